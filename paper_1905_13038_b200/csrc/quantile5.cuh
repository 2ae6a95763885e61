// quantile5.cuh -- K5 rebuilt (round 2): the local-quantile mask by sliding
// CDF windows ("local quantiles such as median of gray levels
// can also be computed recursively by maintaining histograms").
//
// The mask needs one comparison, not the quantile itself: with rank
// rho = max(1, ceil(q n)) and Q the rho-th smallest in-bounds value of the
// window (R10),
//     I <= Q   <=>   #(x < I) < rho,
// so a pixel is decided by the window's count of values below its own grey
// level (SURVEY.md 8(c) identity).  This kernel keeps that count -- the
// window CDF -- at 16 consecutive levels L .. L+15 per "window" (NW windows
// per tile, L chosen per tile from a sample of its pixels), exactly:
//   * per column j (vertical recursion, PAPER.md:119-120 in the other
//     direction): C_j[f] = #{rows of the window: x < L + f}, f = 0..15, as 16
//     bytes (counts <= h <= 127), updated per row by the entering and leaving
//     pixels through a 256-entry thermometer table (entry v: bytes [v < L+f]);
//     an absent pixel (outside the image) is staged as 255, whose entry is 0
//     for every window (L <= 240);
//   * per output (horizontal recursion): W_t = W_{t-1} + C_in - C_out, the 16
//     levels as u16 lanes (n <= 127 * 127 < 2^16), the byte difference taken
//     biased (128 + C_in - C_out in [1, 255]: never carries) and widened by
//     two PRMTs.
// For a pixel with f = I - L in [0, 15], #(x < I) = W[f] exactly; below the
// window (f < 0) #(x < I) <= W[0], above it (f > 15) #(x < I) >= W[15], which
// decides the pixel whenever W[0] < rho, resp. W[15] >= rho.  Pixels no window
// decides go to an exact queue (k_q5fix: the direct count over the window),
// so the mask is exact whatever the windows.
//
// Geometry (as moments5.cuh): one warp per CTA, lane k owns the 16 columns
// c0 + 16k .. +15 and produces the outputs whose entering column is its own
// (shifted ownership); lanes k < KH = ceil(w/16) are halo.  A lane's start
// value (the window just left of its first output) is the sum of the totals
// of the mq = floor(w/16) lanes before it plus the last WR = w mod 16 columns
// of lane k - mq - 1 (shuffles); totals persist across rows, updated with the
// same thermometer differences.
#pragma once
#include <cstdint>
#include <cmath>

namespace abin {
namespace q5 {

constexpr int kG = 16;         // columns per lane
constexpr int kMaxW = 127;     // KH <= 8
constexpr int kMaxH = 127;     // byte column counts; |C_in - C_out| <= 127 for the biased difference
constexpr int kMaxNW = 3;
#ifndef ABIN_Q5_MINB
#define ABIN_Q5_MINB 12  // resident warps / SM the registers are sized for (A/B: 14, 16 spill)
#endif
constexpr int kLut = 256;      // thermometer entries (absent pixels staged as 255: entry 0)

struct Q5Params {
  const uint8_t* in;           // first held row (global row buf_row0) of page 0
  int64_t in_page_stride, in_pitch, W;
  int64_t buf_row0, buf_rows;  // held rows
  int64_t row0, H_out, H_global;
  uint8_t* out;
  int64_t out_pitch, out_page_stride;
  int32_t fmt;
  int32_t h, w, l, r, o, u;
  double q;
  int32_t KH, mq, Tw, B, n_bands, n_strips;
  int32_t nw;
  float qf[kMaxNW];            // window placement: quantile fractions of the tile sample
  int32_t force_L;             // test hook (>= 0): window k starts at force_L + 16 k
  int32_t in_vec, out_vec;     // rows 16-byte aligned for vector loads / the mask rows for vector stores
  uint4* fq;                   // exact queue {page, row, column, 0}
  uint32_t* fq_count;
  uint32_t fq_cap;
  unsigned long long* counters;  // optional: counters[1] += pixels decided by the exact count
};

__host__ __device__ constexpr int lut_bytes(int nw) { return nw * kLut * 16; }
__host__ __device__ constexpr int col_bytes(int nw) { return nw * 16 * 32 * 16; }
__host__ __device__ constexpr int stage_bytes() { return 2 * 33 * 16; }  // entering + leaving row (and the tile histogram)
__host__ __device__ constexpr size_t smem_bytes(int nw) {
  return (size_t)lut_bytes(nw) + col_bytes(nw) + stage_bytes();
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint4 lds4(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }
// ordered shared load (volatile: not hoisted across the other volatile shared
// accesses of the recursion, which bounds the registers in flight)
__device__ __forceinline__ uint4 lds4v(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint8_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// x + a - b as one three-input add (kept out of the front end's common
// subexpressions, which would share a - b and cost three adds for two uses)
__device__ __forceinline__ uint32_t add_sub(uint32_t x, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\tadd.u32 t, %1, %2;\n\tsub.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(x), "r"(a), "r"(b));
  return r;
}

// add the biased byte difference d (128 + delta per byte) to u16 lanes: even
// bytes into e, odd bytes into o
__device__ __forceinline__ void widen_add(uint32_t d, uint32_t& e, uint32_t& o) {
  e = e + prmt(d, 0, 0x4240) - 0x00800080u;
  o = o + prmt(d, 0, 0x4341) - 0x00800080u;
}

// Rank rho = max(1, ceil(q n)) in IEEE double (as the oracle and k_quantile).
__device__ __forceinline__ int rank_of(double q, int64_t n) {
  const int r = (int)ceil(__dmul_rn(q, (double)n));
  return r < 1 ? 1 : r;
}

// Byte-wise 16-byte load of columns [c, c + 16) of a row, 255 (absent)
// outside [0, W) (the unaligned / border path of the staged loads; out of line to
// keep the hot loops small)
static __device__ __noinline__ uint4 load16_bytes(const uint8_t* row, int64_t c, int64_t W) {
  uint32_t wv[4] = {~0u, ~0u, ~0u, ~0u};
#pragma unroll
  for (int b = 0; b < 16; ++b)
    if (c + b >= 0 && c + b < W) wv[b >> 2] ^= (uint32_t)(255 ^ __ldg(row + c + b)) << (8 * (b & 3));
  return make_uint4(wv[0], wv[1], wv[2], wv[3]);
}

// The exact decision of one pixel by all 32 lanes: #(x < I) over the window
// counted directly (rows / columns clipped to the image), then
// I' = [#(x < I) >= rho].  Used by the queue kernel and, when the queue is
// full, inline.
static __device__ __noinline__ uint32_t exact_decide(const Q5Params& p, int page, int64_t i, int64_t j) {
  const int lane = threadIdx.x & 31;
  const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;
  const int64_t lo_row = max((int64_t)0, p.buf_row0);
  const int64_t hi_row = min(p.H_global, p.buf_row0 + p.buf_rows);
  const int I = img[(i - p.buf_row0) * p.in_pitch + j];
  const int64_t r0 = max(i - p.o + 1, lo_row), r1 = min(i + p.u, hi_row - 1);
  const int64_t cl = max(j - p.l + 1, (int64_t)0), cr = min(j + p.r, p.W - 1);
  uint32_t cnt = 0;
  if (((reinterpret_cast<uintptr_t>(img) | (uintptr_t)p.in_pitch) & 15u) == 0) {
    // 16-byte chunks: lane = (chunk lane & 7 of the window's columns, row offset lane >> 3);
    // bytes below I by a SIMD compare, bytes outside [cl, cr] masked (rows are 16-aligned and
    // their last partial chunk readable: abin.h)
    const int64_t ca = cl & ~(int64_t)15;
    const int nch = (int)((cr - ca) / 16 + 1);
    const uint32_t Iw = (uint32_t)I * 0x01010101u;
    for (int k = lane & 7; k < nch; k += 8) {
      const int64_t x0 = ca + 16 * k;
      uint32_t vm[4];
#pragma unroll
      for (int wq = 0; wq < 4; ++wq) {
        uint32_t m = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int64_t x = x0 + 4 * wq + b;
          if (x >= cl && x <= cr) m |= 0xFFu << (8 * b);
        }
        vm[wq] = m;
      }
      for (int64_t g = r0 + (lane >> 3); g <= r1; g += 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(img + (g - p.buf_row0) * p.in_pitch + x0));
        cnt += __popc(__vcmpltu4(v.x, Iw) & vm[0]) + __popc(__vcmpltu4(v.y, Iw) & vm[1]) +
               __popc(__vcmpltu4(v.z, Iw) & vm[2]) + __popc(__vcmpltu4(v.w, Iw) & vm[3]);
      }
    }
    cnt >>= 3;  // 8 bits per byte below I
  } else {
    for (int64_t g = r0 + lane; g <= r1; g += 32) {
      const uint8_t* row = img + (g - p.buf_row0) * p.in_pitch;
      for (int64_t c = cl; c <= cr; ++c) cnt += (int)__ldg(row + c) < I ? 1u : 0u;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
  const int64_t nrow = min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1);
  const int64_t ncol = min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1);
  return (int)cnt >= rank_of(p.q, nrow * ncol) ? 1u : 0u;
}

template <int WR, int NW, bool EDGE>
__device__ __forceinline__ void q5_body(const Q5Params& p, uint8_t* sm, int strip, int band, int page) {
  const int lane = threadIdx.x;
  uint8_t* lut = sm;                                  // [NW][257][16]
  uint8_t* colb = lut + lut_bytes(NW);                // [NW][16 slots][32 lanes][16]
  uint8_t* stg = colb + col_bytes(NW);                // [2][33][16]

  const int64_t J0 = (int64_t)strip * p.Tw;            // first output column of the strip
  const int64_t c0 = J0 - 16 * p.KH + p.r;             // lane 0's first column
  const int64_t A = c0 - (((c0 % 16) + 16) % 16);      // 16-aligned staging origin
  const int s = (int)(c0 - A);
  const int64_t y0 = p.row0 + (int64_t)band * p.B;
  const int nrows = (int)min((int64_t)p.B, p.row0 + p.H_out - y0);
  const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;
  const int64_t lo_row = max((int64_t)0, p.buf_row0);
  const int64_t hi_row = min(p.H_global, p.buf_row0 + p.buf_rows);
  const bool out_lane = lane >= p.KH;
  const int64_t jl = J0 + 16 * (lane - p.KH);          // this lane's first output column

  // one 16-byte staged chunk of row g: columns [A + 16 q, +16), zero outside
  // chunk qc of a row given by its pointer (nullptr: absent row)
  auto load_rchunk = [&](const uint8_t* row, int qc) -> uint4 {
    const uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);  // absent: 255
    if (row == nullptr) return v;
    const int64_t cc = A + 16 * qc;
    if (!EDGE) return p.in_vec ? __ldg(reinterpret_cast<const uint4*>(row + cc)) : load16_bytes(row, cc, p.W);
    if (cc + 16 <= 0 || cc >= p.W) return v;
    if (p.in_vec && cc >= 0 && cc + 16 <= p.W) return __ldg(reinterpret_cast<const uint4*>(row + cc));
    return load16_bytes(row, cc, p.W);
  };
  auto row_at = [&](int64_t g) -> const uint8_t* {
    return (g < lo_row || g >= hi_row) ? nullptr : img + (g - p.buf_row0) * p.in_pitch;
  };
  auto load_chunk = [&](int64_t g, int qc) -> uint4 {
    const uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);  // absent: 255
    if (g < lo_row || g >= hi_row) return v;
    const int64_t cc = A + 16 * qc;
    if (EDGE && (cc + 16 <= 0 || cc >= p.W)) return v;
    const uint8_t* row = img + (g - p.buf_row0) * p.in_pitch;
    if (p.in_vec && (!EDGE || (cc >= 0 && cc + 16 <= p.W))) return __ldg(reinterpret_cast<const uint4*>(row + cc));
    return load16_bytes(row, cc, p.W);
  };
  // this lane's 16 output pixels of row g (aligned chunk jl)
  auto load_centre = [&](int64_t g) -> uint4 {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (!out_lane || g < lo_row || g >= hi_row) return v;
    const uint8_t* row = img + (g - p.buf_row0) * p.in_pitch;
    if (p.in_vec && (!EDGE || (jl >= 0 && jl + 16 <= p.W))) return __ldg(reinterpret_cast<const uint4*>(row + jl));
    return load16_bytes(row, jl, p.W);
  };
  // own 16 bytes of a staged row: words at byte offset 16 lane + s
  auto own16 = [&](const uint8_t* st, uint32_t (&o)[4]) {
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(st) + 4 * lane + (s >> 2);
    const uint32_t x0 = w32[0], x1 = w32[1], x2 = w32[2], x3 = w32[3], x4 = w32[4];
    const uint32_t sh = 8u * (uint32_t)(s & 3);
    o[0] = __funnelshift_r(x0, x1, sh);
    o[1] = __funnelshift_r(x1, x2, sh);
    o[2] = __funnelshift_r(x2, x3, sh);
    o[3] = __funnelshift_r(x3, x4, sh);
  };

  // ---- window placement: quantiles of a sample of the tile's rows ----
  int L[NW];
  {
    uint32_t* hist = reinterpret_cast<uint32_t*>(stg);
#pragma unroll
    for (int b = 0; b < 8; ++b) hist[lane + 32 * b] = 0u;
    __syncwarp();
    const int64_t g0 = y0 - p.o, span = (int64_t)nrows + p.h;
    const int64_t step = max((int64_t)1, span / 16);
    for (int64_t g = g0; g < g0 + span; g += step) {
      if (g < lo_row || g >= hi_row) continue;
      const uint4 v = load_chunk(g, lane);
      const int64_t cc = A + 16 * lane;
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if (!EDGE || (cc + b >= 0 && cc + b < p.W)) atomicAdd(&hist[(wv[b >> 2] >> (8 * (b & 3))) & 255u], 1u);
    }
    __syncwarp();
    uint32_t c8[8], sum = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) { c8[b] = hist[8 * lane + b]; sum += c8[b]; }
    uint32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += x;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t base = incl - sum;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const uint32_t target = max(1u, (uint32_t)ceilf(p.qf[k] * (float)total));
      int g = 255;
      if (target > base && target <= incl) {
        uint32_t cum = base;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          cum += c8[b];
          if (cum >= target) { g = 8 * lane + b; break; }
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, target > base && target <= incl);
      const int Qk = who ? __shfl_sync(0xffffffffu, g, __ffs(who) - 1) : 128;
      L[k] = min(max(Qk - 7, 0), 240);
    }
    // distinct, non-overlapping windows (sorted, pushed apart, kept in [0, 240])
#pragma unroll
    for (int a = 0; a < NW; ++a)
#pragma unroll
      for (int b = a + 1; b < NW; ++b)
        if (L[b] < L[a]) { const int t = L[a]; L[a] = L[b]; L[b] = t; }
#pragma unroll
    for (int k = 1; k < NW; ++k) L[k] = max(L[k], L[k - 1] + 16);
#pragma unroll
    for (int k = NW - 1; k >= 0; --k) {
      const int cap = 240 - 16 * (NW - 1 - k);
      if (L[k] > cap) L[k] = cap;
      if (k + 1 < NW && L[k] > L[k + 1] - 16) L[k] = L[k + 1] - 16;
    }
    if (p.force_L >= 0) {
#pragma unroll
      for (int k = 0; k < NW; ++k) L[k] = min(p.force_L + 16 * k, 240);
    }
    __syncwarp();
  }
  // thermometer tables: entry v, byte f = [v < L + f] (entry 255 = 0: L <= 240)
#pragma unroll
  for (int k = 0; k < NW; ++k)
    for (int v = lane; v < kLut; v += 32) {
      uint32_t wv[4];
      const int e = min(max(v - L[k] + 1, 0), 16);  // bytes f >= e are set
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int z = min(max(e - 4 * i, 0), 4);
        wv[i] = z >= 4 ? 0u : (0x01010101u << (8 * z));
      }
      sts4(lut + k * kLut * 16 + v * 16, make_uint4(wv[0], wv[1], wv[2], wv[3]));
    }
  // column slots and lane totals start empty
#pragma unroll
  for (int k = 0; k < NW; ++k)
#pragma unroll
    for (int m = 0; m < 16; ++m) sts4(colb + k * (16 * 512) + m * 512 + lane * 16, make_uint4(0u, 0u, 0u, 0u));
  uint32_t Te[NW][4], To[NW][4], Pe[NW][4], Po[NW][4];
#pragma unroll
  for (int k = 0; k < NW; ++k)
#pragma unroll
    for (int i = 0; i < 4; ++i) { Te[k][i] = To[k][i] = Pe[k][i] = Po[k][i] = 0u; }
  __syncwarp();

  // ---- per row: the vertical update of the own columns (and the totals) ----
  // a / b: own bytes of the entering / leaving row (absent pixels: 255)
  auto update = [&](const uint32_t (&a)[4], const uint32_t (&b)[4]) {
    uint32_t dT[NW][4], dP[NW][4];
#pragma unroll
    for (int k = 0; k < NW; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) dT[k][i] = dP[k][i] = 0x80808080u;
    // columns m = 4 wq + bq: the word loop stays rolled (code size: the hot
    // loops fit the instruction caches), the byte loop is unrolled; the
    // partial P starts at column 16 - WR = 4 wsnap + bsnap
    constexpr int wsnap = (16 - WR) >> 2, bsnap = (16 - WR) & 3;
#pragma unroll 1
    for (int wq = 0; wq < 4; ++wq) {
      const uint32_t aw = wq == 0 ? a[0] : wq == 1 ? a[1] : wq == 2 ? a[2] : a[3];
      const uint32_t bw = wq == 0 ? b[0] : wq == 1 ? b[1] : wq == 2 ? b[2] : b[3];
#pragma unroll
      for (int bq = 0; bq < 4; ++bq) {
        if (WR > 0 && bq == bsnap && wq == wsnap) {
#pragma unroll
          for (int k = 0; k < NW; ++k)
#pragma unroll
            for (int i = 0; i < 4; ++i) dP[k][i] = dT[k][i];
        }
        const uint32_t va = (aw >> (8 * bq)) & 255u;
        const uint32_t vb = (bw >> (8 * bq)) & 255u;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          const uint8_t* lk = lut + k * kLut * 16;
          const uint4 la = lds4(lk + va * 16), lb = lds4(lk + vb * 16);
          uint8_t* cp = colb + k * (16 * 512) + (4 * wq + bq) * 512 + lane * 16;
          uint4 c = lds4(cp);
          c.x = add_sub(c.x, la.x, lb.x);
          c.y = add_sub(c.y, la.y, lb.y);
          c.z = add_sub(c.z, la.z, lb.z);
          c.w = add_sub(c.w, la.w, lb.w);
          sts4(cp, c);
          dT[k][0] = add_sub(dT[k][0], la.x, lb.x);
          dT[k][1] = add_sub(dT[k][1], la.y, lb.y);
          dT[k][2] = add_sub(dT[k][2], la.z, lb.z);
          dT[k][3] = add_sub(dT[k][3], la.w, lb.w);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NW; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        widen_add(dT[k][i], Te[k][i], To[k][i]);
        if (WR > 0) widen_add(dT[k][i] - dP[k][i] + 0x80808080u, Pe[k][i], Po[k][i]);
      }
  };

  // ---- warm-up: rows y0 - o .. y0 + u - 1 (the window of row y0 - 1) ----
  // column adds only (no leaving pixels, no staging: the lane's own 16 bytes
  // are the funnel of its chunks k, k + 1); the totals follow from the columns
  {
    const uint32_t sh = 8u * (uint32_t)(s & 3);
    uint4 x0 = load_chunk(y0 - p.o, lane), x1 = load_chunk(y0 - p.o, lane + 1);
    for (int64_t g = y0 - p.o; g <= y0 + p.u - 1; ++g) {
      const uint4 c0w = x0, c1w = x1;
      if (g + 1 <= y0 + p.u - 1) {
        x0 = load_chunk(g + 1, lane);
        x1 = load_chunk(g + 1, lane + 1);
      }
      if (g < lo_row || g >= hi_row) continue;
      // bytes s .. s + 15 of the 32 staged bytes c0w : c1w
      const uint32_t wv[8] = {c0w.x, c0w.y, c0w.z, c0w.w, c1w.x, c1w.y, c1w.z, c1w.w};
      uint32_t a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // word (s >> 2) + i and its successor (runtime s: select among the 8)
        uint32_t lo = wv[i], hi = wv[i + 1];
#pragma unroll
        for (int z = 1; z < 4; ++z)
          if ((s >> 2) == z) { lo = wv[i + z]; hi = wv[i + z + 1]; }
        a[i] = __funnelshift_r(lo, hi, sh);
      }
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const uint32_t va = (a[m >> 2] >> (8 * (m & 3))) & 255u;  // absent: 255 (adds nothing)
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          const uint4 la = lds4(lut + k * kLut * 16 + va * 16);
          uint8_t* cp = colb + k * (16 * 512) + m * 512 + lane * 16;
          uint4 c = lds4(cp);
          c.x += la.x;
          c.y += la.y;
          c.z += la.z;
          c.w += la.w;
          sts4(cp, c);
        }
      }
    }
    // lane totals T (all 16 columns) and partials P (the last WR columns)
#pragma unroll
    for (int k = 0; k < NW; ++k)
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const uint4 c = lds4(colb + k * (16 * 512) + m * 512 + lane * 16);
        const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t e = prmt(cw[i], 0, 0x4240), o = prmt(cw[i], 0, 0x4341);
          Te[k][i] += e;
          To[k][i] += o;
          if (m >= 16 - WR) {
            Pe[k][i] += e;
            Po[k][i] += o;
          }
        }
      }
    __syncwarp();
  }

  // ---- output rows ----
  const uint32_t colb_a = static_cast<uint32_t>(__cvta_generic_to_shared(colb));
  const int lo_a = ((lane - p.mq - 1) & 31) * 16, lo_b = ((lane - p.mq) & 31) * 16;  // leaving lanes
  uint8_t* obase = p.out + (int64_t)page * p.out_page_stride;
  uint4 nin, nout, nin32, nout32, nctr;
  if (nrows > 0) {
    const uint8_t* ri = row_at(y0 + p.u);
    const uint8_t* ro = row_at(y0 - p.o);
    nin = load_rchunk(ri, lane);
    nout = load_rchunk(ro, lane);
    nin32 = lane == 0 ? load_rchunk(ri, 32) : make_uint4(0u, 0u, 0u, 0u);
    nout32 = lane == 0 ? load_rchunk(ro, 32) : make_uint4(0u, 0u, 0u, 0u);
    nctr = load_centre(y0);
  }
  for (int qq = 0; qq < nrows; ++qq) {
    const int64_t i = y0 + qq;
    sts4(stg + lane * 16, nin);
    sts4(stg + 33 * 16 + lane * 16, nout);
    if (lane == 0) {
      sts4(stg + 32 * 16, nin32);
      sts4(stg + 33 * 16 + 32 * 16, nout32);
    }
    const uint4 ctr = nctr;
    __syncwarp();
    if (qq + 1 < nrows) {
      const uint8_t* ri = row_at(i + 1 + p.u);
      const uint8_t* ro = row_at(i + 1 - p.o);
      nin = load_rchunk(ri, lane);
      nout = load_rchunk(ro, lane);
      if (lane == 0) {
        nin32 = load_rchunk(ri, 32);
        nout32 = load_rchunk(ro, 32);
      }
      nctr = load_centre(i + 1);
    }
    {
      uint32_t a[4], b[4];
      own16(stg, a);
      own16(stg + 33 * 16, b);
      update(a, b);
    }
    __syncwarp();

    // start values S = sum of the mq previous lanes' totals (+ partial), as
    // V = S + K: with K = 0x8000 - rho per u16 lane, bit 15 of a lane is
    // [W >= rho] (W <= 127 * 127, so V stays inside the lane)
    const int64_t nrow = min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1);
    const int rho_row = rank_of(p.q, (int64_t)p.w * nrow);
    const uint32_t K2 = (uint32_t)(0x8000 - rho_row) * 0x10001u;
    uint32_t We[NW][4], Wo[NW][4];
#pragma unroll
    for (int k = 0; k < NW; ++k)
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {
        uint32_t se = K2, so = K2;
        if (WR > 0) {
          se += __shfl_up_sync(0xffffffffu, Pe[k][i2], p.mq + 1);
          so += __shfl_up_sync(0xffffffffu, Po[k][i2], p.mq + 1);
        }
        switch (p.mq) {  // falls through: lanes k - mq .. k - 1
          case 7: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 7); so += __shfl_up_sync(0xffffffffu, To[k][i2], 7);
          case 6: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 6); so += __shfl_up_sync(0xffffffffu, To[k][i2], 6);
          case 5: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 5); so += __shfl_up_sync(0xffffffffu, To[k][i2], 5);
          case 4: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 4); so += __shfl_up_sync(0xffffffffu, To[k][i2], 4);
          case 3: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 3); so += __shfl_up_sync(0xffffffffu, To[k][i2], 3);
          case 2: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 2); so += __shfl_up_sync(0xffffffffu, To[k][i2], 2);
          case 1: se += __shfl_up_sync(0xffffffffu, Te[k][i2], 1); so += __shfl_up_sync(0xffffffffu, To[k][i2], 1);
          default: break;
        }
        We[k][i2] = se;
        Wo[k][i2] = so;
      }
    uint32_t mbits = 0, ubits = 0;
#pragma unroll 1
    for (int tq = 0; tq < 4; ++tq) {
    const uint32_t cwq = tq == 0 ? ctr.x : tq == 1 ? ctr.y : tq == 2 ? ctr.z : ctr.w;
#pragma unroll
    for (int tb = 0; tb < 4; ++tb) {
      const int t = 4 * tq + tb;
      const int slot_out = (t - WR) & 15;
      const int lo = t < WR ? lo_a : lo_b;
      const int It = (int)((cwq >> (8 * tb)) & 255u);
      uint32_t dK = 0u;  // border columns: their own rank (n = ncol nrow < w nrow)
      if (EDGE) {
        const int64_t j = jl + t;
        const int64_t ncol = min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1);
        dK = (uint32_t)(rho_row - rank_of(p.q, ncol * nrow)) * 0x10001u;
      }
      bool mk = false, unk = true;
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const uint32_t cbk = colb_a + k * (16 * 512);
        const uint4 cin = lds4v(cbk + t * 512 + lane * 16);
        const uint4 cout = lds4v(cbk + slot_out * 512 + lo);
        widen_add(cin.x + 0x80808080u - cout.x, We[k][0], Wo[k][0]);
        widen_add(cin.y + 0x80808080u - cout.y, We[k][1], Wo[k][1]);
        widen_add(cin.z + 0x80808080u - cout.z, We[k][2], Wo[k][2]);
        widen_add(cin.w + 0x80808080u - cout.w, We[k][3], Wo[k][3]);
        // the 16 flags [W[f] >= rho] (bit 15 of each lane; level 4i+b of word
        // pair i lands in bit 7 of byte b of g_i), counted: W is
        // non-decreasing in f, so [W[f] >= rho] = [f >= 16 - fge]
        uint32_t g[4];
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2)
          g[i2] = EDGE ? prmt(We[k][i2] + dK, Wo[k][i2] + dK, 0x7351) : prmt(We[k][i2], Wo[k][i2], 0x7351);
        uint32_t a, b, c;
        asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(a) : "r"(g[0]), "r"(g[1] >> 1), "n"(0x80808080));
        asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(b) : "r"(g[2] >> 2), "r"(g[3] >> 3), "n"(0x20202020));
        asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(c) : "r"(a), "r"(b), "n"(0xC0C0C0C0));
        const int fge = __popc(c & 0xF0F0F0F0u);
        // I' = [I - L >= 16 - fge]; undecided: below the window with every
        // level >= rho, or above it with none
        const int f = It - L[k];
        const bool u_k = (unsigned)f > 15u && fge == (f < 0 ? 16 : 0);
        const bool m_k = f + fge >= 16;
        if (NW == 1) {
          mk = m_k;
          unk = u_k;
        } else {
          mk = mk || (!u_k && m_k);
          unk = unk && u_k;
        }
      }
      if (mk) mbits |= 1u << t;
      if (unk) ubits |= 1u << t;
    }
    }
    // outputs of this lane: columns jl .. jl + 15 (inside the image)
    uint32_t vmask = out_lane ? 0xFFFFu : 0u;
    if (EDGE && out_lane) {
      vmask = 0;
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (jl + t >= 0 && jl + t < p.W) vmask |= 1u << t;
    }
    ubits &= vmask;
    mbits &= vmask & ~ubits;  // undecided pixels: 0 until the exact decision
    if (__any_sync(0xffffffffu, ubits != 0u)) {
      // undecided pixels: exact queue (warp-aggregated slots)
      const uint32_t cnt = __popc(ubits);
      uint32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += x;
      }
      uint32_t base = 0;
      if (lane == 31) base = atomicAdd(p.fq_count, incl);
      base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
      uint32_t ub = ubits, over = 0;
      while (ub) {
        const int t = __ffs(ub) - 1;
        ub &= ub - 1;
        if (base < p.fq_cap) p.fq[base] = make_uint4((uint32_t)page, (uint32_t)i, (uint32_t)(jl + t), 0u);
        else over |= 1u << t;
        ++base;
      }
      if (p.counters && lane == 31) atomicAdd(p.counters + 1, (unsigned long long)incl);
      // a full queue: the warp decides the rest here, one pixel at a time
      for (unsigned who = __ballot_sync(0xffffffffu, over != 0); who; who = __ballot_sync(0xffffffffu, over != 0)) {
        const int src = __ffs(who) - 1;
        const uint32_t mo = __shfl_sync(0xffffffffu, over, src);
        const int t = __ffs(mo) - 1;
        const int64_t jj = __shfl_sync(0xffffffffu, jl, src) + t;
        const uint32_t mk = exact_decide(p, page, i, jj);
        if (lane == src) {
          mbits |= mk << t;
          over &= ~(1u << t);
        }
      }
    }
    if (out_lane) {
      uint8_t* orow = obase + (i - p.row0) * p.out_pitch;
      if (p.fmt == 0) {
        uint32_t wv[4];
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) wv[w4] = ((((mbits >> (4 * w4)) & 15u) * 0x00204081u) & 0x01010101u);
        if (p.out_vec && (!EDGE || vmask == 0xFFFFu)) {
          *reinterpret_cast<uint4*>(orow + jl) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if ((vmask >> t) & 1u) orow[jl + t] = (uint8_t)((mbits >> t) & 1u);
        }
      } else {
        // MSB-first bits: byte 0 = columns jl .. jl + 7 (jl is a multiple of 16)
        const uint32_t rv = __brev(mbits) >> 16;  // column jl at bit 15
        const uint32_t b0 = rv >> 8, b1 = rv & 255u;
        const int64_t ob = jl >> 3;
        if (p.out_vec && (!EDGE || vmask == 0xFFFFu)) {
          *reinterpret_cast<uint16_t*>(orow + ob) = (uint16_t)(b0 | (b1 << 8));
        } else {
          if (vmask & 0x00FFu) orow[ob] = (uint8_t)b0;
          if (vmask & 0xFF00u) orow[ob + 1] = (uint8_t)b1;
        }
      }
    }
  }
}

template <int WR, int NW>
__global__ void __launch_bounds__(32, ABIN_Q5_MINB) k_quant5(const __grid_constant__ Q5Params p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k_q5fix (PDL) may be scheduled
  extern __shared__ __align__(16) uint8_t q5sm[];
  int64_t tile = blockIdx.x;
  const int strip = (int)(tile % p.n_strips);
  tile /= p.n_strips;
  const int band = (int)(tile % p.n_bands);
  const int page = (int)(tile / p.n_bands);
  const int64_t J0 = (int64_t)strip * p.Tw;
  const int64_t c0 = J0 - 16 * p.KH + p.r;
  const int64_t A = c0 - (((c0 % 16) + 16) % 16);
  const bool interior = A >= 0 && A + 33 * 16 <= p.W && J0 + p.Tw <= p.W;
  if (interior) q5_body<WR, NW, false>(p, q5sm, strip, band, page);
  else q5_body<WR, NW, true>(p, q5sm, strip, band, page);
}

// The exact queue: one warp per undecided pixel (exact_decide).
static __global__ void __launch_bounds__(256) k_q5fix(const __grid_constant__ Q5Params p) {
  const int lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: k_quant5's queue and mask
  const uint32_t n_e = min(*p.fq_count, p.fq_cap);
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_e; e += (gridDim.x * blockDim.x) >> 5) {
    const uint4 q = p.fq[e];
    const int page = (int)q.x;
    const int64_t i = (int64_t)q.y, j = (int64_t)q.z;
    const uint32_t mk = exact_decide(p, page, i, j);
    if (lane == 0) {
      uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (i - p.row0) * p.out_pitch;
      if (p.fmt == 0) {
        orow[j] = (uint8_t)mk;
      } else {
        // MSB-first bit j, patched with a 32-bit atomic on the aligned word
        // holding its byte (as fixup.cuh)
        const uintptr_t addr = reinterpret_cast<uintptr_t>(orow + (j >> 3));
        unsigned int* word = reinterpret_cast<unsigned int*>(addr & ~(uintptr_t)3);
        const unsigned int bit = 1u << (8 * (unsigned)(addr & 3) + (7 - (unsigned)(j & 7)));
        if (mk) atomicOr(word, bit);
        else atomicAnd(word, ~bit);
      }
    }
  }
}

}  // namespace q5
}  // namespace abin
