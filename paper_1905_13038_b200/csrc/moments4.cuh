// moments4.cuh -- the warp-CTA moments kernel: K1 (windowed moments) + K2
// (threshold) + K3 (mask store) fused.  Hot path of arXiv 1905.13038
// (reference/PAPER.md): Alg. 1 + Table 1.
//
// Work decomposition
//   One CTA = one warp = one "warp strip": 32 lanes x 16 input columns.  Lane
//   k owns input columns [a, a+16), a = Sw + 16 k, and produces the outputs
//   j = a - r + t (t < 16), so the entering column j + r of the row
//   recursion is its own (shifted ownership).  The first KH = ceil((w+1)/16)
//   lanes are halo: their outputs are not stored.  A CTA runs down a band of
//   B output rows of one page.  Warps never wait for one another: each has
//   its own TMA ring, barriers and shared-memory row.  Strips whose windows
//   reach the left/right image border are launched separately (EDGE = true:
//   per-column counts, masking of the bytes past W); interior strips take the
//   lean path.
//
//  * Rows: the entering row i+u and the leaving row i-o
//    arrive by TMA into a kNS-stage ring re-armed by lane 0 as soon as the
//    warp is done with a stage.  The tensor map views a page as 16-byte
//    chunks x rows, one box = 33 chunks x kR rows (528 contiguous bytes per
//    row); chunks outside the image are zero-filled ("undefined elements are
//    zero") and the bytes of the last partial chunk past W are
//    masked by the lanes that own them.  Box origins are whole chunks, so both
//    rows are staged from Sw - (r mod 16) and realigned by a byte funnel
//    (shared-memory TMA destinations must be 128-byte aligned; probed with
//    tools/tma_probe.cu).  The centre row i (the pixels being decided) is read
//    with one 16-byte global load per lane (it entered the L2 u rows earlier),
//    prefetched one row ahead.
//  * Vertical pass: C_t += x - y, D_t += x^2 - y^2 in
//    registers (uint32, exact: D <= 255^2 h < 2^32).
//  * Horizontal pass: the lane runs the row recursion
//    c_t = c_{t-1} + C[a+t] - C[a+t-w] over its 16 outputs; the leaving
//    column sums C[a+t-w] come from the warp's published row (shared memory,
//    swizzled -> bank-conflict free; columns left of the strip read as zero).
//    The start value c(a - r - 1) = P(a) - P(a - w), P(x) = sum of the strip's
//    column sums left of x, is exact integer arithmetic: P(a) is the warp's
//    exclusive scan of the lanes' column totals, and with a - w =
//    16 (k - m) + RHO (m = ceil(w/16)) P(a - w) = P(a_{k-m}) + the first RHO
//    column sums of lane k - m, fetched with one shuffle.
//  * Epilogue (Alg. 1 l.118-124, Table 1; DESIGN.md section 5 "certified
//    decision"), fused with the recursion pixel pair by pixel pair: stage 1
//    evaluates t~ in fp32 (FFMA2 pairs) from the exact c, d; lanes with a
//    pixel within the certified bound store provisional bits and are queued
//    for k_fixup (fixup.cuh), which recomputes their c, d from the image and
//    decides them exactly: stage 2 in fp32 from the exact V = n d - c^2
//    (bound delta2), stage 3 the canonical IEEE double sequence.  The mask
//    equals the double-precision decision bit for bit; near ties
//    |I - t| < 1e-9 are counted on stage 3.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <type_traits>

#include "moments.cuh"
#include "ptx.cuh"

namespace abin {
namespace v4 {

constexpr int kG = 16;                    // columns per lane
constexpr int kStrip = 32 * kG;           // input columns per warp strip
constexpr int kChunks = 33;               // TMA box: 33 16-byte chunks = 528 bytes per row
constexpr int kSpan = 16 * kChunks;       // staged bytes per row (512 + funnel slack)
constexpr int kR = 3;                     // rows per ring stage (one box per stream; 3 x 2 stages measured best)
constexpr int kNS = 2;                    // ring stages
constexpr int kRowsBytes = (kR * kSpan + 127) / 128 * 128;  // one stream of a stage (128-B aligned)
constexpr int kStageBytes = 2 * kRowsBytes;  // entering + leaving

struct SmemLayout {
  static constexpr int ring = 0;
  static constexpr int pub = kNS * kStageBytes;                 // C[516] then D[516] (4 zero words each)
  static constexpr int nic = pub + 2 * (kStrip + 4) * 4;        // -1/ncol per column (edge strips)
  static constexpr int bar = nic + kStrip * 4;
  static constexpr int total = bar + kNS * 8;
};

constexpr size_t smem_bytes() { return (size_t)SmemLayout::total; }

constexpr int kZero = kStrip;  // word offset of the zero chunk (columns left of the strip)

#ifndef ABIN_V4_MINB
#define ABIN_V4_MINB 16  // resident warp-CTAs per SM the register allocation targets
#endif

// Inclusive warp scan step: v += value of lane - off (if it exists).  The
// shuffle's predicate output says whether the source lane was in range, so
// the add is predicated instead of selected.
__device__ __forceinline__ uint32_t scan_step(uint32_t v, int off) {
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
               "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
               "@p add.u32 %0, %0, t;\n\t}"
               : "+r"(v) : "r"(off));
  return v;
}
__device__ __forceinline__ uint64_t scan_step(uint64_t v, int off) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 tl, th;\n\t"
               "shfl.sync.up.b32 tl|p, %0, %2, 0, 0xffffffff;\n\t"
               "shfl.sync.up.b32 th, %1, %2, 0, 0xffffffff;\n\t"
               "@p add.cc.u32 %0, %0, tl;\n\t"
               "@p addc.u32 %1, %1, th;\n\t}"
               : "+r"(lo), "+r"(hi) : "r"(off));
  return ((uint64_t)hi << 32) | lo;
}

// A warp-uniform value the compiler must keep in a register (a shuffle result
// cannot be re-materialised from the kernel-parameter bank).
__device__ __forceinline__ int64_t opaque(int64_t v) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, 0);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)((uint64_t)v >> 32), 0);
  return (int64_t)(((uint64_t)hi << 32) | lo);
}

// value of lane `src & 31` (no range select)
__device__ __forceinline__ uint32_t shfl_raw(uint32_t v, int src) { return __shfl_sync(0xffffffffu, v, src & 31); }
__device__ __forceinline__ uint64_t shfl_raw(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src & 31);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src & 31);
  return ((uint64_t)hi << 32) | lo;
}

// sum of the values of lanes lane-1 .. lane-M (wrapped; see the start value)
template <int M, typename DT>
__device__ __forceinline__ void lane_sums(uint32_t tc, DT td, int lane, uint32_t& ac, DT& ad) {
#pragma unroll
  for (int q = 1; q <= M; ++q) {
    ac += shfl_raw(tc, lane - q);
    ad += shfl_raw(td, lane - q);
  }
}

// value of lane `src` (0 if src < 0: columns left of the strip are zero)
__device__ __forceinline__ uint32_t shfl_idx(uint32_t v, int src) {
  const uint32_t r = __shfl_sync(0xffffffffu, v, src & 31);
  return src >= 0 ? r : 0u;
}
__device__ __forceinline__ uint64_t shfl_idx(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src & 31);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src & 31);
  return src >= 0 ? (((uint64_t)hi << 32) | lo) : 0ull;
}

template <typename DT>
__device__ __forceinline__ DT shfl_up(DT v, int off) {
  if constexpr (sizeof(DT) == 8) {
    const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, off);
    const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), off);
    return ((uint64_t)hi << 32) | lo;
  } else {
    return __shfl_up_sync(0xffffffffu, v, off);
  }
}

__device__ __forceinline__ float to_f(uint32_t x) { return (float)x; }
__device__ __forceinline__ float to_f(uint64_t x) {  // x < 2^40 here
  return __fmaf_rn((float)(uint32_t)(x >> 32), 4294967296.0f, (float)(uint32_t)x);
}

// Stage-1 residual e = I - t~ of one pixel (the scalar twin of the paired
// evaluation in the row loop; both are the same sequence of correctly
// rounded fp32 operations, so they agree bit for bit).
__device__ __forceinline__ float stage1_e(int method, float cf, float df, float nu, float I, float fa, float fb,
                                          float Lf, float& sv) {
  const float mn = __fmul_rn(cf, nu);
  const float qn = __fmul_rn(df, nu);
  sv = sqrt_approx(fabsf(__fmaf_rn(mn, mn, qn)));
  if (method == M_SAUVOLA) return __fmaf_rn(mn, __fmaf_rn(fb, sv, fa), I);
  if (method == M_NIBLACK) return __fmaf_rn(-fb, sv, __fadd_rn(I, mn));
  return __fmaf_rn(__fmul_rn(-fa, __fadd_rn(mn, Lf)), __fmaf_rn(-fb, sv, 1.0f), __fadd_rn(I, mn));
}

// The stage-1 bound with the data-dependent |s~ - s| (abin_api.cu
// filter_consts): rb0 + rb1 min(sqrt dv, dv / s~).  dv / s~ uses the
// approximate reciprocal (relative error < 2^-22); the 1 + 2^-20 inflation
// keeps the bound an upper bound.
__device__ __forceinline__ float refined_bound(const MomParams& p, float s) {
  float rs;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(s));  // s = 0 -> +inf -> sqrt dv
  return __fmaf_rn(p.rb1, fminf(p.rsdv, p.rdv * rs), p.rb0) * 1.000001f;
}

// Kernel template parameters:
//   W32   w mod 32: fixes the phase PH = (-w) mod 4 of the leaving reads and
//         the byte funnel DL = r mod 16 of the staged rows
//   D64   window square sums d in uint64
//   EDGE  strips whose windows reach the left/right border (per-column counts,
//         bytes past W masked); false: interior strips [sL, sR)
template <int W32, bool D64, int METHOD, bool EDGE>
__device__ __forceinline__ void mom4_body(const CUtensorMap& tin, const MomParams& p, int strip, int band, int page) {
  using DT = typename std::conditional<D64, uint64_t, uint32_t>::type;
  constexpr int W16 = W32 & 15;
  constexpr int PH = (4 - (W16 & 3)) & 3;  // (-w) mod 4
  constexpr int DL = (W32 >> 1) & 15;      // r mod 16
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem + SmemLayout::ring;
  uint32_t* cb = reinterpret_cast<uint32_t*>(smem + SmemLayout::pub);
  uint32_t* db = cb + kStrip + 4;
  float* nicw = reinterpret_cast<float*>(smem + SmemLayout::nic);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SmemLayout::bar);

  const int lane = threadIdx.x;
  const int64_t J0 = (int64_t)strip * p.Tw;               // first output column of the strip
  const int64_t Sw = J0 + p.r - (int64_t)kG * p.KH;       // input column of lane 0
  const int64_t XE = Sw - DL;                             // 16-aligned staging origin
  const int64_t XC = J0 - (int64_t)kG * p.KH;             // = Sw - r, centre-row chunk origin (aligned)
  const int64_t y0 = p.row0 + (int64_t)band * p.B;        // first output row (global)
  const int nrows = (int)min((int64_t)p.B, p.row0 + p.H_out - y0);
  const int WS = (p.h + 2 * kR - 1) / (2 * kR);           // warm-up stages (2 kR rows: both streams' buffers)
  const int total = WS + (nrows + kR - 1) / kR;

  // ---- TMA: one box per stream and stage, chunks [XE/16, XE/16 + 33) x kR rows
  const int32_t xchunk = (int32_t)(XE / 16);
  auto issue = [&](int s) {  // lane 0 only
    const int slot = s % kNS;
    uint8_t* st = ring + slot * kStageBytes;
    const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
    if (s < WS) {  // warm-up rows y0-o+2kR s .. +2kR-1 into both halves of the slot
      const int32_t yw = (int32_t)(y0 - p.o + (int64_t)s * 2 * kR - p.buf_row0);
      mbar_arrive_expect_tx(&full[slot], 2 * kR * kSpan);
      tma_load_4d_hint(st, &tin, 0, xchunk, yw, page, &full[slot], keep);
      tma_load_4d_hint(st + kRowsBytes, &tin, 0, xchunk, yw + kR, page, &full[slot], keep);
    } else {
      const int64_t q0 = (int64_t)(s - WS) * kR;
      mbar_arrive_expect_tx(&full[slot], 2 * kR * kSpan);
      tma_load_4d_hint(st, &tin, 0, xchunk, (int32_t)(y0 + q0 + p.u - p.buf_row0), page, &full[slot], keep);
      tma_load_4d_hint(st + kRowsBytes, &tin, 0, xchunk, (int32_t)(y0 + q0 - p.o - p.buf_row0), page, &full[slot],
                       drop);
    }
  };

  // ---- per-lane geometry
  const int64_t a = Sw + (int64_t)kG * lane;              // first owned input column
  const int64_t j0 = a - p.r;                             // first output column (multiple of 16)
  const int64_t Jend = min(J0 + p.Tw, p.W);
  const bool valid_lane = lane >= p.KH && j0 < Jend;
  const uint32_t vmask = valid_lane ? (Jend - j0 >= kG ? 0xFFFFu : ((1u << (uint32_t)(Jend - j0)) - 1u)) : 0u;
  const int eo = kG * lane;                               // staged offset of the lane's chunk
  // swizzled offsets of the 5 leaving chunks (columns a - w - PH + 4g relative
  // to the strip); chunks left of the strip read the zero chunk
  const int st0 = kG * lane - p.w - PH;
  int lofs[5];
#pragma unroll
  for (int g = 0; g < 5; ++g) {
    const int s = st0 + 4 * g;
    lofs[g] = (s < 0 || s >= kStrip) ? kZero : swz(s);
  }
  const float Lf = (METHOD == M_WOLF) ? (float)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0f;
  const float nic_c = -__frcp_rn((float)p.w);             // interior: ncol = w
  uint32_t km[4] = {~0u, ~0u, ~0u, ~0u};                  // bytes of columns >= W (edge strips)
  if (EDGE) {
#pragma unroll
    for (int t = 0; t < kG; ++t) {
      const int64_t j = j0 + t;
      const int64_t nc = max((int64_t)1, min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));
      nicw[swz(kG * lane + t)] = -__frcp_rn((float)nc);
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t m = 0;
#pragma unroll
      for (int z = 0; z < 4; ++z)
        if (a + 4 * g + z < p.W) m |= 0xFFu << (8 * z);
      km[g] = m;
    }
  }
  auto mask_tail = [&](uint4 x) {
    if (EDGE) { x.x &= km[0]; x.y &= km[1]; x.z &= km[2]; x.w &= km[3]; }
    return x;
  };
  if (lane < 4) { cb[kZero + lane] = 0u; db[kZero + lane] = 0u; }
  if (lane == 0) {
    for (int s = 0; s < kNS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0) {
    fence_proxy_async_smem();
    prefetch_tmap(&tin);
    for (int s = 0; s < kNS && s < total; ++s) issue(s);
  }
  auto stage_end = [&](int s) {
    __syncwarp();
    if (lane == 0 && s + kNS < total) {
      fence_proxy_async_smem();  // generic reads of the slot precede the async-proxy refill
      issue(s + kNS);
    }
  };

  uint32_t C[kG], D[kG];
#pragma unroll
  for (int t = 0; t < kG; ++t) C[t] = D[t] = 0;

  // ---- warm-up: rows y0-o .. y0+u-1
  for (int s = 0; s < WS; ++s) {
    mbar_wait(&full[s % kNS], (s / kNS) & 1);
    const uint8_t* st = ring + (s % kNS) * kStageBytes + eo;
    const int nr = min(2 * kR, p.h - s * 2 * kR);
#pragma unroll 2
    for (int rr = 0; rr < nr; ++rr) {
      const uint8_t* sr = st + (rr < kR ? rr * kSpan : kRowsBytes + (rr - kR) * kSpan);
      const uint4 x = mask_tail(funnel16<DL>(*reinterpret_cast<const uint4*>(sr),
                                             *reinterpret_cast<const uint4*>(sr + 16)));
#pragma unroll
      for (int t = 0; t < kG; ++t) {
        const uint32_t v = byte_of(x, t);
        C[t] += v;
        D[t] += v * v;
      }
    }
    stage_end(s);
  }

  // centre rows: one 16-byte load per lane per row, one row ahead
  const int64_t cx = XC + kG * lane;  // first column of the lane's centre chunk (16-aligned)
  const int cmode = (cx >= 0 && cx + kG <= p.W) ? 1 : ((cx >= 0 && cx < p.W) ? 2 : 0);
  const uint8_t* cptr = p.in + (int64_t)page * p.in_page_stride + (y0 - p.buf_row0) * p.in_pitch + cx;
  auto load_centre = [&](const uint8_t* src, bool ok) -> uint4 {
    if (!ok || cmode == 0) return make_uint4(0, 0, 0, 0);
    if (!EDGE || cmode == 1) return __ldg(reinterpret_cast<const uint4*>(src));
    // columns past W read as 255: their outputs are not stored, but a window
    // wholly outside the image has c = 0 and t~ = 0, and I = 0 there would
    // make the lane ambiguous (queued for the exact fixup) for nothing
    uint32_t wd[4] = {~0u, ~0u, ~0u, ~0u};
    for (int t = 0; t < kG; ++t)
      if (cx + t < p.W) wd[t >> 2] ^= (255u ^ (uint32_t)__ldg(src + t)) << (8 * (t & 3));
    return make_uint4(wd[0], wd[1], wd[2], wd[3]);
  };
  uint4 xc_next = load_centre(cptr, nrows > 0);
  uint8_t* optr = p.out + (int64_t)page * p.out_page_stride + (y0 - p.row0) * p.out_pitch +
                  (p.fmt == 0 ? j0 : (j0 >> 3));
  const bool out_vec = ((reinterpret_cast<uintptr_t>(p.out) | (uintptr_t)p.out_pitch |
                         (uintptr_t)p.out_page_stride) & 15u) == 0 && vmask == 0xFFFFu;
  const float2 fa2 = make_float2(p.fa, p.fa), fb2 = make_float2(p.fb, p.fb);
  constexpr int RHO = (kG - W16) % kG;                        // (-w) mod 16
  const int mW = (p.w + RHO) / kG;                            // ceil(w / 16)
  constexpr int method = METHOD;
  // rows whose window is clipped by the top / bottom image edge: nrow < h
  const int64_t i_full0 = p.o - 1, i_full1 = p.H_global - 1 - p.u;  // nrow == h for i in [i_full0, i_full1]
  // per-row scalars kept in registers: passed through a shuffle, ptxas cannot
  // re-materialise them from the parameter bank every row (which exposed the
  // load latency in the row loop)
  // (not for the uint64 variant: its register budget is tighter and the
  // extra live registers cost more than the re-loads)
  const int64_t in_pitch = D64 ? p.in_pitch : opaque(p.in_pitch);
  const int64_t out_pitch = D64 ? p.out_pitch : opaque(p.out_pitch);
  const float inv_h = D64 ? p.inv_h : __int_as_float((int)opaque((int64_t)__float_as_int(p.inv_h)));
  uint32_t store_mode = !valid_lane ? 0u : (p.fmt != 0 ? 3u : (out_vec ? 1u : 2u));
  int32_t row_lo = (int32_t)max(i_full0, (int64_t)INT32_MIN), row_hi = (int32_t)min(i_full1, (int64_t)INT32_MAX);

  // ---- main rows
  int q = 0;
  for (int s = WS; s < total; ++s) {
    mbar_wait(&full[s % kNS], (s / kNS) & 1);
    const uint8_t* st = ring + (s % kNS) * kStageBytes + eo;
    const int nr = min(kR, nrows - (s - WS) * kR);
#pragma unroll 1
    for (int rr = 0; rr < nr; ++rr, ++q) {
      const int64_t i = y0 + q;  // global output row
      const uint4 xi = mask_tail(funnel16<DL>(*reinterpret_cast<const uint4*>(st + rr * kSpan),
                                              *reinterpret_cast<const uint4*>(st + rr * kSpan + 16)));
      const uint4 xo = mask_tail(funnel16<DL>(*reinterpret_cast<const uint4*>(st + kRowsBytes + rr * kSpan),
                                              *reinterpret_cast<const uint4*>(st + kRowsBytes + rr * kSpan + 16)));
      const uint4 xc = xc_next;
      if (q + 1 < nrows) cptr += in_pitch;  // the last row re-reads itself (harmless)
      xc_next = load_centre(cptr, true);
      // vertical update
#pragma unroll
      for (int t = 0; t < kG; ++t) {
        const uint32_t vi = byte_of(xi, t), vo = byte_of(xo, t);
        C[t] = C[t] + vi - vo;
        D[t] = D[t] + vi * vi - vo * vo;
      }
      // publish the row's column sums (single buffer: the first __syncwarp
      // orders the stores after the previous row's leaving reads)
      __syncwarp();
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        *reinterpret_cast<uint4*>(cb + 128 * g + 4 * lane) = make_uint4(C[4 * g], C[4 * g + 1], C[4 * g + 2], C[4 * g + 3]);
        *reinterpret_cast<uint4*>(db + 128 * g + 4 * lane) = make_uint4(D[4 * g], D[4 * g + 1], D[4 * g + 2], D[4 * g + 3]);
      }
      __syncwarp();
      // ---- start value of the lane's row recursion: the window sum
      // c(a - r - 1) = P(a) - P(a - w), P(x) = sum of the strip's column sums
      // left of column x (zero left of the strip).  P(a) is the exclusive warp
      // scan of the lanes' totals; a - w = 16 (k - m) + RHO, so
      // P(a - w) = P(a_{k-m}) + (first RHO column sums of lane k - m).
      uint32_t Ac;
      DT Ad;
      {
        uint32_t sc = 0, tc;
        DT sd = 0, td;
#pragma unroll
        for (int t = 0; t < RHO; ++t) { sc += C[t]; sd += (DT)D[t]; }
        tc = sc;
        td = sd;
#pragma unroll
        for (int t = RHO; t < kG; ++t) { tc += C[t]; td += (DT)D[t]; }
        if (mW <= 8) {
          // small windows: sum the m lanes' totals directly -- m + 1 independent
          // shuffles instead of a dependent 5-level scan
          // (only the output lanes' start values matter, and for them every
          // source lane k - q >= k - m >= KH - m >= 0: no zero-select needed;
          // the halo lanes read wrapped-around garbage they never use)
          uint32_t ac = 0u - shfl_raw(sc, lane - mW);
          DT ad = (DT)0 - shfl_raw(sd, lane - mW);
          switch (mW) {  // warp-uniform: one branch, then m independent shuffles
            case 1: lane_sums<1>(tc, td, lane, ac, ad); break;
            case 2: lane_sums<2>(tc, td, lane, ac, ad); break;
            case 3: lane_sums<3>(tc, td, lane, ac, ad); break;
            case 4: lane_sums<4>(tc, td, lane, ac, ad); break;
            case 5: lane_sums<5>(tc, td, lane, ac, ad); break;
            case 6: lane_sums<6>(tc, td, lane, ac, ad); break;
            case 7: lane_sums<7>(tc, td, lane, ac, ad); break;
            default: lane_sums<8>(tc, td, lane, ac, ad); break;
          }
          Ac = ac;
          Ad = ad;
        } else {
          uint32_t ic = tc;
          DT id = td;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            ic = scan_step(ic, off);
            id = scan_step(id, off);
          }
          const uint32_t pc = ic - tc;  // P(a_k)
          const DT pd = id - td;
          const uint32_t xc_ = shfl_idx(pc + sc, lane - mW);
          const DT xd_ = shfl_idx(pd + sd, lane - mW);
          Ac = pc - xc_;
          Ad = pd - xd_;
        }
      }
      // ---- epilogue (Alg. 1 l.118-124, Table 1): row recursion
      // c_t = c_{t-1} + C[a+t] - C[a+t-w] fused with stage 1
      // of the certified decision
      uint32_t nrow = (uint32_t)p.h;
      float inv_nrow = inv_h;
      if ((int32_t)i < row_lo || (int32_t)i > row_hi) {
        nrow = (uint32_t)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
        inv_nrow = __frcp_rn((float)nrow);
      }
      const float nu_c = nic_c * inv_nrow;
      uint32_t wv[4];
      float emin = __int_as_float(0x7f800000), smin = emin;
      {
        uint32_t cc = Ac;
        DT dd = Ad;
        uint4 qc = *reinterpret_cast<const uint4*>(cb + lofs[0]), qd = *reinterpret_cast<const uint4*>(db + lofs[0]);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t cl[4], dl[4];
          if (PH == 0) {
            cl[0] = qc.x; cl[1] = qc.y; cl[2] = qc.z; cl[3] = qc.w;
            dl[0] = qd.x; dl[1] = qd.y; dl[2] = qd.z; dl[3] = qd.w;
            if (g < 3) {
              qc = *reinterpret_cast<const uint4*>(cb + lofs[g + 1]);
              qd = *reinterpret_cast<const uint4*>(db + lofs[g + 1]);
            }
          } else {
            const uint4 nc = *reinterpret_cast<const uint4*>(cb + lofs[g + 1]);
            const uint4 nd = *reinterpret_cast<const uint4*>(db + lofs[g + 1]);
            const uint32_t c8[8] = {qc.x, qc.y, qc.z, qc.w, nc.x, nc.y, nc.z, nc.w};
            const uint32_t d8[8] = {qd.x, qd.y, qd.z, qd.w, nd.x, nd.y, nd.z, nd.w};
#pragma unroll
            for (int z = 0; z < 4; ++z) { cl[z] = c8[PH + z]; dl[z] = d8[PH + z]; }
            qc = nc;
            qd = nd;
          }
          float2 nv01 = make_float2(nu_c, nu_c), nv23 = nv01;
          if (EDGE) {
            const float4 n4 = *reinterpret_cast<const float4*>(nicw + 128 * g + 4 * lane);
            nv01 = __fmul2_rn(make_float2(n4.x, n4.y), make_float2(inv_nrow, inv_nrow));
            nv23 = __fmul2_rn(make_float2(n4.z, n4.w), make_float2(inv_nrow, inv_nrow));
          }
          const uint32_t wd = g == 0 ? xc.x : (g == 1 ? xc.y : (g == 2 ? xc.z : xc.w));
          float e4[4];
#pragma unroll
          for (int h2 = 0; h2 < 4; h2 += 2) {
            const int t = 4 * g + h2;
            cc += C[t] - cl[h2];
            dd += (DT)D[t] - (DT)dl[h2];
            const uint32_t c0 = cc;
            const DT d0 = dd;
            cc += C[t + 1] - cl[h2 + 1];
            dd += (DT)D[t + 1] - (DT)dl[h2 + 1];
            const float2 nv = h2 == 0 ? nv01 : nv23;
            const float2 mn = __fmul2_rn(make_float2(to_f(c0), to_f(cc)), nv);  // -m~
            const float2 qn = __fmul2_rn(make_float2(to_f(d0), to_f(dd)), nv);  // -q~
            const float2 vn = __ffma2_rn(mn, mn, qn);                           // -v~
            const float2 sv = make_float2(sqrt_approx(fabsf(vn.x)), sqrt_approx(fabsf(vn.y)));
            // I exactly, off the XU pipe: the byte as the mantissa of 2^23, minus 2^23
            const float2 I = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(wd, 0x4B000000u, 0x7440u | (uint32_t)h2)),
                                                    __uint_as_float(__byte_perm(wd, 0x4B000000u, 0x7440u | (uint32_t)(h2 + 1)))),
                                        make_float2(-8388608.0f, -8388608.0f));
            float2 e;
            if (method == M_SAUVOLA) {
              e = __ffma2_rn(mn, __ffma2_rn(fb2, sv, fa2), I);                                        // I - m g
            } else if (method == M_NIBLACK) {
              e = __ffma2_rn(make_float2(-fb2.x, -fb2.y), sv, __fadd2_rn(I, mn));                      // I - m - k s
            } else {
              const float2 b = __ffma2_rn(make_float2(-fb2.x, -fb2.y), sv, make_float2(1.0f, 1.0f)); // 1 - s/R
              const float2 ka = __fmul2_rn(make_float2(-fa2.x, -fa2.y), __fadd2_rn(mn, make_float2(Lf, Lf)));
              e = __ffma2_rn(ka, b, __fadd2_rn(I, mn));                                              // I - t
            }
            emin = fminf(emin, fminf(fabsf(e.x), fabsf(e.y)));
            if (METHOD == M_NIBLACK) smin = fminf(smin, fminf(sv.x, sv.y));
            e4[h2] = e.x;
            e4[h2 + 1] = e.y;
          }
          // byte t of wv[g] = (e_t >= 0): prmt replicates the selected bytes' sign bits
          const uint32_t lo = prmt_sign(__float_as_uint(e4[0]), __float_as_uint(e4[1]), 0x00FBu);
          const uint32_t hi = prmt_sign(__float_as_uint(e4[2]), __float_as_uint(e4[3]), 0xFB00u);
          wv[g] = ~__byte_perm(lo, hi, 0x7610u) & 0x01010101u;
        }
      }
      // ambiguous lane: some pixel within the certified bound delta1.  For
      // Niblack (t = m + k s: the bound's sqrt(dv) term is large next to the
      // residuals) the lane is re-tested with the data-dependent bound at its
      // smallest s~ (the bound decreases in s~), which keeps the queue ~40x
      // shorter; for Sauvola / Wolf the coarse test alone queues next to
      // nothing, and tracking s~ would cost more than it saves
      uint32_t amb = 0u;
      if (emin < p.delta1) {
        if (METHOD != M_NIBLACK || emin * 0.999999f < refined_bound(p, smin)) amb = vmask;
      }
      // ambiguous lanes (rare) go to the exact fixup kernel (fixup.cuh), which
      // recomputes their pixels' sums and decides them exactly, overwriting
      // the provisional bits stored below; nothing of the exact stages lives
      // in this kernel: its registers go to the hot loop
      if (amb) {
        const uint32_t slot = atomicAdd(p.q_count, 1u);
        if (slot < p.q_cap) p.q_data[slot] = make_uint4((uint32_t)page, (uint32_t)(i - p.row0), (uint32_t)j0, amb);
      }
      // ---- store the mask: outputs j0 .. j0+15 (j0 is a multiple of 16)
      if (store_mode != 0u) {
        if (store_mode != 3u) {
          if (store_mode == 1u) {
            __stcs(reinterpret_cast<uint4*>(optr), make_uint4(wv[0], wv[1], wv[2], wv[3]));  // streaming
          } else {
#pragma unroll
            for (int t = 0; t < kG; ++t)
              if ((vmask >> t) & 1u) optr[t] = (uint8_t)(wv[t >> 2] >> (8 * (t & 3)));
          }
        } else {
          // bytes (0/1) -> bits: nibble of word g = (wv[g] * 0x01020408) >> 24
          uint32_t mbits = 0;
#pragma unroll
          for (int g = 0; g < 4; ++g) mbits |= (((wv[g] * 0x01020408u) >> 24) & 0xFu) << (4 * g);
          const uint32_t mb = __brev(mbits & vmask) >> 16;  // bit 15 - t = mask of output t (MSB-first)
          optr[0] = (uint8_t)(mb >> 8);
          if (vmask >> 8) optr[1] = (uint8_t)(mb & 0xFFu);
        }
      }
      optr += out_pitch;
    }
    stage_end(s);
  }

}

// One launch for all strips: the border strips (slower: per-column counts)
// get the low block indices, so they are scheduled first.
template <int W32, bool D64, int METHOD>
__global__ void __launch_bounds__(32, ABIN_V4_MINB) k_mom4(const __grid_constant__ CUtensorMap tin, const MomParams p) {
  const int nE = p.sL + (p.n_strips - p.sR);
  const int64_t per_strip = (int64_t)p.n_bands * p.n_pages_v4;
  const int64_t te = (int64_t)nE * per_strip;
  int64_t tile = blockIdx.x;
  if (tile < te) {
    const int si = (int)(tile % nE);
    tile /= nE;
    const int strip = si < p.sL ? si : p.sR + (si - p.sL);
    mom4_body<W32, D64, METHOD, true>(tin, p, strip, (int)(tile % p.n_bands), (int)(tile / p.n_bands));
  } else {
    tile -= te;
    const int nI = p.sR - p.sL;
    const int strip = p.sL + (int)(tile % nI);
    tile /= nI;
    mom4_body<W32, D64, METHOD, false>(tin, p, strip, (int)(tile % p.n_bands), (int)(tile / p.n_bands));
  }
}

}  // namespace v4
}  // namespace abin
