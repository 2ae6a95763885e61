// moments_wide.cuh -- the CTA-strip variant of the moments kernel for wide
// windows (effective w > 495, where a 512-column warp strip has no room):
// one CTA-wide strip, a __syncthreads per row, canonical fp64 epilogue.
// K1 (windowed moments) + K2 (threshold) + K3 (mask store) fused.  Hot path of arXiv 1905.13038.
//
// Tile = (page, row band of B output rows, column strip of T output cols).
// A CTA of NT threads owns NT*G consecutive input columns of its strip;
// thread k owns input columns [a, a+G), a = S + G k.
//
//  * Vertical pass ("C_j <- C_j + I_{i+u,j} - I_{i-o,j}"):
//    per-column sums C_j, D_j live in registers and run down the rows of the
//    band.  Input rows arrive by TMA (cp.async.bulk.tensor, OOB -> 0, which is
//    exactly the paper's "undefined elements are zero") into a
//    3-stage shared-memory ring: the entering row i+u, the leaving row i-o
//    and the centre row i for every output row.
//  * Horizontal pass ("c <- c + C_{j+r} - C_{j-l}"):
//    shifted ownership -- thread k produces outputs j = a - r + t, so the
//    entering column j + r = a + t is its own; the leaving column a - w + t is
//    read from the row of C, D the CTA publishes to shared memory; the start
//    value c(a - r - 1) = sum_{b=a-w}^{a-1} C_b comes from a CTA-wide scan.
//    Integer sums are exact (mod 2^32 arithmetic is exact when the true sum
//    fits; D64 keeps window d in uint64).
//  * Epilogue (Alg. 1 l.118-124 + Table 1): n, then either the exact fp64
//    sequence for every pixel, or the certified fp32 filter with the exact
//    fp64 sequence for the few pixels it cannot decide (K2).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <type_traits>

#include "ptx.cuh"
#include "rules.cuh"

namespace abin {
namespace wide {

enum { M_SAUVOLA = 0, M_NIBLACK = 1, M_WOLF = 2 };

struct MomParams {
  int64_t W;          // image width
  int64_t H_out;      // output rows of this call (band rows, or H)
  int64_t row0;       // global row of the first output row
  int64_t H_global;   // image height for n / edges
  int64_t buf_row0;   // global row held at tensor-map row 0
  uint8_t* out;       // mask of global row row0, page 0
  int64_t out_pitch;
  int64_t out_page_stride;
  int32_t h, w, l, r, o, u;  // effective (clamped) window
  int32_t fmt;               // 0 u8, 1 bits
  int32_t T;                 // output cols per strip (multiple of G)
  int32_t n_strips;
  int32_t B;                 // output rows per band
  int32_t n_bands;
  int32_t KH;                // halo threads per strip
  int32_t method;
  int32_t force_fp64;
  int32_t out_vec_ok;        // 8-byte aligned mask rows
  double k, R;
  const uint8_t* L_page;     // per-page global minimum (Wolf), device
  int32_t L_fixed;           // >= 0: use this L
  // fp32 filter constants
  float f_inv_n_dummy;
  uint64_t* counters;        // [near_tie, fallback] or null
  // statistics mode (page 0 only)
  uint64_t* c_out;
  uint64_t* d_out;
  uint32_t* n_out;
  double* t_out;
  uint8_t* mask_out;
  // generic loader (used when the image is not 16-byte aligned for TMA)
  int32_t use_tma;
  const uint8_t* in;
  int64_t in_pitch, in_page_stride, buf_rows;
  RuleParams rp;  // Table 1 rules Feng / Rais / Khurshid / Phansalkar (rules.cuh)
};

// ------------------------------------------------------------------ epilogue
// The canonical sequence: Alg. 1 l.121-122 then the Table-1 row written left
// to right, each operation explicitly rounded (no FMA contraction), so the
// result is the plain IEEE-double evaluation of the paper's formula.
__device__ __forceinline__ double threshold_fp64(int method, uint64_t c, uint64_t d, uint32_t n, double k,
                                                 double R, double L) {
  const double nd = (double)n;
  const double m = __ddiv_rn((double)c, nd);
  double v = __dsub_rn(__ddiv_rn((double)d, nd), __dmul_rn(m, m));
  if (v < 0.0) v = 0.0;
  const double s = __dsqrt_rn(v);
  if (method == M_SAUVOLA) return __dmul_rn(m, __dadd_rn(1.0, __dmul_rn(k, __dsub_rn(__ddiv_rn(s, R), 1.0))));
  if (method == M_NIBLACK) return __dadd_rn(m, __dmul_rn(k, s));
  // Wolf: m - ((k (m - L)) (1 - s/R))
  return __dsub_rn(m, __dmul_rn(__dmul_rn(k, __dsub_rn(m, L)), __dsub_rn(1.0, __ddiv_rn(s, R))));
}

// 8 bytes starting `dl` bytes into the 16-byte pair (a, b): fhi selects the
// 4-byte step, sh (0, 8, 16, 24) the byte step.
__device__ __forceinline__ uint2 funnel8(uint2 a, uint2 b, uint32_t sh, bool fhi) {
  const uint32_t w0 = fhi ? a.y : a.x, w1 = fhi ? b.x : a.y, w2 = fhi ? b.y : b.x;
  return make_uint2(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh));
}

template <int G>
struct Bytes;
template <>
struct Bytes<8> {
  uint2 v;
  __device__ __forceinline__ uint32_t at(int t) const { return ((t < 4 ? v.x : v.y) >> (8 * (t & 3))) & 0xFFu; }
};

// Kernel template parameters:
//   NT   threads per CTA (strip input width NT*G bytes)
//   G    columns per thread (8)
//   PH   (-w) mod 4: alignment phase of the leaving-column reads
//   R_   rows per TMA stage
//   D64  window square sums in uint64
//   STATS write per-pixel c, d, n, t, mask (page 0)
template <int NT, int G, int PH, int R_, bool D64, bool STATS>
__global__ void __launch_bounds__(NT) k_moments(const __grid_constant__ CUtensorMap tin, const MomParams p) {
  constexpr int NW = NT / 32;
  constexpr int STRIP = NT * G;        // input bytes per row per stream
  constexpr int NBOX = STRIP / 256;    // TMA boxes (256 x R_) per row chunk
  constexpr int STREAM_BYTES = R_ * STRIP;
  constexpr int STAGE_BYTES = 3 * STREAM_BYTES;
  constexpr int NS = 3;                // ring depth
  using DT = typename std::conditional<D64, uint64_t, uint32_t>::type;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;                                                   // NS * STAGE_BYTES
  uint32_t* Cb = reinterpret_cast<uint32_t*>(smem + NS * STAGE_BYTES);   // [2][STRIP]
  uint32_t* Db = Cb + 2 * STRIP;                                          // [2][STRIP]
  uint32_t* Qc = Db + 2 * STRIP;                                          // [2][NT]
  DT* Qd = reinterpret_cast<DT*>(Qc + 2 * NT);                            // [2][NT]
  uint32_t* Wc = reinterpret_cast<uint32_t*>(Qd + 2 * NT);                // [2][NW]
  DT* Wd = reinterpret_cast<DT*>(Wc + 2 * NW);                             // [2][NW]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(Wd + 2 * NW);          // [NS] mbarriers

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- tile coordinates
  int64_t tile = blockIdx.x;
  const int strip = (int)(tile % p.n_strips);
  tile /= p.n_strips;
  const int band = (int)(tile % p.n_bands);
  const int page = (int)(tile / p.n_bands);
  const int64_t J0 = (int64_t)strip * p.T;                 // first output column of the strip
  const int64_t S = J0 + p.r - (int64_t)G * p.KH;          // input column of thread 0
  // TMA box starts must be 16-byte aligned: the entering/leaving rows are
  // staged from XE = S - dl (dl = S mod 16, the same for every CTA) and read
  // back with a byte funnel; the centre row starts at XC = S - r = J0 - G KH,
  // a multiple of 16 (J0 and G KH are).
  const int dl = (int)(((S % 16) + 16) % 16);
  const int64_t XE = S - dl;
  const int64_t XC = S - p.r;
  const int64_t y0 = p.row0 + (int64_t)band * p.B;         // first output row (global)
  const int64_t nrows = min((int64_t)p.B, p.row0 + p.H_out - y0);
  const int WS = (p.h + R_ - 1) / R_;                      // warm-up stages
  const int MS = (int)((nrows + R_ - 1) / R_);             // main stages
  const int total = WS + MS;

  if (tid == 0) {
    if (smem_u32(smem) & 127u) __trap();  // TMA destinations must be 128-byte aligned
    prefetch_tmap(&tin);
    for (int s = 0; s < NS; ++s) mbar_init(&full_bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // TMA boxes whose column range misses [0, W) entirely are not issued (the
  // hardware rejects them); their shared-memory bytes are zeroed once, since a
  // CTA's column range never changes.  Rows out of range are zero-filled by TMA.
  auto box_ok = [&](int64_t x) { return x + 256 > 0 && x < p.W; };
  int nbox_el = 0, nbox_c = 0;
#pragma unroll
  for (int b = 0; b < NBOX; ++b) {
    nbox_el += box_ok(XE + 256 * b);
    nbox_c += box_ok(XC + 256 * b);
  }
  auto issue = [&](int s) {
    const int slot = s % NS;
    uint8_t* st = ring + slot * STAGE_BYTES;
    if (s < WS) {
      const int64_t yr = y0 - p.o + (int64_t)s * R_ - p.buf_row0;
      mbar_arrive_expect_tx(&full_bar[slot], nbox_el * R_ * 256);
#pragma unroll
      for (int b = 0; b < NBOX; ++b)
        if (box_ok(XE + 256 * b))
          tma_load_3d(st + b * R_ * 256, &tin, (int32_t)(XE + 256 * b), (int32_t)yr, page, &full_bar[slot]);
    } else {
      const int64_t q0 = (int64_t)(s - WS) * R_;
      const int64_t ye = y0 + q0 + p.u - p.buf_row0;
      const int64_t yc = y0 + q0 - p.buf_row0;
      const int64_t yl = y0 + q0 - p.o - p.buf_row0;
      mbar_arrive_expect_tx(&full_bar[slot], (2 * nbox_el + nbox_c) * R_ * 256);
#pragma unroll
      for (int b = 0; b < NBOX; ++b) {
        if (box_ok(XE + 256 * b)) {
          tma_load_3d(st + b * R_ * 256, &tin, (int32_t)(XE + 256 * b), (int32_t)ye, page, &full_bar[slot]);
          tma_load_3d(st + 2 * STREAM_BYTES + b * R_ * 256, &tin, (int32_t)(XE + 256 * b), (int32_t)yl, page,
                      &full_bar[slot]);
        }
        if (box_ok(XC + 256 * b))
          tma_load_3d(st + STREAM_BYTES + b * R_ * 256, &tin, (int32_t)(XC + 256 * b), (int32_t)yc, page,
                      &full_bar[slot]);
      }
    }
  };
  if (p.use_tma && (nbox_el < NBOX || nbox_c < NBOX)) {
    for (int slot = 0; slot < NS; ++slot)
      for (int sidx = 0; sidx < 3; ++sidx)
        for (int b = 0; b < NBOX; ++b) {
          const int64_t x = (sidx == 1 ? XC : XE) + 256 * b;
          if (box_ok(x)) continue;
          uint4* z = reinterpret_cast<uint4*>(ring + slot * STAGE_BYTES + sidx * STREAM_BYTES + b * R_ * 256);
          for (int e = tid; e < R_ * 16; e += NT) z[e] = make_uint4(0, 0, 0, 0);
        }
    __syncthreads();
  }

  // Generic loader: all threads copy the stage's rows (zero outside the
  // held rows / image columns), the same layout the TMA boxes produce.
  auto fill = [&](int s) {
    uint8_t* st = ring + (s % NS) * STAGE_BYTES;
    const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;
    const int nstream = s < WS ? 1 : 3;
    for (int e = tid; e < nstream * STREAM_BYTES; e += NT) {
      const int sidx = e / STREAM_BYTES, rem = e - sidx * STREAM_BYTES;
      const int b = rem / (R_ * 256), rr = (rem / 256) % R_, cc = rem % 256;
      int64_t y, x = XE + 256 * b + cc;
      if (s < WS) {
        y = y0 - p.o + (int64_t)s * R_ + rr;
      } else {
        const int64_t qrow = y0 + (int64_t)(s - WS) * R_ + rr;
        y = sidx == 0 ? qrow + p.u : (sidx == 1 ? qrow : qrow - p.o);
        if (sidx == 1) x += XC - XE;
      }
      y -= p.buf_row0;
      st[e] = (y >= 0 && y < p.buf_rows && x >= 0 && x < p.W) ? img[y * p.in_pitch + x] : (uint8_t)0;
    }
  };
  if (p.use_tma && tid == 0)
    for (int s = 0; s < NS && s < total; ++s) issue(s);

  // ---- per-thread constants
  const int64_t a = S + (int64_t)G * tid;          // first owned input column
  const int64_t j0 = a - p.r;                      // first output column
  // staged byte e of a row lives at (e / 256) * R_*256 + (e % 256) (+ row * 256)
  auto soff = [&](int e) { return (e >> 8) * (R_ * 256) + (e & 255); };
  const int boff = soff(G * tid);                    // centre stream
  const int e0 = G * tid + (dl & ~7);                // entering/leaving: 8-byte words at e0, e0 + 8
  const int eoff0 = soff(e0), eoff1 = soff(e0 + 8);
  const uint32_t fsh = 8u * (uint32_t)(dl & 3);      // funnel shift within the word pair
  const bool fhi = (dl & 4) != 0;
  const int pp = ((-(p.w + 1)) % G + G) % G;       // partial-prefix position
  const int kp = tid - (p.w + 1 + G - 1) / G;       // thread holding column a - w - 1
  const bool valid_thread = tid >= p.KH;
  int ncol[G];
#pragma unroll
  for (int t = 0; t < G; ++t) {
    const int64_t j = j0 + t;
    ncol[t] = (int)(min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));
  }
  const double Lw = (p.method == M_WOLF || p.method == M_FENG) ? (double)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0;

  uint32_t C[G], D[G];
#pragma unroll
  for (int t = 0; t < G; ++t) C[t] = D[t] = 0;

  uint64_t near_ties = 0;

  // ---- warm-up: rows y0-o .. y0-o+h-1 (h rows; the first output row adds
  // row y0+u and subtracts row y0-o, giving rows (y0-o, y0+u]).
  for (int s = 0; s < WS; ++s) {
    const int slot = s % NS;
    if (p.use_tma) {
      mbar_wait(&full_bar[slot], (s / NS) & 1);
    } else {
      fill(s);
      __syncthreads();
    }
    const uint8_t* st = ring + slot * STAGE_BYTES;
    const int nr = min(R_, p.h - s * R_);
    for (int rr = 0; rr < nr; ++rr) {
      Bytes<G> x;
      x.v = funnel8(*reinterpret_cast<const uint2*>(st + eoff0 + rr * 256),
                    *reinterpret_cast<const uint2*>(st + eoff1 + rr * 256), fsh, fhi);
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const uint32_t v = x.at(t);
        C[t] += v;
        D[t] += v * v;
      }
    }
    __syncthreads();
    if (p.use_tma && tid == 0 && s + NS < total) issue(s + NS);
  }

  // ---- main rows
  int64_t q = 0;
  for (int s = WS; s < total; ++s) {
    const int slot = s % NS;
    if (p.use_tma) {
      mbar_wait(&full_bar[slot], (s / NS) & 1);
    } else {
      fill(s);
      __syncthreads();
    }
    const uint8_t* st = ring + slot * STAGE_BYTES;
    const int nr = (int)min((int64_t)R_, nrows - (int64_t)(s - WS) * R_);
    for (int rr = 0; rr < nr; ++rr, ++q) {
      const int buf = (int)(q & 1);
      Bytes<G> xi, xo, xc;
      xi.v = funnel8(*reinterpret_cast<const uint2*>(st + eoff0 + rr * 256),
                     *reinterpret_cast<const uint2*>(st + eoff1 + rr * 256), fsh, fhi);
      xc.v = *reinterpret_cast<const uint2*>(st + STREAM_BYTES + boff + rr * 256);
      xo.v = funnel8(*reinterpret_cast<const uint2*>(st + 2 * STREAM_BYTES + eoff0 + rr * 256),
                     *reinterpret_cast<const uint2*>(st + 2 * STREAM_BYTES + eoff1 + rr * 256), fsh, fhi);
      // vertical update
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const uint32_t vi = xi.at(t), vo = xo.at(t);
        C[t] = C[t] + vi - vo;
        D[t] = D[t] + vi * vi - vo * vo;
      }
      // thread totals and partial prefix up to position pp
      uint32_t Tc = 0, Pc = 0;
      DT Td = 0, Pd = 0;
#pragma unroll
      for (int t = 0; t < G; ++t) {
        Tc += C[t];
        Td += (DT)D[t];
        if (t <= pp) {
          Pc += C[t];
          Pd += (DT)D[t];
        }
      }
      // warp inclusive scan of (Tc, Td)
      uint32_t ic = Tc;
      DT id = Td;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t oc = __shfl_up_sync(0xffffffffu, ic, off);
        const DT od = __shfl_up_sync(0xffffffffu, id, off);
        if (lane >= off) {
          ic += oc;
          id += od;
        }
      }
      const uint32_t ec = ic - Tc;
      const DT ed = id - Td;
      if (lane == 31) {
        Wc[buf * NW + warp] = ic;
        Wd[buf * NW + warp] = id;
      }
      // publish this row's column sums and the partial prefix
      uint32_t* cb = Cb + buf * STRIP + G * tid;
      uint32_t* db = Db + buf * STRIP + G * tid;
#pragma unroll
      for (int t = 0; t < G; t += 4) {
        *reinterpret_cast<uint4*>(cb + t) = make_uint4(C[t], C[t + 1], C[t + 2], C[t + 3]);
        *reinterpret_cast<uint4*>(db + t) = make_uint4(D[t], D[t + 1], D[t + 2], D[t + 3]);
      }
      Qc[buf * NT + tid] = ec + Pc;
      Qd[buf * NT + tid] = ed + Pd;
      __syncthreads();

      // anchor A = sum_{b=a-w}^{a-1} C_b = P(a-1) - P(a-w-1)
      uint32_t offc_me = 0, offc_kp = 0;
      DT offd_me = 0, offd_kp = 0;
      const int wkp = valid_thread ? (kp >> 5) : 0;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) {
        const uint32_t tc = Wc[buf * NW + ww];
        const DT td = Wd[buf * NW + ww];
        if (ww < warp) { offc_me += tc; offd_me += td; }
        if (ww < wkp) { offc_kp += tc; offd_kp += td; }
      }
      const int kpc = valid_thread ? kp : 0;
      uint32_t cc = (offc_me + ec) - (offc_kp + Qc[buf * NT + kpc]);
      DT dd = (offd_me + ed) - (offd_kp + Qd[buf * NT + kpc]);

      // leaving column sums, columns a - w + t (strip index G*tid - w + t)
      uint32_t Cl[G], Dl[G];
      {
        const int st0 = valid_thread ? (G * tid - p.w - PH) : 0;  // 4-aligned
        uint32_t qv[G + 4], dv[G + 4];
#pragma unroll
        for (int t = 0; t < G + 4; t += 4) {
          if (PH == 0 && t == G) break;
          const uint4 a4 = *reinterpret_cast<const uint4*>(Cb + buf * STRIP + st0 + t);
          const uint4 b4 = *reinterpret_cast<const uint4*>(Db + buf * STRIP + st0 + t);
          qv[t] = a4.x; qv[t + 1] = a4.y; qv[t + 2] = a4.z; qv[t + 3] = a4.w;
          dv[t] = b4.x; dv[t + 1] = b4.y; dv[t + 2] = b4.z; dv[t + 3] = b4.w;
        }
#pragma unroll
        for (int t = 0; t < G; ++t) {
          Cl[t] = qv[t + PH];
          Dl[t] = dv[t + PH];
        }
      }

      const int64_t i = y0 + q;  // global output row
      const int nrow = (int)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
      uint32_t mbits = 0;  // bit t = mask of output j0 + t
#pragma unroll
      for (int t = 0; t < G; ++t) {
        cc += C[t] - Cl[t];
        dd += (DT)D[t] - (DT)Dl[t];
        const uint32_t n = (uint32_t)(ncol[t] * nrow);
        const double tt = is_rule(p.method) ? threshold_rule_fp64(p.method, (uint64_t)cc, (uint64_t)dd, n, p.rp, Lw, page)
                                            : threshold_fp64(p.method, (uint64_t)cc, (uint64_t)dd, n, p.k, p.R, Lw);
        const double I = (double)xc.at(t);
        const uint32_t mk = (I <= tt) ? 0u : 1u;
        mbits |= mk << t;
        const int64_t j = j0 + t;
        const bool in_img = valid_thread && j < p.W && j < J0 + p.T;
        if (in_img && fabs(I - tt) < 1e-9) near_ties++;
        if (STATS && in_img && page == 0) {
          const int64_t idx = (i - p.row0) * p.W + j;
          if (p.c_out) p.c_out[idx] = (uint64_t)cc;
          if (p.d_out) p.d_out[idx] = (uint64_t)dd;
          if (p.n_out) p.n_out[idx] = n;
          if (p.t_out) p.t_out[idx] = tt;
          if (p.mask_out) p.mask_out[idx] = (uint8_t)mk;
        }
      }
      // store the mask (outputs j0 .. j0+G-1; j0 is a multiple of G)
      if (valid_thread && j0 < p.W && j0 < J0 + p.T) {
        const int nvalid = (int)min((int64_t)G, min(p.W, J0 + p.T) - j0);
        uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (i - p.row0) * p.out_pitch;
        if (p.fmt == 0) {
          uint8_t* o = orow + j0;
          if (nvalid == G && p.out_vec_ok) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              lo |= ((mbits >> t) & 1u) << (8 * t);
              hi |= ((mbits >> (t + 4)) & 1u) << (8 * t);
            }
            *reinterpret_cast<uint2*>(o) = make_uint2(lo, hi);
          } else {
            for (int t = 0; t < nvalid; ++t) o[t] = (uint8_t)((mbits >> t) & 1u);
          }
        } else {
          // MSB-first: output j0 + t -> bit 7 - t of byte j0/8; pad bits are 0
          uint32_t byte = 0;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < nvalid) byte |= ((mbits >> t) & 1u) << (7 - t);
          orow[j0 >> 3] = (uint8_t)byte;
        }
      }
    }
    __syncthreads();
    if (p.use_tma && tid == 0 && s + NS < total) issue(s + NS);
  }

  if (p.counters) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) near_ties += __shfl_down_sync(0xffffffffu, near_ties, off);
    if (lane == 0 && near_ties) atomicAdd(reinterpret_cast<unsigned long long*>(&p.counters[0]),
                                         (unsigned long long)near_ties);
  }
}

template <int NT, int G, int R_, bool D64>
constexpr size_t moments_smem_bytes() {
  using DT = typename std::conditional<D64, uint64_t, uint32_t>::type;
  return 3 * 3 * R_ * NT * G          // ring
         + 2 * 2 * NT * G * 4         // Cb, Db
         + 2 * NT * 4 + 2 * NT * sizeof(DT)  // Qc, Qd
         + 2 * (NT / 32) * 4 + 2 * (NT / 32) * sizeof(DT) + 3 * 8;
}

}  // namespace wide
}  // namespace abin
