// small.cuh -- the moments path for small calls (a page of a few hundred
// thousand pixels, windows up to 64 x 64): one launch, one CTA per output
// tile, everything in shared memory.  The streaming kernel (moments5.cuh) is
// built for throughput -- one warp walks a band of rows through a TMA ring
// -- and on a single small page its time is the latency of a lone warp's
// rows (config 1, 512^2: ~19 us for k_mom5 plus the exact-fixup launch).
// Here a CTA of 128 threads takes a 16 x 128 output tile:
//   1. the tile's input region (16 + h - 1 rows x 128 + w - 1 columns; 0
//      outside the image) is loaded into shared memory;
//   2. vertical window sums C, D of every region column for the 16 output
//      rows by the recursion of PAPER.md:107-110 (a thread per column, exact
//      uint32: 255^2 h < 2^32);
//   3. horizontal window sums c, d per output pixel by the row recursion of
//      PAPER.md:119-120 (a thread per 16 outputs of a row, exact uint32), the
//      count n of Alg. 1 l.118, and the decision: the certified fp32 residual
//      of the v5 kernel (residual_pair, bound delta1 of filter_consts_v5) and,
//      for a pixel inside the bound, the canonical IEEE-double threshold
//      (threshold_fp64, Table 1 left to right) inline -- so every mask bit is
//      the double-precision decision and no exact-fixup launch follows.
#pragma once
#include <cstdint>

#include "moments.cuh"
#include "moments5.cuh"

namespace abin {
namespace sm {

constexpr int kTH = 16, kTW = 128, kNT = 128;
constexpr int kMaxWin = 64;  // h, w (effective) of the small path

struct SmallParams {
  const uint8_t* in;          // first held row (global row buf_row0) of page 0
  int64_t in_page_stride, in_pitch, W;
  int64_t buf_row0, row0, H_out, H_global;
  uint8_t* out;
  int64_t out_pitch, out_page_stride;
  int32_t fmt;
  int32_t h, w, l, r, o, u;
  int32_t RWp;                // region row pitch in shared memory (bytes, multiple of 16, >= 128 + w - 1 + 15)
  int32_t CWp;                // pitch of the column sums (words, odd)
  int32_t n_rt, n_ct;         // tiles per page
  float fa, fb, delta1;
  double k, R;
  const uint8_t* L_page;      // Wolf: per-page minimum (device), or L_fixed >= 0
  int32_t L_fixed;
  unsigned long long* counters;  // [near ties, fp64 decisions] or null
};

// region bytes rounded up to 16 (the sums that follow are 32-bit words)
__host__ __device__ inline size_t region_bytes(int RWp, int h) { return (size_t)(kTH + h - 1) * RWp; }
__host__ __device__ inline size_t smem_bytes(int RWp, int CWp, int h) {
  return region_bytes(RWp, h) + (size_t)2 * kTH * CWp * 4;
}

template <int METHOD>
__global__ void __launch_bounds__(kNT) k_small(const SmallParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x;
  int64_t b = blockIdx.x;
  const int ct = (int)(b % p.n_ct);
  b /= p.n_ct;
  const int rt = (int)(b % p.n_rt);
  const int page = (int)(b / p.n_rt);
  const int64_t i0 = p.row0 + (int64_t)rt * kTH, j0 = (int64_t)ct * kTW;
  const int RH = kTH + p.h - 1, RW = kTW + p.w - 1, RWp = p.RWp, CWp = p.CWp;
  uint8_t* reg = smem;                                                 // [RH][RWp]
  uint32_t* Cs = reinterpret_cast<uint32_t*>(smem + region_bytes(RWp, p.h));  // [kTH][CWp]
  uint32_t* Ds = Cs + kTH * CWp;
  const uint8_t* pg = p.in + (int64_t)page * p.in_page_stride;
  const int64_t y0 = i0 - p.o + 1, x0 = j0 - p.l + 1;                 // region origin (global)

  // 1. the region, 0 outside the image (or outside the held rows), staged
  // from the 16-aligned column xa = x0 - dx: 16-byte chunks (byte loads only
  // for chunks that leave the image or rows that are not 16-aligned)
  const int64_t xa = x0 & ~(int64_t)15;
  const int dx = (int)(x0 - xa);
  {
    const int nch = (dx + RW + 15) >> 4;
    const bool vec = ((reinterpret_cast<uintptr_t>(p.in) | (uintptr_t)p.in_pitch | (uintptr_t)p.in_page_stride) &
                      15u) == 0;
    for (int idx = tid; idx < RH * nch; idx += kNT) {
      const int ry = idx / nch, ch = idx - ry * nch;
      const int64_t y = y0 + ry, x = xa + 16 * ch;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (y >= 0 && y < p.H_global) {
        const uint8_t* row = pg + (y - p.buf_row0) * p.in_pitch;
        if (vec && x >= 0 && x + 16 <= p.W) {
          v = __ldg(reinterpret_cast<const uint4*>(row + x));
        } else {
          uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
          for (int b = 0; b < 16; ++b)
            if (x + b >= 0 && x + b < p.W) wv[b >> 2] |= (uint32_t)__ldg(row + x + b) << (8 * (b & 3));
          v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
      *reinterpret_cast<uint4*>(reg + ry * RWp + 16 * ch) = v;
    }
  }
  __syncthreads();
  // 2. vertical sums of each region column for the kTH output rows
  for (int x = tid; x < RW; x += kNT) {
    uint32_t c = 0, d = 0;
#pragma unroll 4
    for (int y = 0; y < p.h; ++y) {
      const uint32_t v = reg[y * RWp + dx + x];
      c += v;
      d += v * v;
    }
    Cs[x] = c;
    Ds[x] = d;
#pragma unroll 4
    for (int t = 1; t < kTH; ++t) {
      const uint32_t vi = reg[(t + p.h - 1) * RWp + dx + x], vo = reg[(t - 1) * RWp + dx + x];
      c += vi - vo;
      d += vi * vi - vo * vo;
      Cs[t * CWp + x] = c;
      Ds[t * CWp + x] = d;
    }
  }
  __syncthreads();
  // 3. a thread = 16 outputs of one row: horizontal sums, then the decision
  const int t = tid >> 3, seg = tid & 7;
  const int64_t i = i0 + t;
  const int64_t jb = j0 + 16 * seg;
  if (i >= p.row0 + p.H_out || jb >= p.W) return;
  const uint32_t* Cr = Cs + t * CWp + 16 * seg;
  const uint32_t* Dr = Ds + t * CWp + 16 * seg;
  uint32_t c = 0, d = 0;
#pragma unroll 4
  for (int x = 0; x < p.w; ++x) {
    c += Cr[x];
    d += Dr[x];
  }
  const uint32_t nrow = (uint32_t)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
  const float inv_nrow = __frcp_rn((float)nrow);
  const float Lf = METHOD == M_WOLF ? (float)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0f;
  v5::f2 fa2, fb2;
  v5::method_consts<METHOD>(p.fa, p.fb, fa2, fb2);
  const v5::f2 Lf2 = v5::splat(Lf);
  const uint8_t* irow = pg + (i - p.buf_row0) * p.in_pitch;
  unsigned long long near = 0, fb64 = 0;
  uint32_t bits = 0;
  uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (i - p.row0) * p.out_pitch;
  const int nval = (int)min((int64_t)16, p.W - jb);
#pragma unroll 1
  for (int s2 = 0; s2 < 16; s2 += 2) {
    uint32_t cq[2], dq[2], nq[2];
    float nuv[2];
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      const int s = s2 + z;
      const int64_t j = jb + s;
      cq[z] = c;
      dq[z] = d;
      const uint32_t ncol = (uint32_t)(min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));
      nq[z] = ncol * nrow;
      nuv[z] = -(__frcp_rn((float)ncol) * inv_nrow);
      // slide to output s + 1: c += C[s + w] - C[s] (region columns of this segment)
      c += Cr[s + p.w] - Cr[s];
      d += Dr[s + p.w] - Dr[s];
    }
    const v5::f2 nu = v5::pk(nuv[0], nuv[1]);
    const v5::f2 nb = v5::mul2(nu, v5::splat(-8388608.0f));
    const uint32_t Ia = s2 < nval ? irow[jb + s2] : 0u, Ib = s2 + 1 < nval ? irow[jb + s2 + 1] : 0u;
    v5::f2 sv;
    const v5::f2 e = v5::residual_pair<METHOD>(v5::kBias + cq[0], v5::kBias + cq[1], dq[0], dq[1], nu, nb,
                                               v5::pk((float)Ia, (float)Ib), fa2, fb2, Lf2, sv);
    const float ez[2] = {v5::lo(e), v5::hi(e)};
    const uint32_t Iz[2] = {Ia, Ib};
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      if (s2 + z >= nval) continue;
      uint32_t mk;
      if (fabsf(ez[z]) >= p.delta1) {
        mk = ez[z] < 0.0f ? 0u : 1u;  // e = I - t~ < 0: I < t, foreground (0)
      } else {
        const double tt = threshold_fp64(METHOD, cq[z], dq[z], nq[z], p.k, p.R, (double)Lf);
        mk = ((double)Iz[z] <= tt) ? 0u : 1u;
        ++fb64;
        if (fabs((double)Iz[z] - tt) < 1e-9) ++near;
      }
      if (p.fmt == 0) orow[jb + s2 + z] = (uint8_t)mk;
      else bits |= mk << (15 - (s2 + z));
    }
  }
  if (p.fmt != 0) {
    orow[jb >> 3] = (uint8_t)(bits >> 8);
    if (nval > 8) orow[(jb >> 3) + 1] = (uint8_t)(bits & 0xFFu);
  }
  if (p.counters) {
    if (near) atomicAdd(&p.counters[0], near);
    if (fb64) atomicAdd(&p.counters[1], fb64);
  }
}

}  // namespace sm
}  // namespace abin
