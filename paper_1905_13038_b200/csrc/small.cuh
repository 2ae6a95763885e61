// small.cuh -- the moments path for small calls (a page of a few hundred
// thousand pixels, windows up to 64 x 64): one launch, one CTA per output
// tile, everything in shared memory.  The streaming kernel (moments5.cuh) is
// built for throughput -- one warp walks a band of rows through a TMA ring
// -- and on a single small page its time is the latency of a lone warp's
// rows (config 1, 512^2: ~19 us for k_mom5 plus the exact-fixup launch).
// Here a CTA of 256 threads takes a 16 x 128 output tile:
//   1. the tile's input region (16 + h - 1 rows x 128 + w - 1 columns; 0
//      outside the image) is loaded into shared memory;
//   2. vertical window sums C, D of every region column for the 16 output
//      rows by the recursion of PAPER.md:107-110 (a thread per column, exact
//      uint32: 255^2 h < 2^32);
//   3. horizontal window sums c, d per output pixel as
//      differences of per-row prefix sums of C, D (exact uint32; a warp per
//      two rows, a lane per column of each 32-column group), the
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

constexpr int kTH = 16, kTW = 128, kNT = 256;  // kTH: the default tile height (the kernel's TH: 16 or 32)
static_assert(kTH % (kNT / 32) == 0 && kTW % 64 == 0, "step 3: a warp takes kRPW rows, a lane pairs of 32-column groups");
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
__host__ __device__ inline size_t region_bytes(int RWp, int h, int TH) { return (size_t)(TH + h - 1) * RWp; }
__host__ __device__ inline size_t smem_bytes(int RWp, int CWp, int h, int TH) {
  return region_bytes(RWp, h, TH) + (size_t)2 * TH * CWp * 4;
}

#ifndef ABIN_SMALL_MINB
#define ABIN_SMALL_MINB 4  // resident CTAs per SM the register budget is set for (64 registers; 1: 80 registers, 1024^2 pages 15 % slower)
#endif
// TH: the tile height -- 16 (more tiles: latency of single small pages) or 32
// (pages of several waves of tiles: the h - 1 re-staged rows and the column
// sums' start-up are amortised over twice the rows)
template <int METHOD, int TH>
__global__ void __launch_bounds__(kNT, ABIN_SMALL_MINB) k_small(const SmallParams p) {
  constexpr int RPW = TH / (kNT / 32);  // output rows per warp in steps 2b, 3
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x;
  uint32_t b = blockIdx.x;  // < 2^31 tiles: 32-bit divisions
  const int ct = (int)(b % (uint32_t)p.n_ct);
  b /= (uint32_t)p.n_ct;
  const int rt = (int)(b % (uint32_t)p.n_rt);
  const int page = (int)(b / (uint32_t)p.n_rt);
  const int64_t i0 = p.row0 + (int64_t)rt * TH, j0 = (int64_t)ct * kTW;
  const int RH = TH + p.h - 1, RW = kTW + p.w - 1, RWp = p.RWp, CWp = p.CWp;
  uint8_t* reg = smem;                                                 // [RH][RWp]
  uint32_t* Cs = reinterpret_cast<uint32_t*>(smem + region_bytes(RWp, p.h, TH));  // [TH][CWp]
  uint32_t* Ds = Cs + TH * CWp;
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
    // a 16-lane group per region row, a lane per 16-byte chunk (nch <= 13), 16
    // rows per pass: no index divisions.  x is a multiple of 16, so a chunk
    // left of the image is wholly outside; chunk classes: 0 zeros, 1 one
    // 16-byte load, 2 byte loads (the chunk holding column W, unaligned rows)
    const int ch = tid & 15, rg = tid >> 4;
    const int64_t x = xa + 16 * ch;
    const bool ch_ok = ch < nch;
    const int cls = (!ch_ok || x + 16 <= 0 || x >= p.W) ? 0 : ((vec && x + 16 <= p.W) ? 1 : 2);
    auto fetch = [&](int ry) {
      const int64_t y = y0 + ry;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (cls != 0 && y >= 0 && y < p.H_global) {
        const uint8_t* row = pg + (y - p.buf_row0) * p.in_pitch;
        if (cls == 1) {
          v = __ldg(reinterpret_cast<const uint4*>(row + x));
        } else {
          uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
          for (int b = 0; b < 16; ++b)
            if (x + b >= 0 && x + b < p.W) wv[b >> 2] |= (uint32_t)__ldg(row + x + b) << (8 * (b & 3));
          v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
      return v;
    };
    // kLD rows in flight per thread (a lone CTA per SM: the loads' latency is the cost)
    constexpr int kLD = 4;
    for (int r0 = rg; r0 < RH; r0 += kLD * (kNT / 16)) {
      uint4 v[kLD];
#pragma unroll
      for (int k = 0; k < kLD; ++k) {
        const int ry = r0 + k * (kNT / 16);
        v[k] = ry < RH ? fetch(ry) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int k = 0; k < kLD; ++k) {
        const int ry = r0 + k * (kNT / 16);
        if (ry < RH && ch_ok) *reinterpret_cast<uint4*>(reg + ry * RWp + 16 * ch) = v[k];
      }
    }
  }
  __syncthreads();
  // 2. vertical sums of each region column for the TH output rows
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
    for (int t = 1; t < TH; ++t) {
      const uint32_t vi = reg[(t + p.h - 1) * RWp + dx + x], vo = reg[(t - 1) * RWp + dx + x];
      c += vi - vo;
      d += vi * vi - vo * vo;
      Cs[t * CWp + x] = c;
      Ds[t * CWp + x] = d;
    }
  }
  __syncthreads();
  // 2b. each warp turns its RPW rows of C and D into exclusive prefix sums
  // along the row (RW + 1 entries: P[x] = C[0] + .. + C[x-1], uint32 wraps
  // cancel in differences), so that the window sums of PAPER.md:119-120 are
  // c(j) = P[j + w] - P[j] for any thread-to-column mapping: step 3 reads
  // consecutive words per warp (no bank conflicts) instead of running the
  // row recursion over a thread's own 16-column segment.
  const int wid = tid >> 5, lane = tid & 31;
  {
    const int NP = RW + 1;             // <= 192 = 32 lanes x 6 (RW <= 128 + 64 - 1)
    constexpr int chunk = 6;
#pragma unroll 1
    for (int q = 0; q < 2 * RPW; ++q) {
      uint32_t* A = ((q & 1) ? Ds : Cs) + (RPW * wid + (q >> 1)) * CWp;
      uint32_t v[6], sum = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int idx = lane * chunk + k;
        v[k] = idx < RW ? A[idx] : 0u;
        sum += v[k];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int dlt = 1; dlt < 32; dlt <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, dlt);
        if (lane >= dlt) inc += y;
      }
      uint32_t run = inc - sum;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int idx = lane * chunk + k;
        if (idx < NP) A[idx] = run;
        run += v[k];
      }
    }
  }
  __syncwarp();
  // 3. a warp = its RPW rows; a lane = the columns lane, lane + 32, lane + 64,
  // lane + 96 of the tile: window sums from the prefix rows, then the decision
  const float Lf = METHOD == M_WOLF ? (float)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0f;
  v5::f2 fa2, fb2;
  v5::method_consts<METHOD>(p.fa, p.fb, fa2, fb2);
  const v5::f2 Lf2 = v5::splat(Lf);
  unsigned long long near = 0, fb64 = 0;
  const int Wi = (int)p.W, j0i = (int)j0;
  // the lane's columns are the same in every row: their counts (Alg. 1 l.118) and reciprocals once
  uint32_t ncl[kTW / 32];
  float rcol[kTW / 32];
#pragma unroll
  for (int q = 0; q < kTW / 32; ++q) {
    const int j = j0i + 32 * q + lane;
    ncl[q] = j < Wi ? (uint32_t)(min(j + p.r, Wi - 1) - max(j - p.l, -1)) : 1u;
    rcol[q] = __frcp_rn((float)ncl[q]);
  }
  uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (i0 + RPW * wid - p.row0) * p.out_pitch - p.out_pitch;
#pragma unroll 1
  for (int rr = 0; rr < RPW; ++rr) {
    const int t = RPW * wid + rr;
    const int64_t i = i0 + t;
    if (i >= p.row0 + p.H_out) break;  // warp-uniform
    const uint32_t* Pc = Cs + t * CWp;
    const uint32_t* Pd = Ds + t * CWp;
    const uint32_t nrow = (uint32_t)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
    const float inv_nrow = __frcp_rn((float)nrow);
    // the centre pixels from the staged region (row t + o - 1, column l - 1 + tile column)
    const uint8_t* irow = reg + (t + p.o - 1) * RWp + dx + (p.l - 1);
    orow += p.out_pitch;
#pragma unroll
    for (int q2 = 0; q2 < kTW / 32; q2 += 2) {
      uint32_t cq[2], dq[2], nq[2], Iz[2];
      float nuv[2];
      bool ok[2];
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int jj = 32 * (q2 + z) + lane;
        const int j = j0i + jj;  // the small path's pages have W < 2^30 (run_small)
        ok[z] = j < Wi;
        cq[z] = Pc[jj + p.w] - Pc[jj];
        dq[z] = Pd[jj + p.w] - Pd[jj];
        nq[z] = ncl[q2 + z] * nrow;
        nuv[z] = -(rcol[q2 + z] * inv_nrow);
        Iz[z] = ok[z] ? irow[jj] : 0u;
      }
      const v5::f2 nu = v5::pk(nuv[0], nuv[1]);
      const v5::f2 nb = v5::mul2(nu, v5::splat(-8388608.0f));
      v5::f2 sv;
      const v5::f2 e = v5::residual_pair<METHOD>(v5::kBias + cq[0], v5::kBias + cq[1], dq[0], dq[1], nu, nb,
                                                 v5::pk((float)Iz[0], (float)Iz[1]), fa2, fb2, Lf2, sv);
      const float ez[2] = {v5::lo(e), v5::hi(e)};
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        uint32_t mk = 0u;
        if (ok[z]) {
          if (fabsf(ez[z]) >= p.delta1) {
            mk = ez[z] < 0.0f ? 0u : 1u;  // e = I - t~ < 0: I < t, foreground (0)
          } else {
            const double tt = threshold_fp64(METHOD, cq[z], dq[z], nq[z], p.k, p.R, (double)Lf);
            mk = ((double)Iz[z] <= tt) ? 0u : 1u;
            ++fb64;
            if (fabs((double)Iz[z] - tt) < 1e-9) ++near;
          }
        }
        const int jq = j0i + 32 * (q2 + z);  // first column of this 32-column group
        if (p.fmt == 0) {
          if (ok[z]) orow[jq + lane] = (uint8_t)mk;
        } else {
          // bit mask, MSB first: lane L's bit is column jq + L, byte b holds columns 8 b .. 8 b + 7
          const uint32_t word = __brev(__ballot_sync(0xffffffffu, mk != 0u));
          if (lane < 4 && jq + 8 * lane < Wi) orow[(jq >> 3) + lane] = (uint8_t)(word >> (24 - 8 * lane));
        }
      }
    }
  }
  if (p.counters) {
    if (near) atomicAdd(&p.counters[0], near);
    if (fb64) atomicAdd(&p.counters[1], fb64);
  }
}

}  // namespace sm
}  // namespace abin
