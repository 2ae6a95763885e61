// fixup.cuh -- the exact stages of the certified decision (DESIGN.md section
// 5) for the lanes the v4 kernel could not decide in fp32.  The v4 kernel
// queues each such lane as (page, output row, first column j0, 16-bit mask of
// its pixels) and stores provisional bits; this kernel recomputes the
// pixels' window sums directly from the image (the definition, PAPER.md:118-
// 124: c = sum of I, d = sum of I^2 over the clamped window, n its size),
// runs stage 2 (fp32 from the exact integer V = n d - c^2, bound delta2) and,
// for what is still ambiguous, the canonical IEEE double sequence (Alg. 1
// l.121-124, Table 1 left to right), then overwrites the provisional bits.
// It also counts near ties (|I - t| < 1e-9), fp64 decisions and stage-2
// pixels.  If the queue overflowed, the v3 kernel re-runs the whole call in
// exact mode instead and this kernel stands aside (no double counting).
#pragma once
#include <cstdint>

#include "moments.cuh"
#include "rules.cuh"

namespace abin {

constexpr int kFixWarps = 4;           // warps per CTA; a warp per queued lane
constexpr int kFixNT = 32 * kFixWarps;
constexpr int kFixLd = 4;              // 16-byte loads in flight per lane

// dynamic shared memory of k_fixup, per warp: one staged row per lane (whole
// 16-byte chunks covering the 16 windows' columns) + the row-sum transpose
__host__ __device__ inline int fixup_chunks(int w) { return (15 + w + 15 + 15) / 16; }
// (a lane's row takes 4 nv + 1 words: an odd stride keeps the 32 lanes' byte
// reads of the same column in 32 different banks)
__host__ __device__ inline int fixup_stage_bytes(int w) { return (32 * (4 * fixup_chunks(w) + 1) * 4 + 15) & ~15; }
__host__ __device__ inline int fixup_warp_bytes(int w) { return fixup_stage_bytes(w) + 32 * 16 * (8 + 4); }
inline size_t fixup_smem_bytes(int w) { return (size_t)kFixWarps * fixup_warp_bytes(w); }

// One exact decision into the output: a byte, or the MSB-first bit j of the
// row patched with a 32-bit atomic on the aligned word holding its byte (the
// word's other bytes -- possibly of a neighbouring row -- are left as they
// are; CUDA allocations are 256-byte aligned, so the word never leaves the
// allocation)
__device__ __forceinline__ void store_mask(const MomParams& p, int page, int64_t y, int64_t j, uint32_t mk) {
  uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + y * p.out_pitch;
  if (p.fmt == 0) {
    orow[j] = (uint8_t)mk;
  } else {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(orow + (j >> 3));
    unsigned int* word = reinterpret_cast<unsigned int*>(addr & ~(uintptr_t)3);
    const unsigned int bit = 1u << (8 * (unsigned)(addr & 3) + (7 - (unsigned)(j & 7)));
    if (mk) atomicOr(word, bit);
    else atomicAnd(word, ~bit);
  }
}

static __global__ void __launch_bounds__(kFixNT, 4) k_fixup(const MomParams p) {
  extern __shared__ __align__(16) uint8_t fsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nvmax = fixup_chunks(p.w);
  const int rstride = 4 * nvmax + 1;                           // words per staged row (odd)
  uint8_t* wbase = fsm + (size_t)warp * fixup_warp_bytes(p.w);
  uint32_t* my = reinterpret_cast<uint32_t*>(wbase) + lane * rstride;  // this lane's staged row
  unsigned long long* sd = reinterpret_cast<unsigned long long*>(wbase + fixup_stage_bytes(p.w));  // [32][16]
  uint32_t* sc = reinterpret_cast<uint32_t*>(sd + 32 * 16);                                          // [32][16]
  // programmatic launch (PDL): wait for the moments kernel's queue and mask
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t count = *p.q_count;
  const uint32_t nq = count > p.q_cap ? 0u : count;
  unsigned long long near = 0, fb64 = 0, st2 = 0;
  const uint32_t gw = blockIdx.x * kFixWarps + warp, nw_all = gridDim.x * kFixWarps;
  uint4 qn = gw < nq ? p.q_data[gw] : make_uint4(0u, 0u, 0u, 0u);
  for (uint32_t e = gw; e < nq; e += nw_all) {
    const uint4 q = qn;
    if (e + nw_all < nq) qn = p.q_data[e + nw_all];  // prefetch the warp's next entry
    const int page = (int)q.x;
    const int64_t i = p.row0 + (int64_t)q.y;  // global row
    const int64_t j0 = (int64_t)q.z;          // the lane's first column
    const uint32_t amb = q.w;
    const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;
    // the 16 windows span columns [x0, x0 + w + 15), x0 = j0 - l + 1, staged
    // as whole 16-byte chunks from xs = x0 rounded down (rows are 16-byte
    // aligned and their last partial chunk readable: abin.h); bytes outside
    // [0, W) are zero (n counts the in-bounds columns)
    const int64_t x0 = j0 - p.l + 1;
    const int64_t xs = x0 >= 0 ? (x0 & ~(int64_t)15) : -((-x0 + 15) & ~(int64_t)15);
    const int off = (int)(x0 - xs);
    const int nv = (off + p.w + 15 + 15) >> 4;
    // window rows (i - o, i + u] clamped to the image; lane = row (strided)
    const int64_t a0 = max(i - p.o + 1, (int64_t)0), a1 = min(i + p.u, p.H_global - 1);
    // the centre pixel, loaded now so its latency overlaps the staging
    const uint32_t I = (lane < 16 && ((amb >> lane) & 1u)) ? __ldg(img + (i - p.buf_row0) * p.in_pitch + j0 + lane) : 0u;
    uint32_t c[16];
    unsigned long long dl[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = 0u, dl[t] = 0ull;
    for (int64_t a = a0 + lane; a <= a1; a += 32) {
      const uint8_t* src = img + (a - p.buf_row0) * p.in_pitch;
      // the row's chunks: kFixLd independent loads in flight (the fixup is
      // latency-bound: a few DRAM round trips per queued lane)
      for (int v0 = 0; v0 < nv; v0 += kFixLd) {
        uint4 x[kFixLd];
#pragma unroll
        for (int z = 0; z < kFixLd; ++z) {
          const int64_t col = xs + 16 * (int64_t)(v0 + z);
          x[z] = make_uint4(0u, 0u, 0u, 0u);
          if (v0 + z < nv && col >= 0 && col < p.W) x[z] = __ldg(reinterpret_cast<const uint4*>(src + col));
        }
#pragma unroll
        for (int z = 0; z < kFixLd; ++z) {
          const int64_t col = xs + 16 * (int64_t)(v0 + z);
          if (v0 + z < nv) {
            if (col + 16 > p.W) {  // the image's last chunk: zero the bytes >= W
              uint32_t wd[4] = {x[z].x, x[z].y, x[z].z, x[z].w};
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const int64_t keep = p.W - (col + 4 * g);
                wd[g] = keep >= 4 ? wd[g] : (keep <= 0 ? 0u : wd[g] & (0xFFFFFFFFu >> (8 * (4 - (int)keep))));
              }
              x[z] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
            }
            my[4 * (v0 + z)] = x[z].x;
            my[4 * (v0 + z) + 1] = x[z].y;
            my[4 * (v0 + z) + 2] = x[z].z;
            my[4 * (v0 + z) + 3] = x[z].w;
          }
        }
      }
      const uint8_t* row = reinterpret_cast<const uint8_t*>(my) + off;  // this lane's own staged row
      uint32_t cr = 0, dr = 0;  // one row: w 255^2 < 2^32 (v4 takes w < 500)
#pragma unroll 8
      for (int b = 0; b < p.w; ++b) {
        const uint32_t x = row[b];
        cr += x;
        dr += x * x;
      }
      c[0] += cr;
      dl[0] += dr;
#pragma unroll
      for (int t = 1; t < 16; ++t) {
        const uint32_t xi = row[p.w - 1 + t], xo = row[t - 1];
        cr += xi - xo;
        dr += xi * xi - xo * xo;
        c[t] += cr;
        dl[t] += dr;
      }
    }
    // transpose through the warp's shared memory: lanes 0-15 sum pixel t's c
    // over the 32 lanes, lanes 16-31 its d
#pragma unroll
    for (int t = 0; t < 16; t += 4)
      *reinterpret_cast<uint4*>(sc + lane * 16 + t) = make_uint4(c[t], c[t + 1], c[t + 2], c[t + 3]);
#pragma unroll
    for (int t = 0; t < 16; t += 2)
      *reinterpret_cast<ulonglong2*>(sd + lane * 16 + t) = make_ulonglong2(dl[t], dl[t + 1]);
    __syncwarp();
    const int t = lane & 15;
    uint64_t acc = 0;
    if (lane < 16) {
#pragma unroll 8
      for (int g = 0; g < 32; ++g) acc += sc[g * 16 + t];
    } else {
#pragma unroll 8
      for (int g = 0; g < 32; ++g) acc += sd[g * 16 + t];
    }
    const uint64_t dsum = __shfl_down_sync(0xffffffffu, acc, 16);
    __syncwarp();  // the staging / transpose buffers are reused by the next entry
    const int64_t j = j0 + t;
    if (lane < 16 && ((amb >> t) & 1u)) {
      const uint64_t c = acc, d = dsum;
      const int64_t ncol = min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1);
      const uint32_t n = (uint32_t)((a1 - a0 + 1) * ncol);
      if (p.method == M_MAXS) {
        // Wolf's adaptive R (R21): the pixel's s by the canonical double
        // sequence (Alg. 1 l.121-122, as threshold_fp64 and the oracle), into
        // the page's maximum (non-negative doubles order as their bits)
        const double nd = (double)n;
        const double mm = __ddiv_rn((double)c, nd);
        double v = __dsub_rn(__ddiv_rn((double)d, nd), __dmul_rn(mm, mm));
        if (v < 0.0) v = 0.0;
        atomicMax(p.smax_bits + page, (unsigned long long)__double_as_longlong(__dsqrt_rn(v)));
        continue;
      }
      if (is_rule(p.method)) {
        // v5 rules (Khurshid, Phansalkar): straight to the Table-1 row in IEEE double
        const double Lr = p.method == M_FENG ? (double)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0;
        const double tt = threshold_rule_fp64(p.method, c, d, n, p.rp, Lr, page);
        const uint32_t mk = ((double)I <= tt) ? 0u : 1u;
        ++fb64;
        if (fabs((double)I - tt) < 1e-9) ++near;
        store_mask(p, page, q.y, j, mk);
        continue;
      }
      const float Lf = (p.method == M_WOLF) ? (float)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0f;
      ++st2;
      // stage 2: exact V = n d - c^2 >= 0, fp32 with the tight bound delta2
      const uint64_t V = (uint64_t)n * d - c * c;
      const float Vf = __fmaf_rn((float)(uint32_t)(V >> 32), 4294967296.0f, (float)(uint32_t)V);
      const float invn = __frcp_rn((float)n);
      const float m = (float)(uint32_t)c * invn;
      const float t2 = threshold_f32(p.method, m, sqrt_approx(Vf) * invn, p.fa, p.fb, Lf);
      const float e2 = t2 - (float)I;
      uint32_t mk;
      if (fabsf(e2) >= p.delta2) {
        mk = e2 < 0.0f ? 1u : 0u;
      } else {
        const double tt = threshold_fp64(p.method, c, d, n, p.k, p.R, (double)Lf);
        mk = ((double)I <= tt) ? 0u : 1u;
        ++fb64;
        if (fabs((double)I - tt) < 1e-9) ++near;
      }
      store_mask(p, page, q.y, j, mk);
    }
  }
  if (p.counters) {
    for (int off = 16; off > 0; off >>= 1) {
      near += __shfl_down_sync(0xffffffffu, near, off);
      fb64 += __shfl_down_sync(0xffffffffu, fb64, off);
      st2 += __shfl_down_sync(0xffffffffu, st2, off);
    }
    if (lane == 0) {
      if (near) atomicAdd(reinterpret_cast<unsigned long long*>(&p.counters[0]), near);
      if (fb64) atomicAdd(reinterpret_cast<unsigned long long*>(&p.counters[1]), fb64);
      if (st2 && p.counters_n > 2) atomicAdd(reinterpret_cast<unsigned long long*>(&p.counters[2]), st2);
    }
  }
}

}  // namespace abin
