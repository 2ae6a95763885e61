// rules.cuh -- the remaining Table 1 rows: "binarization
// methods that can be implemented by changing a single condition in
// Algorithm 1".  Evaluated for every pixel in IEEE double,
// each row written left to right with explicitly rounded operations (no FMA
// contraction), after the canonical m = c/n, v = d/n - m^2 (clamped), s = sqrt v:
//   Feng       t = a1 m + k1 (s/R)^(1+g) (m - L) + k2 (s/R)^g L
//   Rais       t = m + 0.3 (m s - M S) / max{m s, M S} s
//   Khurshid   t = m + k sqrt(s^2 + m^2 (N - 1) / N)
//   Phansalkar t = m (1 + p e^(-q m) + k (s/R - 1))
// L = global minimum, M / S = global mean / standard deviation.
// pow / exp are CUDA's double-precision routines (<= 2 ulp): the masks equal
// the oracle's except possibly at pixels within ~1e-13 of the threshold
// (R18).  Khurshid and Rais use only IEEE-exact operations.
#pragma once
#include <cstdint>

namespace abin {

enum { M_FENG = 5, M_RAIS = 6, M_KHURSHID = 7, M_PHANSALKAR = 8 };

struct RuleParams {
  double p[5];    // Feng {a1, k1, k2, g, R}; Khurshid {k, N_mode}; Phansalkar {k, R, p, q}
  double hw;      // nominal window size h w (Khurshid's N)
  const double* MS;  // Rais: per page {M, S} (device)
};

__device__ __forceinline__ bool is_rule(int method) { return method >= M_FENG && method <= M_PHANSALKAR; }

static __device__ __noinline__ double threshold_rule_fp64(int rule, uint64_t c, uint64_t d, uint32_t n,
                                                          const RuleParams& rp, double L, int page) {
  const double nd = (double)n;
  const double m = __ddiv_rn((double)c, nd);
  double v = __dsub_rn(__ddiv_rn((double)d, nd), __dmul_rn(m, m));
  if (v < 0.0) v = 0.0;
  const double s = __dsqrt_rn(v);
  if (rule == M_FENG) {
    const double a1 = rp.p[0], k1 = rp.p[1], k2 = rp.p[2], g = rp.p[3], R = rp.p[4];
    const double sr = __ddiv_rn(s, R);
    const double t1 = __dmul_rn(a1, m);
    const double t2 = __dmul_rn(__dmul_rn(k1, pow(sr, __dadd_rn(1.0, g))), __dsub_rn(m, L));
    const double t3 = __dmul_rn(__dmul_rn(k2, pow(sr, g)), L);
    return __dadd_rn(__dadd_rn(t1, t2), t3);
  }
  if (rule == M_RAIS) {
    const double M = rp.MS[2 * page], S = rp.MS[2 * page + 1];
    const double a = __dmul_rn(m, s), b = __dmul_rn(M, S);
    const double den = a > b ? a : b;
    const double frac = den > 0.0 ? __ddiv_rn(__dsub_rn(a, b), den) : 0.0;
    return __dadd_rn(m, __dmul_rn(__dmul_rn(0.3, frac), s));
  }
  if (rule == M_KHURSHID) {
    const double k = rp.p[0];
    const double N = rp.p[1] != 0.0 ? nd : rp.hw;
    const double r = __ddiv_rn(__dsub_rn(N, 1.0), N);
    return __dadd_rn(m, __dmul_rn(k, __dsqrt_rn(__dadd_rn(__dmul_rn(s, s), __dmul_rn(__dmul_rn(m, m), r)))));
  }
  // Phansalkar
  const double k = rp.p[0], R = rp.p[1], pp = rp.p[2], q = rp.p[3];
  const double ex = exp(__dmul_rn(-q, m));
  return __dmul_rn(m, __dadd_rn(__dadd_rn(1.0, __dmul_rn(pp, ex)), __dmul_rn(k, __dsub_rn(__ddiv_rn(s, R), 1.0))));
}

// Per-page global sum / sum of squares (exact, uint64) for Rais's M and S.
// grid = (blocks_per_page, n_pages); acc[2 page], acc[2 page + 1] zeroed.
static __global__ void __launch_bounds__(256) k_global_sums(const uint8_t* __restrict__ in, int64_t page_stride, int64_t H,
                                                     int64_t W, int64_t pitch, unsigned long long* acc) {
  const int page = blockIdx.y;
  const uint8_t* img = in + (int64_t)page * page_stride;
  unsigned long long s1 = 0, s2 = 0;
  // 16-byte chunks when the page is aligned: the chunk's byte sum and square
  // sum by dp4a (exact in uint32), accumulated in uint64
  const bool vec = ((reinterpret_cast<uintptr_t>(img) | (uintptr_t)pitch) & 15u) == 0;
  const int64_t nv = vec ? W / 16 : 0;
  for (int64_t row = blockIdx.x; row < H; row += gridDim.x) {
    const uint8_t* r = img + row * pitch;
    for (int64_t q = threadIdx.x; q < nv; q += blockDim.x) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(r) + q);
      uint32_t a1 = __dp4a(v.x, 0x01010101u, 0u), a2 = __dp4a(v.x, v.x, 0u);
      a1 = __dp4a(v.y, 0x01010101u, a1); a1 = __dp4a(v.z, 0x01010101u, a1); a1 = __dp4a(v.w, 0x01010101u, a1);
      a2 = __dp4a(v.y, v.y, a2); a2 = __dp4a(v.z, v.z, a2); a2 = __dp4a(v.w, v.w, a2);
      s1 += a1;
      s2 += a2;
    }
    for (int64_t col = 16 * nv + threadIdx.x; col < W; col += blockDim.x) {
      const unsigned long long x = r[col];
      s1 += x;
      s2 += x * x;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[2 * page], s1);
    atomicAdd(&acc[2 * page + 1], s2);
  }
}

// M = sum / N, S = sqrt(max(0, sumsq / N - M^2)), in the
// oracle's order.
static __global__ void k_mean_std(const unsigned long long* acc, double* MS, int64_t n_pages, double N) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pages) return;
  const double m = __ddiv_rn((double)acc[2 * p], N);
  double v = __dsub_rn(__ddiv_rn((double)acc[2 * p + 1], N), __dmul_rn(m, m));
  if (v < 0.0) v = 0.0;
  MS[2 * p] = m;
  MS[2 * p + 1] = __dsqrt_rn(v);
}

}  // namespace abin
