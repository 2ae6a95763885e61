// otsu.cuh -- Otsu's global threshold (the paper's speed
// comparator), NEXT #4 of SURVEY section 8(f).
//   1. k_otsu_hist: exact 256-bin histogram of each page (warp-private
//      shared-memory sub-histograms, merged with 64-bit global atomics);
//   2. k_otsu_pick: one thread per page scans t = 0..255 for the maximum of
//      the between-class variance w0 w1 (mu0 - mu1)^2 in IEEE double, in the
//      oracle's order (ties keep the smallest t);
//   3. k_otsu_mask: I' = 0 iff I <= t (byte or MSB-first bit mask).
#pragma once
#include <cstdint>

namespace abin {

// grid = (blocks_per_page, n_pages), 256 threads; hist: [n_pages][256] u64 zeroed
static __global__ void __launch_bounds__(256) k_otsu_hist(const uint8_t* __restrict__ in, int64_t page_stride,
                                                          int64_t H, int64_t W, int64_t pitch,
                                                          unsigned long long* hist) {
  __shared__ unsigned int sh[8][256];
  const int warp = threadIdx.x >> 5;
  for (int g = threadIdx.x; g < 8 * 256; g += 256) (&sh[0][0])[g] = 0;
  __syncthreads();
  const uint8_t* img = in + (int64_t)blockIdx.y * page_stride;
  const bool vec = ((reinterpret_cast<uintptr_t>(img) | (uintptr_t)pitch) & 3u) == 0;
  for (int64_t row = blockIdx.x; row < H; row += gridDim.x) {
    const uint8_t* r = img + row * pitch;
    if (vec) {
      const int64_t wq = W >> 2;
      for (int64_t c = threadIdx.x; c < wq; c += blockDim.x) {
        const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(r) + c);
        atomicAdd(&sh[warp][v & 0xFF], 1u);
        atomicAdd(&sh[warp][(v >> 8) & 0xFF], 1u);
        atomicAdd(&sh[warp][(v >> 16) & 0xFF], 1u);
        atomicAdd(&sh[warp][v >> 24], 1u);
      }
      for (int64_t c = (wq << 2) + threadIdx.x; c < W; c += blockDim.x) atomicAdd(&sh[warp][r[c]], 1u);
    } else {
      for (int64_t c = threadIdx.x; c < W; c += blockDim.x) atomicAdd(&sh[warp][r[c]], 1u);
    }
  }
  __syncthreads();
  const int g = threadIdx.x;
  unsigned long long s = 0;
  for (int k = 0; k < 8; ++k) s += sh[k][g];
  if (s) atomicAdd(&hist[(int64_t)blockIdx.y * 256 + g], s);
}

static __global__ void k_otsu_pick(const unsigned long long* hist, uint8_t* t_out, int64_t n_pages, double N) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pages) return;
  const unsigned long long* h = hist + p * 256;
  unsigned long long Stot = 0;
  for (int g = 0; g < 256; ++g) Stot += (unsigned long long)g * h[g];
  const unsigned long long Nt = (unsigned long long)N;
  unsigned long long N0 = 0, S0 = 0;
  double best = -1.0;
  int tbest = 0;
  for (int t = 0; t < 256; ++t) {
    N0 += h[t];
    S0 += (unsigned long long)t * h[t];
    const unsigned long long N1 = Nt - N0, S1 = Stot - S0;
    double sb = 0.0;
    if (N0 > 0 && N1 > 0) {
      const double w0 = __ddiv_rn((double)N0, N), w1 = __ddiv_rn((double)N1, N);
      const double mu0 = __ddiv_rn((double)S0, (double)N0), mu1 = __ddiv_rn((double)S1, (double)N1);
      const double d = __dsub_rn(mu0, mu1);
      sb = __dmul_rn(__dmul_rn(w0, w1), __dmul_rn(d, d));
    }
    if (sb > best) {
      best = sb;
      tbest = t;
    }
  }
  t_out[p] = (uint8_t)tbest;
}

// grid = (blocks_per_page, n_pages); one output byte per pixel (fmt 0) or bit (fmt 1)
static __global__ void __launch_bounds__(256) k_otsu_mask(const uint8_t* __restrict__ in, int64_t page_stride,
                                                          int64_t H, int64_t W, int64_t pitch, const uint8_t* tpage,
                                                          uint8_t* out, int64_t out_pitch, int64_t out_page_stride,
                                                          int32_t fmt) {
  const int64_t page = blockIdx.y;
  const int t = tpage[page];
  const uint8_t* img = in + page * page_stride;
  uint8_t* o = out + page * out_page_stride;
  for (int64_t row = blockIdx.x; row < H; row += gridDim.x) {
    const uint8_t* r = img + row * pitch;
    uint8_t* orow = o + row * out_pitch;
    if (fmt == 0) {
      for (int64_t c = threadIdx.x; c < W; c += blockDim.x) orow[c] = r[c] > t ? 1 : 0;
    } else {
      for (int64_t b = threadIdx.x; b < (W + 7) / 8; b += blockDim.x) {
        uint32_t byte = 0;
        for (int k = 0; k < 8; ++k) {
          const int64_t c = 8 * b + k;
          if (c < W && r[c] > t) byte |= 0x80u >> k;
        }
        orow[b] = (uint8_t)byte;
      }
    }
  }
}

}  // namespace abin
