// globalmin.cuh -- K4: per-page global minimum gray level L (Table 1
// notation), for Wolf's threshold.  One pass, 1 B/px read,
// result stays on the device (no host round trip).
#pragma once
#include <cstdint>

namespace abin {

// grid = (blocks_per_page, n_pages); Lw[page] must be initialised to 0xFF.
#ifndef ABIN_MIN_ROWS
#define ABIN_MIN_ROWS 2
#endif
constexpr int kMinRows = ABIN_MIN_ROWS;  // rows in flight per thread (measured: 2 beats 1, 3, 4 and 8)
__global__ void __launch_bounds__(256) k_global_min(const uint8_t* __restrict__ in, int64_t page_stride, int64_t H,
                                                    int64_t W, int64_t pitch, unsigned int* Lw) {
  const int page = blockIdx.y;
  const uint8_t* img = in + (int64_t)page * page_stride;
  unsigned int m = 0xFFu;
  const bool vec = ((reinterpret_cast<uintptr_t>(img) | (uintptr_t)pitch | (uintptr_t)W) & 15u) == 0;
  if (vec) {
    // rows round-robin over the page's blocks, 16-byte chunks across the
    // threads; kMinRows rows in flight per thread (no per-element division)
    const int64_t wq = W >> 4;  // uint4 per row
    for (int64_t row = blockIdx.x; row < H; row += kMinRows * (int64_t)gridDim.x) {
      for (int64_t c = threadIdx.x; c < wq; c += blockDim.x) {
        uint4 v[kMinRows];
#pragma unroll
        for (int k = 0; k < kMinRows; ++k) {
          const int64_t rk = row + (int64_t)k * gridDim.x;
          v[k] = rk < H ? __ldg(reinterpret_cast<const uint4*>(img + rk * pitch) + c) : make_uint4(~0u, ~0u, ~0u, ~0u);
        }
#pragma unroll
        for (int k = 0; k < kMinRows; ++k) {
          unsigned int x = __vminu4(__vminu4(v[k].x, v[k].y), __vminu4(v[k].z, v[k].w));
          x = min(min(x & 0xFFu, (x >> 8) & 0xFFu), min((x >> 16) & 0xFFu, x >> 24));
          m = min(m, x);
        }
      }
    }
  } else {
    for (int64_t row = blockIdx.x; row < H; row += gridDim.x)
      for (int64_t col = threadIdx.x; col < W; col += blockDim.x) m = min(m, (unsigned int)img[row * pitch + col]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ unsigned int red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int r = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = min(r, red[i]);
    atomicMin(&Lw[page], r);
  }
}

__global__ void k_fill_u32(unsigned int* p, int64_t n, unsigned int v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_narrow_u8(const unsigned int* src, uint8_t* dst, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (uint8_t)src[i];
}

}  // namespace abin
