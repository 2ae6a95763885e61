// globalmin.cuh -- K4: per-page global minimum gray level L (Table 1
// notation), for Wolf's threshold.  One pass, 1 B/px read,
// result stays on the device (no host round trip).
#pragma once
#include <cstdint>

namespace abin {

// grid = (blocks_per_page, n_pages); Lw[page] must be initialised to 0xFF.
__global__ void __launch_bounds__(256) k_global_min(const uint8_t* __restrict__ in, int64_t page_stride, int64_t H,
                                                    int64_t W, int64_t pitch, unsigned int* Lw) {
  const int page = blockIdx.y;
  const uint8_t* img = in + (int64_t)page * page_stride;
  unsigned int m = 0xFFu;
  const bool vec = ((reinterpret_cast<uintptr_t>(img) | (uintptr_t)pitch | (uintptr_t)W) & 15u) == 0;
  if (vec) {
    const int64_t wq = W >> 4;  // uint4 per row
    const int64_t nq = H * wq;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nq; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t row = e / wq, col = e - row * wq;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(img + row * pitch) + col);
      unsigned int x = __vminu4(__vminu4(v.x, v.y), __vminu4(v.z, v.w));
      x = min(min(x & 0xFFu, (x >> 8) & 0xFFu), min((x >> 16) & 0xFFu, x >> 24));
      m = min(m, x);
    }
  } else {
    const int64_t n = H * W;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t row = e / W, col = e - row * W;
      m = min(m, (unsigned int)img[row * pitch + col]);
    }
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
