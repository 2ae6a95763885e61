// otsu.cuh -- Otsu's global threshold (the paper's speed
// comparator), NEXT #4 of SURVEY section 8(f).
//   1. k_otsu_hist: exact 256-bin histogram of each page (warp-private
//      shared-memory sub-histograms, merged with 64-bit global atomics);
//   2. k_otsu_pick: one block per page, thread t evaluates the between-class
//      variance w0 w1 (mu0 - mu1)^2 of split t in IEEE double from exact
//      prefix sums; the argmax keeps the smallest t among ties (the oracle's);
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

// one 256-thread block per page: thread t evaluates the split t.  N0(t), S0(t)
// are exact integer prefix sums (a block scan: order-independent), the
// between-class variance of each t is the oracle's IEEE double sequence, and
// the block argmax keeps the smallest t among equal maxima -- the oracle's
// sequential "if (sb > best)" -- so t is bit-identical.
static __global__ void __launch_bounds__(256) k_otsu_pick(const unsigned long long* hist, uint8_t* t_out,
                                                          int64_t n_pages, double N) {
  __shared__ unsigned long long sn[256], ss[256];
  __shared__ double bsb[8];
  __shared__ int bt[8];
  const int64_t p = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const unsigned long long ht = hist[p * 256 + t];
  sn[t] = ht;
  ss[t] = (unsigned long long)t * ht;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {  // inclusive Hillis-Steele scan
    const unsigned long long a = t >= off ? sn[t - off] : 0ull, b = t >= off ? ss[t - off] : 0ull;
    __syncthreads();
    sn[t] += a;
    ss[t] += b;
    __syncthreads();
  }
  const unsigned long long Nt = sn[255], Stot = ss[255];
  const unsigned long long N0 = sn[t], S0 = ss[t], N1 = Nt - N0, S1 = Stot - S0;
  double sb = 0.0;
  if (N0 > 0 && N1 > 0) {
    const double w0 = __ddiv_rn((double)N0, N), w1 = __ddiv_rn((double)N1, N);
    const double mu0 = __ddiv_rn((double)S0, (double)N0), mu1 = __ddiv_rn((double)S1, (double)N1);
    const double d = __dsub_rn(mu0, mu1);
    sb = __dmul_rn(__dmul_rn(w0, w1), __dmul_rn(d, d));
  }
  // argmax, ties -> smallest t (the sequential scan starts from best = -1, so
  // t = 0 wins when every sb is 0)
  double v = sb;
  int vt = t;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, v, off);
    const int ot = __shfl_down_sync(0xffffffffu, vt, off);
    if (ov > v || (ov == v && ot < vt)) { v = ov; vt = ot; }
  }
  if (lane == 0) { bsb[warp] = v; bt[warp] = vt; }
  __syncthreads();
  if (t == 0) {
    double best = bsb[0];
    int tb = bt[0];
    for (int k = 1; k < 8; ++k)
      if (bsb[k] > best || (bsb[k] == best && bt[k] < tb)) { best = bsb[k]; tb = bt[k]; }
    t_out[p] = (uint8_t)tb;
  }
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
