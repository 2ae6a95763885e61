// quantile.cuh -- K5: local quantile threshold by sliding histograms
// ("local quantiles such as median of gray levels can also be
// computed recursively by maintaining histograms").
//
// Q(i,j) = rho-th smallest in-bounds gray level of the window,
// rho = max(1, ceil(q n)) (SPEC sweep_quantile rank convention), and the mask
// is 0 iff I(i,j) <= Q(i,j).
//
// Design: a CTA owns a strip of NT output columns and a band of output rows;
// thread t owns output column j = J0 + t and keeps the 256-bin histogram of
// its window in shared memory (u16 bins, bin-major so that the 32 lanes of a
// warp touch 32 distinct words of one bin row).  Moving down one row removes
// the w values of row i-o and adds the w values of row i+u (the paper's
// recursion in the vertical direction); the quantile is tracked
// incrementally (Q and below = #(x < Q)), so the search after each step is a
// few bin reads.  Out-of-bounds pixels are excluded (not zero-padded).
#pragma once
#include <cstdint>
#include <cmath>

namespace abin {

struct QuantParams {
  const uint8_t* in;    // first held row (global row buf_row0) of page 0
  int64_t in_page_stride, in_pitch;
  int64_t W;
  int64_t buf_row0, buf_rows;  // held rows [buf_row0, buf_row0 + buf_rows)
  int64_t row0, H_out, H_global;
  uint8_t* out;
  int64_t out_pitch, out_page_stride;
  int32_t fmt;
  int32_t h, w, l, r, o, u;
  double q;
  int32_t B, n_bands, n_strips;
  double* Q_out;  // optional (page 0): Q per pixel as double
};

template <int NT>
__global__ void __launch_bounds__(NT) k_quantile(const QuantParams p) {
  extern __shared__ __align__(16) uint8_t qsm[];
  uint16_t* hist = reinterpret_cast<uint16_t*>(qsm);                      // [256][NT]
  uint8_t* rows = qsm + 256 * NT * sizeof(uint16_t);                       // 3 staged rows
  const int span = NT + p.w - 1;                                           // staged row width
  const int span_pad = (span + 15) & ~15;
  uint8_t* r_in = rows;
  uint8_t* r_out = rows + span_pad;
  uint8_t* r_ctr = rows + 2 * span_pad;

  const int t = threadIdx.x;
  int64_t tile = blockIdx.x;
  const int strip = (int)(tile % p.n_strips);
  tile /= p.n_strips;
  const int band = (int)(tile % p.n_bands);
  const int page = (int)(tile / p.n_bands);
  const int64_t J0 = (int64_t)strip * NT;
  const int64_t j = J0 + t;
  const int64_t x0 = J0 - p.l + 1;  // global column of staged byte 0
  const int64_t y0 = p.row0 + (int64_t)band * p.B;
  const int64_t nrows = min((int64_t)p.B, p.row0 + p.H_out - y0);
  const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;

  for (int g = 0; g < 256; ++g) hist[g * NT + t] = 0;

  // in-bounds columns of this thread's window, as staged offsets
  const int64_t cb0 = max(j - p.l + 1, (int64_t)0), cb1 = min(j + p.r, p.W - 1);
  const int s0 = (int)(cb0 - x0), s1 = (int)(cb1 - x0);  // inclusive
  const int ncol = (int)(min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));

  auto stage = [&](uint8_t* dst, int64_t grow) {
    // global row -> staged bytes, zero outside the image / held rows
    const bool row_ok = grow >= 0 && grow < p.H_global && grow >= p.buf_row0 && grow < p.buf_row0 + p.buf_rows;
    const uint8_t* src = img + (grow - p.buf_row0) * p.in_pitch;
    for (int e = t; e < span; e += NT) {
      const int64_t col = x0 + e;
      dst[e] = (row_ok && col >= 0 && col < p.W) ? src[col] : 0;
    }
  };

  int Q = 0, below = 0;  // below = #(x < Q)
  // warm-up: rows y0-o .. y0+u-1 (the first main step adds y0+u, removes y0-o)
  for (int64_t a = y0 - p.o; a <= y0 + p.u - 1; ++a) {
    __syncthreads();
    stage(r_in, a);
    __syncthreads();
    if (a >= 0 && a < p.H_global && j < p.W) {
      for (int e = s0; e <= s1; ++e) {
        const int v = r_in[e];
        hist[v * NT + t] += 1;
        below += (v < Q);
      }
    }
  }
  for (int64_t qq = 0; qq < nrows; ++qq) {
    const int64_t i = y0 + qq;
    const int64_t ain = i + p.u, aout = i - p.o;
    __syncthreads();
    stage(r_in, ain);
    stage(r_out, aout);
    stage(r_ctr, i);
    __syncthreads();
    uint8_t mk = 0;
    int Qv = 0;
    if (j < p.W) {
      if (ain >= 0 && ain < p.H_global)
        for (int e = s0; e <= s1; ++e) {
          const int v = r_in[e];
          hist[v * NT + t] += 1;
          below += (v < Q);
        }
      if (aout >= 0 && aout < p.H_global)
        for (int e = s0; e <= s1; ++e) {
          const int v = r_out[e];
          hist[v * NT + t] -= 1;
          below -= (v < Q);
        }
      const int nrow = (int)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
      const int n = ncol * nrow;
      int rho = (int)ceil(__dmul_rn(p.q, (double)n));
      if (rho < 1) rho = 1;
      // rank tracking: restore below < rho <= below + hist[Q]
      while (below >= rho) {
        --Q;
        below -= hist[Q * NT + t];
      }
      while (below + hist[Q * NT + t] < rho) {
        below += hist[Q * NT + t];
        ++Q;
      }
      const int I = r_ctr[t + p.l - 1];
      mk = (I <= Q) ? 0 : 1;
      Qv = Q;
    }
    uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (i - p.row0) * p.out_pitch;
    if (p.fmt == 0) {
      if (j < p.W) orow[j] = mk;
    } else {
      // MSB-first bits; gather the 8 lanes of each byte with a ballot
      const unsigned bal = __ballot_sync(0xffffffffu, mk);
      if ((t & 7) == 0 && j < p.W) {
        uint32_t byte = 0;
        for (int b = 0; b < 8; ++b)
          if (j + b < p.W) byte |= ((bal >> ((t & 31) + b)) & 1u) << (7 - b);
        orow[j >> 3] = (uint8_t)byte;
      }
    }
    if (p.Q_out && page == 0 && j < p.W) p.Q_out[(i - p.row0) * p.W + j] = (double)Qv;
  }
}

inline size_t quantile_smem_bytes(int nt, int w) {
  const int span = nt + w - 1;
  return (size_t)256 * nt * 2 + 3 * (size_t)((span + 15) & ~15);
}

}  // namespace abin
