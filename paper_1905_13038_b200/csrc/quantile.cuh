// quantile.cuh -- K5: local quantile threshold by sliding histograms
// ("local quantiles such as median of gray levels can also be
// computed recursively by maintaining histograms"; Θ(HW max{h,w}) time).
//
// Q(i,j) = rho-th smallest in-bounds gray level of the window,
// rho = max(1, ceil(q n)) (SPEC sweep_quantile rank convention, R10),
// and the mask is 0 iff I(i,j) <= Q(i,j).
//
// Design: a CTA owns a strip of NT output columns and a band of output rows;
// thread t owns output column j = J0 + t and the 256-bin histogram of its
// window (u16 counts, packed two bins per 32-bit word, bin-major so the
// threads of a warp touch 32 consecutive words).  Moving down one row adds the
// in-bounds values of row i+u and removes those of row i-o -- the paper's
// recursion in the vertical direction.  Per row the CTA stages both rows
// once and turns every staged pixel into a "bin code" (word offset of its
// bin, which half-word, its value), so a thread's update of one value is one
// shared-memory load of the code, an address and an increment, and one
// fire-and-forget shared atomic (no read-modify-write latency chain).
// The quantile itself is tracked incrementally: below = #(x < Q) follows every
// update, and Q moves by the few bins the row changed.  Out-of-bounds pixels
// are excluded (not zero-padded).
//
// MODE 1 is Bernsen's midrange rule: the same histograms give
// the window extrema -- the minimum / maximum are tracked from the added
// values and walked inward past emptied bins -- and the decision
// I <= (min + max) / 2 is the exact integer test 2 I <= min + max (with the
// local-contrast variant: background where max - min < contrast).
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
  double* Q_out;  // optional (page 0): Q (Bernsen: the midrange) per pixel as double
  int32_t contrast;  // Bernsen: < 0 plain midrange, else background where max - min < contrast
};

// A staged pixel's bin code (uint2): x = byte offset of its bin's word in the
// histogram block, y = (v << 24) | increment (1 or 0x10000: which half-word).
// Pixels outside the image get the trash word and v = 255, increment 0.
// Then: atomic add of (y & 0xFFFFFF) at hb + x, and  y < (Q << 24)  <=>  v < Q.
template <int NT>
__device__ __forceinline__ uint2 bin_code(uint32_t v) {
  return make_uint2((v >> 1) * (uint32_t)(NT * 4), (v << 24) | ((v & 1u) ? 0x10000u : 1u));
}
template <int NT>
__device__ __forceinline__ uint2 skip_code() {
  return make_uint2(128u * (uint32_t)(NT * 4), 255u << 24);
}

template <int NT, int MODE>
__global__ void __launch_bounds__(NT) k_quantile(const QuantParams p) {
  extern __shared__ __align__(16) uint8_t qsm[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(qsm);                        // [129][NT] packed u16 bins (+trash)
  const int span = NT + p.w - 1;                                           // staged row width
  uint2* codes = reinterpret_cast<uint2*>(hist + 129 * NT);                // [2 buffers][in | out][span]
  uint8_t* ctr = reinterpret_cast<uint8_t*>(codes + 4 * span);             // [2][NT] centre row

  const int t = threadIdx.x;
  int64_t tile = blockIdx.x;
  const int strip = (int)(tile % p.n_strips);
  tile /= p.n_strips;
  const int band = (int)(tile % p.n_bands);
  const int page = (int)(tile / p.n_bands);
  const int64_t J0 = (int64_t)strip * NT;
  const int64_t j = J0 + t;
  const int64_t x0 = J0 - p.l + 1;  // global column of staged element 0
  const int64_t y0 = p.row0 + (int64_t)band * p.B;
  const int nrows = (int)min((int64_t)p.B, p.row0 + p.H_out - y0);
  const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;

  for (int g = 0; g < 129; ++g) hist[g * NT + t] = 0u;

  // in-bounds columns of this thread's window, as staged offsets [s0, s1]
  const int64_t cb0 = max(j - p.l + 1, (int64_t)0), cb1 = min(j + p.r, p.W - 1);
  const int s0 = (int)(cb0 - x0), s1 = (int)(cb1 - x0);
  const int ncol = (int)(min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));
  const bool active = j < p.W;
  const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(hist + t));

  // Each thread stages at most KS elements of a row (span <= KS * NT).
  constexpr int KS = 4;
  // raw bytes of global row `grow` for this thread's staged elements (-1: outside the image)
  auto fetch = [&](int64_t grow, int (&raw)[KS]) {
    const bool row_ok = grow >= 0 && grow < p.H_global;
    const uint8_t* src = img + (grow - p.buf_row0) * p.in_pitch;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int e = t + k * NT;
      const int64_t col = x0 + e;
      raw[k] = (e < span && row_ok && col >= 0 && col < p.W) ? (int)__ldg(src + col) : -1;
    }
  };
  auto store_codes = [&](uint2* dst, const int (&raw)[KS]) {
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int e = t + k * NT;
      if (e < span) dst[e] = raw[k] >= 0 ? bin_code<NT>((uint32_t)raw[k]) : skip_code<NT>();
    }
  };
  auto atom_add = [](uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
  };

  int Q = 0, below = 0;  // below = #(x < Q) over the window
  int lo = 255, hi = 0;  // MODE 1: bounds on the window extrema (lo <= min, hi >= max)
  // warm-up: rows y0-o .. y0+u-1 (the first main step adds y0+u, removes y0-o)
  {
    int raw[KS];
    fetch(y0 - p.o, raw);
    for (int64_t a = y0 - p.o; a <= y0 + p.u - 1; ++a) {
      __syncthreads();
      store_codes(codes, raw);
      __syncthreads();
      if (a + 1 <= y0 + p.u - 1) fetch(a + 1, raw);  // overlaps the updates below
      if (active) {
#pragma unroll 4
        for (int e = s0; e <= s1; ++e) {
          const uint2 c = codes[e];
          atom_add(hb + c.x, c.y & 0xFFFFFFu);
          if (MODE == 1 && (c.y & 0xFFFFFFu)) { lo = min(lo, (int)(c.y >> 24)); hi = max(hi, (int)(c.y >> 24)); }
        }
      }
    }
  }
  __syncthreads();  // the warm-up's reads of buffer 0 precede the first main-row stores
  uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (y0 - p.row0) * p.out_pitch;
  int raw_in[KS], raw_out[KS];
  int ctr_next = 0;
  if (nrows > 0) {
    fetch(y0 + p.u, raw_in);
    fetch(y0 - p.o, raw_out);
    ctr_next = active ? (int)__ldg(img + (y0 - p.buf_row0) * p.in_pitch + j) : 0;
  }
  for (int qq = 0; qq < nrows; ++qq, orow += p.out_pitch) {
    const int64_t i = y0 + qq;
    uint2* c_in = codes + (qq & 1) * 2 * span;
    uint2* c_out = c_in + span;
    store_codes(c_in, raw_in);
    store_codes(c_out, raw_out);
    const int I = ctr_next;
    __syncthreads();  // codes of row i visible; (double buffer: row i-1's reads finished before row i+1's stores)
    if (qq + 1 < nrows) {  // prefetch row i+1 while the histogram updates of row i run
      fetch(i + 1 + p.u, raw_in);
      fetch(i + 1 - p.o, raw_out);
      ctr_next = active ? (int)__ldg(img + (i + 1 - p.buf_row0) * p.in_pitch + j) : 0;
    }
    uint8_t mk = 0;
    int Qv = 0;
    if (active) {
      auto cnt = [&](int g) { return (int)((hist[(g >> 1) * NT + t] >> ((g & 1) << 4)) & 0xFFFFu); };
      if (MODE == 0) {
      const uint32_t qk = (uint32_t)Q << 24;  // y < qk  <=>  v < Q
      int dbelow = 0;
#pragma unroll 4
      for (int e = s0; e <= s1; ++e) {
        const uint2 a = c_in[e], b = c_out[e];
        atom_add(hb + a.x, a.y & 0xFFFFFFu);
        atom_add(hb + b.x, 0u - (b.y & 0xFFFFFFu));
        dbelow += (int)(a.y < qk) - (int)(b.y < qk);
      }
      below += dbelow;
      } else {
#pragma unroll 4
        for (int e = s0; e <= s1; ++e) {
          const uint2 a = c_in[e], b = c_out[e];
          atom_add(hb + a.x, a.y & 0xFFFFFFu);
          atom_add(hb + b.x, 0u - (b.y & 0xFFFFFFu));
          const int va = (int)(a.y >> 24);
          if (a.y & 0xFFFFFFu) { lo = min(lo, va); hi = max(hi, va); }
        }
        // removals may have emptied the extreme bins: walk inward (n >= 1)
        while (cnt(lo) == 0) ++lo;
        while (cnt(hi) == 0) --hi;
        if (p.contrast >= 0 && hi - lo < p.contrast) mk = 1;  // low local contrast: background
        else mk = (2 * I <= lo + hi) ? 0 : 1;
        if (p.Q_out && page == 0) p.Q_out[(i - p.row0) * p.W + j] = 0.5 * (double)(lo + hi);
      }
      if (MODE == 0) {
      const int nrow = (int)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
      const int n = ncol * nrow;
      int rho = (int)ceil(__dmul_rn(p.q, (double)n));
      if (rho < 1) rho = 1;
      // rank tracking: restore below < rho <= below + count(Q)
      while (below >= rho) {
        --Q;
        below -= cnt(Q);
      }
      for (int cq = cnt(Q); below + cq < rho; cq = cnt(Q)) {
        below += cq;
        ++Q;
      }
      mk = (I <= Q) ? 0 : 1;
      Qv = Q;
      }
    }
    if (p.fmt == 0) {
      if (active) orow[j] = mk;
    } else {
      // MSB-first bits; gather the 8 lanes of each byte with a ballot
      const unsigned bal = __ballot_sync(0xffffffffu, mk);
      if ((t & 7) == 0 && active) {
        uint32_t byte = 0;
        for (int b = 0; b < 8; ++b)
          if (j + b < p.W) byte |= ((bal >> ((t & 31) + b)) & 1u) << (7 - b);
        orow[j >> 3] = (uint8_t)byte;
      }
    }
    if (MODE == 0 && p.Q_out && page == 0 && active) p.Q_out[(i - p.row0) * p.W + j] = (double)Qv;
  }
}

inline size_t quantile_smem_bytes(int nt, int w) {
  const int span = nt + w - 1;
  return (size_t)129 * nt * 4 + 4 * (size_t)span * 8 + 2 * (size_t)nt;
}

}  // namespace abin
