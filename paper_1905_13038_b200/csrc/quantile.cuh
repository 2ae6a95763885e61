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
    // rows outside the held buffer are never needed for an output: the warm-up
    // adds row y0 - o and the first step removes it again, and for a band that
    // row lies above the held halo (o - 1 rows), so both see it as absent
    const bool row_ok = grow >= 0 && grow < p.H_global && grow >= p.buf_row0 && grow < p.buf_row0 + p.buf_rows;
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
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));  // no memory clobber: code loads may pass it
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
      asm volatile("" ::: "memory");  // the histogram reads below follow the row's reductions
      } else {
#pragma unroll 4
        for (int e = s0; e <= s1; ++e) {
          const uint2 a = c_in[e], b = c_out[e];
          atom_add(hb + a.x, a.y & 0xFFFFFFu);
          atom_add(hb + b.x, 0u - (b.y & 0xFFFFFFu));
          const int va = (int)(a.y >> 24);
          if (a.y & 0xFFFFFFu) { lo = min(lo, va); hi = max(hi, va); }
        }
        asm volatile("" ::: "memory");  // the histogram reads below follow the row's reductions
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

// G = 2 variant of the quantile kernel (MODE 0; MODE 1 = Bernsen): thread t owns the two output
// columns j = J0 + 2t and j + 1.  It keeps the full window histogram of column
// j and only the difference
//   Delta = hist(window(j+1)) - hist(window(j)) = col(j+r+1) - col(j-l+1)
// as biased bytes (128 + Delta, |Delta| <= h <= 127: never carries).  A row
// step then costs the 2w value updates of window(j) (shared by both pixels)
// plus four Delta updates, instead of 4w: the recursion of PAPER.md:172
// shared between neighbouring windows.
// Layout: the u16 bins of threads t and t + NT/2 share a word (low / high
// half), the byte deltas of threads t, t + NT/4, ... share a word, so a
// thread's increments are per-thread constants and a staged pixel's code is
// just the grey level.  The rank of each pixel is tracked as
// in k_quantile (below = #(x < Q)); both pixels' comparisons with (Qa, Qb) come
// from one subtraction of 16-bit lanes: key = (0x8000 + v) * 0x10001,
// key - (Qa | Qb << 16) has bit 15 = [v >= Qa] and bit 31 = [v >= Qb], and a
// sign-replicating byte permute turns them into 0 / 255 lane counters.
// A staged pixel is its grey level v as a u16 code, 256 for pixels outside
// the image: bin offset code * 2NT (256 = the trash row), compare key
// (0x8000 + code) * 0x10001 (256 never compares below Q).
__device__ __forceinline__ uint32_t key2(uint32_t code) { return 0x80008000u + code * 0x10001u; }
__device__ __forceinline__ uint32_t ge_lanes(uint32_t key, uint32_t qq) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x4B49;" : "=r"(r) : "r"(key - qq));  // bytes 0 / 2 = sign of bytes 1 / 3
  return r;
}

template <int NT, int MODE>
__global__ void __launch_bounds__(NT) k_quantile2(const QuantParams p) {
  extern __shared__ __align__(16) uint8_t qsm[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(qsm);                  // [257][NT/2] u16 pairs (+trash row)
  uint32_t* dlt = hist + 257 * (NT / 2);                              // [257][NT/4] biased byte quads (+trash)
  const int span = 2 * NT + p.w;                                      // staged row width
  uint16_t* codes = reinterpret_cast<uint16_t*>(dlt + 257 * (NT / 4));  // [2 buffers][in | out][span]

  const int t = threadIdx.x;
  int64_t tile = blockIdx.x;
  const int strip = (int)(tile % p.n_strips);
  tile /= p.n_strips;
  const int band = (int)(tile % p.n_bands);
  const int page = (int)(tile / p.n_bands);
  const int64_t J0 = (int64_t)strip * 2 * NT;
  const int64_t j = J0 + 2 * t;           // pixels j (a) and j + 1 (b)
  const int64_t x0 = J0 - p.l + 1;        // global column of staged element 0
  const int64_t y0 = p.row0 + (int64_t)band * p.B;
  const int nrows = (int)min((int64_t)p.B, p.row0 + p.H_out - y0);
  const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;

  for (int g = t; g < 257 * (NT / 2); g += NT) hist[g] = 0u;
  for (int g = t; g < 257 * (NT / 4); g += NT) dlt[g] = 0x80808080u;

  const bool act_a = j < p.W, act_b = j + 1 < p.W;
  const int ncol_a = (int)(min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));
  const int ncol_b = (int)(min(j + 1 + p.r, p.W - 1) - max(j + 1 - p.l, (int64_t)-1));
  const int hw_ = t % (NT / 2), hs = 16 * (t / (NT / 2));            // word column / half of my u16 bins
  const int dw_ = t % (NT / 4), ds = 8 * (t / (NT / 4));             // word column / byte of my deltas
  const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(hist + hw_));
  const uint32_t hd = static_cast<uint32_t>(__cvta_generic_to_shared(dlt + dw_));
  const uint32_t inc = 1u << hs, dinc = 1u << ds;
  // window(j) = staged [e0, e0 + w); window(j+1) = [e0 + 1, e0 + w]
  const int e0 = 2 * t, e1 = 2 * t + p.w;

  constexpr int KS = 4;  // staged elements per thread and row (span <= KS NT: checked at launch)
  auto fetch = [&](int64_t grow, int (&raw)[KS]) {
    // rows outside the held buffer are never needed for an output: the warm-up
    // adds row y0 - o and the first step removes it again, and for a band that
    // row lies above the held halo (o - 1 rows), so both see it as absent
    const bool row_ok = grow >= 0 && grow < p.H_global && grow >= p.buf_row0 && grow < p.buf_row0 + p.buf_rows;
    const uint8_t* src = img + (grow - p.buf_row0) * p.in_pitch;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int e = t + k * NT;
      const int64_t col = x0 + e;
      raw[k] = (e < span && row_ok && col >= 0 && col < p.W) ? (int)__ldg(src + col) : -1;
    }
  };
  auto store_codes = [&](uint16_t* dst, const int (&raw)[KS]) {
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int e = t + k * NT;
      if (e < span) dst[e] = (uint16_t)(raw[k] >= 0 ? raw[k] : 256);
    }
  };
  constexpr uint32_t kRow = 2 * NT;  // bytes per bin row of the u16 bins (NT/2 words); the deltas': NT
  auto atom_add = [](uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));  // no memory clobber: code loads may pass it
  };

  int Qa = 0, Qb = 0, below_a = 0, below_b = 0;
  // MODE 1: bounds on the two windows' extrema (lo <= min, hi >= max); codes
  // of pixels outside the image (256) never lower a minimum, and as c & 255 = 0
  // never raise a maximum
  int lo_a = 255, hi_a = 0, lo_b = 255, hi_b = 0;
  {  // warm-up: rows y0-o .. y0+u-1
    int raw[KS];
    fetch(y0 - p.o, raw);
    for (int64_t a = y0 - p.o; a <= y0 + p.u - 1; ++a) {
      __syncthreads();
      store_codes(codes, raw);
      __syncthreads();
      if (a + 1 <= y0 + p.u - 1) fetch(a + 1, raw);
      uint32_t mn = 256u, mx = 0u;
#pragma unroll 4
      for (int e = e0; e < e1; ++e) {
        const uint32_t c = codes[e];
        atom_add(hb + c * kRow, inc);
        if (MODE == 1) { mn = min(mn, c); mx = max(mx, c & 255u); }
      }
      atom_add(hd + codes[e1] * (uint32_t)NT, dinc);
      atom_add(hd + codes[e0] * (uint32_t)NT, 0u - dinc);

      if (MODE == 1) {
        const uint32_t ce = codes[e1];
        lo_a = min(lo_a, (int)mn);
        hi_a = max(hi_a, (int)mx);
        lo_b = min(lo_b, (int)min(mn, ce));
        hi_b = max(hi_b, (int)max(mx, ce & 255u));
      }
    }
  }
  __syncthreads();
  uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (y0 - p.row0) * p.out_pitch;
  int raw_in[KS], raw_out[KS];
  int ca_next = 0, cb_next = 0;
  if (nrows > 0) {
    fetch(y0 + p.u, raw_in);
    fetch(y0 - p.o, raw_out);
    const uint8_t* cr = img + (y0 - p.buf_row0) * p.in_pitch;
    ca_next = act_a ? (int)__ldg(cr + j) : 0;
    cb_next = act_b ? (int)__ldg(cr + j + 1) : 0;
  }
  auto cnt_a = [&](int g) { return (int)((hist[g * (NT / 2) + hw_] >> hs) & 0xFFFFu); };
  auto cnt_b = [&](int g) { return cnt_a(g) + (int)((dlt[g * (NT / 4) + dw_] >> ds) & 0xFFu) - 128; };
  // rank tracking: restore below < rho <= below + cnt(Q).  MODE 2 (low
  // quantiles: on documents the rank jumps across the empty grey levels
  // between the strokes' and the background's, row to row) loads the counts
  // of 8 bins at once once a walk is longer than one step (independent loads,
  // one latency instead of a chain).  (16-bin group counts measured slower.)
  auto walk = [&](int& Q, int& below, int rho, auto cnt) {
    if (MODE != 2) {
      while (below >= rho) {
        --Q;
        below -= cnt(Q);
      }
      for (int cq = cnt(Q); below + cq < rho; cq = cnt(Q)) {
        below += cq;
        ++Q;
      }
      return;
    }
    if (below >= rho) {
      --Q;
      below -= cnt(Q);
    }
    while (below >= rho) {  // down: remove bins Q-1, Q-2, ... while below >= rho
      int c8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) c8[k] = Q - 1 - k >= 0 ? cnt(Q - 1 - k) : 0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (below >= rho) { --Q; below -= c8[k]; }
    }
    {
      const int c0 = cnt(Q);
      if (below + c0 >= rho) return;
      below += c0;
      ++Q;
    }
    for (;;) {  // up: add bins Q, Q+1, ... while below + cnt(Q) < rho
      int c8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) c8[k] = Q + k <= 255 ? cnt(Q + k) : (1 << 20);
      bool done = false;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (!done) {
          if (below + c8[k] < rho) { below += c8[k]; ++Q; }
          else done = true;
        }
      if (done) break;
    }
  };
  for (int qq = 0; qq < nrows; ++qq, orow += p.out_pitch) {
    const int64_t i = y0 + qq;
    uint16_t* c_in = codes + (qq & 1) * 2 * span;
    uint16_t* c_out = c_in + span;
    store_codes(c_in, raw_in);
    store_codes(c_out, raw_out);
    const int Ia = ca_next, Ib = cb_next;
    __syncthreads();
    if (qq + 1 < nrows) {
      fetch(i + 1 + p.u, raw_in);
      fetch(i + 1 - p.o, raw_out);
      const uint8_t* cr = img + (i + 1 - p.buf_row0) * p.in_pitch;
      ca_next = act_a ? (int)__ldg(cr + j) : 0;
      cb_next = act_b ? (int)__ldg(cr + j + 1) : 0;
    }
    uint8_t mka = 0, mkb = 0;
    if (MODE == 1 && act_a) {
      uint32_t mn = 256u, mx = 0u;
#pragma unroll 4
      for (int e = e0; e < e1; ++e) {
        const uint32_t a = c_in[e], b = c_out[e];
        atom_add(hb + a * kRow, inc);
        atom_add(hb + b * kRow, 0u - inc);
        mn = min(mn, a);
        mx = max(mx, a & 255u);
      }
      const uint32_t ai = c_in[e1], a0 = c_in[e0], bi = c_out[e1], b0 = c_out[e0];
      atom_add(hd + ai * (uint32_t)NT, dinc);
      atom_add(hd + a0 * (uint32_t)NT, 0u - dinc);
      atom_add(hd + bi * (uint32_t)NT, 0u - dinc);
      atom_add(hd + b0 * (uint32_t)NT, dinc);
      asm volatile("" ::: "memory");  // the histogram reads below follow the row's reductions
      lo_a = min(lo_a, (int)mn);
      hi_a = max(hi_a, (int)mx);
      lo_b = min(lo_b, (int)min(mn, ai));
      hi_b = max(hi_b, (int)max(mx, ai & 255u));
      // removals may have emptied the extreme bins: walk inward (n >= 1)
      while (cnt_a(lo_a) == 0) ++lo_a;
      while (cnt_a(hi_a) == 0) --hi_a;
      mka = (p.contrast >= 0 && hi_a - lo_a < p.contrast) ? 1 : ((2 * Ia <= lo_a + hi_a) ? 0 : 1);
      if (act_b) {
        while (cnt_b(lo_b) == 0) ++lo_b;
        while (cnt_b(hi_b) == 0) --hi_b;
        mkb = (p.contrast >= 0 && hi_b - lo_b < p.contrast) ? 1 : ((2 * Ib <= lo_b + hi_b) ? 0 : 1);
      }
    } else if (MODE != 1 && act_a) {
      const uint32_t qq2 = (uint32_t)Qa | ((uint32_t)Qb << 16);
      uint32_t acc = 0;  // 16-bit lanes: 255 x (#out >= Q - #in >= Q), |.| <= 255 w < 2^15
#pragma unroll 4
      for (int e = e0; e < e1; ++e) {
        const uint32_t a = c_in[e], b = c_out[e];
        atom_add(hb + a * kRow, inc);
        atom_add(hb + b * kRow, 0u - inc);
        acc += ge_lanes(key2(b), qq2) - ge_lanes(key2(a), qq2);
      }
      // unpack the signed lanes (acc = lo + 65536 hi mod 2^32)
      const int lo = (int)(int16_t)(acc & 0xFFFFu);
      const int hi = (int)(acc - (uint32_t)lo) >> 16;
      below_a += lo / 255;  // #in < Qa - #out < Qa = #out >= Qa - #in >= Qa
      below_b += hi / 255;
      {
        const uint32_t ai = c_in[e1], a0 = c_in[e0], bi = c_out[e1], b0 = c_out[e0];
        atom_add(hd + ai * (uint32_t)NT, dinc);
        atom_add(hd + a0 * (uint32_t)NT, 0u - dinc);
        atom_add(hd + bi * (uint32_t)NT, 0u - dinc);
        atom_add(hd + b0 * (uint32_t)NT, dinc);
        // window(j+1) gains ai, b0 and loses a0, bi: [v < Qb] = 1 - (bit 31 of key - qq2)
        below_b += (int)((key2(a0) - qq2) >> 31) + (int)((key2(bi) - qq2) >> 31) -
                   (int)((key2(ai) - qq2) >> 31) - (int)((key2(b0) - qq2) >> 31);
      }
      asm volatile("" ::: "memory");  // the histogram reads below follow the row's reductions
      const int nrow = (int)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
      int rho = (int)ceil(__dmul_rn(p.q, (double)(ncol_a * nrow)));
      if (rho < 1) rho = 1;
      walk(Qa, below_a, rho, cnt_a);
      mka = (Ia <= Qa) ? 0 : 1;
      if (act_b) {
        int rb = (int)ceil(__dmul_rn(p.q, (double)(ncol_b * nrow)));
        if (rb < 1) rb = 1;
        walk(Qb, below_b, rb, cnt_b);
        mkb = (Ib <= Qb) ? 0 : 1;
      }
    }
    if (p.fmt == 0) {
      if (act_a) orow[j] = mka;
      if (act_b) orow[j + 1] = mkb;
    } else {
      // MSB-first bits; lanes 4m .. 4m+3 hold the 8 columns of one byte
      const unsigned ba = __ballot_sync(0xffffffffu, mka), bb = __ballot_sync(0xffffffffu, mkb);
      const int lt = t & 31;
      if ((lt & 3) == 0 && act_a) {
        uint32_t byte = 0;
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2)
          byte |= (((ba >> (lt + q2)) & 1u) << (7 - 2 * q2)) | (((bb >> (lt + q2)) & 1u) << (6 - 2 * q2));
        orow[j >> 3] = (uint8_t)byte;
      }
    }
    if (p.Q_out && page == 0) {  // Q, or Bernsen's midrange
      if (act_a) p.Q_out[(i - p.row0) * p.W + j] = MODE != 1 ? (double)Qa : 0.5 * (double)(lo_a + hi_a);
      if (act_b) p.Q_out[(i - p.row0) * p.W + j + 1] = MODE != 1 ? (double)Qb : 0.5 * (double)(lo_b + hi_b);
    }
  }
}

inline size_t quantile2_smem_bytes(int nt, int w) {
  const int span = 2 * nt + w;
  return (size_t)257 * (nt / 2) * 4 + (size_t)257 * (nt / 4) * 4 + 4 * (size_t)span * 2;
}

inline size_t quantile_smem_bytes(int nt, int w) {
  const int span = nt + w - 1;
  return (size_t)129 * nt * 4 + 4 * (size_t)span * 8 + 2 * (size_t)nt;
}

}  // namespace abin
