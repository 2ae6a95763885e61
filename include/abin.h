/*
 * abin.h -- C ABI of libabin.so, the B200 (sm_100a) hot path of
 * Chan, "Memory-efficient and fast implementation of local adaptive
 * binarization methods", arXiv 1905.13038.
 *
 * What every binarization entry point computes (the paper's definitions):
 *
 *   window      rows (i-o, i+u], cols (j-l, j+r] with
 *               l = floor((w+1)/2), r = floor(w/2), o = floor((h+1)/2),
 *               u = floor(h/2)                      -- Alg. 1 l.1-4
 *   sums        c = sum I, d = sum I^2 over the in-bounds part of the window
 *               (undefined elements are zero)      -- PAPER.md:27, 83
 *   count       n = (min{j+r,W-1} - max{j-l,-1}) * (min{i+u,H-1} - max{i-o,-1})
 *                                                   -- Alg. 1 l.118
 *   moments     m = c/n, v = d/n - m^2 (clamped at 0), s = sqrt(v)
 *                                                   -- Alg. 1 l.121-122
 *   threshold   Sauvola t = m (1 + k (s/R - 1))     -- PAPER.md:24, Table 1 (l.152)
 *               Niblack t = m + k s                 -- Table 1
 *               Wolf    t = m - k (m - L)(1 - s/R), L = global minimum
 *                                                   -- Table 1
 *   decision    I' = 0 (foreground) if I <= t, else 1 -- Alg. 1 l.124
 *
 * t is evaluated in IEEE double, left to right, with no FMA contraction, so
 * the mask is bit-identical to a plain CPU evaluation of the same formula.
 * (The kernels decide most pixels with a certified fp32 bound and re-evaluate
 * the ambiguous ones in that exact double sequence.)
 *
 * abin_quantile computes, per pixel, Q = the rho-th smallest in-bounds gray
 * level of the window, rho = max(1, ceil(q n)), and I' = 0 iff I <= Q
 * (local quantiles via sliding histograms).
 *
 * Conventions shared by all entry points
 * -------------------------------------
 * - Images are uint8, row-major, `H` rows of `W` pixels, rows `pitch` bytes
 *   apart (pitch >= W).  Page batches place page p at `in + p*in_page_stride`.
 *   When the base, pitch and page stride are multiples of 16 bytes the rows are
 *   staged by TMA in whole 16-byte chunks: the bytes of a row's last partial
 *   chunk (columns W .. ceil(W/16)*16 - 1, inside the pitch) must be readable;
 *   their values are ignored.  Otherwise the moments entry points first copy
 *   the pages into a 16-byte aligned scratch buffer (one 2-D device copy).
 * - Scratch.  SURVEY section 8(b) asked for no O(HW) scratch; the library
 *   keeps that for the aligned production path and departs from it, on
 *   purpose, in three places.  All temporary device memory comes from the
 *   device's default stream-ordered pool (cudaMallocAsync) and is returned on
 *   the same stream; the pool's release threshold is raised to 512 MB so it is
 *   reused across calls instead of re-mapped.
 *     O(1) per call (the aligned production path): per-page minima / sums
 *       (a few bytes per page), the exact-fixup queue -- 16 B per output
 *       lane-row (16 pixels), capped at 64 MB; calls that could exceed the cap
 *       take the exact follow-up kernel instead of growing it.
 *     O(HW) (documented departures): (1) rows TMA cannot stage (base, pitch or
 *       page stride not a multiple of 16 bytes) are re-pitched into a
 *       temporary copy of ceil16(W) x H bytes per page -- about half the
 *       kernel's own traffic, 10x faster than the generic row loader, which
 *       remains the fallback when the pool cannot supply the copy;
 *       (2) ABIN_HOST_IO staging: up to 4 chunks of ~64 MB (pages, or row
 *       bands with halos for larger pages); (3) abin_stats: one H x W mask
 *       for the quantile / Bernsen paths (a debug entry point).
 * - All image / mask pointers are DEVICE pointers (cudaMalloc'd or torch CUDA
 *   tensors) unless the flag ABIN_HOST_IO is given (abin_*_batched only): then
 *   `in` and `out` are HOST pointers (pinned memory recommended) and the
 *   library streams pages through device staging buffers it owns.
 * - The caller owns every buffer.  Input and output must not overlap
 *   (the in-place variant is out of scope) -> ABIN_EALIAS.
 * - Output mask formats: ABIN_MASK_U8: one byte per pixel, value 0 or 1,
 *   row stride out_pitch >= W.  ABIN_MASK_BITS: one bit per pixel,
 *   MSB-first (pixel j -> byte j>>3, bit 7-(j&7)), bit = I', rows padded with
 *   0 bits to whole bytes, out_pitch >= ceil(W/8).
 * - Work is enqueued asynchronously on `stream` (a cudaStream_t; NULL = the
 *   legacy default stream).  The call returns once the work is enqueued;
 *   asynchronous device faults surface at the caller's next synchronisation.
 *   Entry points are reentrant across streams.
 * - `counters` (optional, device pointer to 2 x uint64, may be NULL):
 *   counters[0] += pixels with |I - t| < 1e-9 ("near ties"),
 *   counters[1] += pixels the certified fp32 filter sent to the exact fp64
 *   path.  Accumulated with device atomics; the caller zeroes them.
 * - Windows: any h, w >= 1 are legal, including windows larger than the
 *   image (SPEC window-geometry); even sizes are asymmetric per the floors.
 *
 * Error behaviour: every entry point validates its arguments before touching
 * the device and returns one of abin_status; nothing is enqueued on error.
 */
#ifndef ABIN_H
#define ABIN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ABIN_VERSION_MAJOR 0
#define ABIN_VERSION_MINOR 2

typedef enum {
  ABIN_OK = 0,
  ABIN_EINVAL = 1, /* null pointer, H/W/h/w < 1, pitch too small, non-finite k/R, R <= 0, q not in (0,1], bad format */
  ABIN_EALIAS = 2, /* input and output byte ranges overlap */
  ABIN_ERANGE = 3, /* window or image exceeds what the kernels support (see abin_limits) */
  ABIN_ECUDA = 4,  /* a CUDA runtime call or launch failed */
  ABIN_ENOMEM = 5  /* ABIN_HOST_IO staging allocation failed */
} abin_status;

enum { ABIN_MASK_U8 = 0, ABIN_MASK_BITS = 1 };

enum {
  ABIN_FORCE_U64_SQ = 1u << 0, /* accumulate window square sums d in uint64 even when uint32 is exact */
  ABIN_FORCE_FP64 = 1u << 1,   /* skip the fp32 filter: every pixel takes the exact fp64 sequence */
  ABIN_HOST_IO = 1u << 2,      /* (batched calls) in/out are host pointers; copies are part of the call */
  ABIN_COUNT_STAGES = 1u << 3  /* `counters` has 3 entries; counters[2] += pixels the fp32 filter re-examined
                                  from the exact integers (stage 2) */
};

/* ---- Sauvola (Table 1) --------------------------------------
 * in        device uint8 image, H x W, row pitch in_pitch bytes
 * out       device mask, row pitch out_pitch bytes, format mask_format
 * h, w      window height / width (>= 1)
 * k, R      Sauvola parameters (finite; R > 0).  The paper uses k = 0.5, R = 128.
 */
int abin_sauvola(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                 int32_t mask_format, int32_t h, int32_t w, double k, double R, uint32_t flags,
                 uint64_t* counters, void* stream);

/* ---- Niblack (Table 1); k may be negative (e.g. -0.2) ------- */
int abin_niblack(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                 int32_t mask_format, int32_t h, int32_t w, double k, uint32_t flags, uint64_t* counters,
                 void* stream);

/* ---- Wolf (Table 1) ------------------------------------------
 * L_override < 0: L is the page's global minimum gray level, computed on the
 * device (abin_global_min) without a host round trip.  L_override in 0..255
 * uses that value (band mode: pass the minimum over the WHOLE image). */
int abin_wolf(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
              int32_t mask_format, int32_t h, int32_t w, double k, double R, int32_t L_override, uint32_t flags,
              uint64_t* counters, void* stream);

/* ---- Wolf with the image-adaptive dynamic range (NEXT #3) ------------------
 * PAPER.md:153 gives Wolf's rule with R; Wolf et al. take R = the maximum of
 * s over the image (a "two-pass mode").  R = max over the
 * page of s (each s by the canonical double sequence), or +inf when every
 * window is constant (then s / R = 0: DESIGN.md reading R21); then Wolf with
 * that R (and L as abin_wolf).  The mask equals the oracle's bit for bit.
 * Synchronises `stream` once (R is read back to the host); *R_out (host,
 * optional) receives R.  Windows within the v5 kernel's domain (abin_max_s). */
int abin_wolf_adaptive(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                       int32_t mask_format, int32_t h, int32_t w, double k, int32_t L_override, uint32_t flags,
                       uint64_t* counters, double* R_out, void* stream);

/* Max of s over a band's own rows [row0, row0 + H_band) of an image of height
 * H_global (band geometry as abin_binarize_band: `in` points at the first held
 * row, global row row0 - halo_top, and the halos hold the rows the windows
 * reach; a whole image is row0 = 0, H_global = H_band, halos 0).  Exact: the
 * canonical double s of the maximising pixel (the fp32 filter's variance
 * selects the candidates within twice its certified error, k_fixup evaluates
 * them exactly).  *max_s (host) receives the value; synchronises `stream`.
 * ABIN_ERANGE outside the v5 kernel's window domain (h <= 129, w <= 127) or
 * for rows TMA cannot stage (base / pitch not multiples of 16) beyond the
 * re-pitch copy.  The multi-GPU driver all-reduces it (MAX) over the bands. */
int abin_max_s(const uint8_t* in, int64_t H_band, int64_t W, int64_t in_pitch, int64_t row0, int64_t H_global,
               int32_t halo_top, int32_t halo_bot, int32_t h, int32_t w, double* max_s, void* stream);

/* ---- Local quantile threshold -------------------------------
 * q in (0, 1]: Q = rho-th smallest in-bounds level, rho = max(1, ceil(q n)).
 * q = 0.5 is the (lower) local median. */
int abin_quantile(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                  int32_t mask_format, int32_t h, int32_t w, double q, uint32_t flags, void* stream);

/* ---- Bernsen's midrange rule ----------------------------------
 * min, max = extrema of the in-bounds gray levels of the window; I' = 0 iff
 * I <= (min + max) / 2 (exact integer test 2 I <= min + max).  contrast >= 0
 * selects the local-contrast variant (same paragraph: "estimate local contrast
 * by range of gray levels"): I' = 1 where max - min < contrast.  Work per pixel
 * is independent of h and w (the paragraph's Theta(HW)): separable running
 * extrema by van Herk / Gil-Werman block prefix / suffix extrema, a row pass
 * then a column pass with the decision.  Scratch: 4
 * bytes per pixel from the stream-ordered pool (the row pass's (min, max)
 * pairs and the column pass's suffix pairs), freed stream-ordered;
 * ABIN_ENOMEM if it cannot be had.  ABIN_ERANGE beyond
 * abin_limits().bernsen_max_window_w. */
int abin_bernsen(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                 int32_t mask_format, int32_t h, int32_t w, int32_t contrast, uint32_t flags, void* stream);

/* ---- The remaining Table 1 rows ---------------------------
 * rule and params (host array, n_params >= the count below):
 *   ABIN_FENG        {a1, k1, k2, gamma, R}: t = a1 m + k1 (s/R)^(1+gamma) (m - L) + k2 (s/R)^gamma L,
 *                    L = the page's global minimum (computed on the device)
 *   ABIN_RAIS        {}: t = m + 0.3 (m s - M S) / max{m s, M S} s, M / S = the page's global mean /
 *                    standard deviation (computed on the device); 0/0 -> 0
 *   ABIN_KHURSHID    {k, N_mode}: t = m + k sqrt(s^2 + m^2 (N - 1)/N), N = h w (N_mode = 0) or the
 *                    clamped count n (N_mode != 0)
 *   ABIN_PHANSALKAR  {k, R, p, q}: t = m (1 + p e^(-q m) + k (s/R - 1))
 * The mask is the IEEE-double decision of every pixel (left-to-right
 * evaluation; pow/exp are the device's double routines, <= 2 ulp).  Within
 * h <= 129, w <= 127, Khurshid, Phansalkar with q >= 0, Rais and Feng with
 * gamma >= 1 take the v5 kernel's exact integer window sums and certified
 * fp32 filter (a bound on the fp32 residual derived per parameter set -- for
 * Rais per page, from its M S -- DESIGN.md section 5) and decide in double
 * only the pixels inside the bound: the same mask.  Feng with gamma < 1,
 * Phansalkar with q < 0 and larger windows run the v3 kernel (double for
 * every pixel).  ABIN_EINVAL
 * for an unknown rule, missing or non-finite params, R <= 0. */
int abin_binarize_rule(int32_t rule, const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out,
                       int64_t out_pitch, int32_t mask_format, int32_t h, int32_t w, const double* params,
                       int32_t n_params, uint32_t flags, uint64_t* counters, void* stream);

/* ---- Otsu's global threshold (the paper's speed comparator)
 * t = the gray level maximising the between-class variance w0 w1 (mu0 - mu1)^2 of
 * the page histogram (IEEE double, ties keep the smallest t); I' = 0 iff I <= t.
 * t_out: optional device byte receiving t. */
int abin_otsu(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
              int32_t mask_format, uint8_t* t_out, uint32_t flags, void* stream);

/* ---- Page batches ------------------------------------------------------------
 * n_pages pages of identical H x W geometry; page p is read at
 * in + p * in_page_stride and written at out + p * out_page_stride (bytes).
 * method: 0 Sauvola, 1 Niblack, 2 Wolf (per-page L unless L_override >= 0),
 * 3 quantile (param0 = q), 4 Bernsen (param0 = contrast, < 0: plain midrange).
 * param0 = k (or q, contrast), param1 = R.
 * With ABIN_HOST_IO, in/out are host pointers. */
enum { ABIN_SAUVOLA = 0, ABIN_NIBLACK = 1, ABIN_WOLF = 2, ABIN_QUANTILE = 3, ABIN_BERNSEN = 4 };
enum { ABIN_FENG = 5, ABIN_RAIS = 6, ABIN_KHURSHID = 7, ABIN_PHANSALKAR = 8 };
int abin_binarize_batched(int32_t method, const uint8_t* in, int64_t in_page_stride, uint8_t* out,
                          int64_t out_page_stride, int64_t n_pages, int64_t H, int64_t W, int64_t in_pitch,
                          int64_t out_pitch, int32_t mask_format, int32_t h, int32_t w, double param0,
                          double param1, int32_t L_override, uint32_t flags, uint64_t* counters, void* stream);

/* ---- Row bands of a larger image (multi-GPU row decomposition) --------------
 * The caller holds rows [row0 - halo_top, row0 + H_band + halo_bot) of an
 * image that is H_global rows tall; `in` points at the first held row
 * (global row row0 - halo_top).  Output rows are the band's own rows
 * [row0, row0 + H_band); `out` points at the mask row of global row row0.
 * n and the image-edge convention use the GLOBAL geometry, so the union of
 * all bands' masks equals the whole-image mask bit for bit, provided
 * halo_top >= min(o - 1, row0) and halo_bot >= min(u, H_global - row0 - H_band)
 * (else ABIN_EINVAL).  Wolf needs the global minimum: L_override >= 0 required. */
int abin_binarize_band(int32_t method, const uint8_t* in, int64_t H_band, int64_t W, int64_t in_pitch,
                       int64_t row0, int64_t H_global, int32_t halo_top, int32_t halo_bot, uint8_t* out,
                       int64_t out_pitch, int32_t mask_format, int32_t h, int32_t w, double param0,
                       double param1, int32_t L_override, uint32_t flags, uint64_t* counters, void* stream);

/* ---- Global minimum L (Table 1 notation) ----------------------
 * L_out: device uint8[n_pages], the minimum gray level of each page. */
int abin_global_min(const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t H, int64_t W,
                    int64_t in_pitch, uint8_t* L_out, void* stream);

/* ---- Per-pixel statistics (parity / debugging) -------------------------------
 * Same kernels as the binarization path, additionally storing, per pixel
 * (row-major, H*W elements each, device pointers, any may be NULL):
 *   c_out, d_out  uint64 window sums;   n_out uint32 count;
 *   t_out         double threshold (the exact fp64 sequence, every pixel);
 *   mask_out      uint8 mask (ABIN_MASK_U8 layout, pitch W).
 * method 0..2 as above (L_override as for Wolf).  For method 3 (quantile)
 * t_out receives Q as a double, for method 4 (Bernsen) the midrange
 * (min + max) / 2; c_out/d_out/n_out are not written for methods 3, 4. */
int abin_stats(int32_t method, const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, int32_t h, int32_t w,
               double param0, double param1, int32_t L_override, uint64_t* c_out, uint64_t* d_out,
               uint32_t* n_out, double* t_out, uint8_t* mask_out, void* stream);

/* ---- Test hook: the certified fp32 filter -----------
 * Evaluates the production kernel's fp32 residual e~ = I - t~ (the device
 * function residual_pair of moments5.cuh, shared with the kernel) for `count`
 * tuples of exact window data: c = sum of I, d = sum of I^2 (c < 2^23,
 * d < 2^32), ncol, nrow the window's column / row counts (n = ncol nrow,
 * PAPER.md:118), I the centre pixel -- all device arrays of `count` entries;
 * e_out (device, count floats) receives e~, s_out (optional) s~.  method is
 * 0..2 (Sauvola, Niblack, Wolf with global minimum L; rule_params unused, may
 * be NULL) or the v5 rules 7 (Khurshid: rule_params = {k, N_mode, h w}) and
 * 8 (Phansalkar: rule_params = {k, R, p, q}, q >= 0; k, R arguments unused);
 * ABIN_ERANGE for a rule parameter set the v5 kernel does not take (those run
 * on the exact path).  bounds (optional, host, 5 doubles) receives the
 * certified bound: [0] the coarse bound the kernel tests |e~| against,
 * [1..4] rb0, rb1, rdv, rsdv of the data-dependent bound
 * rb0 + rb1 min(rsdv, rdv / s~) (used for Niblack and Khurshid).  The claim
 * the tests check: |e~ - e*| <= bound for the exact e* = I - t(c, d, n).
 * Asynchronous on `stream`; ABIN_EINVAL on bad arguments. */
int abin_probe_filter(int32_t method, double k, double R, double L, const double* rule_params, const uint32_t* c,
                      const uint32_t* d, const uint32_t* ncol, const uint32_t* nrow, const uint8_t* I, int64_t count,
                      float* e_out,
                      float* s_out, double* bounds, void* stream);

/* ---- Limits, versions, errors ------------------------------------------------ */
/* Effective windows are (min(l,W) + min(r,W)) x (min(o,H) + min(u,H))
 * (PAPER.md:94-97 clamped to the image: same in-bounds window, same n); a call
 * beyond these limits returns ABIN_ERANGE before touching the device. */
typedef struct {
  int64_t max_window_w;          /* Sauvola / Niblack / Wolf / Table-1 rules: effective width */
  int64_t max_window_h;          /*   effective height (255^2 h < 2^32: column square sums in uint32) */
  int64_t max_window_hw;         /*   255 h w < 2^32 (window sums of I in uint32) */
  int64_t max_dim;               /* largest H or W, every method */
  int64_t quantile_max_window_w; /* quantile (and abin_stats of Bernsen): effective width */
  int64_t quantile_max_window_hw;/*   h w <= 65535 (16-bit histogram bins) */
  int64_t bernsen_max_window_w;  /* Bernsen masks: effective width (any height) */
} abin_limits_t;
void abin_limits(abin_limits_t* out);
const char* abin_strerror(int status);
const char* abin_version(void);
/* Last CUDA error string recorded by a failing call on this thread ("" if none). */
const char* abin_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ABIN_H */
