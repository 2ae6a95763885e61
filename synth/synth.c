/*
 * synth.c -- seeded synthetic document pages (input generator only).
 *
 * Shared by the oracle side (tests) and the product side (bench inputs); it
 * holds NONE of the method's arithmetic (no window sums, no thresholds):
 * it only draws the pixels of the BASELINE.json workloads.
 *
 * Recipe (BASELINE.json configs):
 *   background  g(j) = 150 + 80 j / (W-1)   (left->right illumination gradient)
 *   noise       sigma = 8 approx-Gaussian: Irwin-Hall sum of 12 u16 uniforms
 *               drawn from a counter-based SplitMix64 stream keyed by
 *               (seed, pixel index): z = (S - 393210) / 65536, noise = 8 z
 *               (exact in double; no libm => bit-reproducible everywhere)
 *   rounding    nearest, ties to even (rint), clamp to 0..255
 *   strokes     axis-aligned rectangles painted over the noisy background,
 *               horizontal/vertical p=1/2, thickness U{2..6}, length U{5..40},
 *               top-left uniform on the page (clipped at the edges),
 *               flat value U{20..60}; strokes are added until the union covers
 *               >= ceil(0.10 H W) pixels
 *   stain       (optional, config 3) radial Gaussian darkening
 *               -80 exp(-r^2 / (2 sb^2)), centre uniform on the page,
 *               sb uniform in [min(H,W)/8, min(H,W)/4], applied to every pixel
 *               after the strokes, then rounded/clamped.  Evaluated as the
 *               product of the two separable factors exp(-di^2/2sb^2) *
 *               exp(-dj^2/2sb^2) (tabulated per row / per column).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static inline uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline double clamp255(double x) { return x < 0.0 ? 0.0 : (x > 255.0 ? 255.0 : x); }

/* Background + noise for one pixel, as a double (before rounding). */
static inline double bg_noise(uint64_t key, int64_t H, int64_t W, int64_t i, int64_t j) {
  (void)H;
  double g = (W > 1) ? 150.0 + (80.0 * (double)j) / (double)(W - 1) : 150.0;
  uint64_t p = (uint64_t)(i * W + j) * 3ULL;
  uint64_t S = 0;
  for (int k = 0; k < 3; ++k) {
    uint64_t r = sm64(key + p + (uint64_t)k);
    S += (r & 0xFFFF) + ((r >> 16) & 0xFFFF) + ((r >> 32) & 0xFFFF) + (r >> 48);
  }
  double z = ((double)(int64_t)S - 393210.0) / 65536.0;
  return g + 8.0 * z;
}

/* Generate one page into out (row pitch `pitch` bytes).  Returns 0, or -1 on
 * allocation failure.  `stain` != 0 adds the config-3 stain blob. */
int synth_page(uint64_t seed, int64_t H, int64_t W, int32_t stain, uint8_t *out, int64_t pitch) {
  uint64_t key = sm64(seed ^ 0x4E4F495345ULL); /* "NOISE" */
  /* stroke values are painted into a side buffer; 0 = no stroke */
  uint8_t *ink = (uint8_t *)calloc((size_t)(H * W), 1);
  if (!ink) return -1;
  int64_t need = (int64_t)ceil(0.10 * (double)H * (double)W);
  int64_t covered = 0;
  uint64_t skey = sm64(seed ^ 0x5354524F4B45ULL); /* "STROKE" */
  for (uint64_t s = 0; covered < need; ++s) {
    uint64_t r1 = sm64(skey + 2 * s), r2 = sm64(skey + 2 * s + 1);
    int horiz = (int)(r1 & 1);
    int64_t thick = 2 + (int64_t)((r1 >> 1) % 5);
    int64_t len = 5 + (int64_t)((r1 >> 8) % 36);
    uint8_t val = (uint8_t)(20 + (r1 >> 16) % 41);
    int64_t y0 = (int64_t)((r2 >> 32) % (uint64_t)H);
    int64_t x0 = (int64_t)((r2 & 0xFFFFFFFFULL) % (uint64_t)W);
    int64_t hh = horiz ? thick : len, ww = horiz ? len : thick;
    for (int64_t a = y0; a < y0 + hh && a < H; ++a)
      for (int64_t b = x0; b < x0 + ww && b < W; ++b) {
        if (ink[a * W + b] == 0) covered++;
        ink[a * W + b] = val;
      }
  }
  double ci = 0, cj = 0, sb = 1;
  double *ey = NULL, *ex = NULL;
  if (stain) {
    uint64_t t1 = sm64(seed ^ 0x535441494EULL), t2 = sm64(t1), t3 = sm64(t2); /* "STAIN" */
    ci = (double)(t1 % (uint64_t)H);
    cj = (double)(t2 % (uint64_t)W);
    double mnhw = (double)(H < W ? H : W);
    double uu = (double)(t3 >> 11) * (1.0 / 9007199254740992.0);
    sb = mnhw / 8.0 + uu * (mnhw / 4.0 - mnhw / 8.0);
    ey = (double *)malloc((size_t)H * sizeof(double));
    ex = (double *)malloc((size_t)W * sizeof(double));
    if (!ey || !ex) { free(ey); free(ex); free(ink); return -1; }
    for (int64_t i = 0; i < H; ++i) ey[i] = exp(-((double)i - ci) * ((double)i - ci) / (2.0 * sb * sb));
    for (int64_t j = 0; j < W; ++j) ex[j] = exp(-((double)j - cj) * ((double)j - cj) / (2.0 * sb * sb));
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < H; ++i) {
    uint8_t *row = out + i * pitch;
    for (int64_t j = 0; j < W; ++j) {
      uint8_t v = ink[i * W + j];
      double x = v ? (double)v : bg_noise(key, H, W, i, j);
      if (!v) x = clamp255(rint(x));
      if (stain) x = clamp255(rint(x - 80.0 * (ey[i] * ex[j])));
      row[j] = (uint8_t)x;
    }
  }
  free(ink);
  free(ey);
  free(ex);
  return 0;
}

/* Many pages: page p uses seed0 + p (BASELINE seeds: 1905130380 + 1000 cfg + p). */
int synth_pages(uint64_t seed0, int64_t P, int64_t H, int64_t W, int32_t stain, uint8_t *out, int64_t pitch,
                int64_t page_stride) {
  int rc = 0;
  for (int64_t p = 0; p < P; ++p)
    if (synth_page(seed0 + (uint64_t)p, H, W, stain, out + p * page_stride, pitch) != 0) rc = -1;
  return rc;
}

/* FNV-1a 64 of a page (row by row, W bytes per row), for the golden hashes. */
uint64_t synth_hash(const uint8_t *img, int64_t H, int64_t W, int64_t pitch) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) {
      h ^= img[i * pitch + j];
      h *= 0x100000001b3ULL;
    }
  return h;
}
