/*
 * abin_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the hot path of
 * Chan, "Memory-efficient and fast implementation of local adaptive
 * binarization methods" (arXiv 1905.13038), reference/PAPER.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path
 * (paper_1905_13038_b200/) never links, imports or executes it, and this
 * file shares no code, header, table or constant generator with the CUDA
 * path.
 *
 * Everything here is the *definition* written out (Sec. 1,
 * l.27: m and s as direct sums over the h x w window) -- Theta(HWhw) --
 * with the paper's window offsets (Alg. 1 l.1-4), the
 * "undefined elements are zero" border convention and the
 * clamped count n (Alg. 1).  Thresholds follow Table 1
 * evaluated left to right in IEEE double, compiled
 * with -ffp-contract=off -fno-fast-math.
 *
 * Secondary engines (each exact, each pinned against orc_* direct in the
 * CPU tests):
 *   orc_alg1_stats   -- a literal transcription of Algorithm 1's recursion
 *                       (PAPER.md:98-120), used as the "decomposition
 *                       invariance" pin and as the paper-method CPU timing.
 *   orc_integral_stats -- Sec. 2 integral images, u64.
 *
 * Parity unpinned (no value in the paper fixes them):
 *   - the exact fp64 bits of t (pinned only by the literal Table-1 order);
 *   - the quantile rank convention rho = max(1, ceil(q n)) (SPEC choice).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_SAUVOLA 0
#define ORC_NIBLACK 1
#define ORC_WOLF 2

/* Alg. 1 l.1-4. */
static void offsets(int32_t h, int32_t w, int64_t *l, int64_t *r, int64_t *o, int64_t *u) {
  *l = (w + 1) / 2; /* floor((w+1)/2) */
  *r = w / 2;       /* floor(w/2)     */
  *o = (h + 1) / 2; /* floor((h+1)/2) */
  *u = h / 2;       /* floor(h/2)     */
}

static int64_t mn(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t mx(int64_t a, int64_t b) { return a > b ? a : b; }

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* Window offsets exported for the tests (they are pinned against the SPEC
 * examples and against brute-force enumeration of PAPER.md:27's bounds). */
void orc_offsets(int32_t h, int32_t w, int64_t out4[4]) {
  offsets(h, w, &out4[0], &out4[1], &out4[2], &out4[3]);
}

/* n, PAPER.md:118:
 *   n = (min{j+r, W-1} - max{j-l, -1}) * (min{i+u, H-1} - max{i-o, -1}). */
int64_t orc_count(int64_t H, int64_t W, int32_t h, int32_t w, int64_t i, int64_t j) {
  int64_t l, r, o, u;
  offsets(h, w, &l, &r, &o, &u);
  return (mn(j + r, W - 1) - mx(j - l, -1)) * (mn(i + u, H - 1) - mx(i - o, -1));
}

/* Direct window sums, PAPER.md:27 (rows i-h/2 < a <= i+h/2 with the floors of
 * Alg. 1: rows (i-o, i+u], cols (j-l, j+r]); out-of-bounds terms are zero
 * (PAPER.md:83), i.e. only in-bounds pixels contribute. */
static void direct_sums(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w,
                        int64_t i, int64_t j, uint64_t *c, uint64_t *d) {
  int64_t l, r, o, u;
  offsets(h, w, &l, &r, &o, &u);
  uint64_t sc = 0, sd = 0;
  for (int64_t a = i - o + 1; a <= i + u; ++a) {
    if (a < 0 || a >= H) continue; /* undefined element = 0 */
    const uint8_t *row = I + a * pitch;
    for (int64_t b = j - l + 1; b <= j + r; ++b) {
      if (b < 0 || b >= W) continue;
      uint64_t x = row[b];
      sc += x;
      sd += x * x;
    }
  }
  *c = sc;
  *d = sd;
}

/* Canonical fp64 threshold: Alg. 1 l.121-122 (m = c/n, v = d/n - m^2),
 * v clamped at 0 (SPEC sweep_mean_variance; never fires for n <= 66049, see
 * DESIGN.md), s = sqrt(v), then the Table 1 row written left to right:
 *   Niblack  t = m + k s
 *   Sauvola  t = m (1 + k (s/R - 1))
 *   Wolf     t = m - k (m - L)(1 - s/R)       (L = global min PAPER.md:163)
 */
double orc_threshold(int32_t method, uint64_t c, uint64_t d, uint64_t n, double k, double R, double L) {
  double m = (double)c / (double)n;
  double v = (double)d / (double)n - m * m;
  if (v < 0) v = 0;
  double s = sqrt(v);
  switch (method) {
    case ORC_SAUVOLA: return m * (1.0 + k * (s / R - 1.0));
    case ORC_NIBLACK: return m + k * s;
    case ORC_WOLF: return m - k * (m - L) * (1.0 - s / R);
  }
  return NAN;
}

/* Wolf's image-adaptive dynamic range R (NEXT #3; PAPER.md:153 writes Wolf's
 * rule with a constant R; Wolf et al.'s original takes R = the maximum of s
 * over the image -- SPEC.md:303, 319, "two-pass mode"; reading R21):
 * the maximum over the page's pixels of s, each s by the canonical fp64
 * sequence of orc_threshold (m = c/n, v = d/n - m m clamped at 0, s = sqrt v).
 * A page whose windows are all constant has max s = 0: R is then +inf, so
 * s / R = 0 and Wolf's t = m - k (m - L) (the reading R21). */
double orc_max_s(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w) {
  double best = 0.0;
#pragma omp parallel for schedule(static) reduction(max : best)
  for (int64_t i = 0; i < H; ++i) {
    for (int64_t j = 0; j < W; ++j) {
      uint64_t c, d;
      direct_sums(I, H, W, pitch, h, w, i, j, &c, &d);
      const uint64_t n = (uint64_t)orc_count(H, W, h, w, i, j);
      double m = (double)c / (double)n;
      double v = (double)d / (double)n - m * m;
      if (v < 0) v = 0;
      const double sv = sqrt(v);
      if (sv > best) best = sv;
    }
  }
  return best;
}

/* R for Wolf's adaptive mode from the maximum s (R21). */
double orc_adaptive_R(double max_s) { return max_s > 0.0 ? max_s : INFINITY; }

/* Global minimum of gray levels, Table 1 notation L. */
int32_t orc_global_min(const uint8_t *I, int64_t H, int64_t W, int64_t pitch) {
  int32_t L = 255;
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j)
      if (I[i * pitch + j] < L) L = I[i * pitch + j];
  return L;
}

/* Full binarization by the definition.  mask[i*W+j] = 0 if I <= t (foreground,
 * Alg. 1 l.124 "I'_ij <- 0"), else 1.  Optional outputs (NULL to skip):
 * c, d (uint64), n (uint64), t (double).  near_tie counts |I - t| < 1e-9
 * (BASELINE.json north_star).  Returns 0. */
int orc_binarize(int32_t method, const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w,
                 double k, double R, int32_t L_override, uint8_t *mask, uint64_t *c_out, uint64_t *d_out,
                 uint64_t *n_out, double *t_out, uint64_t *near_tie) {
  double L = 0.0;
  if (method == ORC_WOLF) L = (double)(L_override >= 0 ? L_override : orc_global_min(I, H, W, pitch));
  uint64_t ties = 0;
#pragma omp parallel for schedule(static) reduction(+ : ties)
  for (int64_t i = 0; i < H; ++i) {
    for (int64_t j = 0; j < W; ++j) {
      uint64_t c, d;
      direct_sums(I, H, W, pitch, h, w, i, j, &c, &d);
      uint64_t n = (uint64_t)orc_count(H, W, h, w, i, j);
      double t = orc_threshold(method, c, d, n, k, R, L);
      double x = (double)I[i * pitch + j];
      if (mask) mask[i * W + j] = (x <= t) ? 0 : 1;
      if (fabs(x - t) < 1e-9) ties++;
      if (c_out) c_out[i * W + j] = c;
      if (d_out) d_out[i * W + j] = d;
      if (n_out) n_out[i * W + j] = n;
      if (t_out) t_out[i * W + j] = t;
    }
  }
  if (near_tie) *near_tie = ties;
  return 0;
}

/* The same definition evaluated at m sampled positions (rows[k], cols[k]) of
 * a (possibly huge) page: used for parity at the bench's full sizes. */
int orc_binarize_points(int32_t method, const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h,
                        int32_t w, double k, double R, int32_t L, int64_t m, const int64_t *rows,
                        const int64_t *cols, uint8_t *mask, uint64_t *c_out, uint64_t *d_out, uint64_t *n_out,
                        double *t_out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < m; ++q) {
    int64_t i = rows[q], j = cols[q];
    uint64_t c, d;
    direct_sums(I, H, W, pitch, h, w, i, j, &c, &d);
    uint64_t n = (uint64_t)orc_count(H, W, h, w, i, j);
    double t = orc_threshold(method, c, d, n, k, R, (double)L);
    double x = (double)I[i * pitch + j];
    if (mask) mask[q] = (x <= t) ? 0 : 1;
    if (c_out) c_out[q] = c;
    if (d_out) d_out[q] = d;
    if (n_out) n_out[q] = n;
    if (t_out) t_out[q] = t;
  }
  return 0;
}

/* ---- Algorithm 1, transcribed -------------------------
 * The paper's recursion for c, d, with its own loop structure: column
 * accumulators C_j, D_j initialised over rows 0..u-1 (l.98-105), updated by
 * "C_j <- C_j + I_{i+u,j} - I_{i-o,j}" (l.107-110), row accumulators reset
 * and prefilled with C_0..C_{r-1} (l.111-116), then slid with
 * "c <- c + C_{j+r} - C_{j-l}" (l.119-120).  Out-of-range reads are zero
 * (PAPER.md:83).  Outputs c, d per pixel (u64); n from l.118.  Used only as
 * a pin ("decomposition invariance") and as the paper-method timing. */
static uint64_t Iz(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int64_t i, int64_t j) {
  if (i < 0 || i >= H || j < 0 || j >= W) return 0;
  return I[i * pitch + j];
}

int orc_alg1_stats(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w, uint64_t *c_out,
                   uint64_t *d_out) {
  int64_t l, r, o, u;
  offsets(h, w, &l, &r, &o, &u);
  uint64_t *C = (uint64_t *)calloc((size_t)W, sizeof(uint64_t));
  uint64_t *D = (uint64_t *)calloc((size_t)W, sizeof(uint64_t));
  if (!C || !D) { free(C); free(D); return -1; }
  for (int64_t j = 0; j < W; ++j) {
    C[j] = 0;
    D[j] = 0;
    for (int64_t i = 0; i <= u - 1; ++i) {
      uint64_t x = Iz(I, H, W, pitch, i, j);
      C[j] += x;
      D[j] += x * x;
    }
  }
  for (int64_t i = 0; i < H; ++i) {
    for (int64_t j = 0; j < W; ++j) {
      uint64_t a = Iz(I, H, W, pitch, i + u, j), b = Iz(I, H, W, pitch, i - o, j);
      C[j] = C[j] + a - b;
      D[j] = D[j] + a * a - b * b;
    }
    uint64_t c = 0, d = 0;
    for (int64_t j = 0; j <= r - 1; ++j) {
      c += (j < W) ? C[j] : 0;
      d += (j < W) ? D[j] : 0;
    }
    for (int64_t j = 0; j < W; ++j) {
      int64_t jr = j + r, jl = j - l;
      c = c + ((jr < W) ? C[jr] : 0) - ((jl >= 0) ? C[jl] : 0);
      d = d + ((jr < W) ? D[jr] : 0) - ((jl >= 0) ? D[jl] : 0);
      c_out[i * W + j] = c;
      d_out[i * W + j] = d;
    }
  }
  free(C);
  free(D);
  return 0;
}

/* ---- Sec. 2 integral images -------------------------------
 * J_{i,j} = J_{i-1,j} + J_{i,j-1} + f(I_{i,j}) - J_{i-1,j-1}, J = 0 for i<0
 * or j<0; window sum = J_{a1,b1} - J_{a0,b1} - J_{a1,b0} + J_{a0,b0}. */
int orc_integral_stats(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w,
                       uint64_t *c_out, uint64_t *d_out) {
  int64_t l, r, o, u;
  offsets(h, w, &l, &r, &o, &u);
  uint64_t *J1 = (uint64_t *)malloc((size_t)(H * W) * sizeof(uint64_t));
  uint64_t *J2 = (uint64_t *)malloc((size_t)(H * W) * sizeof(uint64_t));
  if (!J1 || !J2) { free(J1); free(J2); return -1; }
#define JV(J, a, b) (((a) < 0 || (b) < 0) ? 0 : (J)[(a) * W + (b)])
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) {
      uint64_t x = I[i * pitch + j];
      J1[i * W + j] = JV(J1, i - 1, j) + JV(J1, i, j - 1) + x - JV(J1, i - 1, j - 1);
      J2[i * W + j] = JV(J2, i - 1, j) + JV(J2, i, j - 1) + x * x - JV(J2, i - 1, j - 1);
    }
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) {
      int64_t a0 = mx(i - o, -1), a1 = mn(i + u, H - 1), b0 = mx(j - l, -1), b1 = mn(j + r, W - 1);
      c_out[i * W + j] = JV(J1, a1, b1) - JV(J1, a0, b1) - JV(J1, a1, b0) + JV(J1, a0, b0);
      d_out[i * W + j] = JV(J2, a1, b1) - JV(J2, a0, b1) - JV(J2, a1, b0) + JV(J2, a0, b0);
    }
#undef JV
  free(J1);
  free(J2);
  return 0;
}

/* ---- Local quantile (rank convention SPEC sweep_quantile) --
 * Gather the in-bounds window (out-of-bounds pixels are excluded, not zero
 * padded: the quantile is of the n gray levels that exist), sort, and take
 * the rho-th smallest, rho = max(1, ceil(q n)).  mask = 0 iff I <= Q. */
static int cmp_u8(const void *a, const void *b) { return (int)*(const uint8_t *)a - (int)*(const uint8_t *)b; }

static uint8_t direct_quantile(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w,
                               double q, int64_t i, int64_t j, uint8_t *buf) {
  int64_t l, r, o, u;
  offsets(h, w, &l, &r, &o, &u);
  int64_t n = 0;
  for (int64_t a = i - o + 1; a <= i + u; ++a) {
    if (a < 0 || a >= H) continue;
    for (int64_t b = j - l + 1; b <= j + r; ++b) {
      if (b < 0 || b >= W) continue;
      buf[n++] = I[a * pitch + b];
    }
  }
  qsort(buf, (size_t)n, 1, cmp_u8);
  int64_t rho = (int64_t)ceil(q * (double)n);
  if (rho < 1) rho = 1;
  return buf[rho - 1];
}

int orc_quantile(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w, double q,
                 uint8_t *mask, uint8_t *Q_out) {
  int rc = 0;
#pragma omp parallel
  {
    uint8_t *buf = (uint8_t *)malloc((size_t)mn(h, H) * (size_t)mn(w, W));
    if (!buf) {
#pragma omp atomic write
      rc = -1;
    } else {
#pragma omp for schedule(static)
      for (int64_t i = 0; i < H; ++i)
        for (int64_t j = 0; j < W; ++j) {
          uint8_t Q = direct_quantile(I, H, W, pitch, h, w, q, i, j, buf);
          if (Q_out) Q_out[i * W + j] = Q;
          if (mask) mask[i * W + j] = (I[i * pitch + j] <= Q) ? 0 : 1;
        }
      free(buf);
    }
  }
  return rc;
}

int orc_quantile_points(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w, double q,
                        int64_t m, const int64_t *rows, const int64_t *cols, uint8_t *mask, uint8_t *Q_out) {
  int rc = 0;
#pragma omp parallel
  {
    uint8_t *buf = (uint8_t *)malloc((size_t)mn(h, H) * (size_t)mn(w, W));
    if (!buf) {
#pragma omp atomic write
      rc = -1;
    } else {
#pragma omp for schedule(dynamic, 64)
      for (int64_t p = 0; p < m; ++p) {
        uint8_t Q = direct_quantile(I, H, W, pitch, h, w, q, rows[p], cols[p], buf);
        if (Q_out) Q_out[p] = Q;
        if (mask) mask[p] = (I[rows[p] * pitch + cols[p]] <= Q) ? 0 : 1;
      }
      free(buf);
    }
  }
  return rc;
}

/* ---- Bernsen: local midrange (Sec. 3.4 "Generalization") ----
 * min and max of the in-bounds gray levels of the window (rows (i-o, i+u],
 * cols (j-l, j+r], out-of-bounds pixels excluded -- the extrema of the
 * pixels that exist), threshold t = (min + max) / 2 ("used midrange as
 * threshold value"), foreground iff I <= t.  With integer gray levels,
 * I <= (min + max)/2  <=>  2 I <= min + max, evaluated exactly.
 * contrast >= 0 selects the local-contrast variant the same paragraph
 * mentions ("estimate local contrast by range of gray levels"): a pixel whose
 * window range max - min is below `contrast` is background (1); otherwise the
 * midrange rule (SPEC threshold-rules, rule bernsen-contrast).  The direct
 * definition: Theta(h w) per pixel. */
static void direct_extrema(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w, int64_t i,
                           int64_t j, int32_t *mn_out, int32_t *mx_out) {
  int64_t l, r, o, u;
  offsets(h, w, &l, &r, &o, &u);
  int32_t lo = 255, hi = 0;
  for (int64_t a = mx(i - o + 1, 0); a <= mn(i + u, H - 1); ++a)
    for (int64_t b = mx(j - l + 1, 0); b <= mn(j + r, W - 1); ++b) {
      const int32_t x = I[a * pitch + b];
      if (x < lo) lo = x;
      if (x > hi) hi = x;
    }
  *mn_out = lo;
  *mx_out = hi;
}

static uint8_t bernsen_decide(int32_t x, int32_t lo, int32_t hi, int32_t contrast) {
  if (contrast >= 0 && hi - lo < contrast) return 1; /* low contrast: background */
  return (2 * x <= lo + hi) ? 0 : 1;
}

int orc_bernsen(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w, int32_t contrast,
                uint8_t *mask, uint8_t *min_out, uint8_t *max_out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) {
      int32_t lo, hi;
      direct_extrema(I, H, W, pitch, h, w, i, j, &lo, &hi);
      if (mask) mask[i * W + j] = bernsen_decide(I[i * pitch + j], lo, hi, contrast);
      if (min_out) min_out[i * W + j] = (uint8_t)lo;
      if (max_out) max_out[i * W + j] = (uint8_t)hi;
    }
  return 0;
}

int orc_bernsen_points(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w,
                       int32_t contrast, int64_t m, const int64_t *rows, const int64_t *cols, uint8_t *mask) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < m; ++q) {
    int32_t lo, hi;
    direct_extrema(I, H, W, pitch, h, w, rows[q], cols[q], &lo, &hi);
    mask[q] = bernsen_decide(I[rows[q] * pitch + cols[q]], lo, hi, contrast);
  }
  return 0;
}

/* ---- The remaining Table 1 rows, "implemented by changing
 * a single condition in Algorithm 1".  Each is the row
 * written left to right in IEEE double (no contraction), after the canonical
 * m = c/n, v = d/n - m^2 (clamped at 0), s = sqrt(v) of orc_threshold:
 *   Feng       t = a1 m + k1 (s/R)^(1+g) (m - L) + k2 (s/R)^g L
 *              params {a1, k1, k2, g, R}; L = global minimum
 *   Rais       t = m + 0.3 (m s - M S) / max{m s, M S} s
 *              M, S = global mean and standard deviation;
 *              reading: 0/0 (both products zero) -> fraction 0 (R16)
 *   Khurshid   t = m + k sqrt(s^2 + m^2 (N - 1) / N)
 *              params {k, N_mode}: N = h w (the table's "hw") or, N_mode = 1,
 *              the clamped count n (R17)
 *   Phansalkar t = m (1 + p e^(-q m) + k (s/R - 1))
 *              params {k, R, p, q}
 */
#define ORC_FENG 5
#define ORC_RAIS 6
#define ORC_KHURSHID 7
#define ORC_PHANSALKAR 8

double orc_threshold_rule(int32_t rule, uint64_t c, uint64_t d, uint64_t n, const double *prm, double L, double M,
                          double S, double hw) {
  double m = (double)c / (double)n;
  double v = (double)d / (double)n - m * m;
  if (v < 0) v = 0;
  double s = sqrt(v);
  switch (rule) {
    case ORC_FENG: {
      const double a1 = prm[0], k1 = prm[1], k2 = prm[2], g = prm[3], R = prm[4];
      return a1 * m + k1 * pow(s / R, 1.0 + g) * (m - L) + k2 * pow(s / R, g) * L;
    }
    case ORC_RAIS: {
      const double a = m * s, b = M * S;
      const double den = a > b ? a : b;
      const double frac = den > 0 ? (a - b) / den : 0.0;
      return m + 0.3 * frac * s;
    }
    case ORC_KHURSHID: {
      const double k = prm[0];
      const double N = prm[1] != 0.0 ? (double)n : hw;
      return m + k * sqrt(s * s + m * m * ((N - 1.0) / N));
    }
    case ORC_PHANSALKAR: {
      const double k = prm[0], R = prm[1], p = prm[2], q = prm[3];
      return m * (1.0 + p * exp(-q * m) + k * (s / R - 1.0));
    }
  }
  return NAN;
}

/* Global mean M and standard deviation S of the gray levels (Table 1
 * notation): exact integer sums, then M = sum/N,
 * S = sqrt(sumsq/N - M^2) (clamped at 0). */
void orc_global_mean_std(const uint8_t *I, int64_t H, int64_t W, int64_t pitch, double *M, double *S) {
  uint64_t s1 = 0, s2 = 0;
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) {
      const uint64_t x = I[i * pitch + j];
      s1 += x;
      s2 += x * x;
    }
  const double N = (double)H * (double)W;
  const double m = (double)s1 / N;
  double v = (double)s2 / N - m * m;
  if (v < 0) v = 0;
  *M = m;
  *S = sqrt(v);
}

/* Binarization by a Table 1 rule at the whole page (rows = NULL) or at m
 * sampled pixels; t_out optional.  mask = 0 iff I <= t. */
int orc_binarize_rule(int32_t rule, const uint8_t *I, int64_t H, int64_t W, int64_t pitch, int32_t h, int32_t w,
                      const double *prm, int64_t m, const int64_t *rows, const int64_t *cols, uint8_t *mask,
                      double *t_out) {
  double L = 0, M = 0, S = 0;
  if (rule == ORC_FENG) L = (double)orc_global_min(I, H, W, pitch);
  if (rule == ORC_RAIS) orc_global_mean_std(I, H, W, pitch, &M, &S);
  const double hw = (double)h * (double)w;
  const int64_t total = rows ? m : H * W;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t q = 0; q < total; ++q) {
    const int64_t i = rows ? rows[q] : q / W, j = rows ? cols[q] : q % W;
    uint64_t c, d;
    direct_sums(I, H, W, pitch, h, w, i, j, &c, &d);
    const uint64_t n = (uint64_t)orc_count(H, W, h, w, i, j);
    const double t = orc_threshold_rule(rule, c, d, n, prm, L, M, S, hw);
    mask[q] = ((double)I[i * pitch + j] <= t) ? 0 : 1;
    if (t_out) t_out[q] = t;
  }
  return 0;
}

/* ---- Otsu's global threshold (the paper's speed
 * comparator; SPEC threshold-rules otsu_threshold) -------------------------
 * Histogram h(g) of the page (exact counts), then the t in 0..255 maximising
 * the between-class variance  sigma_b^2(t) = w0 w1 (mu0 - mu1)^2  with
 * w0 = N0/N, w1 = N1/N (N0 = #(x <= t), N1 = N - N0) and mu0, mu1 the class
 * means; classes with no pixels give sigma_b^2 = 0; ties keep the smallest t.
 * Evaluated in IEEE double in this order:
 *   w0 = N0/N, w1 = N1/N, mu0 = S0/N0, mu1 = S1/N1, d = mu0 - mu1,
 *   sb = (w0 * w1) * (d * d)
 * (S0 = sum of g h(g) over g <= t).  Foreground iff I <= t. */
int32_t orc_otsu(const uint8_t *I, int64_t H, int64_t W, int64_t pitch) {
  uint64_t hist[256] = {0};
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) hist[I[i * pitch + j]]++;
  const uint64_t N = (uint64_t)H * (uint64_t)W;
  uint64_t Stot = 0;
  for (int g = 0; g < 256; ++g) Stot += (uint64_t)g * hist[g];
  const double Nd = (double)N;
  uint64_t N0 = 0, S0 = 0;
  double best = -1.0;
  int32_t tbest = 0;
  for (int t = 0; t < 256; ++t) {
    N0 += hist[t];
    S0 += (uint64_t)t * hist[t];
    const uint64_t N1 = N - N0, S1 = Stot - S0;
    double sb = 0.0;
    if (N0 > 0 && N1 > 0) {
      const double w0 = (double)N0 / Nd, w1 = (double)N1 / Nd;
      const double mu0 = (double)S0 / (double)N0, mu1 = (double)S1 / (double)N1;
      const double d = mu0 - mu1;
      sb = (w0 * w1) * (d * d);
    }
    if (sb > best) {
      best = sb;
      tbest = t;
    }
  }
  return tbest;
}

