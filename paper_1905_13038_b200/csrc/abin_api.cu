// abin_api.cu -- the C ABI of libabin.so (include/abin.h): argument
// validation, tiling decisions, TMA tensor maps and kernel launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <utility>

#include "../../include/abin.h"
#include "globalmin.cuh"
#include "otsu.cuh"
#include "fixup.cuh"
#include "launch.cuh"
#include "bernsen.cuh"
#include "small.cuh"
#include "quantile.cuh"

using namespace abin;

namespace {

thread_local char g_last_cuda_error[256] = "";

int cuda_fail(cudaError_t e) {
  snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s", cudaGetErrorString(e));
  return ABIN_ECUDA;
}

#define CK(x)                          \
  do {                                 \
    cudaError_t e_ = (x);              \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

// ---- driver entry point for cuTensorMapEncodeTiled (no -lcuda needed)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

struct Window {
  int32_t h, w, l, r, o, u;
};

// Experiment and test hooks: read on every call and
// parsed / clamped in one place; unset (or "0" for the flags) means the
// measured defaults.
bool env_flag(const char* name) {
  const char* e = getenv(name);
  return e && *e && strcmp(e, "0") != 0;
}
long long env_int(const char* name, long long def, long long lo, long long hi) {
  const char* e = getenv(name);
  if (!e || !*e) return def;
  return std::max(lo, std::min(hi, atoll(e)));
}
double env_real(const char* name, double def, double lo, double hi) {
  const char* e = getenv(name);
  if (!e || !*e) return def;
  const double v = atof(e);
  return std::isfinite(v) ? std::max(lo, std::min(hi, v)) : def;
}

// Alg. 1 l.1-4, then clamp the reach to the image: replacing
// l by min(l, W) (etc.) changes neither the in-bounds window nor n.
Window effective_window(int32_t h, int32_t w, int64_t Hg, int64_t W) {
  Window x;
  x.l = (int32_t)std::min<int64_t>((w + 1) / 2, W);
  x.r = (int32_t)std::min<int64_t>(w / 2, W);
  x.o = (int32_t)std::min<int64_t>((h + 1) / 2, Hg);
  x.u = (int32_t)std::min<int64_t>(h / 2, Hg);
  x.w = x.l + x.r;
  x.h = x.o + x.u;
  return x;
}

// internal test hook: force the generic (non-TMA) loader
constexpr uint32_t ABIN_NO_TMA_INTERNAL = 1u << 30;
// internal test hook: the 4-warp-CTA kernel (moments.cuh) instead of the warp-CTA kernel (moments4.cuh)
constexpr uint32_t ABIN_V3_INTERNAL = 1u << 29;
constexpr uint32_t ABIN_WIDE_INTERNAL = 1u << 28;  // test hook: the CTA-wide kernel for any window
constexpr uint32_t ABIN_V4_INTERNAL = 1u << 27;    // test hook: the v4 warp-CTA kernel instead of v5
constexpr uint32_t ABIN_Q2_INTERNAL = 1u << 26;    // test hook: the round-1 quantile kernels instead of v5
constexpr int64_t kMaxDim = (int64_t)1 << 30;
constexpr int kQuantNT = 128;  // threads of the single-column quantile kernel (its staging bounds w)

// ---- wide-window fallback (moments_wide.cuh): CTA strips of NT*8 columns
int choose_nt_wide(int32_t w_eff) {
  const int kh = (((w_eff + 1 + 8 - 1) / 8) + 1) & ~1;
  if (kh <= 64) return 128;
  if (kh <= 190) return 256;
  return 0;
}

int launch_fast_any(int w32, bool d64, const CUtensorMap& map, const MomParams& p, int64_t n, cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (w32 >> 2) {
    case 0: e = launch_fast_part0(w32, d64, map, p, n, st); break;
    case 1: e = launch_fast_part1(w32, d64, map, p, n, st); break;
    case 2: e = launch_fast_part2(w32, d64, map, p, n, st); break;
    case 3: e = launch_fast_part3(w32, d64, map, p, n, st); break;
    case 4: e = launch_fast_part4(w32, d64, map, p, n, st); break;
    case 5: e = launch_fast_part5(w32, d64, map, p, n, st); break;
    case 6: e = launch_fast_part6(w32, d64, map, p, n, st); break;
    case 7: e = launch_fast_part7(w32, d64, map, p, n, st); break;
  }
  return e == cudaSuccess ? ABIN_OK : cuda_fail(e);
}

int launch_v4_any(int w32, bool d64, const CUtensorMap& map, const MomParams& p, int64_t n, cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (w32 >> 2) {
    case 0: e = launch_v4_part0(w32, d64, map, p, n, st); break;
    case 1: e = launch_v4_part1(w32, d64, map, p, n, st); break;
    case 2: e = launch_v4_part2(w32, d64, map, p, n, st); break;
    case 3: e = launch_v4_part3(w32, d64, map, p, n, st); break;
    case 4: e = launch_v4_part4(w32, d64, map, p, n, st); break;
    case 5: e = launch_v4_part5(w32, d64, map, p, n, st); break;
    case 6: e = launch_v4_part6(w32, d64, map, p, n, st); break;
    case 7: e = launch_v4_part7(w32, d64, map, p, n, st); break;
  }
  return e == cudaSuccess ? ABIN_OK : cuda_fail(e);
}

int launch_v5_any(int w32, const CUtensorMap& map, const CUtensorMap& mpk, const MomParams& p, int64_t n,
                  cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (w32 >> 2) {
    case 0: e = launch_v5_part0(w32, map, mpk, p, n, st); break;
    case 1: e = launch_v5_part1(w32, map, mpk, p, n, st); break;
    case 2: e = launch_v5_part2(w32, map, mpk, p, n, st); break;
    case 3: e = launch_v5_part3(w32, map, mpk, p, n, st); break;
    case 4: e = launch_v5_part4(w32, map, mpk, p, n, st); break;
    case 5: e = launch_v5_part5(w32, map, mpk, p, n, st); break;
    case 6: e = launch_v5_part6(w32, map, mpk, p, n, st); break;
    case 7: e = launch_v5_part7(w32, map, mpk, p, n, st); break;
  }
  return e == cudaSuccess ? ABIN_OK : cuda_fail(e);
}

// resident v5 warp-CTAs per SM (registers and shared memory, as the runtime reports)
int occupancy_v5_query(int w32, int method) {
  switch (w32 >> 2) {
    case 0: return occupancy_v5_part0(w32, method);
    case 1: return occupancy_v5_part1(w32, method);
    case 2: return occupancy_v5_part2(w32, method);
    case 3: return occupancy_v5_part3(w32, method);
    case 4: return occupancy_v5_part4(w32, method);
    case 5: return occupancy_v5_part5(w32, method);
    case 6: return occupancy_v5_part6(w32, method);
    case 7: return occupancy_v5_part7(w32, method);
  }
  return 16;
}

// resident v5 warp-CTAs per SM, cached per device, w mod 32 and method (the
// runtime's occupancy query costs several microseconds of host time per call)
int occupancy_v5_any(int w32, int method) {
  static std::atomic<int> cache[64][32][16];
  static std::once_flag once;
  std::call_once(once, [] {
    for (auto& a : cache)
      for (auto& b : a)
        for (auto& c : b) c.store(-1, std::memory_order_relaxed);
  });
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || w32 < 0 || w32 >= 32 || method < 0 ||
      method >= 16)
    return occupancy_v5_query(w32, method);
  int v = cache[dev][w32][method].load(std::memory_order_relaxed);
  if (v < 0) {
    v = occupancy_v5_query(w32, method);
    cache[dev][w32][method].store(v, std::memory_order_relaxed);
  }
  return v;
}

int launch_wide_any(bool d64, bool stats, int nt, int ph, const CUtensorMap& map, const wide::MomParams& p,
                    int64_t n, cudaStream_t st) {
  const cudaError_t e = d64 ? launch_wide_d64(d64, stats, nt, ph, map, p, n, st)
                            : launch_wide_d32(d64, stats, nt, ph, map, p, n, st);
  return e == cudaSuccess ? ABIN_OK : cuda_fail(e);
}

// Certified bounds of the fp32 stages (K2).  u = 2^-24; the
// derivation bounds |t~ - t*| from the fp32 roundings of m, q, v, the
// approximate square root (relative error eps_sqrt) and the threshold
// expression, with m <= 255, s <= 128, q <= 255^2; eps64 bounds the
// double-precision sequence's own error |t_fp64 - t*|.
struct FilterConsts {
  float fa, fb, delta1, delta2;
  float rb0, rb1, rdv, rsdv;  // data-dependent stage-1 bound: rb0 + rb1 min(rsdv, rdv / s~)
  // Rais: the parts that scale with 1 / (M S) (the page's): coarse bound delta1 + rais_c / (M S),
  // data-dependent rb0 + rais_r0 / (M S) and rb1 + rais_r1 / (M S)
  float rais_c, rais_r0, rais_r1;
};

FilterConsts filter_consts(int method, double k, double R) {
  const double u = std::ldexp(1.0, -24);
  const double eps_sqrt = 8 * u;
  const double eps64 = 1e-6;
  const double qmax = 255.0 * 255.0;
  const double rv = std::sqrt(16.2 * u * qmax);                     // sqrt of the stage-1 bound on |v~ - v|
  const double ds1 = rv + eps_sqrt * (128.0 + rv);                  // stage 1: |s~ - s|
  const double ds2 = (4 * u + eps_sqrt) * 128.0 * 1.01;             // stage 2: relative error x s_max
  auto bound = [&](double ds) {
    if (method == M_SAUVOLA) {
      const double al = std::fabs(1.0 - k), be = std::fabs(k / R), G = al + be * (128.0 + ds);
      return 255.0 * be * ds + 8.1 * u * 255.0 * G;
    }
    if (method == M_NIBLACK) return std::fabs(k) * ds + u * (8.0 * 255.0 + 4.0 * std::fabs(k) * 128.0);
    return std::fabs(k) * 255.0 * ds / R + u * (8.0 * 255.0 + 12.0 * std::fabs(k) * 255.0);  // Wolf
  };
  FilterConsts f;
  if (method == M_SAUVOLA) { f.fa = (float)(1.0 - k); f.fb = (float)(k / R); }
  else if (method == M_NIBLACK) { f.fa = 0.0f; f.fb = (float)k; }
  else { f.fa = (float)k; f.fb = (float)(1.0 / R); }
  f.delta1 = (float)(1.25 * (bound(ds1) + eps64) + 1e-6);
  f.delta2 = (float)(1.25 * (bound(ds2) + eps64) + 1e-6);
  // The same bound with the data-dependent |s~ - s|: for s0 = sqrt|v~|,
  // |s0 - s| = |v~ - v| / (s0 + s) <= dv / s0 and s0 >= s~ / (1 + eps_sqrt), so
  //   |s~ - s| <= min(sqrt dv, dv (1 + eps_sqrt) / s~) + eps_sqrt (128 + sqrt dv).
  // bound(ds) is affine in ds: bound = b0 + b1 ds.
  const double b0 = bound(0.0), b1 = bound(1.0) - b0;
  const double dv = 16.2 * u * qmax;
  f.rb0 = (float)((1.25 * (b0 + b1 * eps_sqrt * (128.0 + rv) + eps64) + 1e-6) * (1 + 1e-6));
  f.rb1 = (float)(1.25 * b1 * (1 + 1e-6));
  f.rdv = (float)(dv * (1 + eps_sqrt) * (1 + 1e-6));
  f.rsdv = (float)(rv * (1 + 1e-6));
  return f;
}

// Certified bound of the v5 kernel's fp32 residual (moments5.cuh residual2),
// |e~ - e*| with e* = I - t*, t* the exact threshold of the exact integer
// sums ("v5 certified bound").  u = 2^-24.  The
// sequence: m~ = fl(rc nu + Kc), q~ = fl(rd nu + Kd) (Kc = fl(Sc nu),
// Kd = fl(fl(Sd) nu), rd = fl(rel_d), rc exact, nu = -1/n with relative error
// e_nu), w~ = fl(m~^2 - q~), s~ = sqrt.approx|w~|, then the Table-1
// expression.  Counts n lie in [n_min, n_max]; the start value and the
// relative sums are window sums of windows with counts <= n_max, so they are
// bounded by 255 n_max (c) and 255^2 n_max (d).
FilterConsts filter_consts_v5(int method, double k, double R, const double* rprm = nullptr) {
  const double u = std::ldexp(1.0, -24);
  const double eps_sqrt = 8 * u;            // sqrt.approx.f32: relative error < 2^-22 (taken as 2^-21)
  const double eps64 = 1e-6;                // |t_fp64 - t*| (the canonical double sequence)
  const double e_nu = 3.01 * u;             // fl(fl(1/ncol) fl(1/nrow)): three roundings
  const double qmax = 255.0 * 255.0;
  // Khurshid's radicand W = q - m^2 / N lies in [0, 255^2]; the others' v in [0, 127.5^2]
  const double smax = method == M_KHURSHID ? 255.0 : 127.5;
  const double dm = 255.0 * (e_nu + u) * 1.01;                                // |m~ - m|: one rounding of c nu~
  const double dq = qmax * (e_nu + 2 * u) * 1.01;                             // |q~ - q|: fl(d), then fl(fl(d) nu~)
  double dv = (2 * 255.0 + dm) * dm + dq + 1.01 * u * (smax * smax + 1.0);    // |(-w~) - v|, w~ = fl(m~^2 - q~)
  if (method == M_KHURSHID)
    // w~ = fl(m~ fl(m~ iN~) - q~), iN~ = 1/N (1 + e_nu): |m~^2 / N - m^2 / N| <= (510 + dm) dm,
    // the product's two roundings and iN~'s error <= 255^2 (e_nu + u), then q~ and the last rounding
    dv = (2 * 255.0 + dm) * dm * 1.01 + qmax * (e_nu + u) * 1.01 + dq + 1.01 * u * (qmax + 1.0);
  const double rv = std::sqrt(dv);
  const double ds = rv + eps_sqrt * (smax + rv);                               // |s~ - s| (coarse)
  FilterConsts f;
  memset(&f, 0, sizeof(f));
  if (method == M_KHURSHID) k = rprm[0];
  if (method == M_PHANSALKAR) { k = rprm[0]; R = rprm[1]; }
  auto bound = [&](double dsx) {
    if (method == M_SAUVOLA) {
      const double a = std::fabs(1.0 - k), b = std::fabs(k / R);
      const double G = a + b * (smax + dsx);                                   // |g~|
      const double dg = b * (dsx + smax * u) + a * u + 1.01 * u * G;           // |g~ - g|
      return dm * G + 255.0 * dg + dm * dg + 1.01 * u * 255.0 * (1.0 + G);
    }
    if (method == M_PHANSALKAR) {
      // g = (1 - k) + (k/R) s + p E, E = 2^(-q log2(e) m) <= 1 (q >= 0); a~ = fl(fl(q log2 e) (-m~))
      // has |a~ - a| <= q log2(e) (dm + 2.02 u 255); ex2.approx (relative error eps_ex2, flush
      // below 2^-126): |E~ - E| <= 2^|da| (ln2 |da| + eps_ex2) + 2^-126, ln2 log2(e) = 1
      const double pp = std::fabs(rprm[2]), q = rprm[3];
      const double eps_ex2 = 32 * u;
      const double da = q * 1.4426950408889634 * (dm + 2.02 * u * 255.0);
      const double g2 = std::exp2(da);
      const double dE = g2 * (q * (dm + 2.02 * u * 255.0) + eps_ex2) * 1.01 + std::ldexp(1.0, -126);
      const double Em = g2 * (1.0 + eps_ex2);
      const double a = std::fabs(1.0 - k), b = std::fabs(k / R);
      const double G = a + b * (smax + dsx) + pp * Em;
      const double dg = b * (dsx + smax * u) + a * u + pp * (dE + u * Em) + 2.02 * u * G;
      return dm * G + 255.0 * dg + dm * dg + 1.01 * u * 255.0 * (1.0 + G);
    }
    if (method == M_NIBLACK || method == M_KHURSHID) {
      const double ak = std::fabs(k);
      return dm + 2.02 * u * 255.0 + ak * dsx + ak * smax * u + 1.01 * u * (510.0 + ak * smax);
    }
    // Wolf: e = (I - m) + (k (m - L)) (1 - s/R)
    const double ak = std::fabs(k), iR = 1.0 / R;
    const double dka = ak * (dm + 255.0 * u) + 2.02 * u * ak * 255.0;           // |ka~ - k (m - L)|
    const double Bm = 1.0 + (smax + dsx) * iR;                                  // |b~|
    const double db = dsx * iR + smax * iR * u + 1.01 * u * Bm;                 // |b~ - (1 - s/R)|
    return dka * Bm + ak * 255.0 * db + dm + 2.02 * u * 255.0 + 1.01 * u * (510.0 + ak * 255.0 * Bm);
  };
  if (method == M_SAUVOLA || method == M_PHANSALKAR) { f.fa = (float)(1.0 - k); f.fb = (float)(k / R); }
  else if (method == M_NIBLACK || method == M_KHURSHID) { f.fa = 0.0f; f.fb = (float)k; }
  else { f.fa = (float)k; f.fb = (float)(1.0 / R); }
  f.delta1 = (float)(1.25 * (bound(ds) + eps64) + 1e-6);
  if (method == M_FENG) {
    // t = a1 m + k1 x^(1+g) (m - L) + k2 x^g L, x = s / R, g >= 1 (x^g Lipschitz on [0, X]); L <= 255.
    // x~ = fl(s~ fl32(1/R)); x^g = ex2.approx(fl(g lg2.approx x~)): lg2.approx absolute error and
    // ex2.approx relative error each taken as 2^-19, the product's rounding u g |lg2 x| (x^g |lg2 x|
    // <= Z on [0, X]); x^(1+g) = fl(x^g x~); then the three terms and their sums, each rounded.
    const double a1 = rprm[0], k1 = rprm[1], k2 = rprm[2], g = rprm[3], Rr = rprm[4];
    const double iRf = (double)(float)(1.0 / Rr);
    // lg2.approx absolute and ex2.approx relative errors, taken as 2^-19 (as Phansalkar's ex2)
    const double e_lg = std::ldexp(1.0, -19), e_ex = std::ldexp(1.0, -19), ln2 = 0.6931471805599453;
    // the range of x~ and x (with the coarse |s~ - s| <= ds), and Z >= x^g |log2 x| on it
    const double dxc = ds * iRf + 127.5 * 1.01 * u / Rr + u * (127.5 + ds) * iRf;
    const double Xm = (127.5 + ds) * iRf * (1 + u) + dxc;
    const double xs = std::exp(-1.0 / g);  // the maximiser of x^g |ln x| on (0, 1]
    double Z = (xs <= Xm ? std::pow(xs, g) * (1.0 / g) / ln2 : std::pow(Xm, g) * std::fabs(std::log2(Xm)));
    if (Xm > 1.0) Z = std::max(Z, std::pow(Xm, g) * std::log2(Xm));
    const double Pg = std::pow(Xm, g);
    // the bound as a function of the bound xs_ on |s~ - s| (affine in it: Xm, P0m, P1m use the coarse ds)
    auto fb = [&](double xs_) {
      const double dx = xs_ * iRf + 127.5 * 1.01 * u / Rr + u * (127.5 + ds) * iRf;
      const double dP0 = g * std::pow(Xm, g - 1.0) * dx + 1.01 * ln2 * (Pg * g * e_lg + u * g * Z) * 1.01 +
                         Pg * e_ex * 1.01 + std::ldexp(1.0, -126);
      const double dP0c = g * std::pow(Xm, g - 1.0) * dxc + 1.01 * ln2 * (Pg * g * e_lg + u * g * Z) * 1.01 +
                          Pg * e_ex * 1.01 + std::ldexp(1.0, -126);
      const double P0m = Pg * (1 + 1e-5) + dP0c, P1m = P0m * Xm;
      const double dP1 = dP0 * Xm + P0m * dx + 1.01 * u * P1m;
      const double dT1 = std::fabs(a1) * dm + 2.02 * u * std::fabs(a1) * (255.0 + dm);
      const double dT2 = std::fabs(k1) * (dP1 * 255.0 + P1m * (dm + 1.01 * u * 255.0)) +
                         3.03 * u * std::fabs(k1) * P1m * (255.0 + dm);
      const double dT3 = std::fabs(k2) * dP0 * 255.0 + 2.02 * u * std::fabs(k2) * P0m * 255.0;
      const double tmax = (std::fabs(a1) + std::fabs(k1) * P1m + std::fabs(k2) * P0m) * (255.0 + dm);
      return dT1 + dT2 + dT3 + 2.02 * u * tmax + 1.01 * u * (255.0 + tmax);
    };
    f.fa = (float)a1;
    f.fb = (float)iRf;
    f.delta1 = (float)(1.25 * (fb(ds) + eps64) + 1e-6);
    // data-dependent form (as Niblack's): |s~ - s| <= min(sqrt dv, dv (1 + eps) / s~) + eps (smax + sqrt dv)
    const double f0 = fb(0.0), f1 = fb(1.0) - f0, xe = eps_sqrt * (smax + rv);
    f.rb0 = (float)((1.25 * (f0 + f1 * xe + eps64) + 1e-6) * (1 + 1e-6));
    f.rb1 = (float)(1.25 * f1 * (1 + 1e-6));
    f.rdv = (float)(dv * (1 + eps_sqrt) * (1 + 1e-6));
    f.rsdv = (float)(rv * (1 + 1e-6));
    return f;
  }
  if (method == M_RAIS) {
    // t = m + 0.3 f s, f = (a - b) / max(a, b), a = m s, b = M S (the page's).  |df/da|, |df/db| <= 1/b
    // on both sides of a = b, so |f(a~, b~) - f| <= (|a~ - a| + |b~ - b|) / (b (1 - 2u)); f~'s own
    // roundings (subtraction, rcp.approx <= 2u, product) add 4.04u (|f| <= 1).  delta1 holds the part
    // independent of b, rb1 the coefficient of 1/b (the kernel adds rb1 / (M S) per page).
    // As functions of the bound x on |s~ - s| (x <= ds, the coarse one): A(x) (independent of b) and
    // B(x) / b, both affine in x ((sx + x) <= sx + ds in B's product)
    const double sx = 127.5;
    const double dg0 = 0.3 * (4.04 * u * 1.01 + 1.02 * u) + 0.61 * u;   // |g~ - 0.3 f| less the Da / b part
    auto A = [&](double x) {
      return dm + 0.3 * x + (sx + x) * dg0 + 1.01 * u * 0.3 * (sx + x) + 2.02 * u * (255.0 + 0.3 * (sx + x));
    };
    auto B = [&](double x) {  // (sx + ds) 0.3 |a~ - m s|, |a~ - m s| <= 255 x + sx dm + dm x + roundings
      const double Da = 255.0 * x + sx * dm + dm * x + 1.01 * u * (255.0 + dm) * (sx + ds);
      return (sx + ds) * 0.3 * Da * (1.0 + 4 * u);
    };
    f.delta1 = (float)(1.25 * (A(ds) + eps64) + 1e-6);
    f.rais_c = (float)(1.25 * B(ds) * (1 + 1e-6));
    // data-dependent: x = min(sqrt dv, dv (1 + eps) / s~) + eps (smax + sqrt dv), as Niblack's
    const double a0 = A(0.0), a1 = A(1.0) - a0, b0 = B(0.0), b1 = B(1.0) - b0;
    const double xe = eps_sqrt * (smax + rv);
    f.rb0 = (float)((1.25 * (a0 + a1 * xe + eps64) + 1e-6) * (1 + 1e-6));
    f.rais_r0 = (float)(1.25 * (b0 + b1 * xe) * (1 + 1e-6) * (1 + 1e-6));
    f.rb1 = (float)(1.25 * a1 * (1 + 1e-6));
    f.rais_r1 = (float)(1.25 * b1 * (1 + 1e-6));
    f.rdv = (float)(dv * (1 + eps_sqrt) * (1 + 1e-6));
    f.rsdv = (float)(rv * (1 + 1e-6));
    return f;
  }
  // data-dependent form (Niblack, Khurshid): |s~ - s| <= min(sqrt dv, dv (1 + eps) / s~) + eps (smax + sqrt dv);
  // bound(ds) is affine in ds
  const double b0 = bound(0.0), b1 = bound(1.0) - b0;
  f.rb0 = (float)((1.25 * (b0 + b1 * eps_sqrt * (smax + rv) + eps64) + 1e-6) * (1 + 1e-6));
  f.rb1 = (float)(1.25 * b1 * (1 + 1e-6));
  f.rdv = (float)(dv * (1 + eps_sqrt) * (1 + 1e-6));
  f.rsdv = (float)(rv * (1 + 1e-6));
  return f;
}

// The v5 rules' extra operands (MomParams aux0 / aux1, moments5.cuh aux_operand):
// Khurshid 1/(h w) (N_mode 0); Phansalkar p and q log2(e)
void rule_aux_v5(int method, const double* rprm, double hw, float* aux0, float* aux1) {
  *aux0 = *aux1 = 0.0f;
  if (method == M_FENG) { *aux0 = (float)rprm[1]; *aux1 = (float)rprm[2]; }  // k1, k2 (gamma: aux2)
  if (method == M_KHURSHID) *aux0 = (float)(1.0 / hw);
  if (method == M_PHANSALKAR) { *aux0 = (float)rprm[2]; *aux1 = (float)(rprm[3] * 1.4426950408889634); }
}

// Khurshid, Phansalkar (q >= 0), Rais and Feng (gamma >= 1) run on v5 behind
// the certified filter when its bound is usable (small against the 0.5
// spacing of the integer pixels; Rais's is formed per page from M S); other
// parameters stay on the exact v3 path
bool rule_on_v5(int method, const double* rprm, double hw) {
  if (method == M_RAIS) return true;  // the bound is formed per page from M S (filter_consts_v5)
  if (method == M_FENG) {  // gamma >= 1: x^gamma Lipschitz at 0; a bound small against the pixel spacing
    for (int z = 0; z < 5; ++z)
      if (!std::isfinite(rprm[z])) return false;
    if (!(rprm[3] >= 1.0) || !(rprm[4] > 0.0)) return false;
    const FilterConsts f = filter_consts_v5(method, 0.0, 1.0, rprm);
    return std::isfinite(f.delta1) && f.delta1 < 8.0f;
  }
  if (method != M_KHURSHID && method != M_PHANSALKAR) return false;
  for (int z = 0; z < 4; ++z)
    if (!std::isfinite(rprm[z])) return false;
  if (method == M_PHANSALKAR && !(rprm[3] >= 0.0)) return false;
  const FilterConsts f = filter_consts_v5(method, 0.0, 1.0, rprm);
  float a0, a1;
  rule_aux_v5(method, rprm, hw, &a0, &a1);
  return std::isfinite(f.delta1) && f.delta1 < 8.0f && std::isfinite(a0) && std::isfinite(a1);
}

// The device's SM count (cudaDevAttrMultiProcessorCount), cached per device;
// grids and band models are sized in multiples of it.
int num_sms() {
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    cache[dev] = (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0) ? n : 148;
  }
  return cache[dev];
}

// Resident warp-CTAs per SM of the v4/v5 kernels (launch bounds: 16), as the
// dynamic shared memory allows (per-SM capacity less the per-block reserve).
int warp_cta_slots(size_t dyn_smem) {
  int dev = 0, cap = 0, rsv = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 16;
  static std::atomic<int> cap_c[64], rsv_c[64];  // per-device attributes (0: not read yet)
  if (dev >= 0 && dev < 64 && cap_c[dev].load(std::memory_order_relaxed) > 0) {
    cap = cap_c[dev].load(std::memory_order_relaxed);
    rsv = rsv_c[dev].load(std::memory_order_relaxed);
    return std::max(1, std::min(16, (int)(cap / (dyn_smem + (size_t)rsv))));
  }
  if (cudaDeviceGetAttribute(&cap, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess) return 16;
  if (cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) rsv = 1024;
  if (dev >= 0 && dev < 64) {
    rsv_c[dev].store(rsv, std::memory_order_relaxed);
    cap_c[dev].store(cap, std::memory_order_relaxed);
  }
  const int per = (int)(cap / (dyn_smem + (size_t)rsv));
  return std::max(1, std::min(16, per));
}

// Validation shared by every entry point.
int check_common(const void* in, int64_t H, int64_t W, int64_t in_pitch, const void* out, int64_t out_pitch,
                 int32_t fmt, int32_t h, int32_t w) {
  if (!in || !out) return ABIN_EINVAL;
  if (H < 1 || W < 1 || h < 1 || w < 1) return ABIN_EINVAL;
  if (H > kMaxDim || W > kMaxDim) return ABIN_ERANGE;
  if (in_pitch < W) return ABIN_EINVAL;
  if (fmt != ABIN_MASK_U8 && fmt != ABIN_MASK_BITS) return ABIN_EINVAL;
  const int64_t row_bytes = fmt == ABIN_MASK_U8 ? W : (W + 7) / 8;
  if (out_pitch < row_bytes) return ABIN_EINVAL;
  return ABIN_OK;
}

// The moments path (Sauvola / Niblack / Wolf) for a batch of pages or a band.
struct MomCall {
  int32_t method;
  const uint8_t* in;          // first held row of page 0
  int64_t in_page_stride;
  int64_t buf_rows;           // rows held per page (tensor-map height)
  int64_t buf_row0;           // global row of the first held row
  int64_t n_pages;
  int64_t W, in_pitch;
  int64_t row0, H_out, H_global;
  uint8_t* out;
  int64_t out_pitch, out_page_stride;
  int32_t fmt, h, w;
  double k, R;
  int32_t L_override;
  uint32_t flags;
  uint64_t* counters;
  cudaStream_t stream;
  // stats
  uint64_t *c_out, *d_out;
  uint32_t* n_out;
  double* t_out;
  uint8_t* mask_out;
  // Table 1 rules (methods 5..8): parameters, see abin.h
  double rprm[5];
  // M_MAXS (Wolf's adaptive R): per-page max s as double bits (device)
  unsigned long long* smax_out;
};

// Row bands: pick the band count so that the tile count fills whole waves
// of resident CTAs while keeping the h-row warm-up (pure vertical adds) short.
void choose_bands(int64_t col_tiles, int64_t H_out, int32_t h, int resident, int32_t* B, int32_t* n_bands) {
  double best = 1e30;
  int64_t bestB = H_out;
  for (int64_t nb = 1; nb <= std::max<int64_t>(1, H_out / 32); ++nb) {
    const int64_t Bc = (H_out + nb - 1) / nb;
    const int64_t tiles = col_tiles * ((H_out + Bc - 1) / Bc);
    const int64_t waves = (tiles + resident - 1) / resident;
    // cost ~ waves x (B rows + h/3 warm-up rows, warm-up rows are cheaper)
    const double cost = (double)waves * (double)(Bc + h / 3.0);
    if (cost < best * 0.999) { best = cost; bestB = Bc; }
    if (tiles > 64 * resident) break;
  }
  *B = (int32_t)bestB;
  *n_bands = (int32_t)((H_out + bestB - 1) / bestB);
}

// v4 (one warp per CTA, tiles of very different cost at the borders): the
// makespan is about  total work / slots + one tile  (the last wave's tail),
// with a tile costing its B rows plus h warm-up rows at a fraction wu of a row each.
// More, shorter bands shrink the tail; the warm-up rows bound how short.
void choose_bands_v4(int64_t col_tiles, int64_t H_out, int32_t h, int slots, int32_t* B, int32_t* n_bands) {
  double best = 1e300;
  int64_t bestB = H_out;
  const int64_t nb_max = std::max<int64_t>(1, H_out / 16);
  // weight of a warm-up row (vertical sums only) against an output row, fitted
  // on the band-count sweeps (tools/band_w.py, tools/bands.py, tools/abt.py with
  // ABIN_V4_WU): 0.3 for single narrow pages (config 2: +10-14 % at h = 127 /
  // 255), 0.5 for small batches and wide pages (16 config-3 pages, config 4),
  // 0.8 for large batches, whose many waves make warm-up rows count more than
  // the tail (64 config-3 pages: 699 -> 714 Gpx/s)
  const double wu = env_real("ABIN_V4_WU", col_tiles < 32 ? 0.3 : (col_tiles >= 512 ? 0.8 : 0.5), 0.0, 8.0);
  for (int64_t nb = 1; nb <= nb_max; ++nb) {
    const int64_t Bc = (H_out + nb - 1) / nb;
    const int64_t tiles = col_tiles * ((H_out + Bc - 1) / Bc);
    const double cost = (double)Bc + wu * h;
    const double t = (double)tiles * cost / slots + cost;
    if (t < best * 0.999) { best = t; bestB = Bc; }
  }
  *B = (int32_t)bestB;
  *n_bands = (int32_t)((H_out + bestB - 1) / bestB);
}

int encode_map(const MomCall& c, int box_rows, bool tma_ok, CUtensorMap* map) {
  memset(map, 0, sizeof(*map));
  if (!tma_ok) return ABIN_OK;
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "cuTensorMapEncodeTiled unavailable");
    return ABIN_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)c.W, (cuuint64_t)c.buf_rows, (cuuint64_t)c.n_pages};
  cuuint64_t strides[2] = {(cuuint64_t)c.in_pitch,
                           (cuuint64_t)(c.n_pages > 1 ? c.in_page_stride : c.in_pitch * c.buf_rows)};
  cuuint32_t box[3] = {256, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(c.in), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    return ABIN_ECUDA;
  }
  return ABIN_OK;
}

// v4 view of the pages: {16 bytes, ceil(W/16) chunks, rows, pages}; a box is
// `chunks` whole chunks x `rows` rows (moments4.cuh).  Needs 16-byte aligned
// base, pitch and page stride.
int encode_map_chunks(const MomCall& c, int chunks, int rows, CUtensorMap* map, int box_pages = 1) {
  memset(map, 0, sizeof(*map));
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "cuTensorMapEncodeTiled unavailable");
    return ABIN_ECUDA;
  }
  cuuint64_t dims[4] = {16, (cuuint64_t)((c.W + 15) / 16), (cuuint64_t)c.buf_rows, (cuuint64_t)c.n_pages};
  cuuint64_t strides[3] = {16, (cuuint64_t)c.in_pitch,
                           (cuuint64_t)(c.n_pages > 1 ? c.in_page_stride : c.in_pitch * c.buf_rows)};
  cuuint32_t box[4] = {16, (cuuint32_t)chunks, (cuuint32_t)rows, (cuuint32_t)box_pages};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult cr = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(c.in), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "cuTensorMapEncodeTiled (chunks) failed (%d)", (int)cr);
    return ABIN_ECUDA;
  }
  return ABIN_OK;
}

// The library's scratch (fixup queue, Wolf minima, rule accumulators) comes
// from the device's default stream-ordered pool.  Keep up to 512 MB of it
// cached across calls (the default threshold 0 hands it back to the driver
// at every synchronisation, and the next call pays for re-mapping it).
static void keep_pool_warm() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (thr < (512ull << 20)) {
      thr = 512ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  done[dev] = true;
}

int launch_fixup(const MomParams& q, int w, cudaStream_t st);

// The small-call path (small.cuh): one launch of k_small for single small
// pages -- tiles in shared memory, certified fp32 decision with the double
// threshold inline, no fixup launch.  Returns -1 (nothing launched) when the
// call is not one it takes.
int run_small(const MomCall& c, const Window& win) {
  using namespace sm;
  const bool stats = c.c_out || c.d_out || c.n_out || c.t_out || c.mask_out;
  const uint32_t forced = ABIN_FORCE_FP64 | ABIN_FORCE_U64_SQ | ABIN_V3_INTERNAL | ABIN_V4_INTERNAL |
                          ABIN_NO_TMA_INTERNAL;
  // Size limit of the tile kernel, measured against the streaming kernels on one
  // page (tools/dev/small_big.py, us per call at 15 / 31 / 63 windows): 1024^2
  // 10.3 / 10.3 / 12.4 vs 27.9 / 27.7 / 31.9; 2048^2 26.7 / 28.8 / 33.6 vs 31.9 /
  // 31.7 / 35.9; 3300 x 2550 53 / 56 / 68 vs 45 / 44 / 51: 2^22 pixels.
  // ABIN_SMALL_PX: tests / experiments (0: off).
  const int64_t max_px = env_int("ABIN_SMALL_PX", 1ll << 22, 0, 1ll << 30);
  if (stats || (c.flags & forced) || win.h > kMaxWin || win.w > kMaxWin ||
      !(c.method == M_SAUVOLA || c.method == M_NIBLACK || c.method == M_WOLF) ||
      c.n_pages * c.H_out * c.W > max_px)
    return -1;
  SmallParams p;
  memset(&p, 0, sizeof(p));
  p.in = c.in; p.in_page_stride = c.in_page_stride; p.in_pitch = c.in_pitch; p.W = c.W;
  p.buf_row0 = c.buf_row0; p.row0 = c.row0; p.H_out = c.H_out; p.H_global = c.H_global;
  p.out = c.out; p.out_pitch = c.out_pitch; p.out_page_stride = c.out_page_stride; p.fmt = c.fmt;
  p.h = win.h; p.w = win.w; p.l = win.l; p.r = win.r; p.o = win.o; p.u = win.u;
  p.RWp = (kTW + win.w - 1 + 15 + 15) / 16 * 16;
  p.CWp = (kTW + win.w + 3) / 4 * 4 + 1;
  p.n_ct = (int32_t)((c.W + kTW - 1) / kTW);
  // tile height 32 once 16-row tiles would fill the device several times over
  // (4 resident CTAs per SM): measured in tools/dev/small_big.py
  const int64_t tiles16 = (c.H_out + 15) / 16 * p.n_ct * c.n_pages;
  const int TH = tiles16 > env_int("ABIN_SMALL_TH32", 8, 0, 1 << 20) * num_sms() ? 32 : 16;
  p.n_rt = (int32_t)((c.H_out + TH - 1) / TH);
  const FilterConsts f5 = filter_consts_v5(c.method, c.k, c.R, c.rprm);
  p.fa = f5.fa; p.fb = f5.fb; p.delta1 = f5.delta1;
  p.k = c.k; p.R = c.R;
  p.L_fixed = c.L_override;
  p.counters = reinterpret_cast<unsigned long long*>(c.counters);
  unsigned int* Lw = nullptr;
  if (c.method == M_WOLF && c.L_override < 0) {
    CK(cudaMallocAsync(&Lw, (size_t)c.n_pages * 4 + (size_t)c.n_pages, c.stream));
    uint8_t* l8 = reinterpret_cast<uint8_t*>(Lw + c.n_pages);
    k_fill_u32<<<(unsigned)((c.n_pages + 255) / 256), 256, 0, c.stream>>>(Lw, c.n_pages, 0xFFu);
    k_global_min<<<dim3((unsigned)num_sms(), (unsigned)c.n_pages), 256, 0, c.stream>>>(c.in, c.in_page_stride, c.H_out,
                                                                                      c.W, c.in_pitch, Lw);
    k_narrow_u8<<<(unsigned)((c.n_pages + 255) / 256), 256, 0, c.stream>>>(Lw, l8, c.n_pages);
    p.L_page = l8;
  }
  const size_t smem = smem_bytes(p.RWp, p.CWp, win.h, TH);
  static bool attr[3][2][64] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const int mi = c.method == M_SAUVOLA ? 0 : (c.method == M_NIBLACK ? 1 : 2);
  const int ti = TH == 32 ? 1 : 0;
  const void* kerns[3][2] = {{(const void*)k_small<M_SAUVOLA, 16>, (const void*)k_small<M_SAUVOLA, 32>},
                             {(const void*)k_small<M_NIBLACK, 16>, (const void*)k_small<M_NIBLACK, 32>},
                             {(const void*)k_small<M_WOLF, 16>, (const void*)k_small<M_WOLF, 32>}};
  const void* kern = kerns[mi][ti];
  if (dev >= 0 && dev < 64 && !attr[mi][ti][dev]) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr[mi][ti][dev] = true;
  }
  void* args[] = {&p};
  const int64_t n = (int64_t)p.n_rt * p.n_ct * c.n_pages;
  int rc = ABIN_OK;
  if (n > 0) {
    const cudaError_t e = cudaLaunchKernel(kern, dim3((unsigned)n), dim3(sm::kNT), args, smem, c.stream);
    if (e != cudaSuccess) rc = cuda_fail(e);
  }
  if (Lw) {
    const cudaError_t f = cudaFreeAsync(Lw, c.stream);
    if (rc == ABIN_OK && f != cudaSuccess) return cuda_fail(f);
  }
  return rc;
}

int run_moments(const MomCall& c) {
  keep_pool_warm();
  const Window win = effective_window(c.h, c.w, c.H_global, c.W);
  if ((uint64_t)win.h > 66051u) return ABIN_ERANGE;  // column D_j must fit uint32 (255^2 h < 2^32)
  const int KH = (win.w + 1 + kG - 1) / kG;
  const bool fast = KH <= 31 && !(c.flags & ABIN_WIDE_INTERNAL);
  const int nt_wide = fast ? 0 : choose_nt_wide(win.w);
  if (!fast && nt_wide == 0) return ABIN_ERANGE;
  // TMA needs a 16-byte aligned base and strides; otherwise the kernels'
  // generic loader stages the rows.
  const bool tma_ok = !((reinterpret_cast<uintptr_t>(c.in) & 15u) || (c.in_pitch & 15) ||
                        (c.n_pages > 1 && (c.in_page_stride & 15))) && !(c.flags & ABIN_NO_TMA_INTERNAL);
  if (fast && (uint64_t)255 * (uint64_t)win.h * (uint64_t)win.w < (1ull << 32)) {
    const int rs = run_small(c, win);  // single small pages: the one-launch tile kernel
    if (rs >= 0) return rs;
  }
  if (!tma_ok && fast && !(c.flags & ABIN_NO_TMA_INTERNAL)) {
    // Rows TMA cannot stage (unaligned base, pitch or page stride, e.g. a tight
    // 2550-byte row): re-pitch them into a 16-byte aligned scratch copy (one
    // 2-D device copy, about half the kernel's own HBM traffic) and take the
    // TMA kernels, ~10x faster than the generic loader.  If the scratch
    // cannot be had, the generic loader runs.
    const int64_t pitch16 = (c.W + 15) & ~(int64_t)15;
    const int64_t rows = c.buf_rows;
    uint8_t* scratch = nullptr;
    if (cudaMallocAsync(&scratch, (size_t)pitch16 * rows * c.n_pages, c.stream) == cudaSuccess) {
      cudaError_t e = cudaSuccess;
      if (c.n_pages == 1 || c.in_page_stride == rows * c.in_pitch) {
        e = cudaMemcpy2DAsync(scratch, pitch16, c.in, c.in_pitch, c.W, rows * c.n_pages, cudaMemcpyDeviceToDevice,
                              c.stream);
      } else {
        for (int64_t pg = 0; pg < c.n_pages && e == cudaSuccess; ++pg)
          e = cudaMemcpy2DAsync(scratch + pg * pitch16 * rows, pitch16, c.in + pg * c.in_page_stride, c.in_pitch, c.W,
                                rows, cudaMemcpyDeviceToDevice, c.stream);
      }
      int rc = ABIN_OK;
      if (e == cudaSuccess) {
        MomCall c2 = c;
        c2.in = scratch;
        c2.in_pitch = pitch16;
        c2.in_page_stride = pitch16 * rows;
        rc = run_moments(c2);
      }
      const cudaError_t f = cudaFreeAsync(scratch, c.stream);
      if (e != cudaSuccess) return cuda_fail(e);
      if (rc == ABIN_OK && f != cudaSuccess) return cuda_fail(f);
      return rc;
    }
    (void)cudaGetLastError();  // no scratch: the generic loader below
  }
  // window sums c are uint32 in the kernels: exact while 255 h w < 2^32
  if ((uint64_t)255 * (uint64_t)win.h * (uint64_t)win.w >= (1ull << 32)) return ABIN_ERANGE;
  const bool rule = c.method >= ABIN_FENG && c.method <= ABIN_PHANSALKAR;
  const bool stats = c.c_out || c.d_out || c.n_out || c.t_out || c.mask_out;
  // v4 (warp CTAs, certified fp32 + deferred exact fixup) for the production
  // path; the v3 kernel (inline exact path) for rules, statistics, forced fp64
  // and rows TMA cannot stage
  const bool d64_sq = (c.flags & ABIN_FORCE_U64_SQ) || (uint64_t)win.h * (uint64_t)win.w * 65025u >= (1ull << 32);
  const bool v5_rule = rule && rule_on_v5(c.method, c.rprm, (double)win.h * (double)win.w) && !d64_sq &&
                       win.h <= v5::kMaxH && win.w <= v5::kMaxW && !(c.flags & ABIN_V4_INTERNAL);
  const bool use_v4 = fast && tma_ok && !(c.flags & ABIN_V3_INTERNAL) && (!rule || v5_rule) && !stats &&
                      !(c.flags & ABIN_FORCE_FP64);
  CUtensorMap map, map4;
  int rc = encode_map(c, fast ? kR : (nt_wide == 128 ? 8 : 4), tma_ok, &map);
  if (rc == ABIN_OK && use_v4) rc = encode_map_chunks(c, v4::kChunks, v4::kR, &map4);
  if (rc) return rc;

  unsigned int* Lw = nullptr;
  const uint8_t* L8 = nullptr;
  if ((c.method == M_WOLF || c.method == ABIN_FENG) && c.L_override < 0) {
    CK(cudaMallocAsync(&Lw, (size_t)c.n_pages * 4 + (size_t)c.n_pages, c.stream));
    uint8_t* l8 = reinterpret_cast<uint8_t*>(Lw + c.n_pages);
    k_fill_u32<<<(unsigned)((c.n_pages + 255) / 256), 256, 0, c.stream>>>(Lw, c.n_pages, 0xFFu);
    // pages are whole images here (band mode requires L_override)
    k_global_min<<<dim3((unsigned)num_sms(), (unsigned)c.n_pages), 256, 0, c.stream>>>(c.in, c.in_page_stride, c.H_out, c.W,
                                                                         c.in_pitch, Lw);
    k_narrow_u8<<<(unsigned)((c.n_pages + 255) / 256), 256, 0, c.stream>>>(Lw, l8, c.n_pages);
    CK(cudaGetLastError());
    L8 = l8;
  }
  // Rais: per-page global mean / standard deviation M, S
  unsigned long long* acc = nullptr;
  RuleParams rp;
  memset(&rp, 0, sizeof(rp));
  for (int z = 0; z < 5; ++z) rp.p[z] = c.rprm[z];
  rp.hw = (double)c.h * (double)c.w;
  if (c.method == ABIN_RAIS) {
    CK(cudaMallocAsync(&acc, (size_t)c.n_pages * 32, c.stream));
    CK(cudaMemsetAsync(acc, 0, (size_t)c.n_pages * 16, c.stream));
    double* MS = reinterpret_cast<double*>(acc + 2 * c.n_pages);
    k_global_sums<<<dim3((unsigned)num_sms(), (unsigned)c.n_pages), 256, 0, c.stream>>>(c.in, c.in_page_stride, c.H_out, c.W,
                                                                          c.in_pitch, acc);
    k_mean_std<<<(unsigned)((c.n_pages + 127) / 128), 128, 0, c.stream>>>(acc, MS, c.n_pages,
                                                                            (double)c.H_out * (double)c.W);
    CK(cudaGetLastError());
    rp.MS = MS;
  }
  const bool d64 = (c.flags & ABIN_FORCE_U64_SQ) || (uint64_t)win.h * (uint64_t)win.w * 65025u >= (1ull << 32);
  const int ph = ((-win.w) % 4 + 4) % 4;
  uint4* queue = nullptr;

  if (fast) {
    MomParams p;
    memset(&p, 0, sizeof(p));
    p.use_tma = tma_ok ? 1 : 0;
    p.in = c.in; p.in_pitch = c.in_pitch; p.in_page_stride = c.in_page_stride; p.buf_rows = c.buf_rows;
    p.W = c.W; p.H_out = c.H_out; p.row0 = c.row0; p.H_global = c.H_global; p.buf_row0 = c.buf_row0;
    p.out = c.out; p.out_pitch = c.out_pitch; p.out_page_stride = c.out_page_stride;
    p.h = win.h; p.w = win.w; p.l = win.l; p.r = win.r; p.o = win.o; p.u = win.u;
    p.fmt = c.fmt;
    p.KH = KH;
    p.Tw = kG * (32 - KH);
    p.n_strips = (int32_t)((c.W + (int64_t)kCW * p.Tw - 1) / ((int64_t)kCW * p.Tw));
    choose_bands((int64_t)p.n_strips * c.n_pages, c.H_out, win.h, num_sms() * 4, &p.B, &p.n_bands);
    p.method = c.method;
    p.force_fp64 = ((c.flags & ABIN_FORCE_FP64) || rule) ? 1 : 0;  // rules: every pixel in IEEE double
    p.rp = rp;
    p.k = c.k; p.R = c.R;
    p.L_page = L8; p.L_fixed = c.L_override;
    const FilterConsts f = filter_consts(c.method, c.k, c.R);
    p.fa = f.fa; p.fb = f.fb; p.delta1 = f.delta1; p.delta2 = f.delta2;
    p.rb0 = f.rb0; p.rb1 = f.rb1; p.rdv = f.rdv; p.rsdv = f.rsdv;
    p.inv_h = 1.0f / (float)win.h;
    p.counters = c.counters;
    p.counters_n = (c.flags & ABIN_COUNT_STAGES) ? 3 : 2;
    p.c_out = c.c_out; p.d_out = c.d_out; p.n_out = c.n_out; p.t_out = c.t_out; p.mask_out = c.mask_out;
    p.stats = stats ? 1 : 0;
    const int w32 = win.w % 32;
    const int64_t n_tiles3 = (int64_t)p.n_strips * p.n_bands * c.n_pages;
    if (use_v4) {
      MomParams q = p;
      // v5 (moments5.cuh) where its exactness conditions hold: biased fp32
      // column sums need 255^2 h < 2^23, the published row pads ceil(w/16) <= 8
      // lanes; uint32 square sums (no forced uint64)
      const bool use_v5 = !d64 && win.h <= v5::kMaxH && win.w <= v5::kMaxW && !(c.flags & ABIN_V4_INTERNAL);
      if (use_v5) {
        q.KH = (win.w + kG - 1) / kG;
        q.Tw = kG * (32 - q.KH);
        const FilterConsts f5 = filter_consts_v5(c.method, c.k, c.R, c.rprm);
        q.fa = f5.fa; q.fb = f5.fb; q.delta1 = f5.delta1;
        rule_aux_v5(c.method, c.rprm, (double)win.h * (double)win.w, &q.aux0, &q.aux1);
        if (c.method == M_FENG) q.aux2 = (float)c.rprm[3];  // gamma
        if (c.method == M_RAIS) {  // the bounds' 1 / (M S) coefficients
          q.aux1 = f5.rais_c;
          q.aux0 = f5.rais_r0;
          q.rais_r1 = f5.rais_r1;
        }
        q.rb0 = f5.rb0; q.rb1 = f5.rb1; q.rdv = f5.rdv; q.rsdv = f5.rsdv;
      }
      // one warp per CTA; a strip = one warp's 32 - KH valid lanes
      q.n_strips = (int32_t)((c.W + q.Tw - 1) / q.Tw);
      // strips whose windows stay inside [0, W) (ncol = w) are
      // [sL, sR); the others take the border variant of the kernel
      const int64_t Tw = q.Tw;
      const int64_t sL = std::min<int64_t>(q.n_strips, win.l - 1 > 0 ? (win.l - 1 + Tw - 1) / Tw : 0);
      const int64_t nfit = (c.W - win.r - Tw) >= 0 ? (c.W - win.r - Tw) / Tw + 1 : 0;
      q.sL = (int32_t)sL;
      q.sR = (int32_t)std::max<int64_t>(sL, std::min<int64_t>(nfit, q.n_strips));
      q.n_pages_v4 = (int32_t)c.n_pages;
      // Packed last strips (v5, page batches): when the last strip of a page
      // holds only a few output lanes (config 3: 32 of 448 columns), the last
      // strips of NG pages share one warp -- G = KH + its output lanes each,
      // one TMA box of NG pages -- instead of a mostly idle warp per page
      CUtensorMap mpk = map4;
      if (use_v5 && c.method != M_MAXS && c.n_pages >= 2 && q.n_strips >= 2 && !env_flag("ABIN_NO_PACK")) {
        const int64_t rem = c.W - (int64_t)(q.n_strips - 1) * q.Tw;  // outputs of the last strip
        const int G = q.KH + (int)((rem + kG - 1) / kG);
        const int NG = std::min(32 / G, v5::kRowsBytes / (v5::kR * kG * (G + 1)));
        if (NG >= 2 && q.sR <= q.n_strips - 1 && q.sL <= q.n_strips - 1) {
          rc = encode_map_chunks(c, G + 1, v5::kR, &mpk, NG);
          if (rc != ABIN_OK) return rc;
          q.pk_on = 1;
          q.pk_G = G;
          q.pk_NG = NG;
          q.pk_n = (int32_t)((c.n_pages + NG - 1) / NG);
        }
      }
      const int64_t col_tiles = q.pk_on ? (int64_t)(q.n_strips - 1) * c.n_pages + q.pk_n
                                        : (int64_t)q.n_strips * c.n_pages;
      choose_bands_v4(col_tiles, c.H_out, win.h,
                      num_sms() * (use_v5 ? occupancy_v5_any(win.w % 32, c.method) : warp_cta_slots(v4::smem_bytes())),
                      &q.B, &q.n_bands);
      if (const long long want_nb = env_int("ABIN_V4_BANDS", 0, 0, c.H_out)) {  // experiments: force the band count
        const int64_t want = std::max<int64_t>(1, want_nb);
        q.B = (int32_t)((c.H_out + want - 1) / want);
        q.n_bands = (int32_t)((c.H_out + q.B - 1) / q.B);
      }
      // the exact-fixup queue: 16 bytes per ambiguous lane (16 pixels)
      // at most one entry per output lane-row: calls below the cap cannot
      // overflow, so they need no follow-up launch and a smaller queue
      const int64_t max_entries = c.n_pages * c.H_out * ((c.W + 15) / 16 + q.n_strips + 1);
      uint32_t cap = (uint32_t)std::min<int64_t>(1 << 22, max_entries);  // <= 64 MB: one A4 page at 600 dpi fits
      if (env_int("ABIN_QUEUE_CAP", 0, 0, 1ll << 26) > 0)  // tests: exercise the overflow follow-up
        cap = (uint32_t)env_int("ABIN_QUEUE_CAP", 0, 1, 1ll << 26);
      const bool may_overflow = max_entries > (int64_t)cap;
      CK(cudaMallocAsync(&queue, (size_t)cap * 16 + 16, c.stream));
      uint32_t* qcount = reinterpret_cast<uint32_t*>(queue + (size_t)cap);
      CK(cudaMemsetAsync(qcount, 0, 4, c.stream));
      q.q_data = queue;
      q.q_count = qcount;
      q.q_cap = cap;
      const int64_t n_tiles = q.pk_on ? ((int64_t)(q.n_strips - 1) * c.n_pages + q.pk_n) * q.n_bands
                                      : (int64_t)q.n_strips * q.n_bands * c.n_pages;
      if (c.method == M_MAXS) {
        // Wolf's adaptive R (R21): pass 0 = max v~ per page, pass 1 = the
        // pixels within 2 |v~ - v| of it (the true maximum is among them),
        // then their exact s (k_fixup, canonical double sequence)
        if (!use_v5 || may_overflow) {
          cudaFreeAsync(queue, c.stream);
          return ABIN_ERANGE;
        }
        uint32_t* vmax = nullptr;
        CK(cudaMallocAsync(&vmax, (size_t)c.n_pages * 4, c.stream));
        CK(cudaMemsetAsync(vmax, 0, (size_t)c.n_pages * 4, c.stream));
        CK(cudaMemsetAsync(c.smax_out, 0, (size_t)c.n_pages * 8, c.stream));
        q.vmax_bits = vmax;
        q.smax_bits = c.smax_out;
        q.maxs_margin = 2.05f * q.rdv;
        q.maxs_pass = 0;
        rc = launch_v5_any(w32, map4, map4, q, n_tiles, c.stream);
        q.maxs_pass = 1;
        if (rc == ABIN_OK) rc = launch_v5_any(w32, map4, map4, q, n_tiles, c.stream);
        if (rc == ABIN_OK) rc = launch_fixup(q, win.w, c.stream);
        cudaError_t e1 = cudaFreeAsync(vmax, c.stream), e2 = cudaFreeAsync(queue, c.stream);
        if (rc == ABIN_OK && e1 != cudaSuccess) return cuda_fail(e1);
        if (rc == ABIN_OK && e2 != cudaSuccess) return cuda_fail(e2);
        return rc;
      }
      rc = use_v5 ? launch_v5_any(w32, map4, mpk, q, n_tiles, c.stream)
                  : launch_v4_any(w32, d64, map4, q, n_tiles, c.stream);
      if (rc == ABIN_OK) rc = launch_fixup(q, win.w, c.stream);
      if (rc == ABIN_OK && may_overflow) {
        // overflow (pathological inputs only): the v3 kernel redoes the call
        // exactly; its CTAs return at once when the queue held everything
        p.ovf_count = qcount;
        p.ovf_cap = cap;
        // about one CTA per SM: the (normal) empty launch costs little
        const int64_t per_band = (int64_t)p.n_strips * c.n_pages;
        const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(c.H_out, num_sms() / per_band));
        p.B = (int32_t)((c.H_out + nb - 1) / nb);
        p.n_bands = (int32_t)((c.H_out + p.B - 1) / p.B);
        rc = launch_fast_any(w32, d64, map, p, per_band * p.n_bands, c.stream);
      }
    } else {
      rc = launch_fast_any(w32, d64, map, p, n_tiles3, c.stream);
    }
  } else {
    wide::MomParams p;
    memset(&p, 0, sizeof(p));
    p.use_tma = tma_ok ? 1 : 0;
    p.in = c.in; p.in_pitch = c.in_pitch; p.in_page_stride = c.in_page_stride; p.buf_rows = c.buf_rows;
    p.W = c.W; p.H_out = c.H_out; p.row0 = c.row0; p.H_global = c.H_global; p.buf_row0 = c.buf_row0;
    p.out = c.out; p.out_pitch = c.out_pitch; p.out_page_stride = c.out_page_stride;
    p.h = win.h; p.w = win.w; p.l = win.l; p.r = win.r; p.o = win.o; p.u = win.u;
    p.fmt = c.fmt;
    p.KH = ((win.w + 1 + 8 - 1) / 8 + 1) & ~1;
    p.T = (nt_wide - p.KH - 2) * 8;
    p.n_strips = (int32_t)((c.W + p.T - 1) / p.T);
    choose_bands((int64_t)p.n_strips * c.n_pages, c.H_out, win.h, num_sms() * 2, &p.B, &p.n_bands);
    p.method = c.method;
    p.force_fp64 = 1;
    p.rp = rp;
    p.out_vec_ok = ((reinterpret_cast<uintptr_t>(c.out) | (uintptr_t)c.out_pitch |
                     (uintptr_t)(c.n_pages > 1 ? c.out_page_stride : 0)) & 7u) == 0;
    p.k = c.k; p.R = c.R;
    p.L_page = L8; p.L_fixed = c.L_override;
    p.counters = c.counters;
    p.c_out = c.c_out; p.d_out = c.d_out; p.n_out = c.n_out; p.t_out = c.t_out; p.mask_out = c.mask_out;
    const int64_t n_tiles = (int64_t)p.n_strips * p.n_bands * c.n_pages;
    rc = launch_wide_any(d64, stats, nt_wide, ph, map, p, n_tiles, c.stream);
  }
  if (Lw) {
    cudaError_t e = cudaFreeAsync(Lw, c.stream);
    if (rc == ABIN_OK && e != cudaSuccess) return cuda_fail(e);
  }
  if (acc) {
    cudaError_t e = cudaFreeAsync(acc, c.stream);
    if (rc == ABIN_OK && e != cudaSuccess) return cuda_fail(e);
  }
  if (queue) {
    cudaError_t e = cudaFreeAsync(queue, c.stream);
    if (rc == ABIN_OK && e != cudaSuccess) return cuda_fail(e);
  }
  return rc;
}

// Parameters of the batched / band / stats entry points: methods 0..4 (the
// Table-1 rules 5..8 take their own parameter array through
// abin_binarize_rule; these entry points have no place for it).
int check_params(int32_t method, double p0, double p1) {
  if (method < ABIN_SAUVOLA || method > ABIN_BERNSEN) return ABIN_EINVAL;
  if (method == ABIN_QUANTILE) return (std::isfinite(p0) && p0 > 0.0 && p0 <= 1.0) ? ABIN_OK : ABIN_EINVAL;
  if (method == ABIN_BERNSEN) return std::isfinite(p0) ? ABIN_OK : ABIN_EINVAL;  // contrast (< 0: plain midrange)
  if (!std::isfinite(p0)) return ABIN_EINVAL;
  if (method == ABIN_SAUVOLA)
    if (!std::isfinite(p1) || !(p1 > 0.0)) return ABIN_EINVAL;
  // Wolf: R > 0, or +inf (s / R = 0: the adaptive R of an all-constant page, R21)
  if (method == ABIN_WOLF)
    if (std::isnan(p1) || !(p1 > 0.0)) return ABIN_EINVAL;
  return ABIN_OK;
}


// k_fixup after the moments kernel on the same stream.  Its CTAs only read
// the queue count and exit when the fp32 filter decided every pixel, so the
// launch itself is the cost for most calls: occupancy is cached per device
// and window, and the launch is programmatic (PDL): the grid is scheduled as
// the moments kernel drains and waits in griddepcontrol.wait for its results.
int launch_fixup(const MomParams& q, int w, cudaStream_t st) {
  const size_t fsm = fixup_smem_bytes(w);
  static std::mutex mu;
  static int cache_w[64][8];
  static int cache_n[64][8];
  static bool inited[64] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return ABIN_EINVAL;
  int per_sm = -1;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!inited[dev]) {
      for (int z = 0; z < 8; ++z) cache_w[dev][z] = -1;
      inited[dev] = true;
    }
    for (int z = 0; z < 8; ++z)
      if (cache_w[dev][z] == w) per_sm = cache_n[dev][z];
  }
  if (per_sm < 0) {
    if (fsm > 48 * 1024) CK(cudaFuncSetAttribute(k_fixup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fixup, kFixNT, fsm));
    std::lock_guard<std::mutex> lock(mu);
    for (int z = 7; z > 0; --z) { cache_w[dev][z] = cache_w[dev][z - 1]; cache_n[dev][z] = cache_n[dev][z - 1]; }
    cache_w[dev][0] = w;
    cache_n[dev][0] = per_sm;
  }
  const unsigned grid = (unsigned)(num_sms() * std::max(1, per_sm));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFixNT);
    cfg.dynamicSmemBytes = fsm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_fixup, q));
  }
  CK(cudaGetLastError());
  return ABIN_OK;
}

int launch_q5_any(int wr, const q5::Q5Params& p, int64_t n, cudaStream_t st, int* occ) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (wr >> 2) {
    case 0: e = launch_q5_part0(wr, p, n, st, occ); break;
    case 1: e = launch_q5_part1(wr, p, n, st, occ); break;
    case 2: e = launch_q5_part2(wr, p, n, st, occ); break;
    case 3: e = launch_q5_part3(wr, p, n, st, occ); break;
  }
  return e == cudaSuccess ? ABIN_OK : cuda_fail(e);
}

// The v5 quantile kernel (quantile5.cuh) for the mask of method 3 where it
// applies: h <= 255, w <= 127 (vector row loads / mask stores where the
// pointers and pitches are aligned).  Returns -1 (nothing launched) otherwise.
int run_quant5(const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t W, int64_t in_pitch, uint8_t* out,
               int64_t out_pitch, int64_t out_page_stride, int32_t fmt, const Window& win, double q, int64_t row0,
               int64_t H_out, int64_t H_global, int64_t buf_rows, int64_t buf_row0, cudaStream_t st,
               uint64_t* counters) {
  if (win.w > q5::kMaxW || win.h > q5::kMaxH) return -1;
  q5::Q5Params p;
  memset(&p, 0, sizeof(p));
  // vector loads / stores where the rows allow (else byte-wise, same results)
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in), oa = reinterpret_cast<uintptr_t>(out);
  p.in_vec = !((ia & 15) || (in_pitch & 15) || (n_pages > 1 && (in_page_stride & 15)));
  const int64_t oal = fmt == ABIN_MASK_U8 ? 16 : 2;
  p.out_vec = !((int64_t)(oa % oal) || out_pitch % oal || (n_pages > 1 && out_page_stride % oal));
  p.in = in; p.in_page_stride = in_page_stride; p.in_pitch = in_pitch; p.W = W;
  p.buf_row0 = buf_row0; p.buf_rows = buf_rows; p.row0 = row0; p.H_out = H_out; p.H_global = H_global;
  p.out = out; p.out_pitch = out_pitch; p.out_page_stride = out_page_stride; p.fmt = fmt;
  p.h = win.h; p.w = win.w; p.l = win.l; p.r = win.r; p.o = win.o; p.u = win.u;
  p.q = q;
  p.KH = (win.w + 15) / 16;
  p.mq = win.w / 16;
  p.Tw = 16 * (32 - p.KH);
  p.n_strips = (int32_t)((W + p.Tw - 1) / p.Tw);
  // windows per tile: the median-like quantiles of document pages sit in the
  // background's level range (one window); the low ones in either the
  // strokes' or the background's (three windows placed at q/2, q, 2q of the
  // tile sample).  ABIN_Q5_NW overrides (experiments).
  int nw = q >= 0.2 ? 1 : 3;
  nw = (int)env_int("ABIN_Q5_NW", nw, 1, q5::kMaxNW);
  p.nw = nw;
  const float qf = (float)q;
  if (nw == 1) { p.qf[0] = qf; }
  else if (nw == 2) { p.qf[0] = 0.5f * qf; p.qf[1] = std::min(1.0f, 2.0f * qf); }
  else { p.qf[0] = 0.5f * qf; p.qf[1] = qf; p.qf[2] = std::min(1.0f, 2.0f * qf); }
  p.force_L = (int32_t)env_int("ABIN_Q5_FORCE_L", -1, 0, 240);  // tests (unset: -1, the sample's placement)
  const int wr = win.w % 16;
  int occ = 0;
  int rc = launch_q5_any(wr, p, 0, st, &occ);
  if (rc) return rc;
  {
    // bands: minimise waves x tile cost, a tile costing its B output rows plus
    // the h warm-up rows (column adds only: about a fifth of a row each) and
    // its set-up (sample histogram, tables: about four rows)
    const int64_t cols = (int64_t)p.n_strips * n_pages, slots = (int64_t)num_sms() * std::max(1, occ);
    const double wu = env_real("ABIN_Q5_WU", 0.2, 0.0, 8.0);  // experiments: warm-up row weight
    double best = 1e300;
    int64_t bestB = H_out;
    for (int64_t nb = 1; nb <= std::max<int64_t>(1, H_out / 4); ++nb) {
      const int64_t Bc = (H_out + nb - 1) / nb;
      const int64_t waves = (cols * ((H_out + Bc - 1) / Bc) + slots - 1) / slots;
      const double cost = (double)waves * ((double)Bc + wu * win.h + 4.0);
      if (cost < best * 0.999) { best = cost; bestB = Bc; }
      if (cols * nb > 64 * slots) break;
    }
    if (const long long want_nb = env_int("ABIN_Q5_BANDS", 0, 0, H_out)) {  // experiments: force the band count
      const int64_t want = std::max<int64_t>(1, want_nb);
      bestB = (H_out + want - 1) / want;
    }
    p.B = (int32_t)bestB;
    p.n_bands = (int32_t)((H_out + bestB - 1) / bestB);
  }
  // the exact queue: 16 bytes per undecided pixel; a full queue is decided inline
  const int64_t px = n_pages * H_out * W;
  uint32_t cap = (uint32_t)std::min<int64_t>(px, 1 << 20);
  cap = (uint32_t)env_int("ABIN_Q5_QCAP", cap, 1, cap);  // tests: a full queue decides inline
  uint4* queue = nullptr;
  CK(cudaMallocAsync(&queue, (size_t)cap * 16 + 16, st));
  uint32_t* qcount = reinterpret_cast<uint32_t*>(queue + cap);
  CK(cudaMemsetAsync(qcount, 0, 4, st));
  p.fq = queue; p.fq_count = qcount; p.fq_cap = cap;
  p.counters = reinterpret_cast<unsigned long long*>(counters);
  const int64_t n_tiles = (int64_t)p.n_strips * p.n_bands * n_pages;
  if (env_flag("ABIN_DEBUG"))
    fprintf(stderr, "q5: w %d h %d nw %d strips %d bands %d B %d occ %d tiles %lld\n", win.w, win.h, nw, p.n_strips,
            p.n_bands, p.B, occ, (long long)n_tiles);
  rc = launch_q5_any(wr, p, n_tiles, st, nullptr);
  if (rc == ABIN_OK) {
    cudaLaunchConfig_t cfg = {};  // programmatic launch (PDL), as launch_fixup
    cfg.gridDim = dim3((unsigned)(num_sms() * 2));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, q5::k_q5fix, p);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e);
  }
  const cudaError_t f = cudaFreeAsync(queue, st);
  if (rc == ABIN_OK && f != cudaSuccess) return cuda_fail(f);
  return rc;
}

// Bernsen (method 4) masks: the window-independent separable extrema of
// bernsen.cuh (row pass, then column pass with the decision).  Scratch: the
// row pass's (min, 255 - max) pairs and the column pass's suffix pairs, 2
// bytes per pixel each (an O(HW) departure from SURVEY 8(b), stated in abin.h).
int run_bernsen(const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t W, int64_t in_pitch, uint8_t* out,
                int64_t out_pitch, int64_t out_page_stride, int32_t fmt, const Window& win, double contrast,
                int64_t row0, int64_t H_out, int64_t H_global, int64_t buf_row0, cudaStream_t st) {
  using namespace bern;
  if (win.w > kBernMaxW) return ABIN_ERANGE;
  BernParams p;
  memset(&p, 0, sizeof(p));
  p.in = in; p.in_page_stride = in_page_stride; p.in_pitch = in_pitch; p.W = W; p.buf_row0 = buf_row0;
  p.row0 = row0; p.H_out = H_out; p.H_global = H_global;
  p.out = out; p.out_pitch = out_pitch; p.out_page_stride = out_page_stride; p.fmt = fmt;
  p.w = win.w; p.l = win.l; p.h = win.h; p.o = win.o;
  p.contrast = (int32_t)std::max(-1.0, std::min(256.0, std::floor(contrast)));
  p.Y0 = std::max<int64_t>(0, row0 - win.o + 1);
  p.Yn = std::min<int64_t>(H_global, row0 + H_out + win.u) - p.Y0;
  p.hpitch = (W + 7) / 8 * 8;
  p.TW = win.w <= 384 ? 128 : 256;  // (w > TW: one block per tile, its suffix pass spans the window)
  p.SP = (15 + p.TW + win.w + 15) / 16 * 16 + 4;
  p.OBP = p.TW + 2;
  p.n_ctiles = (int32_t)((W + p.TW - 1) / p.TW);
  p.n_rtiles = (int32_t)((p.Yn + 31) / 32);
  p.n_groups = (int32_t)((W + 7) / 8);
  p.n_chunks = (int32_t)((H_out + win.h - 1) / win.h);
  p.n_pages = (int32_t)n_pages;
  const size_t hsm = (size_t)h_smem_bytes(p.SP, p.w, p.OBP);
  if (hsm > 227 * 1024) return ABIN_ERANGE;
  // column pass: split each chunk over R threads until ~1.2M threads are in
  // flight (each keeps 4 row loads in flight); the local suffixes stay in
  // shared memory (16 bytes per thread and row) unless the window is too tall
  p.n_gblocks = (p.n_groups + 31) / 32;
  const int64_t base = (int64_t)p.n_gblocks * 32 * p.n_chunks * n_pages;
  int R = (int)std::max<int64_t>(1, std::min<int64_t>(8, (1200000 + base - 1) / std::max<int64_t>(1, base)));
  R = std::min(R, win.h);
  p.sbs = (win.h + R - 1) / R;
  R = (win.h + p.sbs - 1) / p.sbs;
  const size_t vsm_need = (size_t)R * 32 * p.sbs * 16;
  const bool v_smem = vsm_need <= 96 * 1024 && !env_flag("ABIN_BERN_GSB");  // (experiments: global sb)
  const size_t vsm = v_smem ? vsm_need : 0;
  void* scratch = nullptr;
  const size_t hb_bytes = (size_t)n_pages * p.Yn * p.hpitch * 2;
  const size_t sb_bytes = v_smem ? 0 : (size_t)n_pages * H_out * p.hpitch * 2;
  if (cudaMallocAsync(&scratch, hb_bytes + sb_bytes, st) != cudaSuccess) {
    (void)cudaGetLastError();
    return ABIN_ENOMEM;
  }
  p.hb = reinterpret_cast<uint16_t*>(scratch);
  p.sb = v_smem ? nullptr : reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(scratch) + hb_bytes);
  static bool attr_done[64] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if ((hsm > 48 * 1024 || vsm + sizeof(uint4) * 2 * 8 * 32 > 48 * 1024) && dev >= 0 && dev < 64 && !attr_done[dev]) {
    CK(cudaFuncSetAttribute(k_bern_h, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(k_bern_v, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done[dev] = true;
  }
  int rc = ABIN_OK;
  const int64_t nh = (int64_t)p.n_ctiles * p.n_rtiles * n_pages;
  const int64_t nv = (int64_t)p.n_gblocks * p.n_chunks * n_pages;
  if (nh > 0 && nv > 0) {
    k_bern_h<<<(unsigned)nh, 32, hsm, st>>>(p);
    k_bern_v<<<(unsigned)nv, dim3(32, R), vsm, st>>>(p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e);
  }
  const cudaError_t f = cudaFreeAsync(scratch, st);
  if (rc == ABIN_OK && f != cudaSuccess) return cuda_fail(f);
  return rc;
}

int run_quantile(int32_t method, const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t /*H_held*/, int64_t W,
                 int64_t in_pitch, uint8_t* out, int64_t out_pitch, int64_t out_page_stride, int32_t fmt, int32_t h,
                 int32_t w, double q, int64_t row0, int64_t H_out, int64_t H_global, int64_t buf_rows,
                 int64_t buf_row0, cudaStream_t st, double* Q_out, uint32_t flags, uint64_t* counters) {
  const Window win = effective_window(h, w, H_global, W);
  if (method == ABIN_BERNSEN && !Q_out && !(flags & ABIN_Q2_INTERNAL))
    return run_bernsen(in, in_page_stride, n_pages, W, in_pitch, out, out_pitch, out_page_stride, fmt, win, q, row0,
                       H_out, H_global, buf_row0, st);
  // v5 (quantile5.cuh) for masks at q >= 0.25; low quantiles of document
  // pages sit in either the strokes' or the background's levels, which a few
  // 16-level windows per tile do not cover (measured: 1-35 % of the pixels to
  // the exact queue at q = 0.1), so they keep the round-1 kernels (config-5
  // page, tools/dev/q5_low.py: at q = 0.2 round-1 1.16 ms, v5 1.23-1.46 ms;
  // at q = 0.25 v5 0.70 ms, round-1 1.06 ms).
  // ABIN_Q5_ALWAYS (tests) takes v5 for every q.
  const bool q5_always = env_flag("ABIN_Q5_ALWAYS");
  if (method == ABIN_QUANTILE && !Q_out && !(flags & ABIN_Q2_INTERNAL) && (q >= 0.25 || q5_always)) {
    const int rc = run_quant5(in, in_page_stride, n_pages, W, in_pitch, out, out_pitch, out_page_stride, fmt, win, q,
                              row0, H_out, H_global, buf_rows, buf_row0, st, counters);
    if (rc >= 0) return rc;
  }
  constexpr int NT_ = kQuantNT;
  if ((int64_t)win.h * win.w > 65535) return ABIN_ERANGE;  // u16 bins
  if (NT_ + win.w - 1 > 4 * NT_) return ABIN_ERANGE;  // a thread stages at most 4 elements of a row
  constexpr int NT = 128;
  QuantParams p;
  memset(&p, 0, sizeof(p));
  p.in = in;
  p.in_page_stride = in_page_stride;
  p.in_pitch = in_pitch;
  p.W = W;
  p.buf_row0 = buf_row0;
  p.buf_rows = buf_rows;
  p.row0 = row0;
  p.H_out = H_out;
  p.H_global = H_global;
  p.out = out;
  p.out_pitch = out_pitch;
  p.out_page_stride = out_page_stride;
  p.fmt = fmt;
  p.h = win.h; p.w = win.w; p.l = win.l; p.r = win.r; p.o = win.o; p.u = win.u;
  p.q = q;
  // the paired-column kernel (k_quantile2: two outputs per thread sharing one
  // window histogram) for quantiles and Bernsen whose windows fit its packing
  // and rows it can stage; the rest take k_quantile
  // 32 threads (64 columns) per CTA where the window lets a warp stage its
  // rows (w <= 64: finer tiles, measured 1-10 % faster), else 64
  const int NT2 = win.w <= 64 ? 32 : 64;
  // (shared u16 words: counts + one row's transient adds stay below 2^16;
  // byte deltas 128 + Delta with |Delta| <= h + 2 transiently)
  const bool pair = (method == ABIN_QUANTILE || method == ABIN_BERNSEN) && win.h <= 125 && 2 * NT2 + win.w <= 4 * NT2 &&
                    (int64_t)(win.h + 1) * win.w <= 65535 &&
                    !env_flag("ABIN_QUANTILE_SINGLE");
  p.n_strips = (int32_t)(pair ? (W + 2 * NT2 - 1) / (2 * NT2) : (W + NT - 1) / NT);
  const int64_t cols = (int64_t)p.n_strips * n_pages;
  // low quantiles of document pages sit where the strokes' grey levels end:
  // the rank jumps across the empty bins up to the background's, row to row,
  // so their walks load 8 bins at a time (k_quantile2 MODE 2)
  const bool groups = pair && method == ABIN_QUANTILE && q < 0.25;
  const size_t smem = pair ? quantile2_smem_bytes(NT2, win.w) : quantile_smem_bytes(NT, win.w);
  if (smem > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_quantile<NT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(k_quantile<NT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (const void* f : {(const void*)k_quantile2<32, 0>, (const void*)k_quantile2<32, 1>,
                          (const void*)k_quantile2<32, 2>, (const void*)k_quantile2<64, 0>,
                          (const void*)k_quantile2<64, 1>, (const void*)k_quantile2<64, 2>})
      CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  }
  const int q2_mode = method == ABIN_BERNSEN ? 1 : (groups ? 2 : 0);
  const void* q2 = nullptr;
  if (pair) {
    const void* tab[2][3] = {{(const void*)k_quantile2<32, 0>, (const void*)k_quantile2<32, 1>,
                              (const void*)k_quantile2<32, 2>},
                             {(const void*)k_quantile2<64, 0>, (const void*)k_quantile2<64, 1>,
                              (const void*)k_quantile2<64, 2>}};
    q2 = tab[NT2 == 64][q2_mode];
  }
  // bands: a tile costs its B rows plus h warm-up rows at about half a row
  // each; minimise waves x tile cost over the resident CTA slots (few tiles
  // per page: the last wave's tail and the warm-up rows both matter)
  int per_sm = 0;
  if (pair) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, q2, NT2, smem));
  else if (method == ABIN_BERNSEN) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_quantile<NT, 1>, NT, smem));
  else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_quantile<NT, 0>, NT, smem));
  const int64_t slots = num_sms() * (int64_t)std::max(1, per_sm);
  int64_t B = H_out;
  double best = 1e300;
  const double qwu = env_real("ABIN_Q_WU", 0.5, 0.0, 8.0);  // experiments: warm-up row weight
  for (int64_t nb = 1; nb <= std::max<int64_t>(1, H_out / 16); ++nb) {
    const int64_t Bc = (H_out + nb - 1) / nb;
    const int64_t waves = (cols * ((H_out + Bc - 1) / Bc) + slots - 1) / slots;
    const double cost = (double)waves * ((double)Bc + qwu * win.h);
    if (cost < best * 0.999) { best = cost; B = Bc; }
    if (cols * nb > 64 * slots) break;
  }
  p.B = (int32_t)B;
  p.n_bands = (int32_t)((H_out + B - 1) / B);
  p.Q_out = Q_out;
  p.contrast = method == ABIN_BERNSEN ? (int32_t)std::max(-1.0, std::min(256.0, std::floor(q))) : -1;
  const int64_t n_tiles = (int64_t)p.n_strips * p.n_bands * n_pages;
  if (pair) {
    void* args[] = {&p};
    CK(cudaLaunchKernel(q2, dim3((unsigned)n_tiles), dim3(NT2), args, smem, st));
  } else if (method == ABIN_BERNSEN) k_quantile<NT, 1><<<(unsigned)n_tiles, NT, smem, st>>>(p);
  else k_quantile<NT, 0><<<(unsigned)n_tiles, NT, smem, st>>>(p);
  CK(cudaGetLastError());
  return ABIN_OK;
}


// ---- ABIN_HOST_IO: host buffers streamed through device staging ----------
// Pages move in chunks through NSTR internal streams (H2D copy, kernel, D2H
// copy per chunk; consecutive chunks overlap on different streams / copy
// engines).  The caller's stream waits for all of it.
struct HostIoStreams {
  int device = -1;
  static constexpr int kMax = 8;
  cudaStream_t s[kMax] = {};
  cudaEvent_t done[kMax] = {};
};

int get_host_io_streams(HostIoStreams** out) {
  static std::mutex mu;
  static HostIoStreams per_dev[64];
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return ABIN_EINVAL;
  std::lock_guard<std::mutex> lock(mu);
  HostIoStreams& h = per_dev[dev];
  if (h.device < 0) {
    for (int i = 0; i < HostIoStreams::kMax; ++i) {
      CK(cudaStreamCreateWithFlags(&h.s[i], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h.done[i], cudaEventDisableTiming));
    }
    h.device = dev;
  }
  *out = &h;
  return ABIN_OK;
}

int run_moments(const MomCall& c);
int run_quantile(int32_t method, const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t H_held, int64_t W,
                 int64_t in_pitch, uint8_t* out, int64_t out_pitch, int64_t out_page_stride, int32_t fmt, int32_t h,
                 int32_t w, double q, int64_t row0, int64_t H_out, int64_t H_global, int64_t buf_rows,
                 int64_t buf_row0, cudaStream_t st, double* Q_out, uint32_t flags, uint64_t* counters);

// Host <-> device copies of `rows` rows of `width` bytes.  Only the caller's
// `width` bytes per row are read or written (the padding of a row and the
// bytes past the last row belong to the caller): a single linear DMA when the
// rows are contiguous (pitch == width), else all rows but the last as one
// linear copy of whole pitches (host input only: reading a row's padding is
// harmless, the next row follows it) plus the last row, else a 2-D copy.
cudaError_t copy_rows_h2d(uint8_t* dst, int64_t dpitch, const uint8_t* src, int64_t spitch, int64_t width,
                          int64_t rows, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (spitch == dpitch) {
    cudaError_t e = cudaSuccess;
    if (rows > 1) e = cudaMemcpyAsync(dst, src, (size_t)((rows - 1) * spitch), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dst + (rows - 1) * dpitch, src + (rows - 1) * spitch, (size_t)width, cudaMemcpyHostToDevice, s);
    return e;
  }
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyHostToDevice, s);
}
cudaError_t copy_rows_d2h(uint8_t* dst, int64_t dpitch, const uint8_t* src, int64_t spitch, int64_t width,
                          int64_t rows, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (dpitch == width && spitch == width)
    return cudaMemcpyAsync(dst, src, (size_t)(rows * width), cudaMemcpyDeviceToHost, s);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, s);
}

int run_host_io(int32_t method, const uint8_t* in, int64_t in_page_stride, uint8_t* out, int64_t out_page_stride,
                int64_t P, int64_t H, int64_t W, int64_t in_pitch, int64_t out_pitch, int32_t fmt, int32_t h,
                int32_t w, double p0, double p1, int32_t L, uint32_t flags, uint64_t* counters, cudaStream_t st) {
  HostIoStreams* hs = nullptr;
  int rc = get_host_io_streams(&hs);
  if (rc) return rc;
  // device staging keeps the host pitch when it is TMA-friendly, so the copies are linear
  const int64_t dpitch = (in_pitch % 16 == 0) ? in_pitch : (W + 15) / 16 * 16;
  const int64_t orow = fmt == ABIN_MASK_U8 ? W : (W + 7) / 8;
  // the staged mask rows are tight (row bytes) when the caller's are: one
  // linear D2H copy; otherwise the caller's pitch (a 2-D copy of the row bytes)
  const int64_t dopitch = out_pitch == orow ? orow : ((out_pitch % 16 == 0) ? out_pitch : (orow + 15) / 16 * 16);
  const int64_t dpage = dpitch * H, dopage = dopitch * H;
  // chunk of pages per stream and the number of streams in flight (tunable
  // for experiments through ABIN_HOSTIO_CHUNK_MB / ABIN_HOSTIO_STREAMS)
  const int64_t chunk_mb = env_int("ABIN_HOSTIO_CHUNK_MB", 64, 1, 1 << 16);
  const int streams = (int)env_int("ABIN_HOSTIO_STREAMS", 4, 1, HostIoStreams::kMax);
  const int64_t target = env_int("ABIN_HOSTIO_CHUNK_BYTES", chunk_mb << 20, 1, 1ll << 40);  // tests: tiny chunks
  // row bands for the methods whose band path needs nothing page-global
  // (Wolf / Feng only with a given L; the rules' global sums and Otsu never)
  const bool band_ok = method == ABIN_SAUVOLA || method == ABIN_NIBLACK || method == ABIN_QUANTILE ||
                       method == ABIN_BERNSEN || ((method == ABIN_WOLF || method == ABIN_FENG) && L >= 0);
  const int64_t nb = std::min<int64_t>(H, (dpage + target - 1) / target);
  const bool split = band_ok && nb > 1;
  const int64_t R = (H + nb - 1) / nb;
  const int64_t held_max = std::min<int64_t>(H, R + (h + 1) / 2 - 1 + h / 2);
  int64_t pc = std::max<int64_t>(1, std::min<int64_t>(P, target / std::max<int64_t>(dpage, 1)));
  const int64_t n_chunks = split ? P * ((H + R - 1) / R) : (P + pc - 1) / pc;
  const int nstr = (int)std::min<int64_t>(std::max(1, std::min(streams, (int)HostIoStreams::kMax)), n_chunks);
  uint8_t* buf = nullptr;
  const size_t per = split ? (size_t)(held_max * dpitch + R * dopitch) : (size_t)(pc * (dpage + dopage));
  {
    cudaError_t e = cudaMallocAsync(&buf, per * nstr, st);
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? ABIN_ENOMEM : cuda_fail(e);
  }
  cudaEvent_t ready;
  CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CK(cudaEventRecord(ready, st));
  for (int i = 0; i < nstr; ++i) CK(cudaStreamWaitEvent(hs->s[i], ready, 0));
  const bool contiguous_in = P == 1 || in_page_stride == H * in_pitch;
  const bool contiguous_out = P == 1 || out_page_stride == H * out_pitch;
  if (split) {
    // pages larger than a chunk (a gigapixel scan) travel as row bands with
    // their window halos (o - 1 rows above, u below; the band path evaluates n
    // with the page's geometry): device staging stays a few chunks, not pages.
    // (Smaller chunks for ordinary pages measured slower end to end.)
    const int64_t o = (h + 1) / 2, u = h / 2;
    for (int64_t q = 0, ci = 0; q < P && rc == ABIN_OK; ++q) {
      for (int64_t b = 0; b < nb && rc == ABIN_OK; ++b, ++ci) {
        const int64_t r0 = b * R, r1 = std::min(H, r0 + R);
        if (r0 >= r1) break;
        const int64_t top = std::min(o - 1, r0), bot = std::min(u, H - r1), held = (r1 - r0) + top + bot;
        cudaStream_t s = hs->s[ci % nstr];
        uint8_t* din = buf + (ci % nstr) * per;
        uint8_t* dout = din + held_max * dpitch;
        const uint8_t* src = in + q * in_page_stride + (r0 - top) * in_pitch;
        CK(copy_rows_h2d(din, dpitch, src, in_pitch, W, held, s));
        if (method == ABIN_QUANTILE || method == ABIN_BERNSEN) {
          rc = run_quantile(method, din, 0, 1, held, W, dpitch, dout, dopitch, 0, fmt, h, w, p0, r0, r1 - r0, H, held,
                            r0 - top, s, nullptr, flags, counters);
        } else {
          MomCall m;
          memset(&m, 0, sizeof(m));
          m.method = method; m.in = din; m.buf_rows = held; m.buf_row0 = r0 - top; m.n_pages = 1;
          m.W = W; m.in_pitch = dpitch; m.row0 = r0; m.H_out = r1 - r0; m.H_global = H; m.out = dout;
          m.out_pitch = dopitch; m.fmt = fmt; m.h = h; m.w = w; m.k = p0; m.R = p1; m.L_override = L;
          m.flags = flags & ~(uint32_t)ABIN_HOST_IO; m.counters = counters; m.stream = s;
          rc = run_moments(m);
        }
        if (rc) break;
        CK(copy_rows_d2h(out + q * out_page_stride + r0 * out_pitch, out_pitch, dout, dopitch, orow, r1 - r0, s));
      }
    }
  }
  for (int64_t c0 = 0, ci = 0; !split && c0 < P && rc == ABIN_OK; c0 += pc, ++ci) {
    const int64_t np = std::min(pc, P - c0);
    cudaStream_t s = hs->s[ci % nstr];
    uint8_t* din = buf + (ci % nstr) * per;
    uint8_t* dout = din + pc * dpage;
    // linear DMAs where the layout allows (2-D copies run at about half the PCIe rate)
    if (contiguous_in) {
      CK(copy_rows_h2d(din, dpitch, in + c0 * in_page_stride, in_pitch, W, np * H, s));
    } else {
      for (int64_t q = 0; q < np; ++q) CK(copy_rows_h2d(din + q * dpage, dpitch, in + (c0 + q) * in_page_stride, in_pitch, W, H, s));
    }
    if (method == ABIN_QUANTILE || method == ABIN_BERNSEN) {
      rc = run_quantile(method, din, dpage, np, H, W, dpitch, dout, dopitch, dopage, fmt, h, w, p0, 0, H, H, H, 0, s, nullptr,
                        flags, counters);
    } else {
      MomCall m;
      memset(&m, 0, sizeof(m));
      m.method = method; m.in = din; m.in_page_stride = dpage; m.buf_rows = H; m.n_pages = np;
      m.W = W; m.in_pitch = dpitch; m.H_out = H; m.H_global = H; m.out = dout; m.out_pitch = dopitch;
      m.out_page_stride = dopage; m.fmt = fmt; m.h = h; m.w = w; m.k = p0; m.R = p1; m.L_override = L;
      m.flags = flags & ~(uint32_t)ABIN_HOST_IO; m.counters = counters; m.stream = s;
      rc = run_moments(m);
    }
    if (rc) break;
    if (contiguous_out) {
      CK(copy_rows_d2h(out + c0 * out_page_stride, out_pitch, dout, dopitch, orow, np * H, s));
    } else {
      for (int64_t q = 0; q < np; ++q)
        CK(copy_rows_d2h(out + (c0 + q) * out_page_stride, out_pitch, dout + q * dopage, dopitch, orow, H, s));
    }
  }
  for (int i = 0; i < nstr; ++i) {
    CK(cudaEventRecord(hs->done[i], hs->s[i]));
    CK(cudaStreamWaitEvent(st, hs->done[i], 0));
  }
  CK(cudaFreeAsync(buf, st));
  CK(cudaEventDestroy(ready));
  return rc;
}

}  // namespace

// ============================================================== public ABI

extern "C" {

int abin_binarize_batched(int32_t method, const uint8_t* in, int64_t in_page_stride, uint8_t* out,
                          int64_t out_page_stride, int64_t n_pages, int64_t H, int64_t W, int64_t in_pitch,
                          int64_t out_pitch, int32_t mask_format, int32_t h, int32_t w, double param0,
                          double param1, int32_t L_override, uint32_t flags, uint64_t* counters, void* stream) {
  int rc = check_common(in, H, W, in_pitch, out, out_pitch, mask_format, h, w);
  if (rc) return rc;
  if ((rc = check_params(method, param0, param1))) return rc;
  if (n_pages < 1) return ABIN_EINVAL;
  if (L_override > 255) return ABIN_EINVAL;
  const int64_t in_bytes = (H - 1) * in_pitch + W, out_row = mask_format == ABIN_MASK_U8 ? W : (W + 7) / 8;
  const int64_t out_bytes = (H - 1) * out_pitch + out_row;
  if (n_pages > 1 && (in_page_stride < in_bytes || out_page_stride < out_bytes)) return ABIN_EINVAL;
  const int64_t in_span = (n_pages - 1) * in_page_stride + in_bytes;
  const int64_t out_span = (n_pages - 1) * out_page_stride + out_bytes;
  if (overlaps(in, (size_t)in_span, out, (size_t)out_span)) return ABIN_EALIAS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (flags & ABIN_HOST_IO)
    return run_host_io(method, in, in_page_stride, out, out_page_stride, n_pages, H, W, in_pitch, out_pitch,
                       mask_format, h, w, param0, param1, L_override, flags, counters, st);
  if (method == ABIN_QUANTILE || method == ABIN_BERNSEN)
    return run_quantile(method, in, in_page_stride, n_pages, H, W, in_pitch, out, out_pitch, out_page_stride, mask_format, h,
                        w, param0, 0, H, H, H, 0, st, nullptr, flags, counters);
  MomCall c;
  memset(&c, 0, sizeof(c));
  c.method = method;
  c.in = in;
  c.in_page_stride = in_page_stride;
  c.buf_rows = H;
  c.buf_row0 = 0;
  c.n_pages = n_pages;
  c.W = W;
  c.in_pitch = in_pitch;
  c.row0 = 0;
  c.H_out = H;
  c.H_global = H;
  c.out = out;
  c.out_pitch = out_pitch;
  c.out_page_stride = out_page_stride;
  c.fmt = mask_format;
  c.h = h;
  c.w = w;
  c.k = param0;
  c.R = param1;
  c.L_override = L_override;
  c.flags = flags;
  c.counters = counters;
  c.stream = st;
  return run_moments(c);
}

int abin_sauvola(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                 int32_t mask_format, int32_t h, int32_t w, double k, double R, uint32_t flags, uint64_t* counters,
                 void* stream) {
  return abin_binarize_batched(ABIN_SAUVOLA, in, 0, out, 0, 1, H, W, in_pitch, out_pitch, mask_format, h, w, k, R,
                               -1, flags, counters, stream);
}

int abin_niblack(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                 int32_t mask_format, int32_t h, int32_t w, double k, uint32_t flags, uint64_t* counters,
                 void* stream) {
  return abin_binarize_batched(ABIN_NIBLACK, in, 0, out, 0, 1, H, W, in_pitch, out_pitch, mask_format, h, w, k,
                               128.0, -1, flags, counters, stream);
}

int abin_wolf(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
              int32_t mask_format, int32_t h, int32_t w, double k, double R, int32_t L_override, uint32_t flags,
              uint64_t* counters, void* stream) {
  return abin_binarize_batched(ABIN_WOLF, in, 0, out, 0, 1, H, W, in_pitch, out_pitch, mask_format, h, w, k, R,
                               L_override, flags, counters, stream);
}

int abin_quantile(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                  int32_t mask_format, int32_t h, int32_t w, double q, uint32_t flags, void* stream) {
  return abin_binarize_batched(ABIN_QUANTILE, in, 0, out, 0, 1, H, W, in_pitch, out_pitch, mask_format, h, w, q,
                               0.0, -1, flags, nullptr, stream);
}

int abin_binarize_rule(int32_t rule, const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out,
                       int64_t out_pitch, int32_t mask_format, int32_t h, int32_t w, const double* params,
                       int32_t n_params, uint32_t flags, uint64_t* counters, void* stream) {
  int rc = check_common(in, H, W, in_pitch, out, out_pitch, mask_format, h, w);
  if (rc) return rc;
  static const int need[4] = {5, 0, 2, 4};  // Feng, Rais, Khurshid, Phansalkar
  if (rule < ABIN_FENG || rule > ABIN_PHANSALKAR) return ABIN_EINVAL;
  const int k = need[rule - ABIN_FENG];
  if (n_params < k || (k > 0 && !params)) return ABIN_EINVAL;
  for (int z = 0; z < k; ++z)
    if (!std::isfinite(params[z])) return ABIN_EINVAL;
  if (rule == ABIN_FENG && !(params[4] > 0.0)) return ABIN_EINVAL;        // R
  if (rule == ABIN_PHANSALKAR && !(params[1] > 0.0)) return ABIN_EINVAL;  // R
  const int64_t out_row = mask_format == ABIN_MASK_U8 ? W : (W + 7) / 8;
  if (overlaps(in, (size_t)((H - 1) * in_pitch + W), out, (size_t)((H - 1) * out_pitch + out_row))) return ABIN_EALIAS;
  MomCall c;
  memset(&c, 0, sizeof(c));
  c.method = rule;
  c.in = in;
  c.buf_rows = H;
  c.n_pages = 1;
  c.W = W;
  c.in_pitch = in_pitch;
  c.H_out = H;
  c.H_global = H;
  c.out = out;
  c.out_pitch = out_pitch;
  c.fmt = mask_format;
  c.h = h;
  c.w = w;
  c.k = 0.0;
  c.R = 128.0;
  c.L_override = -1;
  c.flags = flags;
  c.counters = counters;
  c.stream = reinterpret_cast<cudaStream_t>(stream);
  for (int z = 0; z < k; ++z) c.rprm[z] = params[z];
  return run_moments(c);
}

int abin_otsu(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
              int32_t mask_format, uint8_t* t_out, uint32_t flags, void* stream) {
  (void)flags;
  int rc = check_common(in, H, W, in_pitch, out, out_pitch, mask_format, 1, 1);
  if (rc) return rc;
  const int64_t out_row = mask_format == ABIN_MASK_U8 ? W : (W + 7) / 8;
  if (overlaps(in, (size_t)((H - 1) * in_pitch + W), out, (size_t)((H - 1) * out_pitch + out_row))) return ABIN_EALIAS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long* hist = nullptr;
  CK(cudaMallocAsync(&hist, 256 * 8 + 16, st));
  uint8_t* tdev = reinterpret_cast<uint8_t*>(hist + 256);
  CK(cudaMemsetAsync(hist, 0, 256 * 8, st));
  const unsigned nb = (unsigned)std::min<int64_t>(H, 4 * num_sms());
  k_otsu_hist<<<dim3(nb, 1), 256, 0, st>>>(in, 0, H, W, in_pitch, hist);
  k_otsu_pick<<<1, 256, 0, st>>>(hist, t_out ? t_out : tdev, 1, (double)H * (double)W);
  k_otsu_mask<<<dim3(nb, 1), 256, 0, st>>>(in, 0, H, W, in_pitch, t_out ? t_out : tdev, out, out_pitch, 0,
                                            mask_format);
  cudaError_t e = cudaGetLastError();
  cudaError_t f = cudaFreeAsync(hist, st);
  if (e != cudaSuccess) return cuda_fail(e);
  if (f != cudaSuccess) return cuda_fail(f);
  return ABIN_OK;
}

int abin_bernsen(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                 int32_t mask_format, int32_t h, int32_t w, int32_t contrast, uint32_t flags, void* stream) {
  return abin_binarize_batched(ABIN_BERNSEN, in, 0, out, 0, 1, H, W, in_pitch, out_pitch, mask_format, h, w,
                               (double)contrast, 0.0, -1, flags, nullptr, stream);
}

int abin_binarize_band(int32_t method, const uint8_t* in, int64_t H_band, int64_t W, int64_t in_pitch, int64_t row0,
                       int64_t H_global, int32_t halo_top, int32_t halo_bot, uint8_t* out, int64_t out_pitch,
                       int32_t mask_format, int32_t h, int32_t w, double param0, double param1, int32_t L_override,
                       uint32_t flags, uint64_t* counters, void* stream) {
  const int64_t held = H_band + halo_top + halo_bot;
  int rc = check_common(in, held, W, in_pitch, out, out_pitch, mask_format, h, w);
  if (rc) return rc;
  if ((rc = check_params(method, param0, param1))) return rc;
  if (H_band < 1 || row0 < 0 || H_global < row0 + H_band || halo_top < 0 || halo_bot < 0) return ABIN_EINVAL;
  if (row0 - halo_top < 0 || row0 + H_band + halo_bot > H_global) return ABIN_EINVAL;
  const int64_t o = (h + 1) / 2, u = h / 2;
  if (halo_top < std::min<int64_t>(o - 1, row0)) return ABIN_EINVAL;
  if (halo_bot < std::min<int64_t>(u, H_global - row0 - H_band)) return ABIN_EINVAL;
  if (method == ABIN_WOLF && (L_override < 0 || L_override > 255)) return ABIN_EINVAL;
  const int64_t in_bytes = (held - 1) * in_pitch + W;
  const int64_t out_row = mask_format == ABIN_MASK_U8 ? W : (W + 7) / 8;
  if (overlaps(in, (size_t)in_bytes, out, (size_t)((H_band - 1) * out_pitch + out_row))) return ABIN_EALIAS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (method == ABIN_QUANTILE || method == ABIN_BERNSEN)
    return run_quantile(method, in, 0, 1, held, W, in_pitch, out, out_pitch, 0, mask_format, h, w, param0, row0, H_band,
                        H_global, held, row0 - halo_top, st, nullptr, flags, counters);
  MomCall c;
  memset(&c, 0, sizeof(c));
  c.method = method;
  c.in = in;
  c.buf_rows = held;
  c.buf_row0 = row0 - halo_top;
  c.n_pages = 1;
  c.W = W;
  c.in_pitch = in_pitch;
  c.row0 = row0;
  c.H_out = H_band;
  c.H_global = H_global;
  c.out = out;
  c.out_pitch = out_pitch;
  c.fmt = mask_format;
  c.h = h;
  c.w = w;
  c.k = param0;
  c.R = param1;
  c.L_override = L_override;
  c.flags = flags;
  c.counters = counters;
  c.stream = st;
  return run_moments(c);
}

int abin_global_min(const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t H, int64_t W,
                    int64_t in_pitch, uint8_t* L_out, void* stream) {
  if (!in || !L_out || n_pages < 1 || H < 1 || W < 1 || in_pitch < W) return ABIN_EINVAL;
  if (n_pages > 1 && in_page_stride < (H - 1) * in_pitch + W) return ABIN_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned int* Lw = nullptr;
  CK(cudaMallocAsync(&Lw, (size_t)n_pages * 4, st));
  k_fill_u32<<<(unsigned)((n_pages + 255) / 256), 256, 0, st>>>(Lw, n_pages, 0xFFu);
  k_global_min<<<dim3((unsigned)num_sms(), (unsigned)n_pages), 256, 0, st>>>(in, in_page_stride, H, W, in_pitch, Lw);
  k_narrow_u8<<<(unsigned)((n_pages + 255) / 256), 256, 0, st>>>(Lw, L_out, n_pages);
  cudaError_t e = cudaGetLastError();
  cudaError_t f = cudaFreeAsync(Lw, st);
  if (e != cudaSuccess) return cuda_fail(e);
  if (f != cudaSuccess) return cuda_fail(f);
  return ABIN_OK;
}

int abin_stats(int32_t method, const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, int32_t h, int32_t w,
               double param0, double param1, int32_t L_override, uint64_t* c_out, uint64_t* d_out, uint32_t* n_out,
               double* t_out, uint8_t* mask_out, void* stream) {
  if (!in || H < 1 || W < 1 || h < 1 || w < 1 || in_pitch < W) return ABIN_EINVAL;
  int rc = check_params(method, param0, param1);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* scratch = nullptr;  // the mask also goes to a throwaway U8 buffer
  CK(cudaMallocAsync(&scratch, (size_t)(H * W), st));
  if (method == ABIN_QUANTILE || method == ABIN_BERNSEN) {
    rc = run_quantile(method, in, 0, 1, H, W, in_pitch, scratch, W, 0, ABIN_MASK_U8, h, w, param0, 0, H, H, H, 0, st, t_out,
                      0, nullptr);
  } else {
    MomCall c;
    memset(&c, 0, sizeof(c));
    c.method = method;
    c.in = in;
    c.buf_rows = H;
    c.n_pages = 1;
    c.W = W;
    c.in_pitch = in_pitch;
    c.H_out = H;
    c.H_global = H;
    c.out = scratch;
    c.out_pitch = W;
    c.fmt = ABIN_MASK_U8;
    c.h = h;
    c.w = w;
    c.k = param0;
    c.R = param1;
    c.L_override = L_override;
    c.flags = ABIN_FORCE_FP64;
    c.stream = st;
    c.c_out = c_out;
    c.d_out = d_out;
    c.n_out = n_out;
    c.t_out = t_out;
    c.mask_out = mask_out;
    rc = run_moments(c);
  }
  if (mask_out && (method == ABIN_QUANTILE || method == ABIN_BERNSEN) && rc == ABIN_OK) {
    cudaError_t e = cudaMemcpyAsync(mask_out, scratch, (size_t)(H * W), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e);
  }
  cudaError_t f = cudaFreeAsync(scratch, st);
  if (rc == ABIN_OK && f != cudaSuccess) return cuda_fail(f);
  return rc;
}

int abin_max_s(const uint8_t* in, int64_t H_band, int64_t W, int64_t in_pitch, int64_t row0, int64_t H_global,
               int32_t halo_top, int32_t halo_bot, int32_t h, int32_t w, double* max_s, void* stream) {
  if (!in || !max_s || H_band < 1 || W < 1 || h < 1 || w < 1 || in_pitch < W) return ABIN_EINVAL;
  if (H_band > kMaxDim || W > kMaxDim || H_global > kMaxDim) return ABIN_ERANGE;
  if (row0 < 0 || H_global < row0 + H_band || halo_top < 0 || halo_bot < 0) return ABIN_EINVAL;
  const int64_t o = (h + 1) / 2, u = h / 2;
  // the band must hold every in-image row its windows reach (as abin_binarize_band)
  if (halo_top < std::min<int64_t>(o - 1, row0) || halo_bot < std::min<int64_t>(u, H_global - row0 - H_band))
    return ABIN_EINVAL;
  if (row0 - halo_top < 0 || row0 + H_band + halo_bot > H_global) return ABIN_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long* dmax = nullptr;
  CK(cudaMallocAsync(&dmax, 8, st));
  MomCall m;
  memset(&m, 0, sizeof(m));
  m.method = M_MAXS; m.in = in; m.buf_rows = H_band + halo_top + halo_bot; m.buf_row0 = row0 - halo_top;
  m.n_pages = 1; m.W = W; m.in_pitch = in_pitch; m.row0 = row0; m.H_out = H_band; m.H_global = H_global;
  m.out = nullptr; m.out_pitch = W; m.fmt = ABIN_MASK_U8; m.h = h; m.w = w; m.k = 0.0; m.R = 1.0;
  m.L_override = 0; m.stream = st; m.smax_out = dmax;
  int rc = run_moments(m);
  unsigned long long bits = 0;
  if (rc == ABIN_OK) {
    cudaError_t e = cudaMemcpyAsync(&bits, dmax, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e);
  }
  cudaFreeAsync(dmax, st);
  if (rc == ABIN_OK) memcpy(max_s, &bits, 8);
  return rc;
}

int abin_wolf_adaptive(const uint8_t* in, int64_t H, int64_t W, int64_t in_pitch, uint8_t* out, int64_t out_pitch,
                       int32_t mask_format, int32_t h, int32_t w, double k, int32_t L_override, uint32_t flags,
                       uint64_t* counters, double* R_out, void* stream) {
  int rc = check_common(in, H, W, in_pitch, out, out_pitch, mask_format, h, w);
  if (rc) return rc;
  if (!std::isfinite(k) || L_override > 255) return ABIN_EINVAL;
  double ms = 0.0;
  if ((rc = abin_max_s(in, H, W, in_pitch, 0, H, 0, 0, h, w, &ms, stream))) return rc;
  const double R = ms > 0.0 ? ms : INFINITY;  // all windows constant: s / R = 0 (R21)
  if (R_out) *R_out = R;
  return abin_binarize_batched(ABIN_WOLF, in, 0, out, 0, 1, H, W, in_pitch, out_pitch, mask_format, h, w, k, R,
                               L_override, flags, counters, stream);
}

int abin_probe_filter(int32_t method, double k, double R, double L, const double* rule_params, const uint32_t* c,
                      const uint32_t* d, const uint32_t* ncol, const uint32_t* nrow, const uint8_t* I, int64_t count,
                      float* e_out, float* s_out, double* bounds, void* stream) {
  if (count < 0) return ABIN_EINVAL;
  const bool rule = method == ABIN_KHURSHID || method == ABIN_PHANSALKAR || method == ABIN_FENG;
  if (!rule && method != ABIN_RAIS && (method < ABIN_SAUVOLA || method > ABIN_WOLF)) return ABIN_EINVAL;
  float aux0 = 0.0f, aux1 = 0.0f;
  const float aux2 = method == ABIN_FENG && rule_params ? (float)rule_params[3] : 0.0f;
  int nmode = 0;
  float Lprobe = (float)L;
  if (method == ABIN_RAIS) {
    // rule_params[0] = the page's M S; bounds[0] + bounds[2] / (M S) is the bound
    if (!rule_params || !std::isfinite(rule_params[0]) || !(rule_params[0] >= 0.0)) return ABIN_EINVAL;
    Lprobe = (float)rule_params[0];
  } else if (rule) {
    if (!rule_params) return ABIN_EINVAL;
    nmode = method == ABIN_KHURSHID && rule_params[1] != 0.0;
    if (method == ABIN_FENG && !(std::isfinite(L) && L >= 0.0 && L <= 255.0)) return ABIN_EINVAL;
    const double hw = method == ABIN_KHURSHID && !nmode ? rule_params[2] : 1.0;  // Khurshid's N = h w
    if (!(hw >= 1.0)) return ABIN_EINVAL;
    if (!rule_on_v5(method, rule_params, hw)) return ABIN_ERANGE;  // not a parameter set v5 takes
    rule_aux_v5(method, rule_params, hw, &aux0, &aux1);
  } else if (!std::isfinite(k) || !std::isfinite(R) || !(R > 0.0) || !std::isfinite(L)) {
    return ABIN_EINVAL;
  }
  const FilterConsts f = filter_consts_v5(method, k, R, rule_params);
  if (bounds) {
    bounds[0] = f.delta1; bounds[1] = f.rb0; bounds[2] = f.rb1; bounds[3] = f.rdv; bounds[4] = f.rsdv;
    if (method == ABIN_RAIS) {  // the bounds at this M S, as the kernel forms them per page
      const double MS = std::max((double)(float)rule_params[0], 1e-30);
      bounds[0] = f.delta1 + f.rais_c / MS;
      bounds[1] = f.rb0 + f.rais_r0 / MS;
      bounds[2] = f.rb1 + f.rais_r1 / MS;
    }
  }
  if (count == 0) return ABIN_OK;
  if (!c || !d || !ncol || !nrow || !I || !e_out) return ABIN_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned nb = (unsigned)((count + 255) / 256);
  const float Lf = Lprobe;
#define ABIN_PROBE(M) \
  v5::k_probe<M><<<nb, 256, 0, st>>>(c, d, ncol, nrow, I, count, f.fa, f.fb, Lf, aux0, aux1, aux2, nmode, e_out, s_out)
  if (method == M_SAUVOLA) ABIN_PROBE(M_SAUVOLA);
  else if (method == M_RAIS) ABIN_PROBE(M_RAIS);
  else if (method == M_FENG) ABIN_PROBE(M_FENG);
  else if (method == M_NIBLACK) ABIN_PROBE(M_NIBLACK);
  else if (method == M_WOLF) ABIN_PROBE(M_WOLF);
  else if (method == M_KHURSHID) ABIN_PROBE(M_KHURSHID);
  else ABIN_PROBE(M_PHANSALKAR);
#undef ABIN_PROBE
  CK(cudaGetLastError());
  return ABIN_OK;
}

void abin_limits(abin_limits_t* out) {
  if (!out) return;
  out->max_window_w = 190 * 8 - 1;                // the CTA-wide kernel's halo (choose_nt_wide)
  out->max_window_h = 66051;                      // 255^2 h < 2^32
  out->max_window_hw = ((1ll << 32) - 1) / 255;   // 255 h w < 2^32
  out->max_dim = kMaxDim;
  out->quantile_max_window_w = 3 * kQuantNT + 1;  // a thread stages at most 4 elements of a row
  out->quantile_max_window_hw = 65535;            // u16 bins
  out->bernsen_max_window_w = bern::kBernMaxW;    // the row pass's staged tile (no h or h w limit)
}

const char* abin_strerror(int status) {
  switch (status) {
    case ABIN_OK: return "ok";
    case ABIN_EINVAL: return "invalid argument";
    case ABIN_EALIAS: return "input and output overlap";
    case ABIN_ERANGE: return "window, image or alignment outside the supported range";
    case ABIN_ECUDA: return "CUDA error";
    case ABIN_ENOMEM: return "out of memory";
  }
  return "unknown status";
}

const char* abin_version(void) { return "abin 0.2 (sm_100a)"; }

const char* abin_last_cuda_error(void) { return g_last_cuda_error; }

}  // extern "C"
