// abin_api.cu -- the C ABI of libabin.so (include/abin.h): argument
// validation, tiling decisions, TMA tensor maps and kernel launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "../../include/abin.h"
#include "globalmin.cuh"
#include "moments.cuh"
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

constexpr int G = 8;
// internal test hook: force the generic (non-TMA) loader
constexpr uint32_t ABIN_NO_TMA_INTERNAL = 1u << 30;
constexpr int64_t kMaxDim = (int64_t)1 << 30;

int choose_nt(int32_t w_eff) {
  const int kh = (((w_eff + 1 + G - 1) / G) + 1) & ~1;
  if (kh <= 64) return 128;
  if (kh <= 190) return 256;
  return 0;  // unsupported by the strip kernel
}

template <int NT, int PH, bool D64, bool STATS>
int launch_moments_t(const CUtensorMap& map, const MomParams& p, int64_t n_tiles, cudaStream_t st) {
  constexpr int R_ = (NT == 128) ? 8 : 4;
  constexpr size_t smem = moments_smem_bytes<NT, G, R_, D64>();
  auto kern = k_moments<NT, G, PH, R_, D64, STATS>;
  static bool attr_set = false;  // benign race: the attribute value is idempotent
  if (!attr_set) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  kern<<<(unsigned)n_tiles, NT, smem, st>>>(map, p);
  CK(cudaGetLastError());
  return ABIN_OK;
}

template <bool D64, bool STATS>
int launch_moments_nt(int nt, int ph, const CUtensorMap& map, const MomParams& p, int64_t n_tiles,
                      cudaStream_t st) {
#define ABIN_PH(NT_)                                                         \
  switch (ph) {                                                              \
    case 0: return launch_moments_t<NT_, 0, D64, STATS>(map, p, n_tiles, st); \
    case 1: return launch_moments_t<NT_, 1, D64, STATS>(map, p, n_tiles, st); \
    case 2: return launch_moments_t<NT_, 2, D64, STATS>(map, p, n_tiles, st); \
    default: return launch_moments_t<NT_, 3, D64, STATS>(map, p, n_tiles, st); \
  }
  if (nt == 128) ABIN_PH(128)
  ABIN_PH(256)
#undef ABIN_PH
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
};

int run_moments(const MomCall& c) {
  const Window win = effective_window(c.h, c.w, c.H_global, c.W);
  const int nt = choose_nt(win.w);
  if (nt == 0) return ABIN_ERANGE;
  if ((uint64_t)win.h > 66051u) return ABIN_ERANGE;  // column D_j must fit uint32 (255^2 h < 2^32)
  // TMA needs a 16-byte aligned base and strides; otherwise the kernel's
  // generic loader stages the rows.
  const bool tma_ok = !((reinterpret_cast<uintptr_t>(c.in) & 15u) || (c.in_pitch & 15) ||
                        (c.n_pages > 1 && (c.in_page_stride & 15))) && !(c.flags & ABIN_NO_TMA_INTERNAL);
  PFN_encodeTiled enc = get_encode();
  if (tma_ok && !enc) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "cuTensorMapEncodeTiled unavailable");
    return ABIN_ECUDA;
  }
  const int R_ = nt == 128 ? 8 : 4;
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  if (tma_ok) {
  cuuint64_t dims[3] = {(cuuint64_t)c.W, (cuuint64_t)c.buf_rows, (cuuint64_t)c.n_pages};
  cuuint64_t strides[2] = {(cuuint64_t)c.in_pitch,
                           (cuuint64_t)(c.n_pages > 1 ? c.in_page_stride : c.in_pitch * c.buf_rows)};
  cuuint32_t box[3] = {256, (cuuint32_t)R_, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(c.in), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    return ABIN_ECUDA;
  }
  }
  MomParams p;
  memset(&p, 0, sizeof(p));
  p.use_tma = tma_ok ? 1 : 0;
  p.in = c.in;
  p.in_pitch = c.in_pitch;
  p.in_page_stride = c.in_page_stride;
  p.buf_rows = c.buf_rows;
  p.W = c.W;
  p.H_out = c.H_out;
  p.row0 = c.row0;
  p.H_global = c.H_global;
  p.buf_row0 = c.buf_row0;
  p.out = c.out;
  p.out_pitch = c.out_pitch;
  p.out_page_stride = c.out_page_stride;
  p.h = win.h; p.w = win.w; p.l = win.l; p.r = win.r; p.o = win.o; p.u = win.u;
  p.fmt = c.fmt;
  // KH halo threads (>= ceil((w+1)/G), rounded up to even so that strip
  // origins stay 16-byte aligned); the last 2 threads only feed the byte
  // funnel of their neighbours and produce no output.
  p.KH = ((win.w + 1 + G - 1) / G + 1) & ~1;
  p.T = (nt - p.KH - 2) * G;
  p.n_strips = (int32_t)((c.W + p.T - 1) / p.T);
  // Row bands: enough tiles for several waves, long enough to amortise the
  // h-row warm-up.
  {
    const int64_t tiles_cols = (int64_t)p.n_strips * c.n_pages;
    int64_t B = 1024;
    while (B > 64 && tiles_cols * ((c.H_out + B - 1) / B) < 148 * 6) B /= 2;
    p.B = (int32_t)B;
    p.n_bands = (int32_t)((c.H_out + B - 1) / B);
  }
  p.method = c.method;
  p.force_fp64 = (c.flags & ABIN_FORCE_FP64) ? 1 : 0;
  p.out_vec_ok = ((reinterpret_cast<uintptr_t>(c.out) | (uintptr_t)c.out_pitch |
                   (uintptr_t)(c.n_pages > 1 ? c.out_page_stride : 0)) & 7u) == 0;
  p.k = c.k;
  p.R = c.R;
  p.L_fixed = c.L_override;
  p.counters = c.counters;
  p.c_out = c.c_out; p.d_out = c.d_out; p.n_out = c.n_out; p.t_out = c.t_out; p.mask_out = c.mask_out;

  unsigned int* Lw = nullptr;
  uint8_t* L8 = nullptr;
  if (c.method == M_WOLF && c.L_override < 0) {
    CK(cudaMallocAsync(&Lw, (size_t)c.n_pages * 4 + (size_t)c.n_pages, c.stream));
    L8 = reinterpret_cast<uint8_t*>(Lw + c.n_pages);
    k_fill_u32<<<(unsigned)((c.n_pages + 255) / 256), 256, 0, c.stream>>>(Lw, c.n_pages, 0xFFu);
    // pages are whole images here (band mode requires L_override)
    k_global_min<<<dim3(148, (unsigned)c.n_pages), 256, 0, c.stream>>>(c.in, c.in_page_stride, c.H_out, c.W,
                                                                         c.in_pitch, Lw);
    k_narrow_u8<<<(unsigned)((c.n_pages + 255) / 256), 256, 0, c.stream>>>(Lw, L8, c.n_pages);
    CK(cudaGetLastError());
    p.L_page = L8;
  }
  const bool d64 = (c.flags & ABIN_FORCE_U64_SQ) || (uint64_t)win.h * (uint64_t)win.w * 65025u >= (1ull << 32);
  const int ph = ((-win.w) % 4 + 4) % 4;
  const int64_t n_tiles = (int64_t)p.n_strips * p.n_bands * c.n_pages;
  const bool stats = c.c_out || c.d_out || c.n_out || c.t_out || c.mask_out;
  int rc;
  if (stats)
    rc = d64 ? launch_moments_nt<true, true>(nt, ph, map, p, n_tiles, c.stream)
             : launch_moments_nt<false, true>(nt, ph, map, p, n_tiles, c.stream);
  else
    rc = d64 ? launch_moments_nt<true, false>(nt, ph, map, p, n_tiles, c.stream)
             : launch_moments_nt<false, false>(nt, ph, map, p, n_tiles, c.stream);
  if (Lw) {
    cudaError_t e = cudaFreeAsync(Lw, c.stream);
    if (rc == ABIN_OK && e != cudaSuccess) return cuda_fail(e);
  }
  return rc;
}

int check_params(int32_t method, double p0, double p1) {
  if (method == ABIN_QUANTILE) return (std::isfinite(p0) && p0 > 0.0 && p0 <= 1.0) ? ABIN_OK : ABIN_EINVAL;
  if (!std::isfinite(p0)) return ABIN_EINVAL;
  if (method == ABIN_SAUVOLA || method == ABIN_WOLF)
    if (!std::isfinite(p1) || !(p1 > 0.0)) return ABIN_EINVAL;
  if (method < 0 || method > 3) return ABIN_EINVAL;
  return ABIN_OK;
}


int run_quantile(const uint8_t* in, int64_t in_page_stride, int64_t n_pages, int64_t /*H_held*/, int64_t W,
                 int64_t in_pitch, uint8_t* out, int64_t out_pitch, int64_t out_page_stride, int32_t fmt, int32_t h,
                 int32_t w, double q, int64_t row0, int64_t H_out, int64_t H_global, int64_t buf_rows,
                 int64_t buf_row0, cudaStream_t st, double* Q_out) {
  const Window win = effective_window(h, w, H_global, W);
  if (win.w > 8192 || (int64_t)win.h * win.w > 65535) return ABIN_ERANGE;  // u16 bins
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
  p.n_strips = (int32_t)((W + NT - 1) / NT);
  int64_t B = 512;
  const int64_t cols = (int64_t)p.n_strips * n_pages;
  while (B > 4 * (int64_t)win.h && B > 32 && cols * ((H_out + B - 1) / B) < 148 * 4) B /= 2;
  p.B = (int32_t)B;
  p.n_bands = (int32_t)((H_out + B - 1) / B);
  p.Q_out = Q_out;
  const size_t smem = quantile_smem_bytes(NT, win.w);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_quantile<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const int64_t n_tiles = (int64_t)p.n_strips * p.n_bands * n_pages;
  k_quantile<NT><<<(unsigned)n_tiles, NT, smem, st>>>(p);
  CK(cudaGetLastError());
  return ABIN_OK;
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
  if (flags & ABIN_HOST_IO) return ABIN_EINVAL;  // not implemented yet
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (method == ABIN_QUANTILE)
    return run_quantile(in, in_page_stride, n_pages, H, W, in_pitch, out, out_pitch, out_page_stride, mask_format, h,
                        w, param0, 0, H, H, H, 0, st, nullptr);
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
  if (method == ABIN_QUANTILE)
    return run_quantile(in, 0, 1, held, W, in_pitch, out, out_pitch, 0, mask_format, h, w, param0, row0, H_band,
                        H_global, held, row0 - halo_top, st, nullptr);
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
  k_global_min<<<dim3(148, (unsigned)n_pages), 256, 0, st>>>(in, in_page_stride, H, W, in_pitch, Lw);
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
  if (method == ABIN_QUANTILE) {
    rc = run_quantile(in, 0, 1, H, W, in_pitch, scratch, W, 0, ABIN_MASK_U8, h, w, param0, 0, H, H, H, 0, st, t_out);
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
  if (mask_out && method == ABIN_QUANTILE && rc == ABIN_OK) {
    cudaError_t e = cudaMemcpyAsync(mask_out, scratch, (size_t)(H * W), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e);
  }
  cudaError_t f = cudaFreeAsync(scratch, st);
  if (rc == ABIN_OK && f != cudaSuccess) return cuda_fail(f);
  return rc;
}

void abin_limits(abin_limits_t* out) {
  if (!out) return;
  out->max_window_w = 190 * G - 1;
  out->max_window_h = 66051;
  out->max_dim = kMaxDim;
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

const char* abin_version(void) { return "abin 0.1 (sm_100a)"; }

const char* abin_last_cuda_error(void) { return g_last_cuda_error; }

}  // extern "C"
