// moments.cuh -- K1 (windowed moments) + K2 (threshold) + K3 (mask store),
// fused in one kernel.  Hot path of arXiv 1905.13038.
//
// Work decomposition
//   A CTA is 4 warps.  It owns one page, a band of B output rows and a
//   column range that the 4 warps split into 4 independent warp strips: warp strip = 32 lanes x G=16 input columns, the
//   first KH lanes being halo (KH = ceil((w+1)/16)); lane k owns input
//   columns [a, a+16) and produces outputs j = a - r + t (t < 16), so the
//   entering column j + r of the horizontal recursion is its own.
//
//  * Vertical pass ("C_j <- C_j + I_{i+u,j} - I_{i-o,j}"):
//    per-column C_j, D_j (uint32, exact) in registers, running down the band.
//  * Horizontal pass ("c <- c + C_{j+r} - C_{j-l}"):
//    running sums over the lane's 16 outputs; the leaving column a - w + t is
//    read from the warp's published row of C, D (shared memory, __syncwarp
//    only); the start value c(a - r - 1) = sum_{b=a-w}^{a-1} C_b comes from a
//    warp shuffle scan of the lanes' column totals.
//  * Rows arrive by TMA (cp.async.bulk.tensor, OOB -> 0, which is the paper's
//    "undefined elements are zero") into a 2-stage ring: entering
//    (i+u), centre (i) and leaving (i-o) rows; the last warp to finish a stage
//    re-arms its slot, so warps never wait for one another.
//  * Epilogue (Alg. 1 l.118-124, Table 1): a certified fp32 evaluation of t
//    with a host-derived error bound delta1 decides every pixel with
//    |I - t~| >= delta1; the rest go to an fp32 evaluation from the exact
//    integer V = n d - c^2 (tighter bound delta2), and what is still
//    ambiguous to the exact IEEE-double sequence (K2).  The mask
//    therefore equals the double-precision decision bit for bit.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <type_traits>

#include "ptx.cuh"
#include "rules.cuh"

namespace abin {

enum { M_SAUVOLA = 0, M_NIBLACK = 1, M_WOLF = 2, M_MAXS = 3 /* Wolf's adaptive R: max s (v5 + fixup) */ };

struct MomParams {
  int64_t W;          // image width
  int64_t H_out;      // output rows of this call (band rows, or H)
  int64_t row0;       // global row of the first output row
  int64_t H_global;   // image height for n / edges
  int64_t buf_row0;   // global row held at tensor-map row 0
  uint8_t* out;       // mask of global row row0, page 0
  int64_t out_pitch;
  int64_t out_page_stride;
  int32_t h, w, l, r, o, u;  // effective (clamped) window
  int32_t fmt;               // 0 u8, 1 bits
  int32_t Tw;                // outputs per warp strip (multiple of 16)
  int32_t n_strips;          // CTA column tiles per page
  int32_t B;                 // output rows per band
  int32_t n_bands;
  int32_t KH;                // halo lanes per warp strip = ceil((w+1)/16)
  int32_t method;
  int32_t force_fp64;
  double k, R;
  const uint8_t* L_page;     // per-page global minimum (Wolf), device
  int32_t L_fixed;           // >= 0: use this L
  // fp32 filter constants (host-derived, K2)
  float fa, fb;              // Sauvola: 1-k, k/R;  Niblack: -, k;  Wolf: k, 1/R
  float delta1, delta2;      // certified bounds of the two fp32 stages (incl. the fp64 error)
  float rb0, rb1, rdv, rsdv; // v4 ambiguity test: data-dependent stage-1 bound rb0 + rb1 min(rsdv, rdv / s~)
  float inv_h;               // fl(1/h): 1/nrow for interior rows
  int32_t stats;             // statistics mode: every pixel takes the fp64 sequence
  uint64_t* counters;        // [near_tie, fp64 fallbacks(, stage-2 pixels)] or null
  int32_t counters_n;        // 2, or 3 with ABIN_COUNT_STAGES
  int32_t sL, sR;            // v4: strips [sL, sR) are interior (no image border inside their windows)
  RuleParams rp;             // Table 1 rules Feng / Rais / Khurshid / Phansalkar (rules.cuh)
  // v4 -> exact fixup queue (fixup.cuh): one uint4 per ambiguous lane, q_count appends
  uint4* q_data;
  uint32_t* q_count;
  uint32_t q_cap;
  // v3 as the overflow follow-up: run only if *ovf_count > ovf_cap
  const uint32_t* ovf_count;
  uint32_t ovf_cap;
  int32_t n_pages_v4;        // v4: pages of the launch
  // v5 packed last strips: the last strip of NG pages in one warp, G lanes
  // each (KH halo + its output lanes), staged by one TMA box of NG pages
  int32_t pk_on, pk_G, pk_NG, pk_n;  // pk_n: packs per band = ceil(pages / NG)
  // M_MAXS (Wolf's image-adaptive R = max s, R21): pass 0 reduces the
  // fp32 v~ per page into vmax_bits; pass 1 queues the pixels whose v~ is within
  // maxs_margin (>= 2 |v~ - v| bound) of it; k_fixup takes their exact fp64 s
  // into smax_bits (double bits; s >= 0, so they order as unsigned integers)
  uint32_t* vmax_bits;
  unsigned long long* smax_bits;
  int32_t maxs_pass;
  float maxs_margin;
  float aux0, aux1;          // v5 rules: Khurshid 1/(h w); Phansalkar p, q log2(e); Rais the bounds' 1/(M S) parts
  float rais_r1;             // Rais: the data-dependent bound's 1/(M S) slope part
  float aux2;                // Feng: gamma (fa = a1, fb = 1/R, aux0 = k1, aux1 = k2)
  // statistics mode (page 0 only)
  uint64_t* c_out;
  uint64_t* d_out;
  uint32_t* n_out;
  double* t_out;
  uint8_t* mask_out;
  // generic loader (used when the image is not 16-byte aligned for TMA)
  int32_t use_tma;
  const uint8_t* in;
  int64_t in_pitch, in_page_stride, buf_rows;
};

// ------------------------------------------------------------------ epilogue
// The canonical sequence: Alg. 1 l.121-122 then the Table-1 row written left
// to right, each operation explicitly rounded (no FMA contraction), so the
// result is the plain IEEE-double evaluation of the paper's formula.
static __device__ __noinline__ double threshold_fp64(int method, uint64_t c, uint64_t d, uint32_t n, double k, double R,
                                              double L) {
  const double nd = (double)n;
  const double m = __ddiv_rn((double)c, nd);
  double v = __dsub_rn(__ddiv_rn((double)d, nd), __dmul_rn(m, m));
  if (v < 0.0) v = 0.0;
  const double s = __dsqrt_rn(v);
  if (method == M_SAUVOLA) return __dmul_rn(m, __dadd_rn(1.0, __dmul_rn(k, __dsub_rn(__ddiv_rn(s, R), 1.0))));
  if (method == M_NIBLACK) return __dadd_rn(m, __dmul_rn(k, s));
  // Wolf: m - ((k (m - L)) (1 - s/R))
  return __dsub_rn(m, __dmul_rn(__dmul_rn(k, __dsub_rn(m, L)), __dsub_rn(1.0, __ddiv_rn(s, R))));
}

// fp32 threshold from m~ and s~ (both fp32 stages use it; K2 bounds it)
__device__ __forceinline__ float threshold_f32(int method, float m, float s, float fa, float fb, float Lf) {
  if (method == M_SAUVOLA) return m * __fmaf_rn(fb, s, fa);            // m (alpha + beta s)
  if (method == M_NIBLACK) return __fmaf_rn(fb, s, m);                  // m + k s
  const float b = __fmaf_rn(-fb, s, 1.0f);                             // 1 - s/R
  return __fmaf_rn(-(fa * (m - Lf)), b, m);                            // m - k (m - L)(1 - s/R)
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 16 bytes starting DL bytes into the 32-byte window (x0, x1).
template <int DL>
__device__ __forceinline__ uint4 funnel16(uint4 x0, uint4 x1) {
  const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
  constexpr int q = DL >> 2, sh = 8 * (DL & 3);
  if (sh == 0) return make_uint4(w[q], w[q + 1], w[q + 2], w[q + 3]);
  return make_uint4(__funnelshift_r(w[q], w[q + 1], sh), __funnelshift_r(w[q + 1], w[q + 2], sh),
                    __funnelshift_r(w[q + 2], w[q + 3], sh), __funnelshift_r(w[q + 3], w[q + 4], sh));
}

// prmt.b32 with the full 4-bit selector nibbles (__byte_perm ignores bit 3,
// the sign-replicate flag).
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t byte_of(const uint4& v, int t) {
  const uint32_t wd = t < 4 ? v.x : (t < 8 ? v.y : (t < 12 ? v.z : v.w));
  return __byte_perm(wd, 0u, 0x4440u | (uint32_t)(t & 3));
}

constexpr int kG = 16;        // columns per lane

// Bank-conflict-free layout of a warp's published 512-column row (C, D and
// the -1/ncol table): column s lives at word
//   ((s/4) mod 4) * 128 + (s/16) * 4 + s mod 4,
// i.e. [4-column chunk g][lane][4], so a warp-wide 16-byte access to chunk g
// of 32 consecutive lanes (publish) or of 32 lanes offset by a common column
// shift (the leaving reads) touches 512 consecutive bytes.
__device__ __forceinline__ int swz(int s) { return (((s >> 2) & 3) << 7) | ((s >> 4) << 2) | (s & 3); }

__device__ __forceinline__ float ninv_sel(const float (&a)[16], int t) {
  float r = 0.0f;
#pragma unroll
  for (int z = 0; z < 16; ++z)
    if (z == t) r = a[z];
  return r;
}

// The 16 leaving values C[st + t], D[st + t] (t < 16) from shared memory;
// `st` is 4-aligned, so the reads are aligned vectors and the phase PH is a
// register renaming.
template <int PH>
__device__ __forceinline__ void load_leaving(const uint32_t* cs, const uint32_t* ds, uint32_t (&Cl)[16],
                                             uint32_t (&Dl)[16]) {
  uint32_t qv[20], dv[20];
#pragma unroll
  for (int t = 0; t < 20; t += 4) {
    if (PH == 0 && t == 16) break;
    const uint4 a4 = *reinterpret_cast<const uint4*>(cs + t);
    const uint4 b4 = *reinterpret_cast<const uint4*>(ds + t);
    qv[t] = a4.x; qv[t + 1] = a4.y; qv[t + 2] = a4.z; qv[t + 3] = a4.w;
    dv[t] = b4.x; dv[t + 1] = b4.y; dv[t + 2] = b4.z; dv[t + 3] = b4.w;
  }
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    Cl[t] = qv[t + PH];
    Dl[t] = dv[t + PH];
  }
}

// Running sums over a lane's 16 outputs fused with stage 1
// of the certified decision (K2).  The leaving column sums are read
// from the warp's published row progressively (cs/ds point 4-aligned at the
// first one minus PH) and the per-column -1/ncol from shared memory (nic).
// With ninv = -1/n (fp32): mn = c ninv = -m~, qn = d ninv = -q~,
// vn = mn^2 + qn = -v~, s~ = sqrt|vn|, en = I - t~ (en > 0: background).
// Writes the mask bytes (byte t of wv[t/4] = en_t >= 0, taken from the sign
// bits by prmt) and returns min |en|.
template <int METHOD, int PH, typename DT>
__device__ __forceinline__ float row_stage1(const uint32_t (&C)[16], const uint32_t (&D)[16], const uint32_t* cs,
                                            const uint32_t* ds, const int (&lofs)[5], uint32_t cc, DT dd,
                                            const float* nic, float inv_nrow, const uint4& xc, float2 fa2,
                                            float2 fb2, float Lf, uint32_t (&wv)[4]) {
  const float2 nr2 = make_float2(inv_nrow, inv_nrow);
  float emin = __int_as_float(0x7f800000);
  uint4 qc = *reinterpret_cast<const uint4*>(cs + lofs[0]), qd = *reinterpret_cast<const uint4*>(ds + lofs[0]);
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    // leaving values of outputs 4g .. 4g+3 = words PH .. PH+3 of (qc, next)
    uint32_t cl[4], dl[4];
    if (PH == 0) {
      cl[0] = qc.x; cl[1] = qc.y; cl[2] = qc.z; cl[3] = qc.w;
      dl[0] = qd.x; dl[1] = qd.y; dl[2] = qd.z; dl[3] = qd.w;
      if (g < 3) {
        qc = *reinterpret_cast<const uint4*>(cs + lofs[g + 1]);
        qd = *reinterpret_cast<const uint4*>(ds + lofs[g + 1]);
      }
    } else {
      const uint4 nc = *reinterpret_cast<const uint4*>(cs + lofs[g + 1]);
      const uint4 nd = *reinterpret_cast<const uint4*>(ds + lofs[g + 1]);
      const uint32_t c8[8] = {qc.x, qc.y, qc.z, qc.w, nc.x, nc.y, nc.z, nc.w};
      const uint32_t d8[8] = {qd.x, qd.y, qd.z, qd.w, nd.x, nd.y, nd.z, nd.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) { cl[k] = c8[PH + k]; dl[k] = d8[PH + k]; }
      qc = nc;
      qd = nd;
    }
    const float4 ni4 = *reinterpret_cast<const float4*>(nic + 128 * g);
    const float nis[4] = {ni4.x, ni4.y, ni4.z, ni4.w};
    const uint32_t wd = g == 0 ? xc.x : (g == 1 ? xc.y : (g == 2 ? xc.z : xc.w));
    float e4[4];
#pragma unroll
    for (int h2 = 0; h2 < 4; h2 += 2) {
      const int t = 4 * g + h2;
      cc += C[t] - cl[h2];
      dd += (DT)D[t] - (DT)dl[h2];
      const uint32_t ca = cc;
      const DT da = dd;
      cc += C[t + 1] - cl[h2 + 1];
      dd += (DT)D[t + 1] - (DT)dl[h2 + 1];
      const float2 ninv = __fmul2_rn(make_float2(nis[h2], nis[h2 + 1]), nr2);
      const float2 mn = __fmul2_rn(make_float2((float)ca, (float)cc), ninv);
      const float2 qn = __fmul2_rn(make_float2((float)da, (float)dd), ninv);
      const float2 vn = __ffma2_rn(mn, mn, qn);
      const float2 s = make_float2(sqrt_approx(fabsf(vn.x)), sqrt_approx(fabsf(vn.y)));
      // exact I: the byte placed in the mantissa of 2^23, minus 2^23
      const float2 Im = make_float2(__uint_as_float(__byte_perm(wd, 0x4B000000u, 0x7440u | (uint32_t)h2)),
                                    __uint_as_float(__byte_perm(wd, 0x4B000000u, 0x7440u | (uint32_t)(h2 + 1))));
      const float2 I = __fadd2_rn(Im, make_float2(-8388608.0f, -8388608.0f));
      float2 e;
      if (METHOD == M_SAUVOLA) {
        const float2 gg = __ffma2_rn(fb2, s, fa2);                // alpha + beta s
        e = __ffma2_rn(mn, gg, I);                                // I - m g
      } else if (METHOD == M_NIBLACK) {
        e = __ffma2_rn(make_float2(-fb2.x, -fb2.y), s, __fadd2_rn(I, mn));   // I - m - k s
      } else {
        const float2 b = __ffma2_rn(make_float2(-fb2.x, -fb2.y), s, make_float2(1.0f, 1.0f));  // 1 - s/R
        const float2 ka = __fmul2_rn(make_float2(-fa2.x, -fa2.y), __fadd2_rn(mn, make_float2(Lf, Lf)));  // k (m - L)
        e = __ffma2_rn(ka, b, __fadd2_rn(I, mn));                 // I - m + k (m - L)(1 - s/R)
      }
      emin = fminf(emin, fminf(fabsf(e.x), fabsf(e.y)));
      e4[h2] = e.x;
      e4[h2 + 1] = e.y;
    }
    // prmt with selector msb set replicates the selected byte's sign bit
    const uint32_t lo = prmt_sign(__float_as_uint(e4[0]), __float_as_uint(e4[1]), 0x00FBu);
    const uint32_t hi = prmt_sign(__float_as_uint(e4[2]), __float_as_uint(e4[3]), 0xFB00u);
    wv[g] = ~__byte_perm(lo, hi, 0x7610u) & 0x01010101u;
  }
  return emin;
}

constexpr int kCW = 4;        // warps per CTA (each owns one warp strip)
constexpr int kNT = 32 * kCW;
constexpr int kR = 2;         // rows per TMA stage (one 256 x 2 box per TMA op)
constexpr int kNS = 2;        // ring depth (stages)
constexpr int kSPAN = 2048;   // staged bytes per row per stream (8 TMA boxes of 256)
constexpr int kNBOX = kSPAN / 256;
constexpr int kStream = kR * kSPAN;
constexpr int kStage = 3 * kStream;
constexpr int kWarpRow = 32 * kG;  // input columns per warp strip (512)

constexpr size_t moments_smem_bytes() {
  return (size_t)kNS * kStage                          // TMA ring
         + (size_t)kCW * 2 * kWarpRow * 4              // per-warp published C, D row
         + (size_t)kCW * kWarpRow * 4                  // per-column -1/ncol
         + kNS * 8 + kNS * 4 + 8;                      // full mbarriers, stage counters
}

// Kernel template parameters:
//   W32   w mod 32: fixes the alignment phase PH = (-w) mod 4 of the
//         leaving-column reads, the partial-prefix position PP = (-(w+1)) mod 16
//         and the byte funnel DL = r mod 16 of the entering/leaving rows
//   D64   window square sums in uint64
template <int W32, bool D64>
__global__ void __launch_bounds__(kNT, 4) k_moments(const __grid_constant__ CUtensorMap tin, const MomParams p) {
  using DT = typename std::conditional<D64, uint64_t, uint32_t>::type;
  constexpr int W16 = W32 & 15;
  constexpr int PH = (4 - (W16 & 3)) & 3;           // (-w) mod 4
  constexpr int PP = (kG - 1 - W16 + kG) % kG;      // (-(w+1)) mod 16
  constexpr int DL = (W32 >> 1) & 15;               // r mod 16 = S0 mod 16
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  uint32_t* pub = reinterpret_cast<uint32_t*>(smem + kNS * kStage);   // [warp][C|D][512]
  float* nic_all = reinterpret_cast<float*>(pub + kCW * 2 * kWarpRow);  // [warp][512] -1/ncol
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(nic_all + kCW * kWarpRow);
  uint32_t* done_cnt = reinterpret_cast<uint32_t*>(full_bar + kNS);  // warps finished with a slot

  if (p.ovf_count != nullptr && *p.ovf_count <= p.ovf_cap) return;  // follow-up launch, no queue overflow
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // ---- tile coordinates
  int64_t tile = blockIdx.x;
  const int strip = (int)(tile % p.n_strips);
  tile /= p.n_strips;
  const int band = (int)(tile % p.n_bands);
  const int page = (int)(tile / p.n_bands);
  const int64_t Tc = (int64_t)kCW * p.Tw;                   // outputs per CTA
  const int64_t J0 = (int64_t)strip * Tc;                   // first output column of the CTA
  const int64_t S0 = J0 + p.r - (int64_t)kG * p.KH;         // input column of warp 0 lane 0
  // TMA box x-origins must be 16-byte aligned: entering/leaving rows are
  // staged from XE = S0 - dl and read back through a byte funnel; the centre
  // row is staged from XC = S0 - r = J0 - 16 KH, already aligned.
  const int64_t XE = S0 - DL;
  const int64_t XC = S0 - p.r;
  const int64_t y0 = p.row0 + (int64_t)band * p.B;          // first output row (global)
  const int64_t nrows = min((int64_t)p.B, p.row0 + p.H_out - y0);
  const int WS = (p.h + kR - 1) / kR;                       // warm-up stages
  const int MS = (int)((nrows + kR - 1) / kR);              // main stages
  const int total = WS + MS;

  // TMA boxes whose column range misses [0, W) entirely are never issued (the
  // hardware rejects them); their bytes are zeroed once -- a CTA's columns
  // never change.
  auto box_ok = [&](int64_t x) { return x + 256 > 0 && x < p.W; };
  int nbe = 0, nbc = 0;
#pragma unroll
  for (int b = 0; b < kNBOX; ++b) {
    nbe += box_ok(XE + 256 * b);
    nbc += box_ok(XC + 256 * b);
  }
  // Issue stage s into slot s % kNS (one elected thread).
  // L2 policy: input rows are read three times (entering, centre o rows
  // later... leaving h rows later), so they are kept (evict_last); the
  // leaving read is their last use (evict_first).
  auto issue = [&](int s) {
    const int slot = s % kNS;
    uint8_t* st = ring + slot * kStage;
    const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
    if (s < WS) {
      const int32_t yr = (int32_t)(y0 - p.o + (int64_t)s * kR - p.buf_row0);
      mbar_arrive_expect_tx(&full_bar[slot], nbe * kR * 256);
      for (int b = 0; b < kNBOX; ++b)
        if (box_ok(XE + 256 * b))
          tma_load_3d_hint(st + b * kR * 256, &tin, (int32_t)(XE + 256 * b), yr, page, &full_bar[slot], keep);
    } else {
      const int64_t q0 = (int64_t)(s - WS) * kR;
      const int32_t ye = (int32_t)(y0 + q0 + p.u - p.buf_row0);
      const int32_t yc = (int32_t)(y0 + q0 - p.buf_row0);
      const int32_t yl = (int32_t)(y0 + q0 - p.o - p.buf_row0);
      mbar_arrive_expect_tx(&full_bar[slot], (2 * nbe + nbc) * kR * 256);
      for (int b = 0; b < kNBOX; ++b) {
        if (box_ok(XE + 256 * b)) {
          tma_load_3d_hint(st + b * kR * 256, &tin, (int32_t)(XE + 256 * b), ye, page, &full_bar[slot], keep);
          tma_load_3d_hint(st + 2 * kStream + b * kR * 256, &tin, (int32_t)(XE + 256 * b), yl, page,
                           &full_bar[slot], drop);
        }
        if (box_ok(XC + 256 * b))
          tma_load_3d_hint(st + kStream + b * kR * 256, &tin, (int32_t)(XC + 256 * b), yc, page, &full_bar[slot],
                           keep);
      }
    }
  };
  // Generic loader (image not 16-byte aligned for TMA): the whole CTA copies
  // the stage's rows (zero outside the held rows / image columns).
  auto fill = [&](int s) {
    uint8_t* st = ring + (s % kNS) * kStage;
    const uint8_t* img = p.in + (int64_t)page * p.in_page_stride;
    const int nstream = s < WS ? 1 : 3;
    for (int e = tid; e < nstream * kStream; e += kNT) {
      const int sidx = e / kStream, rem = e - sidx * kStream;
      const int b = rem / (kR * 256), rr = (rem / 256) % kR, cc = rem % 256;
      const int64_t x = (sidx == 1 ? XC : XE) + 256 * b + cc;
      int64_t y;
      if (s < WS) {
        y = y0 - p.o + (int64_t)s * kR + rr;
      } else {
        const int64_t qrow = y0 + (int64_t)(s - WS) * kR + rr;
        y = sidx == 0 ? qrow + p.u : (sidx == 1 ? qrow : qrow - p.o);
      }
      y -= p.buf_row0;
      st[e] = (y >= 0 && y < p.buf_rows && x >= 0 && x < p.W) ? img[y * p.in_pitch + x] : (uint8_t)0;
    }
  };

  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&full_bar[s], 1);
      done_cnt[s] = 0;
    }
    fence_mbar_init();
  }
  if (p.use_tma) {
    for (int slot = 0; slot < kNS; ++slot)
      for (int sidx = 0; sidx < 3; ++sidx)
        for (int b = 0; b < kNBOX; ++b) {
          const int64_t x = (sidx == 1 ? XC : XE) + 256 * b;
          if (box_ok(x)) continue;
          uint4* z = reinterpret_cast<uint4*>(ring + slot * kStage + sidx * kStream + b * kR * 256);
          for (int e = tid; e < kR * 16; e += kNT) z[e] = make_uint4(0, 0, 0, 0);
        }
  }
  __syncthreads();
  if (p.use_tma && tid == 0) {
    prefetch_tmap(&tin);
    for (int s = 0; s < kNS && s < total; ++s) issue(s);
  }
  // Stage hand-off.  Each warp, when done with stage s, counts itself out of
  // the slot; the last of the 4 re-arms the slot with stage s + kNS, so no
  // warp ever waits for another to refill (TMA path).  The generic path
  // loads synchronously with CTA barriers.
  auto stage_begin = [&](int s) {
    if (p.use_tma) {
      mbar_wait(&full_bar[s % kNS], (s / kNS) & 1);
    } else {
      __syncthreads();
      fill(s);
      __syncthreads();
    }
  };
  auto stage_end = [&](int s) {
    if (!p.use_tma) return;
    __syncwarp();
    if (lane == 0) {
      const int slot = s % kNS;
      if (atomicAdd_block(&done_cnt[slot], 1u) == kCW - 1) {
        done_cnt[slot] = 0;
        fence_proxy_async_smem();  // generic reads of the slot precede the async-proxy refill
        if (s + kNS < total) issue(s + kNS);
      }
    }
  };

  // =================================================================== consumers
  const int64_t Sw = S0 + (int64_t)warp * p.Tw;       // warp strip input origin
  const int64_t a = Sw + (int64_t)kG * lane;          // first owned input column
  const int64_t j0 = a - p.r;                         // first output column (multiple of 16)
  const int64_t Jend = min(J0 + Tc, p.W);
  const bool valid_lane = lane >= p.KH && j0 < Jend;
  // outputs of this lane that exist (halo lanes and columns past W have none:
  // their garbage windows must never reach the slow path)
  const uint32_t vmask = valid_lane ? (Jend - j0 >= kG ? 0xFFFFu : ((1u << (uint32_t)(Jend - j0)) - 1u)) : 0u;
  const int eoff = warp * p.Tw + kG * lane;           // staged offset of column a, minus DL (16-aligned)
  auto soff = [](int e) { return (e >> 8) * (kR * 256) + (e & 255); };
  const int eo0 = soff(eoff), eo1 = soff(eoff + 16);  // entering / leaving 16-byte chunks
  const int co = soff(eoff);                          // centre row chunk (origin XC = S0 - r)
  const int srcq = (lane - p.KH) & 31;                // lane holding column a - w - 1
  uint32_t* cb = pub + warp * (2 * kWarpRow);         // this warp's published C row
  uint32_t* db = cb + kWarpRow;                       //                      D row
  const int st0 = valid_lane ? (kG * lane - p.w - PH) : 0;  // 4-aligned start of the leaving reads
  int lofs[5];                                        // swizzled word offsets of the leaving chunks
#pragma unroll
  for (int g = 0; g < 5; ++g) lofs[g] = swz(min(st0 + 4 * g, kWarpRow - 4));
  const float Lf = (p.method == M_WOLF || p.method == M_FENG)
                       ? (float)(p.L_fixed >= 0 ? p.L_fixed : (int)p.L_page[page]) : 0.0f;
  const bool slow_all = p.stats || p.force_fp64;
  const int method = p.method;
  const float delta1 = p.delta1;

  // negated reciprocals of the clamped column counts (n = ncol * nrow,
  // PAPER.md:118), kept in shared memory (read back as float4 per 4 outputs)
  float* nicw = nic_all + warp * kWarpRow;
  const float* nic = nicw + 4 * lane;               // chunk g of this lane at nic + 128 g
#pragma unroll
  for (int t = 0; t < kG; ++t) {
    const int64_t j = j0 + t;
    const int64_t nc = max((int64_t)1, min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1));
    nicw[swz(kG * lane + t)] = -__frcp_rn((float)nc);
  }
  __syncwarp();
  const float2 fa2 = make_float2(p.fa, p.fa), fb2 = make_float2(p.fb, p.fb);

  uint32_t C[kG], D[kG];
#pragma unroll
  for (int t = 0; t < kG; ++t) C[t] = D[t] = 0;
  uint64_t near_ties = 0, fallbacks = 0;

  // ---- warm-up: rows y0-o .. y0-o+h-1 (the first output row adds y0+u and
  // subtracts y0-o, giving rows (y0-o, y0+u])
  for (int s = 0; s < WS; ++s) {
    const int slot = s % kNS;
    stage_begin(s);
    const uint8_t* st = ring + slot * kStage;
    const int nr = min(kR, p.h - s * kR);
#pragma unroll 1
    for (int rr = 0; rr < nr; ++rr) {
      const uint4 x = funnel16<DL>(*reinterpret_cast<const uint4*>(st + eo0 + rr * 256),
                                   *reinterpret_cast<const uint4*>(st + eo1 + rr * 256));
#pragma unroll
      for (int t = 0; t < kG; ++t) {
        const uint32_t v = byte_of(x, t);
        C[t] += v;
        D[t] += v * v;
      }
    }
    stage_end(s);
  }

  // ---- main rows
  int32_t q = 0;
  for (int s = WS; s < total; ++s) {
    const int slot = s % kNS;
    stage_begin(s);
    const uint8_t* st = ring + slot * kStage;
    const int nr = min(kR, (int)(nrows - (int64_t)(s - WS) * kR));
    // raw 16-byte chunks of row rr (entering x2, leaving x2, centre), loaded
    // one row ahead so their shared-memory latency overlaps the previous row
    uint4 ri0 = *reinterpret_cast<const uint4*>(st + eo0), ri1 = *reinterpret_cast<const uint4*>(st + eo1);
    uint4 ro0 = *reinterpret_cast<const uint4*>(st + 2 * kStream + eo0);
    uint4 ro1 = *reinterpret_cast<const uint4*>(st + 2 * kStream + eo1);
    uint4 rc = *reinterpret_cast<const uint4*>(st + kStream + co);
#pragma unroll 1
    for (int rr = 0; rr < nr; ++rr, ++q) {
      const uint4 xi = funnel16<DL>(ri0, ri1);
      const uint4 xo = funnel16<DL>(ro0, ro1);
      const uint4 xc = rc;
      if (rr + 1 < nr) {
        const int nx = (rr + 1) * 256;
        ri0 = *reinterpret_cast<const uint4*>(st + eo0 + nx);
        ri1 = *reinterpret_cast<const uint4*>(st + eo1 + nx);
        ro0 = *reinterpret_cast<const uint4*>(st + 2 * kStream + eo0 + nx);
        ro1 = *reinterpret_cast<const uint4*>(st + 2 * kStream + eo1 + nx);
        rc = *reinterpret_cast<const uint4*>(st + kStream + co + nx);
      }
      // vertical update
#pragma unroll
      for (int t = 0; t < kG; ++t) {
        const uint32_t vi = byte_of(xi, t), vo = byte_of(xo, t);
        C[t] = C[t] + vi - vo;
        D[t] = D[t] + vi * vi - vo * vo;
      }
      // publish this row's column sums for the neighbours' leaving reads
      // (single buffer: the __syncwarp orders it after last row's reads)
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kG; t += 4) {
        *reinterpret_cast<uint4*>(cb + 32 * t + 4 * lane) = make_uint4(C[t], C[t + 1], C[t + 2], C[t + 3]);
        *reinterpret_cast<uint4*>(db + 32 * t + 4 * lane) = make_uint4(D[t], D[t + 1], D[t + 2], D[t + 3]);
      }
      // lane totals (pairwise) and the partial prefix up to position PP
      uint32_t partc = 0;
      DT partd = 0;
#pragma unroll
      for (int t = 0; t <= PP; ++t) { partc += C[t]; partd += (DT)D[t]; }
      uint32_t restc = 0;
      DT restd = 0;
#pragma unroll
      for (int t = PP + 1; t < kG; ++t) { restc += C[t]; restd += (DT)D[t]; }
      const uint32_t pc = partc + restc;
      const DT pd = partd + restd;
      // anchor A = sum_{b=a-w}^{a-1} C_b = P(a-1) - P(a-w-1)
      //          = sum_{k=1..KH} T(lane-k) - partial(lane-KH)
      uint32_t c0;
      DT d0;
      if (p.KH <= 8) {
        c0 = 0u - __shfl_sync(0xffffffffu, partc, srcq);
        d0 = (DT)0 - __shfl_sync(0xffffffffu, partd, srcq);
        for (int kk = 1; kk <= p.KH; ++kk) {
          c0 += __shfl_sync(0xffffffffu, pc, (lane - kk) & 31);
          d0 += __shfl_sync(0xffffffffu, pd, (lane - kk) & 31);
        }
      } else {
        uint32_t ic = pc;
        DT id = pd;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t oc = __shfl_up_sync(0xffffffffu, ic, off);
          const DT od = __shfl_up_sync(0xffffffffu, id, off);
          if (lane >= off) { ic += oc; id += od; }
        }
        const uint32_t ec = ic - pc;
        const DT ed = id - pd;
        c0 = ec - __shfl_sync(0xffffffffu, ec + partc, srcq);
        d0 = ed - __shfl_sync(0xffffffffu, ed + partd, srcq);
      }
      __syncwarp();

      const int64_t i = y0 + q;  // global output row
      const uint32_t nrow = (uint32_t)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
      const float inv_nrow = (nrow == (uint32_t)p.h) ? p.inv_h : __frcp_rn((float)nrow);
      // ---- running sums fused with stage 1 of the decision
      uint32_t wv[4];
      float emin;
      switch (method) {  // warp-uniform
        case M_SAUVOLA:
          emin = row_stage1<M_SAUVOLA, PH>(C, D, cb, db, lofs, c0, d0, nic, inv_nrow, xc, fa2, fb2, Lf, wv);
          break;
        case M_NIBLACK:
          emin = row_stage1<M_NIBLACK, PH>(C, D, cb, db, lofs, c0, d0, nic, inv_nrow, xc, fa2, fb2, Lf, wv);
          break;
        default:
          emin = row_stage1<M_WOLF, PH>(C, D, cb, db, lofs, c0, d0, nic, inv_nrow, xc, fa2, fb2, Lf, wv);
          break;
      }
      uint32_t ambits = slow_all ? vmask : 0u;
      if (!slow_all && emin < delta1) ambits = vmask;  // (re-tested per pixel below)
      if (ambits) {
        // ---- stages 2 and 3 for the pixels stage 1 could not decide: recompute
        // (c, d) of each from the anchor and the published rows (rare path).
        // Decided bits are collected in fix (which outputs) / fixv (values).
        uint32_t fix = 0, fixv = 0;
        uint32_t cc = c0;
        DT dd = d0;
#pragma unroll 1
        for (int t = 0; t < kG; ++t) {
          uint32_t Ct = 0, Dt = 0;
#pragma unroll
          for (int z = 0; z < kG; ++z)
            if (z == t) { Ct = C[z]; Dt = D[z]; }
          cc += Ct - cb[swz(st0 + PH + t)];
          dd += (DT)Dt - (DT)db[swz(st0 + PH + t)];
          if (!((ambits >> t) & 1u)) continue;
          const int64_t j = j0 + t;
          const uint32_t n =
              (uint32_t)max((int64_t)1, min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1)) * nrow;
          const uint32_t I = byte_of(xc, t);
          const uint64_t c64 = cc, d64 = (uint64_t)dd;
          bool decided = false;
          uint32_t mk = 0;
          if (!slow_all) {
            // stage 1 again for this pixel (is it really ambiguous?)
            const float ninv = nicw[swz(kG * lane + t)] * inv_nrow;
            const float mn = (float)cc * ninv, qn = (float)dd * ninv;
            const float s1 = sqrt_approx(fabsf(__fmaf_rn(mn, mn, qn)));
            const float e1 = (float)I - threshold_f32(p.method, -mn, s1, p.fa, p.fb, Lf);
            if (!(fabsf(e1) < p.delta1)) continue;  // stage 1 decided it already
            // stage 2: exact V = n d - c^2 >= 0, then fp32 with the tight bound delta2
            const uint64_t V = (uint64_t)n * d64 - c64 * c64;
            const float Vf = __fmaf_rn((float)(uint32_t)(V >> 32), 4294967296.0f, (float)(uint32_t)V);
            const float invn = __frcp_rn((float)n);
            const float m = (float)(uint32_t)c64 * invn;
            const float t2 = threshold_f32(p.method, m, sqrt_approx(Vf) * invn, p.fa, p.fb, Lf);
            const float e2 = t2 - (float)I;
            if (fabsf(e2) >= p.delta2) {
              decided = true;
              mk = e2 < 0.0f ? 1u : 0u;
            }
          }
          double tt = 0.0;
          if (!decided) {
            tt = is_rule(p.method) ? threshold_rule_fp64(p.method, c64, d64, n, p.rp, (double)Lf, page)
                                   : threshold_fp64(p.method, c64, d64, n, p.k, p.R, (double)Lf);
            mk = ((double)I <= tt) ? 0u : 1u;
            fallbacks++;
            if (fabs((double)I - tt) < 1e-9) near_ties++;
          }
          fix |= 1u << t;
          fixv |= mk << t;
          if (p.stats && page == 0) {
            const int64_t idx = (i - p.row0) * p.W + j;
            if (p.c_out) p.c_out[idx] = c64;
            if (p.d_out) p.d_out[idx] = d64;
            if (p.n_out) p.n_out[idx] = n;
            if (p.t_out) p.t_out[idx] = tt;
            if (p.mask_out) p.mask_out[idx] = (uint8_t)mk;
          }
        }
        if (fix) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            // spread 4 bits into the 4 bytes of a word: bit b -> byte b
            const uint32_t fm = (((fix >> (4 * g)) & 0xFu) * 0x00204081u) & 0x01010101u;
            const uint32_t fv = (((fixv >> (4 * g)) & 0xFu) * 0x00204081u) & 0x01010101u;
            wv[g] = (wv[g] & ~(fm * 0xFFu)) | fv;
          }
        }
      }
      // ---- store the mask: outputs j0 .. j0+15 (j0 is a multiple of 16)
      if (valid_lane) {
        const int nvalid = (int)min((int64_t)kG, Jend - j0);
        uint8_t* orow = p.out + (int64_t)page * p.out_page_stride + (i - p.row0) * p.out_pitch;
        if (p.fmt == 0) {
          uint8_t* o = orow + j0;
          if (nvalid == kG && ((reinterpret_cast<uintptr_t>(o) & 15u) == 0)) {
            __stcs(reinterpret_cast<uint4*>(o), make_uint4(wv[0], wv[1], wv[2], wv[3]));  // streaming
          } else {
#pragma unroll
            for (int t = 0; t < kG; ++t)
              if (t < nvalid) o[t] = (uint8_t)(wv[t >> 2] >> (8 * (t & 3)));
          }
        } else {
          // bytes (0/1) -> bits: nibble of word g = (wv[g] * 0x01020408) >> 24
          uint32_t mbits = 0;
#pragma unroll
          for (int g = 0; g < 4; ++g) mbits |= (((wv[g] * 0x01020408u) >> 24) & 0xFu) << (4 * g);
          // MSB-first: output j0 + t -> bit 7 - (t & 7) of byte (j0 + t) / 8; pad bits 0
          const uint32_t keep = (1u << nvalid) - 1u;
          const uint32_t mb = __brev(mbits & keep) >> 16;  // bit 15 - t = mask of output t
          uint8_t* o = orow + (j0 >> 3);
          o[0] = (uint8_t)(mb >> 8);
          if (nvalid > 8) o[1] = (uint8_t)(mb & 0xFFu);
        }
      }
    }
    stage_end(s);
  }

  if (p.counters) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      near_ties += __shfl_down_sync(0xffffffffu, near_ties, off);
      fallbacks += __shfl_down_sync(0xffffffffu, fallbacks, off);
    }
    if (lane == 0) {
      if (near_ties) atomicAdd(reinterpret_cast<unsigned long long*>(&p.counters[0]), (unsigned long long)near_ties);
      if (fallbacks) atomicAdd(reinterpret_cast<unsigned long long*>(&p.counters[1]), (unsigned long long)fallbacks);
    }
  }
}

}  // namespace abin
