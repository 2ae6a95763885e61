// moments5.cuh -- the production moments kernel (v5): K1 (windowed moments)
// + K2 (certified threshold) + K3 (mask store) fused.  Hot path of arXiv
// 1905.13038: Alg. 1 and Table 1
// (PAPER.md:151-153).
//
// Same tiling as v4 (moments4.cuh): one CTA = one warp = one warp strip of
// 32 lanes x 16 input columns; lane k owns input columns [a, a+16),
// a = Sw + 16 k, and produces the outputs j = a - r + t (t < 16), so the
// entering column j + r of the row recursion is its own (shifted ownership);
// the first KH = ceil(w/16) lanes are halo.  Rows arrive by TMA into a
// per-warp ring (entering row i+u and leaving row i-o).
// What changed against v4 ("v5"):
//
//  * Vertical pass in packed fp32 on exact integers.  A
//    staged byte b becomes the float 32768 + b with one PRMT (the byte is
//    placed in the mantissa, no conversion instruction); per column pair
//      x - y  = fin - fout,  x + y = (fin + fout) - 65536   (exact),
//      C += x - y,  D += (x - y)(x + y)                       (FADD2 / FFMA2)
//    C and D are kept biased by 2^23 (C_b = 2^23 + C): they are integers
//    below 2^24, so every operation is exact, and the bit pattern of C_b is
//    the integer 0x4B000000 + C.  (Needs D = sum x^2 <= 255^2 h < 2^23: h <= 129.)
//  * Horizontal pass in exact integer arithmetic on those
//    bit patterns: the lane runs the row recursion relative to its own start,
//      rel_c(t) = rel_c(t-1) + bits C_b[a+t] - bits C_b[a+t-w]   (IADD3),
//    the leaving column sums coming from the warp's published row (shared
//    memory, zero-padded on the left).  The lane's start value
//    c(a - r - 1) = sum of C over [a - w, a) is the exclusive warp scan of the
//    lanes' recursion totals rel(15) (the sum telescopes); it is folded into
//    the epilogue's first multiply-add, so no per-pixel addition is needed.
//  * Epilogue (Alg. 1 l.118-124, Table 1): the certified fp32 decision of v4
//    on the exact (c, d): m = c/n, q = d/n, v = q - m^2, s = sqrt v, the
//    Table-1 expression, residual e = I - t~ (packed FFMA2 on pixel pairs),
//    mask bits from the residuals' signs; a lane with a pixel whose |e| is
//    within the host-derived bound (abin_api.cu filter_consts_v5) stores
//    provisional bits and is queued for k_fixup (fixup.cuh), which decides
//    it exactly (fp32 from the exact V = n d - c^2, then the canonical IEEE
//    double sequence).  The mask therefore equals the double-precision
//    decision bit for bit.
#pragma once
#include <cstdint>
#include <cuda.h>

#include "moments.cuh"
#include "moments4.cuh"
#include "ptx.cuh"
#include "rules.cuh"

namespace abin {
namespace v5 {

constexpr int kG = 16;                    // columns per lane
constexpr int kStrip = 32 * kG;           // input columns per warp strip
constexpr int kChunks = 33;               // TMA box: 33 16-byte chunks = 528 bytes per row
constexpr int kSpan = 16 * kChunks;       // staged bytes per row
#ifndef ABIN_V5_MINB
#define ABIN_V5_MINB 16  // resident warp-CTAs per SM the register allocation targets
#endif
#ifndef ABIN_V5_KR
#define ABIN_V5_KR 3
#endif
#ifndef ABIN_V5_L2
#define ABIN_V5_L2 0  // L2 policy experiments: 1 mask stores evict_first, 2 entering rows evict_normal, 4 leaving rows evict_normal
#endif
constexpr int kR = ABIN_V5_KR;            // rows per ring stage and stream
constexpr int kNS = 2;                    // ring stages
constexpr int kRowsBytes = (kR * kSpan + 127) / 128 * 128;
constexpr int kStageBytes = 2 * kRowsBytes;  // entering + leaving
constexpr int kMaxH = 129;                // 255^2 h < 2^23 (biased column square sums)
constexpr int kMaxW = 127;                // ceil(w/16) <= 8 (start value from <= 9 shuffles), 255 h w < 2^23

struct SmemLayout {
  static constexpr int ring = 0;
  static constexpr int pub = kNS * kStageBytes;           // [8 pairs][32 lanes] x 16 B (C_b, C_b, D_b, D_b)
  static constexpr int nic = pub + 8 * 32 * 16;          // edge strips: -1/ncol, [16 slots][16 columns] floats
  static constexpr int bar = nic + 16 * 16 * 4;
  static constexpr int total = bar + kNS * 8;
};
constexpr size_t smem_bytes() { return (size_t)SmemLayout::total; }

constexpr uint32_t kBias = 0x4B000000u;   // bits of 2^23: C_b = 2^23 + C
constexpr uint32_t kMagic = 0x47000000u;  // bits of 32768: PRMT puts a byte in bits 8..15 -> 32768 + b

// the float 32768 + (byte b of x): bytes [0x00, x.b, 0x00, 0x47]
template <int B>
__device__ __forceinline__ float byte_f(uint32_t x) {
  return __uint_as_float(__byte_perm(x, kMagic, 0x7504u | ((uint32_t)B << 4)));
}

// word holding byte t of the lane's 16 columns when they start DL bytes into
// the staged 32-byte window w[0..7]
template <int DL, int T>
__device__ __forceinline__ float own_f(const uint32_t (&w)[8]) {
  return byte_f<(DL + T) & 3>(w[(DL + T) >> 2]);
}

__device__ __forceinline__ uint32_t scan_add(uint32_t v, int off) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
               "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
               "@p add.u32 %0, %0, t;\n\t}"
               : "+r"(v) : "r"(off));
  return v;
}

// packed f32x2 values held in one 64-bit register pair (PTX .f32x2 on .b64):
// keeps the pairs in place across the loop (no re-pairing moves)
typedef uint64_t f2;
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo(f2 v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi(f2 v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2 splat(float a) { return pk(a, a); }

__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Residual pair e = I - t~ for two pixels (the scalar twin used by the
// filter probe, abin_probe_filter, is the same sequence of correctly rounded
// fp32 operations: both go through this function).
//   mn = -m~, qn = -q~ (pairs), I exact, fa/fb the method constants, Lf (Wolf)
template <int METHOD>
__device__ __forceinline__ f2 residual2(f2 mn, f2 qn, f2 I, f2 fa2, f2 fb2, f2 Lf2, f2& s, f2 y2 = f2(0)) {
  if (METHOD == M_KHURSHID) {
    // t = m + k sqrt(s^2 + m^2 (N-1)/N) = m + k sqrt(q - m^2 / N)   (Lf2 = 1/N)
    const f2 wk = fma2(mn, mul2(mn, Lf2), qn);  // m^2 / N - q
    s = pk(sqrt_approx(fabsf(lo(wk))), sqrt_approx(fabsf(hi(wk))));
    return fma2(fb2, s, add2(I, mn));           // (I - m) - k sqrt(.)   (fb2 = -k)
  }
  const f2 wv = fma2(mn, mn, qn);  // m^2 - q = -v~
  s = pk(sqrt_approx(fabsf(lo(wv))), sqrt_approx(fabsf(hi(wv))));
  if (METHOD == M_FENG) {
    // t = a1 m + k1 x^(1+g) (m - L) + k2 x^g L, x = s/R (g >= 1): fa2 = a1, fb2 = (1/R, g),
    // y2 = (k1, k2), Lf2 = L; x^g = ex2(g lg2 x) (0 at x = 0), x^(1+g) = x^g x; each operation
    // rounded separately, as filter_consts_v5 bounds them
    const float a1 = lo(fa2), iR = lo(fb2), g = hi(fb2), k1 = lo(y2), k2 = hi(y2), L = lo(Lf2);
    float e[2];
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      const float m = -(z ? hi(mn) : lo(mn));
      const float x = __fmul_rn(z ? hi(s) : lo(s), iR);
      float P0 = 0.0f;
      if (x > 0.0f) {
        float lg, ex;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"(__fmul_rn(g, lg)));
        P0 = ex;
      }
      const float P1 = __fmul_rn(P0, x);
      const float T1 = __fmul_rn(a1, m);
      const float T2 = __fmul_rn(__fmul_rn(k1, P1), __fsub_rn(m, L));
      const float T3 = __fmul_rn(__fmul_rn(k2, P0), L);
      e[z] = __fsub_rn(z ? hi(I) : lo(I), __fadd_rn(__fadd_rn(T1, T2), T3));
    }
    return pk(e[0], e[1]);
  }
  if (METHOD == M_RAIS) {
    // t = m + 0.3 f s, f = (m s - M S) / max{m s, M S}  (Lf2 = fl32(M S), the page's; 0/0 -> 0, R16);
    // each operation rounded separately, as filter_consts_v5 bounds them
    const f2 na = mul2(mn, s);  // -a~, a~ = fl(m~ s~)
    const float b = lo(Lf2);
    float e[2];
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      const float a = -(z ? hi(na) : lo(na));
      const float den = fmaxf(fmaxf(a, b), 1e-30f);
      float rc;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(den));
      const float f = __fmul_rn(__fsub_rn(a, b), rc);
      const float r = __fmul_rn(__fmul_rn(0.3f, f), z ? hi(s) : lo(s));
      e[z] = __fsub_rn(__fadd_rn(z ? hi(I) : lo(I), z ? hi(mn) : lo(mn)), r);  // (I - m~) - r~
    }
    return pk(e[0], e[1]);
  }
  if (METHOD == M_SAUVOLA) {
    const f2 g = fma2(s, fb2, fa2);  // (1 - k) + (k/R) s
    return fma2(mn, g, I);           // I - m g
  } else if (METHOD == M_NIBLACK) {
    return fma2(fb2, s, add2(I, mn));  // (I - m) - k s   (fb2 = -k)
  } else if (METHOD == M_PHANSALKAR) {
    // t = m (1 + p e^(-q m) + k (s/R - 1)) = m ((1 - k) + (k/R) s + p e^(-q m)); q >= 0
    const f2 a = mul2(y2, mn);  // -q m log2(e)   (y2 = q log2(e))
    f2 E;
    {
      float e0, e1;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(lo(a)));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(hi(a)));
      E = pk(e0, e1);
    }
    const f2 g = fma2(E, Lf2, fma2(s, fb2, fa2));  // (1 - k) + (k/R) s + p E   (Lf2 = p)
    return fma2(mn, g, I);                         // I - m g
  } else {
    const f2 b = fma2(fb2, s, splat(1.0f));   // 1 - s/R      (fb2 = -1/R)
    const f2 ka = mul2(fa2, add2(mn, Lf2));   // k (m - L)    (fa2 = -k)
    return fma2(ka, b, add2(I, mn));          // (I - m) + k (m - L)(1 - s/R)
  }
}

// the method constants as the packed operands residual2 takes
template <int METHOD>
__device__ __forceinline__ void method_consts(float fa, float fb, f2& fa2, f2& fb2) {
  if (METHOD == M_SAUVOLA || METHOD == M_PHANSALKAR) { fa2 = splat(fa); fb2 = splat(fb); }
  else if (METHOD == M_NIBLACK || METHOD == M_KHURSHID) { fa2 = splat(0.0f); fb2 = splat(-fb); }
  else { fa2 = splat(-fa); fb2 = splat(-fb); }
}

// The certified residual pair from the exact window sums (the epilogue of
// the kernel and of the filter probe, abin_probe_filter):
//   cb = bits of the float 2^23 + c (c < 2^23), d the window square sum,
//   nu = -1/n as fl(fl(1/ncol) fl(1/nrow)), nb = -2^23 nu (exact), I exact.
// -m~ = fl((2^23 + c) nu + nb): the product is exact inside the fma, so this
// is the correctly rounded c (-1/n); -q~ = fl(fl(d) nu).
template <int METHOD>
__device__ __forceinline__ f2 residual_pair(uint32_t cb0, uint32_t cb1, uint32_t d0, uint32_t d1, f2 nu, f2 nb, f2 I,
                                            f2 fa2, f2 fb2, f2 Lf2, f2& s, f2 y2 = f2(0)) {
  const f2 mn = fma2(pk(__uint_as_float(cb0), __uint_as_float(cb1)), nu, nb);
  const f2 qn = mul2(pk((float)d0, (float)d1), nu);
  return residual2<METHOD>(mn, qn, I, fa2, fb2, Lf2, s, y2);
}

// The rules' extra operands: Khurshid's 1/N (N = h w, or the pixel's n when
// N_mode != 0: then -nu), Phansalkar's p and q log2(e); Wolf's L
template <int METHOD>
__device__ __forceinline__ f2 aux_operand(const MomParams& p, f2 Lf2, f2 nu) {
  if (METHOD == M_KHURSHID) return p.rp.p[1] != 0.0 ? mul2(nu, splat(-1.0f)) : splat(p.aux0);
  if (METHOD == M_PHANSALKAR) return splat(p.aux0);
  return Lf2;
}

// The filter probe: one tuple (c, d, ncol, nrow, I) per thread, evaluated by
// residual_pair exactly as the kernel does (a test hook for the certified
// bound; the host checks |e~ - e*| <= the bound over many tuples).
template <int METHOD>
__global__ void k_probe(const uint32_t* c, const uint32_t* d, const uint32_t* ncol, const uint32_t* nrow,
                        const uint8_t* I, int64_t count, float fa, float fb, float Lf, float aux0, float aux1,
                        float aux2, int nmode, float* e_out, float* s_out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const float nu1 = -(__frcp_rn((float)ncol[q]) * __frcp_rn((float)nrow[q]));
  const f2 nu = splat(nu1), nb = mul2(nu, splat(-8388608.0f));
  f2 fa2, fb2;
  method_consts<METHOD>(fa, fb, fa2, fb2);
  f2 x2 = splat(Lf);
  if (METHOD == M_KHURSHID) x2 = nmode ? mul2(nu, splat(-1.0f)) : splat(aux0);
  if (METHOD == M_PHANSALKAR) x2 = splat(aux0);
  f2 y2 = splat(aux1);
  if (METHOD == M_FENG) {
    fa2 = splat(fa);
    fb2 = pk(fb, aux2);
    y2 = pk(aux0, aux1);
  }
  const float If = (float)I[q];
  f2 sv;
  const f2 e = residual_pair<METHOD>(kBias + c[q], kBias + c[q], d[q], d[q], nu, nb, pk(If, If), fa2, fb2, x2, sv,
                                     y2);
  e_out[q] = lo(e);
  if (s_out) s_out[q] = lo(sv);
}

// Kernel template parameters:
//   W32   w mod 32: fixes the byte offset DL = r mod 16 of the lane's columns
//         in the staged rows and the phase RHO = (-w) mod 16 of its leaving
//         columns in the published row
//   EDGE  strips whose windows reach the left/right border (per-column counts,
//         bytes past W masked); false: interior strips [sL, sR)
//   PACK  the packed last strips (implies EDGE): lane = (group grp, lane kl of
//         G in the group), group grp = the last strip of page pack NG + grp,
//         all staged by one TMA box of NG pages x (G + 1) chunks (tin is
//         then the packed tensor map); a group is a strip of G lanes
template <int W32, int METHOD, bool EDGE, bool PACK = false>
__device__ __forceinline__ void mom5_body(const CUtensorMap& tin, const MomParams& p, int strip, int band,
                                          int page_arg) {
  constexpr int W16 = W32 & 15;
  constexpr int DL = (W32 >> 1) & 15;      // r mod 16
  constexpr int RHO = (16 - W16) & 15;     // (-w) mod 16
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem + SmemLayout::ring;
  uint4* pub = reinterpret_cast<uint4*>(smem + SmemLayout::pub);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SmemLayout::bar);

  const int lane = threadIdx.x;
  const int KH = p.KH;
  // packed strips: the lane's group and its place in it
  const int G = PACK ? p.pk_G : 32;
  const int grp = PACK ? lane / G : 0;
  const int kl = PACK ? lane - grp * G : lane;               // lane within its strip
  const int page = PACK ? page_arg * p.pk_NG + grp : page_arg;
  const bool lane_ok = !PACK || (grp < p.pk_NG && page < p.n_pages_v4);
  const int RS = PACK ? kG * (G + 1) : kSpan;                // staged row stride
  const int page0 = PACK ? page_arg * p.pk_NG : page_arg;    // TMA page coordinate
  const int64_t J0 = (int64_t)strip * p.Tw;               // first output column of the strip
  const int64_t Sw = J0 + p.r - (int64_t)kG * KH;         // input column of lane 0
  const int64_t XE = Sw - DL;                             // 16-aligned staging origin
  const int64_t y0 = p.row0 + (int64_t)band * p.B;        // first output row (global)
  const int nrows = (int)min((int64_t)p.B, p.row0 + p.H_out - y0);
  const int WS = (p.h + 2 * kR - 1) / (2 * kR);           // warm-up stages (2 kR rows each)
  const int total = WS + (nrows + kR - 1) / kR;
  const int mW = (p.w + RHO) / kG;                        // ceil(w / 16)

  const int32_t xchunk = (int32_t)(XE / 16);
  auto issue = [&](int s) {  // lane 0 only
    const int slot = s % kNS;
    uint8_t* st = ring + slot * kStageBytes;
    const uint64_t keep = (ABIN_V5_L2 & 2) ? policy_evict_normal() : policy_evict_last();
    const uint64_t drop = (ABIN_V5_L2 & 4) ? policy_evict_normal() : policy_evict_first();
    mbar_arrive_expect_tx(&full[slot], 2 * kR * RS * (PACK ? p.pk_NG : 1));
    if (s < WS) {  // warm-up rows y0-o+2kR s .. +2kR-1 into both halves of the slot
      const int32_t yw = (int32_t)(y0 - p.o + (int64_t)s * 2 * kR - p.buf_row0);
      tma_load_4d_hint(st, &tin, 0, xchunk, yw, page0, &full[slot], keep);
      tma_load_4d_hint(st + kRowsBytes, &tin, 0, xchunk, yw + kR, page0, &full[slot], keep);
    } else {
      const int64_t q0 = (int64_t)(s - WS) * kR;
      tma_load_4d_hint(st, &tin, 0, xchunk, (int32_t)(y0 + q0 + p.u - p.buf_row0), page0, &full[slot], keep);
      tma_load_4d_hint(st + kRowsBytes, &tin, 0, xchunk, (int32_t)(y0 + q0 - p.o - p.buf_row0), page0, &full[slot],
                       drop);
    }
  };

  // ---- per-lane geometry
  const int64_t a = Sw + (int64_t)kG * kl;                // first owned input column
  const int64_t j0 = a - p.r;                             // first output column (multiple of 16)
  const int64_t Jend = min(J0 + (PACK ? (int64_t)kG * (G - KH) : (int64_t)p.Tw), p.W);
  const bool valid_lane = lane_ok && kl >= KH && j0 < Jend;
  const uint32_t vmask = valid_lane ? (Jend - j0 >= kG ? 0xFFFFu : ((1u << (uint32_t)(Jend - j0)) - 1u)) : 0u;
  const float Lf = (METHOD == M_WOLF || METHOD == M_FENG)
                       ? (float)(p.L_fixed >= 0 ? p.L_fixed : (lane_ok ? (int)p.L_page[page] : 0)) : 0.0f;
  // Edge strips.  (1) -1/ncol per output column: ncol = w
  // except within (w+1)/2 columns of a border, so at most 10 lanes of a strip
  // see other counts; they get their own 16-entry slot of the table, every
  // other lane reads slot 0 (all -1/w, a broadcast).  (2) Bytes past W: TMA
  // zero-fills whole 16-byte chunks outside the image, but the chunk holding
  // column W is read as it is, so lane 0 clears its tail in each staged row.
  const float* ncol_tab = nullptr;
  int tail_off = -1;                                      // staged offset of column W (edge strips)
  if (EDGE) {
    float* tab = reinterpret_cast<float*>(smem + SmemLayout::nic);
    auto ncol = [&](int64_t j) { return max((int64_t)1, min(j + p.r, p.W - 1) - max(j - p.l, (int64_t)-1)); };
    // (output lanes only: at most ceil((l-1)/16) + ceil(r/16) + 1 <= 9 of them)
    const bool border = valid_lane && (ncol(j0) != p.w || ncol(j0 + kG - 1) != p.w);
    const uint32_t bal = __ballot_sync(0xffffffffu, border);
    const int slot = border ? 1 + __popc(bal & ((1u << lane) - 1u)) : 0;
    if (lane < kG) tab[lane] = -__frcp_rn((float)p.w);
    if (border && slot < 16) {
#pragma unroll 1
      for (int t = 0; t < kG; ++t) tab[slot * kG + t] = -__frcp_rn((float)ncol(j0 + t));
    }
    ncol_tab = tab + (slot < 16 ? slot : 0) * kG;
    const int64_t to = p.W - XE;
    if (to > 0 && to < kSpan && (to & 15)) tail_off = (int)to;
  }
  if (lane == 0) {
    for (int s = 0; s < kNS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0) {
    fence_proxy_async_smem();
    prefetch_tmap(&tin);
    for (int s = 0; s < kNS && s < total; ++s) issue(s);
  }
  auto stage_end = [&](int s) {
    __syncwarp();
    if (lane == 0 && s + kNS < total) {
      fence_proxy_async_smem();  // generic reads of the slot precede the async-proxy refill
      issue(s + kNS);
    }
  };
  auto load_row = [&](const uint8_t* sr, uint32_t (&w)[8]) {
    const uint4 x0 = *reinterpret_cast<const uint4*>(sr);
    const uint4 x1 = *reinterpret_cast<const uint4*>(sr + 16);
    w[0] = x0.x; w[1] = x0.y; w[2] = x0.z; w[3] = x0.w;
    w[4] = x1.x; w[5] = x1.y; w[6] = x1.z; w[7] = x1.w;
  };
  // edge strips: wait for a stage, then clear the bytes past W (see above)
  auto stage_wait = [&](int s) {
    mbar_wait(&full[s % kNS], (s / kNS) & 1);
    if (EDGE && tail_off >= 0) {
      if (lane == 0) {
        const int c0 = tail_off & ~15, nb = tail_off & 15;
        uint8_t* st = ring + (s % kNS) * kStageBytes;
#pragma unroll 1
        for (int z = 0; z < 2 * kR * (PACK ? p.pk_NG : 1); ++z) {
          const int zg = PACK ? z / (2 * kR) : 0, zr = PACK ? z - zg * 2 * kR : z;
          uint4* q = reinterpret_cast<uint4*>(st + (zr < kR ? zr * RS : kRowsBytes + (zr - kR) * RS) +
                                              zg * kR * RS + c0);
          uint4 v = *q;
          uint32_t* vw = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int keep = min(max(nb - 4 * g, 0), 4);  // bytes of word g below W
            vw[g] &= keep >= 4 ? ~0u : ((1u << (8 * keep)) - 1u);
          }
          *q = v;
        }
      }
      __syncwarp();
    }
  };

  // column sums, biased: C_b = 2^23 + C, D_b = 2^23 + D (exact integers < 2^24);
  // S[P] = (C_b, C_b, D_b, D_b) of columns 2P, 2P+1: one register quad, stored
  // to the published row as it is
  f2 SC[8], SD[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) SC[q] = SD[q] = splat(8388608.0f);
  const f2 M32 = splat(-32768.0f), M64 = splat(-65536.0f);
  const int eo = PACK ? grp * kR * RS + kG * kl : kG * lane;  // staged offset of the lane's 32-byte window

  // ---- warm-up: rows y0-o .. y0+u-1
  for (int s = 0; s < WS; ++s) {
    stage_wait(s);
    const uint8_t* st = ring + (s % kNS) * kStageBytes + eo;
    const int nr = min(2 * kR, p.h - s * 2 * kR);
#pragma unroll 1
    for (int rr = 0; rr < nr; ++rr) {
      uint32_t w[8];
      load_row(st + (rr < kR ? rr * RS : kRowsBytes + (rr - kR) * RS), w);
#define ABIN_V5_WU(P)                                                                          \
  {                                                                                            \
    const f2 x = add2(pk(own_f<DL, 2 * P>(w), own_f<DL, 2 * P + 1>(w)), M32);                 \
    SC[P] = add2(SC[P], x);                                                                    \
    SD[P] = fma2(x, x, SD[P]);                                                                 \
  }
      ABIN_V5_WU(0) ABIN_V5_WU(1) ABIN_V5_WU(2) ABIN_V5_WU(3)
      ABIN_V5_WU(4) ABIN_V5_WU(5) ABIN_V5_WU(6) ABIN_V5_WU(7)
#undef ABIN_V5_WU
    }
    stage_end(s);
  }

  // centre rows (the pixels decided): one 16-byte load per lane per row, one row ahead
  const int64_t cx = j0;
  const int cmode = !lane_ok ? 0 : ((cx >= 0 && cx + kG <= p.W) ? 1 : ((cx >= 0 && cx < p.W) ? 2 : 0));
  const uint8_t* cptr = p.in + (int64_t)page * p.in_page_stride + (y0 - p.buf_row0) * p.in_pitch + cx;
  auto load_centre = [&](const uint8_t* src) -> uint4 {
    if (cmode == 0) return make_uint4(0, 0, 0, 0);
    if (!EDGE || cmode == 1) return __ldg(reinterpret_cast<const uint4*>(src));
    // columns past W read as 255: their outputs are not stored, but a window
    // wholly outside the image has c = 0 and t~ = 0, and I = 0 there would
    // make the lane ambiguous (queued for the exact fixup) for nothing
    uint32_t wd[4] = {~0u, ~0u, ~0u, ~0u};
    for (int t = 0; t < kG; ++t)
      if (cx + t < p.W) wd[t >> 2] ^= (255u ^ (uint32_t)__ldg(src + t)) << (8 * (t & 3));
    return make_uint4(wd[0], wd[1], wd[2], wd[3]);
  };
  uint4 xc_next = nrows > 0 ? load_centre(cptr) : make_uint4(0, 0, 0, 0);
  uint8_t* optr = p.out + (int64_t)page * p.out_page_stride + (y0 - p.row0) * p.out_pitch +
                  (p.fmt == 0 ? j0 : (j0 >> 3));
  const bool out_vec = ((reinterpret_cast<uintptr_t>(p.out) | (uintptr_t)p.out_pitch |
                         (uintptr_t)p.out_page_stride) & 15u) == 0 && vmask == 0xFFFFu;
  const uint32_t store_mode = !valid_lane ? 0u : (p.fmt != 0 ? 3u : (out_vec ? 1u : 2u));
  const int64_t i_full0 = p.o - 1, i_full1 = p.H_global - 1 - p.u;  // nrow == h for i in [i_full0, i_full1]
  const int32_t row_lo = (int32_t)max(i_full0, (int64_t)INT32_MIN), row_hi = (int32_t)min(i_full1, (int64_t)INT32_MAX);

  f2 fa2, fb2;
  method_consts<METHOD>(p.fa, p.fb, fa2, fb2);
  if (METHOD == M_FENG) {
    fa2 = splat(p.fa);
    fb2 = pk(p.fb, p.aux2);
  }
  // Rais: the page's M S (fl32 of the double product) in the L slot, and the
  // certified bound delta1 + aux1 / (M S) (the fraction's derivative is <= 1 / (M S))
  const float MSf = METHOD == M_RAIS && lane_ok ? (float)(p.rp.MS[2 * page] * p.rp.MS[2 * page + 1]) : 0.0f;
  const f2 Lf2 = splat(METHOD == M_RAIS ? MSf : Lf);
  const float delta1 = METHOD == M_RAIS ? p.delta1 + p.aux1 / fmaxf(MSf, 1e-30f) : p.delta1;
  const f2 y2 = METHOD == M_FENG ? pk(p.aux0, p.aux1) : splat(p.aux1);  // Phansalkar: q log2(e); Feng: (k1, k2)
  // interior columns: ncol = w; per-row -1/n = -(1/w)(1/nrow) computed once per row
  const float inv_w = __frcp_rn((float)p.w);
  const int64_t in_pitch = p.in_pitch, out_pitch = p.out_pitch;
  // the leaving reads: column pair slots of blocks lane - m (+1) in the published row
  // the start value's bias: w 2^23 (mod 2^32), less one 2^23 for c (carried as 2^23 + c)
  const uint32_t dbias = (uint32_t)p.w * kBias, cbias = dbias - kBias;
  // (halo lanes k < m point below the row: into the ring, read but unused)
  const uint4* lrow0 = pub + (lane - mW);

  // M_MAXS: pass 0 keeps the lane's smallest -v~; pass 1 selects v~ >= vthr
  float vbest = __int_as_float(0x7f800000);
  const float vthr = (METHOD == M_MAXS && p.maxs_pass == 1)
                         ? __int_as_float((int)p.vmax_bits[page]) - p.maxs_margin : 0.0f;
  // ---- main rows
  int q = 0;
  for (int s = WS; s < total; ++s) {
    stage_wait(s);
    const uint8_t* st = ring + (s % kNS) * kStageBytes + eo;
    const int nr = min(kR, nrows - (s - WS) * kR);
#pragma unroll 1
    for (int rr = 0; rr < nr; ++rr, ++q) {
      const int64_t i = y0 + q;  // global output row
      const uint4 xc = xc_next;
      if (q + 1 < nrows) cptr += in_pitch;  // the last row re-reads itself (harmless)
      xc_next = load_centre(cptr);
      // ---- vertical update, exact in fp32
      {
        uint32_t wi[8], wo[8];
        load_row(st + rr * RS, wi);
        load_row(st + kRowsBytes + rr * RS, wo);
#define ABIN_V5_VU(P)                                                                                 \
  {                                                                                                   \
    const f2 fi = pk(own_f<DL, 2 * P>(wi), own_f<DL, 2 * P + 1>(wi));                                 \
    const f2 fo = pk(own_f<DL, 2 * P>(wo), own_f<DL, 2 * P + 1>(wo));                                 \
    const f2 dx = sub2(fi, fo);            /* x - y */                                                \
    const f2 sx = add2(add2(fi, fo), M64); /* x + y */                                                \
    SC[P] = add2(SC[P], dx);                                                                          \
    SD[P] = fma2(dx, sx, SD[P]);                                                                      \
  }
        ABIN_V5_VU(0) ABIN_V5_VU(1) ABIN_V5_VU(2) ABIN_V5_VU(3)
        ABIN_V5_VU(4) ABIN_V5_VU(5) ABIN_V5_VU(6) ABIN_V5_VU(7)
#undef ABIN_V5_VU
      }
      // ---- the lane's column totals (exact integers mod 2^32, on the biased
      // bit patterns: each carries 2^23 per column): all 16 columns (tc, td)
      // and the first RHO of them (pc, pd) -- for the start value below
      uint32_t tc, td, pc = 0u, pd = 0u;
      {
        uint32_t cA = 0u, dA = 0u, cB = 0u, dB = 0u;
#pragma unroll
        for (int P = 0; P < 8; ++P) {
          const uint32_t c0 = (uint32_t)SC[P], c1 = (uint32_t)(SC[P] >> 32);
          const uint32_t d0 = (uint32_t)SD[P], d1 = (uint32_t)(SD[P] >> 32);
          if (2 * P + 1 < RHO) { pc += c0 + c1; pd += d0 + d1; }
          else if (2 * P < RHO) { pc += c0; pd += d0; }
          if (P & 1) { cB += c0 + c1; dB += d0 + d1; } else { cA += c0 + c1; dA += d0 + d1; }
        }
        tc = cA + cB;
        td = dA + dB;
      }
      // ---- publish the row's column sums (single buffer: the first
      // __syncwarp orders the stores after the previous row's leaving reads)
      __syncwarp();
#pragma unroll
      for (int P = 0; P < 8; ++P) {
        const uint32_t addr = smem_u32(pub + P * 32 + lane);
        asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(addr), "l"(SC[P]), "l"(SD[P]) : "memory");
      }
      __syncwarp();
      // ---- start value: the window sum at column a - r - 1,
      // S = sum of C over [a - w, a) = totals of lanes k-1 .. k-m minus the
      // first RHO columns of lane k - m (a - w = a_{k-m} + RHO, m = ceil(w/16)).
      // The biases cancel but for w 2^23 (mod 2^32).  Halo lanes (k < m) read
      // wrapped-around lanes: their outputs are discarded.
      uint32_t Sc = 0u - __shfl_up_sync(0xffffffffu, pc, mW), Sd = 0u - __shfl_up_sync(0xffffffffu, pd, mW);
      switch (mW) {  // warp-uniform; shfl.up: lanes below q keep their own (unused) value
        case 8: Sc += __shfl_up_sync(0xffffffffu, tc, 8); Sd += __shfl_up_sync(0xffffffffu, td, 8);  // fall through
        case 7: Sc += __shfl_up_sync(0xffffffffu, tc, 7); Sd += __shfl_up_sync(0xffffffffu, td, 7);  // fall through
        case 6: Sc += __shfl_up_sync(0xffffffffu, tc, 6); Sd += __shfl_up_sync(0xffffffffu, td, 6);  // fall through
        case 5: Sc += __shfl_up_sync(0xffffffffu, tc, 5); Sd += __shfl_up_sync(0xffffffffu, td, 5);  // fall through
        case 4: Sc += __shfl_up_sync(0xffffffffu, tc, 4); Sd += __shfl_up_sync(0xffffffffu, td, 4);  // fall through
        case 3: Sc += __shfl_up_sync(0xffffffffu, tc, 3); Sd += __shfl_up_sync(0xffffffffu, td, 3);  // fall through
        case 2: Sc += __shfl_up_sync(0xffffffffu, tc, 2); Sd += __shfl_up_sync(0xffffffffu, td, 2);  // fall through
        default: Sc += __shfl_up_sync(0xffffffffu, tc, 1); Sd += __shfl_up_sync(0xffffffffu, td, 1);
      }
      // ---- row recursion fused with the epilogue (Alg. 1
      // l.118-124, Table 1): c(t) = c(t-1) + C[a+t] - C[a+t-w], exact; c is
      // carried as the bits of the float 2^23 + c (c < 2^23), d as an integer
      uint32_t cc = Sc - cbias, dd = Sd - dbias;
      float inv_nrow = p.inv_h;
      if ((int32_t)i < row_lo || (int32_t)i > row_hi) {
        const uint32_t nrow = (uint32_t)(min(i + p.u, p.H_global - 1) - max(i - p.o, (int64_t)-1));
        inv_nrow = __frcp_rn((float)nrow);
      }
      f2 nu = splat(-(inv_w * inv_nrow));                     // -1/n (interior columns)
      f2 nb = mul2(nu, splat(-8388608.0f));                   // -2^23 nu (exact)
      uint32_t wv[4];
      float emin = __int_as_float(0x7f800000), smin = emin;
      uint32_t amb_m = 0u;  // M_MAXS pass 1: pixels within the margin of the page's max v~
      uint4 L = lrow0[(RHO >> 1) * 32];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint32_t wd = g == 0 ? xc.x : (g == 1 ? xc.y : (g == 2 ? xc.z : xc.w));
        float e4[4];
#pragma unroll
        for (int h2 = 0; h2 < 4; h2 += 2) {
          const int t0 = 4 * g + h2;
          uint32_t cq[2], dq[2];
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            const int t = t0 + z;
            const int pos = RHO + t;               // position in block lane - m (>= 16: next block)
            const int blk = pos >> 4, pp = pos & 15;
            if (t > 0 && (pp & 1) == 0) L = lrow0[(pp >> 1) * 32 + blk];
            const uint32_t lc = (pp & 1) ? L.y : L.x, ld = (pp & 1) ? L.w : L.z;
            const uint32_t oc = (t & 1) ? (uint32_t)(SC[t >> 1] >> 32) : (uint32_t)SC[t >> 1];
            const uint32_t od = (t & 1) ? (uint32_t)(SD[t >> 1] >> 32) : (uint32_t)SD[t >> 1];
            cc += oc - lc;
            dd += od - ld;
            cq[z] = cc;
            dq[z] = dd;
          }
          if (EDGE) {
            const float2 nc = *reinterpret_cast<const float2*>(ncol_tab + t0);  // -1/ncol
            nu = mul2(pk(nc.x, nc.y), splat(inv_nrow));
            nb = mul2(nu, splat(-8388608.0f));
          }
          // I exactly: the byte as 32768 + I, minus 32768
          const f2 I = add2(pk(__uint_as_float(__byte_perm(wd, kMagic, 0x7504u | ((uint32_t)h2 << 4))),
                               __uint_as_float(__byte_perm(wd, kMagic, 0x7504u | ((uint32_t)(h2 + 1) << 4)))),
                            M32);
          if (METHOD == M_MAXS) {
            // v~ = q~ - m~^2 (the filter's own variance, |v~ - v| <= dv)
            const f2 mn = fma2(pk(__uint_as_float(cq[0]), __uint_as_float(cq[1])), nu, nb);
            const f2 wv = fma2(mn, mn, mul2(pk((float)dq[0], (float)dq[1]), nu));  // -v~
            const bool va = (vmask >> t0) & 1u, vb = (vmask >> (t0 + 1)) & 1u;
            const float xa = va ? lo(wv) : __int_as_float(0x7f800000), xb = vb ? hi(wv) : __int_as_float(0x7f800000);
            if (p.maxs_pass == 0) {
              emin = fmin3(emin, xa, xb);                       // min of -v~ = -(max v~)
            } else {
              amb_m |= (-xa >= vthr ? 1u : 0u) << t0;
              amb_m |= (-xb >= vthr ? 1u : 0u) << (t0 + 1);
            }
            e4[h2] = e4[h2 + 1] = 0.0f;
            (void)I;
            continue;
          }
          f2 sv;
          const f2 e = residual_pair<METHOD>(cq[0], cq[1], dq[0], dq[1], nu, nb, I, fa2, fb2,
                                             aux_operand<METHOD>(p, Lf2, nu), sv, y2);
          emin = fmin3(emin, fabsf(lo(e)), fabsf(hi(e)));
          if (METHOD == M_NIBLACK || METHOD == M_KHURSHID || METHOD == M_RAIS || METHOD == M_FENG)
            smin = fmin3(smin, lo(sv), hi(sv));
          e4[h2] = lo(e);
          e4[h2 + 1] = hi(e);
        }
        // byte t of wv[g] = (e_t >= 0): prmt replicates the selected bytes' sign bits
        const uint32_t lo = prmt_sign(__float_as_uint(e4[0]), __float_as_uint(e4[1]), 0x00FBu);
        const uint32_t hi = prmt_sign(__float_as_uint(e4[2]), __float_as_uint(e4[3]), 0xFB00u);
        wv[g] = ~__byte_perm(lo, hi, 0x7610u) & 0x01010101u;
      }
      if (METHOD == M_MAXS) {
        if (p.maxs_pass == 0) {
          vbest = fminf(vbest, emin);
        } else if (amb_m) {
          const uint32_t slot = atomicAdd(p.q_count, 1u);
          if (slot < p.q_cap) p.q_data[slot] = make_uint4((uint32_t)page, (uint32_t)(i - p.row0), (uint32_t)j0, amb_m);
        }
        continue;  // no mask
      }
      // ambiguous lane: a pixel within the certified bound.  Niblack re-tests
      // with the data-dependent bound at its smallest s~ (v4 refined_bound)
      uint32_t amb = 0u;
      if (emin < delta1) {
        if constexpr (METHOD == M_RAIS) {
          // the data-dependent bound at the lane's smallest s~, its 1/(M S) parts added per page
          const float iMS = 1.0f / fmaxf(MSf, 1e-30f);
          const float rb0 = p.rb0 + p.aux0 * iMS, rb1 = p.rb1 + p.rais_r1 * iMS;
          if (emin * 0.999999f < (rb0 + rb1 * fminf(p.rsdv, p.rdv / smin)) * 1.000001f) amb = vmask;
        } else if ((METHOD != M_NIBLACK && METHOD != M_KHURSHID && METHOD != M_FENG) ||
                   emin * 0.999999f < v4::refined_bound(p, smin)) {
          amb = vmask;
        }
      }
      if (amb) {
        const uint32_t slot = atomicAdd(p.q_count, 1u);
        if (slot < p.q_cap) p.q_data[slot] = make_uint4((uint32_t)page, (uint32_t)(i - p.row0), (uint32_t)j0, amb);
      }
      // ---- store the mask: outputs j0 .. j0+15
      if (store_mode != 0u) {
        if (store_mode == 1u) {
          if (ABIN_V5_L2 & 1) st_global_hint(optr, make_uint4(wv[0], wv[1], wv[2], wv[3]), policy_evict_first());
          else __stcs(reinterpret_cast<uint4*>(optr), make_uint4(wv[0], wv[1], wv[2], wv[3]));  // streaming
        } else if (store_mode == 2u) {
#pragma unroll
          for (int t = 0; t < kG; ++t)
            if ((vmask >> t) & 1u) optr[t] = (uint8_t)(wv[t >> 2] >> (8 * (t & 3)));
        } else {
          uint32_t mbits = 0;
#pragma unroll
          for (int g = 0; g < 4; ++g) mbits |= (((wv[g] * 0x01020408u) >> 24) & 0xFu) << (4 * g);
          const uint32_t mb = __brev(mbits & vmask) >> 16;  // bit 15 - t = mask of output t (MSB-first)
          optr[0] = (uint8_t)(mb >> 8);
          if (vmask >> 8) optr[1] = (uint8_t)(mb & 0xFFu);
        }
      }
      optr += out_pitch;
    }
    stage_end(s);
  }
  if (METHOD == M_MAXS && p.maxs_pass == 0) {
    // max v~ of the tile (>= 0: a clamp at 0 keeps the float bits ordered)
    float vb = vbest;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) vb = fminf(vb, __shfl_xor_sync(0xffffffffu, vb, off));
    if (lane == 0 && vb < __int_as_float(0x7f800000)) atomicMax(p.vmax_bits + page, __float_as_uint(fmaxf(-vb, 0.0f)));
  }
}

// One launch for all strips: the border strips get the low block indices.
template <int W32, int METHOD>
__global__ void __launch_bounds__(32, ABIN_V5_MINB) k_mom5(const __grid_constant__ CUtensorMap tin,
                                                           const __grid_constant__ CUtensorMap tpk, const MomParams p) {
  // the dependent k_fixup grid (PDL) may be scheduled once every CTA has started
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // tiles: the edge strips (less the last strip when it is packed), then the
  // packed last strips (pk_n per band), then the interior strips
  const int nE = p.sL + (p.n_strips - (p.pk_on ? 1 : 0) - p.sR);
  const int64_t per_strip = (int64_t)p.n_bands * p.n_pages_v4;
  const int64_t te = (int64_t)nE * per_strip;
  const int64_t tp = p.pk_on ? (int64_t)p.pk_n * p.n_bands : 0;
  int64_t tile = blockIdx.x;
  if (tile < te) {
    const int si = (int)(tile % nE);
    tile /= nE;
    const int strip = si < p.sL ? si : p.sR + (si - p.sL);
    mom5_body<W32, METHOD, true>(tin, p, strip, (int)(tile % p.n_bands), (int)(tile / p.n_bands));
  } else if (tile < te + tp) {
    if constexpr (METHOD != M_MAXS) {  // (the host packs no M_MAXS launch)
      tile -= te;
      mom5_body<W32, METHOD, true, true>(tpk, p, p.n_strips - 1, (int)(tile % p.n_bands), (int)(tile / p.n_bands));
    }
  } else {
    tile -= te + tp;
    const int nI = p.sR - p.sL;
    const int strip = p.sL + (int)(tile % nI);
    tile /= nI;
    mom5_body<W32, METHOD, false>(tin, p, strip, (int)(tile % p.n_bands), (int)(tile / p.n_bands));
  }
}

}  // namespace v5
}  // namespace abin
