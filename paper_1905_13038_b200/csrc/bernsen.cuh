// bernsen.cuh -- Bernsen's midrange rule (Sec. 3.4
// "Generalization": "used midrange as threshold value" of the window's gray
// levels) with work per pixel independent of the window size, the Theta(HW)
// the paragraph claims for it ("it is obvious that ... can be implemented in
// Theta(HW)").  The paper's device is a monotone deque per row/column; on the
// GPU we use the van Herk / Gil-Werman block decomposition instead, which has
// no data-dependent control flow: cut a line into blocks of the window length
// L; a window [a, a+L-1] starting in block b is the suffix of b from a plus the
// prefix of b+1 up to a+L-1, so
//     ext[a] = op(S_b[a], P_{b+1}[a+L-1])
// with S (suffix extrema, one backward pass per block) and P (prefix extrema,
// running forward): three extremum operations per element per direction.
//
// Extrema are separable: the window's min (max) is the min (max) over its rows
// of the row-window mins (maxes).  Min and max are computed together on the
// packed pair (x, 255 - x) in 16-bit lanes: one VIMNMX.U16x2 minimum yields
// (min x, 255 - max x).  Two kernels:
//   k_bern_h  rows: a warp stages 32 rows of a column tile in shared memory
//             (coalesced 16-byte loads), each lane runs the block scan along
//             its own row, and the tile's (min, 255 - max) pairs are written
//             out coalesced (2 bytes per pixel, scratch hb).
//   k_bern_v  columns: a thread owns 8 columns and runs the block scan down
//             them over hb (16-byte loads; suffix extrema kept in scratch sb),
//             then decides I' = 0 iff 2 I <= min + max (exact integers), the
//             local-contrast variant background where max - min < contrast.
// Border convention (PAPER.md:83 applied to extrema, as the oracle's
// direct_extrema): only in-bounds pixels take part.  Columns: an index clamped
// to [0, W-1] repeats the edge pixel, which lies inside every clipped window
// that reaches past the edge, so the extrema are unchanged.  Rows: rows
// outside the image are the identity (255, 255).
#pragma once
#include <cstdint>

namespace abin {
namespace bern {

struct BernParams {
  const uint8_t* in;              // first held row (global row buf_row0) of page 0
  int64_t in_page_stride, in_pitch, W;
  int64_t buf_row0;
  int64_t Y0, Yn;                 // global rows [Y0, Y0 + Yn) of the row pass (clipped to the image)
  int64_t row0, H_out, H_global;  // output rows [row0, row0 + H_out) of an image H_global tall
  uint8_t* out;
  int64_t out_pitch, out_page_stride;
  int32_t fmt;                    // 0 bytes, 1 MSB-first bits
  int32_t w, l, h, o;             // window (effective): columns (j-l, j-l+w], rows (i-o, i-o+h]
  int32_t contrast;               // < 0: plain midrange
  uint16_t* hb;                   // row-pass extrema (min | (255 - max) << 8), [page][Yn][hpitch]
  uint16_t* sb;                   // column-pass suffix extrema, [page][H_out][hpitch] (null: shared memory)
  int64_t hpitch;                 // elements, multiple of 8
  int32_t TW;                     // k_bern_h: output columns per tile
  int32_t SP;                     // k_bern_h: staged row pitch in shared memory (bytes, 4 mod 8)
  int32_t OBP;                    // k_bern_h: output staging row pitch (u16 elements, 2 mod 4)
  int32_t n_ctiles, n_rtiles;     // k_bern_h tiles per page
  int32_t n_groups;               // k_bern_v: 8-column groups per page
  int32_t n_gblocks;              // k_bern_v: CTAs of 32 groups per page and chunk
  int32_t n_chunks;               // k_bern_v: row chunks (one window-length block of outputs each) per page
  int32_t sbs;                    // k_bern_v: rows per sub-block (R = blockDim.y sub-blocks per chunk)
  int32_t n_pages;
};

constexpr int kBernMaxW = 2048;        // effective width (the row pass's shared memory)
constexpr uint32_t kId = 0x00FF00FFu;  // identity of the packed minimum: (255, 255)

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// gray level x -> (x, 255 - x): x (0xFFFF0001) + 0x00FF0000 = x - x 2^16 + 255 2^16 (mod 2^32)
__device__ __forceinline__ uint32_t expand(uint32_t x) { return x * 0xFFFF0001u + 0x00FF0000u; }
// stored pair (bytes m, M') -> (m, M') in 16-bit lanes, and back
__device__ __forceinline__ uint32_t unpack(uint32_t v) { return __byte_perm(v, 0u, 0x4140u); }
__device__ __forceinline__ uint32_t pack(uint32_t v) { return __byte_perm(v, 0u, 0x4420u); }

// shared memory of one k_bern_h warp: staged rows, suffix extrema, output rows
__host__ __device__ inline int h_smem_bytes(int SP, int w, int OBP) { return 32 * SP + 64 * w + 64 * OBP; }

// ---- row pass: one warp = 32 rows x TW output columns
__global__ void __launch_bounds__(32) k_bern_h(const BernParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int lane = threadIdx.x;
  int64_t t = blockIdx.x;
  const int ct = (int)(t % p.n_ctiles);
  t /= p.n_ctiles;
  const int rt = (int)(t % p.n_rtiles);
  const int page = (int)(t / p.n_rtiles);
  const int64_t W = p.W;
  const int w = p.w;
  const int64_t j0 = (int64_t)ct * p.TW;                    // first output column
  const int nout = (int)min((int64_t)p.TW, W - j0);
  const int64_t xs = j0 - p.l + 1;                          // input column of position 0 (window start of j0)
  const int64_t xa = xs & ~(int64_t)15;                     // 16-aligned staging origin
  const int d = (int)(xs - xa);
  const int span = nout + w;                                // positions read: [0, nout + w) (+1 slack read)
  const int nch = (d + span + 15) >> 4;                     // 16-byte chunks per staged row
  uint8_t* tile = sm;                                       // [32][SP]
  uint16_t* S = reinterpret_cast<uint16_t*>(sm + 32 * p.SP);  // [w][32]
  uint16_t* ob = S + 32 * w;                                // [32][OBP]
  const uint8_t* pbase = p.in + (int64_t)page * p.in_page_stride;
  const int64_t Yt = p.Y0 + (int64_t)rt * 32;               // global row of tile row 0
  const int nrows = (int)min((int64_t)32, p.Y0 + p.Yn - Yt);
  const bool vec = ((reinterpret_cast<uintptr_t>(p.in) | (uintptr_t)p.in_pitch |
                     (uintptr_t)p.in_page_stride) & 15u) == 0;

  // ---- stage the rows (chunk c of row k covers input columns xa + 16c ..):
  // 8 rows' loads in flight per lane before their shared-memory stores
  auto load_chunk = [&](int k, int c) -> uint4 {
    const uint8_t* row = pbase + (Yt + k - p.buf_row0) * p.in_pitch;
    const int64_t x = xa + 16 * c;
    if (vec && x >= 0 && x + 16 <= W) return __ldg(reinterpret_cast<const uint4*>(row + x));
    uint32_t v[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t z = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t xx = min(max(x + 4 * g + b, (int64_t)0), W - 1);  // edge repeat
        z |= (uint32_t)__ldg(row + xx) << (8 * b);
      }
      v[g] = z;
    }
    return make_uint4(v[0], v[1], v[2], v[3]);
  };
#pragma unroll 1
  for (int k0 = 0; k0 < nrows; k0 += 8) {
#pragma unroll 1
    for (int c = lane; c < nch; c += 32) {
      uint4 v[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        if (k0 + kk < nrows) v[kk] = load_chunk(k0 + kk, c);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        if (k0 + kk < nrows) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(tile + (k0 + kk) * p.SP) + 4 * c;
          dst[0] = v[kk].x; dst[1] = v[kk].y; dst[2] = v[kk].z; dst[3] = v[kk].w;
        }
    }
  }
  __syncwarp();

  // ---- block scans along the lane's row (positions i = 0 .. nout + w - 1)
  if (lane < nrows) {
    const uint8_t* r = tile + lane * p.SP + d;
    uint16_t* Sl = S + lane;
    uint16_t* ol = ob + lane * p.OBP;
    for (int b0 = 0; b0 < nout; b0 += w) {
      // suffix extrema of block [b0, b0 + w)
      uint32_t s = kId;
      const uint8_t* q = r + b0 + w - 1;
#pragma unroll 4
      for (int i = w - 1; i >= 0; --i, --q) {
        s = vmin2(s, expand(*q));
        Sl[32 * i] = (uint16_t)pack(s);
      }
      // prefix extrema of block [b0 + w, b0 + 2w), outputs b0 .. b0 + tn - 1
      const int tn = min(w, nout - b0);
      uint32_t P = kId;
      q = r + b0 + w;
#pragma unroll 4
      for (int i = 0; i < tn; ++i, ++q) {
        ol[b0 + i] = (uint16_t)pack(vmin2(unpack(Sl[32 * i]), P));
        P = vmin2(P, expand(*q));
      }
    }
  }
  __syncwarp();

  // ---- write the tile's rows out: 16-byte pieces (8 outputs), TW / 8 per row
  // (a piece past W lands in the row padding: hpitch = W rounded up to 8)
  const int cps = p.TW == 128 ? 4 : 5;                      // log2 of the pieces per row
  uint16_t* hbt = p.hb + (int64_t)page * p.Yn * p.hpitch + (Yt - p.Y0) * p.hpitch + j0;
#pragma unroll 2
  for (int idx = lane; idx < (nrows << cps); idx += 32) {
    const int k = idx >> cps, c = idx & ((1 << cps) - 1);
    if (8 * c < nout) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(ob + k * p.OBP) + 4 * c;
      *reinterpret_cast<uint4*>(hbt + (int64_t)k * p.hpitch + 8 * c) = make_uint4(src[0], src[1], src[2], src[3]);
    }
  }
}

// ---- column pass.  A CTA = 32 groups of 8 columns x R sub-blocks; a chunk
// is one window-length block of output rows [yb, yb + h), whose windows start
// in the block A = [ab, ab + h) (ab = yb - o + 1) and end in B = [ab + h,
// ab + 2h).  Thread (g, k) takes rows [k sbs, (k+1) sbs) of A and B:
//   1. suffix extrema over its part of A (backward, stored per output row in
//      sb), its aggregate aggA_k;  2. the aggregate aggB_k of its part of B;
//   3. S_t = min(local suffix_t, aggA of the later parts), P_t = min(aggB of
//      the earlier parts, prefix of its own part of B up to row t-1): the
//      output t is min(S_t, P_t) -- the block scan split over R threads.
// Rows are loaded 4 ahead (16-byte loads; each thread's chain of minima is
// short, the latency of its loads is what it waits for).
constexpr int kVPre = 4;

__device__ __forceinline__ void load_pairs(const BernParams& p, const uint16_t* hb, int64_t Y, uint4& q) {
  if (Y < p.Y0 || Y >= p.Y0 + p.Yn) {
    q = make_uint4(~0u, ~0u, ~0u, ~0u);  // absent row: the identity, bytes (m, M') = (255, 255) per pixel
    return;
  }
  q = __ldg(reinterpret_cast<const uint4*>(hb + (Y - p.Y0) * p.hpitch));
}
// 8 stored pairs (bytes m, M') -> minimum into s[8] (16-bit lanes)
__device__ __forceinline__ void min_in(uint32_t (&s)[8], const uint4& q) {
  s[0] = vmin2(s[0], unpack(q.x)); s[1] = vmin2(s[1], unpack(q.x >> 16));
  s[2] = vmin2(s[2], unpack(q.y)); s[3] = vmin2(s[3], unpack(q.y >> 16));
  s[4] = vmin2(s[4], unpack(q.z)); s[5] = vmin2(s[5], unpack(q.z >> 16));
  s[6] = vmin2(s[6], unpack(q.w)); s[7] = vmin2(s[7], unpack(q.w >> 16));
}
__device__ __forceinline__ uint4 pack8(const uint32_t (&s)[8]) {
  return make_uint4(__byte_perm(s[0], s[1], 0x6420u), __byte_perm(s[2], s[3], 0x6420u),
                    __byte_perm(s[4], s[5], 0x6420u), __byte_perm(s[6], s[7], 0x6420u));
}

__global__ void __launch_bounds__(256) k_bern_v(const BernParams p) {
  __shared__ uint4 agg[2][8][32];                          // packed aggregates of A / B parts
  const int tx = threadIdx.x, k = threadIdx.y, R = blockDim.y;
  int64_t b = blockIdx.x;
  const int gb = (int)(b % p.n_gblocks);
  b /= p.n_gblocks;
  const int chunk = (int)(b % p.n_chunks);
  const int page = (int)(b / p.n_chunks);
  const int g = gb * 32 + tx;
  const int64_t j = 8 * (int64_t)g;
  const bool active = g < p.n_groups;
  const int h = p.h, sbs = p.sbs;
  const int64_t yb = p.row0 + (int64_t)chunk * h;          // first output row of the chunk
  const int nq = (int)min((int64_t)h, p.row0 + p.H_out - yb);
  const int64_t ab = yb - p.o + 1;
  const int i0 = k * sbs, i1 = min(i0 + sbs, h);           // this thread's part of A and B
  const uint16_t* hb = p.hb + (int64_t)page * p.Yn * p.hpitch + (active ? j : 0);
  // the local suffixes: shared memory [k][row - i0][tx] (16 bytes per row), or
  // the global scratch sb for windows too tall for it
  extern __shared__ uint4 ssm[];
  const bool gsb = p.sb != nullptr;
  uint16_t* sb = gsb ? p.sb + (int64_t)page * p.H_out * p.hpitch + (yb - p.row0) * p.hpitch + (active ? j : 0) : nullptr;
  uint4* sl = ssm + (int64_t)k * sbs * 32 + tx;
  auto s_store = [&](int i, const uint4& v) {
    if (gsb) *reinterpret_cast<uint4*>(sb + (int64_t)i * p.hpitch) = v;
    else sl[(i - i0) * 32] = v;
  };
  auto s_load = [&](int i) -> uint4 {
    return gsb ? *reinterpret_cast<const uint4*>(sb + (int64_t)i * p.hpitch) : sl[(i - i0) * 32];
  };

  uint32_t s[8], a[8];
#pragma unroll
  for (int z = 0; z < 8; ++z) s[z] = a[z] = kId;
  if (active) {
    // 1. suffix extrema of A's part (backward), stored for the chunk's outputs
    {
      uint4 q[kVPre];
#pragma unroll
      for (int d = 0; d < kVPre; ++d)
        if (i1 - 1 - d >= i0) load_pairs(p, hb, ab + i1 - 1 - d, q[d]);
      for (int i = i1 - 1; i >= i0; i -= kVPre) {
#pragma unroll
        for (int d = 0; d < kVPre; ++d) {
          const int ii = i - d;
          if (ii >= i0) {
            min_in(s, q[d]);
            if (ii - kVPre >= i0) load_pairs(p, hb, ab + ii - kVPre, q[d]);
            if (ii < nq) s_store(ii, pack8(s));
          }
        }
      }
    }
    // 2. aggregate of B's part (only rows that end some output's window: < nq - 1)
    {
      const int e1 = min(i1, nq - 1);
      uint4 q[kVPre];
#pragma unroll
      for (int d = 0; d < kVPre; ++d)
        if (i0 + d < e1) load_pairs(p, hb, ab + h + i0 + d, q[d]);
      for (int i = i0; i < e1; i += kVPre) {
#pragma unroll
        for (int d = 0; d < kVPre; ++d) {
          const int ii = i + d;
          if (ii < e1) {
            min_in(a, q[d]);
            if (ii + kVPre < e1) load_pairs(p, hb, ab + h + ii + kVPre, q[d]);
          }
        }
      }
    }
  }
  agg[0][k][tx] = pack8(s);
  agg[1][k][tx] = pack8(a);
  __syncthreads();
  if (!active || i0 >= nq) return;
  // 3. the parts' suffix / prefix of aggregates
  uint32_t sa[8], pb[8];
#pragma unroll
  for (int z = 0; z < 8; ++z) sa[z] = pb[z] = kId;
  for (int kk = k + 1; kk < R; ++kk) min_in(sa, agg[0][kk][tx]);
  for (int kk = 0; kk < k; ++kk) min_in(pb, agg[1][kk][tx]);
  // 4. outputs t in [i0, min(i1, nq)): min(S_t, P_t), then the decision
  const int t1 = min(i1, nq);
  const uint8_t* ib = p.in + (int64_t)page * p.in_page_stride + (yb + i0 - p.buf_row0) * p.in_pitch + j;
  uint8_t* obase = p.out + (int64_t)page * p.out_page_stride + (yb + i0 - p.row0) * p.out_pitch;
  const int nval = (int)min((int64_t)8, p.W - j);
  const bool cvec = nval == 8 && ((reinterpret_cast<uintptr_t>(ib) | (uintptr_t)p.in_pitch) & 7u) == 0;
  const bool ovec = p.fmt == 0 && nval == 8 &&
                    ((reinterpret_cast<uintptr_t>(obase + j) | (uintptr_t)p.out_pitch) & 7u) == 0;
  const int c = p.contrast;
  const uint32_t kc = (uint32_t)(0x8000 - 256 + max(c, 0)) * 0x10001u;
  uint4 qb[kVPre], qs[kVPre];
#pragma unroll
  for (int d = 0; d < kVPre; ++d)
    if (i0 + d < t1) {
      load_pairs(p, hb, ab + h + i0 + d, qb[d]);
      qs[d] = s_load(i0 + d);
    }
  for (int t = i0; t < t1; t += kVPre) {
#pragma unroll
    for (int d = 0; d < kVPre; ++d) {
      const int tt = t + d;
      if (tt < t1) {
        uint32_t I0 = 0, I1 = 0;
        if (cvec) {
          const uint2 x = __ldg(reinterpret_cast<const uint2*>(ib));
          I0 = x.x; I1 = x.y;
        } else {
          for (int z = 0; z < nval; ++z) {
            if (z < 4) I0 |= (uint32_t)__ldg(ib + z) << (8 * z);
            else I1 |= (uint32_t)__ldg(ib + z) << (8 * (z - 4));
          }
        }
        uint32_t e[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) e[z] = pb[z];
        min_in(e, qs[d]);
#pragma unroll
        for (int z = 0; z < 8; ++z) e[z] = vmin2(e[z], sa[z]);
        // decision on pixel pairs in 16-bit lanes (lo = min, M' = 255 - max):
        //   0x8000 + (lo + hi - 2 I) = (lo + 0x80FF) - (2 I + M'): bit 15 set iff 2 I <= lo + hi
        //   (lo + M') + 0x8000 - 256 + c: bit 15 set iff lo + M' >= 256 - c, i.e. max - min < c
        uint32_t mw[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t Iw = hh ? I1 : I0;
          uint32_t pr[2];
#pragma unroll
          for (int m2 = 0; m2 < 2; ++m2) {
            const uint32_t e0 = e[4 * hh + 2 * m2], e1 = e[4 * hh + 2 * m2 + 1];
            const uint32_t A = __byte_perm(e0, e1, 0x5410u), B = __byte_perm(e0, e1, 0x7632u);
            const uint32_t Ip = __byte_perm(Iw, 0u, m2 ? 0x4342u : 0x4140u);
            const uint32_t D = A + 0x80FF80FFu - (Ip + Ip + B);
            uint32_t bg = ~D;
            if (c >= 0) bg |= A + B + kc;
            pr[m2] = (bg >> 15) & 0x00010001u;
          }
          mw[hh] = __byte_perm(pr[0], pr[1], 0x6420u);  // bytes: mask of pixels 4hh .. 4hh+3
        }
        if (p.fmt == 0) {
          if (ovec) {
            *reinterpret_cast<uint2*>(obase + j) = make_uint2(mw[0], mw[1]);
          } else {
            for (int z = 0; z < nval; ++z) obase[j + z] = (uint8_t)((z < 4 ? mw[0] : mw[1]) >> (8 * (z & 3)));
          }
        } else {
          // bit z = pixel z, then MSB-first; bits past W are 0
          uint32_t bits = ((mw[0] * 0x01020408u) >> 24 & 0xFu) | ((mw[1] * 0x01020408u) >> 24 & 0xFu) << 4;
          bits &= (1u << nval) - 1u;
          obase[j >> 3] = (uint8_t)(__brev(bits) >> 24);
        }
        // the row entering the prefix (window end of output tt + 1), and the next loads
        min_in(pb, qb[d]);
        if (tt + kVPre < t1) {
          load_pairs(p, hb, ab + h + tt + kVPre, qb[d]);
          qs[d] = s_load(tt + kVPre);
        }
        ib += p.in_pitch;
        obase += p.out_pitch;
      }
    }
  }
}

}  // namespace bern
}  // namespace abin
