// moments_part.cu -- instantiations of the warp-strip moments kernel for
// w mod 32 in [4 ABIN_PART, 4 ABIN_PART + 4), both square-sum widths.
// Compiled ABIN_N_PARTS times (build.py) with -DABIN_PART=0..7.
#include "launch.cuh"

#ifndef ABIN_PART
#error "compile with -DABIN_PART=k"
#endif
#define ABIN_CAT2(a, b) a##b
#define ABIN_CAT(a, b) ABIN_CAT2(a, b)

namespace abin {
namespace {
template <int W32, bool D64>
cudaError_t launch_one(const CUtensorMap& map, const MomParams& p, int64_t n_tiles, cudaStream_t st) {
  constexpr size_t smem = moments_smem_bytes();
  auto kern = k_moments<W32, D64>;
  static bool attr_set[64] = {};
  const cudaError_t e = set_smem_attr_once(kern, smem, attr_set);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)n_tiles, kNT, smem, st>>>(map, p);
  return cudaGetLastError();
}
template <int W32, bool D64, int METHOD>
cudaError_t launch_v4_m(const CUtensorMap& map, const MomParams& p, int64_t n_tiles, cudaStream_t st) {
  constexpr size_t smem = v4::smem_bytes();
  auto kern = v4::k_mom4<W32, D64, METHOD>;
  static bool attr_set[64] = {};
  const cudaError_t e = set_smem_attr_once(kern, smem, attr_set);
  if (e != cudaSuccess) return e;
  if (n_tiles > 0) kern<<<(unsigned)n_tiles, 32, smem, st>>>(map, p);
  return cudaGetLastError();
}

template <int W32, int METHOD>
cudaError_t launch_v5_m(const CUtensorMap& map, const CUtensorMap& mpk, const MomParams& p, int64_t n_tiles,
                        cudaStream_t st) {
  constexpr size_t smem = v5::smem_bytes();
  auto kern = v5::k_mom5<W32, METHOD>;
  static bool attr_set[64] = {};
  const cudaError_t e = set_smem_attr_once(kern, smem, attr_set);
  if (e != cudaSuccess) return e;
  if (n_tiles > 0) kern<<<(unsigned)n_tiles, 32, smem, st>>>(map, mpk, p);
  return cudaGetLastError();
}

template <int W32>
int occ_v5(int method) {
  int n = 0;
  constexpr size_t smem = v5::smem_bytes();
  cudaError_t e;
  static bool a0[64] = {}, a1[64] = {}, a2[64] = {}, a3[64] = {}, a4[64] = {};
  if (method == M_KHURSHID) {
    e = set_smem_attr_once(v5::k_mom5<W32, M_KHURSHID>, smem, a3);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v5::k_mom5<W32, M_KHURSHID>, 32, smem);
  } else if (method == M_PHANSALKAR) {
    e = set_smem_attr_once(v5::k_mom5<W32, M_PHANSALKAR>, smem, a4);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v5::k_mom5<W32, M_PHANSALKAR>, 32, smem);
  } else if (method == M_SAUVOLA) {
    e = set_smem_attr_once(v5::k_mom5<W32, M_SAUVOLA>, smem, a0);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v5::k_mom5<W32, M_SAUVOLA>, 32, smem);
  } else if (method == M_NIBLACK) {
    e = set_smem_attr_once(v5::k_mom5<W32, M_NIBLACK>, smem, a1);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v5::k_mom5<W32, M_NIBLACK>, 32, smem);
  } else {
    e = set_smem_attr_once(v5::k_mom5<W32, M_WOLF>, smem, a2);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v5::k_mom5<W32, M_WOLF>, 32, smem);
  }
  return e == cudaSuccess && n > 0 ? n : 16;
}

template <int W32>
cudaError_t launch_v5(const CUtensorMap& map, const CUtensorMap& mpk, const MomParams& p, int64_t n_tiles,
                      cudaStream_t st) {
  if (p.method == M_SAUVOLA) return launch_v5_m<W32, M_SAUVOLA>(map, mpk, p, n_tiles, st);
  if (p.method == M_NIBLACK) return launch_v5_m<W32, M_NIBLACK>(map, mpk, p, n_tiles, st);
  if (p.method == M_MAXS) return launch_v5_m<W32, M_MAXS>(map, mpk, p, n_tiles, st);
  if (p.method == M_KHURSHID) return launch_v5_m<W32, M_KHURSHID>(map, mpk, p, n_tiles, st);
  if (p.method == M_PHANSALKAR) return launch_v5_m<W32, M_PHANSALKAR>(map, mpk, p, n_tiles, st);
  if (p.method == M_RAIS) return launch_v5_m<W32, M_RAIS>(map, mpk, p, n_tiles, st);
  if (p.method == M_FENG) return launch_v5_m<W32, M_FENG>(map, mpk, p, n_tiles, st);
  return launch_v5_m<W32, M_WOLF>(map, mpk, p, n_tiles, st);
}

template <int W32, bool D64>
cudaError_t launch_v4(const CUtensorMap& map, const MomParams& p, int64_t n_tiles, cudaStream_t st) {
  if (p.method == M_SAUVOLA) return launch_v4_m<W32, D64, M_SAUVOLA>(map, p, n_tiles, st);
  if (p.method == M_NIBLACK) return launch_v4_m<W32, D64, M_NIBLACK>(map, p, n_tiles, st);
  return launch_v4_m<W32, D64, M_WOLF>(map, p, n_tiles, st);
}
}  // namespace

cudaError_t ABIN_CAT(launch_v4_part, ABIN_PART)(int w32, bool d64, const CUtensorMap& map, const MomParams& p,
                                                int64_t n, cudaStream_t st) {
  constexpr int b = 4 * ABIN_PART;
  switch (w32 - b) {
    case 0: return d64 ? launch_v4<b + 0, true>(map, p, n, st) : launch_v4<b + 0, false>(map, p, n, st);
    case 1: return d64 ? launch_v4<b + 1, true>(map, p, n, st) : launch_v4<b + 1, false>(map, p, n, st);
    case 2: return d64 ? launch_v4<b + 2, true>(map, p, n, st) : launch_v4<b + 2, false>(map, p, n, st);
    case 3: return d64 ? launch_v4<b + 3, true>(map, p, n, st) : launch_v4<b + 3, false>(map, p, n, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t ABIN_CAT(launch_v5_part, ABIN_PART)(int w32, const CUtensorMap& map, const CUtensorMap& mpk,
                                                const MomParams& p, int64_t n, cudaStream_t st) {
  constexpr int b = 4 * ABIN_PART;
  switch (w32 - b) {
    case 0: return launch_v5<b + 0>(map, mpk, p, n, st);
    case 1: return launch_v5<b + 1>(map, mpk, p, n, st);
    case 2: return launch_v5<b + 2>(map, mpk, p, n, st);
    case 3: return launch_v5<b + 3>(map, mpk, p, n, st);
  }
  return cudaErrorInvalidValue;
}

int ABIN_CAT(occupancy_v5_part, ABIN_PART)(int w32, int method) {
  constexpr int b = 4 * ABIN_PART;
  switch (w32 - b) {
    case 0: return occ_v5<b + 0>(method);
    case 1: return occ_v5<b + 1>(method);
    case 2: return occ_v5<b + 2>(method);
    case 3: return occ_v5<b + 3>(method);
  }
  return 16;
}

cudaError_t ABIN_CAT(launch_fast_part, ABIN_PART)(int w32, bool d64, const CUtensorMap& map, const MomParams& p,
                                                  int64_t n, cudaStream_t st) {
  constexpr int b = 4 * ABIN_PART;
  switch (w32 - b) {
    case 0: return d64 ? launch_one<b + 0, true>(map, p, n, st) : launch_one<b + 0, false>(map, p, n, st);
    case 1: return d64 ? launch_one<b + 1, true>(map, p, n, st) : launch_one<b + 1, false>(map, p, n, st);
    case 2: return d64 ? launch_one<b + 2, true>(map, p, n, st) : launch_one<b + 2, false>(map, p, n, st);
    case 3: return d64 ? launch_one<b + 3, true>(map, p, n, st) : launch_one<b + 3, false>(map, p, n, st);
  }
  return cudaErrorInvalidValue;
}
}  // namespace abin
