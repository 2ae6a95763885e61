// wide_part.cu -- instantiations of the CTA-strip (wide-window) moments
// kernel; compiled twice (build.py) with -DABIN_WIDE_D64=0 / 1.
#include "launch.cuh"

#ifndef ABIN_WIDE_D64
#error "compile with -DABIN_WIDE_D64=0|1"
#endif

namespace abin {
namespace {
template <int NT, int PH, bool D64, bool STATS>
cudaError_t launch_one(const CUtensorMap& map, const wide::MomParams& p, int64_t n_tiles, cudaStream_t st) {
  constexpr int R_ = (NT == 128) ? 8 : 4;
  constexpr size_t smem = wide::moments_smem_bytes<NT, 8, R_, D64>();
  auto kern = wide::k_moments<NT, 8, PH, R_, D64, STATS>;
  static bool attr_set[64] = {};  // per device
  const cudaError_t e = set_smem_attr_once(kern, smem, attr_set);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)n_tiles, NT, smem, st>>>(map, p);
  return cudaGetLastError();
}

template <bool STATS>
cudaError_t by_shape(int nt, int ph, const CUtensorMap& map, const wide::MomParams& p, int64_t n, cudaStream_t st) {
  constexpr bool D = ABIN_WIDE_D64 != 0;
#define ABIN_PH(NT_)                                              \
  switch (ph) {                                                   \
    case 0: return launch_one<NT_, 0, D, STATS>(map, p, n, st);   \
    case 1: return launch_one<NT_, 1, D, STATS>(map, p, n, st);   \
    case 2: return launch_one<NT_, 2, D, STATS>(map, p, n, st);   \
    default: return launch_one<NT_, 3, D, STATS>(map, p, n, st);  \
  }
  if (nt == 128) ABIN_PH(128)
  ABIN_PH(256)
#undef ABIN_PH
}
}  // namespace

#if ABIN_WIDE_D64
cudaError_t launch_wide_d64(bool, bool stats, int nt, int ph, const CUtensorMap& map, const wide::MomParams& p,
                            int64_t n, cudaStream_t st) {
#else
cudaError_t launch_wide_d32(bool, bool stats, int nt, int ph, const CUtensorMap& map, const wide::MomParams& p,
                            int64_t n, cudaStream_t st) {
#endif
  return stats ? by_shape<true>(nt, ph, map, p, n, st) : by_shape<false>(nt, ph, map, p, n, st);
}
}  // namespace abin
