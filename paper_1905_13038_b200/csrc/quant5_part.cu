// quant5_part.cu -- template instantiations of the v5 quantile kernel
// (quantile5.cuh), split by w mod 16 over four translation units compiled in
// parallel (build.py); ABIN_Q5_PART = 0..3 covers WR = 4 PART .. 4 PART + 3.
#include <cuda_runtime.h>

#include "launch.cuh"
#include "quantile5.cuh"

#define ABIN_CAT2(a, b) a##b
#define ABIN_CAT(a, b) ABIN_CAT2(a, b)

#ifndef ABIN_Q5_PART
#define ABIN_Q5_PART 0
#endif

namespace abin {
namespace {

template <int WR, int NW>
cudaError_t launch_q5_m(const q5::Q5Params& p, int64_t n_tiles, cudaStream_t st, int* occ) {
  constexpr size_t smem = q5::smem_bytes(NW);
  auto kern = q5::k_quant5<WR, NW>;
  static bool attr_set[64] = {};
  cudaError_t e = set_smem_attr_once(kern, smem, attr_set);
  if (e != cudaSuccess) return e;
  if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, 32, smem);
  if (n_tiles > 0) kern<<<(unsigned)n_tiles, 32, smem, st>>>(p);
  return cudaGetLastError();
}

template <int WR>
cudaError_t launch_q5_w(const q5::Q5Params& p, int64_t n, cudaStream_t st, int* occ) {
  if (p.nw == 1) return launch_q5_m<WR, 1>(p, n, st, occ);
  if (p.nw == 2) return launch_q5_m<WR, 2>(p, n, st, occ);
  return launch_q5_m<WR, 3>(p, n, st, occ);
}
}  // namespace

// occ != nullptr: report the resident CTAs per SM instead of launching
cudaError_t ABIN_CAT(launch_q5_part, ABIN_Q5_PART)(int wr, const q5::Q5Params& p, int64_t n, cudaStream_t st,
                                                   int* occ) {
  constexpr int b = 4 * ABIN_Q5_PART;
  switch (wr - b) {
    case 0: return launch_q5_w<b + 0>(p, n, st, occ);
    case 1: return launch_q5_w<b + 1>(p, n, st, occ);
    case 2: return launch_q5_w<b + 2>(p, n, st, occ);
    case 3: return launch_q5_w<b + 3>(p, n, st, occ);
  }
  return cudaErrorInvalidValue;
}

}  // namespace abin
