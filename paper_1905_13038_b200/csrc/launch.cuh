// launch.cuh -- launchers of the moments kernels, split over several
// translation units (moments_part.cu, wide_part.cu) so the 100+ template
// instantiations compile in parallel.  Each returns a cudaError_t.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "moments.cuh"
#include "moments_wide.cuh"
#include "moments4.cuh"
#include "moments5.cuh"
#include "quantile5.cuh"

namespace abin {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, carveout) once per device
// and kernel (the attributes are per-device state; `done` is the caller's
// per-kernel static table).  Benign race: the values set are idempotent.
template <typename K>
inline cudaError_t set_smem_attr_once(K kern, size_t smem, bool (&done)[64]) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}
// warp-strip kernel, w mod 32 = w32 (moments.cuh)
cudaError_t launch_fast(int w32, bool d64, const CUtensorMap& map, const MomParams& p, int64_t n_tiles,
                        cudaStream_t st);
// CTA-strip kernel for wide windows (moments_wide.cuh)
cudaError_t launch_wide(bool d64, bool stats, int nt, int ph, const CUtensorMap& map, const wide::MomParams& p,
                        int64_t n_tiles, cudaStream_t st);
// per-part entry points (defined by moments_part.cu compiled with -DABIN_PART=k)
#define ABIN_N_PARTS 8
#define ABIN_DECL_PART(k)                                                                                 \
  cudaError_t launch_fast_part##k(int w32, bool d64, const CUtensorMap& map, const MomParams& p, int64_t n, \
                                  cudaStream_t st);                                                         \
  cudaError_t launch_v4_part##k(int w32, bool d64, const CUtensorMap& map, const MomParams& p, int64_t n,   \
                                cudaStream_t st);                                                           \
  cudaError_t launch_v5_part##k(int w32, const CUtensorMap& map, const CUtensorMap& mpk, const MomParams& p,       \
                                int64_t n, cudaStream_t st);                                                      \
  int occupancy_v5_part##k(int w32, int method);
ABIN_DECL_PART(0) ABIN_DECL_PART(1) ABIN_DECL_PART(2) ABIN_DECL_PART(3)
ABIN_DECL_PART(4) ABIN_DECL_PART(5) ABIN_DECL_PART(6) ABIN_DECL_PART(7)
// v5 quantile kernel (quantile5.cuh), split by w mod 16 (quant5_part.cu); occ != nullptr: occupancy query
cudaError_t launch_q5_part0(int wr, const q5::Q5Params& p, int64_t n, cudaStream_t st, int* occ);
cudaError_t launch_q5_part1(int wr, const q5::Q5Params& p, int64_t n, cudaStream_t st, int* occ);
cudaError_t launch_q5_part2(int wr, const q5::Q5Params& p, int64_t n, cudaStream_t st, int* occ);
cudaError_t launch_q5_part3(int wr, const q5::Q5Params& p, int64_t n, cudaStream_t st, int* occ);
cudaError_t launch_wide_d64(bool d64, bool stats, int nt, int ph, const CUtensorMap& map, const wide::MomParams& p,
                            int64_t n_tiles, cudaStream_t st);
cudaError_t launch_wide_d32(bool d64, bool stats, int nt, int ph, const CUtensorMap& map, const wide::MomParams& p,
                            int64_t n_tiles, cudaStream_t st);
}  // namespace abin
