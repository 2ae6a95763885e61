// Standalone TMA bring-up: one CTA loads a 256x8 box (3-D map) into smem.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1905_13038_b200/csrc/ptx.cuh"
using namespace abin;
__global__ void k(const __grid_constant__ CUtensorMap tin, int x, int y, int mode, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode & 1) prefetch_tmap(&tin);
    mbar_arrive_expect_tx(bar, 256 * 8);
    tma_load_3d(smem, &tin, x, y, 0, bar);
  }
  mbar_wait(bar, 0);
  unsigned s = 0;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s += smem[i];
  atomicAdd(out, s);
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int mode = atoi(argv[1]), x = atoi(argv[2]), y = atoi(argv[3]);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  int H = 512, W = 512;
  uint8_t* d; cudaMalloc(&d, H * W); cudaMemset(d, 1, H * W);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t strides[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
  cuuint32_t box[3] = {256, 8, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, (mode & 2) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (query %d)\n", (int)r, (int)q);
  unsigned* out; cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<1, 128, 16384>>>(map, x, y, mode, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h = 0; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("mode %d x %d y %d -> %s sum %u\n", mode, x, y, cudaGetErrorString(e), h);
}
