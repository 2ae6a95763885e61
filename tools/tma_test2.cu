#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1905_13038_b200/csrc/ptx.cuh"
using namespace abin;
struct P { int64_t a[40]; };
__global__ void k(const __grid_constant__ CUtensorMap tin, const P p, int mode, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 92224);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nb = mode & 3; if (nb == 0) nb = 3;
    mbar_arrive_expect_tx(bar, nb * 2048);
    for (int b = 0; b < nb; ++b) tma_load_3d(smem + b * 2048, &tin, -24 + 256 * b, (mode & 4) ? 0 : -16, 0, bar);
  }
  mbar_wait(bar, 0);
  unsigned s = 0;
  for (int i = threadIdx.x; i < 6144; i += blockDim.x) s += smem[i];
  atomicAdd(out, s + (unsigned)p.a[0]);
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  int H = 512, W = 512;
  uint8_t* d; cudaMalloc(&d, H * W); cudaMemset(d, 1, H * W);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t strides[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
  cuuint32_t box[3] = {256, 8, 1}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned* out; cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 92248);
  P p = {};
  k<<<1, 128, 92248>>>(map, p, mode, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h = 0; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("mode %d -> %s sum %u\n", mode, cudaGetErrorString(e), h);
}
