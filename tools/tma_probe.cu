// TMA probe: which shared-memory destination alignments and box shapes work on sm_100a.
//  mode 0: 3-D map (x bytes, rows, pages), box {176,1,1}, smem dst offset `off`
//  mode 1: 4-D map (16-byte chunks: {16, W/16, rows, pages}), box {16,33,1,1}, chunk start x, dst offset `off`
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1905_13038_b200/csrc/ptx.cuh"
using namespace abin;
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x0, int x1, int x2, int x3, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(smem_u32(bar)) : "memory");
}
__global__ void k(const __grid_constant__ CUtensorMap tin, int mode, int x, int off, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) smem[i] = 0;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    if (mode == 0) { mbar_arrive_expect_tx(bar, 176); tma_load_3d(smem + off, &tin, x, 3, 0, bar); }
    else { mbar_arrive_expect_tx(bar, 528); tma_load_4d(smem + off, &tin, 0, x, 3, 0, bar); }
  }
  mbar_wait(bar, 0);
  if (threadIdx.x == 0) { out[0] = smem[off]; out[1] = smem[off + 1]; out[2] = smem[off + 175]; out[3] = smem[off + 527]; }
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  const int H = 16, W = 1000, P = 1024;  // pitch 1024
  uint8_t h[H * P]; for (int i = 0; i < H * P; ++i) h[i] = (uint8_t)((i % P) & 0xFF);
  uint8_t* d; cudaMalloc(&d, H * P); cudaMemcpy(d, h, H * P, cudaMemcpyHostToDevice);
  unsigned* out; cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (int mode = 1; mode < 2; ++mode) {
    CUtensorMap map; CUresult r;
    if (mode == 0) {
      cuuint64_t dims[3] = {W, H, 1}, str[2] = {P, (cuuint64_t)P * H};
      cuuint32_t box[3] = {176, 1, 1}, es[3] = {1, 1, 1};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[4] = {16, (W + 15) / 16, H, 1}, str[3] = {16, P, (cuuint64_t)P * H};
      cuuint32_t box[4] = {16, 33, 1, 1}, es[4] = {1, 1, 1, 1};
      r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("mode %d encode %d\n", mode, (int)r);
    int offs[] = {0, 128, 256, 640, 1280, 1408, 768};
    int xs[] = {0, 3, 48, 60, -5};
    for (int oi = 0; oi < 7; ++oi) for (int xi = 0; xi < 5; ++xi) {
      int x = mode == 0 ? xs[xi] * 16 : xs[xi];
      cudaMemset(out, 0xFF, 16);
      k<<<1, 128, 16384>>>(map, mode, x, offs[oi], out);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned o[4] = {0}; cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
      printf("mode %d off %4d x %5d: %s  %u %u %u %u\n", mode, offs[oi], x, cudaGetErrorString(e), o[0], o[1], o[2], o[3]);
      if (e != cudaSuccess) { cudaDeviceReset(); return 1; }
    }
  }
}
