// TMA probe 2: does a 3-D byte map (x bytes, rows, pages) accept box x-origins
// that are not multiples of 16 (data landing 128-byte aligned in shared memory)?
// box {256, 2, 1}; checks every byte of both rows against the expected values.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1905_13038_b200/csrc/ptx.cuh"
using namespace abin;
__global__ void k(const __grid_constant__ CUtensorMap tin, int x, int y, unsigned* bad, uint8_t* dump) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) smem[i] = 0xEE;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, 512);
    tma_load_3d(smem, &tin, x, y, 0, bar);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < 512; i += blockDim.x) dump[i] = smem[i];
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  const int H = 16, W = 1000, P = 1024;
  static uint8_t h[H * P];
  for (int r = 0; r < H; ++r) for (int c = 0; c < P; ++c) h[r * P + c] = (uint8_t)((c * 7 + r * 31 + 1) & 0xFF);
  uint8_t* d; cudaMalloc(&d, H * P); cudaMemcpy(d, h, H * P, cudaMemcpyHostToDevice);
  unsigned* bad; cudaMalloc(&bad, 16);
  uint8_t* dump; cudaMalloc(&dump, 512);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  CUtensorMap map;
  cuuint64_t dims[3] = {W, H, 1}, str[2] = {P, (cuuint64_t)P * H};
  cuuint32_t box[3] = {256, 2, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int xs[] = {0, 3, 14, 17, 255, 761, 900, -5, -250};
  for (int xi = 0; xi < 9; ++xi) {
    const int x = xs[xi], y = 3;
    k<<<1, 128, 16384>>>(map, x, y, bad, dump);
    cudaError_t e = cudaDeviceSynchronize();
    uint8_t o[512]; cudaMemcpy(o, dump, 512, cudaMemcpyDeviceToHost);
    int nbad = 0;
    for (int rr = 0; rr < 2; ++rr) for (int c = 0; c < 256; ++c) {
      const int gx = x + c;
      const uint8_t want = (gx >= 0 && gx < W) ? h[(y + rr) * P + gx] : 0;
      if (o[rr * 256 + c] != want) ++nbad;
    }
    printf("x %5d: %s  mismatches %d  first bytes %u %u %u\n", x, cudaGetErrorString(e), nbad, o[0], o[1], o[2]);
    if (e != cudaSuccess) return 1;
  }
}
