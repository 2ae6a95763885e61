#include <cstdio>
#include <cstdint>
__global__ void k() {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0) printf("dyn smem shared addr = 0x%x\n", (unsigned)__cvta_generic_to_shared(smem));
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 32, 100000>>>(); cudaDeviceSynchronize();
  k<<<1, 32, 1000>>>(); printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
