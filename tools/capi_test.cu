// Calls libabin.so's abin_sauvola from a plain host program (no torch).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../include/abin.h"
int main(int argc, char** argv) {
  int H = atoi(argv[1]), W = atoi(argv[2]), h = atoi(argv[3]), w = atoi(argv[4]);
  uint8_t *d, *o;
  cudaMalloc(&d, (size_t)H * W); cudaMalloc(&o, (size_t)H * W);
  uint8_t* hbuf = (uint8_t*)malloc((size_t)H * W);
  for (long i = 0; i < (long)H * W; ++i) hbuf[i] = (uint8_t)((i * 2654435761u) >> 24);
  cudaMemcpy(d, hbuf, (size_t)H * W, cudaMemcpyHostToDevice);
  int rc = abin_sauvola(d, H, W, W, o, W, 0, h, w, 0.5, 128.0, 0, nullptr, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  printf("rc %d sync %s\n", rc, cudaGetErrorString(e));
  return 0;
}
