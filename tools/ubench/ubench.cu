// Instruction-throughput microbenchmark for sm_100a (B200).
// Measures thread-ops per clock per SM for the integer / fp / conversion / MUFU
// instructions the binarization kernels are built from. Single wave, clock64-timed.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NACC 8
#define ITERS 4096

template <int OP>
__device__ __forceinline__ void step(uint32_t (&a)[NACC], float (&f)[NACC], double (&dd)[NACC], uint32_t k1, uint32_t k2) {
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    if (OP == 0) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k1));
    if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(k1), "r"(k2));
    if (OP == 2) asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(a[i]) : "r"(k1));
    if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k1), "r"(k2));
    if (OP == 4) asm volatile("dp4a.u32.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(k1));
    if (OP == 5) asm volatile("dp2a.lo.u32.u32 %0, %0, %1, %0;" : "+r"(a[i]) : "r"(k1));
    if (OP == 6) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(__uint_as_float(k1)), "f"(__uint_as_float(k2)));
    if (OP == 7) { float2 x = make_float2(f[i], f[(i+1)%NACC]); x = __ffma2_rn(x, make_float2(__uint_as_float(k1),__uint_as_float(k1)), make_float2(__uint_as_float(k2),__uint_as_float(k2))); f[i]=x.x; f[(i+1)%NACC]=x.y; }
    if (OP == 8) { uint32_t t; asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f[i]) : "r"(a[i])); asm volatile("mov.b32 %0, %1;" : "=r"(t) : "f"(f[i])); a[i]=t; }
    if (OP == 9) { asm volatile("sqrt.approx.f32 %0, %0;" : "+f"(f[i])); }
    if (OP == 10) { asm volatile("rsqrt.approx.f32 %0, %0;" : "+f"(f[i])); }
    if (OP == 11) { asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dd[i]) : "d"(0.999), "d"(1e-3)); }
    if (OP == 12) { asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(a[i]) : "r"(k1)); }
    if (OP == 13) { asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[i]) : "d"(dd[i])); asm volatile("cvt.f64.f32 %0, %1;" : "=d"(dd[i]) : "f"(f[i])); }
    if (OP == 14) { // IADD3 + FFMA interleaved
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k1));
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(__uint_as_float(k1)), "f"(__uint_as_float(k2)));
    }
    if (OP == 15) { // IADD3 + IMAD interleaved
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k1));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[(i+4)%NACC]) : "r"(k1), "r"(k2));
    }
    if (OP == 16) { // PRMT + IDP2A
      asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(a[i]) : "r"(k1));
      asm volatile("dp2a.lo.u32.u32 %0, %0, %1, %0;" : "+r"(a[(i+4)%NACC]) : "r"(k1));
    }
    if (OP == 17) { uint64_t w; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(a[i]), "r"(k1)); a[i] = (uint32_t)(w ^ (w >> 32)); }
    if (OP == 18) { uint64_t w = ((uint64_t)a[i] << 20) | k1; asm volatile("cvt.rn.f32.u64 %0, %1;" : "=f"(f[i]) : "l"(w)); a[i] = __float_as_uint(f[i]); }
    if (OP == 19) { asm volatile("min.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k1)); }
    if (OP == 20) { asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A800000;" : "+f"(f[i])); }
    if (OP == 21) { asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f[i]) : "r"(a[i])); a[i] = __float_as_uint(f[i]) ^ k1; }
    if (OP == 22) { // MUFU + FFMA interleaved
      asm volatile("sqrt.approx.f32 %0, %0;" : "+f"(f[i]));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k1));
    }
    if (OP == 23) { asm volatile("add.u32 %0, %0, 1;" : "+r"(a[i])); }
    if (OP == 24) { f[i] = (float)((a[i] >> 8) & 0xffu); a[i] += __float_as_uint(f[i]); }   // I2F.U8 .B1 (+iadd)
    if (OP == 25) { float2 x = make_float2(f[i], __uint_as_float(a[i])); x = __ffma2_rn(x, make_float2(__uint_as_float(k1), __uint_as_float(k2)), make_float2(__uint_as_float(k2), __uint_as_float(k1))); f[i] = x.x; a[i] = __float_as_uint(x.y); }  // FFMA2, NACC independent pairs
    if (OP == 26) { asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(__uint_as_float(k1)), "f"(__uint_as_float(k2))); }  // FMNMX3
    if (OP == 27) { asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f[i]) : "r"(a[i])); a[i] += __float_as_uint(f[i]); }  // I2FP.U32 (+iadd)
    if (OP == 28) { // FFMA2 + IADD3 interleaved
      float2 x = make_float2(f[i], __uint_as_float(a[(i+4)%NACC])); x = __ffma2_rn(x, make_float2(__uint_as_float(k1), __uint_as_float(k2)), make_float2(__uint_as_float(k2), __uint_as_float(k1))); f[i] = x.x; a[(i+4)%NACC] = __float_as_uint(x.y);
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k1));
    }
    if (OP == 29) { // FFMA2 + PRMT interleaved
      float2 x = make_float2(f[i], __uint_as_float(a[(i+4)%NACC])); x = __ffma2_rn(x, make_float2(__uint_as_float(k1), __uint_as_float(k2)), make_float2(__uint_as_float(k2), __uint_as_float(k1))); f[i] = x.x; a[(i+4)%NACC] = __float_as_uint(x.y);
      asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(a[i]) : "r"(k1));
    }
    if (OP == 30) { // PRMT + IADD3 interleaved
      asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(a[i]) : "r"(k1));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a[(i+4)%NACC]) : "r"(k2));
    }
  }
}

template <int OP>
__global__ void __launch_bounds__(256) kbench(uint32_t* out, long long* cyc, uint32_t k1, uint32_t k2) {
  uint32_t a[NACC]; float f[NACC]; double dd[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { a[i] = threadIdx.x * 7 + i; f[i] = 1.0f + i * 0.1f; dd[i] = 1.0 + i; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) step<OP>(a, f, dd, k1, k2);
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i] + __float_as_uint(f[i]) + (uint32_t)__double_as_longlong(dd[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int ops_per_step, int nsm, int blocks_per_sm) {
  int grid = nsm * blocks_per_sm;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, grid * 256 * 4); cudaMalloc(&cyc, grid * 8);
  kbench<OP><<<grid, 256>>>(out, cyc, 0x01020304u, 0x3f800001u);
  kbench<OP><<<grid, 256>>>(out, cyc, 0x01020304u, 0x3f800001u);
  cudaDeviceSynchronize();
  long long* h = new long long[grid];
  cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  double ops = (double)blocks_per_sm * 256 * ITERS * NACC * ops_per_step;
  printf("%-28s %8.1f thread-ops/clk/SM  (cycles %.0f)\n", name, ops / mx, mx);
  delete[] h; cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int nsm = p.multiProcessorCount;
  printf("device %s SMs %d clock %d kHz l2 %d\n", p.name, nsm, p.clockRate, p.l2CacheSize);
  int b = 4;
  run<0>("IADD3", 1, nsm, b);
  run<23>("IADD imm", 1, nsm, b);
  run<1>("LOP3", 1, nsm, b);
  run<2>("PRMT", 1, nsm, b);
  run<19>("IMNMX", 1, nsm, b);
  run<3>("IMAD", 1, nsm, b);
  run<4>("IDP.4A", 1, nsm, b);
  run<5>("IDP.2A", 1, nsm, b);
  run<6>("FFMA", 1, nsm, b);
  run<20>("FFMA imm", 1, nsm, b);
  run<7>("FFMA2 (2 flops-lanes)", 2, nsm, b);
  run<8>("I2F.U32 (+mov)", 1, nsm, b);
  run<21>("I2F.S32 (+lop)", 1, nsm, b);
  run<18>("I2F.U64 (+shift)", 1, nsm, b);
  run<13>("F2F f64->f32->f64 (2 cvt)", 2, nsm, b);
  run<9>("MUFU.SQRT", 1, nsm, b);
  run<10>("MUFU.RSQ", 1, nsm, b);
  run<11>("DFMA", 1, nsm, b);
  run<12>("SHFL", 1, nsm, b);
  run<17>("IMAD.WIDE (+lop)", 1, nsm, b);
  run<14>("IADD3+FFMA pair (ops)", 2, nsm, b);
  run<15>("IADD3+IMAD pair (ops)", 2, nsm, b);
  run<16>("PRMT+IDP.2A pair (ops)", 2, nsm, b);
  run<22>("MUFU.SQRT+IADD pair (ops)", 2, nsm, b);
  run<24>("I2F.U8.B1 + IADD (pair)", 2, nsm, b);
  run<25>("FFMA2 (instr)", 1, nsm, b);
  run<26>("FMNMX3", 1, nsm, b);
  run<27>("I2FP.U32 + IADD (pair)", 2, nsm, b);
  run<28>("FFMA2+IADD3 pair (instr)", 2, nsm, b);
  run<29>("FFMA2+PRMT pair (instr)", 2, nsm, b);
  run<30>("PRMT+IADD3 pair (instr)", 2, nsm, b);
  return 0;
}
