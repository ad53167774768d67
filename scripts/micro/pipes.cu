// Microbenchmark: which pipe executes VIADD.16x2 / IMAD / LOP3 / ISETP on sm_100a, and at
// what rate. Each kernel runs a long dependent-free stream of one instruction type.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_viadd2(unsigned* out, unsigned seed, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  const unsigned nb = __vneg2(seed);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __vadd2(a[i], nb);
  }
  unsigned r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_imad(unsigned* out, unsigned seed, int iters) {
  int a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  int m1 = (int)seed | 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m1), "r"(i));
  }
  int r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_lop3(unsigned* out, unsigned seed, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(a[(i + 1) & 7]), "r"(seed));
  }
  unsigned r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_mix(unsigned* out, unsigned seed, int iters) {  // 2 VIADD.16x2 : 1 LOP3 (the planned fast loop)
  unsigned a[8], acc = 0xffffffffu;
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  unsigned nb = __vneg2(seed);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) acc &= __vadd2(a[i], nb) & __vadd2(a[i + 1], nb);
    nb += 0x00010001u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_iadd(unsigned* out, unsigned seed, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i + 3) & 7]));
  }
  unsigned r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_iadd3(unsigned* out, unsigned seed, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { unsigned t; asm volatile("add.u32 %1, %0, %2;\n\tadd.u32 %0, %1, %3;" : "+r"(a[i]), "=r"(t) : "r"(a[(i + 3) & 7]), "r"(seed)); }
  }
  unsigned r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
// balanced: per 8 pairs -> 5 IMAD (fma) + 3 IADD (alu) + 4 LOP3 (alu, 2-pair OR accumulate)
__global__ void k_bal(unsigned* out, unsigned seed, int iters) {
  unsigned a[8], acc0 = 0, acc1 = 0;
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i + 1);
  unsigned nb = seed & 0x7fff7fffu; const unsigned one = seed >> 31 | 1u;
  for (int it = 0; it < iters; ++it) {
    unsigned s[8];
#pragma unroll
    for (int i = 0; i < 5; ++i) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s[i]) : "r"(a[i]), "r"(one), "r"(nb));
#pragma unroll
    for (int i = 5; i < 8; ++i) asm volatile("add.u32 %0, %1, %2;" : "=r"(s[i]) : "r"(a[i]), "r"(nb));
    acc0 |= s[0] | s[1]; acc1 |= s[2] | s[3]; acc0 |= s[4] | s[5]; acc1 |= s[6] | s[7];
    nb += 0x00010001u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1;
}
int main() {
  unsigned* d;
  cudaMalloc(&d, 148 * 1024 * 4 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  auto run = [&](const char* name, void (*k)(unsigned*, unsigned, int), double ops_per_iter) {
    k<<<148 * 8, 256>>>(d, 7, 10);
    cudaEventRecord(e0);
    k<<<148 * 8, 256>>>(d, 7, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = 148.0 * 8 * 8 * iters * ops_per_iter;
    printf("%-8s %8.3f ms  %.3f warp-instr/clk/SM (at 1965 MHz)\n", name, ms,
           warp_instr / (ms * 1e-3) / 148 / 1.965e9);
  };
  run("viadd2", k_viadd2, 8);
  run("imad", k_imad, 8);
  run("lop3", k_lop3, 8);
  run("mix", k_mix, 8 + 4 + 1);
  run("iadd", k_iadd, 8);
  run("iadd3", k_iadd3, 8);
  run("bal", k_bal, 8 + 4 + 1);
  return 0;
}
