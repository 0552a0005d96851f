// Integer-pipe microbenchmarks (tuning aid): Comba mac3, operand scanning,
// radix-2^28 64-bit column sums, IMAD.HI, IMAD, IADD+LOP3 throughput.
// CAUTION: variant B's carry chains are separate NON-volatile asm statements,
// which the compiler may reorder across the implicit carry flag - its 36
// MACs/clk/SM is not a valid multi-limb product rate (mpsp_imad_bench keeps
// the chains in order with asm volatile: 5.65 T vs Comba's 8.1 T limb-MAC/s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/imad_mb tools/imad_mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int L = 8;
// variant A: current Comba mac3 (product scanning)
__device__ __forceinline__ void mac3(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t a, uint32_t b) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
      : "+r"(c0), "+r"(c1), "+r"(c2) : "r"(a), "r"(b));
}
__global__ void kA(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[L], b[L];
  for (int i = 0; i < L; ++i) { a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u; b[i] = (seed ^ blockIdx.x) * 0x85EBCA6Bu + i * threadIdx.x; }
  for (int it = 0; it < iters; ++it) {
    uint32_t c0 = 0, c1 = 0, c2 = 0, r[L];
#pragma unroll
    for (int k = 0; k < 2 * L - 1; ++k) {
#pragma unroll
      for (int i = 0; i < L; ++i) { int j = k - i; if (j < 0 || j >= L) continue; mac3(c0, c1, c2, a[i], b[j]); }
      if (k >= L - 1) r[k - (L - 1)] = c0;
      c0 = c1; c1 = c2; c2 = 0;
    }
#pragma unroll
    for (int i = 0; i < L; ++i) a[i] ^= r[i];
  }
  uint32_t acc = 0; for (int i = 0; i < L; ++i) acc ^= a[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
// variant M<R>: Comba where every R-th MAC of a column is a split multiply
// (mul.lo + mul.hi on the FMA pipes, three carry adds on the ALU pipe)
__device__ __forceinline__ void mac3s(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t a, uint32_t b) {
  uint32_t lo = a * b, hi = __umulhi(a, b);
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
      : "+r"(c0), "+r"(c1), "+r"(c2) : "r"(lo), "r"(hi));
}
template <int R>
__global__ void kM(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[L], b[L];
  for (int i = 0; i < L; ++i) { a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u; b[i] = (seed ^ blockIdx.x) * 0x85EBCA6Bu + i * threadIdx.x; }
  for (int it = 0; it < iters; ++it) {
    uint32_t c0 = 0, c1 = 0, c2 = 0, r[L];
    int q = 0;
#pragma unroll
    for (int k = 0; k < 2 * L - 1; ++k) {
#pragma unroll
      for (int i = 0; i < L; ++i) {
        int j = k - i; if (j < 0 || j >= L) continue;
        if ((q++ % R) == R - 1) mac3s(c0, c1, c2, a[i], b[j]); else mac3(c0, c1, c2, a[i], b[j]);
      }
      if (k >= L - 1) r[k - (L - 1)] = c0;
      c0 = c1; c1 = c2; c2 = 0;
    }
#pragma unroll
    for (int i = 0; i < L; ++i) a[i] ^= r[i];
  }
  uint32_t acc = 0; for (int i = 0; i < L; ++i) acc ^= a[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
// variant B: operand scanning, lo chain then hi chain per a_i
__global__ void kB(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[L], b[L];
  for (int i = 0; i < L; ++i) { a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u; b[i] = (seed ^ blockIdx.x) * 0x85EBCA6Bu + i * threadIdx.x; }
  for (int it = 0; it < iters; ++it) {
    uint32_t r[2 * L];
#pragma unroll
    for (int i = 0; i < 2 * L; ++i) r[i] = 0;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      asm("mad.lo.cc.u32 %0, %1, %2, %0;" : "+r"(r[i]) : "r"(a[i]), "r"(b[0]));
#pragma unroll
      for (int j = 1; j < L; ++j) asm("madc.lo.cc.u32 %0, %1, %2, %0;" : "+r"(r[i + j]) : "r"(a[i]), "r"(b[j]));
      asm("addc.u32 %0, %0, 0;" : "+r"(r[i + L]));
      asm("mad.hi.cc.u32 %0, %1, %2, %0;" : "+r"(r[i + 1]) : "r"(a[i]), "r"(b[0]));
#pragma unroll
      for (int j = 1; j < L; ++j) asm("madc.hi.cc.u32 %0, %1, %2, %0;" : "+r"(r[i + j + 1]) : "r"(a[i]), "r"(b[j]));
      if (i + L + 1 < 2 * L) asm("addc.u32 %0, %0, 0;" : "+r"(r[i + L + 1]));
    }
#pragma unroll
    for (int i = 0; i < L; ++i) a[i] ^= r[i + L];
  }
  uint32_t acc = 0; for (int i = 0; i < L; ++i) acc ^= a[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
// variant C: radix 2^28 limbs, 64-bit column accumulators, mad.wide.u32 (no carries)
__global__ void kC(uint32_t* out, int iters, uint32_t seed) {
  constexpr int M = 10;   // 280 bits
  uint32_t a[M], b[M];
  for (int i = 0; i < M; ++i) { a[i] = (seed * (threadIdx.x + 1) + i * 0x9E3779B9u) & 0xFFFFFFF; b[i] = ((seed ^ blockIdx.x) * 0x85EBCA6Bu + i * threadIdx.x) & 0xFFFFFFF; }
  for (int it = 0; it < iters; ++it) {
    uint32_t r[M] = {0};
    uint64_t cy = 0;
#pragma unroll
    for (int k = 0; k < 2 * M - 1; ++k) {
      uint64_t c = cy;
#pragma unroll
      for (int i = 0; i < M; ++i) { int j = k - i; if (j < 0 || j >= M) continue; c += (uint64_t)a[i] * b[j]; }
      if (k >= M - 1) r[k - (M - 1)] = (uint32_t)c & 0xFFFFFFF;
      cy = c >> 28;
    }
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] ^= r[i];
  }
  uint32_t acc = 0; for (int i = 0; i < M; ++i) acc ^= a[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
// variant D: IMAD.HI only, and IMAD lo only throughput
__global__ void kD(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[L], b[L], r[L];
  for (int i = 0; i < L; ++i) { a[i] = seed * (threadIdx.x + 1) + i; b[i] = seed ^ (i * threadIdx.x); r[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
      for (int j = 0; j < L; ++j) r[j] = __umulhi(a[i] ^ r[j], b[j]) ;
  }
  uint32_t acc = 0; for (int i = 0; i < L; ++i) acc ^= r[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
__global__ void kE(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[L], b[L], r[L];
  for (int i = 0; i < L; ++i) { a[i] = seed * (threadIdx.x + 1) + i; b[i] = seed ^ (i * threadIdx.x); r[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
      for (int j = 0; j < L; ++j) r[j] = a[i] * r[j] + b[j];
  }
  uint32_t acc = 0; for (int i = 0; i < L; ++i) acc ^= r[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
// IADD3 throughput
__global__ void kF(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[L], b[L], r[L];
  for (int i = 0; i < L; ++i) { a[i] = seed * (threadIdx.x + 1) + i; b[i] = seed ^ (i * threadIdx.x); r[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
      for (int j = 0; j < L; ++j) r[j] = (r[j] + a[i]) ^ b[j];
  }
  uint32_t acc = 0; for (int i = 0; i < L; ++i) acc ^= r[i];
  if (acc == seed + 0x12345678u) out[blockIdx.x] = acc;
}
template <typename K>
double run(K k, const char* name, double ops_per_iter, int iters, int threads, int bps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d; cudaMalloc(&d, 1 << 20);
  int blocks = sms * bps;
  k<<<blocks, threads>>>(d, 8, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<blocks, threads>>>(d, iters, 7); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * ops_per_iter;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s: %.3f ms  %.2f Tops/s  %.2f ops/clk/SM (at 1965MHz) err=%s\n", name, ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  return ms;
}
int main() {
  for (int bps : {4, 8}) {
    printf("blocks/SM %d x 256\n", bps);
    run(kA, "A comba mac3 (MACs)", 64, 4096, 256, bps);
    run(kB, "B operand-scan lo/hi (MACs)", 64, 4096, 256, bps);
    run(kC, "C radix28 wide (MACs)", 100, 4096, 256, bps);
    run(kM<1>, "M1 all split (MACs)", 64, 4096, 256, bps);
    run(kM<2>, "M2 1/2 split (MACs)", 64, 4096, 256, bps);
    run(kM<3>, "M3 1/3 split (MACs)", 64, 4096, 256, bps);
    run(kM<4>, "M4 1/4 split (MACs)", 64, 4096, 256, bps);
    run(kD, "D umulhi", 64, 4096, 256, bps);
    run(kE, "E imad lo", 64, 4096, 256, bps);
    run(kF, "F iadd+xor (2 ops)", 128, 4096, 256, bps);
  }
}
