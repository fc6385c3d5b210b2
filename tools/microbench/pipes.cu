// Throughput probe for the integer instructions the LUT lookup path uses
// (PRMT, IDP.2A, IDP.4A, LOP3, IADD3). Prints ops/clk/SM for each.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c){ uint32_t d; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;}
__device__ __forceinline__ int dp2a_lo(int a, int b, int c){ int d; asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;}
__device__ __forceinline__ int dp4a(int a, int b, int c){ int d; asm volatile("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;}
__device__ __forceinline__ uint32_t lop(uint32_t a, uint32_t b){ uint32_t d; asm volatile("xor.b32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;}
__device__ __forceinline__ uint32_t iadd(uint32_t a, uint32_t b){ uint32_t d; asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;}

constexpr int ITERS = 4096;
constexpr int NACC = 16;

template <int OP>
__global__ void probe(uint32_t seed, uint32_t* out) {
  uint32_t a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) a[i] = seed * (i + 1) + threadIdx.x;
  uint32_t t0 = seed ^ 0x1234567u, t1 = seed + 77u;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      if (OP == 0) a[i] = prmt(t0, t1, a[i]);
      if (OP == 1) a[i] = dp2a_lo(0x80000001, t0, a[i]);
      if (OP == 2) a[i] = dp4a(0x01010101, t0, a[i]);
      if (OP == 3) a[i] = lop(a[i], t0);
      if (OP == 4) a[i] = iadd(a[i], t1);
      if (OP == 5) { a[i] = dp2a_lo(0x80000001, t0, a[i]); }
    }
    if (OP == 5) {
#pragma unroll
      for (int i = 0; i < NACC; i++) t0 = prmt(t0, t1, a[i]);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= a[i];
  if (s == 0xdeadbeef) out[0] = s + t0;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t* out; cudaMalloc(&out, 4);
  const char* names[] = {"PRMT", "IDP.2A", "IDP.4A", "LOP3(xor)", "IADD3", "IDP.2A+PRMT(1:1)"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int op = 0; op < 6; op++) {
    for (int rep = 0; rep < 2; rep++) {
      int blocks = sms * 4, threads = 512;
      cudaEventRecord(e0);
      switch (op) {
        case 0: probe<0><<<blocks, threads>>>(1, out); break;
        case 1: probe<1><<<blocks, threads>>>(1, out); break;
        case 2: probe<2><<<blocks, threads>>>(1, out); break;
        case 3: probe<3><<<blocks, threads>>>(1, out); break;
        case 4: probe<4><<<blocks, threads>>>(1, out); break;
        case 5: probe<5><<<blocks, threads>>>(1, out); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * ITERS * NACC * (op == 5 ? 2 : 1);
      double per_s = ops / (ms * 1e-3);
      if (rep == 1)
        printf("%-18s %8.3f ms  %10.3e thread-ops/s  = %6.1f ops/clk/SM at max clock %d MHz\n",
               names[op], ms, per_s, per_s / sms / (clk * 1e3), clk / 1000);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
