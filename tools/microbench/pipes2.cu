// Which issue pipes do the lookup core's instructions share?  Times single
// opcodes and 1:1 mixes (independent dependency chains) and prints
// warp-instructions per clock per SM.  A mix that runs at the sum of the two
// single rates uses two pipes; one that runs at the single rate shares one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes2 pipes2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define DEV __device__ __forceinline__
DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint32_t dp4a(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint32_t dp2a(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint32_t shr16(uint32_t a, uint32_t b) { uint32_t d; asm volatile("shf.r.wrap.b32 %0, %1, %2, 5;" : "=r"(d) : "r"(a), "r"(b)); return d; }
DEV uint32_t xorc(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0x1e;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint32_t mulhi(uint32_t a, uint32_t b) { uint32_t d; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
DEV uint32_t mad(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint32_t mulwide_hi(uint32_t a, uint32_t b) { uint64_t d; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(d) : "r"(a), "r"(b)); return (uint32_t)(d >> 32); }
DEV float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
DEV uint32_t i2f(uint32_t a) { float d; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(d) : "r"(a)); return __float_as_uint(d); }
DEV uint32_t shfl(uint32_t a) { uint32_t d; asm volatile("shfl.sync.bfly.b32 %0, %1, 1, 31, 0xffffffff;" : "=r"(d) : "r"(a)); return d; }
DEV uint32_t sel(uint32_t a, uint32_t b, uint32_t p) { uint32_t d; asm volatile("{.reg .pred q; setp.ne.u32 q, %3, 0; selp.b32 %0, %1, %2, q;}" : "=r"(d) : "r"(a), "r"(b), "r"(p)); return d; }

enum { PRMT, IDP4, IDP2, SHF, LOP, MULHI, IMAD, MULWIDE, FFMA, I2F, SHFL, NOPS };
const char* kNames[] = {"PRMT", "IDP.4A", "IDP.2A", "SHF", "LOP3", "IMAD.HI", "IMAD", "IMAD.WIDE", "FFMA", "I2FP", "SHFL"};

template <int OP>
DEV uint32_t apply(uint32_t v, uint32_t t0, uint32_t t1) {
  if (OP == PRMT) return prmt(t0, t1, v);
  if (OP == IDP4) return dp4a(t0, 0x08040201u, v);
  if (OP == IDP2) return dp2a(0x80000001u, t0, v);
  if (OP == SHF) return shr16(v, v);
  if (OP == LOP) return xorc(v, t0, t1);
  if (OP == MULHI) return mulhi(v, t1);
  if (OP == IMAD) return mad(v, t0, t1);
  if (OP == MULWIDE) return mulwide_hi(v, t1);
  if (OP == FFMA) return __float_as_uint(ffma(__uint_as_float(v), 1.0001f, 0.5f));
  if (OP == I2F) return i2f(v);
  if (OP == SHFL) return shfl(v);
  return v;
}

constexpr int ITERS = 2048;
constexpr int NCH = 8;     // independent chains per opcode

template <int A, int B, int RA, int RB>
__global__ void probe(uint32_t seed, uint32_t* out) {
  uint32_t a[NCH], b[NCH];
#pragma unroll
  for (int i = 0; i < NCH; i++) { a[i] = seed * (i + 1) + threadIdx.x; b[i] = seed * (i + 77) ^ threadIdx.x; }
  const uint32_t t0 = seed ^ 0x1234567u, t1 = seed + 0x10000u;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int r = 0; r < (RA > RB ? RA : RB); r++) {
#pragma unroll
      for (int i = 0; i < NCH; i++) {
        if (r < RA) a[i] = apply<A>(a[i], t0, t1);
        if (B >= 0 && r < RB) b[i] = apply<(B >= 0 ? B : 0)>(b[i], t0, t1);
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NCH; i++) s ^= a[i] ^ b[i];
  if (s == 0xdeadbeef) out[0] = s;
}

static int g_sms, g_clk;
static uint32_t* g_out;

template <int A, int B, int RA = 1, int RB = 1>
void run(const char* label) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = g_sms * 4, threads = 256;
  float ms = 0;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    probe<A, B, RA, RB><<<blocks, threads>>>(1, g_out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double winstr = (double)blocks * (threads / 32) * ITERS * NCH * (RA + (B >= 0 ? RB : 0));
  const double per_clk = winstr / (ms * 1e-3) / g_sms / (g_clk * 1e3);
  printf("%-28s %8.3f ms  %6.3f warp-instr/clk/SM\n", label, ms, per_clk);
}

int main() {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&g_clk, cudaDevAttrClockRate, 0);
  cudaMalloc(&g_out, 4);
  printf("SMs %d, max clock %d MHz (rates assume max clock)\n", g_sms, g_clk / 1000);
  run<PRMT, -1>("PRMT");
  run<IDP4, -1>("IDP.4A");
  run<IDP2, -1>("IDP.2A");
  run<SHF, -1>("SHF");
  run<LOP, -1>("LOP3");
  run<MULHI, -1>("IMAD.HI");
  run<IMAD, -1>("IMAD");
  run<MULWIDE, -1>("IMAD.WIDE");
  run<FFMA, -1>("FFMA");
  run<I2F, -1>("I2FP");
  run<SHFL, -1>("SHFL");
  run<PRMT, IDP4>("PRMT + IDP.4A");
  run<PRMT, SHF>("PRMT + SHF");
  run<PRMT, LOP>("PRMT + LOP3");
  run<PRMT, MULHI>("PRMT + IMAD.HI");
  run<PRMT, IMAD>("PRMT + IMAD");
  run<PRMT, FFMA>("PRMT + FFMA");
  run<IDP4, IMAD>("IDP.4A + IMAD");
  run<IDP4, MULHI>("IDP.4A + IMAD.HI");
  run<IDP4, FFMA>("IDP.4A + FFMA");
  run<IDP4, SHF>("IDP.4A + SHF");
  run<IDP4, I2F>("IDP.4A + I2FP");
  run<PRMT, I2F>("PRMT + I2FP");
  run<PRMT, SHFL>("PRMT + SHFL");
  run<PRMT, IDP4, 3, 2>("PRMT x3 + IDP.4A x2");
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
