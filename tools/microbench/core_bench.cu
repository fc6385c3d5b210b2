// Lookup-core variants on shared-memory-resident weights (no HBM): clocks per
// 32-bit weight word per SM for the plane-merged W4 / W2 cores of
// csrc/b1_core.cuh and candidates that move selector preparation off the ALU
// pipe (PRMT/SHF/LOP3) onto the FMA pipe (IMAD / IMAD.HI).  The HBM feed at
// 6.5 TB/s is 5.77 clk per word-warp (128 B) per SM; a core has to be well
// below that to leave room for the epilogue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o core_bench core_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define DEV __device__ __forceinline__
DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV int dp4a(uint32_t a, uint32_t b, int c) { int d; asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint32_t mulhi(uint32_t a, uint32_t b) { uint32_t d; asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
DEV uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
DEV uint4 lds128(uint32_t addr) { uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)); return v; }

// V: 0 = shipped core; 1 = high-half selectors by IMAD.HI; 2 = IMAD.HI and
// no LOP3 (Y from the byte-reversed table with the complemented selector,
// ~x = x * -1 - 1 on the FMA pipe); 3 (W2) = two channels per PRMT with
// zeroed multipliers (no selector PRMTs)
template <int BITS, int V>
DEV void core_word(uint32_t x, uint32_t a0, uint32_t a1, uint32_t r0, uint32_t r1, int* acc, uint32_t m1) {
  const uint32_t k16 = 0x10000u;
  if constexpr (BITS == 4) {
    if constexpr (V == 0) {
      const uint32_t xx = x ^ 0x88888888u;
      acc[0] = dp4a(prmt(a0, a1, x), 0x08040201u, acc[0]);
      acc[0] = dp4a(prmt(a0, a1, xx), 0xF8FCFEFFu, acc[0]);
      acc[1] = dp4a(prmt(a0, a1, x >> 16), 0x08040201u, acc[1]);
      acc[1] = dp4a(prmt(a0, a1, xx >> 16), 0xF8FCFEFFu, acc[1]);
    } else if constexpr (V == 1) {
      const uint32_t xx = x ^ 0x88888888u;
      acc[0] = dp4a(prmt(a0, a1, x), 0x08040201u, acc[0]);
      acc[0] = dp4a(prmt(a0, a1, xx), 0xF8FCFEFFu, acc[0]);
      acc[1] = dp4a(prmt(a0, a1, mulhi(x, k16)), 0x08040201u, acc[1]);
      acc[1] = dp4a(prmt(a0, a1, mulhi(xx, k16)), 0xF8FCFEFFu, acc[1]);
    } else {
      const uint32_t nx = madlo(x, m1, m1);
      acc[0] = dp4a(prmt(a0, a1, x), 0x08040201u, acc[0]);
      acc[0] = dp4a(prmt(r0, r1, nx), 0xF8FCFEFFu, acc[0]);
      acc[1] = dp4a(prmt(a0, a1, mulhi(x, k16)), 0x08040201u, acc[1]);
      acc[1] = dp4a(prmt(r0, r1, mulhi(nx, k16)), 0xF8FCFEFFu, acc[1]);
    }
  } else {
    if constexpr (V == 0) {
      const uint32_t xx = x ^ 0x88888888u;
      const uint32_t s01 = prmt(x, xx, 0x5140u), s23 = prmt(x, xx, 0x7362u);
      acc[0] = dp4a(prmt(a0, a1, s01), 0xFEFF0201u, acc[0]);
      acc[1] = dp4a(prmt(a0, a1, s01 >> 16), 0xFEFF0201u, acc[1]);
      acc[2] = dp4a(prmt(a0, a1, s23), 0xFEFF0201u, acc[2]);
      acc[3] = dp4a(prmt(a0, a1, s23 >> 16), 0xFEFF0201u, acc[3]);
    } else if constexpr (V == 1) {
      const uint32_t xx = x ^ 0x88888888u;
      const uint32_t s01 = prmt(x, xx, 0x5140u), s23 = prmt(x, xx, 0x7362u);
      acc[0] = dp4a(prmt(a0, a1, s01), 0xFEFF0201u, acc[0]);
      acc[1] = dp4a(prmt(a0, a1, mulhi(s01, k16)), 0xFEFF0201u, acc[1]);
      acc[2] = dp4a(prmt(a0, a1, s23), 0xFEFF0201u, acc[2]);
      acc[3] = dp4a(prmt(a0, a1, mulhi(s23, k16)), 0xFEFF0201u, acc[3]);
    } else if constexpr (V == 2) {
      // selectors [x.b, ~x.b]: A from (a0,a1), Y from the reversed table --
      // a PRMT reads ONE register pair, so A and Y cannot share a PRMT here:
      // two channels per PRMT, zeroed multipliers
      const uint32_t nx = madlo(x, m1, m1);
      const uint32_t A0 = prmt(a0, a1, x), Y0 = prmt(r0, r1, nx);
      const uint32_t A1 = prmt(a0, a1, mulhi(x, k16)), Y1 = prmt(r0, r1, mulhi(nx, k16));
      acc[0] = dp4a(A0, 0x00000201u, acc[0]);
      acc[0] = dp4a(Y0, 0x0000FEFFu, acc[0]);
      acc[1] = dp4a(A0, 0x02010000u, acc[1]);
      acc[1] = dp4a(Y0, 0xFEFF0000u, acc[1]);
      acc[2] = dp4a(A1, 0x00000201u, acc[2]);
      acc[2] = dp4a(Y1, 0x0000FEFFu, acc[2]);
      acc[3] = dp4a(A1, 0x02010000u, acc[3]);
      acc[3] = dp4a(Y1, 0xFEFF0000u, acc[3]);
    } else {
      const uint32_t xx = x ^ 0x88888888u;
      const uint32_t A0 = prmt(a0, a1, x), Y0 = prmt(a0, a1, xx);
      const uint32_t A1 = prmt(a0, a1, x >> 16), Y1 = prmt(a0, a1, xx >> 16);
      acc[0] = dp4a(A0, 0x00000201u, acc[0]);
      acc[0] = dp4a(Y0, 0x0000FEFFu, acc[0]);
      acc[1] = dp4a(A0, 0x02010000u, acc[1]);
      acc[1] = dp4a(Y0, 0xFEFF0000u, acc[1]);
      acc[2] = dp4a(A1, 0x00000201u, acc[2]);
      acc[2] = dp4a(Y1, 0x0000FEFFu, acc[2]);
      acc[3] = dp4a(A1, 0x02010000u, acc[3]);
      acc[3] = dp4a(Y1, 0xFEFF0000u, acc[3]);
    }
  }
}

constexpr int R = 8;

template <int BITS, int V>
__global__ void __launch_bounds__(128) core_kernel(int tiles, uint32_t seed, int* out, uint32_t m1) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NACC = BITS == 4 ? 8 : 16;
  constexpr int PER = BITS == 4 ? 2 : 4;
  const int tid = threadIdx.x;
  uint32_t* w = reinterpret_cast<uint32_t*>(smem);
  for (int i = tid; i < 2 * 16384 / 4; i += blockDim.x) w[i] = seed * (i + 1) * 2654435761u;
  __syncthreads();
  uint32_t tq[R * 2], tr[R * 2];
#pragma unroll
  for (int i = 0; i < R * 2; i++) { tq[i] = seed * (tid + i) * 40503u; tr[i] = __byte_perm(tq[i ^ 1], 0, 0x0123); }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem) + (tid >> 5) * (32 * R * 16) + (tid & 31) * 16;
  int sum = 0;
  for (int t = 0; t < tiles; t++) {
    int acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = 0;
    const uint32_t sb = base + (t & 1) * 16384;
#pragma unroll
    for (int j = 0; j < R; j++) {
      const uint4 wv = lds128(sb + j * 512);
      const uint32_t ws[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int q = 0; q < 4; q++)
        core_word<BITS, V>(ws[q], tq[2 * j], tq[2 * j + 1], tr[2 * j], tr[2 * j + 1], acc + PER * q, m1);
    }
#pragma unroll
    for (int i = 0; i < NACC; i++) sum += acc[i];
  }
  if (sum == 0x12345678) out[0] = sum;
}

template <int BITS, int V>
void run(const char* label, int sms, int clk, int* out) {
  auto k = core_kernel<BITS, V>;
  const int smem = 36 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 128, smem);
  const int tiles = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    k<<<sms * per, 128, smem>>>(tiles, 3, out, 0xFFFFFFFFu);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  // word-warps per SM: CTAs/SM * 4 warps * tiles * R * 4 words
  const double ww = (double)per * 4 * tiles * R * 4;
  const double clk_per_word = ms * 1e-3 * clk * 1e3 / ww;
  printf("%-34s %d CTAs/SM  %7.3f ms  %5.2f clk per word-warp per SM  (%5.2f TB/s equivalent on %d SMs)\n", label, per, ms,
         clk_per_word, 128.0 / clk_per_word * sms * clk * 1e3 / 1e12, sms);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int* out; cudaMalloc(&out, 4);
  run<4, 0>("W4 shipped", sms, clk, out);
  run<4, 1>("W4 IMAD.HI shifts", sms, clk, out);
  run<4, 2>("W4 IMAD.HI + reversed table", sms, clk, out);
  run<2, 0>("W2 shipped", sms, clk, out);
  run<2, 1>("W2 IMAD.HI shifts", sms, clk, out);
  run<2, 2>("W2 two-channel PRMT, reversed, HI", sms, clk, out);
  run<2, 3>("W2 two-channel PRMT, SHF", sms, clk, out);
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
