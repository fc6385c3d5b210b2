// Shared device helpers for the bitlut B200 kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "../../include/bitlut_b200.h"

#define BL_DEV __device__ __forceinline__

// Device-side bounds checks of the checks build (build.py build_lib(checks=
// True) -> libbitlut_b200_checks.so, -DBITLUT_CHECKS): a violated index
// bound prints the condition and traps.  compute-sanitizer is closed on the
// GPU pool, so the GPU tests are also run against that build.  Compiled out
// of the product library.
#ifdef BITLUT_CHECKS
#include <cstdio>
#define BL_CHECK(c)                                                                       \
  do {                                                                                    \
    if (!(c)) {                                                                           \
      printf("BL_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                          \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define BL_CHECK(c) \
  do {              \
  } while (0)
#endif
namespace bl {
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
}  // namespace bl

namespace bl {

// prmt.b32 in its default mode.  Unlike __byte_perm (which masks each
// selector nibble to 3 bits), bit 3 of a selector nibble is honoured: the
// output byte becomes the sign (msb) of the selected byte replicated.  The
// int8 lookup relies on exactly that (see gemv.cu, "A/B tables").
BL_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// d = c + mult.lo16 * b.byte0 + mult.hi16 * b.byte1   (signed)
BL_DEV int dp2a_lo(uint32_t mult, uint32_t b, int c) {
  int d;
  asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(mult), "r"(b), "r"(c));
  return d;
}
// d = c + mult.lo16 * b.byte2 + mult.hi16 * b.byte3   (signed)
BL_DEV int dp2a_hi(uint32_t mult, uint32_t b, int c) {
  int d;
  asm("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(mult), "r"(b), "r"(c));
  return d;
}

// Unsigned 16-bit multipliers (lo/hi of mult as u16), signed bytes of b.
BL_DEV int dp2a_lo_u(uint32_t mult, uint32_t b, int c) {
  int d;
  asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(mult), "r"(b), "r"(c));
  return d;
}
BL_DEV int dp2a_hi_u(uint32_t mult, uint32_t b, int c) {
  int d;
  asm("dp2a.hi.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(mult), "r"(b), "r"(c));
  return d;
}

// x >> 16 on the FMA-heavy pipe (IDP.2A: x.b2 * 1 + x.b3 * 256) instead of a
// SHF on the ALU pipe, which the lookups' PRMTs saturate (IDP.2A/4A and IMAD
// share one half-rate pipe, PRMT/SHF/LOP3/I2FP another: tools/microbench/pipes2.cu)
BL_DEV uint32_t shr16_idp(uint32_t x) {
  uint32_t d;
  asm("dp2a.hi.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(0x01000001u), "r"(x), "r"(0u));
  return d;
}


// d = c + sum_i a.byte_i * b.byte_i   (signed x signed)
BL_DEV int dp4a(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

struct U8x32 { uint32_t w[8]; };

// 256-bit streaming load (sm_100: LDG.E.256): weights are read exactly once.
BL_DEV U8x32 ld_stream_256(const void* p) {
  U8x32 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]),
                 "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
               : "l"(p));
  return r;
}

// L2-coherent loads (bypass L1): data written by other CTAs of the same
// launch (pipeline.cu) must not be read through the non-coherent path.
BL_DEV uint4 ld_cg_128(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
BL_DEV float ld_cg_f32(const float* p) {
  float r;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

BL_DEV uint4 ld_nc_128(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Programmatic dependent launch (PDL) controls.  Both are no-ops when the
// kernel was not launched with the programmatic-serialization attribute.
BL_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
BL_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Op-list dependency counters (pipeline.cu graph executor).  A kernel
// launched with counters uses no griddepcontrol.wait at all: it spins (one
// thread) until every producer launch has counted all of its CTAs, counts
// itself when done, and exits without waiting for its stream predecessor
// (the list ends with a join kernel that waits for every launch's count).  Producers are always resident when a consumer
// spins: PDL launches a kernel only after every CTA of its predecessor has
// started, and each kernel of the list is launched after its producers.
constexpr int kMaxDepWaits = 8;
struct DepSync {
  const unsigned* wait_cnt[kMaxDepWaits];
  unsigned wait_target[kMaxDepWaits];
  int n_wait;
  int counted;                // 1: launched by the counted executor (no PDL waits at all)
  unsigned* done;             // +1 per CTA after its last global write, or null
  unsigned* total;            // optional: +1 per CTA of every counted launch, or null
};

BL_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// every thread of the CTA must call these
// Callers that read producer data through the async proxy (TMA) afterwards
// must issue fence_proxy_async() in the issuing thread first.
BL_DEV void dep_wait(const DepSync& d) {
  if (threadIdx.x == 0)
    for (int i = 0; i < d.n_wait; i++)
      while (ld_acquire_u32(d.wait_cnt[i]) < d.wait_target[i]) __nanosleep(20);
  __syncthreads();
}
BL_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
BL_DEV void dep_signal(const DepSync& d) {
  if (!d.done) return;
  __syncthreads();           // the CTA's writes happen-before thread 0's release (bar.sync cumulativity)
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(d.done) : "memory");
    if (d.total) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(d.total) : "memory");
  }
}

// max that propagates NaN (max.NaN.f32): a non-finite activation makes its
// group's table scale NaN, so the outputs that read it are non-finite too
// (the CUDA-tensor path has no host-side finiteness check).  Equal to fmaxf
// on non-NaN inputs, so the tables stay bitwise the reference's.
BL_DEV float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

BL_DEV float to_f32(float x) { return x; }
BL_DEV float to_f32(__half x) { return __half2float(x); }

}  // namespace bl

// Host side: the current device's ordinal for per-device once-flags
// (function attributes and SM counts are per device; one process may drive
// several GPUs).
static inline int bl_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= 64 ? 0 : d;
}

// Host-side launch-status helper: every entry point returns one of the
// BITLUT_* codes; a CUDA launch failure maps to BITLUT_EINTERNAL.
static inline int bl_launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}
