// Read-bandwidth probe: how fast can one kernel stream S bytes (LDG.128, all
// loads issued up front), launched back to back in a CUDA graph over buffers
// rotating through > 4x L2, with and without programmatic dependent launch.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U>
__global__ void rd(const uint4* __restrict__ src, size_t n16, uint32_t* out, int pdl) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  for (size_t base = tid; base < n16; base += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      size_t i = base + u * stride;
      v[u] = i < n16 ? ldg_stream(src + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void empty_k(int pdl) {
  if (pdl) { asm volatile("griddepcontrol.launch_dependents;"); asm volatile("griddepcontrol.wait;" ::: "memory"); }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d, L2 %d MB\n", sms, l2 >> 20);
  uint32_t* out; cudaMalloc(&out, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t sizes[] = {2u << 20, 4u << 20, 8u << 20, 11272192, 22544384, 58720256, 117440512, 512u << 20};
  for (size_t bytes : sizes) {
    size_t nbuf = (size_t)(4.0 * l2 / bytes) + 1; if (nbuf < 2) nbuf = 2; if (nbuf > 64) nbuf = 64;
    std::vector<uint4*> bufs(nbuf);
    for (auto& b : bufs) { cudaMalloc(&b, bytes); cudaMemset(b, 1, bytes); }
    size_t n16 = bytes / 16;
    for (int pdl = 0; pdl < 2; pdl++) {
      for (int cfg = 0; cfg < 3; cfg++) {
        int threads = 512;
        int blocks = cfg == 0 ? sms * 4 : (cfg == 1 ? sms * 2 : (int)((n16 + threads * 8 - 1) / (threads * 8)));
        if (blocks > sms * 4) blocks = sms * 4;
        int reps = (int)nbuf * 4;
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < reps; r++) {
          cudaLaunchConfig_t lc{}; lc.gridDim = blocks; lc.blockDim = threads; lc.stream = st;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = pdl; lc.attrs = at; lc.numAttrs = 1;
          cudaLaunchKernelEx(&lc, rd<8>, (const uint4*)bufs[r % nbuf], n16, out, pdl);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        float best = 1e9;
        for (int t = 0; t < 5; t++) {
          cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st);
          cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        double us = best * 1e3 / reps;
        printf("bytes %10zu pdl %d blocks %5d: %8.3f us/launch  %7.1f GB/s\n", bytes, pdl, blocks, us, bytes / (us * 1e-6) / 1e9);
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
      }
    }
    for (auto& b : bufs) cudaFree(b);
  }
  for (int pdl = 0; pdl < 2; pdl++) {
    int reps = 200;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < reps; r++) {
      cudaLaunchConfig_t lc{}; lc.gridDim = sms; lc.blockDim = 256; lc.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl; lc.attrs = at; lc.numAttrs = 1;
      cudaLaunchKernelEx(&lc, empty_k, pdl);
    }
    cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
    cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel pdl %d: %.3f us/launch\n", pdl, ms * 1e3 / reps);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
