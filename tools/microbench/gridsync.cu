// Grid-wide barrier latency on B200: G co-resident CTAs pass N barriers
// (per-barrier arrival counter, red.release.gpu + ld.acquire.gpu spin by one
// thread, then __syncthreads) -- the dependency cost of a persistent
// decode-chain kernel per op.   nvcc -gencode arch=compute_100a,code=sm_100a -o gridsync gridsync.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void barriers(unsigned* cnt, int n, int sleep_ns) {
  for (int i = 0; i < n; i++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + i) : "memory");
      if (sleep_ns > 0) {
        while (ld_acq(cnt + i) < gridDim.x) __nanosleep(sleep_ns);
      } else {
        while (ld_acq(cnt + i) < gridDim.x) {}
      }
    }
    __syncthreads();
  }
}

int main() {
  const int N = 1000;
  unsigned* cnt;
  cudaMalloc(&cnt, sizeof(unsigned) * N);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {1, 2, 4}) {
    for (int sl : {0, 32, 100}) {
      for (int threads : {128, 384}) {
        if (per_sm * threads > 2048) continue;
        const int G = sms * per_sm;
        cudaMemset(cnt, 0, sizeof(unsigned) * N);
        void* args[] = {&cnt, (void*)&N, &sl};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaLaunchCooperativeKernel((void*)barriers, G, threads, args, 0, 0);   // warm
        cudaDeviceSynchronize();
        cudaMemset(cnt, 0, sizeof(unsigned) * N);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)barriers, G, threads, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"ctas\": %d, \"threads\": %d, \"nanosleep\": %d, \"us_per_barrier\": %.3f, \"err\": \"%s\"}\n", G,
               threads, sl, ms * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
