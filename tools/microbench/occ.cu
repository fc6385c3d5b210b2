// Occupancy of the batch-1 lookup kernel per 7B shape (diagnostic).
#include "../../paper_2407_00088_b200/csrc/gemv.cu"
#include <cstdio>

template <int R, int LG>
void report(int m, int k) {
  bl::LayoutV2 L;
  bl::make_layout(m, k, 2, 64, &L);
  auto kern = gemv_kernel<R, LG, __half, true, BITLUT_TABLE_Q8, false>;
  size_t smem = smem_plan<__half>(L, false, true, false).total;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int nb = -1;
  int th = gemv_threads(L);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, th, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  printf("%dx%d R=%d LG=%d: tiles %d threads %d smem %zu regs %d -> %d CTAs/SM (%s)\n", m, k, L.R, L.Lg,
         L.n_tiles, th, smem, fa.numRegs, nb, cudaGetErrorString(e));
}

int main() {
  report<8, 2>(4096, 4096);
  report<8, 2>(11008, 4096);
  report<8, 2>(4096, 11008);
  return 0;
}
