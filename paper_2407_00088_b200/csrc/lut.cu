// Online activation tables on the GPU (reference: pkg/src/bitlut/lut_build.py).
//
// Bit-exactness contract: every float operation below is the one the
// reference performs, in the same order, with explicit round-to-nearest
// intrinsics so nvcc cannot contract or reorder (no --use_fast_math):
//   entries     ((+-a0 +- a1) +- a2) +- a3           lut_build.py:121-125
//   table scale max|e| / 127  (IEEE division)        lut_build.py:172-173
//   q           trunc(e/scale + copysign(0.5, .))   lut_build.py:174-176
//   row sums    left-to-right f32 accumulation        lut_build.py:191-193
#include "lut_core.cuh"

namespace {

template <typename T>
__device__ __forceinline__ float load_act(const void* a, int64_t i) {
  return bl::to_f32(reinterpret_cast<const T*>(a)[i]);
}

__device__ __forceinline__ float act(const void* a, int dtype, int64_t i) {
  return dtype == BITLUT_DT_F16 ? load_act<__half>(a, i) : load_act<float>(a, i);
}

// ---- precompute_lut (lut_build.py:105-127), general g <= 8 ----
__global__ void precompute_lut_kernel(const void* __restrict__ a, int dtype, int n, int k, int g,
                                      float* __restrict__ full) {
  const int kgt = k / g;
  const int W = 1 << g;
  const int64_t total = (int64_t)n * kgt;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / kgt;
    int kg = (int)(t - row * kgt);
    float v[8];
    for (int j = 0; j < g; j++) v[j] = act(a, dtype, row * k + (int64_t)kg * g + j);
    float* dst = full + t * W;
    for (int idx = 0; idx < W; idx++) {
      float e = (idx & 1) ? v[0] : -v[0];
      for (int j = 1; j < g; j++) e = ((idx >> j) & 1) ? __fadd_rn(e, v[j]) : __fsub_rn(e, v[j]);
      dst[idx] = e;
    }
  }
}

// ---- mirror_consolidate (lut_build.py:130-143) ----
__global__ void mirror_kernel(const float* __restrict__ full, int64_t rows, int g,
                              float* __restrict__ half, int* __restrict__ asym) {
  const int H = 1 << (g - 1);
  const int64_t total = rows * H;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / H;
    int w = (int)(t - r * H);
    const float* src = full + r * 2 * H;
    float lo = src[w];
    half[t] = lo;
    // full[half + w] must equal -full[half - 1 - w]
    if (src[H + w] != -src[H - 1 - w]) atomicOr(asym, 1);
  }
}

// ---- quantize_tables (lut_build.py:153-179), one block per (row, quant group) ----
__global__ void quantize_tables_kernel(const float* __restrict__ half, int kg, int width, int gpg,
                                       int8_t* __restrict__ q, float* __restrict__ scales) {
  const int gq = blockIdx.x, row = blockIdx.y;
  const int nq = kg / gpg;
  const int64_t base = ((int64_t)row * kg + (int64_t)gq * gpg) * width;
  const int cnt = gpg * width;
  float mx = 0.f;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) mx = bl::fmax_nan(mx, fabsf(half[base + i]));
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) mx = bl::fmax_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v = bl::fmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  float scale = __fdiv_rn(red[0], 127.0f);
  if (scale == 0.0f) scale = 1.0f;
  if (threadIdx.x == 0) scales[(int64_t)row * nq + gq] = scale;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    float s = __fdiv_rn(half[base + i], scale);
    float r = truncf(__fadd_rn(s, copysignf(0.5f, s)));
    r = fminf(fmaxf(r, -127.f), 127.f);
    q[base + i] = (int8_t)(int)r;
  }
}

// ---- row_sums (lut_build.py:182-194), one thread per (row, group) ----
__global__ void row_sums_kernel(const void* __restrict__ a, int dtype, int n, int k, int gs,
                                float* __restrict__ sums) {
  const int nq = k / gs;
  const int64_t total = (int64_t)n * nq;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / nq;
    int gq = (int)(t - row * nq);
    const int64_t base = row * k + (int64_t)gq * gs;
    float acc = 0.f;
    for (int j = 0; j < gs; j++) acc = __fadd_rn(acc, act(a, dtype, base + j));
    sums[t] = acc;
  }
}

// ---- fused per-call build for g = 4 (kernel.py:226-251) ----
// grid (ceil(KG/256), n), 256 threads, one thread per k-group.  Quant groups
// (gpg k-groups, a power of two <= 128) never straddle a block.
constexpr int kLutThreads = 256;

template <int MODE, typename AT>
__global__ void __launch_bounds__(kLutThreads)
build_lut_kernel(const AT* __restrict__ a, int k, int gs, void* __restrict__ tables,
                 float* __restrict__ tscales, float* __restrict__ rowsums, int independent,
                 const bl::DepSync dep) {
  bl::pdl_launch_dependents();
  if (dep.counted) bl::dep_wait(dep);
  else if (!independent) bl::pdl_wait();   // activations come from the previous kernel
  __shared__ __align__(16) float sa[kLutThreads * 4];
  __shared__ float red[kLutThreads / 32];
  lutk::lut_block<MODE, AT>(a, k, gs, tables, tscales, rowsums, blockIdx.y, blockIdx.x * kLutThreads,
                            sa, red);
  bl::dep_signal(dep);
  if (independent) bl::pdl_wait();      // keep stream completion order
}

// ---- several table builds in one launch (op lists: every activation row a
// layer's GEMVs read) ----
constexpr int kMaxLutJobs = 8;
struct LutJobs {
  bl::DepSync dep;
  int n_jobs, independent;
  bitlut_lut_job job[kMaxLutJobs];
  int block_end[kMaxLutJobs];          // cumulative blocks (ceil(KG/256) * n per job)
};

template <int MODE, typename AT>
__global__ void __launch_bounds__(kLutThreads) build_lut_multi_kernel(const __grid_constant__ LutJobs J) {
  bl::pdl_launch_dependents();
  if (J.dep.counted) bl::dep_wait(J.dep);
  else if (!J.independent) bl::pdl_wait();
  __shared__ __align__(16) float sa[kLutThreads * 4];
  __shared__ float red[kLutThreads / 32];
  int j = 0;
  while (j + 1 < J.n_jobs && (int)blockIdx.x >= J.block_end[j]) j++;
  const int b = blockIdx.x - (j ? J.block_end[j - 1] : 0);
  const bitlut_lut_job& jb = J.job[j];
  const int bx = (jb.k / 4 + kLutThreads - 1) / kLutThreads;
  lutk::lut_block<MODE, AT>(reinterpret_cast<const AT*>(jb.a), jb.k, jb.group_size, jb.tables, jb.tscales,
                            jb.rowsums, b / bx, (b % bx) * kLutThreads, sa, red);
  bl::dep_signal(J.dep);
  if (J.independent) bl::pdl_wait();
}

// ---- any number of table builds, job list in device memory ----
template <int MODE, typename AT>
__global__ void __launch_bounds__(kLutThreads)
build_lut_batch_kernel(const bitlut_lut_job* __restrict__ jobs, const int* __restrict__ block_end, int n_jobs,
                       int independent) {
  __shared__ __align__(16) float sa[kLutThreads * 4];
  __shared__ float red[kLutThreads / 32];
  // job of this block = number of jobs ending at or before it
  int j = 0;
  for (int base = 0; base < n_jobs; base += kLutThreads) {
    const int i = base + threadIdx.x;
    j += __syncthreads_count(i < n_jobs && block_end[i] <= (int)blockIdx.x);
  }
  bl::pdl_launch_dependents();
  if (!independent) bl::pdl_wait();
  const bitlut_lut_job& jb = jobs[j];
  const int b = blockIdx.x - (j ? block_end[j - 1] : 0);
  const int bx = (jb.k / 4 + kLutThreads - 1) / kLutThreads;
  lutk::lut_block<MODE, AT>(reinterpret_cast<const AT*>(jb.a), jb.k, jb.group_size, jb.tables, jb.tscales,
                            jb.rowsums, b / bx, (b % bx) * kLutThreads, sa, red);
  if (independent) bl::pdl_wait();
}

inline int grid_1d(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = 148 * 16 * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

extern "C" int bitlut_precompute_lut(const void* a, int a_dtype, int n, int k, int g,
                                     float* full, void* stream) {
  if (g < 1 || g > 8 || n < 0 || k < 0) return BITLUT_EPARAM;
  if (a_dtype != BITLUT_DT_F32 && a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (k % g != 0) return BITLUT_ELAYOUT;
  int64_t t = (int64_t)n * (k / g);
  if (t == 0) return BITLUT_OK;
  precompute_lut_kernel<<<grid_1d(t, 128), 128, 0, (cudaStream_t)stream>>>(a, a_dtype, n, k, g, full);
  return bl_launch_status();
}

extern "C" int bitlut_mirror_consolidate(const float* full, int n, int kg, int g, float* half,
                                         int* asym_flag, void* stream) {
  if (g < 1 || g > 8 || n < 0 || kg < 0) return BITLUT_EPARAM;
  int64_t rows = (int64_t)n * kg;
  if (rows == 0) return BITLUT_OK;
  mirror_kernel<<<grid_1d(rows << (g - 1), 256), 256, 0, (cudaStream_t)stream>>>(full, rows, g, half,
                                                                                 asym_flag);
  return bl_launch_status();
}

extern "C" int bitlut_quantize_tables(const float* half, int n, int kg, int g, int group_size,
                                      int8_t* qentries, float* table_scales, void* stream) {
  if (g < 1 || g > 8 || n < 0 || kg < 0 || group_size < 1) return BITLUT_EPARAM;
  if (group_size % g != 0) return BITLUT_ELAYOUT;
  int gpg = group_size / g;
  if (kg % gpg != 0) return BITLUT_ELAYOUT;
  if (n == 0 || kg == 0) return BITLUT_OK;
  dim3 grid(kg / gpg, n);
  quantize_tables_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(half, kg, 1 << (g - 1), gpg,
                                                                 qentries, table_scales);
  return bl_launch_status();
}

extern "C" int bitlut_row_sums(const void* a, int a_dtype, int n, int k, int group_size,
                               float* sums, void* stream) {
  if (group_size < 1 || n < 0 || k < 0) return BITLUT_EPARAM;
  if (a_dtype != BITLUT_DT_F32 && a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (k % group_size != 0) return BITLUT_ELAYOUT;
  int64_t t = (int64_t)n * (k / group_size);
  if (t == 0) return BITLUT_OK;
  row_sums_kernel<<<grid_1d(t, 128), 128, 0, (cudaStream_t)stream>>>(a, a_dtype, n, k, group_size, sums);
  return bl_launch_status();
}

int bl_build_lut_launch(const void* a, int a_dtype, int n, int k, int group_size, int mode,
                        void* tables, float* tscales, float* rowsums, cudaStream_t stream, bool pdl,
                        bool independent, const bl::DepSync& dep, int* grid_out) {
  const int ind = (pdl && independent) ? 1 : 0;
  const int KG = k / 4;
  dim3 grid((KG + kLutThreads - 1) / kLutThreads, n);
  if (grid_out) *grid_out = (int)(grid.x * grid.y);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = dim3(kLutThreads); cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaError_t e;
  if (mode == BITLUT_TABLE_Q8) {
    e = a_dtype == BITLUT_DT_F16
            ? cudaLaunchKernelEx(&cfg, build_lut_kernel<BITLUT_TABLE_Q8, __half>, (const __half*)a, k, group_size,
                                 tables, tscales, rowsums, ind, dep)
            : cudaLaunchKernelEx(&cfg, build_lut_kernel<BITLUT_TABLE_Q8, float>, (const float*)a, k, group_size,
                                 tables, tscales, rowsums, ind, dep);
  } else if (mode == BITLUT_TABLE_X16) {
    e = a_dtype == BITLUT_DT_F16
            ? cudaLaunchKernelEx(&cfg, build_lut_kernel<BITLUT_TABLE_X16, __half>, (const __half*)a, k, group_size,
                                 tables, tscales, rowsums, ind, dep)
            : cudaLaunchKernelEx(&cfg, build_lut_kernel<BITLUT_TABLE_X16, float>, (const float*)a, k, group_size,
                                 tables, tscales, rowsums, ind, dep);
  } else {
    e = a_dtype == BITLUT_DT_F16
            ? cudaLaunchKernelEx(&cfg, build_lut_kernel<BITLUT_TABLE_F16, __half>, (const __half*)a, k, group_size,
                                 tables, tscales, rowsums, ind, dep)
            : cudaLaunchKernelEx(&cfg, build_lut_kernel<BITLUT_TABLE_F16, float>, (const float*)a, k, group_size,
                                 tables, tscales, rowsums, ind, dep);
  }
  return e == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

extern "C" int bitlut_build_lut(const void* a, int a_dtype, int n, int k, int group_size, int mode,
                                void* tables, float* tscales, float* rowsums, int flags, void* stream) {
  if (a_dtype != BITLUT_DT_F32 && a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8 && mode != BITLUT_TABLE_F16 && mode != BITLUT_TABLE_X16) return BITLUT_EPARAM;
  if (n < 0 || k < 0 || group_size < 4) return BITLUT_EPARAM;
  if (k % group_size != 0 || group_size % 4 != 0) return BITLUT_ELAYOUT;
  int gpg = group_size / 4;
  if (gpg > 128 || (gpg & (gpg - 1))) return BITLUT_EPARAM;   // CUDA path: power-of-two k-groups per group
  if (n == 0 || k == 0) return BITLUT_OK;
  const bl::DepSync none = {};
  return bl_build_lut_launch(a, a_dtype, n, k, group_size, mode, tables, tscales, rowsums,
                             (cudaStream_t)stream, (flags & BITLUT_FLAG_PDL) != 0,
                             (flags & BITLUT_FLAG_INDEPENDENT) != 0, none, nullptr);
}

int bl_build_lut_multi_launch(const bitlut_lut_job* jobs, int n_jobs, int mode, int flags, void* stream,
                              const bl::DepSync& dep, int* grid_out);

extern "C" int bitlut_build_lut_multi(const bitlut_lut_job* jobs, int n_jobs, int mode, int flags, void* stream) {
  const bl::DepSync none = {};
  return bl_build_lut_multi_launch(jobs, n_jobs, mode, flags, stream, none, nullptr);
}

int bl_build_lut_multi_launch(const bitlut_lut_job* jobs, int n_jobs, int mode, int flags, void* stream,
                              const bl::DepSync& dep, int* grid_out) {
  if (!jobs || n_jobs < 1 || n_jobs > kMaxLutJobs) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8 && mode != BITLUT_TABLE_F16) return BITLUT_EPARAM;
  LutJobs J;
  J.dep = dep;
  J.n_jobs = n_jobs;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  J.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  int blocks = 0;
  for (int i = 0; i < n_jobs; i++) {
    const bitlut_lut_job& jb = jobs[i];
    if (jb.a_dtype != jobs[0].a_dtype) return BITLUT_EPARAM;        // one instantiation per launch
    if (jb.a_dtype != BITLUT_DT_F32 && jb.a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
    if (jb.n < 1 || jb.k < 4 || jb.group_size < 4) return BITLUT_EPARAM;
    if (jb.k % jb.group_size != 0 || jb.group_size % 4 != 0) return BITLUT_ELAYOUT;
    const int gpg = jb.group_size / 4;
    if (gpg > 128 || (gpg & (gpg - 1))) return BITLUT_EPARAM;
    blocks += ((jb.k / 4 + kLutThreads - 1) / kLutThreads) * jb.n;
    J.job[i] = jb;
    J.block_end[i] = blocks;
  }
  if (grid_out) *grid_out = blocks;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(kLutThreads); cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr; cfg.numAttrs = 1;
  const bool f16 = jobs[0].a_dtype == BITLUT_DT_F16;
  cudaError_t e;
  if (mode == BITLUT_TABLE_Q8)
    e = f16 ? cudaLaunchKernelEx(&cfg, build_lut_multi_kernel<BITLUT_TABLE_Q8, __half>, J)
            : cudaLaunchKernelEx(&cfg, build_lut_multi_kernel<BITLUT_TABLE_Q8, float>, J);
  else
    e = f16 ? cudaLaunchKernelEx(&cfg, build_lut_multi_kernel<BITLUT_TABLE_F16, __half>, J)
            : cudaLaunchKernelEx(&cfg, build_lut_multi_kernel<BITLUT_TABLE_F16, float>, J);
  return e == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

extern "C" int bitlut_build_lut_batch_encode(const bitlut_lut_job* jobs, int n_jobs, int* block_end,
                                             int* total_blocks) {
  if (!jobs || n_jobs < 1 || !block_end || !total_blocks) return BITLUT_EPARAM;
  int64_t blocks = 0;
  for (int i = 0; i < n_jobs; i++) {
    const bitlut_lut_job& jb = jobs[i];
    if (jb.a_dtype != jobs[0].a_dtype) return BITLUT_EPARAM;
    if (jb.a_dtype != BITLUT_DT_F32 && jb.a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
    if (!jb.a || !jb.tables || !jb.rowsums) return BITLUT_EPARAM;
    if (jb.n < 1 || jb.k < 4 || jb.group_size < 4) return BITLUT_EPARAM;
    if (jb.k % jb.group_size != 0 || jb.group_size % 4 != 0) return BITLUT_ELAYOUT;
    const int gpg = jb.group_size / 4;
    if (gpg > 128 || (gpg & (gpg - 1))) return BITLUT_EPARAM;
    blocks += (int64_t)((jb.k / 4 + kLutThreads - 1) / kLutThreads) * jb.n;
    if (blocks > 0x7fffffff) return BITLUT_ESHAPE;
    block_end[i] = (int)blocks;
  }
  *total_blocks = (int)blocks;
  return BITLUT_OK;
}

extern "C" int bitlut_build_lut_batch(const bitlut_lut_job* dev_jobs, const int* dev_block_end, int n_jobs,
                                      int total_blocks, int a_dtype, int mode, int flags, void* stream) {
  if (!dev_jobs || !dev_block_end || n_jobs < 1 || total_blocks < 1) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8 && mode != BITLUT_TABLE_F16) return BITLUT_EPARAM;
  if (a_dtype != BITLUT_DT_F32 && a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  const int ind = (pdl && (flags & BITLUT_FLAG_INDEPENDENT)) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(total_blocks); cfg.blockDim = dim3(kLutThreads); cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr; cfg.numAttrs = 1;
  const bool f16 = a_dtype == BITLUT_DT_F16;
  cudaError_t e;
  if (mode == BITLUT_TABLE_Q8)
    e = f16 ? cudaLaunchKernelEx(&cfg, build_lut_batch_kernel<BITLUT_TABLE_Q8, __half>, dev_jobs, dev_block_end,
                                 n_jobs, ind)
            : cudaLaunchKernelEx(&cfg, build_lut_batch_kernel<BITLUT_TABLE_Q8, float>, dev_jobs, dev_block_end,
                                 n_jobs, ind);
  else
    e = f16 ? cudaLaunchKernelEx(&cfg, build_lut_batch_kernel<BITLUT_TABLE_F16, __half>, dev_jobs, dev_block_end,
                                 n_jobs, ind)
            : cudaLaunchKernelEx(&cfg, build_lut_batch_kernel<BITLUT_TABLE_F16, float>, dev_jobs, dev_block_end,
                                 n_jobs, ind);
  return e == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}
