// Lookup-accumulate mpGEMV/mpGEMM for sm_100a (int8 tables, "cuda-q8").
//
// Replaces the reference's hot loop _kernels.gemv_q8_vector
// (pkg/src/bitlut/_kernels.py:141-192) driven by kernel.mpgemm
// (kernel.py:280-371).  Output is bitwise identical to the reference's
// vector-q8 output (zeros == NULL): the int32 staging values are exact
// and the float epilogue replays the reference's order.
//
// ---------------------------------------------------------------------------
// Lookup: the A/B tables trick (register-resident, no shared-memory gathers)
// ---------------------------------------------------------------------------
// For one k-group the mirror-consolidated int8 half table Q[0..7] lives in
// two registers.  Each weight nibble is stored pre-encoded as x = (s<<3)|eff
// (s = mirror flag, eff = half-table slot; layout.cuh).  The value to add is
// sigma*Q[eff], sigma = s ? -1 : +1 (_kernels.py:175-177).
// `prmt` in its default mode treats selector bit 3 as "replicate the sign of
// the selected byte", so with tables
//     a[e] = Q[e] - (Q[e] < 0)          b[e] = ~a[e]
//     A = prmt(a, x)          = s ? signfill(a[eff]) : a[eff]
//     B = prmt(b, x ^ 0x8)    = s ? b[eff]           : signfill(b[eff])
// one gets A + B = sigma*Q[eff] - 1 exactly, for every Q in [-127, 127]
// (checked exhaustively in tests/test_encoding.py).  One prmt does this for
// four nibbles at once.  b is never materialised: prmt(~a, sel) = ~prmt(a,
// sel) byte for byte (sign-replicate mode included) and ~y = -y - 1, so with
// Y = prmt(a, x ^ 0x8) the sum is A - Y = sigma*Q[eff] exactly; Y is
// accumulated with negated multipliers.
//
// Accumulation: dp2a.lo/hi (IDP.2A) adds two looked-up bytes into ONE int32:
// A with unsigned 16-bit multipliers (1, 32768), Y with signed (-1, -32768),
// so acc = X + 32768*Y' where X and Y' are the exact partial sums of two
// streams.  |X| <= 127*gpg < 16384 for gpg <= 128, so X = sext15(acc) and
// Y' = (acc - X) >> 15 recover both exactly.
//
// Per 8 lookups: 3 ALU (shift / xor) + 4 PRMT on the ALU pipe and 8 IDP.2A on
// the FMA pipe -- both pipes run at 64 lanes/clk/SM on B200 (measured,
// tools/microbench/pipes.cu), so ~64 lookups/clk/SM = 32 packed B/clk/SM,
// above the HBM share (~22 B/clk/SM at 6.45 TB/s).
//
// ---------------------------------------------------------------------------
// Work decomposition and latency plan
// ---------------------------------------------------------------------------
// CTA = one tile (tile_ch channels, full K) x one activation row; lane = one
// unit (R consecutive k-groups of one 32-stream group).
//  1. thread 0 starts TMA bulk copies (cp.async.bulk) of the tile's weights
//     and weight scales into shared memory: they do not depend on the
//     previous kernel, so under programmatic dependent launch (PDL) they
//     stream while the previous kernel finishes.  Bulk copies also keep the
//     weight traffic out of the in-order L1TEX load queue, so the table
//     loads issued after griddepcontrol.wait are not stuck behind it
//     (measured with tools/timeline.py: ~1 us lost per CTA otherwise).
//  2. griddepcontrol.wait; each lane loads its own k-groups' encoded tables
//     (kernel-format LUT, L2-resident) straight into registers.
//  3. lookups from shared-memory weights (LDS.128, conflict-free), then a
//     butterfly transpose-reduce across the Lg lanes of a quantization
//     group, unpack to exact int32 staging values P.
//  4. each lane forms its epilogue products ((pf_i*ts)*ws)*f32(P) exactly
//     as the reference (_kernels.py:179-185) into shared memory; one thread
//     per channel then adds them left to right in the reference's order
//     (plane-major, group ascending), while two more threads per channel run
//     the bias (:187-190) and zero-point chains.  The order makes the output
//     bitwise equal to the reference's.
// Shapes whose tile does not fit (K > 16384, or bits = 3 with large K) use
// the same pipeline with per-lane LDG.128 weight loads instead of TMA.
#include "gemv_core.cuh"

#include <cstdlib>

namespace {

using namespace blk;

// MULTI: the CTA keeps its weight tile in smem and walks rows_per_cta
// activation rows (GEMM).  A separate instantiation, so the batch-1 kernel
// keeps its register budget (84 vs 116 regs -> 5 vs 4 CTAs/SM, which is
// one wave vs two for 11008x4096).
template <int R, int LG, typename ST, bool TMA, int MODE, bool MULTI>
__global__ void __launch_bounds__(512)
gemv_kernel(GemvArgs p) {
  const bl::LayoutV2& L = p.L;
  const int tile = blockIdx.x;
  const int rpc = MULTI ? p.rows_per_cta : 1;
  const int row0 = blockIdx.y * rpc;
  const int row1 = MULTI ? min(row0 + rpc, p.n_rows) : row0 + 1;
  const int tid = threadIdx.x;
  const SmemPlan sp = smem_plan<ST>(L, p.zeros != nullptr, TMA, MULTI);
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + sp.bar_off);

  TRACE(0);
  // ---- 1. independent traffic first: weights + scales (+ zeros), once per
  //         CTA however many activation rows it processes ----
  if (TMA && tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tile_issue<ST, TMA>(p, tile, sp, smem, bar);
  __syncthreads();                      // mbarrier initialised / scales staged
  TRACE(1);

  // ---- 2. tables (produced by the previous kernel, unless independent).
  //         A dependent launch lets its successor start only after its own
  //         inputs are complete, so an INDEPENDENT successor (same tables)
  //         can read them without waiting. ----
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  TRACE(2);
  for (int row = row0; row < row1; row++) {
    uint4 tq0[R / 2];
    if (MODE == BITLUT_TABLE_Q8) prefetch_tables_q8<R>(p, row, tq0);
    load_row_vectors<MODE>(p, row, sp, smem);
    if (TMA && row == row0) mbar_wait(bar, 0);
    __syncthreads();                    // tsm / rsm visible; weights landed
    TRACE(3);
    tile_body<R, LG, ST, TMA, MODE>(p, tile, row, sp, smem, tq0);
    if (MULTI) __syncthreads();         // row done before tsm / rsm / psm are reused
  }

  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();    // keep stream completion order
  if (p.trace && tid == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + 7] = smid;
  }
  TRACE(6);
}

int max_threads() {
  static int cap = 0;
  if (!cap) {
    const char* e = getenv("BITLUT_MAX_THREADS");
    cap = e ? atoi(e) : 256;
    if (cap < 96 || cap > 512) cap = 512;
  }
  return cap;
}

int gemv_threads(const bl::LayoutV2& L) {
  const int units = L.n_sg * L.U;
  const int cap = max_threads();
  const int rounds = (units + cap - 1) / cap;
  int t = (units + rounds - 1) / rounds;
  t = (t + 31) / 32 * 32;
  if (t < 96) t = 96;                  // three epilogue chain warps
  return t;
}

template <typename ST>
bool use_tma(const bl::LayoutV2& L, bool zeros, bool keep) {
  return L.n_sg * L.U <= 512 && smem_plan<ST>(L, zeros, true, keep).total <= 112 * 1024;
}

template <int R, int LG, typename ST, bool TMA, int MODE, bool MULTI>
int launch_q8(const GemvArgs& a, int n, cudaStream_t stream, bool pdl) {
  const size_t smem = smem_plan<ST>(a.L, a.zeros != nullptr, TMA, MULTI).total;
  if (smem > 227 * 1024) return BITLUT_ELAYOUT;
  auto kern = gemv_kernel<R, LG, ST, TMA, MODE, MULTI>;
  // Once per instantiation: allow the largest plan, and ask for the
  // max-shared carveout -- weights arrive by TMA and tables by ld.cg, so
  // L1 has little to cache, while the default carveout can leave room for
  // only one CTA of a long-K tile per SM (4096x11008: two waves instead of
  // two co-resident CTAs).
  static bool configured_dev[64] = {};                  // per device
  bool& configured = configured_dev[bl_device()];
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return BITLUT_EINTERNAL;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.L.n_tiles, (n + a.rows_per_cta - 1) / a.rows_per_cta);
  if (a.grid_out) *a.grid_out = (int)(cfg.gridDim.x * cfg.gridDim.y);
  cfg.blockDim = dim3(gemv_threads(a.L));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

template <int R, int LG, typename ST>
int launch_q8_any(const GemvArgs& a0, int n, cudaStream_t s, bool pdl, int mode) {
  GemvArgs a = a0;
  // weight-stationary rows need the tile resident in smem (TMA path)
  if (a.rows_per_cta > 1 && !use_tma<ST>(a.L, a.zeros != nullptr, true)) a.rows_per_cta = 1;
  const bool multi = a.rows_per_cta > 1;
  const bool tma = multi || use_tma<ST>(a.L, a.zeros != nullptr, false);
  if (mode == BITLUT_TABLE_Q8) {
    if (multi) return launch_q8<R, LG, ST, true, BITLUT_TABLE_Q8, true>(a, n, s, pdl);
    return tma ? launch_q8<R, LG, ST, true, BITLUT_TABLE_Q8, false>(a, n, s, pdl)
               : launch_q8<R, LG, ST, false, BITLUT_TABLE_Q8, false>(a, n, s, pdl);
  }
  if (multi) return launch_q8<R, LG, ST, true, BITLUT_TABLE_F16, true>(a, n, s, pdl);
  return tma ? launch_q8<R, LG, ST, true, BITLUT_TABLE_F16, false>(a, n, s, pdl)
             : launch_q8<R, LG, ST, false, BITLUT_TABLE_F16, false>(a, n, s, pdl);
}

template <typename ST>
int dispatch_q8(const GemvArgs& a, int n, cudaStream_t s, bool pdl, int mode) {
  const int R = a.L.R, LG = a.L.Lg;
  if (R == 8) {
    switch (LG) {
      case 1: return launch_q8_any<8, 1, ST>(a, n, s, pdl, mode);
      case 2: return launch_q8_any<8, 2, ST>(a, n, s, pdl, mode);
      case 4: return launch_q8_any<8, 4, ST>(a, n, s, pdl, mode);
      case 8: return launch_q8_any<8, 8, ST>(a, n, s, pdl, mode);
      case 16: return launch_q8_any<8, 16, ST>(a, n, s, pdl, mode);
    }
  } else if (R == 4 && LG == 1) {
    return launch_q8_any<4, 1, ST>(a, n, s, pdl, mode);
  }
  return BITLUT_EPARAM;
}

bool b1_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BITLUT_B1");             // diagnostic: 0 disables the batch-1 kernel
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

}  // namespace

// gemv_b1.cu: persistent batch-1 kernel (fast epilogue, 32-stream tiles)
int bl_gemv_b1_launch(const blk::GemvArgs& g, int scale_dtype, cudaStream_t s, bool pdl);

// Internal launcher shared by the C entry points and the op-list executor
// (pipeline.cu), which passes dependency counters and reads the grid size.
int bl_mpgemm_launch(const uint8_t* wgpu, int m, int k, int bits, int group_size, const void* wscales,
                     const void* zeros, int scale_dtype, const void* tables, const float* tscales,
                     const float* rowsums, int mode, int n, float* out, int32_t* partials, int flags,
                     unsigned long long* trace, void* stream, const bl::DepSync& dep, int* grid_out) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (n < 0) return BITLUT_ESHAPE;
  if (n == 0) return BITLUT_OK;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8 && mode != BITLUT_TABLE_F16 && mode != BITLUT_TABLE_X16) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8 && partials) return BITLUT_EPARAM;    // int32 partials: Q8 only
  if (n > 65535) return BITLUT_ESHAPE;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  GemvArgs a = {};
  a.dep = dep;
  a.grid_out = grid_out;
  a.w = wgpu; a.wscales = wscales; a.zeros = zeros;
  a.qtab = reinterpret_cast<const uint8_t*>(tables); a.tscales = tscales; a.rowsums = rowsums;
  a.out = out; a.partials = partials; a.trace = trace; a.L = L;
  a.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  a.fast = (flags & BITLUT_FLAG_FAST_EPILOGUE) != 0;
  a.n_rows = n;
  // weight-stationary rows: a CTA keeps its tile in smem for up to 32 rows
  // once there are enough (tile, row-block) CTAs to fill the GPU
  a.rows_per_cta = 1;
  if (n >= 8) {
    int r = 32;
    while (r > 1 && (int64_t)L.n_tiles * ((n + r - 1) / r) < 4 * 148) r >>= 1;
    a.rows_per_cta = r;
  }
  const bool combined = (flags & BITLUT_FLAG_COMBINED_PARTIALS) != 0;
  if (combined && (!a.fast || mode != BITLUT_TABLE_Q8 || L.n_sg != 1 || trace)) return BITLUT_EPARAM;
  if (flags & BITLUT_FLAG_LAYER_SET) {
    // operand in the layer-set layout: fast epilogue, int8 tables, the lean
    // batch-1 / rows kernels only (else the caller passes the v2 operand)
    if (!((mode == BITLUT_TABLE_Q8 || (mode == BITLUT_TABLE_X16 && n == 1)) && a.fast && !partials && !trace &&
          L.n_sg == 1))
      return BITLUT_ELAYOUT;
    a.layer_set = 1;
    a.f16_tables = mode == BITLUT_TABLE_X16 ? BITLUT_TABLE_X16 : 0;
    return bl_gemv_b1_launch(a, scale_dtype, (cudaStream_t)stream, pdl);
  }
  if (mode == BITLUT_TABLE_X16) {
    // 16-bit block-fixed-point tables: the lean batch-1 kernel only (the
    // caller uses BITLUT_TABLE_F16 for everything else)
    if (!(a.fast && n == 1 && !trace && L.n_sg == 1)) return BITLUT_ELAYOUT;
    a.f16_tables = BITLUT_TABLE_X16;
    return bl_gemv_b1_launch(a, scale_dtype, (cudaStream_t)stream, pdl);
  }
  if (mode == BITLUT_TABLE_Q8 && (a.fast ? (!partials || combined) : !partials) && !trace &&
      L.n_sg == 1 && (b1_enabled() || combined)) {
    rc = bl_gemv_b1_launch(a, scale_dtype, (cudaStream_t)stream, pdl);
    if (rc != BITLUT_ELAYOUT || combined) return rc;  // else: shape exceeds its smem plan
  }
  return scale_dtype == BITLUT_DT_F16 ? dispatch_q8<__half>(a, n, (cudaStream_t)stream, pdl, mode)
                                      : dispatch_q8<float>(a, n, (cudaStream_t)stream, pdl, mode);
}

extern "C" int bitlut_mpgemm_traced(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                                    const void* wscales, const void* zeros, int scale_dtype,
                                    const void* tables, const float* tscales, const float* rowsums,
                                    int mode, int n, float* out, int32_t* partials, int flags,
                                    unsigned long long* trace, void* stream) {
  const bl::DepSync none = {};
  return bl_mpgemm_launch(wgpu, m, k, bits, group_size, wscales, zeros, scale_dtype, tables, tscales, rowsums,
                          mode, n, out, partials, flags, trace, stream, none, nullptr);
}

extern "C" int bitlut_mpgemm(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                             const void* wscales, const void* zeros, int scale_dtype,
                             const void* tables, const float* tscales, const float* rowsums,
                             int mode, int n, float* out, int32_t* partials, int flags,
                             void* stream) {
  return bitlut_mpgemm_traced(wgpu, m, k, bits, group_size, wscales, zeros, scale_dtype, tables,
                              tscales, rowsums, mode, n, out, partials, flags, nullptr, stream);
}

extern "C" int bitlut_mpgemm_launches(int m, int k, int bits, int group_size, int mode, int n) {
  (void)m; (void)k; (void)bits; (void)group_size; (void)mode;
  return n > 0 ? 1 : 0;
}

extern "C" const char* bitlut_version(void) { return "bitlut_b200 0.1.0 (sm_100a)"; }
