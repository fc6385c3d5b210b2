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
// four nibbles at once.
//
// Accumulation: dp2a.lo/hi (IDP.2A) adds two looked-up bytes into ONE int32
// with 16-bit multipliers (1, -32768): acc = X - 32768*Y, where X and Y are
// the partial sums of two streams.  |X| <= 128*gpg < 16384 for gpg <= 128,
// so X = sext15(acc), Y = (X - acc) >> 15 recover both exactly.
//
// Per 8 lookups: 3 ALU (shift / xor) + 4 PRMT on the ALU pipe and 8 IDP.2A on
// the FMA pipe -- both pipes run at 64 lanes/clk/SM on B200 (measured,
// tools/microbench/pipes.cu), so ~64 lookups/clk/SM = 32 packed B/clk/SM,
// above the HBM share (~22 B/clk/SM at 6.45 TB/s).
//
// ---------------------------------------------------------------------------
// Work decomposition
// ---------------------------------------------------------------------------
// CTA = one tile (tile_ch channels, full K) x one activation row.  Lane =
// one unit (R consecutive k-groups of one 32-stream group).  All of a
// lane's R/2 32-byte weight loads are issued before griddepcontrol.wait, so
// under programmatic dependent launch the weight stream of this kernel
// overlaps the tail of the previous one; only the tables wait.  Partials of
// the Lg lanes sharing a quantization group are combined with a
// transpose-reduce (butterfly halving, no redundant adds), unpacked, and
// parked in shared memory; then one thread per channel replays the
// reference's float epilogue sequentially (plane-major, group ascending),
// which keeps the output bit-exact without any split-K traffic.
#include "common.cuh"
#include "layout.cuh"

namespace {

constexpr uint32_t kMult = 0x80000001u;   // int16 pair (lo = 1, hi = -32768)

struct GemvArgs {
  const uint8_t* w;
  const void* wscales;
  const void* zeros;
  const int8_t* qtab;       // (n, KG, 8)
  const float* tscales;     // (n, NQ)
  const float* rowsums;     // (n, NQ)
  float* out;               // (n, m)
  int32_t* partials;        // (n, bits, m, NQ) or null
  bl::LayoutV2 L;
};

__device__ __forceinline__ uint32_t encode_a(uint32_t q) {
  // per byte: Q - (Q < 0).  Negative bytes are >= 0x81, so no borrow.
  return q - ((q >> 7) & 0x01010101u);
}

template <int R>
__device__ __forceinline__ void lookup_unit(const bl::U8x32 (&wr)[R / 2], const uint8_t* tab_smem,
                                            int tab_off0, int tab_step, int (&acc)[16]) {
#pragma unroll
  for (int jp = 0; jp < R / 2; jp++) {
    const uint4 t = *reinterpret_cast<const uint4*>(tab_smem + tab_off0 + jp * tab_step);
#pragma unroll
    for (int kk = 0; kk < 2; kk++) {
      const uint32_t a0 = kk ? t.z : t.x, a1 = kk ? t.w : t.y;
      const uint32_t b0 = ~a0, b1 = ~a1;
#pragma unroll
      for (int w = 0; w < 4; w++) {
        const uint32_t x = wr[jp].w[kk * 4 + w];
        const uint32_t xx = x ^ 0x88888888u;
        const uint32_t xh = x >> 16, xxh = xx >> 16;
        const uint32_t A0 = bl::prmt(a0, a1, x), B0 = bl::prmt(b0, b1, xx);
        const uint32_t A1 = bl::prmt(a0, a1, xh), B1 = bl::prmt(b0, b1, xxh);
        acc[4 * w + 0] = bl::dp2a_lo(kMult, A0, acc[4 * w + 0]);
        acc[4 * w + 0] = bl::dp2a_lo(kMult, B0, acc[4 * w + 0]);
        acc[4 * w + 1] = bl::dp2a_hi(kMult, A0, acc[4 * w + 1]);
        acc[4 * w + 1] = bl::dp2a_hi(kMult, B0, acc[4 * w + 1]);
        acc[4 * w + 2] = bl::dp2a_lo(kMult, A1, acc[4 * w + 2]);
        acc[4 * w + 2] = bl::dp2a_lo(kMult, B1, acc[4 * w + 2]);
        acc[4 * w + 3] = bl::dp2a_hi(kMult, A1, acc[4 * w + 3]);
        acc[4 * w + 3] = bl::dp2a_hi(kMult, B1, acc[4 * w + 3]);
      }
    }
  }
}

// Butterfly transpose-reduce of 16 packed accumulators across LG aligned
// lanes.  Afterwards lane holds NF = 16/LG fully reduced pairs, starting at
// pair index `base`.
template <int LG>
__device__ __forceinline__ int transpose_reduce(int (&acc)[16], int lane) {
  int base = 0;
  int n = 16;
#pragma unroll
  for (int o = LG / 2; o >= 1; o >>= 1) {
    n >>= 1;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (i < n) {
        const int send = up ? acc[i] : acc[i + n];
        const int keep = up ? acc[i + n] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (up) base += n;
  }
  return base;
}

template <int R, int LG, typename ST>
__global__ void __launch_bounds__(512)
gemv_q8_kernel(GemvArgs p) {
  const bl::LayoutV2& L = p.L;
  constexpr int NF = 16 / LG;
  const int tile = blockIdx.x;
  const int row = blockIdx.y;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int T = blockDim.x;
  const int KG = L.KG, NQ = L.NQ, U = L.U;
  const int units = L.n_sg * U;
  const int pstride = 32 * L.n_sg + 1;
  const int tch = L.tile_ch;

  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* tab = smem;                                              // KG * 8
  int32_t* psm = reinterpret_cast<int32_t*>(smem + (size_t)KG * 8); // NQ * pstride
  float* wsm = reinterpret_cast<float*>(psm + (size_t)NQ * pstride);// tch * NQ
  float* zsm = wsm + (size_t)tch * NQ;                              // tch * NQ (if zeros)
  float* tsm = zsm + (p.zeros ? (size_t)tch * NQ : 0);              // NQ
  float* rsm = tsm + NQ;                                            // NQ
  float* fin = rsm + NQ;                                            // 3 * tch

  // ---- 1. issue this lane's first-round weight loads (independent of the
  //         previous kernel in the stream) ----
  bl::U8x32 wr[R / 2];
  {
    const int u = tid;
    if (u < units) {
      const int sg = u / U, uu = u - sg * U;
      const int ub = uu >> 5, l = uu & 31;
      const int nu_b = min(32, U - 32 * ub);
      const uint8_t* base = p.w + L.sg_row_base(tile, sg) + (int64_t)ub * (32 * R * 16) + l * 32;
#pragma unroll
      for (int jp = 0; jp < R / 2; jp++) wr[jp] = bl::ld_stream_256(base + (int64_t)jp * nu_b * 32);
    }
  }
  bl::pdl_launch_dependents();

  // ---- 2. weight scales / zeros of this tile -> smem (also independent) ----
  {
    const ST* ws = reinterpret_cast<const ST*>(p.wscales) + (int64_t)tile * tch * NQ;
    for (int i = tid; i < tch * NQ; i += T) wsm[i] = bl::to_f32(ws[i]);
    if (p.zeros) {
      const ST* zs = reinterpret_cast<const ST*>(p.zeros) + (int64_t)tile * tch * NQ;
      for (int i = tid; i < tch * NQ; i += T) zsm[i] = bl::to_f32(zs[i]);
    }
  }

  // ---- 3. wait for the table producer, then stage this row's tables ----
  bl::pdl_wait();
  {
    const uint2* q = reinterpret_cast<const uint2*>(p.qtab) + (int64_t)row * KG;
    for (int kg = tid; kg < KG; kg += T) {
      const uint2 v = q[kg];
      const int u = kg / R, r = kg - u * R;
      const int ub = u >> 5, l = u & 31;
      const int nu_b = min(32, U - 32 * ub);
      const int off = ub * (R / 2) * 32 * 16 + ((r >> 1) * nu_b + l) * 16 + (r & 1) * 8;
      *reinterpret_cast<uint2*>(tab + off) = make_uint2(encode_a(v.x), encode_a(v.y));
    }
    for (int i = tid; i < NQ; i += T) {
      tsm[i] = p.tscales[(int64_t)row * NQ + i];
      rsm[i] = p.rowsums[(int64_t)row * NQ + i];
    }
  }
  __syncthreads();

  // ---- 4. lookups, group reduction, unpack into psm[gq][stream] ----
  const int rounds = (units + T - 1) / T;
  for (int rd = 0; rd < rounds; rd++) {
    const int u = tid + rd * T;
    const bool live = u < units;
    int acc[16];
#pragma unroll
    for (int i = 0; i < 16; i++) acc[i] = 0;
    int sg = 0, uu = 0;
    if (live) {
      sg = u / U; uu = u - sg * U;
      const int ub = uu >> 5, l = uu & 31;
      const int nu_b = min(32, U - 32 * ub);
      if (rd > 0) {
        const uint8_t* base = p.w + L.sg_row_base(tile, sg) + (int64_t)ub * (32 * R * 16) + l * 32;
#pragma unroll
        for (int jp = 0; jp < R / 2; jp++) wr[jp] = bl::ld_stream_256(base + (int64_t)jp * nu_b * 32);
      }
      lookup_unit<R>(wr, tab, ub * (R / 2) * 32 * 16 + l * 16, nu_b * 16, acc);
    }
    if (__any_sync(0xffffffffu, live)) {
      const int base = transpose_reduce<LG>(acc, lane);
      if (live) {
        const int gq = uu / LG;
        const int gpg = R * LG;
        const int fix = -32767 * gpg;        // undo the -1 per lookup of both streams
        int32_t* dst = psm + (size_t)gq * pstride + sg * 32;
#pragma unroll
        for (int i = 0; i < NF; i++) {
          const int v = acc[i] + fix;
          const int pe = (v << 17) >> 17;
          const int po = (pe - v) >> 15;
          dst[2 * (base + i)] = pe;
          dst[2 * (base + i) + 1] = po;
        }
      }
    }
  }
  __syncthreads();

  // ---- 5. float epilogue in the reference's order (_kernels.py:179-191) ----
  // thread c: sum_i sum_gq ((pf_i*ts)*ws)*P ; thread tch+c: bias sum_gq ws*rs ;
  // thread 2*tch+c: zero-point correction sum_gq (ws*(2^(b-1)-z))*rs.
  const int bits = L.bits;
  if (tid < tch) {
    const int c = tid;
    const int64_t m = (int64_t)tile * tch + c;
    float o = 0.f;
    for (int i = 0; i < bits; i++) {
      const float pf = 0.5f * (float)(1 << i);
      const int s = c * bits + i;
      for (int gq = 0; gq < NQ; gq++) {
        const int32_t P = psm[gq * pstride + s];
        const float f = __fmul_rn(pf, tsm[gq]);
        o = __fadd_rn(o, __fmul_rn(__fmul_rn(f, wsm[c * NQ + gq]), __int2float_rn(P)));
        if (p.partials) p.partials[(((int64_t)row * bits + i) * L.m + m) * NQ + gq] = P;
      }
    }
    fin[c] = o;
  } else if (tid < 2 * tch) {
    const int c = tid - tch;
    float s = 0.f;
    for (int gq = 0; gq < NQ; gq++) s = __fadd_rn(s, __fmul_rn(wsm[c * NQ + gq], rsm[gq]));
    fin[tch + c] = s;
  } else if (p.zeros && tid < 3 * tch) {
    const int c = tid - 2 * tch;
    const float half_range = (float)(1 << (bits - 1));
    float zc = 0.f;
    for (int gq = 0; gq < NQ; gq++) {
      const float d = __fsub_rn(half_range, zsm[c * NQ + gq]);
      zc = __fadd_rn(zc, __fmul_rn(__fmul_rn(wsm[c * NQ + gq], d), rsm[gq]));
    }
    fin[2 * tch + c] = zc;
  }
  __syncthreads();
  if (tid < tch) {
    float o = __fsub_rn(fin[tid], __fmul_rn(0.5f, fin[tch + tid]));
    if (p.zeros) o = __fadd_rn(o, fin[2 * tch + tid]);
    p.out[(int64_t)row * L.m + (int64_t)tile * tch + tid] = o;
  }
}

size_t gemv_smem_bytes(const bl::LayoutV2& L, bool zeros) {
  size_t b = (size_t)L.KG * 8;
  b += (size_t)L.NQ * (32 * L.n_sg + 1) * 4;
  b += (size_t)L.tile_ch * L.NQ * 4 * (zeros ? 2 : 1);
  b += (size_t)L.NQ * 8 + (size_t)L.tile_ch * 12;
  return (b + 15) & ~(size_t)15;
}

int gemv_threads(const bl::LayoutV2& L) {
  int units = L.n_sg * L.U;
  int rounds = (units + 511) / 512;
  int t = (units + rounds - 1) / rounds;
  t = (t + 31) / 32 * 32;
  int need = 3 * L.tile_ch;      // epilogue helpers
  if (t < need) t = (need + 31) / 32 * 32;
  return t;
}

template <int R, int LG, typename ST>
int launch_q8(const GemvArgs& a, int n, cudaStream_t stream, bool pdl) {
  const size_t smem = gemv_smem_bytes(a.L, a.zeros != nullptr);
  auto kern = gemv_q8_kernel<R, LG, ST>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return BITLUT_EINTERNAL;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.L.n_tiles, n);
  cfg.blockDim = dim3(gemv_threads(a.L));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

template <typename ST>
int dispatch_q8(const GemvArgs& a, int n, cudaStream_t s, bool pdl) {
  const int R = a.L.R, LG = a.L.Lg;
  if (R == 8) {
    switch (LG) {
      case 1: return launch_q8<8, 1, ST>(a, n, s, pdl);
      case 2: return launch_q8<8, 2, ST>(a, n, s, pdl);
      case 4: return launch_q8<8, 4, ST>(a, n, s, pdl);
      case 8: return launch_q8<8, 8, ST>(a, n, s, pdl);
      case 16: return launch_q8<8, 16, ST>(a, n, s, pdl);
    }
  } else if (R == 4 && LG == 1) {
    return launch_q8<4, 1, ST>(a, n, s, pdl);
  }
  return BITLUT_EPARAM;
}

}  // namespace

int bl_build_lut_launch(const void* a, int a_dtype, int n, int k, int group_size, int mode,
                        void* tables, float* tscales, float* rowsums, cudaStream_t stream, bool pdl);

extern "C" int bitlut_mpgemm(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                             const void* wscales, const void* zeros, int scale_dtype,
                             const void* tables, const float* tscales, const float* rowsums,
                             int mode, int n, float* out, int32_t* partials, int flags,
                             void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (n < 0) return BITLUT_ESHAPE;
  if (n == 0) return BITLUT_OK;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8) return BITLUT_EPARAM;
  if (n > 65535) return BITLUT_ESHAPE;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  if (gemv_smem_bytes(L, zeros != nullptr) > 227 * 1024) return BITLUT_ELAYOUT;
  GemvArgs a;
  a.w = wgpu; a.wscales = wscales; a.zeros = zeros;
  a.qtab = reinterpret_cast<const int8_t*>(tables); a.tscales = tscales; a.rowsums = rowsums;
  a.out = out; a.partials = partials; a.L = L;
  return scale_dtype == BITLUT_DT_F16 ? dispatch_q8<__half>(a, n, (cudaStream_t)stream, pdl)
                                      : dispatch_q8<float>(a, n, (cudaStream_t)stream, pdl);
}

extern "C" int bitlut_mpgemm_launches(int m, int k, int bits, int group_size, int mode, int n) {
  (void)m; (void)k; (void)bits; (void)group_size; (void)mode;
  return n > 0 ? 1 : 0;
}

extern "C" const char* bitlut_version(void) { return "bitlut_b200 0.1.0 (sm_100a)"; }
