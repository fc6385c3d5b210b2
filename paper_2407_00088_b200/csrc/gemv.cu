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
#include "common.cuh"
#include "layout.cuh"

namespace {

constexpr uint32_t kMult = 0x80000001u;   // int16 pair (lo = 1, hi = -32768)

struct GemvArgs {
  const uint8_t* w;
  const void* wscales;
  const void* zeros;
  const uint8_t* qtab;       // kernel-format tables (n, KG*8)
  const float* tscales;      // (n, NQ)
  const float* rowsums;      // (n, NQ)
  float* out;                // (n, m)
  int32_t* partials;         // (n, bits, m, NQ) or null
  unsigned long long* trace; // null, or (grid, 8) globaltimer stamps per CTA
  int independent;           // BITLUT_FLAG_INDEPENDENT: wait only before exiting
  bl::LayoutV2 L;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot)                                                                       \
  do {                                                                                    \
    if (p.trace && tid == 0)                                                              \
      p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (slot)] = gtimer();      \
  } while (0)

// ---- TMA bulk copy + mbarrier helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "BL_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra BL_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// One k-group of 32 streams: 4 words x (2 selectors + 4 prmt + 8 dp2a).
__device__ __forceinline__ void lookup_kg(const uint4 w, uint32_t a0, uint32_t a1, int (&acc)[16]) {
  const uint32_t b0 = ~a0, b1 = ~a1;
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t x = ws[q];
    const uint32_t xx = x ^ 0x88888888u;
    const uint32_t A0 = bl::prmt(a0, a1, x), B0 = bl::prmt(b0, b1, xx);
    const uint32_t A1 = bl::prmt(a0, a1, x >> 16), B1 = bl::prmt(b0, b1, xx >> 16);
    acc[4 * q + 0] = bl::dp2a_lo(kMult, A0, acc[4 * q + 0]);
    acc[4 * q + 0] = bl::dp2a_lo(kMult, B0, acc[4 * q + 0]);
    acc[4 * q + 1] = bl::dp2a_hi(kMult, A0, acc[4 * q + 1]);
    acc[4 * q + 1] = bl::dp2a_hi(kMult, B0, acc[4 * q + 1]);
    acc[4 * q + 2] = bl::dp2a_lo(kMult, A1, acc[4 * q + 2]);
    acc[4 * q + 2] = bl::dp2a_lo(kMult, B1, acc[4 * q + 2]);
    acc[4 * q + 3] = bl::dp2a_hi(kMult, A1, acc[4 * q + 3]);
    acc[4 * q + 3] = bl::dp2a_hi(kMult, B1, acc[4 * q + 3]);
  }
}

// Butterfly transpose-reduce of NV accumulators across LG aligned lanes
// (no redundant adds).  Afterwards the lane holds NV/LG fully reduced values,
// starting at index `base`.  Fixed order -> deterministic for floats too.
template <int LG, int NV, typename T>
__device__ __forceinline__ int transpose_reduce(T (&acc)[NV], int lane) {
  int base = 0;
  int n = NV;
#pragma unroll
  for (int o = LG / 2; o >= 1; o >>= 1) {
    n >>= 1;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < NV / 2; i++) {
      if (i < n) {
        const T send = up ? acc[i] : acc[i + n];
        const T keep = up ? acc[i + n] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (up) base += n;
  }
  return base;
}

// fp16-table lookup of one k-group for 32 streams ("cuda-f16").  Tables:
// lo0/lo1 = low bytes of the 8 fp16 half-table entries, hi0/hi1 = high
// bytes.  Per 4 nibbles: two prmt gather the bytes (selector bit 3 masked),
// a third prmt in sign-replicate mode turns the mirror flags into a byte
// mask (flag -> 0x80) that flips the fp16 sign, two prmt interleave the
// bytes into half2, and FHADD (f32 += f16 half) accumulates in fp32.
__device__ __forceinline__ void lookup_kg_f16(const uint4 w, const uint4 t, float (&acc)[32]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t x = ws[q];
    const uint32_t e = x & 0x77777777u;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t eh = h ? e >> 16 : e, xh = h ? x >> 16 : x;
      const uint32_t lo = bl::prmt(t.x, t.y, eh);
      uint32_t hi = bl::prmt(t.z, t.w, eh);
      const uint32_t one = bl::prmt(0x01010101u, 0x01010101u, xh);   // 1 where s = 0
      hi ^= 0x80808080u - one * 128u;                                  // 0x80 where s = 1
      const uint32_t h01 = bl::prmt(lo, hi, 0x5140u), h23 = bl::prmt(lo, hi, 0x7362u);
      float* a = acc + 8 * q + 4 * h;
      asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[0]) : "h"((unsigned short)(h01 & 0xffffu)));
      asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[1]) : "h"((unsigned short)(h01 >> 16)));
      asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[2]) : "h"((unsigned short)(h23 & 0xffffu)));
      asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(a[3]) : "h"((unsigned short)(h23 >> 16)));
    }
  }
}

// Shared-memory plan.  Region A holds the tile's weights (TMA variant) and
// is reused for the epilogue products once the lookups are done.
struct SmemPlan {
  int rowlen;            // floats per channel row of epilogue products (odd)
  size_t a_bytes, p_off, s_off, z_off, t_off, r_off, f_off, bar_off, total;
};

template <typename ST>
__host__ __device__ inline SmemPlan smem_plan(const bl::LayoutV2& L, bool zeros, bool tma) {
  SmemPlan s;
  const int need = (L.bits + 1 + (zeros ? 1 : 0)) * L.NQ;
  s.rowlen = ((need + 3) / 4) * 4;
  if (((s.rowlen / 4) & 1) == 0) s.rowlen += 4;
  const size_t wbytes = tma ? (size_t)L.n_sg * L.KG * 16 : 0;
  const size_t terms = (size_t)L.tile_ch * s.rowlen * 4;
  s.a_bytes = ((wbytes > terms ? wbytes : terms) + 15) & ~(size_t)15;
  const size_t sc = ((size_t)L.tile_ch * L.NQ * sizeof(ST) + 15) & ~(size_t)15;
  s.p_off = s.a_bytes;                                  // psm: NQ x (32*n_sg+1) int32
  s.s_off = s.p_off + (((size_t)L.NQ * (32 * L.n_sg + 1) * 4 + 15) & ~(size_t)15);
  s.z_off = s.s_off + sc;
  s.t_off = s.z_off + (zeros ? sc : 0);
  s.r_off = s.t_off + (((size_t)L.NQ * 4 + 15) & ~(size_t)15);
  s.f_off = s.r_off + (((size_t)L.NQ * 4 + 15) & ~(size_t)15);
  s.bar_off = s.f_off + (size_t)3 * 32 * 4;
  s.total = s.bar_off + 16;
  return s;
}

// Epilogue products for every (channel, group) of the tile; tile_ch is a
// power of two so the (c, gq) split is a shift/mask.  BITS is compile-time so
// the plane loop unrolls; partials / zero points are separate passes.
template <int BITS, int MODE, typename ST>
__device__ __forceinline__ void form_terms(const GemvArgs& p, const ST* sraw, const ST* zraw,
                                           const float* tsm, const float* rsm, const int32_t* psm,
                                           float* terms, int rowlen, int tid, int T, int row, int tile) {
  const bl::LayoutV2& L = p.L;
  const int tch = L.tile_ch, NQ = L.NQ;
  const int pstride = 32 * L.n_sg + 1;
  const int lg_tch = __ffs(tch) - 1;
  const int n = tch * NQ;
  if ((NQ & 3) == 0) {
    // 4 consecutive groups per thread step: float4 / 8-byte vector traffic
    const int n4 = n >> 2;
    for (int idx = tid; idx < n4; idx += T) {
      const int c = idx & (tch - 1), gq = (idx >> lg_tch) << 2;
      float ws[4];
      if (sizeof(ST) == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(sraw + c * NQ + gq);
        const __half2 h0 = *reinterpret_cast<const __half2*>(&v.x), h1 = *reinterpret_cast<const __half2*>(&v.y);
        ws[0] = __low2float(h0); ws[1] = __high2float(h0); ws[2] = __low2float(h1); ws[3] = __high2float(h1);
      } else {
        const float4 v = *reinterpret_cast<const float4*>(sraw + c * NQ + gq);
        ws[0] = v.x; ws[1] = v.y; ws[2] = v.z; ws[3] = v.w;
      }
      const float4 ts4 = *reinterpret_cast<const float4*>(tsm + gq);
      const float4 rs4 = *reinterpret_cast<const float4*>(rsm + gq);
      const float ts[4] = {ts4.x, ts4.y, ts4.z, ts4.w}, rs[4] = {rs4.x, rs4.y, rs4.z, rs4.w};
      float* trow = terms + c * rowlen + gq;
      const int32_t* pr = psm + gq * pstride + c * BITS;
#pragma unroll
      for (int i = 0; i < BITS; i++) {
        float t[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int32_t P = pr[q * pstride + i];
          if (MODE == BITLUT_TABLE_Q8) {
            const float f = __fmul_rn(0.5f * (float)(1 << i), ts[q]);
            t[q] = __fmul_rn(__fmul_rn(f, ws[q]), __int2float_rn(P));
          } else {
            t[q] = __fmul_rn(__fmul_rn(0.5f * (float)(1 << i), ws[q]), __int_as_float(P));
          }
        }
        *reinterpret_cast<float4*>(trow + i * NQ) = make_float4(t[0], t[1], t[2], t[3]);
      }
      *reinterpret_cast<float4*>(trow + BITS * NQ) =
          make_float4(__fmul_rn(ws[0], rs[0]), __fmul_rn(ws[1], rs[1]), __fmul_rn(ws[2], rs[2]),
                      __fmul_rn(ws[3], rs[3]));
    }
  } else
  for (int idx = tid; idx < n; idx += T) {
    const int c = idx & (tch - 1), gq = idx >> lg_tch;
    const float ws = bl::to_f32(sraw[c * NQ + gq]);
    const float ts = tsm[gq];
    float* trow = terms + c * rowlen + gq;
    const int32_t* pr = psm + gq * pstride + c * BITS;
#pragma unroll
    for (int i = 0; i < BITS; i++) {
      if (MODE == BITLUT_TABLE_Q8) {
        // _kernels.py:183-184: ((pf * ts) * ws) * f32(stage)
        const float f = __fmul_rn(0.5f * (float)(1 << i), ts);
        trow[i * NQ] = __fmul_rn(__fmul_rn(f, ws), __int2float_rn(pr[i]));
      } else {
        // _kernels.py:131: (pf * ws) * stage, stage = f32 sum of fp16 lookups
        trow[i * NQ] = __fmul_rn(__fmul_rn(0.5f * (float)(1 << i), ws), __int_as_float(pr[i]));
      }
    }
    trow[BITS * NQ] = __fmul_rn(ws, rsm[gq]);
  }
  if (p.zeros) {
    const float half_range = (float)(1 << (BITS - 1));
    for (int idx = tid; idx < n; idx += T) {
      const int c = idx & (tch - 1), gq = idx >> lg_tch;
      const float ws = bl::to_f32(sraw[c * NQ + gq]);
      terms[c * rowlen + (BITS + 1) * NQ + gq] =
          __fmul_rn(__fmul_rn(ws, __fsub_rn(half_range, bl::to_f32(zraw[c * NQ + gq]))), rsm[gq]);
    }
  }
  if (MODE == BITLUT_TABLE_Q8 && p.partials) {
    for (int idx = tid; idx < n * BITS; idx += T) {
      const int gq = idx % NQ, ci = idx / NQ, c = ci / BITS, i = ci - c * BITS;
      p.partials[(((int64_t)row * BITS + i) * L.m + (int64_t)tile * tch + c) * NQ + gq] =
          psm[gq * pstride + c * BITS + i];
    }
  }
}

template <int R, int LG, typename ST, bool TMA, int MODE>
__global__ void __launch_bounds__(512)
gemv_kernel(GemvArgs p) {
  const bl::LayoutV2& L = p.L;
  constexpr int NF = 16 / LG;
  const int tile = blockIdx.x;
  const int row = blockIdx.y;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int T = blockDim.x;
  const int KG = L.KG, NQ = L.NQ, U = L.U;
  const int units = L.n_sg * U;
  const int tch = L.tile_ch;
  const int bits = L.bits;
  const bool has_zeros = p.zeros != nullptr;
  const SmemPlan sp = smem_plan<ST>(L, has_zeros, TMA);

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* wbuf = smem;
  float* terms = reinterpret_cast<float*>(smem);      // after the lookups (TMA)
  int32_t* psm = reinterpret_cast<int32_t*>(smem + sp.p_off);
  const int pstride = 32 * L.n_sg + 1;
  const ST* sraw = reinterpret_cast<const ST*>(smem + sp.s_off);
  const ST* zraw = reinterpret_cast<const ST*>(smem + sp.z_off);
  float* tsm = reinterpret_cast<float*>(smem + sp.t_off);
  float* rsm = reinterpret_cast<float*>(smem + sp.r_off);
  float* fin = reinterpret_cast<float*>(smem + sp.f_off);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + sp.bar_off);

  TRACE(0);
  // ---- 1. independent traffic first: weights + scales (+ zeros) ----
  const uint32_t sc_bytes = (uint32_t)((size_t)tch * NQ * sizeof(ST));
  const int64_t sc_elem0 = (int64_t)tile * tch * NQ;
  if (TMA) {
    if (tid == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t wbytes = (uint32_t)((size_t)L.n_sg * KG * 16);
      mbar_expect_tx(bar, wbytes + sc_bytes * (has_zeros ? 2u : 1u));
      const uint64_t pol = policy_evict_first();
      const uint8_t* src = p.w + L.sg_row_base(tile, 0);
      for (uint32_t off = 0; off < wbytes; off += 32768u) {   // the tile is contiguous
        const uint32_t nb = wbytes - off < 32768u ? wbytes - off : 32768u;
        bulk_g2s(wbuf + off, src + off, nb, bar, pol);
      }
      bulk_g2s((void*)sraw, reinterpret_cast<const ST*>(p.wscales) + sc_elem0, sc_bytes, bar, pol);
      if (has_zeros)
        bulk_g2s((void*)zraw, reinterpret_cast<const ST*>(p.zeros) + sc_elem0, sc_bytes, bar, pol);
    }
  } else {
    const uint4* s4 = reinterpret_cast<const uint4*>(reinterpret_cast<const ST*>(p.wscales) + sc_elem0);
    for (int i = tid; i < (int)(sc_bytes / 16); i += T)
      reinterpret_cast<uint4*>(smem + sp.s_off)[i] = bl::ld_nc_128(s4 + i);
    if (has_zeros) {
      const uint4* z4 = reinterpret_cast<const uint4*>(reinterpret_cast<const ST*>(p.zeros) + sc_elem0);
      for (int i = tid; i < (int)(sc_bytes / 16); i += T)
        reinterpret_cast<uint4*>(smem + sp.z_off)[i] = bl::ld_nc_128(z4 + i);
    }
  }
  __syncthreads();                      // mbarrier initialised / scales staged
  TRACE(1);

  // ---- 2. tables (produced by the previous kernel, unless independent).
  //         A dependent launch lets its successor start only after its own
  //         inputs are complete, so an INDEPENDENT successor (same tables)
  //         can read them without waiting. ----
  if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  TRACE(2);
  for (int i = tid; i < NQ; i += T) {
    if (MODE == BITLUT_TABLE_Q8) tsm[i] = p.tscales[(int64_t)row * NQ + i];
    rsm[i] = p.rowsums[(int64_t)row * NQ + i];
  }
  if (TMA) mbar_wait(bar, 0);
  __syncthreads();                      // tsm / rsm visible; weights landed
  TRACE(3);

  // ---- 3. lookups, reduction, exact staging values -> psm[gq][stream] ----
  const int rowlen = sp.rowlen;
  const int rounds = (units + T - 1) / T;
  for (int rd = 0; rd < rounds; rd++) {
    const int u = tid + rd * T;
    const bool live = u < units;
    int sg = 0, uu = 0, ub = 0, l = 0, nu_b = 32;
    if (live) {
      sg = u / U; uu = u - sg * U;
      ub = uu >> 5; l = uu & 31;
      nu_b = min(32, U - 32 * ub);
    }
    const uint8_t* wsrc = TMA ? wbuf + (size_t)sg * KG * 16 + (size_t)ub * (32 * R * 16) + l * 16
                              : p.w + L.sg_row_base(tile, sg) + (int64_t)ub * (32 * R * 16) + l * 16;
    if constexpr (MODE == BITLUT_TABLE_Q8) {
      int acc[16];
#pragma unroll
      for (int i = 0; i < 16; i++) acc[i] = 0;
      if (live) {
        uint4 tq[R / 2];
        uint4 wr[R];
        const uint8_t* tb = p.qtab + (int64_t)row * KG * 8 + (int64_t)ub * (32 * R * 8) + l * 16;
        // full unit blocks (nu_b == 32) get compile-time strides
        const int stride = nu_b == 32 ? 512 : nu_b * 16;
#pragma unroll
        for (int jp = 0; jp < R / 2; jp++) tq[jp] = bl::ld_nc_128(tb + jp * stride);
#pragma unroll
        for (int j = 0; j < R; j++)
          wr[j] = TMA ? *reinterpret_cast<const uint4*>(wsrc + j * stride)
                      : bl::ld_nc_128(wsrc + (int64_t)j * stride);
#pragma unroll
        for (int j = 0; j < R; j++)
          lookup_kg(wr[j], (j & 1) ? tq[j >> 1].z : tq[j >> 1].x, (j & 1) ? tq[j >> 1].w : tq[j >> 1].y, acc);
      }
      int base = 0;
      if (__any_sync(0xffffffffu, live)) base = transpose_reduce<LG, 16, int>(acc, lane);
      if (live) {
        // undo the -1 per lookup of both streams, split each pair
        const int fix = -32767 * (R * LG);
        int32_t* dst = psm + (size_t)(uu / LG) * pstride + sg * 32 + 2 * base;
#pragma unroll
        for (int i = 0; i < NF; i++) {
          const int v = acc[i] + fix;
          const int pe = (v << 17) >> 17;
          dst[2 * i] = pe;
          dst[2 * i + 1] = (pe - v) >> 15;
        }
      }
    } else {
      float acc[32];
#pragma unroll
      for (int i = 0; i < 32; i++) acc[i] = 0.f;
      if (live) {
        const uint8_t* tb = p.qtab + (int64_t)row * KG * 16 + (int64_t)ub * (32 * R * 16) + l * 16;
#pragma unroll
        for (int j = 0; j < R; j++) {
          const uint4 t = bl::ld_nc_128(tb + j * nu_b * 16);
          const uint4 w = TMA ? *reinterpret_cast<const uint4*>(wsrc + j * nu_b * 16)
                              : bl::ld_nc_128(wsrc + (int64_t)j * nu_b * 16);
          lookup_kg_f16(w, t, acc);
        }
      }
      int base = 0;
      if (__any_sync(0xffffffffu, live)) base = transpose_reduce<LG, 32, float>(acc, lane);
      if (live) {
        int32_t* dst = psm + (size_t)(uu / LG) * pstride + sg * 32 + base;
#pragma unroll
        for (int i = 0; i < 32 / LG; i++) dst[i] = __float_as_int(acc[i]);
      }
    }
  }
  TRACE(4);
  __syncthreads();                      // psm complete; region A (weights) free

  // ---- 4. epilogue products, formed exactly as the reference does:
  //         ((pf_i*ts)*ws)*f32(P)  (_kernels.py:183-184), ws*rs (:188) and the
  //         zero-point term (ws*(2^(b-1)-z))*rs ----
  switch (bits) {
    case 1: form_terms<1, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, terms, rowlen, tid, T, row, tile); break;
    case 2: form_terms<2, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, terms, rowlen, tid, T, row, tile); break;
    case 3: form_terms<3, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, terms, rowlen, tid, T, row, tile); break;
    default: form_terms<4, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, terms, rowlen, tid, T, row, tile); break;
  }
  __syncthreads();
  TRACE(5);

  // ---- 5. left-to-right chains, one per channel, each kind in its own warp
  //         (warp 0: main sum, warp 1: bias, warp 2: zero points) ----
  {
    const int w = tid >> 5, c = tid & 31;
    int start = 0, len = 0;
    bool run = c < tch;
    if (w == 0) { start = 0; len = bits * NQ; }
    else if (w == 1) { start = bits * NQ; len = NQ; }
    else if (w == 2 && has_zeros) { start = (bits + 1) * NQ; len = NQ; }
    else run = false;
    if (run) {
      const float* t = terms + c * rowlen + start;
      float o = 0.f;
      int j = 0;
      if ((start & 3) == 0) {
        // 16-byte loads (rowlen/4 odd: conflict-free across the 16..32 lanes),
        // two loads ahead of the serial add chain
        const float4* t4 = reinterpret_cast<const float4*>(t);
        const int n4 = len >> 2;
        float4 a0 = n4 > 0 ? t4[0] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 a1 = n4 > 1 ? t4[1] : a0;
        for (int q = 0; q < n4; q++) {
          const float4 cur = a0;
          a0 = a1;
          if (q + 2 < n4) a1 = t4[q + 2];
          o = __fadd_rn(o, cur.x); o = __fadd_rn(o, cur.y);
          o = __fadd_rn(o, cur.z); o = __fadd_rn(o, cur.w);
        }
        j = n4 << 2;
      }
      for (; j < len; j++) o = __fadd_rn(o, t[j]);
      fin[w * 32 + c] = o;
    }
  }
  __syncthreads();
  if (tid < tch) {
    float o = __fsub_rn(fin[tid], __fmul_rn(0.5f, fin[32 + tid]));
    if (has_zeros) o = __fadd_rn(o, fin[64 + tid]);
    p.out[(int64_t)row * L.m + (int64_t)tile * tch + tid] = o;
  }
  if (p.independent) bl::pdl_wait();    // keep stream completion order
  if (p.trace && tid == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + 7] = smid;
  }
  TRACE(6);
}

int gemv_threads(const bl::LayoutV2& L) {
  const int units = L.n_sg * L.U;
  const int rounds = (units + 511) / 512;
  int t = (units + rounds - 1) / rounds;
  t = (t + 31) / 32 * 32;
  if (t < 96) t = 96;                  // three epilogue chain warps
  return t;
}

template <typename ST>
bool use_tma(const bl::LayoutV2& L, bool zeros) {
  return L.n_sg * L.U <= 512 && smem_plan<ST>(L, zeros, true).total <= 112 * 1024;
}

template <int R, int LG, typename ST, bool TMA, int MODE>
int launch_q8(const GemvArgs& a, int n, cudaStream_t stream, bool pdl) {
  const size_t smem = smem_plan<ST>(a.L, a.zeros != nullptr, TMA).total;
  if (smem > 227 * 1024) return BITLUT_ELAYOUT;
  auto kern = gemv_kernel<R, LG, ST, TMA, MODE>;
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

template <int R, int LG, typename ST>
int launch_q8_any(const GemvArgs& a, int n, cudaStream_t s, bool pdl, int mode) {
  const bool tma = use_tma<ST>(a.L, a.zeros != nullptr);
  if (mode == BITLUT_TABLE_Q8)
    return tma ? launch_q8<R, LG, ST, true, BITLUT_TABLE_Q8>(a, n, s, pdl)
               : launch_q8<R, LG, ST, false, BITLUT_TABLE_Q8>(a, n, s, pdl);
  return tma ? launch_q8<R, LG, ST, true, BITLUT_TABLE_F16>(a, n, s, pdl)
             : launch_q8<R, LG, ST, false, BITLUT_TABLE_F16>(a, n, s, pdl);
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

}  // namespace

extern "C" int bitlut_mpgemm_traced(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                                    const void* wscales, const void* zeros, int scale_dtype,
                                    const void* tables, const float* tscales, const float* rowsums,
                                    int mode, int n, float* out, int32_t* partials, int flags,
                                    unsigned long long* trace, void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (n < 0) return BITLUT_ESHAPE;
  if (n == 0) return BITLUT_OK;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (mode != BITLUT_TABLE_Q8 && mode != BITLUT_TABLE_F16) return BITLUT_EPARAM;
  if (mode == BITLUT_TABLE_F16 && partials) return BITLUT_EPARAM;   // int32 partials: Q8 only
  if (n > 65535) return BITLUT_ESHAPE;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  GemvArgs a;
  a.w = wgpu; a.wscales = wscales; a.zeros = zeros;
  a.qtab = reinterpret_cast<const uint8_t*>(tables); a.tscales = tscales; a.rowsums = rowsums;
  a.out = out; a.partials = partials; a.trace = trace; a.L = L;
  a.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  return scale_dtype == BITLUT_DT_F16 ? dispatch_q8<__half>(a, n, (cudaStream_t)stream, pdl, mode)
                                      : dispatch_q8<float>(a, n, (cudaStream_t)stream, pdl, mode);
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
