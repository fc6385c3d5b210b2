// Shared device code of the lookup-accumulate kernels (gemv.cu: per-call
// kernel; pipeline.cu: persistent executor).  Design notes: gemv.cu.
#pragma once
#include "common.cuh"
#include "layout.cuh"

namespace blk {


// Stream-pair packing: v = P_even + 32768 * P_odd.  The looked-up A bytes go
// in with unsigned multipliers (1, 32768), the complementary Y bytes (see
// lookup_kg) with signed (-1, -32768).
constexpr uint32_t kMult = 0x80000001u;      // u16 pair (lo = 1, hi = 32768)
constexpr uint32_t kMultNeg = 0x8000FFFFu;   // s16 pair (lo = -1, hi = -32768)


// Fused all-gather epilogue (SURVEY §8(e) "B200-native upgrade"): every
// output element is also stored into the gathered output buffer of each of
// n_peers ranks (peer-accessible memory, e.g. torch symmetric memory over
// NVLink), at column col_offset + channel; after the last CTA of the grid
// has finished its stores it adds 1 to every peer's flag with release
// semantics at system scope.  A rank's gathered buffer is complete when its
// flag reaches (epoch) x world.  `ticket` is a zero-initialised device
// counter of the caller, reset by the last CTA.
constexpr int kMaxPeers = 8;
struct GatherArgs {
  int n_peers;
  int col_offset;
  float* peer_out[kMaxPeers];
  unsigned* peer_flag[kMaxPeers];
  unsigned* ticket;
};

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
  int fast;                  // BITLUT_FLAG_FAST_EPILOGUE: fixed-order parallel fp32 sums
  int rows_per_cta;          // activation rows processed per CTA (weights loaded once)
  int n_rows;
  bl::LayoutV2 L;
  bl::DepSync dep;           // op-list counters (n_wait == 0 and done == null otherwise)
  int* grid_out;             // host: receives the launch's CTA count (op-list executor), or null
  int f16_tables;            // BITLUT_TABLE_F16 (batch-1 fast lean kernel only; 0 = int8 tables)
  int mixed_tables;          // matrices carry their own tables (bitlut_mpgemv_multi_tab): lean kernel only
  int layer_set;             // BITLUT_FLAG_LAYER_SET: operand in the layer-set layout (lean / rows-lean kernels only)
  const GatherArgs* gather;  // host side: fused all-gather epilogue (batch-1 fast kernel), or null
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
// try_wait suspend-time hint: a waiting warp sleeps until the phase completes
// (or this many ns pass) instead of re-issuing the probe -- the spin cost
// issue slots the lookups of other warps could use
constexpr uint32_t kSuspendNs = 20000;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "BL_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra BL_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(kSuspendNs)
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
// A/B tables: with a = Q - (Q<0) per byte and b = ~a, prmt(a, x) +
// prmt(b, x ^ 8) = sQ - 1 for every nibble (s = mirror flag, bit 3 of x).
// Since prmt(~a, sel) = ~prmt(a, sel) byte for byte (sign-replicate mode
// included) and ~y = -y - 1, the B term is -(Y + 1) with Y = prmt(a, x ^ 8):
// A - Y = sQ exactly, so the B lookup reuses the A table and enters dp2a
// with negated multipliers -- no complement, no per-lookup constant.
__device__ __forceinline__ void lookup_kg(const uint4 w, uint32_t a0, uint32_t a1, int (&acc)[16]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t x = ws[q];
    const uint32_t xx = x ^ 0x88888888u;
    const uint32_t A0 = bl::prmt(a0, a1, x), Y0 = bl::prmt(a0, a1, xx);
    const uint32_t A1 = bl::prmt(a0, a1, x >> 16), Y1 = bl::prmt(a0, a1, xx >> 16);
    acc[4 * q + 0] = bl::dp2a_lo_u(kMult, A0, acc[4 * q + 0]);
    acc[4 * q + 0] = bl::dp2a_lo(kMultNeg, Y0, acc[4 * q + 0]);
    acc[4 * q + 1] = bl::dp2a_hi_u(kMult, A0, acc[4 * q + 1]);
    acc[4 * q + 1] = bl::dp2a_hi(kMultNeg, Y0, acc[4 * q + 1]);
    acc[4 * q + 2] = bl::dp2a_lo_u(kMult, A1, acc[4 * q + 2]);
    acc[4 * q + 2] = bl::dp2a_lo(kMultNeg, Y1, acc[4 * q + 2]);
    acc[4 * q + 3] = bl::dp2a_hi_u(kMult, A1, acc[4 * q + 3]);
    acc[4 * q + 3] = bl::dp2a_hi(kMultNeg, Y1, acc[4 * q + 3]);
  }
}

// Batch-1 fast-path lookup (gemv_stream.cu, gemv_pack.cu): plane-merging
// accumulators, S_c = sum_p 2^p P_p per channel.
// One k-group of 32 streams.  A = prmt(a, x), Y = prmt(a, x ^ 8): A - Y = sQ
// exactly for every nibble (gemv_core.cuh lookup_kg).
template <int BITS, int NACC>
__device__ __forceinline__ void lookup_merged(const uint4 w, uint32_t a0, uint32_t a1, int (&acc)[NACC]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t x = ws[q];
    const uint32_t xx = x ^ 0x88888888u;
    if constexpr (BITS == 4) {
      // nibbles 0..3 = planes 0..3 of channel 2q, nibbles 4..7 of channel 2q+1
      const uint32_t A0 = bl::prmt(a0, a1, x), Y0 = bl::prmt(a0, a1, xx);
      const uint32_t A1 = bl::prmt(a0, a1, x >> 16), Y1 = bl::prmt(a0, a1, xx >> 16);
      acc[2 * q] = bl::dp4a(A0, 0x08040201u, acc[2 * q]);
      acc[2 * q] = bl::dp4a(Y0, 0xF8FCFEFFu, acc[2 * q]);
      acc[2 * q + 1] = bl::dp4a(A1, 0x08040201u, acc[2 * q + 1]);
      acc[2 * q + 1] = bl::dp4a(Y1, 0xF8FCFEFFu, acc[2 * q + 1]);
    } else if constexpr (BITS == 2) {
      // byte b of x = channel 4q+b (nibbles: plane 0, plane 1); the selector
      // [x.b, xx.b] looks up [A_p0, A_p1, Y_p0, Y_p1] in one prmt
      const uint32_t s01 = bl::prmt(x, xx, 0x5140u), s23 = bl::prmt(x, xx, 0x7362u);
      acc[4 * q + 0] = bl::dp4a(bl::prmt(a0, a1, s01), 0xFEFF0201u, acc[4 * q + 0]);
      acc[4 * q + 1] = bl::dp4a(bl::prmt(a0, a1, s01 >> 16), 0xFEFF0201u, acc[4 * q + 1]);
      acc[4 * q + 2] = bl::dp4a(bl::prmt(a0, a1, s23), 0xFEFF0201u, acc[4 * q + 2]);
      acc[4 * q + 3] = bl::dp4a(bl::prmt(a0, a1, s23 >> 16), 0xFEFF0201u, acc[4 * q + 3]);
    } else {
      // W1: acc[4q+h] = channels (8q+2h, 8q+2h+1) packed P_even + 32768 P_odd
      const uint32_t A0 = bl::prmt(a0, a1, x), Y0 = bl::prmt(a0, a1, xx);
      const uint32_t A1 = bl::prmt(a0, a1, x >> 16), Y1 = bl::prmt(a0, a1, xx >> 16);
      acc[4 * q + 0] = bl::dp2a_lo_u(kMult, A0, acc[4 * q + 0]);
      acc[4 * q + 0] = bl::dp2a_lo(kMultNeg, Y0, acc[4 * q + 0]);
      acc[4 * q + 1] = bl::dp2a_hi_u(kMult, A0, acc[4 * q + 1]);
      acc[4 * q + 1] = bl::dp2a_hi(kMultNeg, Y0, acc[4 * q + 1]);
      acc[4 * q + 2] = bl::dp2a_lo_u(kMult, A1, acc[4 * q + 2]);
      acc[4 * q + 2] = bl::dp2a_lo(kMultNeg, Y1, acc[4 * q + 2]);
      acc[4 * q + 3] = bl::dp2a_hi_u(kMult, A1, acc[4 * q + 3]);
      acc[4 * q + 3] = bl::dp2a_hi(kMultNeg, Y1, acc[4 * q + 3]);
    }
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
      // high halves on the FMA-heavy pipe (the five PRMTs below saturate the ALU pipe)
      const uint32_t eh = h ? bl::shr16_idp(e) : e, xh = h ? bl::shr16_idp(x) : x;
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
  size_t a_bytes, terms_off, p_off, s_off, z_off, t_off, r_off, f_off, bar_off, total;
};

// keep_weights: the products get their own region instead of reusing the
// weights' (multi-row CTAs keep the tile's weights for every row).
template <typename ST>
__host__ __device__ inline SmemPlan smem_plan(const bl::LayoutV2& L, bool zeros, bool tma,
                                              bool keep_weights = false) {
  SmemPlan s;
  const int need = (L.bits + 1 + (zeros ? 1 : 0)) * L.NQ;
  s.rowlen = ((need + 3) / 4) * 4;
  if (((s.rowlen / 4) & 1) == 0) s.rowlen += 4;
  const size_t wbytes = tma ? (size_t)L.n_sg * L.KG * 16 : 0;
  const size_t terms = (size_t)L.tile_ch * s.rowlen * 4;
  if (keep_weights) {
    s.terms_off = (wbytes + 15) & ~(size_t)15;
    s.a_bytes = s.terms_off + ((terms + 15) & ~(size_t)15);
  } else {
    s.terms_off = 0;
    s.a_bytes = ((wbytes > terms ? wbytes : terms) + 15) & ~(size_t)15;
  }
  const size_t sc = ((size_t)L.tile_ch * L.NQ * sizeof(ST) + 15) & ~(size_t)15;
  s.p_off = s.a_bytes;                                  // psm: NQ x (32*n_sg+1) int32
  // psm rows: 32*n_sg+1 int32 staging values, or tile_ch+4 floats (register epilogue)
  const int prow = 32 * L.n_sg + 1 > L.tile_ch + 4 ? 32 * L.n_sg + 1 : L.tile_ch + 4;
  s.s_off = s.p_off + (((size_t)L.NQ * prow * 4 + 15) & ~(size_t)15);
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

// Start a tile's independent traffic: TMA bulk copies of its weights and
// scales (+ zeros) into smem (thread 0; completion on `bar` via expect_tx),
// or plain loads of the scales for the LDG variant (all threads).
template <typename ST, bool TMA>
__device__ __forceinline__ void tile_issue(const GemvArgs& p, int tile, const SmemPlan& sp, uint8_t* smem,
                                           uint64_t* bar) {
  const bl::LayoutV2& L = p.L;
  const int tid = threadIdx.x, T = blockDim.x;
  const int tch = L.tile_ch, NQ = L.NQ, KG = L.KG;
  const bool has_zeros = p.zeros != nullptr;
  const uint32_t sc_bytes = (uint32_t)((size_t)tch * NQ * sizeof(ST));
  const int64_t sc_elem0 = (int64_t)tile * tch * NQ;
  if (TMA) {
    if (tid == 0) {
      const uint32_t wbytes = (uint32_t)((size_t)L.n_sg * KG * 16);
      mbar_expect_tx(bar, wbytes + sc_bytes * (has_zeros ? 2u : 1u));
      const uint64_t pol = policy_evict_first();
      const uint8_t* src = p.w + L.sg_row_base(tile, 0);
      for (uint32_t off = 0; off < wbytes; off += 32768u) {   // the tile is contiguous
        const uint32_t nb = wbytes - off < 32768u ? wbytes - off : 32768u;
        bulk_g2s(smem + off, src + off, nb, bar, pol);
      }
      bulk_g2s(smem + sp.s_off, reinterpret_cast<const ST*>(p.wscales) + sc_elem0, sc_bytes, bar, pol);
      if (has_zeros)
        bulk_g2s(smem + sp.z_off, reinterpret_cast<const ST*>(p.zeros) + sc_elem0, sc_bytes, bar, pol);
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
}

// Row-dependent per-group vectors (table scales, row sums) -> smem.
template <int MODE>
__device__ __forceinline__ void load_row_vectors(const GemvArgs& p, int row, const SmemPlan& sp,
                                                 uint8_t* smem) {
  const int NQ = p.L.NQ;
  float* tsm = reinterpret_cast<float*>(smem + sp.t_off);
  float* rsm = reinterpret_cast<float*>(smem + sp.r_off);
  for (int i = threadIdx.x; i < NQ; i += blockDim.x) {
    if (MODE == BITLUT_TABLE_Q8) tsm[i] = bl::ld_cg_f32(p.tscales + (int64_t)row * NQ + i);
    rsm[i] = bl::ld_cg_f32(p.rowsums + (int64_t)row * NQ + i);
  }
}

// Fast epilogue (BITLUT_FLAG_FAST_EPILOGUE): the int32 staging values are
// the same exact ones, but the fp32 combination is a fixed-order parallel
// reduction instead of the reference's left-to-right chain: tpc threads per
// channel each sum a strided subset of the groups (all planes' products,
// minus half the bias product, plus the zero-point product), then a
// butterfly over the tpc lanes.  Deterministic; differs from the reference
// in the last bits only (tolerance-tested).
template <int BITS, int MODE, typename ST>
__device__ __forceinline__ void fast_epilogue(const GemvArgs& p, const ST* sraw, const ST* zraw,
                                              const float* tsm, const float* rsm, const int32_t* psm,
                                              int tid, int T, int row, int tile) {
  const bl::LayoutV2& L = p.L;
  const int tch = L.tile_ch, NQ = L.NQ;
  const int pstride = 32 * L.n_sg + 1;
  int tpc = 32;
  while (tpc * tch > T) tpc >>= 1;            // threads per channel, power of two <= 32
  const int c = tid / tpc, j = tid - c * tpc;
  float acc = 0.f;
  if (c < tch) {
    const float half_range = (float)(1 << (BITS - 1));
    for (int gq = j; gq < NQ; gq += tpc) {
      const float ws = bl::to_f32(sraw[c * NQ + gq]);
      const int32_t* pr = psm + gq * pstride + c * BITS;
      float v = 0.f;
#pragma unroll
      for (int i = 0; i < BITS; i++) {
        float t;
        if (MODE == BITLUT_TABLE_Q8)
          t = __fmul_rn(__fmul_rn(__fmul_rn(0.5f * (float)(1 << i), tsm[gq]), ws), __int2float_rn(pr[i]));
        else
          t = __fmul_rn(__fmul_rn(0.5f * (float)(1 << i), ws), __int_as_float(pr[i]));
        v = __fadd_rn(v, t);
      }
      float corr = __fmul_rn(-0.5f, ws);
      if (p.zeros) corr = __fadd_rn(corr, __fmul_rn(ws, __fsub_rn(half_range, bl::to_f32(zraw[c * NQ + gq]))));
      v = __fadd_rn(v, __fmul_rn(corr, rsm[gq]));
      acc = __fadd_rn(acc, v);
    }
  }
  for (int o = tpc / 2; o >= 1; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (c < tch && j == 0) p.out[(int64_t)row * L.m + (int64_t)tile * tch + c] = acc;
  if (MODE == BITLUT_TABLE_Q8 && p.partials) {
    for (int idx = tid; idx < tch * NQ * BITS; idx += T) {
      const int gq = idx % NQ, ci = idx / NQ, cc = ci / BITS, i = ci - cc * BITS;
      p.partials[(((int64_t)row * BITS + i) * L.m + (int64_t)tile * tch + cc) * NQ + gq] =
          psm[gq * pstride + cc * BITS + i];
    }
  }
}

// Register epilogue (fast mode, int8 tables, 32-stream tiles): right after
// the transpose-reduce a lane holds NF packed stream pairs of ONE quant
// group.  It splits them, combines the bit planes of each channel in exact
// integer arithmetic (S = sum_p 2^p P_p, |S| < 2^24 so f32(S) is exact) and
// writes one float per (group, channel):
//     y = ws * (ts*S - rs [+ 2(2^(b-1) - z) rs])
// so out = 0.5 * sum_g y, reduced in a fixed order by reg_final.  The int32
// staging values are the exact ones; only the float combination differs
// from the reference's order (last bits, tolerance-tested).
// Stream pair i = streams (2i, 2i+1), streams channel-major (c*bits + p).
template <int BITS, int NF, typename ST>
__device__ __forceinline__ void reg_terms(const GemvArgs& p, const int (&acc)[16], int fix, int base, int g,
                                          const ST* sraw, const ST* zraw, const float* tsm, const float* rsm,
                                          float* ysm, int ystride, int NQ) {
  constexpr int NCH = BITS == 1 ? 2 * NF : (BITS == 2 ? NF : NF / 2);
  int S[NCH];
#pragma unroll
  for (int i = 0; i < NF; i++) {
    const int v = acc[i] + fix;
    const int pe = (v << 17) >> 17;
    const int po = (v - pe) >> 15;
    if (BITS == 1) { S[2 * i] = pe; S[2 * i + 1] = po; }
    else if (BITS == 2) { S[i] = pe + 2 * po; }
    else { if (i & 1) S[i >> 1] += 4 * (pe + 2 * po); else S[i >> 1] = pe + 2 * po; }
  }
  const int ch0 = BITS == 1 ? 2 * base : (BITS == 2 ? base : base / 2);
  const float ts = tsm[g], rs = rsm[g];
  const float h2 = (float)(2 << (BITS - 1));            // 2 * 2^(b-1)
  float y[NCH];
#pragma unroll
  for (int j = 0; j < NCH; j++) {
    const int c = ch0 + j;
    const float ws = bl::to_f32(sraw[c * NQ + g]);
    float t = fmaf(ts, (float)S[j], -rs);
    if (p.zeros) t = fmaf(fmaf(-2.f, bl::to_f32(zraw[c * NQ + g]), h2), rs, t);
    y[j] = ws * t;
  }
  float* dst = ysm + g * ystride + ch0;
  if constexpr (NCH % 4 == 0) {
#pragma unroll
    for (int j = 0; j < NCH; j += 4)
      *reinterpret_cast<float4*>(dst + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
  } else if constexpr (NCH % 2 == 0) {
#pragma unroll
    for (int j = 0; j < NCH; j += 2) *reinterpret_cast<float2*>(dst + j) = make_float2(y[j], y[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < NCH; j++) dst[j] = y[j];
  }
}

// out[c] = 0.5 * sum_g y[g][c]: tpc threads per channel, strided partial
// sums then a shuffle tree (fixed order -> deterministic).
__device__ __forceinline__ void reg_final(const GemvArgs& p, const float* ysm, int ystride, int row, int tile) {
  const bl::LayoutV2& L = p.L;
  const int tch = L.tile_ch, NQ = L.NQ, T = blockDim.x, tid = threadIdx.x;
  int tpc = 32;
  while (tpc * tch > T) tpc >>= 1;
  const int c = tid / tpc, j = tid - c * tpc;
  float acc = 0.f;
  if (c < tch)
    for (int g = j; g < NQ; g += tpc) acc += ysm[g * ystride + c];
  for (int o = tpc / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (c < tch && j == 0) p.out[(int64_t)row * L.m + (int64_t)tile * tch + c] = 0.5f * acc;
}

// Issue this thread's first-round table loads (Q8 kernel-format tables)
// into registers right after the dependency is met, so they overlap the
// row-vector loads and the weight-arrival wait instead of following them.
template <int R>
__device__ __forceinline__ void prefetch_tables_q8(const GemvArgs& p, int row, uint4 (&tq)[R / 2]) {
  const bl::LayoutV2& L = p.L;
  const int u = threadIdx.x;
  if (u < L.n_sg * L.U) {
    const int uu = u % L.U, ub = uu >> 5, l = uu & 31;
    const int nu_b = min(32, L.U - 32 * ub);
    const int stride = nu_b == 32 ? 512 : nu_b * 16;
    const uint8_t* tb = p.qtab + (int64_t)row * L.KG * 8 + (int64_t)ub * (32 * R * 8) + l * 16;
#pragma unroll
    for (int jp = 0; jp < R / 2; jp++) tq[jp] = bl::ld_cg_128(tb + jp * stride);
  }
}

// Left-to-right chains of the epilogue products, one per channel, each kind
// in its own warp (warp 0: main sum, warp 1: bias, warp 2: zero points),
// then out[c] = main - 0.5 * bias (+ zero term) -- the reference's fp32
// order (_kernels.py:179-191).  All threads of the CTA must call it.
__device__ __forceinline__ void chains_and_out(const bl::LayoutV2& L, const float* terms, float* fin, int rowlen,
                                               bool has_zeros, float* out) {
  const int tid = threadIdx.x;
  const int tch = L.tile_ch, NQ = L.NQ, bits = L.bits;
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
    out[tid] = o;
  }
}

// Phases 3-5 of one (tile, row): lookups -> exact staging values ->
// epilogue products -> left-to-right chains -> out.  Requires the tile's
// weights (TMA variant) and scales in `smem`, tsm / rsm filled, and a
// __syncthreads() before the call.  Shared by the per-call kernel (gemv.cu)
// and the persistent pipeline (pipeline.cu).  Tables are read with
// ld.global.cg (L2, coherent): in the pipeline they are written by other
// CTAs of the same launch.
template <int R, int LG, typename ST, bool TMA, int MODE>
__device__ __forceinline__ void tile_body(const GemvArgs& p, int tile, int row, const SmemPlan& sp,
                                          uint8_t* smem, const uint4 (&tq0)[R / 2]) {
  const bl::LayoutV2& L = p.L;
  constexpr int NF = 16 / LG;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int T = blockDim.x;
  const int KG = L.KG, NQ = L.NQ, U = L.U;
  const int units = L.n_sg * U;
  const int tch = L.tile_ch;
  const int bits = L.bits;
  const bool has_zeros = p.zeros != nullptr;
  uint8_t* wbuf = smem;
  float* terms = reinterpret_cast<float*>(smem + sp.terms_off);   // after the lookups
  int32_t* psm = reinterpret_cast<int32_t*>(smem + sp.p_off);
  const int pstride = 32 * L.n_sg + 1;
  const ST* sraw = reinterpret_cast<const ST*>(smem + sp.s_off);
  const ST* zraw = reinterpret_cast<const ST*>(smem + sp.z_off);
  float* tsm = reinterpret_cast<float*>(smem + sp.t_off);
  float* rsm = reinterpret_cast<float*>(smem + sp.r_off);
  float* fin = reinterpret_cast<float*>(smem + sp.f_off);
  // ---- 3. lookups, reduction, exact staging values -> psm[gq][stream] ----
  const int rowlen = sp.rowlen;
  const int rounds = (units + T - 1) / T;
  // fast mode without partials on 32-stream tiles: epilogue from registers
  const bool regepi = MODE == BITLUT_TABLE_Q8 && p.fast && !p.partials && L.n_sg == 1 &&
                      (NF >= 2 || bits < 4);
  const int ystride = tch + 4;          // floats per group row of y (16 B aligned, spreads banks)
  float* ysm = reinterpret_cast<float*>(psm);
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
        if (rd == 0) {                  // round 0: tables already in flight (prefetch_tables_q8)
#pragma unroll
          for (int jp = 0; jp < R / 2; jp++) tq[jp] = tq0[jp];
        } else {
#pragma unroll
          for (int jp = 0; jp < R / 2; jp++) tq[jp] = bl::ld_cg_128(tb + jp * stride);
        }
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
      if (regepi) {
        if (live) {
          const int fix = 0;                  // lookup_kg sums are exact
          const int g = uu / LG;
          switch (bits) {
            case 1: reg_terms<1, NF, ST>(p, acc, fix, base, g, sraw, zraw, tsm, rsm, ysm, ystride, NQ); break;
            case 2: reg_terms<2, NF, ST>(p, acc, fix, base, g, sraw, zraw, tsm, rsm, ysm, ystride, NQ); break;
            default:
              if constexpr (NF >= 2) reg_terms<4, NF, ST>(p, acc, fix, base, g, sraw, zraw, tsm, rsm, ysm, ystride, NQ);
              break;
          }
        }
      } else if (live) {
        // undo the -1 per lookup of both streams, split each pair
        // split each packed pair v = P_even + 32768 P_odd (|P| < 16384)
        int32_t* dst = psm + (size_t)(uu / LG) * pstride + sg * 32 + 2 * base;
#pragma unroll
        for (int i = 0; i < NF; i++) {
          const int v = acc[i];
          const int pe = (v << 17) >> 17;
          dst[2 * i] = pe;
          dst[2 * i + 1] = (v - pe) >> 15;
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
          const uint4 t = bl::ld_cg_128(tb + j * nu_b * 16);
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
  if (regepi) {
    reg_final(p, ysm, ystride, row, tile);
    return;
  }
  if (p.fast) {
    switch (bits) {
      case 1: fast_epilogue<1, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, tid, T, row, tile); break;
      case 2: fast_epilogue<2, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, tid, T, row, tile); break;
      case 3: fast_epilogue<3, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, tid, T, row, tile); break;
      default: fast_epilogue<4, MODE, ST>(p, sraw, zraw, tsm, rsm, psm, tid, T, row, tile); break;
    }
    return;
  }

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

  // ---- 5. left-to-right chains, one per channel ----
  chains_and_out(L, terms, fin, rowlen, has_zeros, p.out + (int64_t)row * L.m + (int64_t)tile * tch);
}

}  // namespace blk
