// The batch executor's lookup kernel: any number of independent batch-1
// mpGEMV calls of one K (a layer set), each with its own int8 tables, in ONE
// launch (bitlut_mpgemv_batch; replaces that many kernel.py:374-382 mpgemv
// calls, fast epilogue).
//
// Work split: the matrices' tiles (tile = 32/b channels x all K, contiguous
// in layout v2) are numbered matrix after matrix; CTA b streams the
// contiguous range [b*T/G, (b+1)*T/G), so every CTA gets the same number of
// tiles and the launch has one tail.  Per tile: one TMA bulk copy of the
// weights (+ the tile's fp16 group scales / zero points) into a 1-2 stage
// ring (mbarrier completion, L2 evict_first), thread u looks up unit u
// (R k-groups) with the plane-merged prmt/dp4a core of b1_core.cuh against
// its register-resident tables, the unit sums are reduced over the lanes of
// a quantization group (exact int32 S = sum_p 2^p P_p), scaled per
// (channel, group) in registers, reduced over the groups of the warp by
// shuffles and over the warps in a fixed order through shared memory.
//
// Weight encodings (template MODE, bitlut_b200.h BITLUT_W_*), per
// (channel, group) term t and output y = f * sum_g t:
//   OFFSET   t = ws (ts S - rs)                     f = 1/2   (reference)
//   ZEROS    t = ws ((2^b - 2z) rs + ts S - rs)     f = 1/2
//   SIGN     t = ws ts S                            f = 1
//   TERNARY  t = ts S + rs                          f = s_t / 2
// (_kernels.py:179-191 is OFFSET in the reference's order; ZEROS adds
// 2 (2^(b-1) - z) rs per group; SIGN, w = s (2q - 1), is ZEROS at b = 1
// with scale 2s and z = 1/2, where the row-sum terms cancel; TERNARY,
// w = s_t (q - 1), is ZEROS at b = 2, z = 1 with one scale per tensor, so
// the tile carries no scale stream at all.)
//
// Per tile the CTA-wide barrier publishes the cross-warp sums and frees the
// stage; thread 0 refills it and warp 0 adds the cross-warp sums.  Measured
// and not kept (same-box A/B, 32-layer 7B layer sets):
// rotating the refill and the final sums over the warps (-3 %); a producer
// warp with full/empty mbarriers instead of the CTA barrier (-2..-10 %: the
// extra warp costs a CTA per SM); a leader warp waiting on an "empty"
// mbarrier while the others run ahead (-1 %); the integer lane reduction
// through shared memory (W1 -2 %); two units per thread (-2..-5 %: half the
// resident warps).  The kernel is issue-bound at ~2.6 (W2) / ~3.0 (W1)
// warp-instructions per 4-weight lookup.
#include "b1_core.cuh"

#include <cstdlib>

namespace {

using namespace blk;

constexpr int kStagesMax = 2;
constexpr int kYBufs = 2;             // cross-warp sum buffers (power of two)
// Per-tile duties after the CTA barrier: thread kRefillThread refills the
// consumed stage, warp kSumWarp adds the cross-warp sums.  On different warps
// neither delays the other's arrival at the next barrier (same-box A/B over
// thread 0/32/64 x warp 0/1/2: refill on warp 0, sums on warp 1 is +1.1..1.5 %
// on the W2 / W1 / ternary layer sets; macros for further A/Bs).
#ifndef BITLUT_REFILL_THREAD
#define BITLUT_REFILL_THREAD 0
#endif
constexpr int kRefillThread = BITLUT_REFILL_THREAD;   // (a thread's own issue cursor: advance() catches up)
#ifndef BITLUT_SUM_WARP
#define BITLUT_SUM_WARP 1
#endif
constexpr int kSumWarp = BITLUT_SUM_WARP;

struct BatchArgs {
  bl::LayoutV2 L;             // the launch's k, bits, group size (m unused)
  int independent;            // BITLUT_FLAG_INDEPENDENT
  int stages;                 // 1 or 2
  uint32_t stage_bytes, w_bytes, s_off, s_bytes, z_off;
  uint32_t y_off, bar_off;
};

__host__ __device__ inline uint32_t al16(size_t x) { return (uint32_t)((x + 15) & ~(size_t)15); }



// The issuing thread keeps the current matrix's operand pointers in registers
// (reloaded at a matrix change only): the per-tile refill, which sits between
// the CTA barrier and the thread's own lookups, reads no descriptor memory.
struct IssuePtrs {
  const uint8_t* w;
  const uint8_t* s;
  const uint8_t* z;
};
__device__ __forceinline__ IssuePtrs issue_ptrs(const bitlut_batch_mat& mt) {
  return {mt.wgpu, reinterpret_cast<const uint8_t*>(mt.wscales), reinterpret_cast<const uint8_t*>(mt.zeros)};
}

template <typename ST, int MODE>
__device__ __forceinline__ void issue_tile(const BatchArgs& a, const IssuePtrs& mt, int local, uint8_t* sb,
                                           uint64_t* bar, uint64_t pol) {
  const bl::LayoutV2& L = a.L;
  const uint32_t s_bytes = MODE == BITLUT_W_TERNARY ? 0u : a.s_bytes;
  mbar_expect_tx(bar, a.w_bytes + s_bytes * (MODE == BITLUT_W_ZEROS ? 2u : 1u));
  const uint8_t* src = mt.w + (int64_t)local * L.KG * 16;
  for (uint32_t off = 0; off < a.w_bytes; off += 32768u) {
    const uint32_t nb = a.w_bytes - off < 32768u ? a.w_bytes - off : 32768u;
    bulk_g2s(sb + off, src + off, nb, bar, pol);
  }
  if constexpr (MODE != BITLUT_W_TERNARY) {
    const int64_t b0 = (int64_t)local * s_bytes;        // layer-set layout: s_bytes per tile
    bulk_g2s(sb + a.s_off, mt.s + b0, s_bytes, bar, pol);
    if constexpr (MODE == BITLUT_W_ZEROS) bulk_g2s(sb + a.z_off, mt.z + b0, s_bytes, bar, pol);
  }
}

// matrix cursor: advance (j, begin, end) until tile t < end (bounded by the
// descriptor count: a tile number past the last matrix stays on it)
__device__ __forceinline__ void advance(const bitlut_batch_mat* dm, int n_mats, int t, int& j, int& jb, int& je) {
  while (t >= je && j + 1 < n_mats) {
    j++;
    jb = je;
    je = dm[j].tile_end;
  }
}

template <int R, int LG, int BITS, typename ST, int MODE, bool PART>
__global__ void __launch_bounds__(384) gemv_batch_kernel(const __grid_constant__ BatchArgs a,
                                                         const bitlut_batch_mat* __restrict__ dm, int n_mats) {
  const bl::LayoutV2& L = a.L;
  constexpr int TCH = 32 / BITS;
  constexpr int NACC = BITS == 4 ? 8 : 16;
  constexpr int NV = reduced_count<NACC, 1, LG>();
  constexpr int NCH = BITS == 1 ? 2 * NV : NV;
  constexpr int NF = reduced_count<NCH, LG, 32>();
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x >> 5;
  const int NQ = L.NQ, U = L.U;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  float* ysm = reinterpret_cast<float*>(smem + a.y_off);
  const int S = a.stages;
  // the tile count is the descriptors' own (not a host-side copy)
  const int T = dm[n_mats - 1].tile_end, G = gridDim.x;
  const int t0 = (int)((int64_t)blockIdx.x * T / G), t1 = (int)((int64_t)(blockIdx.x + 1) * T / G);
  // matrix holding t0 = number of matrices ending at or before it
  int j0 = 0;
  for (int base = 0; base < n_mats; base += blockDim.x) {
    const int i = base + tid;
    j0 += __syncthreads_count(i < n_mats && dm[i].tile_end <= t0);
  }
  if (j0 >= n_mats) j0 = n_mats - 1;
  if (t0 >= t1) {                                       // more CTAs than tiles
    if (!a.independent) bl::pdl_wait();
    bl::pdl_launch_dependents();
    if (a.independent) bl::pdl_wait();
    return;
  }
  // consumer cursor (every thread): the matrix of the current tile
  int jc = j0, jc_begin = j0 ? dm[j0 - 1].tile_end : 0, jc_end = dm[j0].tile_end;
  // issue cursor (thread 0): the matrix of the next tile to stage
  int ji = jc, ji_begin = jc_begin, ji_end = jc_end;
  IssuePtrs ip = {nullptr, nullptr, nullptr};
  if (tid == kRefillThread) ip = issue_ptrs(dm[ji]);
  if (tid == 0) {
    for (int s = 0; s < kStagesMax; s++) {
      mbar_init(bar + s, 1);                            // the stage's TMA bytes landed
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t pol = policy_evict_first();
    static_assert(kRefillThread == 0, "the initial stages are issued by the refill thread");
    for (int s = 0; s < S; s++) {
      const int t = t0 + s;
      if (t >= t1) break;
      if (t >= ji_end) {
        advance(dm, n_mats, t, ji, ji_begin, ji_end);
        ip = issue_ptrs(dm[ji]);
      }
      issue_tile<ST, MODE>(a, ip, t - ji_begin, smem + s * a.stage_bytes, bar + s, pol);
    }
  }
  const uint64_t pol = policy_evict_first();
  if (!a.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  // thread u looks up unit u; a thread past the last unit (U is not a
  // multiple of 32) shadows the last unit with all-zero tables, so it adds
  // exact zeros everywhere and the tile loop needs no "live" branches
  const bool live = tid < U;
  const int u = live ? tid : U - 1;
  const int ub = u >> 5, l = u & 31;
  const int nu_b = min(32, U - 32 * ub);
  const int g = u / LG;
  float* outp = nullptr;
  int32_t* part = nullptr;                              // PART: exact integer sums, (m, NQ)
  uint4 tq[R / 2];
  float ts = 0.f, rs = 0.f, fin = MODE == BITLUT_W_SIGN ? 1.f : 0.5f;
  auto load_matrix = [&](const bitlut_batch_mat& mt) {
    outp = mt.out;
    if constexpr (PART) part = mt.partials;
    if constexpr (MODE == BITLUT_W_TERNARY) fin = 0.5f * bl::to_f32(*reinterpret_cast<const ST*>(mt.wscales));
    const uint8_t* tb = reinterpret_cast<const uint8_t*>(mt.tables) + (int64_t)ub * (32 * R * 8) + l * 16;
#pragma unroll
    for (int jp = 0; jp < R / 2; jp++) tq[jp] = live ? bl::ld_cg_128(tb + jp * nu_b * 16) : make_uint4(0, 0, 0, 0);
    ts = live ? bl::ld_cg_f32(mt.tscales + g) : 0.f;
    rs = live ? bl::ld_cg_f32(mt.rowsums + g) : 0.f;
  };
  load_matrix(dm[jc]);
  const uint32_t woff = (uint32_t)(ub * (32 * R * 16) + l * 16);
  const int stride = nu_b == 32 ? 512 : nu_b * 16;
  // layer-set layout: value j of this lane is channel j ^ cmask; the unit's
  // NCH scales (zero points) are contiguous at unit * NCH
  const int cmask = perm_mask<TCH>(lane);
  const uint32_t soff = a.s_off + (uint32_t)u * (NCH * (uint32_t)sizeof(ST));
  const uint32_t zoff = a.z_off + (uint32_t)u * (NCH * (uint32_t)sizeof(ST));
  BL_CHECK(MODE == BITLUT_W_TERNARY || (u + 1) * NCH * (int)sizeof(ST) <= (int)a.s_bytes);
  BL_CHECK(a.bar_off + 8u * kStagesMax <= bl::dyn_smem_bytes());
  BL_CHECK(woff + (R - 1) * stride + 16 <= a.w_bytes);
  __syncthreads();                                      // barriers initialised
  int it = 0;
  for (int tile = t0; tile < t1; tile++, it++) {
    if (tile >= jc_end) {                               // next matrix: its tables and output
      advance(dm, n_mats, tile, jc, jc_begin, jc_end);
      load_matrix(dm[jc]);
    }
    const int stage = S == 1 ? 0 : (it & 1);
    uint8_t* sb = smem + stage * a.stage_bytes;
    mbar_wait(bar + stage, (S == 1 ? it : it >> 1) & 1);
    int acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = 0;
    {
      const uint8_t* wsrc = sb + woff;
#pragma unroll
      for (int j = 0; j < R; j += 2) {
        const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
        const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
        lookup_kg_merged<BITS, NACC>(wa, tq[j >> 1].x, tq[j >> 1].y, acc);
        lookup_kg_merged<BITS, NACC>(wc, tq[j >> 1].z, tq[j >> 1].w, acc);
      }
    }
    reduce_lanes_perm<NACC, 1, LG>(acc);                // exact integer sums of the quantization group
    const int local = tile - jc_begin;
    BL_CHECK(jc < n_mats && local >= 0 && (local + 1) * TCH <= dm[jc].m);
    float y[NCH];
    {
      int Sv[NCH];
      if constexpr (BITS == 1) {
#pragma unroll
        for (int i = 0; i < NV; i++) {
          const int v = acc[i];
          const int pe = (v << 17) >> 17;
          Sv[2 * i] = pe;
          Sv[2 * i + 1] = (v - pe) >> 15;
        }
      } else {
#pragma unroll
        for (int i = 0; i < NV; i++) Sv[i] = acc[i];
      }
      if (PART && live) {                               // exact integer sums (parity tests)
#pragma unroll
        for (int j = 0; j < NCH; j++)                   // value j of this lane = channel j ^ cmask
          part[((int64_t)local * TCH + (j ^ cmask)) * NQ + g] = Sv[j];
      }
      // the lane's NCH scales (+ zero points) are one vector in the layer-set
      // layout; __fmul_rn: the products must not contract into the first add
      // of the reduction (outputs stay bitwise those of the per-call lookups)
      constexpr int SB = NCH * (int)sizeof(ST);
      uint32_t sv[(SB + 3) / 4];
      if constexpr (MODE != BITLUT_W_TERNARY) lds_vec<SB>(sb + soff, sv);
      if constexpr (MODE == BITLUT_W_OFFSET) {
#pragma unroll
        for (int j = 0; j < NCH; j++) y[j] = __fmul_rn(vec_elem<ST>(sv, j), fmaf(ts, (float)Sv[j], -rs));
      } else if constexpr (MODE == BITLUT_W_ZEROS) {
        uint32_t zv[(SB + 3) / 4];
        lds_vec<SB>(sb + zoff, zv);
        const float h2 = (float)(2 << (BITS - 1));
#pragma unroll
        for (int j = 0; j < NCH; j++)
          y[j] = __fmul_rn(vec_elem<ST>(sv, j),
                           fmaf(fmaf(-2.f, vec_elem<ST>(zv, j), h2), rs, fmaf(ts, (float)Sv[j], -rs)));
      } else if constexpr (MODE == BITLUT_W_SIGN) {
#pragma unroll
        for (int j = 0; j < NCH; j++) y[j] = __fmul_rn(vec_elem<ST>(sv, j), __fmul_rn(ts, (float)Sv[j]));
      } else {
#pragma unroll
        for (int j = 0; j < NCH; j++) y[j] = fmaf(ts, (float)Sv[j], rs);
      }
    }
    reduce_lanes_perm<NCH, LG, 32>(y);                  // over the groups of the warp: y[0] = channel cmask
    static_assert(NF == 1, "one channel sum per lane");
    ysm[(it & (kYBufs - 1)) * NW * TCH + warp * TCH + cmask] = y[0];
    __syncthreads();                                    // stage consumed, ysm complete
    if (tid == kRefillThread) {                         // refill the consumed stage
      const int t = tile + S;
      if (t < t1) {
        if (t >= ji_end) {
          advance(dm, n_mats, t, ji, ji_begin, ji_end);
          ip = issue_ptrs(dm[ji]);
        }
        issue_tile<ST, MODE>(a, ip, t - ji_begin, sb, bar + stage, pol);
      }
    }
    if (tid >= kSumWarp * 32 && tid < kSumWarp * 32 + TCH) {   // fixed warp order: deterministic
      const int c = tid - kSumWarp * 32;
      const float* yr = ysm + (it & (kYBufs - 1)) * NW * TCH + c;
      float s = 0.f;
      for (int w = 0; w < NW; w++) s += yr[w * TCH];
      outp[(int64_t)local * TCH + c] = fin * s;
    }
  }
  if (a.independent) bl::pdl_wait();
}

// ---------------------------------------------------------------- host side

int device_sms(int dev) {
  static int n[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

template <int R, int LG, int BITS, typename ST, int MODE, bool PART>
int launch(const bl::LayoutV2& L, const bitlut_batch_mat* dm, int n_mats, int total_tiles, bool independent,
           bool pdl, cudaStream_t stream) {
  if (L.U > 384) return BITLUT_ELAYOUT;
  int T = (L.U + 31) & ~31;                             // one thread per unit
  if (T < 128) T = 128;
  const int NW = T / 32;
  constexpr int TCH = 32 / BITS;
  auto kern = gemv_batch_kernel<R, LG, BITS, ST, MODE, PART>;
  int dev = 0;
  cudaGetDevice(&dev);
  static bool configured[64] = {false};                // per device (attributes are per device)
  if (dev < 0 || dev >= 64) return BITLUT_EINTERNAL;
  if (!configured[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return BITLUT_EINTERNAL;
    configured[dev] = true;
  }
  BatchArgs a;
  a.L = L;
  a.independent = independent ? 1 : 0;
  a.w_bytes = (uint32_t)((size_t)L.KG * 16);
  constexpr int NV = reduced_count<BITS == 4 ? 8 : 16, 1, LG>();
  constexpr int NCH = BITS == 1 ? 2 * NV : NV;
  a.s_bytes = MODE == BITLUT_W_TERNARY ? 0u : (uint32_t)((size_t)L.U * NCH * sizeof(ST));
  if (a.s_bytes != (uint32_t)bl::layer_set_scale_bytes(L, (int)sizeof(ST)) && MODE != BITLUT_W_TERNARY)
    return BITLUT_EINTERNAL;
  a.s_off = al16(a.w_bytes);
  a.z_off = a.s_off + al16(a.s_bytes);
  a.stage_bytes = a.z_off + (MODE == BITLUT_W_ZEROS ? al16(a.s_bytes) : 0u);
  a.stage_bytes = (a.stage_bytes + 127) & ~127u;
  auto total_for = [&](int stages) {
    const uint32_t y_off = stages * a.stage_bytes;
    const uint32_t bar_off = y_off + al16((size_t)kYBufs * NW * TCH * 4);
    return bar_off + 8u * kStagesMax;
  };
  static int st_env = -1;
  if (st_env < 0) {
    const char* e = getenv("BITLUT_BATCH_STAGES");       // diagnostic: force 1 or 2
    st_env = e ? atoi(e) : 0;
  }
  int per_sm2 = 0, per_sm1 = 0;
  if (total_for(2) > 227 * 1024 ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, kern, T, total_for(2)) != cudaSuccess)
    per_sm2 = 0;
  if (total_for(1) > 227 * 1024 ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm1, kern, T, total_for(1)) != cudaSuccess)
    per_sm1 = 0;
  // two stages, or one when double buffering leaves <= 2 CTAs per SM and a
  // single stage fits twice as many (long K)
  int best_s = 2, best_per = per_sm2;
  if (st_env == 1 || (st_env == 0 && per_sm2 <= 2 && per_sm1 >= 2 * per_sm2) || per_sm2 < 1) {
    best_s = 1;
    best_per = per_sm1;
  }
  if (best_per < 1) return BITLUT_ELAYOUT;
  a.stages = best_s;
  a.y_off = best_s * a.stage_bytes;
  a.bar_off = a.y_off + al16((size_t)kYBufs * NW * TCH * 4);
  int grid = device_sms(dev) * best_per;
  if (grid > total_tiles) grid = total_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = total_for(best_s);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, dm, n_mats) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

template <int R, int LG, int BITS, typename ST, int MODE>
int by_part(const bl::LayoutV2& L, const bitlut_batch_mat* dm, int n, int tt, bool ind, bool pdl, cudaStream_t s,
            bool part) {
  return part ? launch<R, LG, BITS, ST, MODE, true>(L, dm, n, tt, ind, pdl, s)
              : launch<R, LG, BITS, ST, MODE, false>(L, dm, n, tt, ind, pdl, s);
}

template <int R, int LG, int BITS>
int by_mode(const bl::LayoutV2& L, const bitlut_batch_mat* dm, int n, int tt, bool ind, bool pdl, cudaStream_t s,
            int sdt, int mode, bool part) {
  const bool f16 = sdt == BITLUT_DT_F16;
  switch (mode) {
    case BITLUT_W_OFFSET:
      return f16 ? by_part<R, LG, BITS, __half, BITLUT_W_OFFSET>(L, dm, n, tt, ind, pdl, s, part)
                 : by_part<R, LG, BITS, float, BITLUT_W_OFFSET>(L, dm, n, tt, ind, pdl, s, part);
    case BITLUT_W_ZEROS:
      return f16 ? by_part<R, LG, BITS, __half, BITLUT_W_ZEROS>(L, dm, n, tt, ind, pdl, s, part)
                 : by_part<R, LG, BITS, float, BITLUT_W_ZEROS>(L, dm, n, tt, ind, pdl, s, part);
    case BITLUT_W_SIGN:
      if constexpr (BITS == 1)
        return f16 ? by_part<R, LG, BITS, __half, BITLUT_W_SIGN>(L, dm, n, tt, ind, pdl, s, part)
                   : by_part<R, LG, BITS, float, BITLUT_W_SIGN>(L, dm, n, tt, ind, pdl, s, part);
      return BITLUT_EPARAM;
    case BITLUT_W_TERNARY:
      if constexpr (BITS == 2)
        return f16 ? by_part<R, LG, BITS, __half, BITLUT_W_TERNARY>(L, dm, n, tt, ind, pdl, s, part)
                   : by_part<R, LG, BITS, float, BITLUT_W_TERNARY>(L, dm, n, tt, ind, pdl, s, part);
      return BITLUT_EPARAM;
  }
  return BITLUT_EPARAM;
}

template <int R, int LG>
int by_bits(const bl::LayoutV2& L, const bitlut_batch_mat* dm, int n, int tt, bool ind, bool pdl, cudaStream_t s,
            int sdt, int mode, bool part) {
  switch (L.bits) {
    case 1: return by_mode<R, LG, 1>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
    case 2: return by_mode<R, LG, 2>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
    case 4: return by_mode<R, LG, 4>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
  }
  return BITLUT_ELAYOUT;
}

int dispatch(const bl::LayoutV2& L, const bitlut_batch_mat* dm, int n, int tt, bool ind, bool pdl, cudaStream_t s,
             int sdt, int mode, bool part) {
  if (L.R == 8) {
    switch (L.Lg) {
      case 1: return by_bits<8, 1>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
      case 2: return by_bits<8, 2>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
      case 4: return by_bits<8, 4>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
      case 8: return by_bits<8, 8>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
      case 16: return by_bits<8, 16>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
    }
  } else if (L.R == 4 && L.Lg == 1) {
    return by_bits<4, 1>(L, dm, n, tt, ind, pdl, s, sdt, mode, part);
  }
  return BITLUT_ELAYOUT;
}

bool mode_ok(int mode, int bits) {
  switch (mode) {
    case BITLUT_W_OFFSET:
    case BITLUT_W_ZEROS: return true;
    case BITLUT_W_SIGN: return bits == 1;
    case BITLUT_W_TERNARY: return bits == 2;
  }
  return false;
}

}  // namespace

// Host-side check and tile numbering of a batched launch (see the header).
extern "C" int bitlut_mpgemv_batch_encode(bitlut_batch_mat* mats, int n_mats, int k, int bits, int group_size,
                                          int weight_mode, int* total_tiles) {
  if (!mats || n_mats < 1 || !total_tiles) return BITLUT_EPARAM;
  if (!mode_ok(weight_mode, bits)) return BITLUT_EPARAM;
  int64_t tiles = 0;
  int n_part = 0;
  for (int j = 0; j < n_mats; j++) {
    bl::LayoutV2 L;
    const int rc = bl::make_layout(mats[j].m, k, bits, group_size, &L);
    if (rc) return rc;
    if (!mats[j].wgpu || !mats[j].wscales || !mats[j].out || !mats[j].tables || !mats[j].tscales ||
        !mats[j].rowsums)
      return BITLUT_EPARAM;
    if ((weight_mode == BITLUT_W_ZEROS) != (mats[j].zeros != nullptr)) return BITLUT_EPARAM;
    n_part += mats[j].partials != nullptr;
    if (L.n_sg != 1 || L.bits == 3 || L.U > 384) return BITLUT_ELAYOUT;
    tiles += L.n_tiles;
    if (tiles > (int64_t)1 << 30) return BITLUT_ESHAPE;
    mats[j].tile_end = (int)tiles;
  }
  if (n_part != 0 && n_part != n_mats) return BITLUT_EPARAM;   // all or none
  *total_tiles = (int)tiles;
  return BITLUT_OK;
}

extern "C" int bitlut_mpgemv_batch(const bitlut_batch_mat* dev_mats, int n_mats, int total_tiles, int k, int bits,
                                   int group_size, int scale_dtype, int weight_mode, int flags, void* stream) {
  if (!dev_mats || n_mats < 1 || total_tiles < 1) return BITLUT_EPARAM;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (!(flags & BITLUT_FLAG_FAST_EPILOGUE)) return BITLUT_EPARAM;
  if (!mode_ok(weight_mode, bits)) return BITLUT_EPARAM;
  bl::LayoutV2 L;
  const int rc = bl::make_layout(32, k, bits, group_size, &L);
  if (rc) return rc;
  if (L.n_sg != 1 || L.bits == 3 || L.U > 384) return BITLUT_ELAYOUT;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  const bool independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  return dispatch(L, dev_mats, n_mats, total_tiles, independent, pdl, (cudaStream_t)stream, scale_dtype,
                  weight_mode, (flags & BITLUT_FLAG_COMBINED_PARTIALS) != 0);
}
