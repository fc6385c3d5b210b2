// Batch-1 lookup kernel for the decode path (fast epilogue, int8 tables,
// 1/2/4-bit weights): persistent CTAs that walk tiles with a 2-stage TMA
// pipeline, so the per-CTA setup (barriers, tables, table scales / row sums)
// is paid once and tile i+1's weights stream in while tile i is looked up.
//
// Per tile (tile_ch channels x bits planes = 32 streams, all k-groups):
//   lookups   the A/B prmt lookup of gemv.cu with the bit planes merged by
//             the dp2a multipliers instead of packed as independent streams:
//               W2  pair (c, p0 p1)           mult (1, 2)     -> S_c
//               W4  pairs (c, p0 p1)(c, p2 p3) mult (1,2),(4,8) -> S_c
//               W1  pair (c, c+1)             mult (1, -32768) (packed, split later)
//             so each accumulator already holds the exact integer
//             S = sum_p 2^p P_p of one channel (|S| < 2^24: exact in f32);
//   epilogue  y_c += ws_cg * (ts_g * S - rs_g [+ 2 (2^(b-1) - z) rs_g]) per
//             (channel, group) in registers, fixed-order shuffle + smem
//             reduction, out_c = 0.5 * sum.  Deterministic; the int32 sums
//             are exact, only the float combination order differs from the
//             reference (<= 1e-5 relative, tests/test_gpu_parity.py).
// The reference-order (bit-exact float) epilogue stays in gemv.cu.
#include "gemv_core.cuh"
#include "b1_core.cuh"

#include <cstdlib>


namespace {

using namespace blk;

constexpr int kMaxStages = 2;

constexpr int kMaxMats = 8;

// One weight matrix of a (multi-matrix) launch: matrices that share the
// activation tables (q/k/v, gate/up) are looked up by one launch whose tiles
// are numbered matrix after matrix.
struct B1Mat {
  const uint8_t* w;
  const void* wscales;
  const void* zeros;
  float* out;
  int tile_end;               // cumulative tile count up to and including this matrix
  const uint8_t* qtab;        // per-matrix tables (lean kernel, partitioned launch), or null
  const float* tscales;
  const float* rowsums;
};

struct B1Args {
  GemvArgs g;                 // L: the shared layout (k, bits, gs); tables, flags
  int n_mats, total_tiles;
  int n_rows, rows_per_cta;   // activation rows (mpGEMM): CTA y walks rows [y*rpc, y*rpc + rpc)
  B1Mat mats[kMaxMats];
  const __half* act;          // fused variant: fp16 activation row (tables built in-kernel)
  uint32_t sa_off, red_off;   // fused: activation staging (4*T floats) + group-max scratch
  uint32_t psm_off, terms_off, fin_off;   // exact variant: staging values, products, chain ends
  int rowlen;                 // exact: floats per channel row of products
  int rounds;                 // unit rounds per tile (units = KG / R)
  int stages;                 // weight pipeline depth: 1 (one tile per CTA) or 2
  int tab_smem;               // tables staged in smem (rounds > 1), else registers
  uint32_t stage_bytes;       // per pipeline stage: weights | scales | zeros
  uint32_t w_bytes, s_off, s_bytes, z_off;
  uint32_t tab_off, ts_off, rs_off, y_off, bar_off;
  GatherArgs gth;             // fused all-gather epilogue (fast kernel), n_peers == 0 otherwise
  int ldg_w;                  // fast kernel: weights loaded straight into registers (stage = scales only)
  int partition;              // lean kernel: CTAs [cta_begin[j], cta_begin[j+1]) serve matrix j only
  int cta_begin[kMaxMats + 1];
};

struct B1Plan {
  uint32_t stage_bytes, w_bytes, s_off, s_bytes, z_off, tab_off, ts_off, rs_off, y_off, sa_off, red_off,
      psm_off, terms_off, fin_off, bar_off, total;
  int rowlen;
};

// kFastRows / kExactRows: the mpGEMM instantiations (several activation rows
// per CTA); separate so the batch-1 kernels keep their register budget
enum B1Kind { kFast = 0, kFused = 1, kExact = 2, kFastRows = 3, kExactRows = 4 };
__host__ __device__ constexpr bool kind_exact(int k) { return k == kExact || k == kExactRows; }
__host__ __device__ constexpr bool kind_rows(int k) { return k == kFastRows || k == kExactRows; }

__host__ __device__ inline uint32_t al16(size_t x) { return (uint32_t)((x + 15) & ~(size_t)15); }

template <typename ST>
B1Plan b1_plan(const bl::LayoutV2& L, bool zeros, bool tab_smem, int T, int stages, int kind = kFast,
               bool ldg_w = false) {
  const bool fused = kind == kFused, exact = kind_exact(kind);
  B1Plan s;
  s.w_bytes = ldg_w ? 0u : (uint32_t)((size_t)L.KG * 16);
  s.s_bytes = (uint32_t)((size_t)L.tile_ch * L.NQ * sizeof(ST));
  s.s_off = al16(s.w_bytes);
  s.z_off = s.s_off + al16(s.s_bytes);
  s.stage_bytes = s.z_off + (zeros ? al16(s.s_bytes) : 0);
  s.stage_bytes = (s.stage_bytes + 127) & ~127u;
  s.tab_off = stages * s.stage_bytes;
  s.ts_off = s.tab_off + (tab_smem ? al16((size_t)L.KG * 8) : 0);
  s.rs_off = s.ts_off + al16((size_t)L.NQ * 4);
  s.y_off = s.rs_off + al16((size_t)L.NQ * 4);
  // cross-warp sums, double-buffered; the rows kernel stores two rows per buffer
  // (batch-1 plans stay as small as before: K = 4096 fits six CTAs per SM)
  s.sa_off = s.y_off + al16((size_t)(kind_rows(kind) ? 4 : 2) * (T / 32) * L.tile_ch * 4);
  s.red_off = s.sa_off + (fused ? al16((size_t)4 * T * 4) : 0);
  s.psm_off = s.red_off + (fused ? al16((size_t)(T / 32) * 4) : 0);
  // exact epilogue (reference order): staging values NQ x 33 int32, products
  // tile_ch x rowlen floats (rowlen/4 odd: conflict-free chain loads), chain ends
  const int need = (L.bits + 1 + (zeros ? 1 : 0)) * L.NQ;
  s.rowlen = ((need + 3) / 4) * 4;
  if (((s.rowlen / 4) & 1) == 0) s.rowlen += 4;
  s.terms_off = s.psm_off + (exact ? al16((size_t)L.NQ * 33 * 4) : 0);
  s.fin_off = s.terms_off + (exact ? al16((size_t)L.tile_ch * s.rowlen * 4) : 0);
  s.bar_off = s.fin_off + (exact ? al16((size_t)3 * 32 * 4) : 0);
  s.total = s.bar_off + 8 * (kMaxStages + 1);
  return s;
}

__device__ __forceinline__ int find_mat(const B1Args& a, int tile, int& local) {
  int j = 0;
  while (j + 1 < a.n_mats && tile >= a.mats[j].tile_end) j++;
  local = tile - (j ? a.mats[j - 1].tile_end : 0);
  return j;
}

template <typename ST>
__device__ __forceinline__ void issue_stage(const B1Args& a, int tile, uint8_t* sb, uint64_t* bar, uint64_t pol) {
  const bl::LayoutV2& L = a.g.L;
  int local;
  const B1Mat& mt = a.mats[find_mat(a, tile, local)];
  const bool zeros = mt.zeros != nullptr;
  mbar_expect_tx(bar, a.w_bytes + a.s_bytes * (zeros ? 2u : 1u));
  const uint8_t* src = mt.w + L.sg_row_base(local, 0);
  for (uint32_t off = 0; off < a.w_bytes; off += 32768u) {
    const uint32_t nb = a.w_bytes - off < 32768u ? a.w_bytes - off : 32768u;
    bulk_g2s(sb + off, src + off, nb, bar, pol);
  }
  const int64_t e0 = (int64_t)local * L.tile_ch * L.NQ;
  bulk_g2s(sb + a.s_off, reinterpret_cast<const ST*>(mt.wscales) + e0, a.s_bytes, bar, pol);
  if (zeros) bulk_g2s(sb + a.z_off, reinterpret_cast<const ST*>(mt.zeros) + e0, a.s_bytes, bar, pol);
}

// ---- fused table build (cluster-cooperative) ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store to the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void st_cluster_v2(const void* local, uint32_t rank, uint32_t x, uint32_t y) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" ::"r"(ra), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void st_cluster_f32(const void* local, uint32_t rank, float x) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(x) : "memory");
}

// Each CTA of the cluster builds the int8 tables, table scales and row sums
// of a slice of the quantization groups -- the arithmetic of lut_core.cuh
// lut_block, operation for operation, so the tables are bitwise those of
// bitlut_build_lut -- and stores them into the shared memory of EVERY CTA
// of the cluster (DSMEM).  Requires T % (gs/4) == 0.
template <int R>
__device__ __forceinline__ void fused_tables(const B1Args& a, uint8_t* smem) {
  const bl::LayoutV2& L = a.g.L;
  const int tid = threadIdx.x, T = blockDim.x;
  const int NQ = L.NQ, gs = L.gs, gpg = gs >> 2, U = L.U;
  const uint32_t rank = cluster_rank(), cs = cluster_size();
  const int gpr = (NQ + (int)cs - 1) / (int)cs;
  const int g0 = (int)rank * gpr, g1 = min(NQ, g0 + gpr);
  float* sa = reinterpret_cast<float*>(smem + a.sa_off);
  float* red = reinterpret_cast<float*>(smem + a.red_off);
  uint8_t* tab = smem + a.tab_off;
  float* tsm = reinterpret_cast<float*>(smem + a.ts_off);
  float* rsm = reinterpret_cast<float*>(smem + a.rs_off);
  bool waited = false;
  for (int kb = g0 * gpg; kb < g1 * gpg; kb += T) {
    const int kg = kb + tid;
    const bool live = kg < g1 * gpg;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (live) {
      uint2 r;
      asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(a.act + 4 * (int64_t)kg));
      const __half2 h0 = *reinterpret_cast<const __half2*>(&r.x), h1 = *reinterpret_cast<const __half2*>(&r.y);
      v[0] = __low2float(h0); v[1] = __high2float(h0); v[2] = __low2float(h1); v[3] = __high2float(h1);
    }
#pragma unroll
    for (int j = 0; j < 4; j++) sa[tid * 4 + j] = v[j];
    float e[8];
#pragma unroll
    for (int idx = 0; idx < 8; idx++) {
      float x = (idx & 1) ? v[0] : -v[0];
      x = (idx & 2) ? __fadd_rn(x, v[1]) : __fsub_rn(x, v[1]);
      x = (idx & 4) ? __fadd_rn(x, v[2]) : __fsub_rn(x, v[2]);
      e[idx] = __fsub_rn(x, v[3]);
    }
    float mx = 0.f;
#pragma unroll
    for (int idx = 0; idx < 8; idx++) mx = bl::fmax_nan(mx, fabsf(e[idx]));
    const int seg = gpg < 32 ? gpg : 32;
    for (int o = 1; o < seg; o <<= 1) mx = bl::fmax_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (gpg > 32) {
      if ((tid & 31) == 0) red[tid >> 5] = mx;
      __syncthreads();
      const int wpg = gpg >> 5;
      const int w0 = (tid >> 5) / wpg * wpg;
      mx = 0.f;
      for (int w = 0; w < wpg; w++) mx = bl::fmax_nan(mx, red[w0 + w]);
    }
    float scale = __fdiv_rn(mx, 127.0f);
    if (scale == 0.0f) scale = 1.0f;
    uint32_t packed[2] = {0u, 0u};
#pragma unroll
    for (int idx = 0; idx < 8; idx++) {
      const float q = __fdiv_rn(e[idx], scale);
      float r = truncf(__fadd_rn(q, copysignf(0.5f, q)));
      r = fminf(fmaxf(r, -127.f), 127.f);
      packed[idx >> 2] |= ((uint32_t)(int)r & 0xffu) << (8 * (idx & 3));
    }
    if (!waited) {                 // every CTA of the cluster is running: DSMEM is safe
      cluster_wait();
      waited = true;
    }
    if (live) {
      const uint32_t e0 = packed[0] - ((packed[0] >> 7) & 0x01010101u);
      const uint32_t e1 = packed[1] - ((packed[1] >> 7) & 0x01010101u);
      const int u = kg / R, r = kg - u * R, ub = u >> 5, l = u & 31;
      const int nu_b = min(32, U - 32 * ub);
      const uint8_t* dst = tab + ub * (32 * R * 8) + ((r >> 1) * nu_b + l) * 16 + (r & 1) * 8;
      for (uint32_t d = 0; d < cs; d++) st_cluster_v2(dst, d, e0, e1);
      if ((kg & (gpg - 1)) == 0)
        for (uint32_t d = 0; d < cs; d++) st_cluster_f32(tsm + kg / gpg, d, scale);
    }
    __syncthreads();               // sa complete
    if (live && (kg & (gpg - 1)) == 0) {
      const float4* s4 = reinterpret_cast<const float4*>(sa + tid * 4);
      float acc = 0.f;
      for (int q = 0; q < gs / 4; q++) {
        const float4 c = s4[q];
        acc = __fadd_rn(acc, c.x); acc = __fadd_rn(acc, c.y); acc = __fadd_rn(acc, c.z); acc = __fadd_rn(acc, c.w);
      }
      for (uint32_t d = 0; d < cs; d++) st_cluster_f32(rsm + kg / gpg, d, acc);
    }
    __syncthreads();               // sa / red reusable
  }
  if (!waited) cluster_wait();
  cluster_arrive_release();        // this CTA's slice is in every CTA's smem
  cluster_wait();                  // ... and every other slice is in ours
}

template <int R, int LG, int BITS, typename ST, int KIND>
__global__ void __launch_bounds__(384) gemv_b1_kernel(const __grid_constant__ B1Args a) {
  constexpr bool FUSED = KIND == kFused, EXACT = kind_exact(KIND), ROWS = kind_rows(KIND);
  const GemvArgs& p = a.g;
  const bl::LayoutV2& L = p.L;
  constexpr int TCH = 32 / BITS;                        // channels per tile
  constexpr int NACC = BITS == 4 ? 8 : 16;              // int accumulators per lane
  constexpr int NV = reduced_count<NACC, 1, LG>();      // after the in-group reduction
  constexpr int NCH = BITS == 1 ? 2 * NV : NV;          // float channel values per lane
  constexpr int NF = reduced_count<NCH, LG, 32>();      // after the cross-group reduction
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, NW = T >> 5;
  const int NQ = L.NQ, KG = L.KG, U = L.U;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  float* tsm = reinterpret_cast<float*>(smem + a.ts_off);
  float* rsm = reinterpret_cast<float*>(smem + a.rs_off);
  float* ysm = reinterpret_cast<float*>(smem + a.y_off);
  const uint8_t* tab = smem + a.tab_off;
  const int ntl = a.total_tiles, step = gridDim.x;
  const int S = a.stages;

  if (FUSED) cluster_arrive_relaxed();                 // paired with the wait in fused_tables
  // ---- 1. weights + scales of the first tiles: independent of the predecessor ----
  if (tid == 0) {
    for (int s = 0; s <= kMaxStages; s++) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t pol = policy_evict_first();
    for (int s = 0; s < S; s++) {
      const int t = blockIdx.x + s * step;
      if (t < ntl) issue_stage<ST>(a, t, smem + s * a.stage_bytes, bar + s, pol);
    }
  }
  // ---- 2. tables / table scales / row sums come from the previous kernel ----
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  if (!FUSED && a.tab_smem && tid == 0) {
    if (p.dep.counted) bl::fence_proxy_async();        // tables were written by another launch
    const uint32_t tb = (uint32_t)KG * 8;
    mbar_expect_tx(bar + kMaxStages, tb);
    for (uint32_t off = 0; off < tb; off += 32768u) {
      const uint32_t nb = tb - off < 32768u ? tb - off : 32768u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + a.tab_off + off)),
          "l"(p.qtab + off), "r"(nb), "r"(smem_u32(bar + kMaxStages))
          : "memory");
    }
  }
  const int row0 = ROWS ? blockIdx.y * a.rows_per_cta : 0;
  const int row1 = ROWS ? min(row0 + a.rows_per_cta, a.n_rows) : 1;
  uint4 tq0[R / 2];
  // this thread's unit tables (one round of units per tile) and the row's
  // table scales / row sums -> smem; rows after the CTA's first reload them
  auto load_row = [&](int row) {
    if (!FUSED && !a.tab_smem && tid < U) {
      const int ub = tid >> 5, l = tid & 31;
      const int nu_b = min(32, U - 32 * ub);
      const uint8_t* tb = p.qtab + (int64_t)row * KG * 8 + (int64_t)ub * (32 * R * 8) + l * 16;
#pragma unroll
      for (int jp = 0; jp < R / 2; jp++) tq0[jp] = bl::ld_cg_128(tb + jp * nu_b * 16);
    }
    for (int i = tid; i < NQ; i += T) {
      tsm[i] = bl::ld_cg_f32(p.tscales + (int64_t)row * NQ + i);
      rsm[i] = bl::ld_cg_f32(p.rowsums + (int64_t)row * NQ + i);
    }
  };
  if (FUSED) {
    fused_tables<R>(a, smem);                           // includes the block-wide syncs
  } else {
    load_row(row0);
  }
  __syncthreads();                                      // barriers initialised, tsm / rsm ready
  if (!FUSED && a.tab_smem) mbar_wait(bar + kMaxStages, 0);

  const bool has_zeros = a.mats[0].zeros != nullptr;     // uniform across the matrices
  const float h2 = (float)(2 << (BITS - 1));
  int it = 0, yit = 0;
  for (int tile = blockIdx.x; tile < ntl; tile += step, it++) {
    const int stage = S == 1 ? 0 : (it & 1);
    uint8_t* sb = smem + stage * a.stage_bytes;
    mbar_wait(bar + stage, (S == 1 ? it : it >> 1) & 1);
    const ST* sraw = reinterpret_cast<const ST*>(sb + a.s_off);
    const ST* zraw = reinterpret_cast<const ST*>(sb + a.z_off);
  for (int row = row0; row < row1; row++, yit++) {      // mpGEMM: the tile stays in smem
    if constexpr (ROWS) {
      if (row != row0 || it > 0) {
        __syncthreads();                                // previous row done with tsm / rsm
        load_row(row);
        __syncthreads();
      }
    }
    const bool last_row = !ROWS || row + 1 == row1;

    float y[NCH];
#pragma unroll
    for (int j = 0; j < NCH; j++) y[j] = 0.f;
    int ch0 = 0;
    for (int rd = 0; rd < a.rounds; rd++) {
      const int u = tid + rd * T;
      const bool live = u < U;
      if constexpr (EXACT) {
        // reference epilogue: per-plane staging values (packed stream pairs)
        int acc[16];
#pragma unroll
        for (int i = 0; i < 16; i++) acc[i] = 0;
        if (live) {
          const int ub = u >> 5, l = u & 31;
          const int nu_b = min(32, U - 32 * ub);
          const int stride = nu_b == 32 ? 512 : nu_b * 16;
          uint4 tq[R / 2];
          if (a.tab_smem) {
            const uint8_t* tb = tab + ub * (32 * R * 8) + l * 16;
#pragma unroll
            for (int jp = 0; jp < R / 2; jp++) tq[jp] = *reinterpret_cast<const uint4*>(tb + jp * stride);
          } else {
#pragma unroll
            for (int jp = 0; jp < R / 2; jp++) tq[jp] = tq0[jp];
          }
          const uint8_t* wsrc = sb + ub * (32 * R * 16) + l * 16;
#pragma unroll
          for (int j = 0; j < R; j++) {
            const uint4 wr = *reinterpret_cast<const uint4*>(wsrc + j * stride);
            lookup_kg(wr, (j & 1) ? tq[j >> 1].z : tq[j >> 1].x, (j & 1) ? tq[j >> 1].w : tq[j >> 1].y, acc);
          }
        }
        const int base = transpose_reduce<LG, 16, int>(acc, lane);
        if (live) {
          constexpr int NFP = 16 / LG;
          int32_t* dst = reinterpret_cast<int32_t*>(smem + a.psm_off) + (u / LG) * 33 + 2 * base;
#pragma unroll
          for (int i = 0; i < NFP; i++) {             // v = P_even + 32768 P_odd
            const int v = acc[i];
            const int pe = (v << 17) >> 17;
            dst[2 * i] = pe;
            dst[2 * i + 1] = (v - pe) >> 15;
          }
        }
        continue;
      }
      int acc[NACC];
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = 0;
      if (live) {
        const int ub = u >> 5, l = u & 31;
        const int nu_b = min(32, U - 32 * ub);
        const int stride = nu_b == 32 ? 512 : nu_b * 16;
        const uint8_t* wsrc = sb + ub * (32 * R * 16) + l * 16;
        if (KIND == kFast && a.ldg_w) {
          // weights straight from HBM into registers (the warp reads 512
          // contiguous bytes per k-step), no shared-memory stage
          int local;
          const B1Mat& mt = a.mats[find_mat(a, tile, local)];
          const uint8_t* gsrc = mt.w + L.sg_row_base(local, 0) + ub * (32 * R * 16) + l * 16;
          uint4 wv[R];
#pragma unroll
          for (int j = 0; j < R; j++) wv[j] = bl::ld_nc_128(gsrc + j * stride);
          if (a.tab_smem) {
            const uint8_t* tb = tab + ub * (32 * R * 8) + l * 16;
#pragma unroll
            for (int j = 0; j < R; j += 2) {
              const uint4 t = *reinterpret_cast<const uint4*>(tb + (j >> 1) * stride);
              lookup_kg_merged<BITS, NACC>(wv[j], t.x, t.y, acc);
              lookup_kg_merged<BITS, NACC>(wv[j + 1], t.z, t.w, acc);
            }
          } else {
#pragma unroll
            for (int j = 0; j < R; j += 2) {
              lookup_kg_merged<BITS, NACC>(wv[j], tq0[j >> 1].x, tq0[j >> 1].y, acc);
              lookup_kg_merged<BITS, NACC>(wv[j + 1], tq0[j >> 1].z, tq0[j >> 1].w, acc);
            }
          }
        } else if (FUSED || a.tab_smem) {
          const uint8_t* tb = tab + ub * (32 * R * 8) + l * 16;
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            const uint4 t = *reinterpret_cast<const uint4*>(tb + (j >> 1) * stride);
            const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
            const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
            lookup_kg_merged<BITS, NACC>(wa, t.x, t.y, acc);
            lookup_kg_merged<BITS, NACC>(wc, t.z, t.w, acc);
          }
        } else if (nu_b == 32) {                        // register tables, full unit block
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * 512);
            const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * 512);
            lookup_kg_merged<BITS, NACC>(wa, tq0[j >> 1].x, tq0[j >> 1].y, acc);
            lookup_kg_merged<BITS, NACC>(wc, tq0[j >> 1].z, tq0[j >> 1].w, acc);
          }
        } else {
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
            const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
            lookup_kg_merged<BITS, NACC>(wa, tq0[j >> 1].x, tq0[j >> 1].y, acc);
            lookup_kg_merged<BITS, NACC>(wc, tq0[j >> 1].z, tq0[j >> 1].w, acc);
          }
        }
      }
      // sum the LG lanes of each quantization group (exact int32)
      const int base = reduce_lanes<NACC, 1, LG>(acc, lane);
      ch0 = BITS == 1 ? 2 * base : base;
      if (live) {
        const int g = u / LG;
        const float ts = tsm[g], rs = rsm[g];
        int S[NCH];
        if constexpr (BITS == 1) {
#pragma unroll
          for (int i = 0; i < NV; i++) {
            const int v = acc[i];                       // P_even + 32768 P_odd
            const int pe = (v << 17) >> 17;
            S[2 * i] = pe;
            S[2 * i + 1] = (v - pe) >> 15;
          }
        } else {
#pragma unroll
          for (int i = 0; i < NV; i++) S[i] = acc[i];
        }
        if (p.partials) {                                 // exact integer sums (single-matrix launches)
          int local;
          find_mat(a, tile, local);
#pragma unroll
          for (int j = 0; j < NCH; j++)
            p.partials[((int64_t)row * L.m + (int64_t)local * TCH + ch0 + j) * NQ + g] = S[j];
        }
#pragma unroll
        for (int j = 0; j < NCH; j++) {
          const int c = ch0 + j;
          float t = fmaf(ts, (float)S[j], -rs);
          if (has_zeros) t = fmaf(fmaf(-2.f, bl::to_f32(zraw[c * NQ + g]), h2), rs, t);
          y[j] = fmaf(bl::to_f32(sraw[c * NQ + g]), t, y[j]);
        }
      }
    }
    if constexpr (EXACT) {
      __syncthreads();                                  // staging values complete
      float* terms = reinterpret_cast<float*>(smem + a.terms_off);
      const int32_t* psm = reinterpret_cast<const int32_t*>(smem + a.psm_off);
      form_terms<BITS, BITLUT_TABLE_Q8, ST>(p, sraw, zraw, tsm, rsm, psm, terms, a.rowlen, tid, T, 0, 0);
      __syncthreads();                                  // products complete; stage consumed
      if (tid == 0 && last_row) {
        const int t = tile + S * step;
        if (t < ntl) issue_stage<ST>(a, t, sb, bar + stage, policy_evict_first());
      }
      int local;
      const int j = find_mat(a, tile, local);
      chains_and_out(L, terms, reinterpret_cast<float*>(smem + a.fin_off), a.rowlen, has_zeros,
                     a.mats[j].out + (int64_t)row * L.m + (int64_t)local * TCH);
      __syncthreads();                                  // psm / terms / fin reusable
      continue;
    }
    // ---- cross-group reduction: lanes of this warp, then the warps ----
    const int fb = reduce_lanes<NCH, LG, 32>(y, lane);
    float* yb = ysm + (yit & 1) * NW * TCH + warp * TCH;
#pragma unroll
    for (int j = 0; j < NF; j++) yb[ch0 + fb + j] = y[j];   // lanes holding a duplicate write the same value
    __syncthreads();                                    // stage consumed, ysm complete
    if (tid == 0 && last_row) {
      const int t = tile + S * step;
      if (t < ntl) issue_stage<ST>(a, t, sb, bar + stage, policy_evict_first());
    }
    if (tid < TCH) {
      const float* yr = ysm + (yit & 1) * NW * TCH + tid;
      float s = 0.f;
      for (int w = 0; w < NW; w++) s += yr[w * TCH];
      int local;
      const int j = find_mat(a, tile, local);
      a.mats[j].out[(int64_t)row * L.m + (int64_t)local * TCH + tid] = 0.5f * s;
      if constexpr (KIND == kFast) {
        // fused all-gather: the same value into every rank's gathered row
        for (int q = 0; q < a.gth.n_peers; q++)
          a.gth.peer_out[q][a.gth.col_offset + local * TCH + tid] = 0.5f * s;
      }
    }
  }
  }
  if constexpr (KIND == kFast) {
    if (a.gth.n_peers > 0) {
      __syncthreads();                                  // the CTA's peer stores are issued
      if (tid == 0) {
        __threadfence_system();
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.gth.ticket) : "memory");
        if (old == gridDim.x - 1) {                     // last CTA: every store of the grid is ordered before
          *a.gth.ticket = 0;
          __threadfence_system();
          for (int q = 0; q < a.gth.n_peers; q++)
            asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.gth.peer_flag[q]) : "memory");
        }
      }
    }
  }
  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();                    // keep stream completion order
}


// Lean specialisation of the fast batch-1 kernel for its common case: one
// round of units per tile (thread u = unit u), tables in registers, no zero
// points, no partials export, no fused gather, weights staged by TMA.  Same
// arithmetic, same shared-memory plan and launch plan as gemv_b1_kernel
// (launch_b1 picks it), so outputs are bitwise identical; what it drops is
// the per-tile cost of the general kernel's mode branches, round / row loops
// and per-tile reloads: the thread's group, table scale, row sum and smem
// addresses are fixed for the launch.
// F16: the fast path of variant cuda-f16, on 16-bit block-fixed-point tables
// (BITLUT_TABLE_X16: two balanced base-127 int8 digit tables per k-group, 16 B
// in registers): the int8 core runs once per digit with shared selectors,
// S = 127 S_H + S_L exactly, then the int8 epilogue with the 16-bit table
// scale (scalar-real semantics _kernels.py:101-137 within the fp16-table
// tolerance, tested).  Round 1's fp16 byte-plane lookups (5 PRMT + sign fix
// per 4 lookups, fp32 adds) ran at 0.49 of the HBM peak.
// PERM: the operand is in the layer-set layout (layout.cuh; BITLUT_FLAG_LAYER_SET):
// select-free lane reductions and one scale vector per lane, like gemv_batch_kernel.
template <int R, int LG, int BITS, typename ST, bool ZEROS, bool F16 = false, bool PERM = false>
__global__ void __launch_bounds__(384) gemv_b1_lean_kernel(const __grid_constant__ B1Args a) {
  const GemvArgs& p = a.g;
  const bl::LayoutV2& L = p.L;
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
  // tiles of this CTA: all matrices strided by the grid, or (partitioned
  // launch) the CTA's own matrix strided by that matrix's CTAs -- then the
  // matrix's own tables, when it has them
  int t_first = blockIdx.x, step = gridDim.x, ntl = a.total_tiles;
  const uint8_t* qtab = p.qtab;
  const float* tsc = p.tscales;
  const float* rsum = p.rowsums;
  if (a.partition) {
    int pj = 0;
    while (pj + 1 < a.n_mats && (int)blockIdx.x >= a.cta_begin[pj + 1]) pj++;
    t_first = (pj ? a.mats[pj - 1].tile_end : 0) + ((int)blockIdx.x - a.cta_begin[pj]);
    step = a.cta_begin[pj + 1] - a.cta_begin[pj];
    ntl = a.mats[pj].tile_end;
    if (a.mats[pj].qtab) {
      qtab = a.mats[pj].qtab;
      tsc = a.mats[pj].tscales;
      rsum = a.mats[pj].rowsums;
    }
  }

  if (tid == 0) {
    for (int s = 0; s <= kMaxStages; s++) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t pol = policy_evict_first();
    for (int s = 0; s < S; s++) {
      const int t = t_first + s * step;
      if (t < ntl) issue_stage<ST>(a, t, smem + s * a.stage_bytes, bar + s, pol);
    }
  }
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  // the thread's unit, group and tables: fixed for the launch
  // a thread past the last unit shadows the last unit with all-zero int8
  // tables (exact zeros everywhere): the int8 tile loop has no "live" branch
  const bool live = tid < U;
  const int u = live ? tid : U - 1;
  const int ub = u >> 5, l = u & 31;
  const int nu_b = min(32, U - 32 * ub);
  const int g = u / LG;
  uint4 tq[F16 ? R : R / 2];
  float ts = 0.f, rs = 0.f;
  if (live) {
    if constexpr (F16) {
      const uint8_t* tb = qtab + (int64_t)ub * (32 * R * 16) + l * 16;
#pragma unroll
      for (int j = 0; j < R; j++) tq[j] = bl::ld_cg_128(tb + j * nu_b * 16);
      ts = bl::ld_cg_f32(tsc + g);
    } else {
      const uint8_t* tb = qtab + (int64_t)ub * (32 * R * 8) + l * 16;
#pragma unroll
      for (int jp = 0; jp < R / 2; jp++) tq[jp] = bl::ld_cg_128(tb + jp * nu_b * 16);
      ts = bl::ld_cg_f32(tsc + g);
    }
    rs = bl::ld_cg_f32(rsum + g);
  } else {
#pragma unroll
    for (int jp = 0; jp < (F16 ? R : R / 2); jp++) tq[jp] = make_uint4(0, 0, 0, 0);
  }
  const uint32_t woff = (uint32_t)(ub * (32 * R * 16) + l * 16);
  BL_CHECK(a.bar_off + 8u * (kMaxStages + 1) <= bl::dyn_smem_bytes());
  BL_CHECK(!live || woff + (R - 1) * (nu_b == 32 ? 512 : nu_b * 16) + 16 <= a.w_bytes);
  __syncthreads();                                      // barriers initialised
  int it = 0;
  for (int tile = t_first; tile < ntl; tile += step, it++) {
    const int stage = S == 1 ? 0 : (it & 1);
    uint8_t* sb = smem + stage * a.stage_bytes;
    mbar_wait(bar + stage, (S == 1 ? it : it >> 1) & 1);
    float y[NCH];
    int ch0 = 0;
    // integer sums: int8 tables, or (F16) the two digit tables of the 16-bit
    // block-fixed-point tables (BITLUT_TABLE_X16: the H and L digit tables of a
    // k-group are one uint4; the int8 core runs once per digit with shared
    // selectors), combined per lane as S = 127 S_H + S_L -- exact -- before
    // the lane reduction (W1: after it, the packed pair fields would overflow)
    int acc[NACC];
    int accL[F16 && BITS == 1 ? NACC : 1];
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = 0;
    {
      const uint8_t* wsrc = sb + woff;
      const int stride = nu_b == 32 ? 512 : nu_b * 16;
      if constexpr (F16) {
        int lo[NACC];
#pragma unroll
        for (int i = 0; i < NACC; i++) lo[i] = 0;
#pragma unroll
        for (int j = 0; j < R; j++)
          lookup_kg_merged2<BITS, NACC>(*reinterpret_cast<const uint4*>(wsrc + j * stride), tq[j].x, tq[j].y,
                                        tq[j].z, tq[j].w, acc, lo);
        if constexpr (BITS == 1) {
#pragma unroll
          for (int i = 0; i < NACC; i++) accL[i] = lo[i];
        } else {
#pragma unroll
          for (int i = 0; i < NACC; i++) acc[i] = 127 * acc[i] + lo[i];
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; j += 2) {
          const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
          const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
          lookup_kg_merged<BITS, NACC>(wa, tq[j >> 1].x, tq[j >> 1].y, acc);
          lookup_kg_merged<BITS, NACC>(wc, tq[j >> 1].z, tq[j >> 1].w, acc);
        }
      }
    }
    if constexpr (PERM) {
      reduce_lanes_perm<NACC, 1, LG>(acc);
      if constexpr (F16 && BITS == 1) reduce_lanes_perm<NACC, 1, LG>(accL);
    } else {
      const int base = reduce_lanes<NACC, 1, LG>(acc, lane);
      if constexpr (F16 && BITS == 1) reduce_lanes<NACC, 1, LG>(accL, lane);
      ch0 = BITS == 1 ? 2 * base : base;
    }
    {
      int Sv[NCH];
      if constexpr (BITS == 1) {
#pragma unroll
        for (int i = 0; i < NV; i++) {
          const int v = acc[i];
          const int pe = (v << 17) >> 17;
          Sv[2 * i] = pe;
          Sv[2 * i + 1] = (v - pe) >> 15;
          if constexpr (F16) {
            const int vl = accL[i];
            const int le = (vl << 17) >> 17;
            Sv[2 * i] = 127 * Sv[2 * i] + le;
            Sv[2 * i + 1] = 127 * Sv[2 * i + 1] + ((vl - le) >> 15);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < NV; i++) Sv[i] = acc[i];
      }
      if constexpr (PERM) {
        // the unit's NCH scales (zero points) are one vector; __fmul_rn keeps the
        // products out of the reduction's first add (bitwise == the v2 path)
        constexpr int SB = NCH * (int)sizeof(ST);
        uint32_t sv[(SB + 3) / 4];
        lds_vec<SB>(sb + a.s_off + (uint32_t)u * SB, sv);
        if constexpr (ZEROS) {
          uint32_t zv[(SB + 3) / 4];
          lds_vec<SB>(sb + a.z_off + (uint32_t)u * SB, zv);
          const float h2 = (float)(2 << (BITS - 1));
#pragma unroll
          for (int j = 0; j < NCH; j++)
            y[j] = __fmul_rn(vec_elem<ST>(sv, j),
                             fmaf(fmaf(-2.f, vec_elem<ST>(zv, j), h2), rs, fmaf(ts, (float)Sv[j], -rs)));
        } else {
#pragma unroll
          for (int j = 0; j < NCH; j++) y[j] = __fmul_rn(vec_elem<ST>(sv, j), fmaf(ts, (float)Sv[j], -rs));
        }
      } else {
        const ST* sp = reinterpret_cast<const ST*>(sb + a.s_off) + ch0 * NQ + g;
        if constexpr (ZEROS) {
          // asymmetric zero points: + 2 (2^(b-1) - z) rs per (channel, group)
          const ST* zp = reinterpret_cast<const ST*>(sb + a.z_off) + ch0 * NQ + g;
          const float h2 = (float)(2 << (BITS - 1));
#pragma unroll
          for (int j = 0; j < NCH; j++) {
            const float t = fmaf(fmaf(-2.f, bl::to_f32(zp[j * NQ]), h2), rs, fmaf(ts, (float)Sv[j], -rs));
            y[j] = bl::to_f32(sp[j * NQ]) * t;
          }
        } else {
#pragma unroll
          for (int j = 0; j < NCH; j++) y[j] = bl::to_f32(sp[j * NQ]) * fmaf(ts, (float)Sv[j], -rs);
        }
      }
    }
    float* yb = ysm + (it & 1) * NW * TCH + warp * TCH;
    if constexpr (PERM) {
      reduce_lanes_perm<NCH, LG, 32>(y);
      yb[perm_mask<TCH>(lane)] = y[0];
    } else {
      const int fb = reduce_lanes<NCH, LG, 32>(y, lane);
#pragma unroll
      for (int j = 0; j < NF; j++) yb[ch0 + fb + j] = y[j];
    }
    __syncthreads();                                    // stage consumed, ysm complete
    if (tid == 0) {
      const int t = tile + S * step;
      if (t < ntl) issue_stage<ST>(a, t, sb, bar + stage, policy_evict_first());
    }
    if (tid >= 32 && tid < 32 + TCH) {                  // warp 1 adds the sums (thread 0 refills: gemv_batch.cu)
      const int c = tid - 32;
      const float* yr = ysm + (it & 1) * NW * TCH + c;
      float s = 0.f;
      for (int w = 0; w < NW; w++) s += yr[w * TCH];
      int local;
      const int j = find_mat(a, tile, local);
      BL_CHECK(j < a.n_mats && local >= 0 && local * TCH + c < (a.mats[j].tile_end - (j ? a.mats[j - 1].tile_end : 0)) * TCH);
      a.mats[j].out[(int64_t)local * TCH + c] = 0.5f * s;
    }
  }
  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();
}


// Lean mpGEMM rows kernel (kFastRows common case: one unit round, register
// tables, no zeros / partials): the tile is staged once and stays in shared
// memory while the CTA walks its rows TWO AT A TIME -- the weights are read
// from shared memory once per row pair and the selector preparation is
// shared (lookup_kg_merged2); one barrier per pair publishes the cross-warp
// partial sums (double-buffered).
// Bitwise equal to gemv_b1_kernel<kFastRows>.
template <int R, int LG, int BITS, typename ST, bool PERM = false>
__global__ void __launch_bounds__(384) gemv_b1_rows_lean_kernel(const __grid_constant__ B1Args a) {
  const GemvArgs& p = a.g;
  const bl::LayoutV2& L = p.L;
  constexpr int TCH = 32 / BITS;
  constexpr int NACC = BITS == 4 ? 8 : 16;
  constexpr int NV = reduced_count<NACC, 1, LG>();
  constexpr int NCH = BITS == 1 ? 2 * NV : NV;
  constexpr int NF = reduced_count<NCH, LG, 32>();
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x >> 5;
  const int NQ = L.NQ, KG = L.KG, U = L.U;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  float* ysm = reinterpret_cast<float*>(smem + a.y_off);     // [2 pairs][2 rows][NW][TCH]
  const int tile = blockIdx.x;
  const int row0 = blockIdx.y * a.rows_per_cta;
  const int row1 = min(row0 + a.rows_per_cta, a.n_rows);
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue_stage<ST>(a, tile, smem, bar, policy_evict_first());
  }
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  const int u = tid;
  const bool live = u < U;
  const int ub = u >> 5, l = u & 31;
  const int nu_b = min(32, U - 32 * ub);
  const int g = u / LG;
  const uint8_t* tb0 = p.qtab + (int64_t)ub * (32 * R * 8) + l * 16;
  uint4 tqA[R / 2], tqB[R / 2];
  float tsA = 0.f, rsA = 0.f, tsB = 0.f, rsB = 0.f;
  auto fetch = [&](int row, uint4 (&t)[R / 2], float& s1, float& s2) {
    if (live && row < row1) {
      const uint8_t* tb = tb0 + (int64_t)row * KG * 8;
#pragma unroll
      for (int jp = 0; jp < R / 2; jp++) t[jp] = bl::ld_cg_128(tb + jp * nu_b * 16);
      s1 = bl::ld_cg_f32(p.tscales + (int64_t)row * NQ + g);
      s2 = bl::ld_cg_f32(p.rowsums + (int64_t)row * NQ + g);
    }
  };
  __syncthreads();                                      // barrier initialised
  mbar_wait(bar, 0);
  const uint8_t* wsrc = smem + (uint32_t)(ub * (32 * R * 16) + l * 16);
  int local;
  const int mj = find_mat(a, tile, local);
  float* outp = a.mats[mj].out + (int64_t)local * TCH;
  const int stride = nu_b * 16;
  // the lane's NCH weight scales are the same for every row: converted once
  float wsf[NCH];
  if constexpr (PERM) {                                 // layer-set operand: the unit's scale vector
    constexpr int SB = NCH * (int)sizeof(ST);
    uint32_t sv[(SB + 3) / 4];
    lds_vec<SB>(smem + a.s_off + (uint32_t)(live ? u : U - 1) * SB, sv);
#pragma unroll
    for (int j = 0; j < NCH; j++) wsf[j] = live ? vec_elem<ST>(sv, j) : 0.f;
  } else {
    const int b0 = lane_base<NACC, 1, LG>(lane);
    const ST* sp = reinterpret_cast<const ST*>(smem + a.s_off) + (BITS == 1 ? 2 * b0 : b0) * NQ + g;
#pragma unroll
    for (int j = 0; j < NCH; j++) wsf[j] = live ? bl::to_f32(sp[j * NQ]) : 0.f;
  }
  // one row's sums: group reduction, scaling, reduction over the warp's groups -> ysm
  auto finish_row = [&](int (&acc)[NACC], float ts, float rs, float* ybuf) {
    int ch0 = 0;
    if constexpr (PERM) {
      reduce_lanes_perm<NACC, 1, LG>(acc);
    } else {
      const int base = reduce_lanes<NACC, 1, LG>(acc, lane);
      ch0 = BITS == 1 ? 2 * base : base;
    }
    float y[NCH];
    if (live) {
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
#pragma unroll
      for (int j = 0; j < NCH; j++) y[j] = __fmul_rn(wsf[j], fmaf(ts, (float)Sv[j], -rs));
    } else {
#pragma unroll
      for (int j = 0; j < NCH; j++) y[j] = 0.f;
    }
    float* yb = ybuf + warp * TCH;
    if constexpr (PERM) {
      reduce_lanes_perm<NCH, LG, 32>(y);
      yb[perm_mask<TCH>(lane)] = y[0];
    } else {
      const int fb = reduce_lanes<NCH, LG, 32>(y, lane);
#pragma unroll
      for (int j = 0; j < NF; j++) yb[ch0 + fb + j] = y[j];
    }
  };
  for (int row = row0, it = 0; row < row1; row += 2, it++) {
    const bool two = row + 1 < row1;                    // uniform over the CTA
    fetch(row, tqA, tsA, rsA);                          // (other CTAs of the SM hide the L2 latency)
    fetch(row + 1, tqB, tsB, rsB);
    int accA[NACC], accB[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) accA[i] = accB[i] = 0;
    if (live) {
      if (two) {
#pragma unroll
        for (int j = 0; j < R; j += 2) {
          const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
          const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
          lookup_kg_merged2<BITS, NACC>(wa, tqA[j >> 1].x, tqA[j >> 1].y, tqB[j >> 1].x, tqB[j >> 1].y, accA, accB);
          lookup_kg_merged2<BITS, NACC>(wc, tqA[j >> 1].z, tqA[j >> 1].w, tqB[j >> 1].z, tqB[j >> 1].w, accA, accB);
        }
      } else {
#pragma unroll
        for (int j = 0; j < R; j += 2) {
          const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
          const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
          lookup_kg_merged<BITS, NACC>(wa, tqA[j >> 1].x, tqA[j >> 1].y, accA);
          lookup_kg_merged<BITS, NACC>(wc, tqA[j >> 1].z, tqA[j >> 1].w, accA);
        }
      }
    }
    float* ybase = ysm + (it & 1) * 2 * NW * TCH;
    finish_row(accA, tsA, rsA, ybase);
    if (two) finish_row(accB, tsB, rsB, ybase + NW * TCH);
    __syncthreads();                                    // this pair's partials complete
    if (tid >= 32 && tid < 32 + 2 * TCH) {              // warps 1.. add the sums: one thread per (row, channel)
      const int r = (tid - 32) / TCH, c = (tid - 32) - r * TCH;
      if (r == 0 || two) {
        const float* yr = ybase + r * NW * TCH + c;
        float sum = 0.f;
        for (int w = 0; w < NW; w++) sum += yr[w * TCH];
        outp[(int64_t)(row + r) * L.m + c] = 0.5f * sum;
      }
    }
  }
  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();
}


// Long-K batch-1 fast lookups split over a thread-block cluster: CS CTAs share
// every tile, rank r owning quantization groups [r*NG/CS, (r+1)*NG/CS) (its
// unit blocks are TMA-copied; a block two ranks touch is copied by both).
// Per tile each CTA forms its partial channel sums exactly like the lean
// kernel (one unit per thread, register tables, fixed group), stores them
// into rank 0's shared memory (DSMEM) and arrives on the cluster barrier;
// rank 0 adds the CS partials in rank order one tile later, after the
// matching wait -- the barrier's latency overlaps the next tile's lookups.
// Deterministic for a given CS (the fp32 order differs from the unsplit
// kernel's in the last bits; the integer sums are the same).
struct ClArgs {
  int cs;                     // CTAs per cluster (tile split)
  int u0[9];                  // unit ranges per rank: [u0[r], u0[r+1])
  uint32_t stage_bytes, w_bytes_max, s_off, s_bytes, z_off, y_off, part_off, bar_off;
  int stages;
};

template <int R, int LG, int BITS, typename ST, bool ZEROS>
__global__ void __launch_bounds__(256) gemv_b1_cluster_kernel(const __grid_constant__ B1Args a,
                                                              const __grid_constant__ ClArgs c) {
  const GemvArgs& p = a.g;
  const bl::LayoutV2& L = p.L;
  constexpr int TCH = 32 / BITS;
  constexpr int NACC = BITS == 4 ? 8 : 16;
  constexpr int NV = reduced_count<NACC, 1, LG>();
  constexpr int NCH = BITS == 1 ? 2 * NV : NV;
  constexpr int NF = reduced_count<NCH, LG, 32>();
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x >> 5;
  const int NQ = L.NQ, U = L.U;
  const uint32_t rank = cluster_rank();
  const int CS = c.cs;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + c.bar_off);
  float* ysm = reinterpret_cast<float*>(smem + c.y_off);
  float* part = reinterpret_cast<float*>(smem + c.part_off);      // [2][CS][TCH] (rank 0's is read)
  const int ntl = a.total_tiles;
  const int ncl = gridDim.x / CS, cl = blockIdx.x / CS;
  const int S = c.stages;
  const int ua = c.u0[rank], ue = c.u0[rank + 1];
  const int b0 = ua >> 5, b1 = (ue + 31) >> 5;
  uint32_t wbytes = 0;
  for (int b = b0; b < b1; b++) wbytes += (uint32_t)(min(32, U - 32 * b) * R * 16);

  auto issue = [&](int tile, uint8_t* sb, uint64_t* br, uint64_t pol) {
    int local;
    const B1Mat& mt = a.mats[find_mat(a, tile, local)];
    const bool z = mt.zeros != nullptr;
    mbar_expect_tx(br, wbytes + c.s_bytes * (z ? 2u : 1u));
    const uint8_t* src = mt.w + L.sg_row_base(local, 0) + (int64_t)b0 * (32 * R * 16);
    for (uint32_t off = 0; off < wbytes; off += 32768u) {
      const uint32_t nb = wbytes - off < 32768u ? wbytes - off : 32768u;
      bulk_g2s(sb + off, src + off, nb, br, pol);
    }
    const int64_t e0 = (int64_t)local * L.tile_ch * L.NQ;
    bulk_g2s(sb + c.s_off, reinterpret_cast<const ST*>(mt.wscales) + e0, c.s_bytes, br, pol);
    if (z) bulk_g2s(sb + c.z_off, reinterpret_cast<const ST*>(mt.zeros) + e0, c.s_bytes, br, pol);
  };
  if (tid == 0) {
    for (int s = 0; s < S; s++) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t pol = policy_evict_first();
    for (int s = 0; s < S; s++) {
      const int t = cl + s * ncl;
      if (t < ntl) issue(t, smem + s * c.stage_bytes, bar + s, pol);
    }
  }
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  // a thread past the rank's last unit shadows it with all-zero tables (exact
  // zeros everywhere): the tile loop has no "live" branches
  const bool live = ua + tid < ue;
  const int u = live ? ua + tid : max(ue - 1, ua);
  const int ub = u >> 5, l = u & 31;
  const int nu_b = min(32, U - 32 * ub);
  const int g = u / LG;
  uint4 tq[R / 2];
  float ts = 0.f, rs = 0.f;
  if (live) {
    const uint8_t* tb = p.qtab + (int64_t)ub * (32 * R * 8) + l * 16;
#pragma unroll
    for (int jp = 0; jp < R / 2; jp++) tq[jp] = bl::ld_cg_128(tb + jp * nu_b * 16);
    ts = bl::ld_cg_f32(p.tscales + g);
    rs = bl::ld_cg_f32(p.rowsums + g);
  } else {
#pragma unroll
    for (int jp = 0; jp < R / 2; jp++) tq[jp] = make_uint4(0, 0, 0, 0);
  }
  const uint32_t woff = (uint32_t)((ub - b0) * (32 * R * 16) + l * 16);
  __syncthreads();                                      // barriers initialised
  cluster_arrive_relaxed();                             // every CTA of the cluster has started:
  cluster_wait();                                       // DSMEM stores are safe from here on
  int it = 0, prev_tile = -1;
  for (int tile = cl; tile < ntl; tile += ncl, it++) {
    const int stage = S == 1 ? 0 : (it & 1);
    uint8_t* sb = smem + stage * c.stage_bytes;
    mbar_wait(bar + stage, (S == 1 ? it : it >> 1) & 1);
    int acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = 0;
    {
      const uint8_t* wsrc = sb + woff;
      const int stride = nu_b * 16;
#pragma unroll
      for (int j = 0; j < R; j += 2) {
        const uint4 wa = *reinterpret_cast<const uint4*>(wsrc + j * stride);
        const uint4 wc = *reinterpret_cast<const uint4*>(wsrc + (j + 1) * stride);
        lookup_kg_merged<BITS, NACC>(wa, tq[j >> 1].x, tq[j >> 1].y, acc);
        lookup_kg_merged<BITS, NACC>(wc, tq[j >> 1].z, tq[j >> 1].w, acc);
      }
    }
    const int base = reduce_lanes<NACC, 1, LG>(acc, lane);
    const int ch0 = BITS == 1 ? 2 * base : base;
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
      const ST* sp = reinterpret_cast<const ST*>(sb + c.s_off) + ch0 * NQ + g;
      if constexpr (ZEROS) {
        const ST* zp = reinterpret_cast<const ST*>(sb + c.z_off) + ch0 * NQ + g;
        const float h2 = (float)(2 << (BITS - 1));
#pragma unroll
        for (int j = 0; j < NCH; j++) {
          const float t = fmaf(fmaf(-2.f, bl::to_f32(zp[j * NQ]), h2), rs, fmaf(ts, (float)Sv[j], -rs));
          y[j] = bl::to_f32(sp[j * NQ]) * t;
        }
      } else {
#pragma unroll
        for (int j = 0; j < NCH; j++) y[j] = bl::to_f32(sp[j * NQ]) * fmaf(ts, (float)Sv[j], -rs);
      }
    }
    const int fb = reduce_lanes<NCH, LG, 32>(y, lane);
    float* yb = ysm + (it & 1) * NW * TCH + warp * TCH;
#pragma unroll
    for (int j = 0; j < NF; j++) yb[ch0 + fb + j] = y[j];
    __syncthreads();                                    // stage consumed, ysm complete
    if (tid == 0) {
      const int t = tile + S * ncl;
      if (t < ntl) issue(t, sb, bar + stage, policy_evict_first());
    }
    if (it > 0) {
      cluster_wait();                                   // partials of the previous tile are in rank 0
      if (rank == 0 && tid < TCH) {
        const float* pr = part + ((it - 1) & 1) * CS * TCH + tid;
        float sum = 0.f;
        for (int r = 0; r < CS; r++) sum += pr[r * TCH];
        int local;
        const int j = find_mat(a, prev_tile, local);
        a.mats[j].out[(int64_t)local * TCH + tid] = 0.5f * sum;
      }
    }
    if (tid >= 32 && tid < 32 + TCH) {                  // warp 1 adds the sums (thread 0 refills)
      const int cc = tid - 32;
      const float* yr = ysm + (it & 1) * NW * TCH + cc;
      float sum = 0.f;
      for (int w = 0; w < NW; w++) sum += yr[w * TCH];
      st_cluster_f32(part + (it & 1) * CS * TCH + rank * TCH + cc, 0, sum);
    }
    cluster_arrive_release();
    prev_tile = tile;
  }
  if (it > 0) {
    cluster_wait();
    if (rank == 0 && tid < TCH) {
      const float* pr = part + ((it - 1) & 1) * CS * TCH + tid;
      float sum = 0.f;
      for (int r = 0; r < CS; r++) sum += pr[r * TCH];
      int local;
      const int j = find_mat(a, prev_tile, local);
      a.mats[j].out[(int64_t)local * TCH + tid] = 0.5f * sum;
    }
  }
  cluster_arrive_relaxed();                             // no CTA leaves while a peer may still
  cluster_wait();                                       // store into its shared memory
  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();
}

template <int R, int LG, int BITS, typename ST>
int launch_b1_cluster(const GemvArgs& g, const B1Mat* mats, int n_mats, cudaStream_t stream, bool pdl,
                      bool* handled) {
  const bl::LayoutV2& L = g.L;
  *handled = false;
  const int NG = L.U / LG;
  int cs = 2;
  while (cs < 8 && (NG + cs - 1) / cs * LG > 256) cs <<= 1;
  if ((NG + cs - 1) / cs * LG > 256) return BITLUT_OK;   // not handled
  ClArgs c;
  c.cs = cs;
  int tmax = 0;
  for (int r = 0; r <= cs; r++) c.u0[r] = (int)((int64_t)NG * r / cs) * LG;
  for (int r = 0; r < cs; r++) tmax = max(tmax, c.u0[r + 1] - c.u0[r]);
  const int T = ((tmax + 31) / 32) * 32 < 64 ? 64 : ((tmax + 31) / 32) * 32;
  uint32_t wmax = 0;
  for (int r = 0; r < cs; r++) {
    const int b0 = c.u0[r] >> 5, b1 = (c.u0[r + 1] + 31) >> 5;
    uint32_t w = 0;
    for (int b = b0; b < b1; b++) w += (uint32_t)(min(32, L.U - 32 * b) * L.R * 16);
    wmax = max(wmax, w);
  }
  const bool zeros = mats[0].zeros != nullptr;
  B1Args a;
  a.g = g;
  a.act = nullptr;
  a.gth = GatherArgs{};
  a.ldg_w = 0;
  a.n_mats = n_mats;
  for (int j = 0; j < n_mats; j++) a.mats[j] = mats[j];
  a.total_tiles = mats[n_mats - 1].tile_end;
  c.s_bytes = (uint32_t)((size_t)L.tile_ch * L.NQ * sizeof(ST));
  c.w_bytes_max = wmax;
  c.s_off = al16(wmax);
  c.z_off = c.s_off + al16(c.s_bytes);
  c.stage_bytes = ((c.z_off + (zeros ? al16(c.s_bytes) : 0)) + 127) & ~127u;
  auto kern = zeros ? gemv_b1_cluster_kernel<R, LG, BITS, ST, true> : gemv_b1_cluster_kernel<R, LG, BITS, ST, false>;
  static bool configured[64][2] = {};                  // per device
  if (!configured[bl_device()][zeros]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return BITLUT_EINTERNAL;
    configured[bl_device()][zeros] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cs;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.blockDim = dim3(T);
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // two stages when that keeps as many clusters resident, else one
  int best_cl = 0;
  size_t best_total = 0;
  for (int st = 1; st <= 2; st++) {
    const uint32_t y_off = st * c.stage_bytes;
    const uint32_t part_off = y_off + al16((size_t)2 * (T / 32) * L.tile_ch * 4);
    const uint32_t bar_off = part_off + al16((size_t)2 * cs * L.tile_ch * 4);
    const size_t total = bar_off + 16;
    if (total > 227 * 1024) break;
    cfg.dynamicSmemBytes = total;
    cfg.gridDim = dim3(cs * 148);
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) ncl = 0;
    if (ncl >= 1 && ncl >= best_cl) {
      best_cl = ncl; best_total = total;
      c.stages = st; c.y_off = y_off; c.part_off = part_off; c.bar_off = bar_off;
    }
  }
  if (best_cl < 1) return BITLUT_OK;                  // not handled
  int ncl = best_cl;
  if (ncl > a.total_tiles) ncl = a.total_tiles;
  if (g.grid_out) *g.grid_out = ncl * cs;
  cfg.gridDim = dim3(ncl * cs);
  cfg.dynamicSmemBytes = best_total;
  *handled = true;
  return cudaLaunchKernelEx(&cfg, kern, a, c) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

int sm_count() {
  static int n_dev[64] = {};                           // per device
  const int dev = bl_device();
  int& n = n_dev[dev];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

constexpr int kClusterCTAs = 8;

// CTA size.  A dependent launch (its inputs complete only when it starts)
// wants the shortest per-tile path: as few rounds of units as a <= 384-thread
// CTA allows, units spread evenly (U = 344 at K = 11008 -> one round of 352
// threads).  An overlapped (INDEPENDENT) launch wants more resident CTAs:
// at most 256 threads.  Never fewer than 128.
int b1_threads(const bl::LayoutV2& L, bool overlapped) {
  static int cap_env = -1;
  if (cap_env < 0) {
    const char* e = getenv("BITLUT_B1_CAP");             // diagnostic: overlapped-launch CTA cap
    cap_env = e ? atoi(e) : 0;
  }
  // one round of units per tile whenever U <= 384: the lean kernel needs it,
  // and at K = 11008 one round of 352 threads beats two of 176 (4096x11008
  // overlapped W2 3.38 -> 3.09 us, W4 5.36 -> 4.86 us)
  const int cap = overlapped ? (cap_env > 0 ? cap_env : 384) : 384;
  const int rounds = (L.U + cap - 1) / cap;
  int t = (L.U + rounds - 1) / rounds;
  t = (t + 31) & ~31;
  return t < 128 ? 128 : t;
}

template <int R, int LG, int BITS, typename ST, int KIND>
int launch_b1(const GemvArgs& g, const B1Mat* mats, int n_mats, const __half* act, cudaStream_t stream,
              bool pdl) {
  constexpr bool FUSED = KIND == kFused;
  const bl::LayoutV2& L = g.L;
  if constexpr (KIND == kFast) {
    static int cl_env = -1;
    if (cl_env < 0) {
      const char* e = getenv("BITLUT_B1_CLUSTER");       // diagnostic: 0 disables the split-K cluster kernel
      cl_env = e ? atoi(e) : 1;
    }
    // long tile rows only (> 64 KB, K > 16384: the 70B down projection and
    // its shards): 4096x28672 W2 8.3 vs 11.0 us, 2048x28672 4.7 vs 5.9 us;
    // at K = 11008 the unsplit lean kernel is faster (2.6 vs 3.8 us)
    if (cl_env != 0 && (size_t)L.KG * 16 > 65536 && L.U > 256 && !g.partials && !g.gather && !g.trace &&
        g.n_rows <= 1 && !g.f16_tables && !g.layer_set) {
      bool handled = false;
      const int rc = launch_b1_cluster<R, LG, BITS, ST>(g, mats, n_mats, stream, pdl, &handled);
      if (handled || rc != BITLUT_OK) return rc;
    }
  }
  // the exact epilogue's serial chains favour one tile per CTA and one round
  const int T = b1_threads(L, !kind_exact(KIND) && (g.independent || g.dep.counted));
  if (FUSED && T % (L.gs / 4) != 0) return BITLUT_ELAYOUT;
  if (n_mats < 1 || n_mats > kMaxMats) return BITLUT_EPARAM;
  B1Args a;
  a.g = g;
  a.act = act;
  a.gth = GatherArgs{};
  if (g.gather) {
    if (KIND != kFast) return BITLUT_EPARAM;
    a.gth = *g.gather;
  }
  a.n_mats = n_mats;
  for (int j = 0; j < n_mats; j++) a.mats[j] = mats[j];
  a.total_tiles = mats[n_mats - 1].tile_end;
  a.rounds = (L.U + T - 1) / T;
  a.tab_smem = FUSED || a.rounds > 1;
  const int n_rows = kind_rows(KIND) ? (g.n_rows > 0 ? g.n_rows : 1) : 1;
  // several activation rows: one round of units (register tables reloaded per row)
  if (kind_rows(KIND) && (a.rounds > 1 || n_mats > 1)) return BITLUT_ELAYOUT;
  a.n_rows = n_rows;
  a.rows_per_cta = n_rows;
  static int ldg_env = -1;
  if (ldg_env < 0) {
    // diagnostic: weights via registers, no smem stage -- measured slower
    // (4096^2 W4 overlapped 2.01 vs 1.75 us, W2 on par), off by default
    const char* e = getenv("BITLUT_B1_LDG");
    ldg_env = e ? atoi(e) : 0;
  }
  a.ldg_w = (KIND == kFast && ldg_env > 0) ? 1 : 0;
  static int lean_env = -1;
  if (lean_env < 0) {
    const char* e = getenv("BITLUT_B1_LEAN");            // diagnostic: 0 = always the general kernel
    lean_env = e ? atoi(e) : 1;
  }
  const bool lean_common = lean_env != 0 && a.rounds == 1 && !a.tab_smem && !g.partials && !g.gather &&
                           !g.trace && !a.ldg_w;
  const bool has_z = mats[0].zeros != nullptr;
  const bool lean = KIND == kFast && lean_common;
  const bool lean_rows = KIND == kFastRows && lean_common && n_mats == 1 && !has_z && !g.f16_tables;
  if (g.f16_tables && !lean) return BITLUT_ELAYOUT;     // X16 tables: the lean kernel only
  const bool f16 = g.f16_tables != 0;
  // layer-set operand: the lean kernels only, and only where the per-unit scale
  // vectors are a permutation of the (channel, group) block (same stage plan)
  const bool perm = g.layer_set != 0;
  if (perm && (!(lean || lean_rows) ||
               bl::layer_set_scale_bytes(L, (int)sizeof(ST)) != (int64_t)L.tile_ch * L.NQ * (int64_t)sizeof(ST)))
    return BITLUT_ELAYOUT;
  auto kern = lean ? (f16 ? (perm ? (has_z ? gemv_b1_lean_kernel<R, LG, BITS, ST, true, true, true>
                                           : gemv_b1_lean_kernel<R, LG, BITS, ST, false, true, true>)
                                  : (has_z ? gemv_b1_lean_kernel<R, LG, BITS, ST, true, true>
                                           : gemv_b1_lean_kernel<R, LG, BITS, ST, false, true>))
                          : (perm ? (has_z ? gemv_b1_lean_kernel<R, LG, BITS, ST, true, false, true>
                                           : gemv_b1_lean_kernel<R, LG, BITS, ST, false, false, true>)
                                  : (has_z ? gemv_b1_lean_kernel<R, LG, BITS, ST, true>
                                           : gemv_b1_lean_kernel<R, LG, BITS, ST, false>)))
                   : (lean_rows ? (perm ? gemv_b1_rows_lean_kernel<R, LG, BITS, ST, true>
                                        : gemv_b1_rows_lean_kernel<R, LG, BITS, ST, false>)
                                : gemv_b1_kernel<R, LG, BITS, ST, KIND>);
  static bool configured_k[64][16] = {};               // per device and kernel variant
  // 0 general; 1,2 lean (zeros); 4,5 lean X16; 6 rows; + 8 with the layer-set operand
  const int ki = (lean ? (has_z ? 2 : 1) + (f16 ? 3 : 0) : (lean_rows ? 6 : 0)) + (perm ? 8 : 0);
  bool& configured = configured_k[bl_device()][ki];
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return BITLUT_EINTERNAL;
    configured = true;
  }
  // Tiles per CTA: a dependent launch wants the most CTAs (shortest path
  // once its inputs are ready); an INDEPENDENT one overlaps its predecessor
  // and gains from amortising the CTA setup over two tiles.
  static int tpc_env = -1;
  if (tpc_env < 0) {
    const char* e = getenv("BITLUT_B1_TILES_PER_CTA");   // diagnostic override
    tpc_env = e ? atoi(e) : 0;
  }

  // one stage when every CTA gets a single tile, else double-buffer
  const bool zeros = mats[0].zeros != nullptr;
  B1Plan s = b1_plan<ST>(L, zeros, a.tab_smem, T, 1, KIND, a.ldg_w != 0);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, s.total) != cudaSuccess || per_sm < 1)
    return BITLUT_ELAYOUT;
  const B1Plan s2 = b1_plan<ST>(L, zeros, a.tab_smem, T, 2, KIND, a.ldg_w != 0);
  int per_sm2 = 0;
  if (s2.total > 227 * 1024 ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, kern, T, s2.total) != cudaSuccess)
    per_sm2 = 0;
  // two tiles per CTA only where the double-buffered plan still leaves
  // several CTAs per SM (short K); long-K tiles want every CTA they can get
  static int tpc_ovl = -1, tpc_dep = -1;
  if (tpc_ovl < 0) {
    const char* e1 = getenv("BITLUT_B1_TPC_OVL");         // diagnostic: tiles per CTA, overlapped launches
    const char* e2 = getenv("BITLUT_B1_TPC_DEP");         // ... dependent launches
    // overlapped fast launches: three tiles per double-buffered CTA (layer
    // set 0.405 -> 0.401 ms, lookups alone 0.402 -> 0.390 ms, 3 of 3 A/B runs)
    tpc_ovl = e1 ? atoi(e1) : 3;
    tpc_dep = e2 ? atoi(e2) : 0;
  }
  const bool ovl = g.independent || g.dep.counted;
  int tiles_per_cta = tpc_env > 0 ? tpc_env
                                  : ((!kind_exact(KIND) && ovl && per_sm2 >= 3) ? 2 : 1);
  if (tpc_env <= 0 && !kind_exact(KIND)) {
    if (ovl && tpc_ovl > 0 && per_sm2 >= 1) tiles_per_cta = tpc_ovl;
    if (!ovl && tpc_dep > 0 && per_sm2 >= 1) tiles_per_cta = tpc_dep;
  }
  if (tpc_env <= 0 && (a.total_tiles + tiles_per_cta - 1) / tiles_per_cta < sm_count() / 2) tiles_per_cta = 1;
  const int want = (a.total_tiles + tiles_per_cta - 1) / tiles_per_cta;
  // double-buffer when CTAs get several tiles -- by choice (tiles_per_cta)
  // or because one wave cannot hold every tile -- unless that costs
  // resident CTAs (then the single stage refills after each tile)
  a.stages = 1;
  if (per_sm2 >= 1 && (tiles_per_cta > 1 || (sm_count() * per_sm < a.total_tiles && per_sm2 >= per_sm))) {
    s = s2; per_sm = per_sm2; a.stages = 2;
  }
  if (s.total > 227 * 1024) return BITLUT_ELAYOUT;
  a.stage_bytes = s.stage_bytes; a.w_bytes = s.w_bytes; a.s_off = s.s_off; a.s_bytes = s.s_bytes;
  a.z_off = s.z_off; a.tab_off = s.tab_off; a.ts_off = s.ts_off; a.rs_off = s.rs_off;
  a.y_off = s.y_off; a.bar_off = s.bar_off; a.sa_off = s.sa_off; a.red_off = s.red_off;
  a.psm_off = s.psm_off; a.terms_off = s.terms_off; a.fin_off = s.fin_off; a.rowlen = s.rowlen;
  int grid = sm_count() * per_sm;
  if (grid > want) grid = want;
  a.partition = 0;
  if (g.mixed_tables) {
    if (!lean) return BITLUT_ELAYOUT;                   // per-matrix tables: the lean kernel only
    // CTAs per matrix in proportion to its tiles (>= 1, <= its tiles); a CTA
    // then serves one matrix and loads that matrix's tables once
    const int G = grid < n_mats ? n_mats : grid;
    a.partition = 1;
    a.cta_begin[0] = 0;
    for (int j = 0; j < n_mats; j++) {
      const int nj = mats[j].tile_end - (j ? mats[j - 1].tile_end : 0);
      int cj = (int)(((int64_t)G * nj + a.total_tiles / 2) / a.total_tiles);
      if (cj < 1) cj = 1;
      if (cj > nj) cj = nj;
      a.cta_begin[j + 1] = a.cta_begin[j] + cj;
    }
    grid = a.cta_begin[n_mats];
  }
  const int cs = FUSED ? kClusterCTAs : 1;
  grid = (grid + cs - 1) / cs * cs;                     // spare CTAs only build their table slice
  int grid_y = 1;
  if (kind_rows(KIND)) {
    // mpGEMM: one tile per CTA (weights stay in smem for the CTA's rows);
    // rows per CTA as large as keeps >= 4 CTAs per SM busy
    int r = 32;
    while (r > 1 && (int64_t)a.total_tiles * ((n_rows + r - 1) / r) < 4 * sm_count()) r >>= 1;
    a.rows_per_cta = r;
    grid_y = (n_rows + r - 1) / r;
    if (grid_y > 65535) return BITLUT_ESHAPE;
    grid = a.total_tiles;
    a.stages = 1;
    s = b1_plan<ST>(L, zeros, a.tab_smem, T, 1, KIND);
    a.stage_bytes = s.stage_bytes; a.tab_off = s.tab_off; a.ts_off = s.ts_off; a.rs_off = s.rs_off;
    a.y_off = s.y_off; a.bar_off = s.bar_off; a.sa_off = s.sa_off; a.red_off = s.red_off;
    a.psm_off = s.psm_off; a.terms_off = s.terms_off; a.fin_off = s.fin_off;
  }
  if (g.grid_out) *g.grid_out = grid * grid_y;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, grid_y);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = s.total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cs;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = FUSED ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

template <int R, int LG, typename ST, int KIND>
int launch_b1_bits(const GemvArgs& g, const B1Mat* m, int nm, const __half* act, cudaStream_t s, bool pdl) {
  switch (g.L.bits) {
    case 1: return launch_b1<R, LG, 1, ST, KIND>(g, m, nm, act, s, pdl);
    case 2: return launch_b1<R, LG, 2, ST, KIND>(g, m, nm, act, s, pdl);
    case 4: return launch_b1<R, LG, 4, ST, KIND>(g, m, nm, act, s, pdl);
  }
  return BITLUT_EPARAM;
}

template <typename ST, int KIND>
int dispatch_b1(const GemvArgs& g, const B1Mat* m, int nm, const __half* act, cudaStream_t s, bool pdl) {
  const int R = g.L.R, LG = g.L.Lg;
  if (R == 8) {
    switch (LG) {
      case 1: return launch_b1_bits<8, 1, ST, KIND>(g, m, nm, act, s, pdl);
      case 2: return launch_b1_bits<8, 2, ST, KIND>(g, m, nm, act, s, pdl);
      case 4: return launch_b1_bits<8, 4, ST, KIND>(g, m, nm, act, s, pdl);
      case 8: return launch_b1_bits<8, 8, ST, KIND>(g, m, nm, act, s, pdl);
      case 16: return launch_b1_bits<8, 16, ST, KIND>(g, m, nm, act, s, pdl);
    }
  } else if (R == 4 && LG == 1) {
    return launch_b1_bits<4, 1, ST, KIND>(g, m, nm, act, s, pdl);
  }
  return BITLUT_EPARAM;
}

B1Mat single_mat(const GemvArgs& g) {
  B1Mat m;
  m.w = g.w; m.wscales = g.wscales; m.zeros = g.zeros; m.out = g.out; m.tile_end = g.L.n_tiles;
  return m;
}

}  // namespace

// Internal entry used by bitlut_mpgemm_traced (gemv.cu) for batch-1 fast
// calls: returns BITLUT_ELAYOUT when the shape does not fit the kernel's
// shared-memory plan (the caller then uses the per-tile kernel).
int bl_gemv_b1_launch(const GemvArgs& g, int scale_dtype, cudaStream_t s, bool pdl) {
  if (g.L.n_sg != 1) return BITLUT_ELAYOUT;
  const B1Mat m = single_mat(g);
  const bool f16 = scale_dtype == BITLUT_DT_F16;
  if (g.n_rows > 1) {
    if (g.fast)
      return f16 ? dispatch_b1<__half, kFastRows>(g, &m, 1, nullptr, s, pdl)
                 : dispatch_b1<float, kFastRows>(g, &m, 1, nullptr, s, pdl);
    return f16 ? dispatch_b1<__half, kExactRows>(g, &m, 1, nullptr, s, pdl)
               : dispatch_b1<float, kExactRows>(g, &m, 1, nullptr, s, pdl);
  }
  if (g.fast)
    return f16 ? dispatch_b1<__half, kFast>(g, &m, 1, nullptr, s, pdl)
               : dispatch_b1<float, kFast>(g, &m, 1, nullptr, s, pdl);
  return f16 ? dispatch_b1<__half, kExact>(g, &m, 1, nullptr, s, pdl)
             : dispatch_b1<float, kExact>(g, &m, 1, nullptr, s, pdl);
}

bool bl_gemv_b1_fused_fits(const bl::LayoutV2& L, bool zeros, int scale_dtype) {
  if (L.n_sg != 1) return false;
  const int T = b1_threads(L, false);
  if (T % (L.gs / 4) != 0) return false;
  const size_t total = scale_dtype == BITLUT_DT_F16 ? b1_plan<__half>(L, zeros, true, T, 1, kFused).total
                                                    : b1_plan<float>(L, zeros, true, T, 1, kFused).total;
  return total <= 227 * 1024;
}

// Table build + lookup in ONE launch for a batch-1 fp16 activation row
// (fast epilogue): see include/bitlut_b200.h.
int bl_mpgemv_fused_launch(const void* a, int a_dtype, const uint8_t* wgpu, int m, int k, int bits,
                           int group_size, const void* wscales, const void* zeros, int scale_dtype, float* out,
                           int flags, void* stream, const bl::DepSync& dep, int* grid_out);

extern "C" int bitlut_mpgemv_fused(const void* a, int a_dtype, const uint8_t* wgpu, int m, int k, int bits,
                                   int group_size, const void* wscales, const void* zeros, int scale_dtype,
                                   float* out, int flags, void* stream) {
  const bl::DepSync none = {};
  return bl_mpgemv_fused_launch(a, a_dtype, wgpu, m, k, bits, group_size, wscales, zeros, scale_dtype, out,
                                flags, stream, none, nullptr);
}

int bl_mpgemv_fused_launch(const void* a, int a_dtype, const uint8_t* wgpu, int m, int k, int bits,
                           int group_size, const void* wscales, const void* zeros, int scale_dtype, float* out,
                           int flags, void* stream, const bl::DepSync& dep, int* grid_out) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (!a || !wgpu || !wscales || !out) return BITLUT_EPARAM;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (!(flags & BITLUT_FLAG_FAST_EPILOGUE)) return BITLUT_EPARAM;     // reference order: build_lut + mpgemm
  if (a_dtype != BITLUT_DT_F16 || L.n_sg != 1) return BITLUT_ELAYOUT;  // caller falls back to two launches
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  GemvArgs g = {};
  g.w = wgpu; g.wscales = wscales; g.zeros = zeros;
  g.out = out; g.L = L;
  g.dep = dep;
  g.grid_out = grid_out;
  g.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  g.fast = 1;
  g.rows_per_cta = 1; g.n_rows = 1;
  const __half* act = reinterpret_cast<const __half*>(a);
  const B1Mat mt = single_mat(g);
  return scale_dtype == BITLUT_DT_F16 ? dispatch_b1<__half, kFused>(g, &mt, 1, act, (cudaStream_t)stream, pdl)
                                      : dispatch_b1<float, kFused>(g, &mt, 1, act, (cudaStream_t)stream, pdl);
}

int bl_mpgemv_multi_launch(const bitlut_mat* mats, int n_mats, int k, int bits, int group_size,
                           int scale_dtype, const void* tables, const float* tscales, const float* rowsums,
                           int flags, void* stream, const bl::DepSync& dep, int* grid_out);

// Several matrices sharing one activation row's tables in ONE batch-1 launch
// (q/k/v, gate/up): see include/bitlut_b200.h.
extern "C" int bitlut_mpgemv_multi(const bitlut_mat* mats, int n_mats, int k, int bits, int group_size,
                                   int scale_dtype, const void* tables, const float* tscales,
                                   const float* rowsums, int flags, void* stream) {
  const bl::DepSync none = {};
  return bl_mpgemv_multi_launch(mats, n_mats, k, bits, group_size, scale_dtype, tables, tscales, rowsums,
                                flags, stream, none, nullptr);
}

int bl_mpgemv_multi_launch(const bitlut_mat* mats, int n_mats, int k, int bits, int group_size,
                           int scale_dtype, const void* tables, const float* tscales, const float* rowsums,
                           int flags, void* stream, const bl::DepSync& dep, int* grid_out) {
  if (!mats || n_mats < 1 || n_mats > kMaxMats || !tables || !tscales || !rowsums) return BITLUT_EPARAM;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  bl::LayoutV2 L;
  B1Mat ms[kMaxMats];
  int tiles = 0;
  for (int j = 0; j < n_mats; j++) {
    int rc = bl::make_layout(mats[j].m, k, bits, group_size, &L);
    if (rc) return rc;
    if (!mats[j].wgpu || !mats[j].wscales || !mats[j].out) return BITLUT_EPARAM;
    if ((mats[j].zeros != nullptr) != (mats[0].zeros != nullptr)) return BITLUT_EPARAM;
    tiles += L.n_tiles;
    ms[j].w = mats[j].wgpu; ms[j].wscales = mats[j].wscales; ms[j].zeros = mats[j].zeros;
    ms[j].out = mats[j].out; ms[j].tile_end = tiles;
  }
  if (L.n_sg != 1) return BITLUT_ELAYOUT;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  GemvArgs g = {};
  g.qtab = reinterpret_cast<const uint8_t*>(tables); g.tscales = tscales; g.rowsums = rowsums;
  g.L = L;
  g.dep = dep;
  g.grid_out = grid_out;
  g.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  g.fast = (flags & BITLUT_FLAG_FAST_EPILOGUE) != 0;
  g.layer_set = (flags & BITLUT_FLAG_LAYER_SET) != 0;   // operands in the layer-set layout (fast, lean kernel)
  if (g.layer_set && !g.fast) return BITLUT_ELAYOUT;
  g.zeros = mats[0].zeros;                              // presence flag for the epilogue
  g.rows_per_cta = 1; g.n_rows = 1;
  const cudaStream_t st = (cudaStream_t)stream;
  if (g.fast)
    return scale_dtype == BITLUT_DT_F16 ? dispatch_b1<__half, kFast>(g, ms, n_mats, nullptr, st, pdl)
                                        : dispatch_b1<float, kFast>(g, ms, n_mats, nullptr, st, pdl);
  return scale_dtype == BITLUT_DT_F16 ? dispatch_b1<__half, kExact>(g, ms, n_mats, nullptr, st, pdl)
                                      : dispatch_b1<float, kExact>(g, ms, n_mats, nullptr, st, pdl);
}

// Batch-1 fast lookup of this rank's output-channel shard with the all-gather
// fused into the epilogue: see include/bitlut_b200.h.
extern "C" int bitlut_mpgemv_gather(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                                    const void* wscales, const void* zeros, int scale_dtype, const void* tables,
                                    const float* tscales, const float* rowsums, float* out, int n_peers,
                                    float* const* peer_out, unsigned* const* peer_flags, unsigned* ticket,
                                    int col_offset, int flags, void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (!wgpu || !wscales || !tables || !tscales || !rowsums || !out || !ticket) return BITLUT_EPARAM;
  if (n_peers < 1 || n_peers > kMaxPeers || !peer_out || !peer_flags || col_offset < 0) return BITLUT_EPARAM;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (!(flags & BITLUT_FLAG_FAST_EPILOGUE)) return BITLUT_EPARAM;
  if (L.n_sg != 1) return BITLUT_ELAYOUT;
  GatherArgs ga = {};
  ga.n_peers = n_peers;
  ga.col_offset = col_offset;
  for (int q = 0; q < n_peers; q++) {
    if (!peer_out[q] || !peer_flags[q]) return BITLUT_EPARAM;
    ga.peer_out[q] = peer_out[q];
    ga.peer_flag[q] = peer_flags[q];
  }
  ga.ticket = ticket;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  GemvArgs g = {};
  g.w = wgpu; g.wscales = wscales; g.zeros = zeros;
  g.qtab = reinterpret_cast<const uint8_t*>(tables); g.tscales = tscales; g.rowsums = rowsums;
  g.out = out; g.L = L;
  g.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  g.fast = 1;
  g.rows_per_cta = 1; g.n_rows = 1;
  g.gather = &ga;
  const B1Mat mt = single_mat(g);
  const cudaStream_t st = (cudaStream_t)stream;
  return scale_dtype == BITLUT_DT_F16 ? dispatch_b1<__half, kFast>(g, &mt, 1, nullptr, st, pdl)
                                      : dispatch_b1<float, kFast>(g, &mt, 1, nullptr, st, pdl);
}

namespace {
// bounded: gives up after timeout_ns (a peer that never arrives must not
// hang the stream) and then sets *timed_out, when given
__global__ void gather_wait_kernel(const unsigned* flag, unsigned target, unsigned long long timeout_ns,
                                   unsigned* timed_out) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = gtimer();
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if ((int)(v - target) >= 0) break;
      if (gtimer() - t0 > timeout_ns) {
        if (timed_out) *timed_out = 1u;
        break;
      }
      __nanosleep(100);
    }
  }
}
}  // namespace

// Stream-ordered wait until this rank's gather flag reaches `target`
// (wrap-around safe): kernels after it on `stream` see the gathered row.
extern "C" int bitlut_gather_wait(const unsigned* flag, unsigned target, unsigned* timed_out, void* stream) {
  if (!flag) return BITLUT_EPARAM;
  gather_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(flag, target, 10000000000ull, timed_out);
  return bl_launch_status();
}

// Shapes whose batch-1 fast launches run the lean kernel (one unit round,
// no split-K): the op-list planner groups lookups with different tables only
// for these (pipeline.cu).
bool bl_mixed_tables_ok(const bl::LayoutV2& L) {
  static int lean_env = -1, mixed_env = -1;
  if (lean_env < 0) {
    const char* e = getenv("BITLUT_B1_LEAN");
    lean_env = e ? atoi(e) : 1;
    const char* m = getenv("BITLUT_MIXED_TABLES");       // diagnostic: 0 = group same-table lookups only
    mixed_env = m ? atoi(m) : 1;
  }
  return lean_env != 0 && mixed_env != 0 && L.n_sg == 1 && L.U <= 384 && (size_t)L.KG * 16 <= 65536 && L.bits != 3;
}

int bl_mpgemv_multi_tab_launch(const bitlut_mat_tab* mats, int n_mats, int k, int bits, int group_size,
                               int scale_dtype, int flags, void* stream, const bl::DepSync& dep, int* grid_out);

// Several batch-1 matrices, each with its OWN activation tables, in one launch
// (fast epilogue): see include/bitlut_b200.h.
extern "C" int bitlut_mpgemv_multi_tab(const bitlut_mat_tab* mats, int n_mats, int k, int bits, int group_size,
                                       int scale_dtype, int flags, void* stream) {
  const bl::DepSync none = {};
  return bl_mpgemv_multi_tab_launch(mats, n_mats, k, bits, group_size, scale_dtype, flags, stream, none, nullptr);
}

int bl_mpgemv_multi_tab_launch(const bitlut_mat_tab* mats, int n_mats, int k, int bits, int group_size,
                               int scale_dtype, int flags, void* stream, const bl::DepSync& dep, int* grid_out) {
  if (!mats || n_mats < 1 || n_mats > kMaxMats) return BITLUT_EPARAM;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  if (!(flags & BITLUT_FLAG_FAST_EPILOGUE)) return BITLUT_EPARAM;
  bl::LayoutV2 L;
  B1Mat ms[kMaxMats];
  int tiles = 0;
  for (int j = 0; j < n_mats; j++) {
    int rc = bl::make_layout(mats[j].m, k, bits, group_size, &L);
    if (rc) return rc;
    if (!mats[j].wgpu || !mats[j].wscales || !mats[j].out || !mats[j].tables || !mats[j].tscales ||
        !mats[j].rowsums)
      return BITLUT_EPARAM;
    if ((mats[j].zeros != nullptr) != (mats[0].zeros != nullptr)) return BITLUT_EPARAM;
    tiles += L.n_tiles;
    ms[j].w = mats[j].wgpu; ms[j].wscales = mats[j].wscales; ms[j].zeros = mats[j].zeros;
    ms[j].out = mats[j].out; ms[j].tile_end = tiles;
    ms[j].qtab = reinterpret_cast<const uint8_t*>(mats[j].tables);
    ms[j].tscales = mats[j].tscales;
    ms[j].rowsums = mats[j].rowsums;
  }
  if (L.n_sg != 1) return BITLUT_ELAYOUT;
  const bool pdl = (flags & BITLUT_FLAG_PDL) != 0;
  GemvArgs g = {};
  g.qtab = ms[0].qtab; g.tscales = ms[0].tscales; g.rowsums = ms[0].rowsums;
  g.L = L;
  g.independent = pdl && (flags & BITLUT_FLAG_INDEPENDENT) != 0;
  g.fast = 1;
  g.layer_set = (flags & BITLUT_FLAG_LAYER_SET) != 0;   // operands in the layer-set layout
  g.zeros = mats[0].zeros;
  g.rows_per_cta = 1; g.n_rows = 1;
  g.mixed_tables = 1;
  g.dep = dep;
  g.grid_out = grid_out;
  const cudaStream_t st = (cudaStream_t)stream;
  return scale_dtype == BITLUT_DT_F16 ? dispatch_b1<__half, kFast>(g, ms, n_mats, nullptr, st, pdl)
                                      : dispatch_b1<float, kFast>(g, ms, n_mats, nullptr, st, pdl);
}
