// Batch-1 lookup kernel for the decode path, fast epilogue ("pack" kernel,
// opt-in with BITLUT_PACK=1: measured slower than gemv_b1_kernel on every
// Llama shape -- e.g. 4096x4096 W2 overlapped 1.76 vs 1.13 us, 65536x4096
// steady state 20.3 vs 17.9 us -- although it issues ~35% fewer
// instructions per lookup: with half as many threads per tile each thread
// owns twice the staged bytes, so fewer warps are resident to hide the
// lookup and copy latencies.  Kept as the measured alternative.)
//
// Same arithmetic as gemv_b1.cu's fast epilogue -- the exact integer
// S = sum_p 2^p P_p per (channel, quantization group), then
// out_c = 0.5 * sum_g ws_cg * (ts_g * S_cg - rs_g [+ 2 (2^(b-1) - z_cg) rs_g])
// (_kernels.py:179-191 regrouped) -- with the work laid out so that the
// instructions outside the lookup core are paid per quantization group, not
// per unit of eight k-groups:
//
//   * a thread owns a fixed group of every tile it sees (UPL = 2 adjacent
//     units, or one unit when a unit is a whole group): its tables (UPL x R
//     k-groups, registers), table scale and row sum are loaded once per CTA;
//     at gs = 128 (4 units per group) two neighbouring lanes share a group
//     and add their integer sums with one shuffle step;
//   * a CTA streams PACKS of TPK consecutive tiles (TMA bulk copies of the
//     weights and scales, 1-2 stages, issued before the dependency wait);
//     each thread writes its group's per-channel products to a shared row,
//     and after one barrier per pack the outputs are summed over the groups
//     by several threads each plus a shuffle tree -- fixed order, so the
//     result is deterministic and does not depend on the grid;
//   * lookups: gemv_core.cuh lookup_merged (dp4a, W4 1,2,4,8 / W2 A-Y
//     selector form / W1 packed pairs).
#include "gemv_core.cuh"

#include <cstdlib>

namespace {

using namespace blk;

constexpr int kMaxMatsP = 4;
constexpr int kMaxStagesP = 2;

struct PArgs {
  GemvArgs g;
  int n_mats, total_tiles;
  blk::StreamMat mats[kMaxMatsP];
  int tpk;                    // tiles per pack
  int tt;                     // threads per tile (U / UPL)
  int stages;
  int rowp;                   // floats per product row (TCH + 4: conflict-free STS.128)
  uint32_t w_tile, s_tile;    // bytes of one tile's weights / scales in a stage
  uint32_t stage_bytes, y_off, y_bytes, bar_off;
};

__device__ __forceinline__ int find_mat_p(const PArgs& a, int tile, int& local) {
  int j = 0;
  while (j + 1 < a.n_mats && tile >= a.mats[j].tile_end) j++;
  local = tile - (j ? a.mats[j - 1].tile_end : 0);
  return j;
}

// Zero-point terms (BASELINE configs[0]), out of line so the common path has
// no predicated loads: d_c += (2^b - 2 z_c) rs.
template <typename ST, int N>
__device__ __noinline__ void add_zero_terms_p(float (&d)[N], const void* zeros, int64_t e0, int stride, float h2,
                                              float rs) {
  const ST* zp = reinterpret_cast<const ST*>(zeros) + e0;
#pragma unroll
  for (int c = 0; c < N; c++, zp += stride) d[c] = fmaf(fmaf(-2.f, bl::to_f32(*zp), h2), rs, d[c]);
}

template <int N>
__device__ __noinline__ void store_partials_p(int32_t* dst, int stride, const int (&S)[N]) {
#pragma unroll
  for (int c = 0; c < N; c++) dst[(int64_t)c * stride] = S[c];
}

// lane 0 of the CTA: TMA the pack's tiles (weights + scales) into one stage
template <typename ST>
__device__ __forceinline__ void issue_pack(const PArgs& a, int pk, uint8_t* sb, uint64_t* bar, uint64_t pol) {
  const bl::LayoutV2& L = a.g.L;
  const int t0 = pk * a.tpk;
  const int nt = min(a.tpk, a.total_tiles - t0);
  mbar_expect_tx(bar, (uint32_t)nt * (a.w_tile + a.s_tile));
  for (int p = 0; p < nt; p++) {
    int local;
    const blk::StreamMat& mt = a.mats[find_mat_p(a, t0 + p, local)];
    const uint8_t* src = mt.w + L.sg_row_base(local, 0);
    uint8_t* dst = sb + p * a.w_tile;
    for (uint32_t off = 0; off < a.w_tile; off += 32768u) {
      const uint32_t nb = a.w_tile - off < 32768u ? a.w_tile - off : 32768u;
      bulk_g2s(dst + off, src + off, nb, bar, pol);
    }
    bulk_g2s(sb + a.tpk * a.w_tile + p * a.s_tile,
             reinterpret_cast<const ST*>(mt.wscales) + (int64_t)local * L.tile_ch * L.NQ, a.s_tile, bar, pol);
  }
}

template <int BITS, int R, int LG, typename ST>
__global__ void __launch_bounds__(512, 1) gemv_pack_kernel(const __grid_constant__ PArgs a) {
  constexpr int TCH = 32 / BITS;                        // channels per tile
  constexpr int NACC = BITS == 4 ? 8 : 16;              // int accumulators per thread
  constexpr int UPL = LG < 2 ? LG : 2;                  // units per thread
  constexpr int LPG = LG / UPL;                         // threads per group (1 or 2)
  constexpr int NCL = LPG == 2 ? TCH / 2 : TCH;         // channels a thread scales
  const GemvArgs& p = a.g;
  const bl::LayoutV2& L = p.L;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31;
  const int NQ = L.NQ, U = L.U, TPK = a.tpk, tt = a.tt, rowp = a.rowp;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  const int npacks = (a.total_tiles + TPK - 1) / TPK;
  const int S = a.stages;

  // this thread's tile-in-pack and group (fixed for the whole launch)
  const int tp = tid / tt, v = tid - tp * tt;
  const bool lane_live = tp < TPK;
  const int g = v / LPG;
  const int ug = v * UPL;                               // first unit
  const int ub = ug >> 5, pos = ug & 31;                // unit block, position in it
  const int nu = min(32, U - 32 * ub);
  const int cb = LPG == 2 ? (v & 1) * NCL : 0;

  // ---- 1. barriers; the first packs stream in before the dependency wait ----
  if (tid == 0) {
    for (int s = 0; s < S; s++) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t pol = policy_evict_first();
    for (int s = 0; s < S; s++) {
      const int pk = blockIdx.x + s * gridDim.x;
      if (pk < npacks) issue_pack<ST>(a, pk, smem + s * a.stage_bytes, bar + s, pol);
    }
  }
  // ---- 2. tables / table scale / row sum of this thread's group (from the previous kernel) ----
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  uint4 tq[UPL][R / 2];
  float ts = 0.f, rs = 0.f;
  if (lane_live) {
    const uint8_t* tb = p.qtab + (int64_t)ub * (32 * R * 8) + pos * 16;
#pragma unroll
    for (int u = 0; u < UPL; u++)
#pragma unroll
      for (int jp = 0; jp < R / 2; jp++) tq[u][jp] = bl::ld_cg_128(tb + (jp * nu + u) * 16);
    ts = bl::ld_cg_f32(p.tscales + g);
    rs = bl::ld_cg_f32(p.rowsums + g);
  }
  __syncthreads();                                      // barriers initialised

  const bool has_zeros = p.zeros != nullptr;
  const float h2 = (float)(2 << (BITS - 1));
  int it = 0;
  for (int pk = blockIdx.x; pk < npacks; pk += gridDim.x, it++) {
    const int stage = S == 1 ? 0 : (it & 1);
    uint8_t* sb = smem + stage * a.stage_bytes;
    float* ysm = reinterpret_cast<float*>(smem + a.y_off + (it & 1) * a.y_bytes);
    mbar_wait(bar + stage, (S == 1 ? it : it >> 1) & 1);
    const int tile = pk * TPK + tp;
    const bool live = lane_live && tile < a.total_tiles;
    int acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = 0;
    if (live) {
      const uint8_t* wb = sb + tp * a.w_tile + (int64_t)ub * (32 * R * 16) + pos * 16;
      if (nu == 32) {
#pragma unroll
        for (int u = 0; u < UPL; u++)
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            const uint4 wa = *reinterpret_cast<const uint4*>(wb + j * 512 + u * 16);
            const uint4 wc = *reinterpret_cast<const uint4*>(wb + (j + 1) * 512 + u * 16);
            lookup_merged<BITS, NACC>(wa, tq[u][j >> 1].x, tq[u][j >> 1].y, acc);
            lookup_merged<BITS, NACC>(wc, tq[u][j >> 1].z, tq[u][j >> 1].w, acc);
          }
      } else {                                          // the tile row's last, partial unit block
        const int st = nu * 16;
#pragma unroll
        for (int u = 0; u < UPL; u++)
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            const uint4 wa = *reinterpret_cast<const uint4*>(wb + j * st + u * 16);
            const uint4 wc = *reinterpret_cast<const uint4*>(wb + (j + 1) * st + u * 16);
            lookup_merged<BITS, NACC>(wa, tq[u][j >> 1].x, tq[u][j >> 1].y, acc);
            lookup_merged<BITS, NACC>(wc, tq[u][j >> 1].z, tq[u][j >> 1].w, acc);
          }
      }
    }
    if constexpr (LPG == 2) {
      // the group's other half is in the neighbour lane: exact int32 sums;
      // the even lane keeps channels [0, TCH/2), the odd one the rest
#pragma unroll
      for (int q = 0; q < NACC / 2; q++) {
        const bool up = (lane & 1) != 0;
        const int send = up ? acc[q] : acc[q + NACC / 2];
        const int keep = up ? acc[q + NACC / 2] : acc[q];
        acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
    }
    if (live) {
      int Sv[NCL];
      if constexpr (BITS == 1) {
#pragma unroll
        for (int i = 0; i < NCL / 2; i++) {
          const int x = acc[i];                          // P_even + 32768 P_odd
          const int pe = (x << 17) >> 17;
          Sv[2 * i] = pe;
          Sv[2 * i + 1] = (x - pe) >> 15;
        }
      } else {
#pragma unroll
        for (int i = 0; i < NCL; i++) Sv[i] = acc[i];
      }
      int local;
      const int mj = find_mat_p(a, tile, local);
      if (p.partials) store_partials_p<NCL>(p.partials + ((int64_t)local * TCH + cb) * NQ + g, NQ, Sv);
      float d[NCL];
#pragma unroll
      for (int c = 0; c < NCL; c++) d[c] = fmaf(ts, (float)Sv[c], -rs);
      if (has_zeros)
        add_zero_terms_p<ST, NCL>(d, a.mats[mj].zeros, ((int64_t)local * TCH + cb) * NQ + g, NQ, h2, rs);
      const ST* sraw = reinterpret_cast<const ST*>(sb + TPK * a.w_tile + tp * a.s_tile) + cb * NQ + g;
      float* yrow = ysm + (tp * NQ + g) * rowp + cb;
#pragma unroll
      for (int c = 0; c < NCL; c += 4) {
        float4 o;
        o.x = bl::to_f32(sraw[(c + 0) * NQ]) * d[c + 0];
        o.y = bl::to_f32(sraw[(c + 1) * NQ]) * d[c + 1];
        o.z = bl::to_f32(sraw[(c + 2) * NQ]) * d[c + 2];
        o.w = bl::to_f32(sraw[(c + 3) * NQ]) * d[c + 3];
        *reinterpret_cast<float4*>(yrow + c) = o;
      }
    }
    __syncthreads();                                    // rows complete; the stage is consumed
    if (tid == 0) {
      const int nx = pk + S * gridDim.x;
      if (nx < npacks) issue_pack<ST>(a, nx, sb, bar + stage, policy_evict_first());
    }
    // out_c = 0.5 * sum over the groups: tpo threads per output, strided
    // partial sums then a shuffle tree (fixed order)
    {
      const int nout = TPK * TCH;
      int tpo = 32;
      while (tpo > 1 && tpo * nout > T) tpo >>= 1;
      const int o = tid / tpo, j = tid - o * tpo;
      float s = 0.f;
      const int p2 = o / TCH, c = o - p2 * TCH;
      const int tile2 = pk * TPK + p2;
      const bool ok = o < nout && tile2 < a.total_tiles;
      if (ok) {
        const float* col = ysm + (p2 * NQ) * rowp + c;
        for (int gg = j; gg < NQ; gg += tpo) s += col[gg * rowp];
      }
      for (int off = tpo / 2; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (ok && j == 0) {
        int local;
        const int mj = find_mat_p(a, tile2, local);
        a.mats[mj].out[(int64_t)local * TCH + c] = 0.5f * s;
      }
    }
  }
  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();                    // keep stream completion order
}

int sm_count_p() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BITS, int R, int LG, typename ST>
int launch_p(const GemvArgs& g, const blk::StreamMat* mats, int n_mats, cudaStream_t stream, bool pdl) {
  constexpr int UPL = LG < 2 ? LG : 2;
  const bl::LayoutV2& L = g.L;
  auto kern = gemv_pack_kernel<BITS, R, LG, ST>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return BITLUT_EINTERNAL;
    configured = true;
  }
  PArgs a;
  a.g = g;
  a.n_mats = n_mats;
  for (int j = 0; j < n_mats; j++) a.mats[j] = mats[j];
  a.total_tiles = mats[n_mats - 1].tile_end;
  a.tt = L.U / UPL;
  if (a.tt * UPL != L.U || a.tt > 512) return BITLUT_ELAYOUT;
  static int tpk_env = -1;
  if (tpk_env < 0) {
    const char* e = getenv("BITLUT_PACK_TPK");           // diagnostic override
    tpk_env = e ? atoi(e) : 0;
  }
  a.tpk = tpk_env > 0 ? tpk_env : (128 / a.tt > 1 ? 128 / a.tt : 1);
  while (a.tpk > 1 && a.tpk * a.tt > 512) a.tpk--;
  const int T = ((a.tpk * a.tt + 31) / 32) * 32;
  a.rowp = L.tile_ch + 4;
  a.w_tile = (uint32_t)((size_t)L.KG * 16);
  a.s_tile = (uint32_t)(((size_t)L.tile_ch * L.NQ * sizeof(ST) + 15) & ~(size_t)15);
  a.stage_bytes = (uint32_t)(((size_t)a.tpk * (a.w_tile + a.s_tile) + 127) & ~(size_t)127);
  a.y_bytes = (uint32_t)(((size_t)a.tpk * L.NQ * a.rowp * 4 + 127) & ~(size_t)127);
  // stages: double-buffer unless that costs resident CTAs
  int best_stages = 1, best_per_sm = 0;
  size_t best_total = 0;
  for (int s = 1; s <= kMaxStagesP; s++) {
    const size_t total = (size_t)s * a.stage_bytes + 2 * (size_t)a.y_bytes + 8 * kMaxStagesP;
    if (total > 227 * 1024) break;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, total) != cudaSuccess) per_sm = 0;
    if (per_sm >= 1 && per_sm >= best_per_sm) { best_stages = s; best_per_sm = per_sm; best_total = total; }
  }
  if (best_per_sm < 1) return BITLUT_ELAYOUT;
  a.stages = best_stages;
  a.y_off = (uint32_t)(best_stages * a.stage_bytes);
  a.bar_off = a.y_off + 2 * a.y_bytes;
  const int npacks = (a.total_tiles + a.tpk - 1) / a.tpk;
  int grid = sm_count_p() * best_per_sm;
  if (grid > npacks) grid = npacks;
  if (g.grid_out) *g.grid_out = grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = best_total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

template <int R, int LG, typename ST>
int launch_p_bits(const GemvArgs& g, const blk::StreamMat* m, int nm, cudaStream_t s, bool pdl) {
  switch (g.L.bits) {
    case 1: return launch_p<1, R, LG, ST>(g, m, nm, s, pdl);
    case 2: return launch_p<2, R, LG, ST>(g, m, nm, s, pdl);
    case 4: return launch_p<4, R, LG, ST>(g, m, nm, s, pdl);
  }
  return BITLUT_ELAYOUT;
}

template <typename ST>
int dispatch_p(const GemvArgs& g, const blk::StreamMat* m, int nm, cudaStream_t s, bool pdl) {
  const int R = g.L.R, LG = g.L.Lg;
  if (R == 8) {
    switch (LG) {
      case 1: return launch_p_bits<8, 1, ST>(g, m, nm, s, pdl);
      case 2: return launch_p_bits<8, 2, ST>(g, m, nm, s, pdl);
      case 4: return launch_p_bits<8, 4, ST>(g, m, nm, s, pdl);
    }
  } else if (R == 4 && LG == 1) {
    return launch_p_bits<4, 1, ST>(g, m, nm, s, pdl);
  }
  return BITLUT_ELAYOUT;
}

}  // namespace

// Batch-1 fast-epilogue lookups through the pack kernel when BITLUT_PACK=1.
// Returns BITLUT_ELAYOUT otherwise or when the shape is outside its envelope
// (the caller then uses gemv_b1_kernel).
int bl_gemv_pack_launch(const blk::GemvArgs& g, const blk::StreamMat* mats, int n_mats, int scale_dtype,
                        cudaStream_t s, bool pdl) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BITLUT_PACK");               // opt-in: 1 enables the pack kernel
    on = e ? atoi(e) != 0 : 0;
  }
  const bl::LayoutV2& L = g.L;
  if (!on || !g.fast || g.n_rows > 1 || L.n_sg != 1 || n_mats < 1 || n_mats > kMaxMatsP) return BITLUT_ELAYOUT;
  return scale_dtype == BITLUT_DT_F16 ? dispatch_p<__half>(g, mats, n_mats, s, pdl)
                                      : dispatch_p<float>(g, mats, n_mats, s, pdl);
}
