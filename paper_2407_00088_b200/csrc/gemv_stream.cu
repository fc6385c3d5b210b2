// Batch-1 streaming lookup kernel (fast epilogue, int8 tables, 1/2/4-bit
// weights, layout v2): the decode-path GEMV written for steady-state HBM
// streaming.  Same arithmetic as gemv_b1.cu's fast epilogue (the exact
// integer S = sum_p 2^p P_p per (channel, quantization group), then
// y_c = 0.5 * sum_g ws_cg * (ts_g * S_cg - rs_g [+ 2 (2^(b-1) - z_cg) rs_g]),
// i.e. _kernels.py:179-191 regrouped), different work mapping:
//
//   * a lane owns whole quantization groups: its LG = gs/4/R units of one
//     group are adjacent in the unit block, so the group's integer sum never
//     crosses lanes (no per-unit shuffle reduction);
//   * a slice = 32 consecutive groups of one tile (one per lane); a warp
//     walks a contiguous range of slices, accumulating each channel's fp32
//     partial in registers until its tile changes (one shuffle reduction
//     per tile, not per unit);
//   * every warp streams its own weights through a private 3-slot ring of
//     4 KB sub-slices (cp.async.bulk + mbarrier, issued by lane 0 two
//     sub-slices ahead): no CTA-wide barrier inside the main loop;
//   * lookups with dp4a: W4 adds a channel's 4 planes in one IDP per
//     looked-up word (multipliers 1,2,4,8), W2 gathers the A and Y bytes of
//     one channel into one word (selector built with one prmt per two
//     channels) and adds them with (1,2,-1,-2); W1 keeps the packed
//     (1, 32768) stream pairs;
//   * each CTA owns a contiguous range of whole tiles; the few tiles split
//     between two warps are combined once at the end from shared memory in
//     warp order (deterministic).
// Tables (kernel format, one activation row) live in shared memory for the
// whole launch.
#include "gemv_core.cuh"

namespace {

using namespace blk;

constexpr int kMaxMatsS = 4;
constexpr int kMaxWarps = 16;
constexpr int kSlotsPerWarp = 2;

struct SArgs {
  GemvArgs g;
  int n_mats, total_tiles;
  int nsl;                    // slices per tile row (64 units = two unit blocks each)
  int nslots;                 // ring slots per warp (one slice each)
  blk::StreamMat mats[kMaxMatsS];
  uint32_t tab_off, ts_off, rs_off, rec_off, cnt_off, wb_off, warp_off, bar_off;
};


// Fixed-order transpose-reduce of NV floats over the 32 lanes: halving
// exchanges while more than one value is left, butterfly adds afterwards.
// The lane then holds the full sum of value `base` (returned).
template <int NV>
__device__ __forceinline__ int warp_reduce(float (&v)[NV], int lane) {
  int base = 0;
#pragma unroll
  for (int o = 1, n = NV; o < 32; o <<= 1) {
    if (n > 1) {
      n >>= 1;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; i++) {
        if (i < n) {
          const float send = up ? v[i] : v[i + n];
          const float keep = up ? v[i + n] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (up) base += n;
    } else {
      v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  return base;
}

__device__ __forceinline__ int find_mat_s(const SArgs& a, int tile, int& local) {
  int j = 0;
  while (j + 1 < a.n_mats && tile >= a.mats[j].tile_end) j++;
  local = tile - (j ? a.mats[j - 1].tile_end : 0);
  return j;
}

template <typename ST>
__device__ __forceinline__ uint32_t ld_scale_raw(const void* base, int64_t i) {
  uint32_t r;
  if constexpr (sizeof(ST) == 2) {
    unsigned short h;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(h) : "l"(reinterpret_cast<const __half*>(base) + i));
    r = h;
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(reinterpret_cast<const float*>(base) + i));
  }
  return r;
}
template <typename ST>
__device__ __forceinline__ float raw_to_f32(uint32_t r) {
  if constexpr (sizeof(ST) == 2) return __half2float(__ushort_as_half((unsigned short)r));
  else return __uint_as_float(r);
}

template <typename ST>
__device__ __forceinline__ float ld_scale(const void* base, int64_t i) {
  if constexpr (sizeof(ST) == 2) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(reinterpret_cast<const __half*>(base) + i));
    return __half2float(__ushort_as_half(r));
  } else {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(reinterpret_cast<const float*>(base) + i));
    return r;
  }
}

// Zero-point terms (BASELINE config 1: asymmetric per-group zeros), out of
// line so the common path carries no predicated loads:
// d_c += (2^b - 2 z_c) * rs, i.e. 2 (2^(b-1) - z) rs.
template <typename ST, int N>
__device__ __noinline__ void add_zero_terms(float (&d)[N], const void* zeros, int64_t e0, int stride, float h2,
                                            float rs) {
  const ST* zp = reinterpret_cast<const ST*>(zeros) + e0;
#pragma unroll
  for (int c = 0; c < N; c++, zp += stride) d[c] = fmaf(fmaf(-2.f, bl::to_f32(*zp), h2), rs, d[c]);
}

// Exact integer sums S of one lane's channels (BITLUT_FLAG_COMBINED_PARTIALS),
// out of line so the common path carries no predicated stores.
template <int N>
__device__ __noinline__ void store_partials(int32_t* dst, int stride, const int (&S)[N]) {
#pragma unroll
  for (int c = 0; c < N; c++) dst[(int64_t)c * stride] = S[c];
}

// The R k-steps of one unit: wb / tb point at the unit's chunk / table pair
// in step row 0; `stride` = bytes per k-step row of the unit block (512 for
// full blocks: immediate offsets).
template <int BITS, int NACC, int R, bool FULL>
__device__ __forceinline__ void unit_lookups(const uint8_t* wb, const uint8_t* tb, int stride_rt,
                                             int (&acc)[NACC]) {
  const int stride = FULL ? 512 : stride_rt;
#pragma unroll
  for (int j = 0; j < R; j += 2) {
    const uint4 t = *reinterpret_cast<const uint4*>(tb + (j >> 1) * stride);
    const uint4 wa = *reinterpret_cast<const uint4*>(wb + j * stride);
    const uint4 wc = *reinterpret_cast<const uint4*>(wb + (j + 1) * stride);
    lookup_merged<BITS, NACC>(wa, t.x, t.y, acc);
    lookup_merged<BITS, NACC>(wc, t.z, t.w, acc);
  }
}

template <int BITS, int R, int LG, typename ST>
__global__ void __launch_bounds__(512, 1) gemv_stream_kernel(const __grid_constant__ SArgs a) {
  constexpr int TCH = 32 / BITS;                        // channels per tile
  constexpr int NACC = BITS == 4 ? 8 : 16;              // int accumulators per lane
  constexpr int NCL = LG == 4 ? TCH / 2 : TCH;          // channels a lane scales per group
  constexpr int BLK = 32 * R * 16;                      // bytes of a full unit block
  const GemvArgs& p = a.g;
  const bl::LayoutV2& L = p.L;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  const int NQ = L.NQ, KG = L.KG, U = L.U, nsl = a.nsl, NS = a.nslots;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* bar = bars + warp * NS;
  uint64_t* tbar = bars + NW * NS;
  uint8_t* ring = smem + a.warp_off + (size_t)warp * NS * (2 * BLK);
  const uint8_t* tab = smem + a.tab_off;
  float* tsm = reinterpret_cast<float*>(smem + a.ts_off);
  float* rsm = reinterpret_cast<float*>(smem + a.rs_off);
  float* rec = reinterpret_cast<float*>(smem + a.rec_off);   // [NW*2][TCH]
  int* cnt = reinterpret_cast<int*>(smem + a.cnt_off);        // per CTA tile: warps done

  // ---- this CTA's whole tiles, this warp's contiguous slice range ----
  const int G = gridDim.x;
  const int t0 = (int)((int64_t)a.total_tiles * blockIdx.x / G);
  const int t1 = (int)((int64_t)a.total_tiles * (blockIdx.x + 1) / G);
  const int cs0 = t0 * nsl, ncs = (t1 - t0) * nsl;
  int* wsm = reinterpret_cast<int*>(smem + a.wb_off);           // warp range starts [NW + 1]
  auto wbeg = [&](int w) { return wsm[w]; };
  for (int w = tid; w <= NW; w += blockDim.x) wsm[w] = cs0 + (int)((int64_t)ncs * w / NW);
  __syncthreads();
  const int w0 = wbeg(warp), w1 = wbeg(warp + 1);
  const int nsw = w1 - w0;                              // slices of this warp

  // copy cursor (lane 0): slice w0 + i -> slot i % NS
  int c_tile = nsw > 0 ? w0 / nsl : 0, c_s = nsw > 0 ? w0 - c_tile * nsl : 0;
  const uint8_t* c_base = nullptr;
  auto c_rebase = [&]() {
    int local;
    const blk::StreamMat& mt = a.mats[find_mat_s(a, c_tile, local)];
    c_base = mt.w + L.sg_row_base(local, 0);
  };
  auto issue = [&](int i, uint64_t pol) {
    const int u0 = c_s * 64;
    const uint32_t bytes = (uint32_t)(min(64, U - u0) * R * 16);
    uint64_t* b = bar + i % NS;
    mbar_expect_tx(b, bytes);
    bulk_g2s(ring + (i % NS) * (2 * BLK), c_base + (int64_t)c_s * (2 * BLK), bytes, b, pol);
    if (++c_s == nsl) {
      c_s = 0;
      c_tile++;
      c_rebase();
    }
  };

  // ---- 1. barriers; the first slices stream in before the dependency wait ----
  if (lane == 0) {
    for (int k = 0; k < NS; k++) mbar_init(bar + k, 1);
    if (warp == 0) mbar_init(tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (nsw > 0) {
      c_rebase();
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < NS && i < nsw; i++) issue(i, pol);
    }
  }
  // ---- 2. tables / table scales / row sums come from the previous kernel ----
  if (p.dep.counted) bl::dep_wait(p.dep);
  else if (!p.independent) bl::pdl_wait();
  bl::pdl_launch_dependents();
  if (tid == 0) {
    if (p.dep.counted) bl::fence_proxy_async();
    const uint32_t tb = (uint32_t)KG * 8;
    mbar_expect_tx(tbar, tb);
    for (uint32_t off = 0; off < tb; off += 32768u) {
      const uint32_t nb = tb - off < 32768u ? tb - off : 32768u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + a.tab_off + off)),
          "l"(p.qtab + off), "r"(nb), "r"(smem_u32(tbar))
          : "memory");
    }
  }
  for (int i = tid; i < NQ; i += blockDim.x) {
    tsm[i] = bl::ld_cg_f32(p.tscales + i);
    rsm[i] = bl::ld_cg_f32(p.rowsums + i);
  }
  for (int i = tid; i < t1 - t0; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  mbar_wait(tbar, 0);

  const bool has_zeros = p.zeros != nullptr;
  const float h2 = (float)(2 << (BITS - 1));
  const int lb = lane >> 4;                             // which of the slice's two blocks
  const int p0 = 2 * (lane & 15);                       // first of the lane's two unit positions
  // LG == 4: lanes (2i, 2i+1) share a group; after the pair reduction the
  // even lane scales channels [0, TCH/2), the odd one [TCH/2, TCH)
  const int cb = LG == 4 ? (lane & 1) * (TCH / 2) : 0;
  float y[TCH];
#pragma unroll
  for (int c = 0; c < TCH; c++) y[c] = 0.f;

  // the lane's group of slice (tile, s) and the raw scales of its channels
  auto group_of = [&](int s) { return (s * 64 + 32 * lb + p0) / LG; };
  uint32_t wcur[NCL];
  auto load_ws = [&](uint32_t (&dst)[NCL], int local, int mj, int g) {
    if (g < NQ) {
      const ST* wp = reinterpret_cast<const ST*>(a.mats[mj].wscales) + (((int64_t)local * TCH + cb) * NQ + g);
#pragma unroll
      for (int c = 0; c < NCL; c++, wp += NQ) dst[c] = ld_scale_raw<ST>(wp, 0);
    }
  };
  // y[c] += ws * (ts*S - rs [+ zero term]) for the lane's channels of group g
  auto scale_group = [&](const int (&acc)[NACC], const uint32_t (&wr)[NCL], int tile, int g, int local, int mj) {
    int S[NCL];
    if constexpr (BITS == 1) {
#pragma unroll
      for (int i = 0; i < NCL / 2; i++) {
        const int v = acc[i];                            // P_even + 32768 P_odd
        const int pe = (v << 17) >> 17;
        S[2 * i] = pe;
        S[2 * i + 1] = (v - pe) >> 15;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NCL; i++) S[i] = acc[i];
    }
    if (p.partials) store_partials<NCL>(p.partials + ((int64_t)local * TCH + cb) * NQ + g, NQ, S);
    const float ts = tsm[g], rs = rsm[g];
    float d[NCL];
#pragma unroll
    for (int c = 0; c < NCL; c++) d[c] = fmaf(ts, (float)S[c], -rs);
    if (has_zeros) add_zero_terms<ST, NCL>(d, a.mats[mj].zeros, ((int64_t)local * TCH + cb) * NQ + g, NQ, h2, rs);
    if (LG == 4 && cb) {                                 // static register indices either way
#pragma unroll
      for (int c = 0; c < NCL; c++) y[TCH - NCL + c] = fmaf(raw_to_f32<ST>(wr[c]), d[c], y[TCH - NCL + c]);
    } else {
#pragma unroll
      for (int c = 0; c < NCL; c++) y[c] = fmaf(raw_to_f32<ST>(wr[c]), d[c], y[c]);
    }
  };

  // tile finished by this warp: reduce over the lanes; whole tiles are
  // written, tiles shared with neighbouring warps go through the records and
  // the last warp to finish one combines them in warp order
  auto flush = [&](int tile) {
    const int base = warp_reduce<TCH>(y, lane);
    int local;
    const int mj = find_mat_s(a, tile, local);
    float* out = a.mats[mj].out + (int64_t)local * TCH;
    const bool whole = tile * nsl >= w0 && (tile + 1) * nsl <= w1;
    if (whole) {
      if (lane < TCH) out[base] = 0.5f * y[0];
    } else {
      const int k = tile == w0 / nsl ? 0 : 1;
      if (lane < TCH) rec[(warp * 2 + k) * TCH + base] = y[0];
      // warps whose range meets this tile (contiguous, non-empty ranges)
      int wf = -1, wl = -1;
      for (int w = 0; w < NW; w++) {
        const int b0 = wbeg(w), b1 = wbeg(w + 1);
        if (b0 < b1 && b0 < (tile + 1) * nsl && b1 > tile * nsl) { if (wf < 0) wf = w; wl = w; }
      }
      __threadfence_block();
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(cnt + (tile - t0), 1) == wl - wf;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence_block();
        if (lane < TCH) {
          float acc = 0.f;
          for (int w = wf; w <= wl; w++) {
            const int kw = tile == wbeg(w) / nsl ? 0 : 1;
            acc += *reinterpret_cast<volatile float*>(rec + (w * 2 + kw) * TCH + lane);
          }
          out[lane] = 0.5f * acc;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < TCH; c++) y[c] = 0.f;
  };

  int tile = nsw > 0 ? w0 / nsl : 0, s = nsw > 0 ? w0 - tile * nsl : 0;
  for (int i = 0; i < nsw; i++) {
    int ntile = tile, ns = s + 1;
    if (ns == nsl) { ns = 0; ntile++; }
    int local;
    const int mj = find_mat_s(a, tile, local);
    // this slice's scales: issued before the slot wait, used after the lookups
    if (LG >= 2) load_ws(wcur, local, mj, group_of(s));
    const int ub = 2 * s + lb;                          // the lane's unit block
    const int nu = min(32, U - 32 * ub);
    const int u0 = s * 64 + 32 * lb + p0;               // the lane's first unit
    const uint8_t* tb = tab + (size_t)ub * (32 * R * 8) + p0 * 16;
    mbar_wait(bar + i % NS, (i / NS) & 1);
    const uint8_t* wb = ring + (i % NS) * (2 * BLK) + lb * BLK + p0 * 16;
    int acc[NACC];
#pragma unroll
    for (int q = 0; q < NACC; q++) acc[q] = 0;
    if constexpr (LG == 1) {
      // a unit is a whole group: two groups per lane, one after the other
      uint32_t wr[NCL];
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int g = u0 + u;
        if (g < U) {
          load_ws(wr, local, mj, g);
          if (nu == 32) unit_lookups<BITS, NACC, R, true>(wb + u * 16, tb + u * 16, 512, acc);
          else unit_lookups<BITS, NACC, R, false>(wb + u * 16, tb + u * 16, nu * 16, acc);
          scale_group(acc, wr, tile, g, local, mj);
#pragma unroll
          for (int q = 0; q < NACC; q++) acc[q] = 0;
        }
      }
    } else {
      if (u0 < U) {
        if (nu == 32) {
          unit_lookups<BITS, NACC, R, true>(wb, tb, 512, acc);
          unit_lookups<BITS, NACC, R, true>(wb + 16, tb + 16, 512, acc);
        } else {
          unit_lookups<BITS, NACC, R, false>(wb, tb, nu * 16, acc);
          unit_lookups<BITS, NACC, R, false>(wb + 16, tb + 16, nu * 16, acc);
        }
      }
      if constexpr (LG == 4) {
        // the group's other half is in the neighbour lane: exact int32 pair sum
#pragma unroll
        for (int q = 0; q < NACC / 2; q++) {
          const bool up = (lane & 1) != 0;
          const int send = up ? acc[q] : acc[q + NACC / 2];
          const int keep = up ? acc[q + NACC / 2] : acc[q];
          acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
      }
      if (u0 < U) scale_group(acc, wcur, tile, u0 / LG, local, mj);
    }
    __syncwarp();
    if (lane == 0 && i + NS < nsw) issue(i + NS, policy_evict_first());
    if (ns == 0 || i + 1 == nsw) flush(tile);           // the tile's last slice in this warp
    tile = ntile;
    s = ns;
  }
  bl::dep_signal(p.dep);
  if (p.independent) bl::pdl_wait();                    // keep stream completion order
}

int sm_count_s() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct SPlan {
  uint32_t tab_off, ts_off, rs_off, rec_off, cnt_off, wb_off, warp_off, bar_off, total;
};

SPlan s_plan(const bl::LayoutV2& L, int nw, int ns, int tiles_per_cta) {
  auto al = [](size_t x, size_t a) { return (uint32_t)((x + a - 1) & ~(a - 1)); };
  SPlan s;
  s.tab_off = 0;
  s.ts_off = al((size_t)L.KG * 8, 16);
  s.rs_off = s.ts_off + al((size_t)L.NQ * 4, 16);
  s.rec_off = s.rs_off + al((size_t)L.NQ * 4, 16);
  s.cnt_off = s.rec_off + al((size_t)nw * 2 * L.tile_ch * 4, 16);
  s.wb_off = s.cnt_off + al((size_t)tiles_per_cta * 4, 16);
  s.warp_off = al(s.wb_off + (size_t)(nw + 1) * 4, 128);
  s.bar_off = s.warp_off + (uint32_t)(nw * ns * 2 * 32 * L.R * 16);
  s.total = s.bar_off + (uint32_t)((nw * ns + 1) * 8);
  return s;
}

template <int BITS, int R, int LG, typename ST>
int launch_s(const GemvArgs& g, const blk::StreamMat* mats, int n_mats, cudaStream_t stream, bool pdl) {
  const bl::LayoutV2& L = g.L;
  auto kern = gemv_stream_kernel<BITS, R, LG, ST>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return BITLUT_EINTERNAL;
    configured = true;
  }
  SArgs a;
  a.g = g;
  a.n_mats = n_mats;
  for (int j = 0; j < n_mats; j++) a.mats[j] = mats[j];
  a.total_tiles = mats[n_mats - 1].tile_end;
  a.nsl = (L.U + 63) / 64;
  a.nslots = kSlotsPerWarp;
  static int nw_env = -1;
  if (nw_env < 0) {
    const char* e = getenv("BITLUT_STREAM_WARPS");       // diagnostic override
    nw_env = e ? atoi(e) : 0;
  }
  // warps per CTA: as many as the shared memory holds (one CTA per SM),
  // fewer when the CTA's tiles have fewer slices than that
  const int sms = sm_count_s();
  int tiles_per_cta = (a.total_tiles + sms - 1) / sms;
  int nw = nw_env > 0 ? nw_env : kMaxWarps;
  SPlan s = s_plan(L, nw, a.nslots, tiles_per_cta);
  while (nw > 1 && s.total > 227 * 1024) s = s_plan(L, --nw, a.nslots, tiles_per_cta);
  if (s.total > 227 * 1024) return BITLUT_ELAYOUT;
  int grid = a.total_tiles < sms ? a.total_tiles : sms;
  const int slices_per_cta = (a.total_tiles / grid) * a.nsl;
  if (slices_per_cta < nw) {
    nw = slices_per_cta < 1 ? 1 : slices_per_cta;
    s = s_plan(L, nw, a.nslots, tiles_per_cta);
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, s.total) != cudaSuccess || per_sm < 1)
    return BITLUT_ELAYOUT;
  a.tab_off = s.tab_off; a.ts_off = s.ts_off; a.rs_off = s.rs_off; a.rec_off = s.rec_off;
  a.cnt_off = s.cnt_off; a.wb_off = s.wb_off; a.warp_off = s.warp_off; a.bar_off = s.bar_off;
  if (g.grid_out) *g.grid_out = grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(nw * 32);
  cfg.dynamicSmemBytes = s.total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}

template <int R, int LG, typename ST>
int launch_s_bits(const GemvArgs& g, const blk::StreamMat* m, int nm, cudaStream_t s, bool pdl) {
  switch (g.L.bits) {
    case 1: return launch_s<1, R, LG, ST>(g, m, nm, s, pdl);
    case 2: return launch_s<2, R, LG, ST>(g, m, nm, s, pdl);
    case 4: return launch_s<4, R, LG, ST>(g, m, nm, s, pdl);
  }
  return BITLUT_ELAYOUT;
}

template <typename ST>
int dispatch_s(const GemvArgs& g, const blk::StreamMat* m, int nm, cudaStream_t s, bool pdl) {
  const int R = g.L.R, LG = g.L.Lg;
  if (R == 8) {
    switch (LG) {
      case 1: return launch_s_bits<8, 1, ST>(g, m, nm, s, pdl);
      case 2: return launch_s_bits<8, 2, ST>(g, m, nm, s, pdl);
      case 4: return launch_s_bits<8, 4, ST>(g, m, nm, s, pdl);
    }
  } else if (R == 4 && LG == 1) {
    return launch_s_bits<4, 1, ST>(g, m, nm, s, pdl);
  }
  return BITLUT_ELAYOUT;
}

}  // namespace

// Kernel choice for a batch-1 fast launch: only when forced by
// BITLUT_FLAG_STREAM (or BITLUT_STREAM=1 in the environment).  It used to be
// the automatic choice for long-K launches; the split-K cluster kernel
// (gemv_b1.cu) now beats it there too (8192x28672 W2 15.0 vs 19.8 us, W4
// 24.3 vs 26.7 us overlapped).
bool bl_gemv_stream_wanted(const bl::LayoutV2& L, int total_tiles, bool force) {
  (void)L; (void)total_tiles;
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("BITLUT_STREAM");
    env = e ? atoi(e) : -1;
  }
  if (env >= 0) return env != 0;
  return force;
}

// Batch-1 fast-epilogue lookups through the streaming kernel.  Returns
// BITLUT_ELAYOUT when it is not wanted or the shape is outside its envelope
// (the caller then uses gemv_b1_kernel).
int bl_gemv_stream_launch(const blk::GemvArgs& g, const blk::StreamMat* mats, int n_mats, int scale_dtype,
                          cudaStream_t s, bool pdl) {
  const bl::LayoutV2& L = g.L;
  if (!g.fast || g.n_rows > 1 || L.n_sg != 1 || n_mats < 1 || n_mats > kMaxMatsS) return BITLUT_ELAYOUT;
  if (!bl_gemv_stream_wanted(L, mats[n_mats - 1].tile_end, g.force_stream != 0)) return BITLUT_ELAYOUT;
  return scale_dtype == BITLUT_DT_F16 ? dispatch_s<__half>(g, mats, n_mats, s, pdl)
                                      : dispatch_s<float>(g, mats, n_mats, s, pdl);
}
