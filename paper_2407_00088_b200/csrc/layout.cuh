// Layout v2: the GPU weight layout consumed by the lookup kernels.
//
// Terms:
//   stream   = (output channel c, bit plane p): one int32 staging accumulator
//              per quantization group, exactly the reference's `stage[m]` of
//              plane p (_kernels.py:154-185).
//   tile     = tile_channels consecutive channels; its streams are flattened
//              channel-major (c*bits + p) and cut into 32-stream groups (SG).
//   chunk    = 16 bytes = 32 nibbles = the 32 streams of one SG at one
//              k-group kg (4 activations).  Nibble j of word w holds stream
//              8w+j.  The nibble is the mirror-encoded index
//              x = idx ^ (7 * (idx >> 3)): bit 3 = mirror flag s, bits 0-2 =
//              the half-table slot eff (_kernels.py:175-177 computes the same
//              s/eff at run time; here it is done once, offline).
//   unit     = unit_kg (R) consecutive k-groups of one SG, processed by one lane.
//              Units are interleaved 32 at a time ("unit block", ub): within
//              a unit block the order is [j = kg-in-unit][lane][16 B], so at
//              step j the 32 lanes of a warp touch 512 contiguous bytes
//              (conflict-free LDS.128 from shared memory, coalesced from HBM).
//   tables   = the kernel-format LUT (bitlut_build_lut, mode Q8) uses the
//              same interleave at 8 B per k-group, pairs of k-groups packed:
//              [ub][j/2][lane][2 x 8 B], so one LDG.128 per lane fetches the
//              encoded half tables of two consecutive k-groups.
#pragma once
#include <cstdint>

namespace bl {

struct LayoutV2 {
  int m, k, bits, gs;
  int tile_ch, n_sg, R, Lg;   // channels per tile, SGs per tile, kg per unit, units per group
  int KG, NQ, U;              // k-groups, quant groups, units per SG row
  int n_tiles;

  __host__ __device__ int64_t sg_row_base(int tile, int sg) const {
    return ((int64_t)tile * n_sg + sg) * (int64_t)KG * 16;
  }
  // byte offset of the 16-byte chunk (tile, sg, kg)
  __host__ __device__ int64_t chunk_offset(int tile, int sg, int kg) const {
    int u = kg / R, r = kg - u * R;
    int ub = u >> 5, l = u & 31;
    int nu_b = U - 32 * ub; if (nu_b > 32) nu_b = 32;
    return sg_row_base(tile, sg) + (int64_t)ub * (32 * R * 16) + (int64_t)(r * nu_b + l) * 16;
  }
  // byte offset of k-group kg's 8-byte encoded half table in one table row
  __host__ __device__ int64_t table_offset(int kg) const {
    int u = kg / R, r = kg - u * R;
    int ub = u >> 5, l = u & 31;
    int nu_b = U - 32 * ub; if (nu_b > 32) nu_b = 32;
    return (int64_t)ub * (32 * R * 8) + (int64_t)((r >> 1) * nu_b + l) * 16 + (r & 1) * 8;
  }
};

// Returns BITLUT_OK or an error code; fills L on success.
__host__ __device__ inline int unit_kg_for(int gs) { return ((gs / 4) % 8 == 0) ? 8 : 4; }

inline int make_layout(int m, int k, int bits, int gs, LayoutV2* L) {
  if (bits < 1 || bits > 4) return -1;          // EPARAM
  if (gs < 4 || k <= 0 || m <= 0) return -1;
  if (gs % 16 != 0) return -1;                   // CUDA path: gs multiple of 16
  int gpg = gs / 4;
  if (gpg > 128) return -1;                      // packed int32 accumulator bound
  int R = unit_kg_for(gs);
  int Lg = gpg / R;
  if (Lg & (Lg - 1)) return -1;                  // lanes per group must be a power of two
  if (k % gs != 0) return -4;                    // ELAYOUT
  if (m % 32 != 0) return -4;
  L->m = m; L->k = k; L->bits = bits; L->gs = gs;
  L->tile_ch = (bits == 3) ? 32 : 32 / bits;
  L->n_sg = (bits == 3) ? 3 : 1;
  L->R = R; L->Lg = Lg;
  L->KG = k / 4; L->NQ = k / gs; L->U = L->KG / R;
  L->n_tiles = m / L->tile_ch;
  return 0;
}

// ---- layer-set layout (consumed by bitlut_mpgemv_batch, csrc/gemv_batch.cu) ----
// The same chunks at the same offsets as layout v2, but inside the chunk of
// lane l (l = unit & 31) position pos holds stream pos ^ pmask(l), with
// pmask(l) = bits * bitrev_{log2 tile_ch}(l): the lane reductions of the
// batch kernel then need no selects (b1_core.cuh reduce_lanes_perm).  The
// group scales (zero points) of a tile are stored per unit: unit u holds the
// NCH = max(1, tile_ch / Lg) values of its quantization group g = u / Lg in
// the order of the lane's reduced sums, value j = channel j ^ cmask(u & 31)
// -- one vector load per lane instead of NCH strided 2-byte loads.
__host__ __device__ inline int layer_set_cmask(int lane, int tile_ch) {
  int m = 0;
  for (int o = 1, n = tile_ch >> 1; n >= 1; o <<= 1, n >>= 1)
    if (lane & o) m |= n;
  return m;
}
__host__ __device__ inline int layer_set_nch(const LayoutV2& L) {
  const int nacc = L.bits == 4 ? 8 : 16;                 // accumulators per lane (W1: stream pairs)
  int nv = nacc / L.Lg; if (nv < 1) nv = 1;
  return L.bits == 1 ? 2 * nv : nv;
}
__host__ __device__ inline int64_t layer_set_scale_bytes(const LayoutV2& L, int elem_bytes) {
  return (int64_t)L.U * layer_set_nch(L) * elem_bytes;   // per tile
}

}  // namespace bl
