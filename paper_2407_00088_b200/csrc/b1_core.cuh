// Batch-1 lookup core shared by gemv_b1.cu (per-call kernels) and
// gemv_batch.cu (the batch executor's kernel): the plane-merged k-group
// lookup and the lane reductions.
#pragma once
#include "gemv_core.cuh"

namespace blk {

// The high half of a selector word.  The PRMT lookups, the selector
// preparation (LOP3, PRMT, SHF) and the epilogue's SEL/FSEL/I2FP all issue to
// the ALU pipe and the dot products (IDP) to the FMA-heavy pipe, each at one
// warp instruction per two clocks per scheduler (tools/microbench/pipes2.cu,
// profiles/r02cc_pipes.txt).  W2 has 9 ALU and 4 IDP instructions per weight
// word, so its two shifts go to the IDP pipe (7 + 6): +8 % on the W2 layer
// set.  W1 is already IDP-heavy (7 ALU, 8 IDP) and keeps SHF.
template <bool IDP>
__device__ __forceinline__ uint32_t sel_hi(uint32_t x) {
  if constexpr (IDP) return bl::shr16_idp(x);
  return x >> 16;
}

// Lookup of one k-group for 32 streams with plane-merging multipliers (the
// A/Y form of gemv_core.cuh lookup_kg: A - Y = sQ exactly, Y enters with the
// negated multiplier).
template <int BITS, int NACC>
__device__ __forceinline__ void lookup_kg_merged(const uint4 w, uint32_t a0, uint32_t a1, int (&acc)[NACC]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t x = ws[q];
    const uint32_t xx = x ^ 0x88888888u;
    if constexpr (BITS == 2) {
      // byte b of x = channel 4q+b (nibbles: plane 0, plane 1): the selector
      // [x.b, xx.b] looks up [A_p0, A_p1, Y_p0, Y_p1] in one prmt, dp4a with
      // (1, 2, -1, -2) adds S_c = P0 + 2 P1 -- 13 instead of 15 instructions
      // per 8 lookups
      const uint32_t s01 = bl::prmt(x, xx, 0x5140u), s23 = bl::prmt(x, xx, 0x7362u);
      acc[4 * q + 0] = bl::dp4a(bl::prmt(a0, a1, s01), 0xFEFF0201u, acc[4 * q + 0]);
      acc[4 * q + 1] = bl::dp4a(bl::prmt(a0, a1, sel_hi<true>(s01)), 0xFEFF0201u, acc[4 * q + 1]);
      acc[4 * q + 2] = bl::dp4a(bl::prmt(a0, a1, s23), 0xFEFF0201u, acc[4 * q + 2]);
      acc[4 * q + 3] = bl::dp4a(bl::prmt(a0, a1, sel_hi<true>(s23)), 0xFEFF0201u, acc[4 * q + 3]);
      continue;
    }
    const uint32_t A0 = bl::prmt(a0, a1, x), Y0 = bl::prmt(a0, a1, xx);
    // W4: 7 ALU + 4 IDP per word -> one of the two shifts on the IDP pipe
    const uint32_t A1 = bl::prmt(a0, a1, sel_hi<BITS == 4>(x)), Y1 = bl::prmt(a0, a1, xx >> 16);
    if constexpr (BITS == 4) {
      // bytes 0..3 of A0/Y0 = planes 0..3 of channel 2q, of A1/Y1: channel
      // 2q+1; dp4a with (1,2,4,8) adds a channel's planes in one instruction
      acc[2 * q] = bl::dp4a(A0, 0x08040201u, acc[2 * q]);
      acc[2 * q] = bl::dp4a(Y0, 0xF8FCFEFFu, acc[2 * q]);
      acc[2 * q + 1] = bl::dp4a(A1, 0x08040201u, acc[2 * q + 1]);
      acc[2 * q + 1] = bl::dp4a(Y1, 0xF8FCFEFFu, acc[2 * q + 1]);
    } else {
      // W1: pair i = channels (2i, 2i+1), packed P_even + 32768 P_odd
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

// The same k-group of weights against the tables of TWO activation rows
// (mpGEMM row blocks): the selector preparation -- the LOP3, the shifts and
// W2's two selector PRMTs -- is done once per weight word and only the
// lookups and dot products repeat per row (W2: 5.5 ALU + 5 IDP instructions
// per word and row instead of 7 + 6).  Same sums as lookup_kg_merged.
template <int BITS, int NACC>
__device__ __forceinline__ void lookup_kg_merged2(const uint4 w, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1,
                                                  int (&accA)[NACC], int (&accB)[NACC]) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t x = ws[q];
    const uint32_t xx = x ^ 0x88888888u;
    if constexpr (BITS == 2) {
      const uint32_t s01 = bl::prmt(x, xx, 0x5140u), s23 = bl::prmt(x, xx, 0x7362u);
      const uint32_t h01 = sel_hi<true>(s01), h23 = sel_hi<true>(s23);
      accA[4 * q + 0] = bl::dp4a(bl::prmt(a0, a1, s01), 0xFEFF0201u, accA[4 * q + 0]);
      accA[4 * q + 1] = bl::dp4a(bl::prmt(a0, a1, h01), 0xFEFF0201u, accA[4 * q + 1]);
      accA[4 * q + 2] = bl::dp4a(bl::prmt(a0, a1, s23), 0xFEFF0201u, accA[4 * q + 2]);
      accA[4 * q + 3] = bl::dp4a(bl::prmt(a0, a1, h23), 0xFEFF0201u, accA[4 * q + 3]);
      accB[4 * q + 0] = bl::dp4a(bl::prmt(b0, b1, s01), 0xFEFF0201u, accB[4 * q + 0]);
      accB[4 * q + 1] = bl::dp4a(bl::prmt(b0, b1, h01), 0xFEFF0201u, accB[4 * q + 1]);
      accB[4 * q + 2] = bl::dp4a(bl::prmt(b0, b1, s23), 0xFEFF0201u, accB[4 * q + 2]);
      accB[4 * q + 3] = bl::dp4a(bl::prmt(b0, b1, h23), 0xFEFF0201u, accB[4 * q + 3]);
      continue;
    }
    const uint32_t xh = sel_hi<BITS == 4>(x), xxh = xx >> 16;
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const uint32_t t0 = r ? b0 : a0, t1 = r ? b1 : a1;
      int (&acc)[NACC] = r ? accB : accA;
      const uint32_t A0 = bl::prmt(t0, t1, x), Y0 = bl::prmt(t0, t1, xx);
      const uint32_t A1 = bl::prmt(t0, t1, xh), Y1 = bl::prmt(t0, t1, xxh);
      if constexpr (BITS == 4) {
        acc[2 * q] = bl::dp4a(A0, 0x08040201u, acc[2 * q]);
        acc[2 * q] = bl::dp4a(Y0, 0xF8FCFEFFu, acc[2 * q]);
        acc[2 * q + 1] = bl::dp4a(A1, 0x08040201u, acc[2 * q + 1]);
        acc[2 * q + 1] = bl::dp4a(Y1, 0xF8FCFEFFu, acc[2 * q + 1]);
      } else {
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
}

// Reduce NV values across the lanes that differ in lane bits [O0, O1):
// halving exchanges while more than one value is left (each lane keeps a
// disjoint half, no redundant adds), plain butterfly adds afterwards.
// Returns the index of the lane's first remaining value; the count is
// reduced_count<NV, O0, O1>().
template <int NV, int O0, int O1>
__host__ __device__ constexpr int reduced_count() {
  int n = NV;
  for (int o = O0; o < O1; o <<= 1)
    if (n > 1) n >>= 1;
  return n;
}

// The index reduce_lanes<NV, O0, O1> returns for this lane (it depends on the lane only).
template <int NV, int O0, int O1>
__device__ __forceinline__ int lane_base(int lane) {
  int base = 0;
#pragma unroll
  for (int o = O0, n = NV; o < O1; o <<= 1) {
    if (n > 1) {
      n >>= 1;
      if (lane & o) base += n;
    }
  }
  return base;
}

template <int NV, int O0, int O1, typename T>
__device__ __forceinline__ int reduce_lanes(T (&v)[NV], int lane) {
  int base = 0;
#pragma unroll
  for (int o = O0, n = NV; o < O1; o <<= 1) {
    if (n > 1) {
      n >>= 1;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; i++) {
        if (i < n) {
          const T send = up ? v[i] : v[i + n];
          const T keep = up ? v[i + n] : v[i];
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

// ---- layer-set layout (layout.cuh: lane-permuted chunks) ----
// In a chunk of lane l, position pos holds stream pos ^ (BITS * perm_mask<TCH>(l)):
// value index i of lane l means logical index i ^ mask(l), and the mask of
// the partner at halving step o differs exactly in the bit that step splits
// on, so BOTH lanes keep the low half and send the high half -- the halving
// needs no selects (reduce_lanes spends 2 SEL/FSEL per exchanged value), and
// after all steps lane l holds logical index perm_mask(l).
template <int NIDX>
__host__ __device__ constexpr int perm_mask(int lane) {
  int m = 0;
  for (int o = 1, n = NIDX >> 1; n >= 1; o <<= 1, n >>= 1)
    if (lane & o) m |= n;
  return m;
}

template <int NV, int O0, int O1, typename T>
__device__ __forceinline__ void reduce_lanes_perm(T (&v)[NV]) {
#pragma unroll
  for (int o = O0, n = NV; o < O1; o <<= 1) {
    if (n > 1) {
      n >>= 1;
#pragma unroll
      for (int i = 0; i < NV / 2; i++)
        if (i < n) v[i] = v[i] + __shfl_xor_sync(0xffffffffu, v[i + n], o);
    } else {
      v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}

// NB consecutive bytes from shared memory (NB = 4, 8 or a multiple of 16)
template <int NB>
__device__ __forceinline__ void lds_vec(const void* p, uint32_t (&d)[(NB + 3) / 4]) {
  if constexpr (NB % 16 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 16; i++) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      d[4 * i] = v.x; d[4 * i + 1] = v.y; d[4 * i + 2] = v.z; d[4 * i + 3] = v.w;
    }
  } else if constexpr (NB == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    d[0] = v.x; d[1] = v.y;
  } else if constexpr (NB == 4) {
    d[0] = *reinterpret_cast<const uint32_t*>(p);
  } else {
    static_assert(NB == 2, "vector width");
    d[0] = *reinterpret_cast<const uint16_t*>(p);
  }
}

// element j of a packed fp16 / fp32 vector held in 32-bit registers
template <typename ST, int NW>
__device__ __forceinline__ float vec_elem(const uint32_t (&d)[NW], int j) {
  if constexpr (sizeof(ST) == 4) {
    return __uint_as_float(d[j]);
  } else {
    const __half2 h = *reinterpret_cast<const __half2*>(&d[j >> 1]);
    return (j & 1) ? __high2float(h) : __low2float(h);
  }
}

}  // namespace blk
