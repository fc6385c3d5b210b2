// Per-block table build for g = 4 (kernel.py:226-251: precompute_lut ->
// mirror_consolidate -> quantize_tables / fp16 rounding, and row_sums), one
// thread per k-group.  Shared by the per-call kernel (lut.cu) and the
// persistent pipeline (pipeline.cu).  Bit-exactness notes: lut.cu.
#pragma once
#include "common.cuh"
#include "layout.cuh"

namespace lutk {

// 4 consecutive activations -> f32 (exact for fp16); L2-coherent loads
// because in the pipeline they may come from an earlier op of the launch.
__device__ __forceinline__ void load4(const float* p, float (&v)[4]) {
  const uint4 r = bl::ld_cg_128(p);
  v[0] = __uint_as_float(r.x); v[1] = __uint_as_float(r.y);
  v[2] = __uint_as_float(r.z); v[3] = __uint_as_float(r.w);
}
__device__ __forceinline__ void load4(const __half* p, float (&v)[4]) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  const __half2 h0 = *reinterpret_cast<const __half2*>(&r.x), h1 = *reinterpret_cast<const __half2*>(&r.y);
  v[0] = __low2float(h0); v[1] = __high2float(h0); v[2] = __low2float(h1); v[3] = __high2float(h1);
}

// blockDim.x threads cover k-groups [kg0, kg0 + blockDim.x) of row `row`;
// blockDim.x must be a multiple of gs/4 and <= 256.  sa: 4*blockDim.x floats,
// red: blockDim.x/32 floats of shared memory.
template <int MODE, typename AT>
__device__ __forceinline__ void lut_block(const AT* __restrict__ a, int k, int gs, void* __restrict__ tables,
                                          float* __restrict__ tscales, float* __restrict__ rowsums,
                                          int row, int kg0, float* sa, float* red) {
  const int KG = k >> 2;
  const int gpg = gs >> 2;
  const int NQ = k / gs;
  const int kg = kg0 + threadIdx.x;
  const bool live = kg < KG;

  float v[4] = {0.f, 0.f, 0.f, 0.f};
  if (live) load4(a + (int64_t)row * k + 4 * (int64_t)kg, v);
#pragma unroll
  for (int j = 0; j < 4; j++) sa[threadIdx.x * 4 + j] = v[j];

  // half table (index bit 3 clear): e[idx] = ((s0 a0 + s1 a1) + s2 a2) - a3
  float e[8];
#pragma unroll
  for (int idx = 0; idx < 8; idx++) {
    float x = (idx & 1) ? v[0] : -v[0];
    x = (idx & 2) ? __fadd_rn(x, v[1]) : __fsub_rn(x, v[1]);
    x = (idx & 4) ? __fadd_rn(x, v[2]) : __fsub_rn(x, v[2]);
    e[idx] = __fsub_rn(x, v[3]);
  }

  if (MODE == BITLUT_TABLE_Q8 || MODE == BITLUT_TABLE_X16) {
    float mx = 0.f;
#pragma unroll
    for (int idx = 0; idx < 8; idx++) mx = bl::fmax_nan(mx, fabsf(e[idx]));
    const int seg = gpg < 32 ? gpg : 32;
    for (int o = 1; o < seg; o <<= 1) mx = bl::fmax_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (gpg > 32) {
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
      __syncthreads();
      const int wpg = gpg >> 5;                       // warps per group
      const int w0 = (threadIdx.x >> 5) / wpg * wpg;
      mx = 0.f;
      for (int w = 0; w < wpg; w++) mx = bl::fmax_nan(mx, red[w0 + w]);
    }
    if (MODE == BITLUT_TABLE_X16) {
      // two balanced base-127 digits per entry (bitlut_b200.h BITLUT_TABLE_X16)
      float scale = __fdiv_rn(mx, 16129.0f);
      if (scale == 0.0f) scale = 1.0f;
      uint32_t ph[2] = {0u, 0u}, pl[2] = {0u, 0u};
#pragma unroll
      for (int idx = 0; idx < 8; idx++) {
        float s = __fdiv_rn(e[idx], scale);
        float r = truncf(__fadd_rn(s, copysignf(0.5f, s)));
        r = fminf(fmaxf(r, -16129.f), 16129.f);
        const int q = (int)r;
        const int h = (q + (q >= 0 ? 63 : -63)) / 127;      // nearest, ties cannot occur (127 odd)
        const int lo = q - 127 * h;                          // [-63, 63]
        ph[idx >> 2] |= ((uint32_t)h & 0xffu) << (8 * (idx & 3));
        pl[idx >> 2] |= ((uint32_t)lo & 0xffu) << (8 * (idx & 3));
      }
      if (live) {
        // both digit tables in the kernel's encoded form a = Q - (Q < 0), at
        // the 16-byte-per-k-group offsets of the fp16 tables
        uint4 o;
        o.x = ph[0] - ((ph[0] >> 7) & 0x01010101u); o.y = ph[1] - ((ph[1] >> 7) & 0x01010101u);
        o.z = pl[0] - ((pl[0] >> 7) & 0x01010101u); o.w = pl[1] - ((pl[1] >> 7) & 0x01010101u);
        const int R = bl::unit_kg_for(gs), U = KG / R;
        const int u = kg / R, r = kg - u * R, ub = u >> 5, l = u & 31;
        const int nu_b = min(32, U - 32 * ub);
        const int64_t off = (int64_t)ub * (32 * R * 16) + (int64_t)(r * nu_b + l) * 16;
        BL_CHECK(off >= 0 && off + 16 <= (int64_t)KG * 16);
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(tables) + (int64_t)row * KG * 16 + off) = o;
        if ((kg & (gpg - 1)) == 0) tscales[(int64_t)row * NQ + kg / gpg] = scale;
      }
    } else {
    float scale = __fdiv_rn(mx, 127.0f);
    if (scale == 0.0f) scale = 1.0f;
    uint32_t packed[2] = {0u, 0u};
#pragma unroll
    for (int idx = 0; idx < 8; idx++) {
      float s = __fdiv_rn(e[idx], scale);
      float r = truncf(__fadd_rn(s, copysignf(0.5f, s)));
      r = fminf(fmaxf(r, -127.f), 127.f);
      packed[idx >> 2] |= ((uint32_t)(int)r & 0xffu) << (8 * (idx & 3));
    }
    if (live) {
      // kernel-format table: encoded a = Q - (Q < 0) per byte (gemv.cu "A/B
      // tables"), unit-interleaved like the weights (layout.cuh table_offset)
      const uint32_t e0 = packed[0] - ((packed[0] >> 7) & 0x01010101u);
      const uint32_t e1 = packed[1] - ((packed[1] >> 7) & 0x01010101u);
      const int R = bl::unit_kg_for(gs), U = KG / R;
      const int u = kg / R, r = kg - u * R, ub = u >> 5, l = u & 31;
      const int nu_b = min(32, U - 32 * ub);
      const int64_t off = (int64_t)ub * (32 * R * 8) + (int64_t)((r >> 1) * nu_b + l) * 16 + (r & 1) * 8;
      BL_CHECK(off >= 0 && off + 8 <= (int64_t)KG * 8);
      *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(tables) + (int64_t)row * KG * 8 + off) =
          make_uint2(e0, e1);
      if ((kg & (gpg - 1)) == 0) tscales[(int64_t)row * NQ + kg / gpg] = scale;
    }
    }
  } else {
    // fp16 half table, kernel format: 8 low bytes then 8 high bytes of the
    // 8 entries (byte planes for prmt lookups), unit-interleaved at 16 B
    // per k-group like the weights (layout.cuh chunk order)
    uint32_t lo[2] = {0u, 0u}, hi[2] = {0u, 0u};
#pragma unroll
    for (int idx = 0; idx < 8; idx++) {
      const uint32_t h = __half_as_ushort(__float2half_rn(e[idx]));
      lo[idx >> 2] |= (h & 0xffu) << (8 * (idx & 3));
      hi[idx >> 2] |= (h >> 8) << (8 * (idx & 3));
    }
    if (live) {
      const int R = bl::unit_kg_for(gs), U = KG / R;
      const int u = kg / R, r = kg - u * R, ub = u >> 5, l = u & 31;
      const int nu_b = min(32, U - 32 * ub);
      const int64_t off = (int64_t)ub * (32 * R * 16) + (int64_t)(r * nu_b + l) * 16;
      BL_CHECK(off >= 0 && off + 16 <= (int64_t)KG * 16);
      *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(tables) + (int64_t)row * KG * 16 + off) =
          make_uint4(lo[0], lo[1], hi[0], hi[1]);
    }
  }

  __syncthreads();
  // row sums: the first thread of each quant group adds its gs activations
  // left to right (lut_build.py:191-193)
  if (live && (kg & (gpg - 1)) == 0) {
    // loads 16 ahead of the serial add chain (gs is a multiple of 16)
    const float4* s4 = reinterpret_cast<const float4*>(sa + threadIdx.x * 4);
    float acc = 0.f;
    float4 c0 = s4[0], c1 = s4[1], c2 = s4[2], c3 = s4[3];
    for (int q = 0; q < gs / 4; q += 4) {
      float4 n0 = c0, n1 = c1, n2 = c2, n3 = c3;
      if (q + 4 < gs / 4) { n0 = s4[q + 4]; n1 = s4[q + 5]; n2 = s4[q + 6]; n3 = s4[q + 7]; }
      acc = __fadd_rn(acc, c0.x); acc = __fadd_rn(acc, c0.y); acc = __fadd_rn(acc, c0.z); acc = __fadd_rn(acc, c0.w);
      acc = __fadd_rn(acc, c1.x); acc = __fadd_rn(acc, c1.y); acc = __fadd_rn(acc, c1.z); acc = __fadd_rn(acc, c1.w);
      acc = __fadd_rn(acc, c2.x); acc = __fadd_rn(acc, c2.y); acc = __fadd_rn(acc, c2.z); acc = __fadd_rn(acc, c2.w);
      acc = __fadd_rn(acc, c3.x); acc = __fadd_rn(acc, c3.y); acc = __fadd_rn(acc, c3.z); acc = __fadd_rn(acc, c3.w);
      c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    rowsums[(int64_t)row * NQ + kg / gpg] = acc;
  }
}

}  // namespace lutk
