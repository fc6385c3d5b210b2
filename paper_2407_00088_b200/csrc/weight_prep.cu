// Offline weight pipeline on the GPU (reference: pkg/src/bitlut/weight_prep.py).
//
//   decompose_bits   q (m,k) -> plane indices (bits, m, k/g)       :86-105
//   pack_v1          indices -> v1 planes (tile-major, interleaved)  :193-246
//   unpack_v1        v1 planes -> indices                           :249-257
//   repack_gpu       indices -> layout v2 (layout.cuh)     [north-star kernel (1)]
//   unrepack_gpu     layout v2 -> indices
//
// All are one-thread-per-output-element kernels: offline, HBM-bound byte
// shuffles with no reuse, so no shared-memory staging is needed; grids are
// sized in multiples of 148 SMs x 8 resident blocks.
#include "common.cuh"
#include "layout.cuh"

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  const int64_t cap = 148 * 8 * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

inline int slot_bits(int g) { return g == 1 ? 1 : (g == 2 ? 2 : (g <= 4 ? 4 : 8)); }

__device__ __forceinline__ int bitrev(int v, int nbits) {
  int r = 0;
  for (int i = 0; i < nbits; i++) r |= ((v >> i) & 1) << (nbits - 1 - i);
  return r;
}

// ---- decompose_bits (weight_prep.py:86-105) ----
__global__ void decompose_kernel(const uint8_t* __restrict__ q, int m, int k, int bits, int g,
                                 uint8_t* __restrict__ idx) {
  const int kgt = k / g;
  const int64_t total = (int64_t)m * kgt;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / kgt;
    int kg = (int)(t - row * kgt);
    const uint8_t* src = q + row * k + (int64_t)kg * g;
    uint32_t v[8];
    for (int j = 0; j < g; j++) v[j] = src[j];
    for (int i = 0; i < bits; i++) {
      uint32_t x = 0;
      for (int j = 0; j < g; j++) x |= ((v[j] >> i) & 1u) << j;
      idx[(int64_t)i * total + t] = (uint8_t)x;
    }
  }
}

// v1 stream position -> (row, kg) of the plane (docs/formats.md:60-71):
// order (mb, kb, lb, kg-in-tile, lane).
__device__ __forceinline__ void v1_stream_to_rc(int64_t pos, int m_tile, int ktg, int lanes,
                                                int kgt, int64_t* row, int* kg) {
  const int64_t tile_sz = (int64_t)m_tile * ktg;
  const int n_kb = kgt / ktg;
  int64_t tile = pos / tile_sz;
  int64_t rem = pos - tile * tile_sz;
  int64_t mb = tile / n_kb;
  int kb = (int)(tile - mb * n_kb);
  int lb_sz = lanes * ktg;
  int lb = (int)(rem / lb_sz);
  int r2 = (int)(rem - (int64_t)lb * lb_sz);
  int kgi = r2 / lanes;
  int lane = r2 - kgi * lanes;
  *row = mb * m_tile + lb * lanes + lane;
  *kg = kb * ktg + kgi;
}

// ---- pack_and_permute, v1 (weight_prep.py:131-156, 193-246) ----
// One thread per output byte.  Byte j of an interleave unit (per*lanes
// indices) holds, in slot s (bits s*sb .. s*sb+sb-1), the index at unit
// position bitrev(s)*lanes + j: that is what the reference's recursive
// low/high split produces (weight_prep.py:150-155).
__global__ void pack_v1_kernel(const uint8_t* __restrict__ idx, int bits, int m, int k, int g,
                               int m_tile, int k_tile, int lanes, uint8_t* __restrict__ planes) {
  const int kgt = k / g;
  const int sb = g == 1 ? 1 : (g == 2 ? 2 : (g <= 4 ? 4 : 8));
  const int per = 8 / sb;
  const int lg_per = per == 1 ? 0 : (per == 2 ? 1 : (per == 4 ? 2 : 3));
  const int ktg = k_tile / g;
  const int64_t plane_idx = (int64_t)m * kgt;
  const int64_t plane_bytes = plane_idx / per;
  const int64_t total = plane_bytes * bits;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / plane_bytes);
    int64_t p = t - (int64_t)i * plane_bytes;
    int64_t unit = p / lanes;
    int j = (int)(p - unit * lanes);
    uint32_t byte = 0;
    for (int s = 0; s < per; s++) {
      int64_t pos = unit * per * lanes + (int64_t)bitrev(s, lg_per) * lanes + j;
      int64_t row; int kg;
      v1_stream_to_rc(pos, m_tile, ktg, lanes, kgt, &row, &kg);
      byte |= (uint32_t)idx[(int64_t)i * plane_idx + row * kgt + kg] << (s * sb);
    }
    planes[t] = (uint8_t)byte;
  }
}

// ---- unpack_planes, v1 (weight_prep.py:249-257) ----  one thread per index
__global__ void unpack_v1_kernel(const uint8_t* __restrict__ planes, int bits, int m, int k, int g,
                                 int m_tile, int k_tile, int lanes, uint8_t* __restrict__ idx) {
  const int kgt = k / g;
  const int sb = g == 1 ? 1 : (g == 2 ? 2 : (g <= 4 ? 4 : 8));
  const int per = 8 / sb;
  const int lg_per = per == 1 ? 0 : (per == 2 ? 1 : (per == 4 ? 2 : 3));
  const int ktg = k_tile / g;
  const int64_t plane_idx = (int64_t)m * kgt;
  const int64_t plane_bytes = plane_idx / per;
  const int64_t total = plane_idx * bits;
  const int64_t tile_sz = (int64_t)m_tile * ktg;
  const int n_kb = kgt / ktg;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / plane_idx);
    int64_t rc = t - (int64_t)i * plane_idx;
    int64_t row = rc / kgt;
    int kg = (int)(rc - row * kgt);
    // (row, kg) -> v1 stream position
    int64_t mb = row / m_tile;
    int rin = (int)(row - mb * m_tile);
    int lb = rin / lanes, lane = rin - lb * lanes;
    int kb = kg / ktg, kgi = kg - kb * ktg;
    int64_t pos = (mb * n_kb + kb) * tile_sz + (int64_t)lb * lanes * ktg + (int64_t)kgi * lanes + lane;
    int64_t unit = pos / (per * lanes);
    int upos = (int)(pos - unit * per * lanes);
    int tslot = upos / lanes, j = upos - tslot * lanes;
    int s = bitrev(tslot, lg_per);
    uint32_t byte = planes[(int64_t)i * plane_bytes + unit * lanes + j];
    idx[t] = (uint8_t)((byte >> (s * sb)) & ((1u << sb) - 1u));
  }
}

// ---- repack to layout v2 (north-star kernel 1) ----  one thread per 16-byte chunk
__global__ void repack_kernel(const uint8_t* __restrict__ idx, bl::LayoutV2 L, uint8_t* __restrict__ out) {
  const int64_t chunks = (int64_t)L.n_tiles * L.n_sg * L.KG;
  const int64_t plane = (int64_t)L.m * L.KG;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    int kg = (int)(t % L.KG);
    int64_t ts = t / L.KG;
    int sg = (int)(ts % L.n_sg);
    int tile = (int)(ts / L.n_sg);
    uint32_t w[4] = {0, 0, 0, 0};
    for (int s = 0; s < 32; s++) {
      int f = sg * 32 + s;
      int c = f / L.bits, p = f - c * L.bits;
      int64_t row = (int64_t)tile * L.tile_ch + c;
      uint32_t x = idx[(int64_t)p * plane + row * L.KG + kg];
      x ^= 7u * (x >> 3);                    // mirror encoding: (s, eff)
      w[s >> 3] |= x << (4 * (s & 7));
    }
    *reinterpret_cast<uint4*>(out + L.chunk_offset(tile, sg, kg)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void unrepack_kernel(const uint8_t* __restrict__ in, bl::LayoutV2 L, uint8_t* __restrict__ idx) {
  const int64_t chunks = (int64_t)L.n_tiles * L.n_sg * L.KG;
  const int64_t plane = (int64_t)L.m * L.KG;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    int kg = (int)(t % L.KG);
    int64_t ts = t / L.KG;
    int sg = (int)(ts % L.n_sg);
    int tile = (int)(ts / L.n_sg);
    uint4 v = *reinterpret_cast<const uint4*>(in + L.chunk_offset(tile, sg, kg));
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    for (int s = 0; s < 32; s++) {
      int f = sg * 32 + s;
      int c = f / L.bits, p = f - c * L.bits;
      int64_t row = (int64_t)tile * L.tile_ch + c;
      uint32_t x = (w[s >> 3] >> (4 * (s & 7))) & 15u;
      x ^= 7u * (x >> 3);                    // the encoding is an involution
      idx[(int64_t)p * plane + row * L.KG + kg] = (uint8_t)x;
    }
  }
}

// ---- layer-set layout (layout.cuh) ----  one thread per 16-byte chunk:
// nibble pos of the output = nibble pos ^ pmask(lane) of the v2 chunk (an
// involution, so the same kernel converts back)
__global__ void layer_set_weights_kernel(const uint8_t* __restrict__ in, bl::LayoutV2 L, uint8_t* __restrict__ out) {
  const int64_t chunks = (int64_t)L.n_tiles * L.KG;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int kg = (int)(t % L.KG);
    const int tile = (int)(t / L.KG);
    const int64_t off = L.chunk_offset(tile, 0, kg);
    const int lane = (kg / L.R) & 31;
    const int pmask = L.bits * bl::layer_set_cmask(lane, L.tile_ch);
    const uint4 v = *reinterpret_cast<const uint4*>(in + off);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4] = {0, 0, 0, 0};
    for (int pos = 0; pos < 32; pos++) {
      const int src = pos ^ pmask;
      o[pos >> 3] |= ((w[src >> 3] >> (4 * (src & 7))) & 15u) << (4 * (pos & 7));
    }
    *reinterpret_cast<uint4*>(out + off) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// group scales / zero points (m, NQ) -> per tile, per unit, the lane's NCH values
template <typename ST>
__global__ void layer_set_scales_kernel(const ST* __restrict__ in, bl::LayoutV2 L, int nch, ST* __restrict__ out) {
  const int64_t per_tile = (int64_t)L.U * nch;
  const int64_t total = per_tile * L.n_tiles;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(t / per_tile);
    const int r = (int)(t - (int64_t)tile * per_tile);
    const int u = r / nch, j = r - u * nch;
    const int c = j ^ bl::layer_set_cmask(u & 31, L.tile_ch);
    out[t] = in[((int64_t)tile * L.tile_ch + c) * L.NQ + u / L.Lg];
  }
}

int check_v1(int bits, int m, int k, int g, int m_tile, int k_tile, int lanes) {
  if (bits < 1 || bits > 4 || g < 1 || g > 8 || lanes < 1 || m_tile < 1 || k_tile < 1)
    return BITLUT_EPARAM;
  if (k % g != 0 || k_tile % g != 0 || m_tile % lanes != 0) return BITLUT_ELAYOUT;
  if (m % m_tile != 0 || k % k_tile != 0) return BITLUT_ELAYOUT;
  int per = 8 / slot_bits(g);
  if ((k_tile / g) % per != 0) return BITLUT_ELAYOUT;
  return BITLUT_OK;
}

}  // namespace

extern "C" int bitlut_gpu_layout_query(int m, int k, int bits, int group_size, bitlut_gpu_layout* out) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc != 0) return rc;
  if (out) {
    out->m = m; out->k = k; out->bits = bits; out->group_size = group_size;
    out->tile_channels = L.tile_ch; out->stream_groups = L.n_sg;
    out->unit_kg = L.R; out->lanes_per_group = L.Lg;
    out->bytes = (int64_t)m * bits * (k / 4) / 2;
  }
  return BITLUT_OK;
}

extern "C" int bitlut_decompose_bits(const uint8_t* q, int m, int k, int bits, int g,
                                     uint8_t* indices, void* stream) {
  if (bits < 1 || bits > 4 || g < 1 || g > 8 || m < 0 || k < 0) return BITLUT_EPARAM;
  if (k % g != 0) return BITLUT_ELAYOUT;
  int64_t n = (int64_t)m * (k / g);
  if (n == 0) return BITLUT_OK;
  decompose_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(q, m, k, bits, g, indices);
  return bl_launch_status();
}

extern "C" int bitlut_pack_v1(const uint8_t* indices, int bits, int m, int k, int g,
                              int m_tile, int k_tile, int lanes, uint8_t* planes, void* stream) {
  int rc = check_v1(bits, m, k, g, m_tile, k_tile, lanes);
  if (rc) return rc;
  int64_t n = (int64_t)m * (k / g) / (8 / slot_bits(g)) * bits;
  if (n == 0) return BITLUT_OK;
  pack_v1_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(indices, bits, m, k, g, m_tile,
                                                                     k_tile, lanes, planes);
  return bl_launch_status();
}

extern "C" int bitlut_unpack_v1(const uint8_t* planes, int bits, int m, int k, int g,
                                int m_tile, int k_tile, int lanes, uint8_t* indices, void* stream) {
  int rc = check_v1(bits, m, k, g, m_tile, k_tile, lanes);
  if (rc) return rc;
  int64_t n = (int64_t)m * (k / g) * bits;
  if (n == 0) return BITLUT_OK;
  unpack_v1_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(planes, bits, m, k, g, m_tile,
                                                                       k_tile, lanes, indices);
  return bl_launch_status();
}

extern "C" int bitlut_repack_gpu(const uint8_t* indices, int bits, int m, int k, int group_size,
                                 uint8_t* wgpu, void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  int64_t n = (int64_t)L.n_tiles * L.n_sg * L.KG;
  repack_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(indices, L, wgpu);
  return bl_launch_status();
}

extern "C" int bitlut_unrepack_gpu(const uint8_t* wgpu, int bits, int m, int k, int group_size,
                                   uint8_t* indices, void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  int64_t n = (int64_t)L.n_tiles * L.n_sg * L.KG;
  unrepack_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(wgpu, L, indices);
  return bl_launch_status();
}

// Layer-set layout (the operand format of bitlut_mpgemv_batch): see layout.cuh.
extern "C" int64_t bitlut_layer_set_scales_bytes(int m, int k, int bits, int group_size, int scale_dtype) {
  bl::LayoutV2 L;
  if (bl::make_layout(m, k, bits, group_size, &L) != 0 || L.n_sg != 1) return -1;
  if (scale_dtype != BITLUT_DT_F32 && scale_dtype != BITLUT_DT_F16) return -1;
  return bl::layer_set_scale_bytes(L, scale_dtype == BITLUT_DT_F16 ? 2 : 4) * L.n_tiles;
}

extern "C" int bitlut_layer_set_weights(const uint8_t* wgpu, int bits, int m, int k, int group_size,
                                        uint8_t* out, void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (L.n_sg != 1) return BITLUT_ELAYOUT;
  if (!wgpu || !out || wgpu == out) return BITLUT_EPARAM;
  int64_t n = (int64_t)L.n_tiles * L.KG;
  layer_set_weights_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(wgpu, L, out);
  return bl_launch_status();
}

extern "C" int bitlut_layer_set_scales(const void* scales, int scale_dtype, int bits, int m, int k,
                                       int group_size, void* out, void* stream) {
  bl::LayoutV2 L;
  int rc = bl::make_layout(m, k, bits, group_size, &L);
  if (rc) return rc;
  if (L.n_sg != 1) return BITLUT_ELAYOUT;
  if (!scales || !out || scales == out) return BITLUT_EPARAM;
  const int nch = bl::layer_set_nch(L);
  int64_t n = (int64_t)L.n_tiles * L.U * nch;
  if (scale_dtype == BITLUT_DT_F16)
    layer_set_scales_kernel<__half><<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const __half*>(scales), L, nch, reinterpret_cast<__half*>(out));
  else if (scale_dtype == BITLUT_DT_F32)
    layer_set_scales_kernel<float><<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float*>(scales), L, nch, reinterpret_cast<float*>(out));
  else
    return BITLUT_EPARAM;
  return bl_launch_status();
}
