/*
 * C restatement of the reference's CPU hot path -- TEST INFRASTRUCTURE ONLY
 * (checker for tests/, smoke() and bench.py's cpu_baseline / --impl
 * reference legs; never linked into the product).
 *
 * Restates, for g = 4, with the reference's exact float32 operation order
 * (compiled with -ffp-contract=off: no fused multiply-add, like the
 * reference's numba code):
 *   lut_build.py:105-127  precompute_lut (half tables, doubling order)
 *   lut_build.py:153-179  quantize_tables
 *   lut_build.py:182-194  row_sums
 *   _kernels.py:141-192   gemv_q8_vector  (walks the v1 packed planes with
 *                         the byte decode of weight_prep.py:179-190)
 *   _kernels.py:85-138    gemv_real       (scalar-real, fp32 tables)
 *   kernel.py:254-263     M-block slicing over threads (OpenMP here; outputs
 *                         are independent of the thread count).
 *   _kernels.py:20-82     quantize_groups (core.py:227-262 quantize_weights),
 *                         with numba's types: the products x*l and sum(x*l)
 *                         in float64 (float32 * int64 promotes), sum(l*l) in
 *                         float32, candidate scores in float64, round() half
 *                         to even -- pinned by sha256 to the reference's own
 *                         output (tests/golden/nmse.json).
 * The v1 layout comes from weight_prep.py:193-246 (pack it with the numpy
 * oracle or the CUDA bitlut_pack_v1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* half tables: tabs (KG, 8) float, entry idx (bit 3 clear) = ((+-a0 +- a1) +- a2) - a3 */
static void half_tables(const float* a, int k, float* tabs) {
  for (int kg = 0; kg < k / 4; kg++) {
    const float* v = a + 4 * kg;
    for (int idx = 0; idx < 8; idx++) {
      float x = (idx & 1) ? v[0] : -v[0];
      x = (idx & 2) ? x + v[1] : x - v[1];
      x = (idx & 4) ? x + v[2] : x - v[2];
      tabs[kg * 8 + idx] = x - v[3];
    }
  }
}

void orc_tables_q8(const float* a, int k, int gs, int8_t* qtab, float* tscales, float* rowsums,
                   float* scratch /* (k/4)*8 floats */) {
  const int KG = k / 4, gpg = gs / 4, NQ = k / gs;
  half_tables(a, k, scratch);
  for (int gq = 0; gq < NQ; gq++) {
    float mx = 0.f;
    for (int i = gq * gpg * 8; i < (gq + 1) * gpg * 8; i++) {
      float v = fabsf(scratch[i]);
      if (v > mx) mx = v;
    }
    float s = mx / 127.0f;
    if (s == 0.0f) s = 1.0f;
    tscales[gq] = s;
    for (int i = gq * gpg * 8; i < (gq + 1) * gpg * 8; i++) {
      float sc = scratch[i] / s;
      float r = truncf(sc + copysignf(0.5f, sc));
      if (r > 127.f) r = 127.f;
      if (r < -127.f) r = -127.f;
      qtab[i] = (int8_t)r;
    }
    float acc = 0.f;
    for (int j = 0; j < gs; j++) acc += a[gq * gs + j];
    rowsums[gq] = acc;
  }
  (void)KG;
}

void orc_tables_real(const float* a, int k, int gs, float* tabs, float* rowsums) {
  const int NQ = k / gs;
  half_tables(a, k, tabs);
  for (int gq = 0; gq < NQ; gq++) {
    float acc = 0.f;
    for (int j = 0; j < gs; j++) acc += a[gq * gs + j];
    rowsums[gq] = acc;
  }
}

/* _kernels.py:141-192 over M-blocks [mb0, mb1); g = 4, 2 indices per byte */
static void gemv_q8_vector(const uint8_t* planes, int64_t plane_bytes, const int8_t* qtabs,
                           const float* tscales, const float* wscales, const float* rowsums,
                           float* out, int K, int bits, int m_tile, int k_tile, int lanes, int gs,
                           int mb0, int mb1) {
  const int g = 4, per = 2;
  const int KG = K / g, ktg = k_tile / g, gpg = gs / g, n_kb = K / k_tile, n_lb = m_tile / lanes;
  const int64_t mb_bytes = (int64_t)m_tile * KG / per;
  const int NQ = K / gs;
  int32_t* stage = (int32_t*)calloc((size_t)m_tile, sizeof(int32_t));
  uint8_t buf[64];
  for (int i = 0; i < bits; i++) {
    const float pf = (float)(0.5 * (double)(1 << i));
    const uint8_t* pl = planes + (int64_t)i * plane_bytes;
    for (int mb = mb0; mb < mb1; mb++) {
      memset(stage, 0, sizeof(int32_t) * (size_t)m_tile);
      int64_t pos = mb * mb_bytes;
      for (int kb = 0; kb < n_kb; kb++) {
        for (int lb = 0; lb < n_lb; lb++) {
          const int moff = lb * lanes;
          for (int u = 0; u < ktg / per; u++) {
            const int kgu = kb * ktg + u * per;
            for (int j = 0; j < lanes; j++) buf[j] = pl[pos + j];
            for (int t = 0; t < per; t++) {
              const int kg = kgu + t;
              for (int j = 0; j < lanes; j++) {
                int32_t idx = t ? (buf[j] >> 4) : (buf[j] & 15);
                int32_t s = idx >> 3;
                int32_t eff = idx ^ (15 * s);
                int32_t v = qtabs[kg * 8 + eff];
                stage[moff + j] += (v ^ -s) + s;
              }
              if ((kg + 1) % gpg == 0) {
                const int gq = kg / gpg;
                const float f = pf * tscales[gq];
                for (int j = 0; j < lanes; j++) {
                  const int64_t m = (int64_t)mb * m_tile + moff + j;
                  out[m] += f * wscales[m * NQ + gq] * (float)stage[moff + j];
                  stage[moff + j] = 0;
                }
              }
            }
            pos += lanes;
          }
        }
      }
    }
  }
  for (int64_t m = (int64_t)mb0 * m_tile; m < (int64_t)mb1 * m_tile; m++) {
    float s = 0.f;
    for (int gq = 0; gq < NQ; gq++) s += wscales[m * NQ + gq] * rowsums[gq];
    out[m] -= 0.5f * s;
  }
  free(stage);
}

/* _kernels.py:85-138 (scalar-real) over M-blocks [mb0, mb1) */
static void gemv_real(const uint8_t* planes, int64_t plane_bytes, const float* tabs,
                      const float* wscales, const float* rowsums, float* out, int K, int bits,
                      int m_tile, int k_tile, int lanes, int gs, int mb0, int mb1) {
  const int g = 4, per = 2;
  const int KG = K / g, ktg = k_tile / g, gpg = gs / g, n_kb = K / k_tile, n_lb = m_tile / lanes;
  const int64_t mb_bytes = (int64_t)m_tile * KG / per;
  const int NQ = K / gs;
  float* stage = (float*)calloc((size_t)m_tile, sizeof(float));
  uint8_t buf[64];
  for (int i = 0; i < bits; i++) {
    const float pf = (float)(0.5 * (double)(1 << i));
    const uint8_t* pl = planes + (int64_t)i * plane_bytes;
    for (int mb = mb0; mb < mb1; mb++) {
      for (int j = 0; j < m_tile; j++) stage[j] = 0.f;
      int64_t pos = mb * mb_bytes;
      for (int kb = 0; kb < n_kb; kb++) {
        for (int lb = 0; lb < n_lb; lb++) {
          const int moff = lb * lanes;
          for (int u = 0; u < ktg / per; u++) {
            const int kgu = kb * ktg + u * per;
            for (int j = 0; j < lanes; j++) buf[j] = pl[pos + j];
            for (int t = 0; t < per; t++) {
              const int kg = kgu + t;
              for (int j = 0; j < lanes; j++) {
                int32_t idx = t ? (buf[j] >> 4) : (buf[j] & 15);
                int32_t s = idx >> 3;
                int32_t eff = idx ^ (15 * s);
                float v = tabs[kg * 8 + eff];
                if (s == 1) v = -v;
                stage[moff + j] += v;
              }
              if ((kg + 1) % gpg == 0) {
                const int gq = kg / gpg;
                for (int j = 0; j < lanes; j++) {
                  const int64_t m = (int64_t)mb * m_tile + moff + j;
                  out[m] += pf * wscales[m * NQ + gq] * stage[moff + j];
                  stage[moff + j] = 0.f;
                }
              }
            }
            pos += lanes;
          }
        }
      }
    }
  }
  for (int64_t m = (int64_t)mb0 * m_tile; m < (int64_t)mb1 * m_tile; m++) {
    float s = 0.f;
    for (int gq = 0; gq < NQ; gq++) s += wscales[m * NQ + gq] * rowsums[gq];
    out[m] -= 0.5f * s;
  }
  free(stage);
}

/* kernel.py:280-371 for variant vector-q8 (mode 0) or scalar-real (mode 1):
 * a (n, K) f32, planes v1 (bits, plane_bytes), wscales (M, NQ) f32 -> out (n, M).
 * threads <= 0: use all OpenMP threads.  Returns 0. */
int orc_mpgemm(const float* a, int n, const uint8_t* planes, int M, int K, int bits, int gs,
               int m_tile, int k_tile, int lanes, const float* wscales, int mode, int threads,
               float* out) {
  const int KG = K / 4, NQ = K / gs, n_mb = M / m_tile;
  const int64_t plane_bytes = (int64_t)M * KG / 2;
  float* tabs = (float*)malloc(sizeof(float) * (size_t)KG * 8);
  int8_t* qtab = (int8_t*)malloc((size_t)KG * 8);
  float* ts = (float*)malloc(sizeof(float) * (size_t)NQ);
  float* rs = (float*)malloc(sizeof(float) * (size_t)NQ);
#ifdef _OPENMP
  int nt = threads > 0 ? threads : omp_get_max_threads();
#else
  int nt = 1;
  (void)threads;
#endif
  if (nt > n_mb) nt = n_mb;
  if (nt < 1) nt = 1;
  for (int r = 0; r < n; r++) {
    const float* ar = a + (int64_t)r * K;
    float* o = out + (int64_t)r * M;
    memset(o, 0, sizeof(float) * (size_t)M);
    if (mode == 0) orc_tables_q8(ar, K, gs, qtab, ts, rs, tabs);
    else orc_tables_real(ar, K, gs, tabs, rs);
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int w = 0; w < nt; w++) {
      /* kernel.py:254-263: contiguous M-block slices */
      int base = n_mb / nt, extra = n_mb % nt;
      int mb0 = w * base + (w < extra ? w : extra);
      int mb1 = mb0 + base + (w < extra ? 1 : 0);
      if (mb1 > mb0) {
        if (mode == 0)
          gemv_q8_vector(planes, plane_bytes, qtab, ts, wscales, rs, o, K, bits, m_tile, k_tile,
                         lanes, gs, mb0, mb1);
        else
          gemv_real(planes, plane_bytes, tabs, wscales, rs, o, K, bits, m_tile, k_tile, lanes, gs,
                    mb0, mb1);
      }
    }
  }
  free(tabs); free(qtab); free(ts); free(rs);
  return 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* _kernels.py:20-82: one group per row of x (ng, gs); q_out (ng, gs) u8,
 * d_out (ng) f32. */
int orc_quantize_groups(const float* x, int64_t ng, int gs, int half, int nstep, uint8_t* q_out,
                        float* d_out, int threads) {
#ifdef _OPENMP
  int nt = threads > 0 ? threads : omp_get_max_threads();
#else
  int nt = 1;
  (void)threads;
#endif
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t gi = 0; gi < ng; gi++) {
    const float* xr = x + gi * gs;
    uint8_t* qr = q_out + gi * gs;
    float amax = 0.0f, smax = 0.0f;
    for (int j = 0; j < gs; j++) {
      const float ax = fabsf(xr[j]);
      if (ax > amax) {
        amax = ax;
        smax = xr[j];
      }
    }
    if (amax == 0.0f) {
      d_out[gi] = 0.0f;
      for (int j = 0; j < gs; j++) qr[j] = (uint8_t)half;
      continue;
    }
    const float inv = (float)(-half) / smax;
    if (nstep == 0) {
      const float d = smax / (float)(-half);
      for (int j = 0; j < gs; j++) {
        long l = lrintf(xr[j] * inv);
        if (l < -half) l = -half;
        if (l > half - 1) l = half - 1;
        qr[j] = (uint8_t)(l + half);
      }
      d_out[gi] = d;
      continue;
    }
    double best_score = -1.0;
    float best_inv = inv;
    for (int t = -nstep; t <= nstep; t++) {
      const float cand = ((float)(-half) + 0.1f * (float)t) / smax;
      double sumlx = 0.0;
      float suml2 = 0.0f;
      for (int j = 0; j < gs; j++) {
        long l = lrintf(xr[j] * cand);
        if (l < -half) l = -half;
        if (l > half - 1) l = half - 1;
        sumlx += (double)xr[j] * (double)l;
        suml2 += (float)(l * l);
      }
      if (suml2 > 0.0f && sumlx * sumlx > best_score * (double)suml2) {
        best_score = sumlx * sumlx / (double)suml2;
        best_inv = cand;
      }
    }
    double sumlx = 0.0;
    float suml2 = 0.0f;
    for (int j = 0; j < gs; j++) {
      long l = lrintf(xr[j] * best_inv);
      if (l < -half) l = -half;
      if (l > half - 1) l = half - 1;
      qr[j] = (uint8_t)(l + half);
      sumlx += (double)xr[j] * (double)l;
      suml2 += (float)(l * l);
    }
    d_out[gi] = suml2 > 0.0f ? (float)(sumlx / (double)suml2) : 0.0f;
  }
  return 0;
}
