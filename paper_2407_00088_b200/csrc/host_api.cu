// Host-buffer drop-in call: the reference's mpgemm/mpgemv contract (numpy in,
// numpy out: kernel.py:280-382) as ONE C entry point.  The activations come
// from a host pointer and the f32 result goes back to one; the H2D copy, the
// table build, the lookup launch(es) and the D2H copy are enqueued on one
// stream and the call returns after that stream drained -- no torch
// dispatch, no per-call allocation (the caller passes device scratch), one
// synchronization per call.  Python's mpgemm uses it for numpy inputs.
#include "common.cuh"

extern "C" int bitlut_build_lut(const void* a, int a_dtype, int n, int k, int group_size, int mode, void* tables,
                                float* tscales, float* rowsums, int flags, void* stream);
extern "C" int bitlut_mpgemm(const uint8_t* wgpu, int m, int k, int bits, int group_size, const void* wscales,
                             const void* zeros, int scale_dtype, const void* tables, const float* tscales,
                             const float* rowsums, int mode, int n, float* out, int32_t* partials, int flags,
                             void* stream);
extern "C" int bitlut_mpgemv_fused(const void* a, int a_dtype, const uint8_t* wgpu, int m, int k, int bits,
                                   int group_size, const void* wscales, const void* zeros, int scale_dtype,
                                   float* out, int flags, void* stream);

extern "C" int bitlut_mpgemm_host(const void* a_host, int a_dtype, int n, int k, const uint8_t* wgpu, int m,
                                  int bits, int group_size, const void* wscales, const void* zeros,
                                  int scale_dtype, int mode, int flags, void* a_dev, void* tables,
                                  float* tscales, float* rowsums, float* out_dev, float* out_host,
                                  void* stream) {
  if (!a_host || !wgpu || !wscales || !a_dev || !tables || !tscales || !rowsums || !out_dev || !out_host)
    return BITLUT_EPARAM;
  if (n < 1 || k < 1 || m < 1) return BITLUT_EPARAM;
  if (a_dtype != BITLUT_DT_F32 && a_dtype != BITLUT_DT_F16) return BITLUT_EPARAM;
  const cudaStream_t st = (cudaStream_t)stream;
  const size_t a_bytes = (size_t)n * k * (a_dtype == BITLUT_DT_F16 ? 2 : 4);
  // a_dev == a_host / out_dev == out_host: pinned (mapped) host memory the
  // kernels read / write directly over the bus -- no copy operations
  if (a_dev != a_host &&
      cudaMemcpyAsync(a_dev, a_host, a_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return BITLUT_EINTERNAL;
  int rc = BITLUT_ELAYOUT;
  // batch 1, fast epilogue, fp16 row: table build + lookup in one launch
  if (n == 1 && mode == BITLUT_TABLE_Q8 && (flags & BITLUT_FLAG_FAST_EPILOGUE) && a_dtype == BITLUT_DT_F16 &&
      bits != 3)
    rc = bitlut_mpgemv_fused(a_dev, a_dtype, wgpu, m, k, bits, group_size, wscales, zeros, scale_dtype, out_dev,
                             flags, stream);
  if (rc == BITLUT_ELAYOUT) {
    rc = bitlut_build_lut(a_dev, a_dtype, n, k, group_size, mode, tables, tscales, rowsums,
                          flags & BITLUT_FLAG_PDL, stream);
    if (rc) return rc;
    rc = bitlut_mpgemm(wgpu, m, k, bits, group_size, wscales, zeros, scale_dtype, tables, tscales, rowsums, mode,
                       n, out_dev, nullptr, flags, stream);
  }
  if (rc) return rc;
  if (out_dev != out_host &&
      cudaMemcpyAsync(out_host, out_dev, (size_t)n * m * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return BITLUT_EINTERNAL;
  return cudaStreamSynchronize(st) == cudaSuccess ? BITLUT_OK : BITLUT_EINTERNAL;
}
