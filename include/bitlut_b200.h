/*
 * bitlut_b200 -- C ABI of the B200 (sm_100a) LUT mixed-precision GEMV/GEMM.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `bitlut` (arXiv 2407.00088 reimplementation, /root/reference/pkg).  The
 * reference has no native ABI of its own: its "native layer" is numba-JIT'd
 * Python (`_kernels.py`) called from `kernel.py`.  Each entry point below
 * names the reference function it replaces (file:line relative to
 * pkg/src/bitlut/).  Python binds these through ctypes underneath
 * torch.library custom ops (paper_2407_00088_b200/_native.py); INTEGRATION.md
 * shows the binding a maintainer would add to the reference itself.
 *
 * Conventions:
 *   - every pointer is a DEVICE pointer allocated by the caller; the library
 *     never allocates, frees, or synchronizes, and keeps no global state;
 *   - kernels are enqueued on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream);
 *   - the return value is BITLUT_OK or a negative code mapping 1:1 onto the
 *     reference's error classes (errors.py:8-69); shape/parameter checks
 *     happen before any launch, a launch failure returns BITLUT_EINTERNAL;
 *   - no C++ exception crosses the ABI.
 */
#ifndef BITLUT_B200_H
#define BITLUT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> errors.py classes */
#define BITLUT_OK          0
#define BITLUT_EPARAM     -1   /* ParameterError      errors.py:15  */
#define BITLUT_EDATA      -2   /* DataError           errors.py:21  */
#define BITLUT_ESHAPE     -3   /* ShapeError          errors.py:27  */
#define BITLUT_ELAYOUT    -4   /* LayoutError         errors.py:33  */
#define BITLUT_EOVERFLOW  -5   /* OverflowConfigError errors.py:39  */
#define BITLUT_EINTERNAL -100  /* BitLutError (launch failure)  errors.py:8 */

/* element types of activations / weight scales / zeros */
#define BITLUT_DT_F32 0
#define BITLUT_DT_F16 1

/* lookup-table modes */
#define BITLUT_TABLE_Q8  0  /* int8 half tables + per-group table scales (vector-q8 semantics) */
#define BITLUT_TABLE_F16 1  /* fp16 half tables (BASELINE "fp16 tables") */
/* 16-bit block fixed point: per quantization group scale = max|entry| / 16129,
 * entry = scale * (127 H + L) with two balanced base-127 digits H in
 * [-127, 127], L in [-63, 63] -- each an int8 half table, so the mirror flag
 * negates digit by digit and the int8 lookup core applies twice.  At least
 * fp16-table accuracy (<= 3.1e-5 of the group maximum per entry; fp16:
 * 4.9e-4 of the entry).  The fast batch-1 path of variant "cuda-f16":
 * bitlut_build_lut (single row) + bitlut_mpgemm with
 * BITLUT_FLAG_FAST_EPILOGUE, n = 1, 1/2/4-bit weights; anything else
 * returns BITLUT_ELAYOUT (use BITLUT_TABLE_F16).  16 bytes per k-group
 * like BITLUT_TABLE_F16; table scales are written. */
#define BITLUT_TABLE_X16 2

/* launch flags (bitlut_build_lut, bitlut_mpgemm) */
#define BITLUT_FLAG_PDL 1   /* launch with programmatic dependent launch */
/* With BITLUT_FLAG_PDL: the call's inputs (tables, weights, scales) were
 * complete before the PREVIOUS kernel in the stream started (e.g. k and v
 * after q, all reading one table).  The kernel then does its whole
 * computation without griddepcontrol.wait and waits only before exiting, so
 * completion order is preserved while the work overlaps the predecessor. */
#define BITLUT_FLAG_INDEPENDENT 2
/* Fast epilogue: the int32 staging values are the same exact ones, but the
 * float combination is a fixed-order parallel reduction instead of the
 * reference's left-to-right chain (deterministic; last-bits differences). */
#define BITLUT_FLAG_FAST_EPILOGUE 4
/* With BITLUT_FLAG_FAST_EPILOGUE at batch 1 on 1/2/4-bit weights:
 * `partials` receives, instead of the per-plane staging values, the exact
 * integer combination S[m][gq] = sum_p 2^p P_p (shape (1, m, k/gs)) that the
 * fast kernel scales -- SURVEY §8(c)'s bit-exactness object. */
#define BITLUT_FLAG_COMBINED_PARTIALS 32
/* bitlut_mpgemm: wgpu / wscales / zeros are in the LAYER-SET layout
 * (bitlut_layer_set_weights / _scales) instead of layout v2.  Fast epilogue,
 * int8 tables; served by the lean batch-1 and mpGEMM rows kernels with
 * select-free lane reductions (outputs bitwise those of the v2 operand);
 * BITLUT_ELAYOUT where those kernels do not apply (exact epilogue, long K,
 * zero points at N >= 8, groups wider than a lane's accumulators) -- pass
 * the v2 operand then.  Also accepted by bitlut_mpgemv_multi and
 * bitlut_mpgemv_multi_tab (every matrix of the launch in the layer-set
 * layout) and, per lookup op, by the op-list executor. */
#define BITLUT_FLAG_LAYER_SET 64

/*
 * GPU weight layout ("layout v2", this library's own; the reference's v1
 * layout is docs/formats.md:60-90).  Filled by bitlut_gpu_layout_query.
 *   tile_channels : output channels per tile (32/bits, or 32 for bits=3)
 *   stream_groups : 32-stream groups per tile (1, or 3 for bits=3)
 *   unit_kg       : k-groups (4 activations each) per lane unit
 *   lanes_per_group : lane units per quantization group
 *   bytes         : total bytes (== bits*m*k/8, same as v1)
 */
typedef struct {
  int32_t m, k, bits, group_size;
  int32_t tile_channels, stream_groups, unit_kg, lanes_per_group;
  int64_t bytes;
} bitlut_gpu_layout;

/* Validate (m, k, bits, group_size) for the CUDA path and describe layout v2. */
int bitlut_gpu_layout_query(int m, int k, int bits, int group_size, bitlut_gpu_layout* out);

/* ---------------- offline weight pipeline (weight_prep.py) ---------------- */

/* decompose_bits  weight_prep.py:86-105.
 * q (m,k) u8 -> indices (bits, m, k/g) u8, index = sum_j bit_i(q[m,kg*g+j]) << j */
int bitlut_decompose_bits(const uint8_t* q, int m, int k, int bits, int g,
                          uint8_t* indices, void* stream);

/* pack_and_permute (v1 layout)  weight_prep.py:214-246, _permute_plane :193-201,
 * interleave_layout :131-156.  indices (bits, m, k/g) -> planes (bits, m*(k/g)/per) */
int bitlut_pack_v1(const uint8_t* indices, int bits, int m, int k, int g,
                   int m_tile, int k_tile, int lanes, uint8_t* planes, void* stream);

/* unpack_planes  weight_prep.py:249-257 (inverse of bitlut_pack_v1). */
int bitlut_unpack_v1(const uint8_t* planes, int bits, int m, int k, int g,
                     int m_tile, int k_tile, int lanes, uint8_t* indices, void* stream);

/* The offline weight-permutation kernel of the north star: plane indices
 * (bits, m, k/4) -> layout v2 (mirror-encoded nibbles, 16 B per 32 streams
 * x 1 k-group, unit-interleaved so each warp load is one coalesced span). */
int bitlut_repack_gpu(const uint8_t* indices, int bits, int m, int k, int group_size,
                      uint8_t* wgpu, void* stream);

/* Inverse of bitlut_repack_gpu (verification / round trips). */
int bitlut_unrepack_gpu(const uint8_t* wgpu, int bits, int m, int k, int group_size,
                        uint8_t* indices, void* stream);

/* ---------------- online activation tables (lut_build.py) ---------------- */

/* precompute_lut  lut_build.py:105-127.  a (n,k) -> full (n, k/g, 2^g) f32 */
int bitlut_precompute_lut(const void* a, int a_dtype, int n, int k, int g,
                          float* full, void* stream);

/* mirror_consolidate  lut_build.py:130-143.  full (n,kg,2^g) -> half (n,kg,2^(g-1));
 * *asym_flag (device int, caller zeroes it) is set to 1 if the input is not
 * exactly sign-symmetric (the reference raises DataError). */
int bitlut_mirror_consolidate(const float* full, int n, int kg, int g, float* half,
                              int* asym_flag, void* stream);

/* quantize_tables  lut_build.py:153-179.  half (n,kg,w) f32 ->
 * qentries (n,kg,w) i8 + table_scales (n, kg*g/group_size) f32 */
int bitlut_quantize_tables(const float* half, int n, int kg, int g, int group_size,
                           int8_t* qentries, float* table_scales, void* stream);

/* row_sums  lut_build.py:182-194.  a (n,k) -> sums (n, k/group_size) f32 */
int bitlut_row_sums(const void* a, int a_dtype, int n, int k, int group_size,
                    float* sums, void* stream);

/* Fused per-call table build used by mpgemm (kernel.py:226-251,
 * _build_block_tables): one launch produces, for g = 4,
 *   mode Q8 : tables = int8 (n, k/4, 8) holding quantize_tables(mirror_consolidate(
 *             precompute_lut(a))) in KERNEL FORMAT: each byte Q stored as
 *             Q - (Q < 0), k-groups unit-interleaved like the weights
 *             (layout.cuh table_offset); tscales (n, k/gs) f32, rowsums f32
 *   mode F16: tables = fp16-rounded half tables (n, k/4, 8 x 2 B) in KERNEL
 *             FORMAT: per k-group 8 low bytes then 8 high bytes of the 8
 *             entries, unit-interleaved at 16 B; rowsums (tscales unused). */
int bitlut_build_lut(const void* a, int a_dtype, int n, int k, int group_size, int mode,
                     void* tables, float* tscales, float* rowsums, int flags, void* stream);

/* Several table builds (up to 8 activation blocks, one dtype) in ONE launch:
 * each job is exactly a bitlut_build_lut call. */
typedef struct {
  const void* a;            /* (n, k) activations */
  int a_dtype, n, k, group_size;
  void* tables;
  float* tscales;
  float* rowsums;
} bitlut_lut_job;
int bitlut_build_lut_multi(const bitlut_lut_job* jobs, int n_jobs, int mode, int flags, void* stream);

/* Any number of table builds in ONE launch, the job list in DEVICE memory
 * (e.g. every activation row of an independent layer set).  Each job is
 * exactly a bitlut_build_lut call (one dtype for the list).
 * bitlut_build_lut_batch_encode (host) validates the HOST copy of the jobs
 * and writes block_end[j] = cumulative CTA count through job j; the caller
 * copies jobs and block_end to device memory and passes those copies. */
int bitlut_build_lut_batch_encode(const bitlut_lut_job* jobs, int n_jobs, int* block_end, int* total_blocks);
int bitlut_build_lut_batch(const bitlut_lut_job* dev_jobs, const int* dev_block_end, int n_jobs,
                           int total_blocks, int a_dtype, int mode, int flags, void* stream);

/* ---------------- lookup-accumulate (kernel.py / _kernels.py) ---------------- */

/* mpgemm  kernel.py:280-371 with _kernels.gemv_q8_vector :141-192 (mode Q8)
 * or an fp16-table analogue of _kernels.gemv_real :85-138 (mode F16).
 *   wgpu      layout-v2 weights (bitlut_repack_gpu)
 *   wscales   (m, k/gs) per-group weight scales, dtype scale_dtype
 *   zeros     (m, k/gs) zero points or NULL (= implicit 2^(bits-1), the
 *             reference's symmetric scheme core.py:86-100)
 *   tables/tscales/rowsums  from bitlut_build_lut (tscales unused for F16)
 *   out       (n, m) f32, overwritten
 *   partials  NULL, or (n, bits, m, k/gs) int32: the exact per-(row, plane,
 *             channel, group) int32 staging values (Q8 mode only)
 * In Q8 mode with zeros == NULL, `out` is bitwise identical to the
 * reference's vector-q8 output. */
int bitlut_mpgemm(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                  const void* wscales, const void* zeros, int scale_dtype,
                  const void* tables, const float* tscales, const float* rowsums,
                  int mode, int n, float* out, int32_t* partials, int flags,
                  void* stream);

/* Batch-1 table build + lookup in ONE launch (decode path, fast epilogue):
 * a = one fp16 activation row (k).  The CTAs of each 8-CTA thread-block
 * cluster build the int8 tables of disjoint quantization-group slices --
 * bitwise the tables of bitlut_build_lut -- and broadcast them through
 * distributed shared memory, then look up their tiles (gemv_b1.cu).
 * flags must include BITLUT_FLAG_FAST_EPILOGUE; BITLUT_FLAG_INDEPENDENT
 * means `a` was complete before the previous kernel in the stream started.
 * Returns BITLUT_ELAYOUT when the call does not fit this kernel (3-bit
 * weights, fp32 activations, shared-memory plan) -- use bitlut_build_lut +
 * bitlut_mpgemm instead. */
int bitlut_mpgemv_fused(const void* a, int a_dtype, const uint8_t* wgpu, int m, int k, int bits,
                        int group_size, const void* wscales, const void* zeros, int scale_dtype,
                        float* out, int flags, void* stream);

/* Several weight matrices that read the same activation row's tables
 * (q/k/v, gate/up) looked up by ONE batch-1 launch (fast or, without
 * BITLUT_FLAG_FAST_EPILOGUE, the reference-order epilogue; 1/2/4-bit
 * weights sharing k, bits, group_size, scale dtype and zero-point presence).
 * tables / tscales / rowsums as produced by bitlut_build_lut (mode Q8, n = 1).
 * Up to 4 matrices.  Returns BITLUT_ELAYOUT for 3-bit weights. */
typedef struct {
  const uint8_t* wgpu;      /* layout-v2 weights (m, k) */
  const void* wscales;      /* (m, k/gs) */
  const void* zeros;        /* (m, k/gs) or NULL (all or none) */
  int m;
  float* out;               /* (1, m) f32 */
} bitlut_mat;
int bitlut_mpgemv_multi(const bitlut_mat* mats, int n_mats, int k, int bits, int group_size,
                        int scale_dtype, const void* tables, const float* tscales, const float* rowsums,
                        int flags, void* stream);

/* Several batch-1 matrices with DIFFERENT activation rows (each its own
 * tables from bitlut_build_lut, mode Q8, n = 1) in one launch -- e.g. the
 * q,k,v,o,gate,up lookups of a layer set whose tables are all complete:
 * fewer, larger launches.  Fast epilogue only; matrices share k, bits,
 * group_size, scale dtype and zero-point presence; up to 8.  Outputs equal
 * the per-matrix bitlut_mpgemm calls bitwise.  Returns BITLUT_ELAYOUT when
 * the shape needs a kernel without per-matrix tables (callers then launch
 * the matrices separately). */
typedef struct {
  const uint8_t* wgpu;
  const void* wscales;
  const void* zeros;        /* or NULL (all or none) */
  int m;
  float* out;               /* (1, m) f32 */
  const void* tables;       /* this matrix's activation row: (1, k/4*8) int8 kernel format */
  const float* tscales;     /* (1, k/gs) */
  const float* rowsums;     /* (1, k/gs) */
} bitlut_mat_tab;
int bitlut_mpgemv_multi_tab(const bitlut_mat_tab* mats, int n_mats, int k, int bits, int group_size,
                            int scale_dtype, int flags, void* stream);

/* Any number of independent batch-1 mpgemv calls of one k (each its own
 * activation row and int8 tables: a layer set) in ONE launch, fast epilogue;
 * replaces that many kernel.py:374-382 mpgemv calls.  The descriptors live
 * in DEVICE memory: bitlut_mpgemv_batch_encode (host) validates the host copy
 * and fills tile_end (cumulative tiles) and *total_tiles; the caller copies
 * the array to the device.  Every CTA streams one contiguous tile range of
 * the concatenated matrices (csrc/gemv_batch.cu).  Scales of one dtype, one
 * weight encoding per launch (BITLUT_W_*); shapes with one unit round per
 * tile (bits 1/2/4, k/4/R <= 384 units), else BITLUT_ELAYOUT.
 *
 * Weight encodings (w = the dequantized weight of code q):
 *   BITLUT_W_OFFSET   w = s (q - 2^(b-1)): the reference's implicit zero
 *                     (core.py:121-123, _kernels.py:187-191); zeros NULL
 *   BITLUT_W_ZEROS    w = s (q - z), z per (channel, group) in `zeros`
 *                     (BASELINE configs[0]: asymmetric)
 *   BITLUT_W_SIGN     1-bit sign planes w = s (2q - 1): the table entry is
 *                     already the signed sum, no row-sum term (configs[2])
 *   BITLUT_W_TERNARY  2-bit codes q in {0,1,2}, w = s_t (q - 1) with ONE
 *                     per-tensor scale s_t (`wscales` points at it; no
 *                     per-group scale stream) (configs[2])
 * partials (optional, all or none, BITLUT_FLAG_COMBINED_PARTIALS): the exact
 * int32 S = sum_p 2^p P_p per (channel, group), (m, k/gs) row-major -- the
 * integer object SURVEY §8(c) pins against the reference's staging values.
 *
 * Operand format: the LAYER-SET layout (csrc/layout.cuh), made from the
 * layout-v2 weights and the (m, k/gs) group scales / zero points by
 * bitlut_layer_set_weights / bitlut_layer_set_scales below: the chunks of
 * v2 with the streams of each chunk permuted per lane (so the kernel's lane
 * reductions exchange without selects) and the scales regrouped per unit
 * (one vector load per lane).  `wgpu`, `wscales` (BITLUT_W_OFFSET / ZEROS /
 * SIGN) and `zeros` of bitlut_batch_mat are in that format; the per-tensor
 * BITLUT_W_TERNARY scale is one plain value.  The outputs are bitwise those
 * of the per-call fast lookups on the v2 operand. */
#define BITLUT_W_OFFSET 0
#define BITLUT_W_ZEROS 1
#define BITLUT_W_SIGN 2
#define BITLUT_W_TERNARY 3
typedef struct {
  const uint8_t* wgpu;      /* layer-set weights */
  const void* wscales;      /* layer-set scales, or 1 value (BITLUT_W_TERNARY) */
  const void* zeros;        /* layer-set zero points for BITLUT_W_ZEROS, else NULL */
  float* out;               /* (1, m) f32 */
  const void* tables;       /* (1, k/4*8) int8 kernel format */
  const float* tscales;     /* (1, k/gs) */
  const float* rowsums;     /* (1, k/gs) */
  int32_t* partials;        /* (m, k/gs) int32, or NULL */
  int m;
  int tile_end;             /* filled by bitlut_mpgemv_batch_encode */
} bitlut_batch_mat;
int bitlut_mpgemv_batch_encode(bitlut_batch_mat* mats, int n_mats, int k, int bits, int group_size,
                               int weight_mode, int* total_tiles);
int bitlut_mpgemv_batch(const bitlut_batch_mat* dev_mats, int n_mats, int total_tiles, int k, int bits,
                        int group_size, int scale_dtype, int weight_mode, int flags, void* stream);

/* Layer-set layout conversion (offline; part of the north star's repack
 * step, replaces nothing in the reference -- weight_prep.py:193-246 is the
 * analogous pack_and_permute).  bitlut_layer_set_weights: layout v2 ->
 * layer-set weights, same size (m*bits*k/8 bytes), out != wgpu; it is an
 * involution (applying it to layer-set weights gives v2 back).
 * bitlut_layer_set_scales: (m, k/gs) f16/f32 scales or zero points ->
 * bitlut_layer_set_scales_bytes(...) bytes (the same m*k/gs elements,
 * reordered; more only when a group spans more lanes than a lane has
 * accumulators: 4-bit gs >= 256, 2-bit gs = 512).  1/2/4-bit weights only
 * (BITLUT_ELAYOUT otherwise). */
int64_t bitlut_layer_set_scales_bytes(int m, int k, int bits, int group_size, int scale_dtype);
int bitlut_layer_set_weights(const uint8_t* wgpu, int bits, int m, int k, int group_size, uint8_t* out,
                             void* stream);
int bitlut_layer_set_scales(const void* scales, int scale_dtype, int bits, int m, int k, int group_size,
                            void* out, void* stream);

/* The drop-in call with HOST buffers (replaces kernel.py:280-371 mpgemm /
 * :374-382 mpgemv as a numpy caller sees them): copies a_host (n, k) f16/f32
 * to a_dev, builds the tables (or, batch 1 fast epilogue fp16, runs the fused
 * build + lookup launch), looks up, copies the (n, m) f32 result to out_host
 * and synchronizes `stream`.  The device scratch (a_dev, tables, tscales,
 * rowsums, out_dev: sizes as for bitlut_build_lut / bitlut_mpgemm) is the
 * caller's; flags as bitlut_mpgemm.  Passing a_dev == a_host (out_dev ==
 * out_host) makes the kernels read (write) the pinned, UVA-mapped host
 * buffer directly instead of a copy operation.  csrc/host_api.cu. */
int bitlut_mpgemm_host(const void* a_host, int a_dtype, int n, int k, const uint8_t* wgpu, int m, int bits,
                       int group_size, const void* wscales, const void* zeros, int scale_dtype, int mode,
                       int flags, void* a_dev, void* tables, float* tscales, float* rowsums, float* out_dev,
                       float* out_host, void* stream);

/* Tensor-parallel batch-1 lookup with the all-gather fused into the epilogue
 * (SURVEY §8(e) B200-native upgrade; replaces kernel.py:374-382 mpgemv on
 * this rank's output-channel shard + parallel.py's NCCL all-gather).  Same
 * arguments as bitlut_mpgemm at n = 1 with BITLUT_FLAG_FAST_EPILOGUE (the
 * local (1, m) result also goes to `out`), plus:
 *   peer_out[q]   (HOST array of n_peers device pointers, q = 0..n_peers-1):
 *                 the gathered (1, m_total) f32 row of rank q, peer-accessible
 *                 (symmetric memory / IPC over NVLink); this call writes
 *                 columns [col_offset, col_offset + m) of every one;
 *   peer_flags[q] (HOST array of device pointers): rank q's u32 gather flag;
 *                 the last CTA adds 1 to each with release semantics at
 *                 system scope after every store of the launch;
 *   ticket        a zero-initialised u32 of this rank (reset by the kernel).
 * Rank r's row is complete once its flag reaches epoch * world
 * (bitlut_gather_wait).  1 <= n_peers <= 8. */
int bitlut_mpgemv_gather(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                         const void* wscales, const void* zeros, int scale_dtype, const void* tables,
                         const float* tscales, const float* rowsums, float* out, int n_peers,
                         float* const* peer_out, unsigned* const* peer_flags, unsigned* ticket,
                         int col_offset, int flags, void* stream);
/* Stream-ordered wait (one thread, ld.acquire.sys) until *flag - target >= 0
 * as signed 32-bit (wrap-around safe).  Bounded: after 10 s without the
 * peers' arrivals it gives up and sets *timed_out (device u32, nullable), so
 * a missing peer cannot hang the stream. */
int bitlut_gather_wait(const unsigned* flag, unsigned target, unsigned* timed_out, void* stream);

/* bitlut_mpgemm plus a timeline: `trace` (device, (n * tiles) x 8 u64) gets
 * per-CTA %globaltimer stamps [start, loads issued, after griddepcontrol.wait,
 * tables staged, lookups done, epilogue products done, end] and %smid in
 * slot 7.  Diagnostic only (tools/timeline.py). */
int bitlut_mpgemm_traced(const uint8_t* wgpu, int m, int k, int bits, int group_size,
                         const void* wscales, const void* zeros, int scale_dtype,
                         const void* tables, const float* tscales, const float* rowsums,
                         int mode, int n, float* out, int32_t* partials, int flags,
                         unsigned long long* trace, void* stream);

/* ---------------- op lists (this library's executors) ----------------
 * A list of table builds and lookup GEMVs -- e.g. every projection of every
 * decoder layer of a batch-1 decode step.  Each op names up to three earlier
 * ops it depends on.  Per-op arithmetic is identical to bitlut_build_lut
 * (mode Q8) + bitlut_mpgemm (mode Q8). */
#define BITLUT_OP_TABLES 0
#define BITLUT_OP_LOOKUP 1
typedef struct {
  int type;                 /* BITLUT_OP_TABLES or BITLUT_OP_LOOKUP */
  int dep[3];               /* earlier op indices this op needs complete, -1 = none */
  const void* a;            /* TABLES: activations (n, k), a_dtype */
  int a_dtype;
  int n, k, group_size;     /* rows, reduction length, quantization group */
  void* tables;             /* TABLES: written; LOOKUP: read (kernel-format int8) */
  float* tscales;           /* (n, k/gs) */
  float* rowsums;           /* (n, k/gs) */
  const uint8_t* wgpu;      /* LOOKUP: layout-v2 weights */
  const void* wscales;      /* LOOKUP: (m, k/gs), scale_dtype */
  const void* zeros;        /* LOOKUP: (m, k/gs) or NULL */
  int scale_dtype;
  int m, bits;
  float* out;               /* LOOKUP: (n, m) f32 */
  int flags;                /* LOOKUP: BITLUT_FLAG_FAST_EPILOGUE or 0; TABLES: BITLUT_FLAG_FUSED_TABLES
                               = may be folded into its consumers (bitlut_mpgemv_fused) */
} bitlut_pipe_op;

/* Per-op executor: stream-ordered launches of the
 * bitlut_build_lut / bitlut_mpgemm kernels (mode Q8) chained with
 * programmatic dependent launch, for capture into a CUDA graph.  Lookups
 * whose deps are already complete when they start are launched with
 * BITLUT_FLAG_INDEPENDENT; batch-1 fp16 table ops marked
 * BITLUT_FLAG_FUSED_TABLES whose consumers are all fast-epilogue 32-stream
 * lookups are folded into them (each consumer runs
 * as bitlut_mpgemv_fused); consecutive table builds, and consecutive
 * batch-1 fast lookups over the same tables, share one launch.
 * bitlut_pipeline_plan_flags writes the per-op plan: launch flags,
 * BITLUT_PLAN_SKIP, BITLUT_FLAG_FUSED_TABLES, BITLUT_PLAN_JOINED (see
 * pipeline.cu for the rules). */
#define BITLUT_PLAN_SKIP (-1)          /* plan: table op folded into its consumers */
#define BITLUT_FLAG_FUSED_TABLES 8     /* plan: lookup launched as bitlut_mpgemv_fused */
#define BITLUT_PLAN_JOINED 16          /* plan: launched together with the previous op
                                          (bitlut_build_lut_multi / bitlut_mpgemv_multi) */
int bitlut_pipeline_plan_flags(const bitlut_pipe_op* specs, int n_ops, int* flags_out);
int bitlut_pipeline_launch_ops(const bitlut_pipe_op* specs, int n_ops, void* stream);
/* The same launches, but inputs are tracked with per-launch completion
 * counters instead of PDL waits (no launch drains the stream): `counters` =
 * device scratch of n_ops + 1 uint32, zeroed by the call (a captured memset);
 * a final 1-CTA join kernel completes when every CTA of the list has. */
int bitlut_pipeline_launch_ops_counted(const bitlut_pipe_op* specs, int n_ops, unsigned* counters, void* stream);

/* Number of kernel launches one bitlut_mpgemm call enqueues (for accounting). */
int bitlut_mpgemm_launches(int m, int k, int bits, int group_size, int mode, int n);

/* Library version string. */
const char* bitlut_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BITLUT_B200_H */
