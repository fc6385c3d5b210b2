"""Binding of the C ABI (include/bitlut_b200.h) and the torch custom ops.

The shared library ``_lib/libbitlut_b200.so`` is built in-tree by
``paper_2407_00088_b200.build`` (nvcc, sm_100a).  There is no CPU
fallback: if the library or a CUDA device is missing, every op raises.

torch.library custom ops (namespace ``bitlut_b200``) wrap the C entry
points so the ops compose with torch streams, CUDA graphs and
torch.compile (fake/meta implementations give shapes without a GPU).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

from .errors import BitLutError, ParameterError, raise_for_status

LIB_PATH = os.environ.get("BITLUT_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libbitlut_b200.so")   # env: A/B builds

DT_F32, DT_F16 = 0, 1
TABLE_Q8, TABLE_F16, TABLE_X16 = 0, 1, 2     # X16: 16-bit block fixed point (bitlut_b200.h)
FLAG_PDL = 1
FLAG_INDEPENDENT = 2
FLAG_FAST_EPILOGUE = 4
FLAG_FUSED_TABLES = 8       # table op may fold into its consumers (graph executor)
PLAN_JOINED = 16            # plan: launched together with the previous op
FLAG_COMBINED_PARTIALS = 32
FLAG_LAYER_SET = 64         # lookup operand in the layer-set layout (lean kernels)

_vp, _i = ctypes.c_void_p, ctypes.c_int

_SIGS = {
    "bitlut_gpu_layout_query": [_i, _i, _i, _i, _vp],
    "bitlut_decompose_bits": [_vp, _i, _i, _i, _i, _vp, _vp],
    "bitlut_pack_v1": [_vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "bitlut_unpack_v1": [_vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "bitlut_repack_gpu": [_vp, _i, _i, _i, _i, _vp, _vp],
    "bitlut_unrepack_gpu": [_vp, _i, _i, _i, _i, _vp, _vp],
    "bitlut_precompute_lut": [_vp, _i, _i, _i, _i, _vp, _vp],
    "bitlut_mirror_consolidate": [_vp, _i, _i, _i, _vp, _vp, _vp],
    "bitlut_quantize_tables": [_vp, _i, _i, _i, _i, _vp, _vp, _vp],
    "bitlut_row_sums": [_vp, _i, _i, _i, _i, _vp, _vp],
    "bitlut_build_lut": [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp],
    "bitlut_mpgemm": [_vp, _i, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _vp, _vp, _i, _vp],
    "bitlut_mpgemm_traced": [_vp, _i, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _vp, _vp, _i,
                             _vp, _vp],
    "bitlut_mpgemm_launches": [_i, _i, _i, _i, _i, _i],
    "bitlut_mpgemv_fused": [_vp, _i, _vp, _i, _i, _i, _i, _vp, _vp, _i, _vp, _i, _vp],
    "bitlut_mpgemm_host": [_vp, _i, _i, _i, _vp, _i, _i, _i, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp,
                           _vp],
    "bitlut_mpgemv_multi": [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp],
    "bitlut_mpgemv_gather": [_vp, _i, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i,
                             _vp],
    "bitlut_gather_wait": [_vp, ctypes.c_uint32, _vp, _vp],
    "bitlut_mpgemv_multi_tab": [_vp, _i, _i, _i, _i, _i, _i, _vp],
    "bitlut_mpgemv_batch_encode": [_vp, _i, _i, _i, _i, _i, _vp],
    "bitlut_mpgemv_batch": [_vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp],
    "bitlut_layer_set_weights": [_vp, _i, _i, _i, _i, _vp, _vp],
    "bitlut_layer_set_scales": [_vp, _i, _i, _i, _i, _i, _vp, _vp],
    "bitlut_build_lut_batch_encode": [_vp, _i, _vp, _vp],
    "bitlut_build_lut_batch": [_vp, _vp, _i, _i, _i, _i, _i, _vp],
}


class BitlutMat(ctypes.Structure):
    """include/bitlut_b200.h bitlut_mat: one matrix of a grouped batch-1 launch."""
    _fields_ = [("wgpu", ctypes.c_void_p), ("wscales", ctypes.c_void_p), ("zeros", ctypes.c_void_p),
                ("m", ctypes.c_int32), ("out", ctypes.c_void_p)]


class BitlutMatTab(ctypes.Structure):
    """include/bitlut_b200.h bitlut_mat_tab: one matrix with its own tables."""
    _fields_ = [("wgpu", ctypes.c_void_p), ("wscales", ctypes.c_void_p), ("zeros", ctypes.c_void_p),
                ("m", ctypes.c_int32), ("out", ctypes.c_void_p), ("tables", ctypes.c_void_p),
                ("tscales", ctypes.c_void_p), ("rowsums", ctypes.c_void_p)]


class BitlutBatchMat(ctypes.Structure):
    """include/bitlut_b200.h bitlut_batch_mat: one GEMV of a batched launch
    (device-resident descriptor array)."""
    _fields_ = [("wgpu", ctypes.c_void_p), ("wscales", ctypes.c_void_p), ("zeros", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("tables", ctypes.c_void_p), ("tscales", ctypes.c_void_p),
                ("rowsums", ctypes.c_void_p), ("partials", ctypes.c_void_p),
                ("m", ctypes.c_int32), ("tile_end", ctypes.c_int32)]


# weight encodings of the batch executor (bitlut_b200.h BITLUT_W_*)
W_OFFSET, W_ZEROS, W_SIGN, W_TERNARY = 0, 1, 2, 3
W_MODES = {"offset": W_OFFSET, "zeros": W_ZEROS, "sign": W_SIGN, "ternary": W_TERNARY}


class BitlutLutJob(ctypes.Structure):
    """include/bitlut_b200.h bitlut_lut_job: one table build."""
    _fields_ = [("a", ctypes.c_void_p), ("a_dtype", ctypes.c_int32), ("n", ctypes.c_int32),
                ("k", ctypes.c_int32), ("group_size", ctypes.c_int32), ("tables", ctypes.c_void_p),
                ("tscales", ctypes.c_void_p), ("rowsums", ctypes.c_void_p)]


def _to_device_bytes(arr, device) -> torch.Tensor:
    host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
    return host.to(device)


def layer_set_weights(wgpu: torch.Tensor, bits: int, m: int, k: int, group_size: int) -> torch.Tensor:
    """Layout-v2 weights -> the layer-set layout bitlut_mpgemv_batch reads
    (csrc/layout.cuh; an involution)."""
    require_cuda(wgpu, "wgpu")
    out = torch.empty_like(wgpu)
    rc = lib().bitlut_layer_set_weights(ptr(wgpu), bits, m, k, group_size, ptr(out),
                                        ctypes.c_void_p(torch.cuda.current_stream(wgpu.device).cuda_stream))
    raise_for_status(rc, "bitlut_layer_set_weights")
    return out


def layer_set_scales(t: torch.Tensor, bits: int, m: int, k: int, group_size: int) -> torch.Tensor:
    """(m, k/gs) f16/f32 group scales or zero points -> layer-set order (flat)."""
    require_cuda(t, "scales")
    t = t.contiguous()
    dt = dtype_code(t)
    nbytes = lib().bitlut_layer_set_scales_bytes(m, k, bits, group_size, dt)
    if nbytes < 0:
        raise_for_status(-4, "bitlut_layer_set_scales_bytes")
    out = torch.empty((nbytes // t.element_size(),), dtype=t.dtype, device=t.device)
    rc = lib().bitlut_layer_set_scales(ptr(t), dt, bits, m, k, group_size, ptr(out),
                                       ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream))
    raise_for_status(rc, "bitlut_layer_set_scales")
    return out


class LookupBatch:
    """Encoded bitlut_mpgemv_batch launch: independent batch-1 fast GEMVs of
    one (k, bits, group_size, scale dtype), each with its own int8 tables.
    `arr`: ctypes array of BitlutBatchMat (host); copied to `device`."""

    def __init__(self, arr, k: int, bits: int, group_size: int, scale_dtype: int, device, weight_mode: int = W_OFFSET):
        tt = ctypes.c_int(0)
        raise_for_status(lib().bitlut_mpgemv_batch_encode(arr, len(arr), k, bits, group_size, weight_mode,
                                                          ctypes.byref(tt)), "bitlut_mpgemv_batch_encode")
        self.n, self.total_tiles = len(arr), tt.value
        self.k, self.bits, self.group_size, self.scale_dtype = k, bits, group_size, scale_dtype
        self.weight_mode = weight_mode
        self.partials = bool(arr[0].partials)          # all or none (checked by the encoder)
        self.dev = _to_device_bytes(arr, device)

    @classmethod
    def from_tensors(cls, mats, k: int, bits: int, group_size: int, weight_mode: int = W_OFFSET) -> "LookupBatch":
        """mats = [(wgpu, wscales, m, out (1, m) f32, tables, tscales, rowsums[, zeros[, partials]]), ...]
        with layout-v2 weights and (m, k/gs) scales / zero points: converted
        here to the layer-set layout the launch reads (one copy per call --
        Pipeline caches the converted operand per PackedWeights instead)."""
        arr = (BitlutBatchMat * len(mats))()
        conv = []
        for i, mt in enumerate(mats):
            w, sc, m, out, t, ts, rs = mt[:7]
            z = mt[7] if len(mt) > 7 else None
            pp = mt[8] if len(mt) > 8 else None
            w = layer_set_weights(w, bits, m, k, group_size)
            if weight_mode != W_TERNARY:
                sc = layer_set_scales(sc, bits, m, k, group_size)
            if z is not None:
                z = layer_set_scales(z, bits, m, k, group_size)
            conv += [w, sc, z]
            arr[i].wgpu, arr[i].wscales, arr[i].out = w.data_ptr(), sc.data_ptr(), out.data_ptr()
            arr[i].tables, arr[i].tscales, arr[i].rowsums = t.data_ptr(), ts.data_ptr(), rs.data_ptr()
            arr[i].zeros = z.data_ptr() if z is not None else None
            arr[i].partials = pp.data_ptr() if pp is not None else None
            arr[i].m = m
        b = cls(arr, k, bits, group_size, dtype_code(mats[0][1]), mats[0][0].device, weight_mode)
        b.keep = [x for mt in mats for x in mt if isinstance(x, torch.Tensor)] + conv
        return b

    def launch(self, flags: int, stream) -> None:
        rc = lib().bitlut_mpgemv_batch(ptr(self.dev), self.n, self.total_tiles, self.k, self.bits, self.group_size,
                                       self.scale_dtype, self.weight_mode,
                                       flags | (FLAG_COMBINED_PARTIALS if self.partials else 0),
                                       ctypes.c_void_p(stream.cuda_stream))
        raise_for_status(rc, "bitlut_mpgemv_batch")


class TableBatch:
    """Encoded bitlut_build_lut_batch launch.  `arr`: ctypes array of
    BitlutLutJob (host, one activation dtype); copied to `device`."""

    def __init__(self, arr, mode: int, device):
        ends = (ctypes.c_int * len(arr))()
        tb = ctypes.c_int(0)
        raise_for_status(lib().bitlut_build_lut_batch_encode(arr, len(arr), ends, ctypes.byref(tb)),
                         "bitlut_build_lut_batch_encode")
        self.n, self.total_blocks, self.mode, self.a_dtype = len(arr), tb.value, mode, arr[0].a_dtype
        self.dev_jobs = _to_device_bytes(arr, device)
        self.dev_ends = _to_device_bytes(ends, device)

    @classmethod
    def from_tensors(cls, jobs, mode: int) -> "TableBatch":
        """jobs = [(a (n, k), group_size, tables, tscales, rowsums), ...]"""
        arr = (BitlutLutJob * len(jobs))()
        for i, (a, gs, t, ts, rs) in enumerate(jobs):
            arr[i].a, arr[i].a_dtype = a.data_ptr(), dtype_code(a)
            arr[i].n, arr[i].k, arr[i].group_size = a.shape[0], a.shape[1], gs
            arr[i].tables, arr[i].tscales, arr[i].rowsums = t.data_ptr(), ts.data_ptr(), rs.data_ptr()
        b = cls(arr, mode, jobs[0][0].device)
        b.keep = [x for jb in jobs for x in jb if isinstance(x, torch.Tensor)]
        return b

    def launch(self, flags: int, stream) -> None:
        rc = lib().bitlut_build_lut_batch(ptr(self.dev_jobs), ptr(self.dev_ends), self.n, self.total_blocks,
                                          self.a_dtype, self.mode, flags, ctypes.c_void_p(stream.cuda_stream))
        raise_for_status(rc, "bitlut_build_lut_batch")


class GpuLayout(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("k", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("tile_channels", ctypes.c_int32),
                ("stream_groups", ctypes.c_int32), ("unit_kg", ctypes.c_int32),
                ("lanes_per_group", ctypes.c_int32), ("bytes", ctypes.c_int64)]


_LIB: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise BitLutError(
                f"native library not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.bitlut_version.restype = ctypes.c_char_p
        L.bitlut_version.argtypes = []
        L.bitlut_layer_set_scales_bytes.restype = ctypes.c_int64
        L.bitlut_layer_set_scales_bytes.argtypes = [_i, _i, _i, _i, _i]
        _LIB = L
    return _LIB


def exported_symbols() -> list[str]:
    return list(_SIGS) + ["bitlut_version", "bitlut_layer_set_scales_bytes",
                          "bitlut_pipeline_plan_flags", "bitlut_pipeline_launch_ops",
                          "bitlut_build_lut_multi", "bitlut_mpgemv_multi",
                          "bitlut_pipeline_launch_ops_counted"]


def require_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise BitLutError(f"{what} must be a CUDA tensor (the B200 package has no CPU path)")


def ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_of(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DT_F32
    if t.dtype == torch.float16:
        return DT_F16
    raise BitLutError(f"unsupported dtype {t.dtype} (float32 or float16)")


def layout_query(m: int, k: int, bits: int, group_size: int) -> GpuLayout:
    out = GpuLayout()
    rc = lib().bitlut_gpu_layout_query(m, k, bits, group_size, ctypes.byref(out))
    raise_for_status(rc, f"GPU layout for m={m}, k={k}, bits={bits}, group_size={group_size}")
    return out


# ---------------------------------------------------------------------------
# torch custom ops
# ---------------------------------------------------------------------------

@torch.library.custom_op("bitlut_b200::build_lut", mutates_args=())
def build_lut(a: torch.Tensor, group_size: int, mode: int, flags: int = 0) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Fused table build (kernel.py:226-251): a (n, k) f16/f32 ->
    (tables (n, k/4, 8) int8|fp16, table scales (n, k/gs), row sums (n, k/gs))."""
    require_cuda(a, "activations")
    a = a.contiguous()
    n, k = a.shape
    nq = k // group_size
    tdt = torch.int8 if mode == TABLE_Q8 else torch.float16
    tables = torch.empty((n, k // 4, 8), dtype=tdt, device=a.device)
    ts = torch.empty((n, nq), dtype=torch.float32, device=a.device)
    rs = torch.empty((n, nq), dtype=torch.float32, device=a.device)
    rc = lib().bitlut_build_lut(ptr(a), dtype_code(a), n, k, group_size, mode, ptr(tables),
                                ptr(ts), ptr(rs), flags, stream_of(a))
    raise_for_status(rc, "bitlut_build_lut")
    return tables, ts, rs


@build_lut.register_fake
def _(a, group_size, mode, flags=0):
    n, k = a.shape
    tdt = torch.int8 if mode == TABLE_Q8 else torch.float16
    nq = k // group_size
    return (a.new_empty((n, k // 4, 8), dtype=tdt), a.new_empty((n, nq), dtype=torch.float32),
            a.new_empty((n, nq), dtype=torch.float32))


@torch.library.custom_op("bitlut_b200::lookup", mutates_args=())
def lookup(wgpu: torch.Tensor, wscales: torch.Tensor, zeros: Optional[torch.Tensor],
           tables: torch.Tensor, tscales: torch.Tensor, rowsums: torch.Tensor,
           m: int, k: int, bits: int, group_size: int, mode: int, flags: int,
           want_partials: bool) -> tuple[torch.Tensor, torch.Tensor]:
    """Lookup-accumulate (kernel.py:280-371 / _kernels.py:141-192):
    returns (out (n, m) f32, partials (n, bits, m, k/gs) int32 or empty)."""
    require_cuda(wgpu, "packed weights")
    n = tables.shape[0]
    out = torch.empty((n, m), dtype=torch.float32, device=wgpu.device)
    nq = k // group_size
    pb = 1 if flags & FLAG_COMBINED_PARTIALS else bits
    partials = (torch.empty((n, pb, m, nq), dtype=torch.int32, device=wgpu.device)
                if want_partials else torch.empty(0, dtype=torch.int32, device=wgpu.device))
    rc = lib().bitlut_mpgemm(ptr(wgpu), m, k, bits, group_size, ptr(wscales), ptr(zeros),
                             dtype_code(wscales), ptr(tables), ptr(tscales), ptr(rowsums), mode, n,
                             ptr(out), ptr(partials) if want_partials else None, flags,
                             stream_of(wgpu))
    raise_for_status(rc, "bitlut_mpgemm")
    return out, partials


def mpgemv_multi(mats, tables: torch.Tensor, tscales: torch.Tensor, rowsums: torch.Tensor, k: int, bits: int,
                 group_size: int, flags: int) -> list:
    """Several batch-1 matrices sharing one activation row's tables in ONE
    launch (bitlut_mpgemv_multi): mats = [(wgpu, wscales, zeros, m), ...];
    returns one (1, m) f32 output per matrix."""
    require_cuda(tables, "tables")
    outs = [torch.empty((1, m), dtype=torch.float32, device=tables.device) for (_, _, _, m) in mats]
    arr = (BitlutMat * len(mats))()
    for i, ((w, sc, z, m), o) in enumerate(zip(mats, outs)):
        arr[i].wgpu, arr[i].wscales = w.data_ptr(), sc.data_ptr()
        arr[i].zeros = None if z is None else z.data_ptr()
        arr[i].m, arr[i].out = m, o.data_ptr()
    rc = lib().bitlut_mpgemv_multi(arr, len(mats), k, bits, group_size, dtype_code(mats[0][1]), ptr(tables),
                                   ptr(tscales), ptr(rowsums), flags, stream_of(tables))
    raise_for_status(rc, "bitlut_mpgemv_multi")
    return outs


def mpgemv_multi_tab(mats, k: int, bits: int, group_size: int, flags: int) -> list:
    """bitlut_mpgemv_multi_tab: batch-1 matrices with their own tables in one
    launch; mats = [(wgpu, wscales, zeros, m, tables, tscales, rowsums), ...]
    (fast epilogue).  Returns one (1, m) f32 output per matrix."""
    dev = mats[0][0].device
    outs = [torch.empty((1, m), dtype=torch.float32, device=dev) for (_, _, _, m, _, _, _) in mats]
    arr = (BitlutMatTab * len(mats))()
    for i, ((w, sc, z, m, t, ts, rs), o) in enumerate(zip(mats, outs)):
        arr[i].wgpu, arr[i].wscales = w.data_ptr(), sc.data_ptr()
        arr[i].zeros = None if z is None else z.data_ptr()
        arr[i].m, arr[i].out = m, o.data_ptr()
        arr[i].tables, arr[i].tscales, arr[i].rowsums = t.data_ptr(), ts.data_ptr(), rs.data_ptr()
    rc = lib().bitlut_mpgemv_multi_tab(arr, len(mats), k, bits, group_size, dtype_code(mats[0][1]), flags,
                                       stream_of(mats[0][0]))
    raise_for_status(rc, "bitlut_mpgemv_multi_tab")
    return outs


def mpgemv_gather(wgpu: torch.Tensor, wscales: torch.Tensor, zeros: Optional[torch.Tensor],
                  tables: torch.Tensor, tscales: torch.Tensor, rowsums: torch.Tensor, m: int, k: int, bits: int,
                  group_size: int, peer_out_ptrs: list, peer_flag_ptrs: list,
                  ticket: torch.Tensor, col_offset: int, flags: int) -> torch.Tensor:
    """bitlut_mpgemv_gather: this rank's batch-1 shard lookup with the
    all-gather fused into the epilogue.  peer_out_ptrs / peer_flag_ptrs are
    the device addresses (ints) of every rank's gathered row / flag; returns
    the local (1, m) f32 result."""
    require_cuda(wgpu, "packed weights")
    out = torch.empty((1, m), dtype=torch.float32, device=wgpu.device)
    n = len(peer_out_ptrs)
    if n != len(peer_flag_ptrs):
        raise ParameterError("peer_out_ptrs and peer_flag_ptrs differ in length")
    outs = (ctypes.c_void_p * n)(*peer_out_ptrs)
    fls = (ctypes.c_void_p * n)(*peer_flag_ptrs)
    rc = lib().bitlut_mpgemv_gather(ptr(wgpu), m, k, bits, group_size, ptr(wscales), ptr(zeros),
                                    dtype_code(wscales), ptr(tables), ptr(tscales), ptr(rowsums), ptr(out), n,
                                    outs, fls, ptr(ticket), col_offset, flags, stream_of(wgpu))
    raise_for_status(rc, "bitlut_mpgemv_gather")
    return out


def gather_wait(flag: torch.Tensor, target: int, timed_out: Optional[torch.Tensor] = None) -> None:
    """bitlut_gather_wait on the flag's stream (bounded; sets `timed_out`
    (device int32) when the peers never arrive)."""
    require_cuda(flag, "gather flag")
    raise_for_status(lib().bitlut_gather_wait(ptr(flag), target & 0xFFFFFFFF, ptr(timed_out), stream_of(flag)),
                     "bitlut_gather_wait")


@torch.library.custom_op("bitlut_b200::mpgemv_fused", mutates_args=())
def mpgemv_fused(a: torch.Tensor, wgpu: torch.Tensor, wscales: torch.Tensor,
                 zeros: Optional[torch.Tensor], m: int, k: int, bits: int, group_size: int,
                 flags: int) -> torch.Tensor:
    """Batch-1 table build + lookup in one launch (fast epilogue): a (1, k)
    fp16 -> out (1, m) f32.  Raises LayoutError when the call does not fit
    the fused kernel (callers fall back to build_lut + lookup)."""
    require_cuda(a, "activations")
    out = torch.empty((1, m), dtype=torch.float32, device=wgpu.device)
    rc = lib().bitlut_mpgemv_fused(ptr(a), dtype_code(a), ptr(wgpu), m, k, bits, group_size,
                                   ptr(wscales), ptr(zeros), dtype_code(wscales), ptr(out), flags,
                                   stream_of(wgpu))
    raise_for_status(rc, "bitlut_mpgemv_fused")
    return out


@mpgemv_fused.register_fake
def _(a, wgpu, wscales, zeros, m, k, bits, group_size, flags):
    return wgpu.new_empty((1, m), dtype=torch.float32)


@lookup.register_fake
def _(wgpu, wscales, zeros, tables, tscales, rowsums, m, k, bits, group_size, mode, flags,
      want_partials):
    n = tables.shape[0]
    nq = k // group_size
    pb = 1 if flags & FLAG_COMBINED_PARTIALS else bits
    return (wgpu.new_empty((n, m), dtype=torch.float32),
            wgpu.new_empty((n, pb, m, nq) if want_partials else (0,), dtype=torch.int32))
