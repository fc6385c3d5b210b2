"""mpGEMV / mpGEMM drop-in (reference: pkg/src/bitlut/kernel.py).

Same entry points, argument meaning and error behaviour as the reference's
``mpgemm``/``mpgemv`` (kernel.py:280-382), dispatching to the CUDA kernels
through the torch custom ops in ``_native``:

    a --(bitlut_b200::build_lut)--> int8 tables, table scales, row sums
      --(bitlut_b200::lookup)-----> out (n, m) float32

Variants (``KernelVariant``):
  * ``cuda-q8``  -- int8 tables; output bitwise identical to the
    reference's ``vector-q8`` (and hence ``scalar-q8``), int32 staging
    values exact.  Default.
  * ``cuda-f16`` -- fp16 tables (BASELINE "fp16 tables"); matches the
    reference's fp32-table ``scalar-real`` within max|dy| <= 1e-3 max|y|.
The reference's CPU variants (scalar-real, scalar-q8, vector-q8, fast-agg)
are rejected: this package has no CPU path.

Inputs may be numpy arrays or torch tensors (CPU or CUDA).  Numpy/CPU
inputs are copied to the device and the result is returned the same way
(numpy float32 for numpy input), so host callers see the reference's
contract; CUDA inputs return CUDA tensors without synchronizing.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .core import Matrix, TileConfig, as_tensor
from .errors import DataError, LayoutError, OverflowConfigError, ParameterError, ShapeError, raise_for_status
from .lut_build import REAL, LookupTables
from .weight_prep import LAYOUT_VERSION, PackedWeights

INT32_MAX = 2**31 - 1


class KernelVariant(Enum):
    CUDA_Q8 = "cuda-q8"
    CUDA_F16 = "cuda-f16"


_REFERENCE_CPU_VARIANTS = ("scalar-real", "scalar-q8", "vector-q8", "fast-agg")


def _variant(v) -> KernelVariant:
    if isinstance(v, KernelVariant):
        return v
    name = getattr(v, "value", v)
    if name in _REFERENCE_CPU_VARIANTS:
        raise ParameterError(
            f"variant {name!r} is a CPU kernel of the reference; the B200 package "
            "provides 'cuda-q8' (bitwise identical to vector-q8/scalar-q8) and 'cuda-f16'")
    try:
        return KernelVariant(name)
    except ValueError:
        raise ParameterError(f"unknown kernel variant {name!r}") from None


@dataclass
class KernelStats:
    """kernel.py:41-46.  Filled analytically (the GPU does exactly these)."""

    lookups: int = 0
    lut_builds: int = 0


@dataclass
class Accumulators:
    """kernel.py:49-64 (definitional tile primitive state)."""

    real: torch.Tensor
    integer: torch.Tensor

    @classmethod
    def zeros(cls, channels: int, device=None) -> "Accumulators":
        dev = device or ("cuda" if torch.cuda.is_available() else "cpu")
        return cls(real=torch.zeros(channels, dtype=torch.float32, device=dev),
                   integer=torch.zeros(channels, dtype=torch.int32, device=dev))


def validate_kernel_config(tile: TileConfig, bits: int, group_size: int, m: int, k: int) -> None:
    """kernel.py:67-87, plus the CUDA path's own constraints."""
    if group_size % tile.g != 0:
        raise LayoutError(f"group_size={group_size} not divisible by g={tile.g}")
    if m % tile.m_tile != 0:
        raise LayoutError(f"m={m} not divisible by m_tile={tile.m_tile}")
    if k % tile.k_tile != 0:
        raise LayoutError(f"k={k} not divisible by k_tile={tile.k_tile}")
    if k % group_size != 0:
        raise LayoutError(f"k={k} not divisible by group_size={group_size}")
    if (group_size // tile.g) * 127 > INT32_MAX:
        raise OverflowConfigError(
            f"group accumulation bound exceeded: {group_size // tile.g} "
            f"lookups of magnitude 127 cannot be staged in int32")
    if tile.g != 4:
        raise ParameterError(f"the CUDA kernels implement g=4 (got g={tile.g})")
    if m % 32 != 0:
        raise LayoutError(f"m={m} not divisible by 32 (CUDA tile)")
    gpg = group_size // 4
    if group_size % 16 != 0 or gpg > 128 or (gpg & (gpg - 1)):
        raise ParameterError(
            f"group_size={group_size}: the CUDA kernels need group_size in "
            "{16, 32, 64, 128, 256, 512}")


def _check_layout_match(cfg: TileConfig, pw: PackedWeights) -> None:
    """kernel.py:90-100."""
    if pw.layout_version != LAYOUT_VERSION:
        raise LayoutError(f"packed weights use layout version {pw.layout_version}, "
                          f"kernel implements {LAYOUT_VERSION}")
    t = pw.tile
    if (cfg.m_tile, cfg.k_tile, cfg.g, cfg.lanes) != (t.m_tile, t.k_tile, t.g, t.lanes):
        raise LayoutError("tile config does not match the layout the weights were packed "
                          f"for: {cfg} vs {t}")


def _host_rows(a):
    """Numpy activations (kernel.py:266-277): contiguous (n, k) f16/f32 with the
    reference's host-side finiteness check, or None for tensor inputs."""
    if isinstance(a, Matrix):
        a = a.to_array()
    if not isinstance(a, np.ndarray):
        return None
    arr = a if a.dtype in (np.float16, np.float32) else a.astype(np.float32)
    if arr.ndim == 1:
        arr = arr.reshape(1, -1)
    if arr.ndim != 2:
        raise ShapeError("activations must be 1-D or 2-D")
    arr = np.ascontiguousarray(arr)
    if arr.dtype == np.float16:      # finite <=> exponent bits not all ones (fast integer test)
        bad = bool(((arr.view(np.uint16) & 0x7C00) == 0x7C00).any())
    else:
        bad = not np.isfinite(arr).all()
    if bad:
        raise DataError("activations contain non-finite values")
    return arr


def _activation_rows(a, check_finite=None):
    """kernel.py:266-277: -> (device tensor (n, k) f16/f32, how-to-return).

    Host inputs (numpy, CPU tensors) are checked for non-finite values on the
    host, as the reference does.  CUDA inputs are not checked unless
    ``check_finite=True`` (that check needs a host synchronization); a
    non-finite activation then yields non-finite outputs (the table build
    propagates NaN/Inf into the table scales and row sums)."""
    kind = "cuda"
    if isinstance(a, Matrix):
        a = a.to_array()
    if isinstance(a, np.ndarray):
        kind = "numpy"
        t = torch.from_numpy(_host_rows(a).copy())
    else:
        t = as_tensor(a)
        if t.dtype not in (torch.float16, torch.float32):
            t = t.to(torch.float32)
        if t.dim() == 1:
            t = t.reshape(1, -1)
        if t.dim() != 2:
            raise ShapeError("activations must be 1-D or 2-D")
        if not t.is_cuda:
            kind = "cpu"
            if not bool(torch.isfinite(t).all()):
                raise DataError("activations contain non-finite values")
        elif check_finite and not bool(torch.isfinite(t).all()):
            raise DataError("activations contain non-finite values")
    if not t.is_cuda:
        if not torch.cuda.is_available():
            raise N.BitLutError("a CUDA device is required (the B200 package has no CPU path)")
        t = t.to("cuda", non_blocking=True)
    return t.contiguous(), kind


_TLS = threading.local()
_SCRATCH_MAX = 16
# the lookup writes the result straight into the pinned (UVA-mapped) staging
# buffer (no D2H copy operation: -5..-8 us per call, tools/per_call_profile.py);
# reading the activations the same way was slower (the fused build reads them
# from every CTA).  BITLUT_ZERO_COPY = "in,out" (diagnostic)
import os as _os
_ZERO_COPY = tuple(bool(int(x)) for x in _os.environ.get("BITLUT_ZERO_COPY", "0,1").split(","))


class _HostScratch:
    """Per-thread, per-shape buffers of the host-buffer call: pinned staging
    for the activations and the result, device scratch for the tables and
    the output (allocated once, reused by every later call of the shape)."""

    def __init__(self, dev, n, k, m, gs, a_dtype, mode):
        tdt = torch.int8 if mode == N.TABLE_Q8 else torch.float16
        self.a_host = torch.empty((n, k), dtype=a_dtype, pin_memory=True)
        self.a_np = self.a_host.numpy()
        self.a_dev = torch.empty((n, k), dtype=a_dtype, device=dev)
        self.tables = torch.empty((n, k // 4, 8), dtype=tdt, device=dev)
        self.ts = torch.empty((n, k // gs), dtype=torch.float32, device=dev)
        self.rs = torch.empty((n, k // gs), dtype=torch.float32, device=dev)
        self.out_dev = torch.empty((n, m), dtype=torch.float32, device=dev)
        self.out_host = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
        self.out_np = self.out_host.numpy()


def _scratch(dev, n, k, m, gs, a_dtype, mode) -> _HostScratch:
    cache = getattr(_TLS, "scratch", None)
    if cache is None:
        cache = _TLS.scratch = {}
    key = (dev.index, n, k, m, gs, a_dtype, mode)
    b = cache.get(key)
    if b is None:
        if len(cache) >= _SCRATCH_MAX:
            cache.pop(next(iter(cache)))
        b = cache[key] = _HostScratch(dev, n, k, m, gs, a_dtype, mode)
    return b


def _host_call(rows: np.ndarray, pw: PackedWeights, mode: int, flags: int) -> np.ndarray:
    """numpy in -> numpy out through bitlut_mpgemm_host: one C call does the
    H2D copy, the table build + lookup launch(es), the D2H copy and the
    stream synchronization (csrc/host_api.cu)."""
    n, k = rows.shape
    a_dtype = torch.float16 if rows.dtype == np.float16 else torch.float32
    dev = pw.gpu.device
    b = _scratch(dev, n, k, pw.m, pw.group_size, a_dtype, mode)
    np.copyto(b.a_np, rows)
    if torch.cuda.current_device() != dev.index:
        torch.cuda.set_device(dev)
    zc_in, zc_out = _ZERO_COPY
    rc = N.lib().bitlut_mpgemm_host(
        b.a_host.data_ptr(), N.DT_F16 if a_dtype == torch.float16 else N.DT_F32, n, k, pw.gpu.data_ptr(), pw.m,
        pw.bits, pw.group_size, pw.scales.data_ptr(), None if pw.zeros is None else pw.zeros.data_ptr(),
        N.dtype_code(pw.scales), mode, flags, b.a_host.data_ptr() if zc_in else b.a_dev.data_ptr(),
        b.tables.data_ptr(), b.ts.data_ptr(), b.rs.data_ptr(),
        b.out_host.data_ptr() if zc_out else b.out_dev.data_ptr(), b.out_host.data_ptr(),
        torch.cuda.current_stream(dev).cuda_stream)
    raise_for_status(rc, "bitlut_mpgemm_host")
    return b.out_np.copy()


def mpgemm(a, pw: PackedWeights, cfg: TileConfig | None = None,
           variant: KernelVariant | str = KernelVariant.CUDA_Q8,
           threads: int = 1, stats: KernelStats | None = None, *,
           check_finite: bool | None = None, return_partials: bool = False, pdl: bool = True,
           exact_epilogue: bool = True):
    """Mixed-precision GEMM: (N, K) activations x packed low-bit weights.

    Returns (N, M) float32 (numpy for numpy input, a CUDA tensor for CUDA
    input).  ``return_partials`` (cuda-q8) additionally returns the exact
    int32 staging values, shape (N, bits, M, K/group_size).
    ``exact_epilogue=False`` keeps those exact int32 values but combines
    them with a fixed-order parallel float reduction instead of the
    reference's sequential one (faster; last-bits differences only).
    """
    variant = _variant(variant)
    cfg = pw.tile if cfg is None else cfg
    if cfg.n_tile < 1:
        raise ParameterError("n_tile must be >= 1")
    _check_layout_match(cfg, pw)
    validate_kernel_config(cfg, pw.bits, pw.group_size, pw.m, pw.k)
    if threads < 1:
        raise ParameterError("threads must be >= 1")
    if pw.gpu is None:
        raise LayoutError("packed weights carry no GPU layout (prepare them with prepare_weights)")
    mode = N.TABLE_Q8 if variant is KernelVariant.CUDA_Q8 else N.TABLE_F16
    if return_partials and mode != N.TABLE_Q8:
        raise ParameterError("exact int32 partials exist only for int8 tables (cuda-q8)")
    flags = (N.FLAG_PDL if pdl else 0) | (0 if exact_epilogue else N.FLAG_FAST_EPILOGUE)
    host = None if return_partials else _host_rows(a)
    if host is not None:                       # numpy in, numpy out: one C call, one sync
        if host.shape[1] != pw.k:
            raise ShapeError(f"activation length {host.shape[1]} != weight k {pw.k}")
        # cuda-f16 fast at batch 1: 16-bit block-fixed-point tables (BITLUT_TABLE_X16)
        x16 = mode == N.TABLE_F16 and not exact_epilogue and host.shape[0] == 1 and pw.bits != 3
        try:
            out = _host_call(host, pw, N.TABLE_X16 if x16 else mode, flags)
        except LayoutError:
            if not x16:
                raise
            out = _host_call(host, pw, mode, flags)
        if stats is not None:
            stats.lookups += pw.bits * host.shape[0] * pw.m * (pw.k // pw.g)
            stats.lut_builds += -(-host.shape[0] // cfg.n_tile) * (pw.k // cfg.k_tile)
        return out
    rows, kind = _activation_rows(a, check_finite)
    n, k = rows.shape
    if k != pw.k:
        raise ShapeError(f"activation length {k} != weight k {pw.k}")
    if rows.device != pw.gpu.device:
        rows = rows.to(pw.gpu.device)
    out = None
    if (mode == N.TABLE_Q8 and not exact_epilogue and not return_partials and n == 1
            and rows.dtype == torch.float16 and pw.bits != 3):
        try:      # table build + lookup in one launch (csrc/gemv_b1.cu)
            out = N.mpgemv_fused(rows, pw.gpu, pw.scales, pw.zeros, pw.m, pw.k, pw.bits,
                                 pw.group_size, flags)
            partials = None
        except LayoutError:
            out = None
    if out is None and mode == N.TABLE_F16 and not exact_epilogue and n == 1 and pw.bits != 3:
        try:      # cuda-f16 fast at batch 1: 16-bit block-fixed-point tables (BITLUT_TABLE_X16)
            tables, ts, rs = N.build_lut(rows, pw.group_size, N.TABLE_X16, N.FLAG_PDL if pdl else 0)
            ls = pw.__dict__.get("_layer_set") if pw.encoding in ("offset", "zeros") else None
            if ls is not None:
                try:
                    out, partials = N.lookup(ls[0], ls[1], ls[2], tables, ts, rs, pw.m, pw.k, pw.bits,
                                             pw.group_size, N.TABLE_X16, flags | N.FLAG_LAYER_SET, False)
                except LayoutError:
                    out = None
            if out is None:
                out, partials = N.lookup(pw.gpu, pw.scales, pw.zeros, tables, ts, rs, pw.m, pw.k, pw.bits,
                                         pw.group_size, N.TABLE_X16, flags, False)
        except LayoutError:
            out = None
    if out is None:
        tables, ts, rs = N.build_lut(rows, pw.group_size, mode, N.FLAG_PDL if pdl else 0)
        ls = pw.__dict__.get("_layer_set")        # set by pw.layer_set_operand() (opt-in, second copy)
        if (ls is not None and mode == N.TABLE_Q8 and not exact_epilogue and not return_partials
                and pw.encoding in ("offset", "zeros")):   # (sign / ternary: their layer-set scales are the native ones)
            try:      # the layer-set operand in the lean kernels (select-free reductions): same bits
                out, partials = N.lookup(ls[0], ls[1], ls[2], tables, ts, rs,
                                         pw.m, pw.k, pw.bits, pw.group_size, mode, flags | N.FLAG_LAYER_SET, False)
            except LayoutError:
                out = None
    if out is None:
        out, partials = N.lookup(pw.gpu, pw.scales, pw.zeros, tables, ts, rs, pw.m, pw.k, pw.bits,
                                 pw.group_size, mode, flags, return_partials)
    if stats is not None:
        stats.lookups += pw.bits * n * pw.m * (pw.k // pw.g)
        stats.lut_builds += -(-n // cfg.n_tile) * (pw.k // cfg.k_tile)
    if kind == "numpy":
        out = out.cpu().numpy()
        partials = partials.cpu().numpy() if return_partials else None
    elif kind == "cpu":
        out = out.cpu()
        partials = partials.cpu() if return_partials else None
    return (out, partials) if return_partials else out


def mpgemv(a_row, pw: PackedWeights, cfg: TileConfig | None = None,
           variant: KernelVariant | str = KernelVariant.CUDA_Q8,
           threads: int = 1, stats: KernelStats | None = None, **kw):
    """kernel.py:374-382: one activation row, returns a length-M vector."""
    if isinstance(a_row, np.ndarray):
        if a_row.ndim != 1:
            raise ShapeError("mpgemv expects a 1-D activation row")
    elif isinstance(a_row, torch.Tensor) and a_row.dim() != 1:
        raise ShapeError("mpgemv expects a 1-D activation row")
    res = mpgemm(a_row.reshape(1, -1), pw, cfg=cfg, variant=variant, threads=threads,
                 stats=stats, **kw)
    if kw.get("return_partials"):
        return res[0][0], res[1][0]
    return res[0]


def lookup_accumulate_tile(indices, lut: LookupTables, acc: Accumulators, row: int = 0,
                           kg_offset: int = 0) -> Accumulators:
    """kernel.py:190-223: definitional tile primitive (device tensor ops; not
    the hot path -- the hot path is csrc/gemv.cu)."""
    idx = as_tensor(indices).to(acc.integer.device)
    if idx.dim() != 2:
        raise ShapeError("index tile must be 2-D")
    if idx.numel() and int(idx.max()) >= (1 << lut.g):
        raise ParameterError("tile contains indices out of range")
    ii = idx.to(torch.int64)
    if lut.consolidated:
        flip = ii >> (lut.g - 1)
        eff = ii ^ (flip * ((1 << lut.g) - 1))
    else:
        flip = torch.zeros_like(ii)
        eff = ii
    kg = kg_offset + torch.arange(idx.shape[1], device=ii.device)
    if lut.mode == REAL:
        vals = lut.entries[row].to(ii.device)[kg[None, :], eff]
        vals = torch.where(flip == 1, -vals, vals)
        acc.real += vals.sum(dim=1, dtype=torch.float32)
    else:
        vals = lut.qentries[row].to(ii.device)[kg[None, :], eff].to(torch.int32)
        vals = torch.where(flip == 1, -vals, vals)
        acc.integer += vals.sum(dim=1, dtype=torch.int32)
    return acc
