"""The rest of the reference package's public names (bitlut/__init__.py
`__all__`), so code written against the reference imports unchanged.

* Offline weight helpers: `pad_weights` (weight_prep.py:108-128),
  `interleave_layout` / `deinterleave_layout` (weight_prep.py:131-176).
* Lookup primitives whose semantics the GPU kernels implement with PRMT
  (kernel.py:157-187): `byte_parallel_lookup`, `wide_lookup`,
  `split_wide_table`; and the reference's approximate aggregation
  (kernel.py:103-154): `rhadd`, `rhadd_tree`, `bias_correction`,
  `fast_aggregate` (excluded from the exactness guarantees there as here).
* Definitional references (oracle.py:26-100) computed on the GPU with torch:
  `reference_gemm` (fp32 GEMM), `reference_mpgemm` (dequantize then GEMM),
  `reference_lut_mpgemv` (literal lookup over full, unconsolidated tables).
  They are validation utilities for NMSE reports, not the lookup path: the
  fp32 summation order is torch's, so they agree with the reference's
  ascending-k loops to rounding, not bitwise.

The tuner names (`tune`, `enumerate_configs`, `TuneResult`) are not provided:
the CUDA kernels choose their tiling from the shape (SURVEY.md §2 marks the
tuner out of scope).
"""
from __future__ import annotations

import numpy as np
import torch

from .core import QuantizedWeights, as_tensor, indices_per_byte, slot_bits
from .errors import LayoutError, ParameterError, ShapeError


# ---------------------------------------------------------------- weights

def pad_weights(qw: QuantizedWeights, m_multiple: int, k_multiple: int) -> QuantizedWeights:
    """Grow (m, k) to multiples of (m_multiple, lcm(k_multiple, group_size)).
    New K positions hold the implicit zero point 2^(b-1) with zero scales
    (they dequantize to 0); new rows are zero rows with zero scales.  Zero
    points, when present, are extended with the implicit value."""
    if m_multiple < 1 or k_multiple < 1:
        raise ParameterError("padding multiples must be positive")
    if qw.k % qw.group_size != 0:
        raise LayoutError("k must remain a multiple of group_size")
    k_step = int(np.lcm(k_multiple, qw.group_size))
    new_k = -(-qw.k // k_step) * k_step
    new_m = -(-qw.m // m_multiple) * m_multiple
    if (new_m, new_k) == (qw.m, qw.k):
        return qw
    q0, s0 = as_tensor(qw.qvalues), as_tensor(qw.scales)
    q = torch.full((new_m, new_k), qw.offset, dtype=torch.uint8, device=q0.device)
    q[:qw.m, :qw.k] = q0
    s = torch.zeros((new_m, new_k // qw.group_size), dtype=s0.dtype, device=s0.device)
    s[:qw.m, :qw.k // qw.group_size] = s0
    z = None
    if qw.zeros is not None:
        z0 = as_tensor(qw.zeros)
        z = torch.full(tuple(s.shape), float(qw.offset), dtype=z0.dtype, device=z0.device)
        z[:qw.m, :qw.k // qw.group_size] = z0
    return QuantizedWeights(m=new_m, k=new_k, bits=qw.bits, group_size=qw.group_size, qvalues=q, scales=s,
                            zeros=z)


def interleave_layout(indices, g: int, lanes: int) -> np.ndarray:
    """Pack an index stream into bytes so that unpacking is mask and shift
    only.  The stream is cut into units of indices_per_byte(g) * lanes
    indices; each unit is folded in halves, the second half shifted above
    the first: for g = 4, byte j = idx[j] | idx[j + lanes] << 4; narrower
    slots fold again (2-bit, then 1-bit fields)."""
    idx = np.ascontiguousarray(as_tensor(indices).cpu().numpy(), dtype=np.uint8).reshape(-1)
    per = indices_per_byte(g)
    if lanes < 1 or idx.size % lanes != 0:
        raise LayoutError(f"index span {idx.size} not divisible by lanes={lanes}")
    if per == 1:
        return idx.copy()
    unit = per * lanes
    if idx.size % unit != 0:
        raise LayoutError(f"index span {idx.size} not divisible by the {unit}-index packing unit for g={g}")
    out = idx.reshape(-1, unit).astype(np.uint16)
    width = slot_bits(g)
    while out.shape[1] > lanes:
        h = out.shape[1] // 2
        out = out[:, :h] | (out[:, h:] << width)
        width *= 2
    return out.astype(np.uint8).reshape(-1)


def deinterleave_layout(packed, g: int, lanes: int) -> np.ndarray:
    """Inverse of interleave_layout: bytes back to the index stream."""
    b = np.ascontiguousarray(as_tensor(packed).cpu().numpy(), dtype=np.uint8).reshape(-1)
    per = indices_per_byte(g)
    if lanes < 1 or b.size % lanes != 0:
        raise LayoutError(f"byte span {b.size} not divisible by lanes={lanes}")
    if per == 1:
        return b.copy()
    cur = b.reshape(-1, lanes).astype(np.uint16)
    width = 8
    while width > slot_bits(g):
        width //= 2
        mask = (1 << width) - 1
        cur = np.concatenate([cur & mask, cur >> width], axis=1)
    return cur.astype(np.uint8).reshape(-1)


# ---------------------------------------------------------------- lookup primitives

def byte_parallel_lookup(table, indices) -> np.ndarray:
    """The bytes of a one-dimensional table selected by index bytes (the
    semantics the kernels' PRMT lookups implement)."""
    tab = np.asarray(as_tensor(table).cpu().numpy() if isinstance(table, torch.Tensor) else table)
    idx = np.asarray(as_tensor(indices).cpu().numpy() if isinstance(indices, torch.Tensor) else indices,
                     dtype=np.uint8)
    if tab.ndim != 1:
        raise ShapeError("table must be one-dimensional")
    if idx.size and int(idx.max()) >= tab.shape[0]:
        raise ParameterError("lookup index out of table range")
    return tab[idx]


def split_wide_table(table_i16) -> tuple[np.ndarray, np.ndarray]:
    """int16 table -> (low, high) byte planes for wide_lookup."""
    t = np.asarray(table_i16, dtype=np.int16).view(np.uint16)
    return (t & 0xFF).astype(np.uint8), (t >> 8).astype(np.uint8)


def wide_lookup(table_lo, table_hi, indices) -> np.ndarray:
    """16-bit lookups as two byte lookups recombined (exact int16 values;
    the fp16 table path gathers its low / high byte planes the same way)."""
    lo = byte_parallel_lookup(np.asarray(table_lo, dtype=np.uint8), indices).astype(np.uint16)
    hi = byte_parallel_lookup(np.asarray(table_hi, dtype=np.uint8), indices).astype(np.uint16)
    return ((hi << 8) | lo).view(np.int16)


def rhadd(a: int, b: int) -> int:
    """Rounding halving add of two integers: floor((a + b + 1) / 2)."""
    return (int(a) + int(b) + 1) >> 1


def rhadd_tree(values) -> int:
    """Balanced pairwise rhadd reduction of a power-of-two count of values."""
    vals = [int(v) for v in np.asarray(values).reshape(-1)]
    if not vals or len(vals) & (len(vals) - 1):
        raise ParameterError("rhadd_tree needs a power-of-two value count")
    while len(vals) > 1:
        vals = [rhadd(vals[i], vals[i + 1]) for i in range(0, len(vals), 2)]
    return vals[0]


def bias_correction(depth: int) -> float:
    """Expected upward bias of a depth-level rhadd tree rescaled by 2^depth:
    each of the 2^depth - 1 halving adds rounds ties up (+1/4 expected at its
    own scale), which sums to depth * 2^(depth-2)."""
    if depth < 0:
        raise ParameterError("depth must be >= 0")
    return depth * 2.0 ** (depth - 2)


def chain_bias_correction(depth: int, bits: int) -> float:
    """Expected bias of per-plane rhadd trees followed by a halving chain
    over the bit planes (plane i weighted 2^(i-1)):
    2^(depth-1) * (2^bits - 1) * (depth + 2) / 4."""
    if depth < 0 or bits < 1:
        raise ParameterError("invalid fast-aggregation shape")
    return 2.0 ** (depth - 1) * ((1 << bits) - 1) * (depth + 2) / 4.0


def fast_aggregate(partials, depth: int) -> float:
    """Approximate sum of 2^depth 8-bit partials: rhadd tree * 2^depth minus
    the expected bias (approximate by construction)."""
    vals = np.asarray(partials).reshape(-1)
    if vals.size != 1 << depth:
        raise ParameterError(f"expected {1 << depth} partials for depth {depth}, got {vals.size}")
    return float(rhadd_tree(vals)) * (1 << depth) - bias_correction(depth)


# ---------------------------------------------------------------- definitional references (GPU)

def _cuda(x) -> torch.Tensor:
    t = as_tensor(x)
    if not torch.cuda.is_available():
        raise ParameterError("the definitional references run on the GPU (torch, CUDA)")
    return t.to("cuda")


def reference_gemm(a, w) -> np.ndarray:
    """Plain fp32 GEMM: activations (N, K) times weights (M, K) transposed,
    on the GPU (TF32 off); returns numpy (N, M) float32."""
    x = _cuda(a).float()
    x = x.reshape(1, -1) if x.dim() == 1 else x
    wm = _cuda(w).float()
    if x.shape[1] != wm.shape[1]:
        raise ShapeError(f"activation length {x.shape[1]} != weight k {wm.shape[1]}")
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        y = x @ wm.t()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return y.cpu().numpy().astype(np.float32)


def reference_mpgemm(a, qw: QuantizedWeights) -> np.ndarray:
    """Dequantize, then multiply (the semantics every mpGEMM variant must
    reproduce up to its tolerance)."""
    from .quantize import dequantize
    return reference_gemm(a, dequantize(qw))


def reference_lut_mpgemv(a_row, planes, params, scales) -> np.ndarray:
    """Literal table-lookup GEMV over full (unconsolidated) 2^g tables: per
    quantization group sum_i alpha_i 2^i P_i plus (combined_bias - 2^(b-1))
    times the group's activation sum, times the group scale; no packing,
    tiling or mirroring, so it validates the offline pipeline and the
    kernels jointly."""
    row = _cuda(a_row).float().reshape(-1)
    g = planes[0].g
    k = row.shape[0]
    idx0 = _cuda(planes[0].indices)
    m, kg = idx0.shape
    if kg * g != k:
        raise ShapeError("plane width does not match activation length")
    sc = _cuda(scales).float()
    nq = sc.shape[1]
    if k % nq != 0:
        raise ShapeError("scales width does not divide k")
    gpg = (k // nq) // g
    grouped = row.reshape(kg, g)
    bits_of = ((torch.arange(1 << g, device=row.device)[:, None] >> torch.arange(g, device=row.device)) & 1)
    signs = bits_of.float() * 2 - 1                                   # (2^g, g)
    table = grouped @ signs.t()                                       # (kg, 2^g)
    per_group = torch.zeros((m, nq), dtype=torch.float32, device=row.device)
    cols = torch.arange(kg, device=row.device)[None, :]
    for i, pl in enumerate(planes):
        looked = table[cols, _cuda(pl.indices).long()]                # (m, kg)
        per_group += float(params.alpha[i] * (1 << i)) * looked.reshape(m, nq, gpg).sum(dim=2)
    bias = float(params.combined_bias - (1 << (params.bits - 1)))
    per_group += bias * row.reshape(nq, -1).sum(dim=1)[None, :]
    return (per_group * sc).sum(dim=1).cpu().numpy().astype(np.float32)
