"""Offline weight pipeline on the GPU (reference: pkg/src/bitlut/weight_prep.py).

``prepare_weights`` runs three CUDA kernels (csrc/weight_prep.cu):
decompose q into bit-plane indices (weight_prep.py:86-105), pack them into
the reference's v1 layout (tile permutation + interleave, :193-246) so
``PackedWeights.planes`` is byte-identical to the reference's, and repack
them into layout v2 -- the mirror-encoded, unit-interleaved layout the
lookup kernel streams with coalesced 256-bit loads (layout.cuh).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _native as N
from .core import DEFAULT_TILE, QuantizedWeights, TileConfig, as_tensor, indices_per_byte
from .errors import LayoutError, ParameterError, ShapeError, raise_for_status

LAYOUT_VERSION = 1       # PackedWeights.planes (reference layout, docs/formats.md)
GPU_LAYOUT_VERSION = 2   # PackedWeights.gpu (this package's kernel layout)


def _device(dev=None) -> torch.device:
    if dev is not None:
        return torch.device(dev)
    if not torch.cuda.is_available():
        raise N.BitLutError("a CUDA device is required (the B200 package has no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, device, dtype=None) -> torch.Tensor:
    t = as_tensor(x, dtype)
    return t.to(device, non_blocking=True).contiguous()


@dataclass(frozen=True)
class BitPlane:
    """g-bit-grouped indices of one bit position (weight_prep.py:35-47)."""

    bit: int
    g: int
    indices: torch.Tensor  # uint8 (m, k // g), on the device

    def __post_init__(self):
        if self.indices.dtype != torch.uint8:
            raise ParameterError("plane indices must be uint8")


@dataclass(frozen=True)
class PackedWeights:
    """Kernel-side weight operand (weight_prep.py:50-83).

    ``planes`` is the reference's v1 layout (byte-identical);
    ``gpu`` is layout v2 consumed by the CUDA lookup kernel (None when the
    shape is outside the CUDA path, e.g. g != 4).
    """

    m: int
    k: int
    bits: int
    g: int
    group_size: int
    tile: TileConfig
    planes: torch.Tensor                 # uint8 (bits, plane_bytes)
    scales: torch.Tensor                 # float32/float16 (m, k // group_size)
    zeros: Optional[torch.Tensor] = None
    gpu: Optional[torch.Tensor] = field(default=None, compare=False)
    layout_version: int = LAYOUT_VERSION
    # QuantizedWeights.encoding; native_scales: what the batch executor reads
    # for it (sign: s of w = s (2q - 1); ternary: the one per-tensor scale)
    encoding: str = "offset"
    native_scales: Optional[torch.Tensor] = field(default=None, compare=False)

    def __post_init__(self):
        expected = self.m * (self.k // self.g) // indices_per_byte(self.g)
        if tuple(self.planes.shape) != (self.bits, expected):
            raise ShapeError(f"planes shape {tuple(self.planes.shape)} does not match "
                             f"(bits={self.bits}, plane_bytes={expected})")
        if tuple(self.scales.shape) != (self.m, self.k // self.group_size):
            raise ShapeError("scales shape mismatch")
        if self.encoding == "offset" and self.zeros is not None:
            object.__setattr__(self, "encoding", "zeros")

    def layer_set_operand(self):
        """(weights, scales, zeros) in the layer-set layout the batch executor
        reads (include/bitlut_b200.h bitlut_layer_set_*; csrc/layout.cuh),
        converted from the v2 operand on first use and cached.  scales: the
        encoding's scale stream (sign planes: native_scales; ternary: None,
        the one per-tensor value is passed as is)."""
        cached = self.__dict__.get("_layer_set")
        if cached is None:
            if self.gpu is None:
                raise LayoutError("packed weights carry no GPU layout")
            args = (self.bits, self.m, self.k, self.group_size)
            w = N.layer_set_weights(self.gpu, *args)
            src = self.native_scales if self.encoding == "sign" else self.scales
            sc = None if self.encoding == "ternary" else N.layer_set_scales(src, *args)
            z = N.layer_set_scales(self.zeros, *args) if self.encoding == "zeros" else None
            cached = (w, sc, z)
            object.__setattr__(self, "_layer_set", cached)
        return cached

    @property
    def plane_bytes(self) -> int:
        return self.planes.shape[1]

    @property
    def index_slots(self) -> int:
        return self.bits * self.m * (self.k // self.g)

    @property
    def n_groups(self) -> int:
        return self.k // self.group_size

    @property
    def packed_bytes(self) -> int:
        """Packed-weight bytes per call = bits*M*K/8 (the BASELINE metric's
        numerator; the reference's weight_bytes, cli.py:153)."""
        return self.bits * self.plane_bytes

    @property
    def device(self) -> torch.device:
        return self.planes.device


def decompose_bits(qw: QuantizedWeights, g: int, device=None) -> list[BitPlane]:
    """weight_prep.py:86-105 on the GPU."""
    if not 1 <= g <= 8:
        raise ParameterError(f"g must be in [1, 8], got {g}")
    if qw.k % g != 0:
        raise LayoutError(f"k={qw.k} not divisible by g={g}; pad the weights first")
    dev = _device(device if device is not None else
                  (qw.qvalues.device if isinstance(qw.qvalues, torch.Tensor) and qw.qvalues.is_cuda
                   else None))
    q = to_device(qw.qvalues, dev, torch.uint8)
    idx = torch.empty((qw.bits, qw.m, qw.k // g), dtype=torch.uint8, device=dev)
    rc = N.lib().bitlut_decompose_bits(N.ptr(q), qw.m, qw.k, qw.bits, g, N.ptr(idx), N.stream_of(q))
    raise_for_status(rc, "bitlut_decompose_bits")
    return [BitPlane(bit=i, g=g, indices=idx[i]) for i in range(qw.bits)]


def _stack(planes: list[BitPlane]) -> torch.Tensor:
    idx = torch.stack([p.indices for p in planes]).contiguous()
    if not idx.is_cuda:
        idx = idx.to(_device())
    return idx


def repack_gpu(indices: torch.Tensor, m: int, k: int, bits: int, group_size: int) -> torch.Tensor:
    """Plane indices (bits, m, k/4) -> layout v2 bytes (north-star kernel 1)."""
    lay = N.layout_query(m, k, bits, group_size)
    out = torch.empty(int(lay.bytes), dtype=torch.uint8, device=indices.device)
    rc = N.lib().bitlut_repack_gpu(N.ptr(indices), bits, m, k, group_size, N.ptr(out),
                                   N.stream_of(indices))
    raise_for_status(rc, "bitlut_repack_gpu")
    return out


def unrepack_gpu(pw: PackedWeights) -> torch.Tensor:
    """Inverse of repack_gpu: layout v2 -> plane indices (bits, m, k/4)."""
    idx = torch.empty((pw.bits, pw.m, pw.k // 4), dtype=torch.uint8, device=pw.gpu.device)
    rc = N.lib().bitlut_unrepack_gpu(N.ptr(pw.gpu), pw.bits, pw.m, pw.k, pw.group_size,
                                     N.ptr(idx), N.stream_of(idx))
    raise_for_status(rc, "bitlut_unrepack_gpu")
    return idx


def gpu_layout_ok(m: int, k: int, bits: int, g: int, group_size: int) -> bool:
    if g != 4:
        return False
    try:
        N.layout_query(m, k, bits, group_size)
        return True
    except Exception:
        return False


def pack_and_permute(planes: list[BitPlane], tile: TileConfig, scales, group_size: int,
                     zeros=None, encoding=None) -> PackedWeights:
    """weight_prep.py:214-246: v1 planes (byte-identical to the reference)
    plus the layout-v2 operand for the CUDA kernel."""
    if not planes:
        raise ParameterError("no bit planes given")
    g = planes[0].g
    m, kg_total = planes[0].indices.shape
    k = kg_total * g
    if tile.g != g:
        raise LayoutError(f"tile g={tile.g} does not match plane g={g}")
    if m % tile.m_tile != 0:
        raise LayoutError(f"m={m} not divisible by m_tile={tile.m_tile}")
    if kg_total % tile.k_groups_per_tile != 0:
        raise LayoutError(f"k={k} not divisible by k_tile={tile.k_tile}")
    if group_size % g != 0:
        raise LayoutError(f"group_size={group_size} not divisible by g={g}")
    if k % group_size != 0:
        raise LayoutError(f"k={k} not divisible by group_size={group_size}")
    idx = _stack(planes)
    dev = idx.device
    bits = idx.shape[0]
    plane_bytes = m * kg_total // indices_per_byte(g)
    v1 = torch.empty((bits, plane_bytes), dtype=torch.uint8, device=dev)
    rc = N.lib().bitlut_pack_v1(N.ptr(idx), bits, m, k, g, tile.m_tile, tile.k_tile, tile.lanes,
                                N.ptr(v1), N.stream_of(idx))
    raise_for_status(rc, "bitlut_pack_v1")
    gpu = repack_gpu(idx, m, k, bits, group_size) if gpu_layout_ok(m, k, bits, g, group_size) else None
    s = to_device(scales, dev)
    if s.dtype not in (torch.float32, torch.float16):
        s = s.float()
    z = None if zeros is None else to_device(zeros, dev, s.dtype)
    enc = encoding or ("offset" if z is None else "zeros")
    native = None
    if enc == "sign":           # generic form (2s, 1/2) -> s (exact halving)
        native = (s.float() * 0.5).to(s.dtype).contiguous()
    elif enc == "ternary":      # the one per-tensor scale
        native = s.reshape(-1)[:1].clone()
    return PackedWeights(m=m, k=k, bits=bits, g=g, group_size=group_size, tile=tile, planes=v1,
                         scales=s, zeros=z, gpu=gpu, encoding=enc, native_scales=native)


def unpack_planes(pw: PackedWeights) -> list[BitPlane]:
    """weight_prep.py:249-257 on the GPU (inverse of the v1 packing)."""
    kg_total = pw.k // pw.g
    idx = torch.empty((pw.bits, pw.m, kg_total), dtype=torch.uint8, device=pw.planes.device)
    rc = N.lib().bitlut_unpack_v1(N.ptr(pw.planes), pw.bits, pw.m, pw.k, pw.g, pw.tile.m_tile,
                                  pw.tile.k_tile, pw.tile.lanes, N.ptr(idx), N.stream_of(idx))
    raise_for_status(rc, "bitlut_unpack_v1")
    return [BitPlane(bit=i, g=pw.g, indices=idx[i]) for i in range(pw.bits)]


def prepare_weights(qw: QuantizedWeights, tile: TileConfig = DEFAULT_TILE, device=None) -> PackedWeights:
    """weight_prep.py:260-263: decompose, pack (v1), repack (v2) -- all on the GPU."""
    planes = decompose_bits(qw, tile.g, device=device)
    return pack_and_permute(planes, tile, qw.scales, qw.group_size, zeros=qw.zeros, encoding=qw.encoding)


def from_v1(pw: PackedWeights) -> PackedWeights:
    """Attach the layout-v2 operand to v1-only packed weights (e.g. planes
    loaded from an LMPW file): unpack v1 on the GPU, repack to v2."""
    if pw.gpu is not None:
        return pw
    planes = unpack_planes(pw)
    return pack_and_permute(planes, pw.tile, pw.scales, pw.group_size, zeros=pw.zeros, encoding=pw.encoding)
