"""Core domain types (reference: pkg/src/bitlut/core.py).

Same names, fields and validation as the reference, with two extensions
the north star needs:

* ``QuantizedWeights.zeros`` -- optional per-group zero points (fp16/fp32).
  ``None`` keeps the reference's symmetric scheme with the implicit zero
  ``2**(bits-1)`` (core.py:86-100).  A zero point z gives w = s*(q - z); 1-bit
  sign planes (w = +-s) are (scale 2s, z = 0.5) and ternary {-1,0,+1} is
  (bits 2, q = v+1, z = 1) -- see ``QuantizedWeights.sign_planes`` /
  ``QuantizedWeights.ternary``.
* arrays may be numpy arrays or torch tensors (CPU or CUDA); fp16 scales,
  zeros and activations are accepted as-is (they upcast exactly to fp32).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import DataError, LayoutError, ParameterError, ShapeError

DEFAULT_GROUP_SIZE = 32
DEFAULT_LANES = 16


def slot_bits(g: int) -> int:
    """core.py:18-37: power-of-two slot width of one packed index."""
    if not 1 <= g <= 8:
        raise ParameterError(f"g must be in [1, 8], got {g}")
    if g == 1:
        return 1
    if g == 2:
        return 2
    if g <= 4:
        return 4
    return 8


def indices_per_byte(g: int) -> int:
    return 8 // slot_bits(g)


def as_tensor(x, dtype=None) -> torch.Tensor:
    """numpy / torch -> torch tensor (no copy when already a tensor of dtype)."""
    if isinstance(x, torch.Tensor):
        return x if dtype is None or x.dtype == dtype else x.to(dtype)
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t if dtype is None or t.dtype == dtype else t.to(dtype)


def _shape(x):
    return tuple(x.shape)


def _all_finite(x) -> bool:
    if isinstance(x, torch.Tensor):
        return bool(torch.isfinite(x.float()).all())
    return bool(np.isfinite(np.asarray(x, dtype=np.float32)).all())


def _max(x) -> int:
    if isinstance(x, torch.Tensor):
        return int(x.max()) if x.numel() else 0
    return int(np.asarray(x).max(initial=0))


@dataclass(frozen=True)
class Matrix:
    """Row-major real matrix (core.py:40-83); ``data`` float32, finite."""

    data: object

    def __post_init__(self):
        a = self.data
        if len(_shape(a)) != 2:
            raise ShapeError(f"matrix data must be 2-D, got {len(_shape(a))}-D")
        dt = a.dtype
        if dt not in (np.float32, torch.float32):
            raise ParameterError(f"matrix data must be float32, got {dt}")
        if not _all_finite(a):
            raise DataError("matrix contains non-finite values")

    @classmethod
    def from_array(cls, arr) -> "Matrix":
        if isinstance(arr, torch.Tensor):
            a = arr.to(torch.float32).contiguous()
            if a.dim() == 1:
                a = a.reshape(1, -1)
        else:
            a = np.ascontiguousarray(arr, dtype=np.float32)
            if a.ndim == 1:
                a = a.reshape(1, -1)
        return cls(a)

    @property
    def rows(self) -> int:
        return _shape(self.data)[0]

    @property
    def cols(self) -> int:
        return _shape(self.data)[1]

    def to_array(self):
        return self.data


@dataclass(frozen=True)
class QuantizedWeights:
    """Low-bit weights with per-group scales (core.py:86-127).

    Dequantized value: ``scale[m][k // gs] * (q - zero)`` with
    ``zero = zeros[m][k // gs]`` if ``zeros`` is given, else the reference's
    implicit ``2**(bits-1)``.
    """

    m: int
    k: int
    bits: int
    group_size: int
    qvalues: object   # uint8 (m, k)
    scales: object    # float32/float16 (m, k // group_size)
    zeros: object = None
    # weight encoding (batch executor, bitlut_b200.h BITLUT_W_*): "offset"
    # (zeros None: the reference's implicit zero), "zeros" (asymmetric),
    # "sign" (1-bit sign planes, built by sign_planes) or "ternary" (built by
    # ternary); None = derived from zeros.  sign/ternary keep the equivalent
    # (scale, zero) pair in scales/zeros, so every kernel can run them.
    encoding: object = None

    ENCODINGS = ("offset", "zeros", "sign", "ternary")

    def __post_init__(self):
        if not 1 <= self.bits <= 4:
            raise ParameterError(f"bits must be in [1, 4], got {self.bits}")
        if self.group_size < 1:
            raise ParameterError("group_size must be positive")
        if self.k % self.group_size != 0:
            raise LayoutError(f"k={self.k} not divisible by group_size={self.group_size}")
        if _shape(self.qvalues) != (self.m, self.k):
            raise ShapeError("qvalues shape mismatch")
        if _shape(self.scales) != (self.m, self.k // self.group_size):
            raise ShapeError("scales shape mismatch")
        if self.qvalues.dtype not in (np.uint8, torch.uint8):
            raise ParameterError("qvalues must be uint8")
        if _max(self.qvalues) >= (1 << self.bits):
            raise DataError(f"qvalues exceed {self.bits}-bit range")
        if self.scales.dtype not in (np.float32, np.float16, torch.float32, torch.float16):
            raise ParameterError("scales must be float32 or float16")
        if not _all_finite(self.scales):
            raise DataError("scales contain non-finite values")
        if self.zeros is not None:
            if _shape(self.zeros) != _shape(self.scales):
                raise ShapeError("zeros shape mismatch")
            if not _all_finite(self.zeros):
                raise DataError("zeros contain non-finite values")
        enc = self.encoding
        if enc is None:
            enc = "offset" if self.zeros is None else "zeros"
        if enc not in self.ENCODINGS:
            raise ParameterError(f"encoding must be one of {self.ENCODINGS}, got {enc!r}")
        if (enc == "offset") != (self.zeros is None):
            raise ParameterError(f"encoding {enc!r} {'takes no' if enc == 'offset' else 'needs'} zero points")
        if enc == "sign" and self.bits != 1:
            raise ParameterError("sign planes are 1-bit")
        if enc == "ternary" and self.bits != 2:
            raise ParameterError("ternary weights use 2 bit planes")
        object.__setattr__(self, "encoding", enc)

    @property
    def offset(self) -> int:
        return 1 << (self.bits - 1)

    @property
    def n_groups(self) -> int:
        return self.k // self.group_size

    @classmethod
    def sign_planes(cls, signs_q, scales, group_size):
        """1-bit sign planes: w = +s where q = 1, -s where q = 0
        (BASELINE config 3).  Stored as bits=1, scale 2s, zero 0.5 (the
        generic zero-point form); encoding "sign" lets the batch executor
        drop the zero points and the row-sum term (BITLUT_W_SIGN)."""
        s = as_tensor(scales)
        return cls(m=_shape(signs_q)[0], k=_shape(signs_q)[1], bits=1, group_size=group_size,
                   qvalues=signs_q, scales=(2 * s.float()).to(s.dtype),
                   zeros=torch.full(tuple(s.shape), 0.5, dtype=s.dtype), encoding="sign")

    @classmethod
    def ternary(cls, values, scale, group_size):
        """Ternary weights v in {-1, 0, +1} with ONE per-tensor scale:
        q = v + 1 in 2 bit planes, zero 1 (BASELINE config 3).  `scale` is
        a scalar (or an (m, k/gs) array of one value); encoding "ternary"
        lets the batch executor read that one value instead of a scale
        stream (BITLUT_W_TERNARY)."""
        v = as_tensor(values)
        q = (v.to(torch.int16) + 1).to(torch.uint8)
        m, k = q.shape
        s = as_tensor(scale)
        if s.dim() == 0 or s.numel() == 1:
            s = s.reshape(1, 1).expand(m, k // group_size).contiguous()
        flat = s.reshape(-1)
        if flat.numel() and not bool((flat == flat[0]).all()):
            raise DataError("ternary weights take one per-tensor scale")
        return cls(m=m, k=k, bits=2, group_size=group_size, qvalues=q,
                   scales=s, zeros=torch.ones(tuple(s.shape), dtype=s.dtype), encoding="ternary")


@dataclass(frozen=True)
class BitSerialParams:
    """core.py:130-167: constants of f(v) = s0 + (s1 - s0) v with s0=-1,
    s1=+1, alpha = beta = 1/2 (every bit v = f(v)/2 + 1/2)."""

    bits: int
    s0: float = -1.0
    s1: float = 1.0
    alpha: tuple = field(default=())
    beta: tuple = field(default=())
    combined_bias: float = 0.0

    def map_bit(self, v: int) -> float:
        return self.s0 + (self.s1 - self.s0) * v

    def reconstruct(self, value: int) -> float:
        acc = self.combined_bias
        for i in range(self.bits):
            acc += self.alpha[i] * (1 << i) * self.map_bit((value >> i) & 1)
        return acc


def bit_serial_params(bits: int) -> BitSerialParams:
    if not isinstance(bits, (int, np.integer)) or not 1 <= bits <= 4:
        raise ParameterError(f"bits must be an integer in [1, 4], got {bits!r}")
    bits = int(bits)
    half = tuple(0.5 for _ in range(bits))
    return BitSerialParams(bits=bits, alpha=half, beta=half,
                           combined_bias=sum(0.5 * (1 << i) for i in range(bits)))


@dataclass(frozen=True)
class TileConfig:
    """core.py:170-213: tiling of the reference's v1 packed layout.  The
    CUDA kernels use their own layout (layout v2); TileConfig
    still defines PackedWeights.planes so v1 round trips are exact."""

    n_tile: int = 1
    m_tile: int = 32
    k_tile: int = 128
    g: int = 4
    lanes: int = DEFAULT_LANES

    def __post_init__(self):
        if not 1 <= self.g <= 8:
            raise ParameterError(f"g must be in [1, 8], got {self.g}")
        if self.n_tile < 1:
            raise ParameterError("n_tile must be >= 1")
        if self.lanes < 1:
            raise ParameterError("lanes must be >= 1")
        if self.k_tile % self.g != 0:
            raise LayoutError(f"k_tile={self.k_tile} not divisible by g={self.g}")
        if self.m_tile % self.lanes != 0:
            raise LayoutError(f"m_tile={self.m_tile} not divisible by lanes={self.lanes}")
        ipb = indices_per_byte(self.g)
        if (self.k_tile // self.g) % ipb != 0:
            raise LayoutError(f"k_tile/g={self.k_tile // self.g} not divisible by the "
                              f"packing density {ipb} for g={self.g}")

    @property
    def k_groups_per_tile(self) -> int:
        return self.k_tile // self.g

    def lut_working_set_entries(self, n_rows: int | None = None) -> int:
        n = self.n_tile if n_rows is None else n_rows
        return n * self.k_groups_per_tile * (1 << (self.g - 1))


DEFAULT_TILE = TileConfig()
