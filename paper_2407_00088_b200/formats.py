"""Binary containers (reference pkg/docs/formats.md; pkg/src/bitlut/fileio.py,
weight_prep.py:266-350): LMRM raw matrices, LMQW quantized weights, LMPW
packed weights.

* LMRM / LMQW and LMPW **format version 1** are the reference's containers,
  byte for byte (a file written here loads in the reference and vice
  versa), with the same validation order and error classes.
* LMPW **format version 2** (this package) stores the GPU operand instead:
  header + layout-v2 payload (csrc/layout.cuh) + scales in their dtype
  (fp16 or fp32) + optional zero points, so a deployment loads kernel-ready
  bytes without the v1 -> v2 repack.  Same error rules as version 1.

All integers little-endian; arrays row-major, no padding.
"""
from __future__ import annotations

import struct
from pathlib import Path
from typing import Union

import numpy as np
import torch

from . import _native as N
from .core import Matrix, QuantizedWeights, TileConfig, indices_per_byte
from .errors import (BadMagicError, FormatVersionError, LayoutError, PayloadLengthError,
                     TruncatedStreamError)
from .weight_prep import (LAYOUT_VERSION, BitPlane, PackedWeights, from_v1, pack_and_permute,
                          unpack_planes, unrepack_gpu)

RAW_MAGIC, QUANT_MAGIC, PACKED_MAGIC = b"LMRM", b"LMQW", b"LMPW"
RAW_VERSION = QUANT_VERSION = 1
PACKED_V1, PACKED_V2 = 1, 2
GPU_LAYOUT_VERSION = 2

_RAW = struct.Struct("<4sIII")
_QUANT = struct.Struct("<4sIIIII")
_PACKED_V1 = struct.Struct("<4sIIIIIIIIIIIIII")     # magic + 14 u32 (formats.md "Container")
# v2: magic, format 2, layout 2, m, k, bits, group_size, scale dtype (0 f32 / 1 f16),
#     has_zeros, scale_count, gpu_bytes, then the v1 tile (n_tile, m_tile, k_tile, lanes)
_PACKED_V2 = struct.Struct("<4sIIIIIIIIIIIIII")

PathLike = Union[str, Path]


def _check_magic(data: bytes, magic: bytes, header: struct.Struct, what: str) -> None:
    if len(data) < 4 or data[:4] != magic:
        raise BadMagicError(f"not an {what} stream (magic {data[:4]!r})")
    if len(data) < header.size:
        raise TruncatedStreamError(f"{what} stream ends inside the header ({len(data)} bytes)")


def _check_total(data: bytes, expected: int, what: str) -> None:
    if len(data) < expected:
        raise TruncatedStreamError(f"{what} stream has {len(data)} bytes, header declares {expected}")
    if len(data) > expected:
        raise PayloadLengthError(f"{what} stream has {len(data)} bytes, header declares {expected}")


def _np(t) -> np.ndarray:
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


# ---------------------------------------------------------------- LMRM

def write_matrix(path: PathLike, matrix) -> None:
    arr = np.ascontiguousarray(_np(matrix.to_array() if isinstance(matrix, Matrix) else matrix),
                               dtype="<f4")
    Path(path).write_bytes(_RAW.pack(RAW_MAGIC, RAW_VERSION, arr.shape[0], arr.shape[1]) + arr.tobytes())


def read_matrix(path: PathLike) -> Matrix:
    data = Path(path).read_bytes()
    _check_magic(data, RAW_MAGIC, _RAW, "LMRM")
    _, version, rows, cols = _RAW.unpack_from(data)
    if version != RAW_VERSION:
        raise FormatVersionError(f"unsupported LMRM version {version} (expected {RAW_VERSION})")
    _check_total(data, _RAW.size + 4 * rows * cols, "LMRM")
    arr = np.frombuffer(data, dtype="<f4", count=rows * cols, offset=_RAW.size)
    return Matrix(np.ascontiguousarray(arr.reshape(rows, cols), dtype=np.float32))


# ---------------------------------------------------------------- LMQW

def write_quantized(path: PathLike, qw: QuantizedWeights) -> None:
    if qw.zeros is not None:
        raise LayoutError("LMQW (format 1) has no zero points; use LMPW format 2")
    out = bytearray(_QUANT.pack(QUANT_MAGIC, QUANT_VERSION, qw.m, qw.k, qw.bits, qw.group_size))
    out += np.ascontiguousarray(_np(qw.qvalues), dtype=np.uint8).tobytes()
    out += np.ascontiguousarray(_np(qw.scales).astype(np.float32), dtype="<f4").tobytes()
    Path(path).write_bytes(bytes(out))


def read_quantized(path: PathLike) -> QuantizedWeights:
    data = Path(path).read_bytes()
    _check_magic(data, QUANT_MAGIC, _QUANT, "LMQW")
    _, version, m, k, bits, group_size = _QUANT.unpack_from(data)
    if version != QUANT_VERSION:
        raise FormatVersionError(f"unsupported LMQW version {version} (expected {QUANT_VERSION})")
    if group_size < 1 or k % group_size != 0:
        raise PayloadLengthError("LMQW header dimensions are inconsistent")
    nq = k // group_size
    _check_total(data, _QUANT.size + m * k + 4 * m * nq, "LMQW")
    q = np.frombuffer(data, dtype=np.uint8, count=m * k, offset=_QUANT.size).reshape(m, k)
    s = np.frombuffer(data, dtype="<f4", count=m * nq, offset=_QUANT.size + m * k).reshape(m, nq)
    return QuantizedWeights(m=m, k=k, bits=bits, group_size=group_size,
                            qvalues=q.copy(), scales=s.astype(np.float32))


# ---------------------------------------------------------------- LMPW

def serialize(pw: PackedWeights, format_version: int = PACKED_V1) -> bytes:
    """Packed weights -> LMPW bytes.  Version 1 = the reference's stream
    (weight_prep.py:266-277: v1 planes + f32 scales); version 2 = the GPU
    layout-v2 operand + scales in their dtype + zero points."""
    if format_version == PACKED_V1:
        if pw.zeros is not None:
            raise LayoutError("LMPW format 1 has no zero points; use format_version=2")
        scales = np.ascontiguousarray(_np(pw.scales).astype(np.float32), dtype="<f4")
        planes = np.ascontiguousarray(_np(pw.planes), dtype=np.uint8)
        header = _PACKED_V1.pack(PACKED_MAGIC, PACKED_V1, pw.layout_version, pw.m, pw.k, pw.bits, pw.g,
                                 pw.group_size, pw.tile.n_tile, pw.tile.m_tile, pw.tile.k_tile,
                                 pw.tile.lanes, scales.size, pw.plane_bytes, pw.bits * pw.plane_bytes)
        return header + scales.tobytes() + planes.tobytes()
    if format_version == PACKED_V2:
        if pw.gpu is None:
            raise LayoutError("packed weights carry no GPU layout (prepare them with prepare_weights)")
        f16 = pw.scales.dtype == torch.float16
        sdt = "<f2" if f16 else "<f4"
        scales = np.ascontiguousarray(_np(pw.scales), dtype=sdt)
        gpu = np.ascontiguousarray(_np(pw.gpu), dtype=np.uint8)
        header = _PACKED_V2.pack(PACKED_MAGIC, PACKED_V2, GPU_LAYOUT_VERSION, pw.m, pw.k, pw.bits,
                                 pw.group_size, 1 if f16 else 0, 1 if pw.zeros is not None else 0,
                                 scales.size, gpu.size, pw.tile.n_tile, pw.tile.m_tile, pw.tile.k_tile,
                                 pw.tile.lanes)
        out = header + scales.tobytes()
        if pw.zeros is not None:
            out += np.ascontiguousarray(_np(pw.zeros), dtype=sdt).tobytes()
        return out + gpu.tobytes()
    raise FormatVersionError(f"unsupported format version {format_version}")


def _validate_index_range(planes: np.ndarray, g: int) -> None:
    """Indices must fit g bits (only slot widths wider than g can encode
    invalid values: g = 3 nibbles, g in [5, 7] bytes; weight_prep.py:280-293)."""
    if g == 3:
        if (planes & 0x88).any():
            raise PayloadLengthError("payload contains indices >= 8 for g=3")
    elif 5 <= g <= 7:
        if planes.max(initial=0) >= (1 << g):
            raise PayloadLengthError(f"payload contains indices out of range for g={g}")


def deserialize(data: bytes, device=None, gpu: bool = True) -> PackedWeights:
    """LMPW bytes -> PackedWeights on `device` (default: the current CUDA
    device).  Version 1 streams are validated like the reference
    (weight_prep.py:296-350) and, with gpu=True and g = 4, also repacked to
    layout v2; version 2 streams come back with both layouts."""
    if len(data) < 4 or data[:4] != PACKED_MAGIC:
        raise BadMagicError(f"not an LMPW stream (magic {data[:4]!r})")
    if len(data) < 8:
        raise TruncatedStreamError(f"stream ends inside the header ({len(data)} bytes)")
    version = struct.unpack_from("<I", data, 4)[0]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if version == PACKED_V1:
        if len(data) < _PACKED_V1.size:
            raise TruncatedStreamError(f"stream ends inside the header ({len(data)} bytes)")
        (_, _, layout, m, k, bits, g, gs, n_tile, m_tile, k_tile, lanes, scale_count, plane_bytes,
         payload_bytes) = _PACKED_V1.unpack_from(data)
        if layout != LAYOUT_VERSION:
            raise FormatVersionError(f"unsupported layout version {layout} (expected {LAYOUT_VERSION})")
        if g < 1 or g > 8 or bits < 1 or bits > 4 or gs < 1:
            raise PayloadLengthError("header fields out of range")
        if k % g != 0 or k % gs != 0:
            raise PayloadLengthError("header dimensions are inconsistent")
        if scale_count != m * (k // gs):
            raise PayloadLengthError(f"scale count {scale_count} disagrees with m={m}, k={k}, group_size={gs}")
        expected_plane = m * (k // g) // indices_per_byte(g)
        if plane_bytes != expected_plane:
            raise PayloadLengthError(f"plane size {plane_bytes} disagrees with header dimensions "
                                     f"(expected {expected_plane})")
        if payload_bytes != bits * plane_bytes:
            raise PayloadLengthError(f"declared payload {payload_bytes} disagrees with bits={bits} x "
                                     f"plane_bytes={plane_bytes}")
        _check_total(data, _PACKED_V1.size + 4 * scale_count + bits * plane_bytes, "LMPW")
        off = _PACKED_V1.size
        scales = np.frombuffer(data, dtype="<f4", count=scale_count, offset=off).reshape(m, k // gs)
        off += 4 * scale_count
        planes = np.frombuffer(data, dtype=np.uint8, count=bits * plane_bytes, offset=off)
        planes = np.ascontiguousarray(planes.reshape(bits, plane_bytes))
        _validate_index_range(planes, g)
        tile = TileConfig(n_tile=n_tile, m_tile=m_tile, k_tile=k_tile, g=g, lanes=lanes)
        pw = PackedWeights(m=m, k=k, bits=bits, g=g, group_size=gs, tile=tile,
                           planes=torch.from_numpy(planes.copy()).to(dev),
                           scales=torch.from_numpy(scales.astype(np.float32)).to(dev))
        if gpu and g == 4:
            try:
                pw = from_v1(pw)
            except LayoutError:
                pass                        # shape outside the CUDA path: v1 only
        return pw
    if version == PACKED_V2:
        if len(data) < _PACKED_V2.size:
            raise TruncatedStreamError(f"stream ends inside the header ({len(data)} bytes)")
        (_, _, layout, m, k, bits, gs, f16, has_z, scale_count, gpu_bytes, n_tile, m_tile, k_tile,
         lanes) = _PACKED_V2.unpack_from(data)
        if layout != GPU_LAYOUT_VERSION:
            raise FormatVersionError(f"unsupported GPU layout version {layout} (expected {GPU_LAYOUT_VERSION})")
        if bits < 1 or bits > 4 or gs < 1 or f16 > 1 or has_z > 1:
            raise PayloadLengthError("header fields out of range")
        if k % gs != 0 or scale_count != m * (k // gs):
            raise PayloadLengthError("header dimensions are inconsistent")
        lay = N.layout_query(m, k, bits, gs)
        if gpu_bytes != lay.bytes:
            raise PayloadLengthError(f"GPU payload {gpu_bytes} disagrees with the layout ({lay.bytes})")
        esz = 2 if f16 else 4
        _check_total(data, _PACKED_V2.size + esz * scale_count * (1 + has_z) + gpu_bytes, "LMPW")
        sdt = "<f2" if f16 else "<f4"
        off = _PACKED_V2.size
        scales = np.frombuffer(data, dtype=sdt, count=scale_count, offset=off).reshape(m, k // gs)
        off += esz * scale_count
        zeros = None
        if has_z:
            zeros = np.frombuffer(data, dtype=sdt, count=scale_count, offset=off).reshape(m, k // gs)
            off += esz * scale_count
        g_bytes = np.frombuffer(data, dtype=np.uint8, count=gpu_bytes, offset=off)
        tdt = torch.float16 if f16 else torch.float32
        gpu_t = torch.from_numpy(g_bytes.copy()).to(dev)
        s_t = torch.from_numpy(scales.astype(np.float16 if f16 else np.float32)).to(dev)
        z_t = torch.from_numpy(zeros.astype(np.float16 if f16 else np.float32)).to(dev) if has_z else None
        # v1 planes from the GPU layout (the drop-in operand): unrepack, then pack v1 on the GPU
        tile = TileConfig(n_tile=n_tile, m_tile=m_tile, k_tile=k_tile, g=4, lanes=lanes)
        shell = PackedWeights(m=m, k=k, bits=bits, g=4, group_size=gs, tile=tile,
                              planes=torch.zeros((bits, m * (k // 4) // 2), dtype=torch.uint8, device=dev),
                              scales=s_t, zeros=z_t, gpu=gpu_t)
        idx = unrepack_gpu(shell)
        planes = [BitPlane(bit=i, g=4, indices=idx[i].contiguous()) for i in range(bits)]
        pw = pack_and_permute(planes, tile, s_t.to(tdt), gs, zeros=z_t)
        if not torch.equal(pw.gpu, gpu_t):
            raise PayloadLengthError("GPU payload is not a canonical layout-v2 stream")
        return pw
    raise FormatVersionError(f"unsupported format version {version} (expected 1 or 2)")


def write_packed(path: PathLike, pw: PackedWeights, format_version: int = PACKED_V1) -> None:
    Path(path).write_bytes(serialize(pw, format_version))


def read_packed(path: PathLike, device=None, gpu: bool = True) -> PackedWeights:
    return deserialize(Path(path).read_bytes(), device=device, gpu=gpu)


def verify_round_trip(pw: PackedWeights, data: bytes) -> bool:
    """The stream decodes to the same plane indices (cli.py:100-108)."""
    back = deserialize(data)
    a, b = unpack_planes(pw), unpack_planes(back)
    return all(torch.equal(x.indices, y.indices) for x, y in zip(a, b))
