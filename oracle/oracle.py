"""CPU oracle for the LUT mpGEMV/mpGEMM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference package
``bitlut`` (arXiv 2407.00088 reimplementation under /root/reference/pkg)
for the functions on the north-star path.  It exists so that tests,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg can check
the CUDA product path against the reference algorithm.  Nothing in the
product package (``paper_2407_00088_b200``) imports it; the product path
has no CPU fallback.

Every function cites the reference file:line it restates (paths relative
to /root/reference/pkg/src/bitlut/).  The restatement is pinned against
vectors produced by running the real reference (``oracle/make_golden.py``
-> ``tests/golden/``); see tests/test_oracle_pins.py.

All floating-point work is float32 with the reference's exact operation
order (numpy float32 elementwise arithmetic is IEEE round-to-nearest with
no fused multiply-add, matching the reference's numba loops, which were
verified to compile to separate mulss/addss).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


# --------------------------------------------------------------------------
# Offline weight pipeline (weight_prep.py)
# --------------------------------------------------------------------------

def slot_bits(g: int) -> int:
    """core.py:18-37 -- power-of-two slot width of one packed index."""
    if g == 1:
        return 1
    if g == 2:
        return 2
    if g <= 4:
        return 4
    return 8


def indices_per_byte(g: int) -> int:
    return 8 // slot_bits(g)


def decompose_bits(q: np.ndarray, bits: int, g: int) -> np.ndarray:
    """weight_prep.py:86-105.

    Plane i, entry (m, kg) = sum_j bit_i(q[m, kg*g + j]) << j.
    Returns uint8 array of shape (bits, M, K/g).
    """
    q = np.asarray(q, dtype=np.uint8)
    m, k = q.shape
    kg = k // g
    grouped = q.reshape(m, kg, g).astype(np.uint32)
    out = np.zeros((bits, m, kg), dtype=np.uint8)
    for i in range(bits):
        plane = np.zeros((m, kg), dtype=np.uint32)
        for j in range(g):
            plane |= ((grouped[:, :, j] >> i) & 1) << j
        out[i] = plane.astype(np.uint8)
    return out


def permute_plane_v1(indices: np.ndarray, m_tile: int, k_tile: int,
                     g: int, lanes: int) -> np.ndarray:
    """weight_prep.py:193-201 and docs/formats.md:60-71.

    Flatten (M, K/g) indices in the order (mb, kb, lb, kg-in-tile, lane).
    """
    m, kg_total = indices.shape
    ktg = k_tile // g
    out = np.empty(m * kg_total, dtype=np.uint8)
    pos = 0
    for mb in range(m // m_tile):
        for kb in range(kg_total // ktg):
            for lb in range(m_tile // lanes):
                rows = slice(mb * m_tile + lb * lanes, mb * m_tile + (lb + 1) * lanes)
                blk = indices[rows, kb * ktg:(kb + 1) * ktg]  # (lanes, ktg)
                flat = np.ascontiguousarray(blk.T).reshape(-1)  # kg-major, lane-minor
                out[pos:pos + flat.size] = flat
                pos += flat.size
    return out


def interleave_v1(stream: np.ndarray, g: int, lanes: int) -> np.ndarray:
    """weight_prep.py:131-156 and docs/formats.md:73-90.

    Units of per*lanes indices; recursive low/high split with the slot
    width doubling each level (for g=4: byte j = U[j] | U[j+lanes] << 4).
    """
    per = indices_per_byte(g)
    if per == 1:
        return stream.astype(np.uint8).copy()
    units = stream.astype(np.uint16).reshape(-1, per * lanes)
    width = slot_bits(g)
    while units.shape[1] > lanes:
        h = units.shape[1] // 2
        units = units[:, :h] | (units[:, h:] << width)
        width *= 2
    return units.astype(np.uint8).reshape(-1)


def deinterleave_v1(packed: np.ndarray, g: int, lanes: int) -> np.ndarray:
    """weight_prep.py:159-176 (inverse of interleave_v1)."""
    per = indices_per_byte(g)
    if per == 1:
        return packed.astype(np.uint8).copy()
    cur = packed.astype(np.uint8).reshape(-1, lanes)
    width = 4
    sb = slot_bits(g)
    while True:
        mask = np.uint8((1 << width) - 1)
        cur = np.concatenate([cur & mask, cur >> np.uint8(width)], axis=1)
        if width == sb:
            break
        width //= 2
    return cur.reshape(-1)


def unpermute_plane_v1(stream: np.ndarray, m: int, kg_total: int, m_tile: int,
                       k_tile: int, g: int, lanes: int) -> np.ndarray:
    """weight_prep.py:204-211."""
    ktg = k_tile // g
    out = np.empty((m, kg_total), dtype=np.uint8)
    pos = 0
    for mb in range(m // m_tile):
        for kb in range(kg_total // ktg):
            for lb in range(m_tile // lanes):
                n = lanes * ktg
                blk = stream[pos:pos + n].reshape(ktg, lanes).T
                out[mb * m_tile + lb * lanes:mb * m_tile + (lb + 1) * lanes,
                    kb * ktg:(kb + 1) * ktg] = blk
                pos += n
    return out


def pack_v1(indices: np.ndarray, m_tile: int, k_tile: int, g: int,
            lanes: int) -> np.ndarray:
    """weight_prep.py:214-246 (pack_and_permute): (bits, M, KG) -> (bits, plane_bytes)."""
    return np.stack([interleave_v1(permute_plane_v1(p, m_tile, k_tile, g, lanes), g, lanes)
                     for p in indices])


def unpack_v1(planes: np.ndarray, m: int, k: int, m_tile: int, k_tile: int,
              g: int, lanes: int) -> np.ndarray:
    """weight_prep.py:249-257 (unpack_planes)."""
    kg_total = k // g
    return np.stack([unpermute_plane_v1(deinterleave_v1(p, g, lanes), m, kg_total,
                                        m_tile, k_tile, g, lanes) for p in planes])


# --------------------------------------------------------------------------
# Online activation tables (lut_build.py)
# --------------------------------------------------------------------------

def precompute_lut(a: np.ndarray, g: int) -> np.ndarray:
    """lut_build.py:105-127.

    Entry (n, kg, idx) = signed sum of a[n, kg*g + j] (+ when bit j of idx is
    set), summed in ascending j in float32: ((+-a0 +- a1) +- a2) +- a3.
    Returns (N, K/g, 2**g) float32.
    """
    a = np.ascontiguousarray(a, dtype=F32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    n, k = a.shape
    ag = a.reshape(n, k // g, g)
    idx = np.arange(1 << g)
    bit0 = ((idx & 1) != 0)[None, None, :]
    e = np.where(bit0, ag[:, :, 0:1], -ag[:, :, 0:1]).astype(F32)
    for j in range(1, g):
        bj = (((idx >> j) & 1) != 0)[None, None, :]
        aj = ag[:, :, j:j + 1]
        e = np.where(bj, e + aj, e - aj).astype(F32)
    return e


def mirror_consolidate(full: np.ndarray) -> np.ndarray:
    """lut_build.py:130-143 -- keep indices with the top bit clear."""
    half = full.shape[2] // 2
    assert np.array_equal(full[:, :, half:], -full[:, :, half - 1::-1])
    return np.ascontiguousarray(full[:, :, :half])


def quantize_tables(half: np.ndarray, g: int, group_size: int):
    """lut_build.py:153-179.

    One scale per (row, quantization group): max|e| / 127 (1 for all-zero
    groups); q = clip(trunc(e/scale + copysign(0.5, e/scale)), -127, 127).
    Returns (qentries int8 (N, KG, 2**(g-1)), table_scales f32 (N, NQ)).
    """
    gpg = group_size // g
    n, kg, width = half.shape
    grouped = half.reshape(n, kg // gpg, gpg * width)
    scales = (np.abs(grouped).max(axis=2) / F32(127.0)).astype(F32)
    scales = np.where(scales == F32(0.0), F32(1.0), scales).astype(F32)
    per_kg = np.repeat(scales, gpg, axis=1)[:, :, None]
    scaled = (half / per_kg).astype(F32)
    q = np.trunc((scaled + np.copysign(F32(0.5), scaled)).astype(F32))
    q = np.clip(q, -127, 127).astype(np.int8)
    return q, scales


def row_sums(a: np.ndarray, group_size: int) -> np.ndarray:
    """lut_build.py:182-194 -- per-group sums accumulated left to right."""
    a = np.ascontiguousarray(a, dtype=F32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    n, k = a.shape
    ag = a.reshape(n, k // group_size, group_size)
    acc = np.zeros((n, k // group_size), dtype=F32)
    for j in range(group_size):
        acc = (acc + ag[:, :, j]).astype(F32)
    return acc


# --------------------------------------------------------------------------
# Lookup-accumulate (kernel.py / _kernels.py)
# --------------------------------------------------------------------------

def _mirror(indices: np.ndarray, g: int):
    """_kernels.py:154-177: s = idx >> (g-1); eff = idx ^ (mask * s)."""
    ii = indices.astype(np.int32)
    s = ii >> (g - 1)
    eff = ii ^ (((1 << g) - 1) * s)
    return s, eff


def stage_partials_q8(indices: np.ndarray, qtab: np.ndarray, g: int,
                      group_size: int) -> np.ndarray:
    """_kernels.py:141-186 (int32 staging) == kernel.py:190-223 (integer mode).

    P[i, n, m, gq] = sum over kg in group gq of +-qtab[n, kg, eff] -- the
    exact int32 value the reference stages per (plane, channel, group)
    before the float epilogue.  Returns int32 (bits, N, M, NQ).
    """
    bits, m, kgt = indices.shape
    n = qtab.shape[0]
    gpg = group_size // g
    nq = kgt // gpg
    out = np.zeros((bits, n, m, nq), dtype=np.int32)
    kg_idx = np.arange(kgt)[None, :]
    for i in range(bits):
        s, eff = _mirror(indices[i], g)
        sign = 1 - 2 * s
        for r in range(n):
            vals = qtab[r][kg_idx, eff].astype(np.int32) * sign
            out[i, r] = vals.reshape(m, nq, gpg).sum(axis=2, dtype=np.int32)
    return out


def epilogue_q8(P: np.ndarray, tscales: np.ndarray, wscales: np.ndarray,
                rsums: np.ndarray) -> np.ndarray:
    """_kernels.py:179-191 float epilogue, in the reference's order.

    out[m] += ((pf_i * ts[gq]) * ws[m, gq]) * f32(P) for i ascending, gq
    ascending; then out[m] -= 0.5 * sum_gq(ws[m, gq] * rs[gq]).
    """
    bits, n, m, nq = P.shape
    ws = np.asarray(wscales, dtype=F32)
    y = np.zeros((n, m), dtype=F32)
    for r in range(n):
        out = np.zeros(m, dtype=F32)
        for i in range(bits):
            pf = F32(0.5 * (1 << i))
            for gq in range(nq):
                f = F32(pf * tscales[r, gq])
                out = (out + (f * ws[:, gq]).astype(F32) * P[i, r, :, gq].astype(F32)).astype(F32)
        out = (out - F32(0.5) * bias_sum(ws, rsums[r])).astype(F32)
        y[r] = out
    return y


def bias_sum(ws: np.ndarray, rs_row: np.ndarray) -> np.ndarray:
    """_kernels.py:187-190: s = sum_gq ws[m, gq] * rs[gq], left to right."""
    s = np.zeros(ws.shape[0], dtype=F32)
    for gq in range(ws.shape[1]):
        s = (s + (ws[:, gq] * rs_row[gq]).astype(F32)).astype(F32)
    return s


def gemv_real(indices: np.ndarray, half_tables: np.ndarray, wscales: np.ndarray,
              rsums: np.ndarray, g: int, group_size: int) -> np.ndarray:
    """_kernels.py:85-138 (scalar-real): float32 stage summed in ascending kg
    within each group, out[m] += (pf * ws[m, gq]) * stage, then the bias."""
    bits, m, kgt = indices.shape
    n = half_tables.shape[0]
    gpg = group_size // g
    nq = kgt // gpg
    ws = np.asarray(wscales, dtype=F32)
    y = np.zeros((n, m), dtype=F32)
    for r in range(n):
        out = np.zeros(m, dtype=F32)
        for i in range(bits):
            s, eff = _mirror(indices[i], g)
            looked = half_tables[r][np.arange(kgt)[None, :], eff]
            looked = np.where(s == 1, -looked, looked).astype(F32)
            pf = F32(0.5 * (1 << i))
            for gq in range(nq):
                stage = np.zeros(m, dtype=F32)
                for j in range(gpg):
                    stage = (stage + looked[:, gq * gpg + j]).astype(F32)
                out = (out + (pf * ws[:, gq]).astype(F32) * stage).astype(F32)
        out = (out - F32(0.5) * bias_sum(ws, rsums[r])).astype(F32)
        y[r] = out
    return y


# --------------------------------------------------------------------------
# Generalized zero point (BASELINE extension; not in the reference)
# --------------------------------------------------------------------------

def zero_correction(wscales: np.ndarray, zeros: np.ndarray, bits: int,
                    rsums_row: np.ndarray) -> np.ndarray:
    """Correction turning the reference's implicit zero 2**(b-1) into z.

    w = s * (q - z) = s * (q - 2**(b-1)) + s * (2**(b-1) - z), so
    y = reference(q, s) + sum_gq (s * d) * R with d = 2**(b-1) - z.
    Order (defined by this package, mirrored by the CUDA epilogue):
    d = f32(2**(b-1)) - z; c = 0; c += (ws*d)*rs per gq ascending; y += c.
    Validated against the reference's dequantize-then-GEMM oracle
    (oracle.py:26-42) in tests/test_oracle_pins.py.
    """
    ws = np.asarray(wscales, dtype=F32)
    d = (F32(1 << (bits - 1)) - np.asarray(zeros, dtype=F32)).astype(F32)
    c = np.zeros(ws.shape[0], dtype=F32)
    for gq in range(ws.shape[1]):
        c = (c + ((ws[:, gq] * d[:, gq]).astype(F32) * rsums_row[gq]).astype(F32)).astype(F32)
    return c


def mpgemm_q8(a: np.ndarray, q: np.ndarray, wscales: np.ndarray, bits: int,
              group_size: int, zeros=None, g: int = 4, return_partials=False):
    """Full int8-table path: tables -> int32 partials -> float epilogue.

    Equals the reference ``mpgemm(..., variant="vector-q8")`` bit for bit
    when ``zeros`` is None (kernel.py:280-371 with _kernels.py:141-192).
    """
    a = np.ascontiguousarray(a, dtype=F32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    idx = decompose_bits(q, bits, g)
    half = mirror_consolidate(precompute_lut(a, g))
    qtab, ts = quantize_tables(half, g, group_size)
    rs = row_sums(a, group_size)
    P = stage_partials_q8(idx, qtab, g, group_size)
    y = epilogue_q8(P, ts, wscales, rs)
    if zeros is not None:
        for r in range(a.shape[0]):
            y[r] = (y[r] + zero_correction(wscales, zeros, bits, rs[r])).astype(F32)
    if return_partials:
        return y, P
    return y


def mpgemm_real(a: np.ndarray, q: np.ndarray, wscales: np.ndarray, bits: int,
                group_size: int, zeros=None, g: int = 4):
    """Full fp32-table path == reference ``variant="scalar-real"`` bit for bit
    when ``zeros`` is None."""
    a = np.ascontiguousarray(a, dtype=F32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    idx = decompose_bits(q, bits, g)
    half = mirror_consolidate(precompute_lut(a, g))
    rs = row_sums(a, group_size)
    y = gemv_real(idx, half, wscales, rs, g, group_size)
    if zeros is not None:
        for r in range(a.shape[0]):
            y[r] = (y[r] + zero_correction(wscales, zeros, bits, rs[r])).astype(F32)
    return y


def dequant_gemm(a: np.ndarray, q: np.ndarray, wscales: np.ndarray, bits: int,
                 group_size: int, zeros=None) -> np.ndarray:
    """core.py:265-273 + oracle.py:26-42 semantics (float64 here: used only
    as an accuracy yardstick, never for bitwise checks)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    m, k = q.shape
    z = (np.full((m, k // group_size), float(1 << (bits - 1)))
         if zeros is None else np.asarray(zeros, dtype=np.float64))
    w = (q.reshape(m, k // group_size, group_size).astype(np.float64) - z[:, :, None]) \
        * np.asarray(wscales, dtype=np.float64)[:, :, None]
    return a @ w.reshape(m, k).T


# --------------------------------------------------------------------------
# C restatement (oracle/bitlut_oracle.c): same arithmetic, fast enough to be
# the timed CPU baseline.  Built by `make -C oracle` (build() runs it).
# --------------------------------------------------------------------------

_CLIB = None


def c_lib():
    import ctypes
    import os
    import subprocess
    global _CLIB
    if _CLIB is None:
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "_build", "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", here], check=True)
        _CLIB = ctypes.CDLL(path)
        _CLIB.orc_mpgemm.restype = ctypes.c_int
        _CLIB.orc_max_threads.restype = ctypes.c_int
    return _CLIB


def c_mpgemm(a, planes_v1, m, k, bits, group_size, wscales, mode="vector-q8",
             threads=0, m_tile=32, k_tile=128, lanes=16):
    """Reference mpgemm (kernel.py:280-371) via the C port, v1 planes in."""
    import ctypes
    P = ctypes.c_void_p
    a = np.ascontiguousarray(a, dtype=F32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    planes = np.ascontiguousarray(planes_v1, dtype=np.uint8)
    ws = np.ascontiguousarray(wscales, dtype=F32)
    out = np.empty((a.shape[0], m), dtype=F32)
    c_lib().orc_mpgemm(a.ctypes.data_as(P), a.shape[0], planes.ctypes.data_as(P), m, k, bits,
                       group_size, m_tile, k_tile, lanes, ws.ctypes.data_as(P),
                       0 if mode == "vector-q8" else 1, int(threads), out.ctypes.data_as(P))
    return out


def c_quantize_weights(w: np.ndarray, bits: int, group_size: int, refine: bool = True, threads: int = 0):
    """core.py:227-262 quantize_weights via the C port of _kernels.py:20-82:
    -> (q (M, K) uint8, scales (M, K/gs) float32)."""
    import ctypes
    P = ctypes.c_void_p
    w = np.ascontiguousarray(w, dtype=F32)
    m, k = w.shape
    ng = m * k // group_size
    q = np.empty((m, k), dtype=np.uint8)
    d = np.empty((m, k // group_size), dtype=F32)
    fn = c_lib().orc_quantize_groups
    fn.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int]
    fn(w.ctypes.data_as(P), ng, group_size, 1 << (bits - 1), 9 if refine else 0, q.ctypes.data_as(P),
       d.ctypes.data_as(P), int(threads))
    return q, d


def c_max_threads() -> int:
    return int(c_lib().orc_max_threads())
