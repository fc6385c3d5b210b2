"""Golden vectors for the auxiliary public names (TEST INFRASTRUCTURE).

Runs the REAL reference (/root/reference/pkg/src, read-only) on seeded
inputs for pad_weights, interleave_layout, the byte/wide lookup primitives,
the rhadd aggregation helpers and reference_lut_mpgemv / reference_mpgemm,
and writes tests/golden/api_extras.npz, which tests/test_api_extras.py
checks paper_2407_00088_b200.api_extras against.

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden_extras.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, REF)

import bitlut  # noqa: E402  (the real reference)
from bitlut import kernel as RK  # noqa: E402
from bitlut import oracle as RO  # noqa: E402
from bitlut import weight_prep as RW  # noqa: E402


def main():
    rng = np.random.default_rng(2407)
    out = {}
    # interleave_layout over every g and two lane counts
    for g in range(1, 9):
        for lanes in (16, 32):
            per = bitlut.core.indices_per_byte(g)
            n = per * lanes * 3
            idx = rng.integers(0, 1 << g, n, dtype=np.uint8)
            out[f"il_in_g{g}_l{lanes}"] = idx
            out[f"il_out_g{g}_l{lanes}"] = RW.interleave_layout(idx, g, lanes)
    # pad_weights (the reference has no zero points)
    for tag, bits, gs, m, k, mm, km in (("a", 2, 8, 5, 24, 4, 16), ("b", 3, 4, 7, 12, 8, 6),
                                        ("c", 4, 16, 16, 32, 16, 16)):
        q = rng.integers(0, 1 << bits, (m, k), dtype=np.uint8)
        s = rng.uniform(0.5, 1.5, (m, k // gs)).astype(np.float32)
        qw = bitlut.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=s)
        p = RW.pad_weights(qw, mm, km)
        out[f"pad_{tag}_q"], out[f"pad_{tag}_s"] = q, s
        out[f"pad_{tag}_args"] = np.array([bits, gs, m, k, mm, km], np.int64)
        out[f"pad_{tag}_outq"] = np.asarray(p.qvalues)
        out[f"pad_{tag}_outs"] = np.asarray(p.scales)
    # lookups
    tab = rng.integers(-128, 128, 16).astype(np.int8)
    li = rng.integers(0, 16, 64, dtype=np.uint8)
    out["bpl_tab"], out["bpl_idx"], out["bpl_out"] = tab, li, RK.byte_parallel_lookup(tab, li)
    wt = rng.integers(-32768, 32768, 16).astype(np.int16)
    lo, hi = RK.split_wide_table(wt)
    out["wide_tab"], out["wide_lo"], out["wide_hi"] = wt, lo, hi
    out["wide_out"] = RK.wide_lookup(lo, hi, li)
    # aggregation
    for depth in range(0, 6):
        vals = rng.integers(-128, 128, 1 << depth)
        out[f"agg_in_d{depth}"] = vals
        out[f"agg_tree_d{depth}"] = np.array(RK.rhadd_tree(vals))
        out[f"agg_fast_d{depth}"] = np.array(RK.fast_aggregate(vals, depth))
        out[f"agg_bias_d{depth}"] = np.array(RK.bias_correction(depth))
        for bits in (1, 2, 4):
            out[f"agg_chain_d{depth}_b{bits}"] = np.array(RK.chain_bias_correction(depth, bits))
    # definitional references
    for tag, bits, g, gs, m, k in (("w2", 2, 4, 32, 16, 128), ("w3", 3, 2, 16, 8, 64), ("w4", 4, 4, 64, 32, 256)):
        q = rng.integers(0, 1 << bits, (m, k), dtype=np.uint8)
        s = rng.uniform(0.01, 0.1, (m, k // gs)).astype(np.float32)
        qw = bitlut.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=s)
        a = rng.standard_normal((3, k)).astype(np.float32)
        planes = bitlut.decompose_bits(qw, g)
        params = bitlut.bit_serial_params(bits)
        out[f"ref_{tag}_args"] = np.array([bits, g, gs, m, k], np.int64)
        out[f"ref_{tag}_q"], out[f"ref_{tag}_s"], out[f"ref_{tag}_a"] = q, s, a
        out[f"ref_{tag}_mpgemm"] = RO.reference_mpgemm(a, qw)
        out[f"ref_{tag}_lut"] = RO.reference_lut_mpgemv(a[0], planes, params, s)
    path = os.path.join(ROOT, "tests", "golden", "api_extras.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays")


if __name__ == "__main__":
    main()
