"""Seeded synthetic workloads for BASELINE.json configs.

Part of the package (not the oracle) so bench.py can draw inputs without
touching oracle/.  Shared by oracle/make_golden.py (which runs the real reference on them),
the tests and bench.py.  Inputs are drawn with numpy's PCG64
``default_rng(seed)`` in the fixed order q -> scales -> zeros -> a, as
SURVEY.md §8(d) specifies; the reference uses the same generator family
(cli.py:142).  No dataset is involved: BASELINE names none.
"""
from __future__ import annotations

import numpy as np

LLAMA2_7B_SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]   # (M out, K in)
LLAMA2_70B_SHAPES = [(8192, 8192), (28672, 8192), (8192, 28672), (1024, 8192)]
# one decode layer of Llama-2-7B: q, k, v, o (4096x4096), gate, up (11008x4096),
# down (4096x11008)
LLAMA2_7B_LAYER = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)]


def _scales(rng, m, nq):
    return (np.abs(rng.normal(0.0, 0.02, (m, nq))) + 1e-3).astype(np.float16)


def config1(seed=1, m=4096, k=4096):
    """C1: single mpGEMV, W4 asymmetric (fp16 zeros), gs=128, fp16 tables."""
    rng = np.random.default_rng(seed)
    gs = 128
    q = rng.integers(0, 16, (m, k), dtype=np.uint8)
    s = _scales(rng, m, k // gs)
    z = rng.uniform(0, 15, (m, k // gs)).astype(np.float16)
    a = rng.standard_normal((1, k)).astype(np.float16)
    return dict(name=f"c1_{m}x{k}_w4_g128_asym", q=q, scales=s, zeros=z, a=a,
                bits=4, group_size=gs)


def config2(shape_index=0, n=1):
    """C2: Llama-2-7B decode shapes, W2 in [0,4), gs=64, implicit zero 2,
    int8 tables (bit-exact)."""
    m, k = LLAMA2_7B_SHAPES[shape_index]
    rng = np.random.default_rng(2 * 100 + shape_index)
    gs = 64
    q = rng.integers(0, 4, (m, k), dtype=np.uint8)
    s = _scales(rng, m, k // gs)
    a = rng.standard_normal((n, k)).astype(np.float16)
    return dict(name=f"c2_{m}x{k}_w2_g64", q=q, scales=s, zeros=None, a=a,
                bits=2, group_size=gs)


def config3(shape_index=0, kind="sign"):
    """C3: 1-bit sign planes (w = +-s, per-group fp16 scale, gs=128) or
    ternary {-1,0,+1} (p=1/3 each, 2 planes, per-tensor fp16 scale).

    Both map onto the generalized zero: sign -> bits=1, scale 2s, zero 0.5;
    ternary -> bits=2, q = v+1, zero 1.
    """
    m, k = LLAMA2_7B_SHAPES[shape_index]
    rng = np.random.default_rng(3 * 100 + shape_index + (50 if kind == "ternary" else 0))
    gs = 128
    nq = k // gs
    if kind == "sign":
        q = rng.integers(0, 2, (m, k), dtype=np.uint8)
        s = _scales(rng, m, nq)
        scales = (2.0 * s.astype(np.float32)).astype(np.float16)   # exact (x2)
        zeros = np.full((m, nq), 0.5, dtype=np.float16)
        bits = 1
    else:
        v = rng.choice(np.array([-1, 0, 1], dtype=np.int8), size=(m, k), p=[1 / 3] * 3)
        q = (v + 1).astype(np.uint8)
        s = np.float16(abs(rng.normal(0.0, 0.02)) + 1e-3)
        scales = np.full((m, nq), s, dtype=np.float16)
        zeros = np.full((m, nq), 1.0, dtype=np.float16)
        bits = 2
    a = rng.standard_normal((1, k)).astype(np.float16)
    return dict(name=f"c3_{m}x{k}_{kind}", q=q, scales=scales, zeros=zeros, a=a,
                bits=bits, group_size=gs)


def config4(n_tokens=32, bits=4, shape_index=0):
    """C4: prefill mpGEMM, N tokens, W4/W2, gs=128, implicit zero."""
    m, k = LLAMA2_7B_SHAPES[shape_index]
    rng = np.random.default_rng(4 * 1000 + n_tokens + 10 * bits + shape_index)
    gs = 128
    q = rng.integers(0, 1 << bits, (m, k), dtype=np.uint8)
    s = _scales(rng, m, k // gs)
    a = rng.standard_normal((n_tokens, k)).astype(np.float16)
    return dict(name=f"c4_{m}x{k}_w{bits}_n{n_tokens}", q=q, scales=s, zeros=None,
                a=a, bits=bits, group_size=gs)


def config5(shape_index=0, bits=2, n=1):
    """C5: Llama-2-70B decode shapes, W2/W4, gs=128, batch 1 or 8."""
    m, k = LLAMA2_70B_SHAPES[shape_index]
    rng = np.random.default_rng(5 * 1000 + 10 * shape_index + bits + 100 * n)
    gs = 128
    q = rng.integers(0, 1 << bits, (m, k), dtype=np.uint8)
    s = _scales(rng, m, k // gs)
    a = rng.standard_normal((n, k)).astype(np.float16)
    return dict(name=f"c5_{m}x{k}_w{bits}_n{n}", q=q, scales=s, zeros=None, a=a,
                bits=bits, group_size=gs)


def small_instance(seed, m, k, bits, group_size, n=1, zeros=False, dtype=np.float16):
    """Small random instance (tests): q uniform, fp16-valued scales/acts."""
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 1 << bits, (m, k), dtype=np.uint8)
    s = _scales(rng, m, k // group_size)
    z = (rng.uniform(0, (1 << bits) - 1, (m, k // group_size)).astype(np.float16)
         if zeros else None)
    a = rng.standard_normal((n, k)).astype(dtype)
    return dict(name=f"small_{m}x{k}_w{bits}_g{group_size}_n{n}", q=q, scales=s,
                zeros=z, a=a, bits=bits, group_size=group_size)
