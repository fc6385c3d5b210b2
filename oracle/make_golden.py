"""Generate golden vectors by running the REAL reference (TEST INFRASTRUCTURE).

Runs the reference package ``bitlut`` in place from
/root/reference/pkg/src (read-only; numba JIT cache redirected to /tmp) on
seeded inputs and writes its outputs to tests/golden/.  The reference
cannot travel to the GPU box, so these committed fixtures are how the GPU
tests and the oracle restatement are pinned to it.

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden.py

Small instances store inputs and every intermediate; BASELINE-sized
instances store outputs only (inputs are regenerated from the seeds in
paper_2407_00088_b200/workloads.py), with sha256 digests plus sampled rows
where the full output would be too large to commit.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import bitlut  # noqa: E402  (the real reference)
from bitlut import (KernelVariant, QuantizedWeights, TileConfig, decompose_bits,  # noqa: E402
                    mirror_consolidate, mpgemm, precompute_lut, prepare_weights,
                    quantize_tables, row_sums)
from bitlut.kernel import Accumulators, lookup_accumulate_tile  # noqa: E402
from bitlut.oracle import reference_gemm  # noqa: E402

from paper_2407_00088_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
THREADS = os.cpu_count() or 1


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def ref_packed(inst, tile=None):
    q, s = inst["q"], inst["scales"].astype(np.float32)
    m, k = q.shape
    qw = QuantizedWeights(m=m, k=k, bits=inst["bits"], group_size=inst["group_size"],
                          qvalues=q, scales=s)
    tile = tile or TileConfig(n_tile=1, m_tile=32, k_tile=128, g=4, lanes=16)
    return qw, prepare_weights(qw, tile)


def ref_partials(inst):
    """Per-(plane, row, channel, group) int32 staging values computed with the
    reference's own definitional tile primitive (kernel.py:190-223)."""
    qw, _ = ref_packed(inst)
    a = inst["a"].astype(np.float32)
    gs = inst["group_size"]
    planes = decompose_bits(qw, 4)
    lut = quantize_tables(mirror_consolidate(precompute_lut(a, 4)), gs)
    gpg = gs // 4
    nq = qw.k // gs
    P = np.zeros((qw.bits, a.shape[0], qw.m, nq), dtype=np.int32)
    for i, p in enumerate(planes):
        for r in range(a.shape[0]):
            for gq in range(nq):
                acc = Accumulators.zeros(qw.m)
                lookup_accumulate_tile(p.indices[:, gq * gpg:(gq + 1) * gpg], lut, acc,
                                       row=r, kg_offset=gq * gpg)
                P[i, r, :, gq] = acc.integer
    return P


def explicit_dequant_ref(inst):
    """reference_gemm (oracle.py:26-42) on explicitly dequantized weights
    w = s * (q - z): the yardstick for the generalized-zero extension."""
    q = inst["q"].astype(np.float32)
    m, k = q.shape
    gs = inst["group_size"]
    s = inst["scales"].astype(np.float32)
    z = (np.full(s.shape, float(1 << (inst["bits"] - 1)), np.float32) if inst["zeros"] is None
         else inst["zeros"].astype(np.float32))
    w = ((q.reshape(m, k // gs, gs) - z[:, :, None]) * s[:, :, None]).reshape(m, k)
    return reference_gemm(inst["a"].astype(np.float32), w.astype(np.float32))


def small_cases():
    cases = []
    specs = [
        # seed, m, k, bits, gs, n, zeros
        (11, 64, 256, 1, 32, 1, False),
        (12, 64, 256, 2, 32, 1, False),
        (13, 64, 256, 3, 32, 1, False),
        (14, 64, 256, 4, 32, 1, False),
        (15, 96, 512, 2, 64, 3, False),
        (16, 96, 512, 4, 128, 2, False),
        (17, 32, 1024, 1, 128, 1, False),
        (18, 64, 512, 4, 64, 1, True),
        (19, 64, 384, 2, 128, 5, False),
        (20, 128, 256, 3, 64, 2, True),
    ]
    store = {}
    for (seed, m, k, bits, gs, n, zeros) in specs:
        inst = W.small_instance(seed, m, k, bits, gs, n=n, zeros=zeros)
        name = inst["name"] + f"_s{seed}"
        qw, pw = ref_packed(inst)
        a = inst["a"].astype(np.float32)
        full = precompute_lut(a, 4)
        half = mirror_consolidate(full)
        qt = quantize_tables(half, gs)
        rs = row_sums(a, gs)
        planes = decompose_bits(qw, 4)
        d = {
            "q": inst["q"], "scales": inst["scales"], "a": inst["a"],
            "indices": np.stack([p.indices for p in planes]),
            "planes_v1": pw.planes,
            "lut_full": full.entries, "lut_half": half.entries,
            "qentries": qt.qentries, "tscales": qt.table_scales, "rowsums": rs.sums,
            "y_vector_q8": mpgemm(a, pw, variant=KernelVariant.VECTOR_QUANTIZED),
            "y_scalar_q8": mpgemm(a, pw, variant=KernelVariant.SCALAR_QUANTIZED),
            "y_scalar_real": mpgemm(a, pw, variant=KernelVariant.SCALAR_REAL),
            "partials": ref_partials(inst),
            "meta": np.array([m, k, bits, gs, n, 1 if zeros else 0, seed], dtype=np.int64),
        }
        if zeros:
            d["zeros"] = inst["zeros"]
            d["y_dequant_ref"] = explicit_dequant_ref(inst)
        for key, val in d.items():
            store[f"{name}/{key}"] = val
        cases.append(name)
    np.savez_compressed(os.path.join(OUT, "small_cases.npz"), **store)
    return cases


def run_cfg(inst, variants=("vector-q8", "scalar-real"), partial_sample=True, rows=None,
            dequant=False):
    """Run the reference on one BASELINE-sized instance; return arrays and
    a JSON-able summary (hashes)."""
    qw, pw = ref_packed(inst)
    a = inst["a"].astype(np.float32)
    arrays, meta = {}, {"name": inst["name"], "m": int(qw.m), "k": int(qw.k),
                        "bits": int(qw.bits), "group_size": int(qw.group_size),
                        "n": int(a.shape[0])}
    gs = inst["group_size"]
    lut = quantize_tables(mirror_consolidate(precompute_lut(a, 4)), gs)
    rs = row_sums(a, gs)
    meta["sha_qentries"] = sha(lut.qentries)
    meta["sha_tscales"] = sha(lut.table_scales)
    meta["sha_rowsums"] = sha(rs.sums)
    if a.shape[0] == 1:
        arrays["qentries"] = lut.qentries
        arrays["tscales"] = lut.table_scales
        arrays["rowsums"] = rs.sums
    for v in variants:
        t0 = time.perf_counter()
        y = mpgemm(a, pw, variant=v, threads=THREADS)
        meta[f"time_{v}_s"] = time.perf_counter() - t0
        meta[f"sha_y_{v}"] = sha(y)
        if rows is None:
            arrays[f"y_{v}"] = y
        else:
            arrays[f"y_{v}_rows"] = y[rows]
            arrays["rows"] = np.asarray(rows, dtype=np.int64)
    if partial_sample and a.shape[0] == 1:
        P = ref_partials(inst)
        meta["sha_partials"] = sha(P)
        arrays["partials_head"] = P[:, :, :64, :]
    if dequant:
        arrays["y_dequant_ref"] = explicit_dequant_ref(inst)
    return arrays, meta


def main():
    os.makedirs(OUT, exist_ok=True)
    t0 = time.time()
    small = small_cases()
    print(f"small cases: {len(small)} ({time.time() - t0:.1f}s)", flush=True)

    store, index = {}, {"reference": bitlut.__file__, "threads": THREADS,
                        "numpy": np.__version__, "configs": []}

    def add(arrays, meta):
        for key, val in arrays.items():
            store[f"{meta['name']}/{key}"] = val
        index["configs"].append(meta)
        print(f"  {meta['name']}: " + ", ".join(f"{k}={v:.2f}" for k, v in meta.items()
                                                  if k.startswith("time")), flush=True)

    add(*run_cfg(W.config1(), dequant=True))
    for si in range(3):
        add(*run_cfg(W.config2(si)))
    for si in range(3):
        for kind in ("sign", "ternary"):
            add(*run_cfg(W.config3(si, kind), dequant=True, partial_sample=False))
    for bits in (4, 2):
        for si in (0, 1):
            for n in (32, 128, 512):
                variants = ("vector-q8", "scalar-real") if n == 32 else ("vector-q8",)
                add(*run_cfg(W.config4(n, bits, si), variants=variants,
                             partial_sample=False, rows=[0, 1, n // 2, n - 1]))
    for si in range(4):
        for bits in (2, 4):
            for n in (1, 8):
                add(*run_cfg(W.config5(si, bits, n), variants=("vector-q8",),
                             partial_sample=False, rows=[0, n - 1] if n > 1 else None))
    np.savez_compressed(os.path.join(OUT, "configs.npz"), **store)
    with open(os.path.join(OUT, "configs.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"done in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
