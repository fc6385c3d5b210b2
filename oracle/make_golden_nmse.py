"""Golden values of the reference's NMSE acceptance criterion C2
(pkg/tests/test_acceptance.py:61-82, :121-138; recorded values
pkg/test_output.txt:220) -- TEST INFRASTRUCTURE.

Runs the REAL reference (read-only, numba cache in /tmp) on the three
Table-4 shapes exactly as its acceptance test does -- w, a from
default_rng(0), quantize_weights(w, 4, 32), prepare_weights, mpgemv
vector-q8 vs reference_gemm(a, w) -- and writes tests/golden/nmse.json:
sha256 of the quantized codes and scales (pins oracle.c_quantize_weights)
and the NMSE values (the CUDA path must reproduce them).

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden_nmse.py
"""
import hashlib
import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
from bitlut import KernelVariant, TileConfig, mpgemv, prepare_weights, quantize_weights  # noqa: E402
from bitlut.oracle import reference_gemm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "nmse.json")
SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def main():
    rows = []
    for (m, k) in SHAPES:
        rng = np.random.default_rng(0)
        w = rng.standard_normal((m, k), dtype=np.float32)
        a = rng.standard_normal(k, dtype=np.float32)
        qw = quantize_weights(w, 4, 32)
        pw = prepare_weights(qw, TileConfig(m_tile=32, k_tile=128))
        y = reference_gemm(a, w)[0]
        out = mpgemv(a, pw, variant=KernelVariant.VECTOR_QUANTIZED, threads=os.cpu_count() or 1)
        nmse = float(((y - out) ** 2).sum()) / float((y ** 2).sum())
        rows.append({"m": m, "k": k, "bits": 4, "group_size": 32, "seed": 0,
                     "sha_q": sha(qw.qvalues), "sha_scales": sha(qw.scales), "sha_y_ref": sha(y),
                     "sha_y_vector_q8": sha(out), "nmse_vector_q8": nmse})
        print(m, k, nmse, flush=True)
    with open(OUT, "w") as f:
        json.dump({"source": "pkg/tests/test_acceptance.py:61-82 (criterion 2)", "shapes": rows}, f, indent=1)


if __name__ == "__main__":
    main()
