"""Golden container files written by the REAL reference (TEST INFRASTRUCTURE).

The reference's own writers (bitlut.fileio.write_matrix / write_quantized,
bitlut.weight_prep.serialize) on small seeded inputs -> tests/golden/formats/.
tests/test_formats.py checks that this package writes the same bytes and
reads them back.

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden_formats.py
"""
import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from bitlut import Matrix, QuantizedWeights, TileConfig, prepare_weights  # noqa: E402
from bitlut.fileio import write_matrix, write_quantized  # noqa: E402
from bitlut.weight_prep import serialize  # noqa: E402

from paper_2407_00088_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "formats")


def main():
    os.makedirs(OUT, exist_ok=True)
    index = []
    for seed, (m, k, bits, gs, g) in enumerate([(64, 256, 2, 64, 4), (32, 512, 4, 128, 4),
                                                 (96, 256, 1, 32, 4), (32, 256, 3, 64, 2)]):
        inst = W.small_instance(500 + seed, m, k, bits, gs)
        qw = QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=inst["q"],
                              scales=inst["scales"].astype(np.float32))
        tile = TileConfig(n_tile=1, m_tile=32, k_tile=128, g=g, lanes=16)
        pw = prepare_weights(qw, tile)
        name = f"w{bits}_{m}x{k}_gs{gs}_g{g}"
        with open(os.path.join(OUT, name + ".lmpw"), "wb") as f:
            f.write(serialize(pw))
        write_quantized(os.path.join(OUT, name + ".lmqw"), qw)
        write_matrix(os.path.join(OUT, name + "_a.lmrm"), Matrix(inst["a"].astype(np.float32)))
        index.append({"name": name, "m": m, "k": k, "bits": bits, "group_size": gs, "g": g, "seed": 500 + seed})
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print("wrote", len(index), "cases")


if __name__ == "__main__":
    main()
