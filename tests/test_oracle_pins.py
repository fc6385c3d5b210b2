"""Pin the oracle (numpy and C restatements) to the REAL reference.

The golden vectors in tests/golden/ were produced by running the reference
package (oracle/make_golden.py).  These CPU tests show the oracle
reproduces them bit for bit, so the GPU parity tests that compare against
the oracle inherit the pin.
"""
import numpy as np
import pytest

from paper_2407_00088_b200 import workloads as W
from oracle import oracle as O


def test_small_cases_bitwise(small_golden):
    for name, c in small_golden.items():
        m, k, bits, gs, n, hz, seed = [int(x) for x in c["meta"]]
        q, s, a = c["q"], c["scales"].astype(np.float32), c["a"].astype(np.float32)
        idx = O.decompose_bits(q, bits, 4)
        assert np.array_equal(idx, c["indices"]), name
        pv1 = O.pack_v1(idx, 32, 128, 4, 16)
        assert np.array_equal(pv1, c["planes_v1"]), name
        assert np.array_equal(O.unpack_v1(pv1, m, k, 32, 128, 4, 16), idx), name
        full = O.precompute_lut(a, 4)
        assert np.array_equal(full, c["lut_full"]), name
        half = O.mirror_consolidate(full)
        assert np.array_equal(half, c["lut_half"]), name
        qt, ts = O.quantize_tables(half, 4, gs)
        assert np.array_equal(qt, c["qentries"]) and np.array_equal(ts, c["tscales"]), name
        assert np.array_equal(O.row_sums(a, gs), c["rowsums"]), name
        y, P = O.mpgemm_q8(a, q, s, bits, gs, return_partials=True)
        assert np.array_equal(P, c["partials"]), name
        assert np.array_equal(y, c["y_vector_q8"]), name
        assert np.array_equal(O.mpgemm_real(a, q, s, bits, gs), c["y_scalar_real"]), name


def test_c_oracle_small_bitwise(small_golden):
    for name, c in small_golden.items():
        m, k, bits, gs, n, hz, seed = [int(x) for x in c["meta"]]
        s = c["scales"].astype(np.float32)
        for mode, key in (("vector-q8", "y_vector_q8"), ("scalar-real", "y_scalar_real")):
            for threads in (1, 3):
                y = O.c_mpgemm(c["a"], c["planes_v1"], m, k, bits, gs, s, mode=mode,
                               threads=threads)
                assert np.array_equal(y, c[key]), (name, mode, threads)


def test_zero_point_extension_vs_reference_dequant(small_golden):
    """Generalized zero (BASELINE extension): reference kernel + correction
    agrees with the reference's dequantize-then-GEMM oracle (oracle.py:26-42)."""
    for name, c in small_golden.items():
        if int(c["meta"][5]) == 0:
            continue
        bits, gs = int(c["meta"][2]), int(c["meta"][3])
        y = O.mpgemm_real(c["a"], c["q"], c["scales"].astype(np.float32), bits, gs,
                          zeros=c["zeros"])
        ref = c["y_dequant_ref"]
        assert np.abs(y - ref).max() <= 1e-5 * np.abs(ref).max(), name


@pytest.mark.parametrize("si", [0, 1, 2])
def test_config2_full_size_bitwise(config_golden, si):
    """BASELINE config 2 (Llama-2-7B W2 g64) at full size: tables, int32
    partials and vector-q8/scalar-real outputs equal the reference's."""
    inst = W.config2(si)
    g = config_golden[inst["name"]]
    a = inst["a"].astype(np.float32)
    s = inst["scales"].astype(np.float32)
    half = O.mirror_consolidate(O.precompute_lut(a, 4))
    qt, ts = O.quantize_tables(half, 4, 64)
    assert np.array_equal(qt, g["qentries"]) and np.array_equal(ts, g["tscales"])
    assert np.array_equal(O.row_sums(a, 64), g["rowsums"])
    planes = O.pack_v1(O.decompose_bits(inst["q"], 2, 4), 32, 128, 4, 16)
    y = O.c_mpgemm(a, planes, inst["q"].shape[0], inst["q"].shape[1], 2, 64, s)
    assert np.array_equal(y, g["y_vector-q8"])
    yr = O.c_mpgemm(a, planes, inst["q"].shape[0], inst["q"].shape[1], 2, 64, s,
                    mode="scalar-real")
    assert np.array_equal(yr, g["y_scalar-real"])


def test_config1_zero_correction_vs_dequant(config_golden):
    inst = W.config1()
    g = config_golden[inst["name"]]
    a = inst["a"].astype(np.float32)
    rs = O.row_sums(a, inst["group_size"])
    y = g["y_scalar-real"][0] + O.zero_correction(inst["scales"], inst["zeros"], 4, rs[0])
    ref = g["y_dequant_ref"][0]
    assert np.abs(y - ref).max() <= 1e-5 * np.abs(ref).max()


def test_known_answers():
    # test_oracle.py:66-75 / SPEC.md:283: bits (1,0,1,0), a=(1,2,3,4) -> -6
    q = np.array([[1, 0, 1, 0]], dtype=np.uint8)
    a = np.array([[1, 2, 3, 4]], dtype=np.float32)
    idx = O.decompose_bits(q, 1, 4)
    assert idx[0, 0, 0] == 0b0101
    y = O.mpgemm_real(a, q, np.ones((1, 1), np.float32), 1, 4)
    assert y[0, 0] == np.float32(-6.0)
    # test_weight_prep.py:27-30: [0,1,2,3] -> plane0 0b1010, plane1 0b1100
    idx2 = O.decompose_bits(np.array([[0, 1, 2, 3]], np.uint8), 2, 4)
    assert idx2[0, 0, 0] == 0b1010 and idx2[1, 0, 0] == 0b1100
    # test_lut_build.py:24-34 endpoints
    t = O.precompute_lut(np.array([1.5, -2.0, 0.25, 3.0], np.float32), 4)
    assert t[0, 0, 0] == -(1.5 - 2.0 + 0.25 + 3.0)
    ones = O.precompute_lut(np.ones(4, np.float32), 4)
    assert ones[0, 0, 0] == -4 and ones[0, 0, 15] == 4 and ones[0, 0, 5] == 0
    # test_lut_build.py:105-110: scale 4/127, stored -4 -> -127
    qt, ts = O.quantize_tables(O.mirror_consolidate(ones), 4, 4)
    assert ts[0, 0] == np.float32(4.0 / 127.0) and qt[0, 0, 0] == -127
    # all-zero tables -> scale 1
    z = O.mirror_consolidate(O.precompute_lut(np.zeros(8, np.float32), 4))
    qz, tz = O.quantize_tables(z, 4, 8)
    assert np.all(tz == 1.0) and np.all(qz == 0)


def _table4_inputs(m, k):
    """pkg/tests/test_acceptance.py:65-68: w, a from default_rng(0)."""
    rng = np.random.default_rng(0)
    w = rng.standard_normal((m, k), dtype=np.float32)
    a = rng.standard_normal(k, dtype=np.float32)
    return w, a


def test_c_quantizer_pinned_to_reference():
    """The C restatement of the reference's group quantizer (_kernels.py:20-82)
    reproduces its codes and scales bit for bit on the Table-4 shapes of the
    NMSE criterion (sha256 from oracle/make_golden_nmse.py)."""
    import hashlib
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "nmse.json")))
    for row in gold["shapes"]:
        w, _ = _table4_inputs(row["m"], row["k"])
        q, d = O.c_quantize_weights(w, row["bits"], row["group_size"])
        assert hashlib.sha256(q.tobytes()).hexdigest() == row["sha_q"], (row["m"], row["k"])
        assert hashlib.sha256(d.tobytes()).hexdigest() == row["sha_scales"], (row["m"], row["k"])
