"""The auxiliary public names (api_extras.py) against golden vectors from the
real reference (oracle/make_golden_extras.py -> tests/golden/api_extras.npz)."""
import os

import numpy as np
import pytest
import torch

import paper_2407_00088_b200 as B

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "api_extras.npz"))


@pytest.mark.parametrize("g", range(1, 9))
@pytest.mark.parametrize("lanes", (16, 32))
def test_interleave_layout_matches_reference(g, lanes):
    idx = GOLD[f"il_in_g{g}_l{lanes}"]
    packed = B.interleave_layout(idx, g, lanes)
    np.testing.assert_array_equal(packed, GOLD[f"il_out_g{g}_l{lanes}"])
    np.testing.assert_array_equal(B.deinterleave_layout(packed, g, lanes), idx)


def test_interleave_layout_known_answer_and_errors():
    idx = np.arange(32, dtype=np.uint8) % 16
    out = B.interleave_layout(idx, 4, 16)
    assert out.tolist() == [(j % 16) | ((j + 16) % 16) << 4 for j in range(16)]
    with pytest.raises(B.LayoutError):
        B.interleave_layout(idx[:30], 4, 16)
    with pytest.raises(B.LayoutError):
        B.interleave_layout(idx[:16], 4, 16)         # not a whole 2*lanes unit


@pytest.mark.parametrize("tag", ("a", "b", "c"))
def test_pad_weights_matches_reference(tag):
    bits, gs, m, k, mm, km = (int(v) for v in GOLD[f"pad_{tag}_args"])
    qw = B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=GOLD[f"pad_{tag}_q"],
                            scales=GOLD[f"pad_{tag}_s"])
    p = B.pad_weights(qw, mm, km)
    np.testing.assert_array_equal(np.asarray(B.core.as_tensor(p.qvalues)), GOLD[f"pad_{tag}_outq"])
    np.testing.assert_array_equal(np.asarray(B.core.as_tensor(p.scales)), GOLD[f"pad_{tag}_outs"])
    assert p.m % mm == 0 and p.k % int(np.lcm(km, gs)) == 0


def test_pad_weights_extends_zero_points():
    q = np.ones((3, 8), np.uint8)
    s = np.ones((3, 2), np.float32)
    z = np.full((3, 2), 1.5, np.float32)
    p = B.pad_weights(B.QuantizedWeights(m=3, k=8, bits=2, group_size=4, qvalues=q, scales=s, zeros=z), 4, 12)
    assert (p.m, p.k) == (4, 12)
    zz = np.asarray(B.core.as_tensor(p.zeros))
    assert zz[:3, :2].tolist() == z.tolist() and (zz[3] == 2).all() and (zz[:, 2] == 2).all()
    with pytest.raises(B.ParameterError):
        B.pad_weights(B.QuantizedWeights(m=3, k=8, bits=2, group_size=4, qvalues=q, scales=s), 0, 4)


def test_lookup_primitives_match_reference():
    np.testing.assert_array_equal(B.byte_parallel_lookup(GOLD["bpl_tab"], GOLD["bpl_idx"]), GOLD["bpl_out"])
    lo, hi = B.split_wide_table(GOLD["wide_tab"])
    np.testing.assert_array_equal(lo, GOLD["wide_lo"])
    np.testing.assert_array_equal(hi, GOLD["wide_hi"])
    np.testing.assert_array_equal(B.wide_lookup(lo, hi, GOLD["bpl_idx"]), GOLD["wide_out"])
    np.testing.assert_array_equal(B.wide_lookup(lo, hi, np.arange(16, dtype=np.uint8)), GOLD["wide_tab"])
    with pytest.raises(B.ParameterError):
        B.byte_parallel_lookup(GOLD["bpl_tab"], np.array([16], np.uint8))
    with pytest.raises(B.ShapeError):
        B.byte_parallel_lookup(GOLD["bpl_tab"].reshape(4, 4), np.array([1], np.uint8))


@pytest.mark.parametrize("depth", range(0, 6))
def test_aggregation_helpers_match_reference(depth):
    vals = GOLD[f"agg_in_d{depth}"]
    assert B.rhadd_tree(vals) == int(GOLD[f"agg_tree_d{depth}"])
    assert B.fast_aggregate(vals, depth) == float(GOLD[f"agg_fast_d{depth}"])
    assert B.bias_correction(depth) == float(GOLD[f"agg_bias_d{depth}"])
    for bits in (1, 2, 4):
        assert B.chain_bias_correction(depth, bits) == float(GOLD[f"agg_chain_d{depth}_b{bits}"])


def test_aggregation_errors():
    with pytest.raises(B.ParameterError):
        B.rhadd_tree([1, 2, 3])
    with pytest.raises(B.ParameterError):
        B.fast_aggregate([1, 2], 2)
    with pytest.raises(B.ParameterError):
        B.bias_correction(-1)
    with pytest.raises(B.ParameterError):
        B.chain_bias_correction(1, 0)


def test_reference_names_exported():
    for name in ("pad_weights", "interleave_layout", "fast_aggregate", "reference_lut_mpgemv",
                 "reference_mpgemm"):
        assert name in B.__all__ and callable(getattr(B, name))


def _qw(tag):
    bits, g, gs, m, k = (int(v) for v in GOLD[f"ref_{tag}_args"])
    qw = B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=GOLD[f"ref_{tag}_q"],
                            scales=GOLD[f"ref_{tag}_s"])
    return qw, g


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ("w2", "w3", "w4"))
def test_definitional_references_match_reference(tag):
    """reference_mpgemm / reference_lut_mpgemv on the GPU (planes from our
    decompose_bits kernel) against the reference's own outputs; fp32
    summation order differs, so rtol 1e-5 of the output scale."""
    qw, g = _qw(tag)
    a = GOLD[f"ref_{tag}_a"]
    got = B.reference_mpgemm(a, qw)
    want = GOLD[f"ref_{tag}_mpgemm"]
    tol = 1e-5 * float(np.abs(want).max())
    np.testing.assert_allclose(got, want, rtol=0, atol=tol)
    planes = B.decompose_bits(qw, g, device="cuda")
    got = B.reference_lut_mpgemv(a[0], planes, B.bit_serial_params(qw.bits), GOLD[f"ref_{tag}_s"])
    want = GOLD[f"ref_{tag}_lut"]
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-5 * float(np.abs(want).max()))
    if qw.m % 32:
        return                       # below the CUDA layout's tile height
    # the CUDA lookup path agrees with the literal lookup within the fp16-table bound
    y = B.mpgemv(a[0], B.prepare_weights(qw), variant="cuda-f16")
    y = np.asarray(torch.as_tensor(y).float().cpu())
    np.testing.assert_allclose(y.reshape(-1), want, rtol=0, atol=1e-2 * float(np.abs(want).max()))
