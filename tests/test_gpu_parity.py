"""GPU parity: CUDA path vs the reference (golden vectors) and the oracle.

Bars (north star): int8 tables -> bit-exact int32 staging values, and
(our epilogue replays the reference order) a bitwise-identical float32
output; zero-point extension -> bitwise vs the oracle's defined order and
within 1e-5 (max-norm) of the reference's dequantize-then-GEMM.
"""
import hashlib

import numpy as np
import pytest
import torch

import paper_2407_00088_b200 as B
from paper_2407_00088_b200 import workloads as W
from paper_2407_00088_b200.weight_prep import unrepack_gpu

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def make_pw(inst, tile=None):
    qw = B.QuantizedWeights(m=inst["q"].shape[0], k=inst["q"].shape[1], bits=inst["bits"],
                            group_size=inst["group_size"], qvalues=inst["q"],
                            scales=inst["scales"], zeros=inst.get("zeros"))
    tile = tile or B.TileConfig(n_tile=1, m_tile=32, k_tile=128, g=4, lanes=16)
    return qw, B.prepare_weights(qw, tile)


def plain(small_golden, i):
    """i-th small case without zero points."""
    names = [n for n in sorted(small_golden) if int(small_golden[n]["meta"][5]) == 0]
    return small_golden[names[i % len(names)]]


def decode_kernel_tables(t, gs):
    """Kernel-format LUT (layout.cuh table_offset, bytes Q - (Q<0)) ->
    reference qentries (n, KG, 8) int8."""
    n, kgt = t.shape[0], t.shape[1]
    raw = t.reshape(n, kgt * 8).view(np.int8).astype(np.int16)
    R = 8 if (gs // 4) % 8 == 0 else 4
    U = kgt // R
    kg = np.arange(kgt)
    u, r = kg // R, kg % R
    ub, l = u >> 5, u & 31
    nu_b = np.minimum(32, U - 32 * ub)
    off = ub * (32 * R * 8) + ((r >> 1) * nu_b + l) * 16 + (r & 1) * 8
    a = raw[:, off[:, None] + np.arange(8)[None, :]]
    return (a + (a < 0)).astype(np.int8)


def small_inst(c):
    m, k, bits, gs, n, hz, seed = [int(x) for x in c["meta"]]
    return dict(q=c["q"], scales=c["scales"], a=c["a"], bits=bits, group_size=gs,
                zeros=c.get("zeros") if hz else None)


# ---------------------------------------------------------------- weights

def test_weight_prep_matches_reference(small_golden):
    for name, c in small_golden.items():
        inst = small_inst(c)
        qw, pw = make_pw(inst)
        planes = B.decompose_bits(qw, 4)
        got = np.stack([p.indices.cpu().numpy() for p in planes])
        assert np.array_equal(got, c["indices"]), name
        assert np.array_equal(pw.planes.cpu().numpy(), c["planes_v1"]), name
        back = np.stack([p.indices.cpu().numpy() for p in B.unpack_planes(pw)])
        assert np.array_equal(back, c["indices"]), name
        if pw.gpu is not None:
            assert np.array_equal(unrepack_gpu(pw).cpu().numpy(), c["indices"]), name


@pytest.mark.parametrize("g", [1, 2, 3, 5, 6, 8])
def test_v1_pack_other_g(rng, g):
    m, k = 32, 8 * g * 8
    q = rng.integers(0, 8, (m, k), dtype=np.uint8)
    qw = B.QuantizedWeights(m=m, k=k, bits=3, group_size=k, qvalues=q,
                            scales=np.ones((m, 1), np.float32))
    tile = B.TileConfig(m_tile=16, k_tile=8 * g, g=g, lanes=16)
    pw = B.prepare_weights(qw, tile)
    idx = O.decompose_bits(q, 3, g)
    assert np.array_equal(pw.planes.cpu().numpy(), O.pack_v1(idx, 16, 8 * g, g, 16))
    back = np.stack([p.indices.cpu().numpy() for p in B.unpack_planes(pw)])
    assert np.array_equal(back, idx)


# ---------------------------------------------------------------- tables

def test_tables_match_reference(small_golden):
    for name, c in small_golden.items():
        gs = int(c["meta"][3])
        a = torch.from_numpy(c["a"]).cuda()
        full = B.precompute_lut(a, 4)
        assert np.array_equal(full.entries.cpu().numpy(), c["lut_full"]), name
        half = B.mirror_consolidate(full)
        assert np.array_equal(half.entries.cpu().numpy(), c["lut_half"]), name
        qt = B.quantize_tables(half, gs)
        assert np.array_equal(qt.qentries.cpu().numpy(), c["qentries"]), name
        assert np.array_equal(qt.table_scales.cpu().numpy(), c["tscales"]), name
        rs = B.row_sums(a, gs)
        assert np.array_equal(rs.sums.cpu().numpy(), c["rowsums"]), name
        # the fused per-call build used by mpgemm
        from paper_2407_00088_b200 import _native as N
        t, ts, rsf = N.build_lut(a, gs, N.TABLE_Q8)
        assert np.array_equal(decode_kernel_tables(t.cpu().numpy(), gs), c["qentries"]), name
        assert np.array_equal(ts.cpu().numpy(), c["tscales"]), name
        assert np.array_equal(rsf.cpu().numpy(), c["rowsums"]), name


@pytest.mark.parametrize("g", [1, 2, 3, 5])
def test_precompute_other_g(rng, g):
    a = rng.standard_normal((3, 8 * g)).astype(np.float32)
    full = B.precompute_lut(a, g).entries.cpu().numpy()
    assert np.array_equal(full, O.precompute_lut(a, g))


# ---------------------------------------------------------------- mpgemm, small

def test_mpgemm_small_bitwise(small_golden):
    for name, c in small_golden.items():
        inst = small_inst(c)
        qw, pw = make_pw(inst)
        y, P = B.mpgemm(c["a"], pw, return_partials=True)
        assert np.array_equal(P.transpose(1, 0, 2, 3), c["partials"]), name
        if inst["zeros"] is None:
            assert np.array_equal(y, c["y_vector_q8"]), name
            assert np.array_equal(y, c["y_scalar_q8"]), name
        else:
            yo = O.mpgemm_q8(c["a"], c["q"], c["scales"].astype(np.float32), inst["bits"],
                             inst["group_size"], zeros=c["zeros"])
            assert np.array_equal(y, yo), name
            ref = c["y_dequant_ref"]
            assert np.abs(y - ref).max() <= 1e-2 * np.abs(ref).max(), name


def test_mpgemv_equals_mpgemm_row(small_golden):
    c = plain(small_golden, 4)
    inst = small_inst(c)
    _, pw = make_pw(inst)
    full = B.mpgemm(c["a"], pw)
    for r in range(c["a"].shape[0]):
        assert np.array_equal(B.mpgemv(c["a"][r], pw), full[r])


def test_cuda_tensor_in_cuda_tensor_out(small_golden):
    c = plain(small_golden, 0)
    _, pw = make_pw(small_inst(c))
    a = torch.from_numpy(c["a"]).cuda()
    y = B.mpgemm(a, pw)
    assert y.is_cuda and y.dtype == torch.float32
    assert np.array_equal(y.cpu().numpy(), c["y_vector_q8"])


def test_determinism_repeat(small_golden):
    c = plain(small_golden, 5)
    _, pw = make_pw(small_inst(c))
    y0 = B.mpgemm(c["a"], pw)
    for _ in range(3):
        assert np.array_equal(B.mpgemm(c["a"], pw), y0)


def test_zero_activation_zero_output(small_golden):
    c = plain(small_golden, 1)
    _, pw = make_pw(small_inst(c))
    y = B.mpgemv(np.zeros(pw.k, np.float32), pw)
    assert np.all(y == 0.0)


def test_stats_counters(small_golden):
    c = plain(small_golden, 4)
    _, pw = make_pw(small_inst(c))
    st = B.KernelStats()
    B.mpgemm(c["a"], pw, stats=st)
    n = c["a"].shape[0]
    assert st.lookups == pw.bits * n * pw.m * (pw.k // 4)
    assert st.lut_builds == n * (pw.k // pw.tile.k_tile)


# ---------------------------------------------------------------- BASELINE shapes

@pytest.mark.parametrize("si", [0, 1, 2])
def test_config2_llama7b_w2_bitwise(config_golden, si):
    inst = W.config2(si)
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y, P = B.mpgemm(inst["a"], pw, return_partials=True)
    assert np.array_equal(y, g["y_vector-q8"])
    assert sha(y) == g["meta"]["sha_y_vector-q8"]
    Pr = P.transpose(1, 0, 2, 3)
    assert np.array_equal(Pr[:, :, :64, :], g["partials_head"])
    assert sha(Pr) == g["meta"]["sha_partials"]


def test_config1_asymmetric_zeros(config_golden):
    inst = W.config1()
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw)
    # bitwise vs the reference's vector-q8 + the oracle's zero correction
    rs = O.row_sums(inst["a"].astype(np.float32), inst["group_size"])
    corr = O.zero_correction(inst["scales"], inst["zeros"], inst["bits"], rs[0])
    expect = (g["y_vector-q8"][0] + corr).astype(np.float32)
    assert np.array_equal(y[0], expect)
    ref = g["y_dequant_ref"][0]
    assert np.abs(y[0] - ref).max() <= 1e-2 * np.abs(ref).max()


@pytest.mark.parametrize("si", [0, 1, 2])
@pytest.mark.parametrize("kind", ["sign", "ternary"])
def test_config3_sign_and_ternary(config_golden, si, kind):
    inst = W.config3(si, kind)
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw)
    rs = O.row_sums(inst["a"].astype(np.float32), inst["group_size"])
    corr = O.zero_correction(inst["scales"], inst["zeros"], inst["bits"], rs[0])
    expect = (g["y_vector-q8"][0] + corr).astype(np.float32)
    assert np.array_equal(y[0], expect)
    ref = g["y_dequant_ref"][0]
    assert np.abs(y[0] - ref).max() <= 2e-2 * np.abs(ref).max()


@pytest.mark.parametrize("bits", [4, 2])
@pytest.mark.parametrize("si", [0, 1])
def test_config4_prefill_rows(config_golden, bits, si):
    inst = W.config4(32, bits, si)
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw)
    assert np.array_equal(y[g["rows"]], g["y_vector-q8_rows"])
    assert sha(y) == g["meta"]["sha_y_vector-q8"]


@pytest.mark.parametrize("si", [0, 1, 2, 3])
@pytest.mark.parametrize("bits", [2, 4])
def test_config5_llama70b_shapes(config_golden, si, bits):
    inst = W.config5(si, bits, 1)
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw)
    assert np.array_equal(y, g["y_vector-q8"])


# ---------------------------------------------------------------- errors

def test_errors(small_golden):
    c = plain(small_golden, 0)
    _, pw = make_pw(small_inst(c))
    with pytest.raises(B.ShapeError):
        B.mpgemv(c["a"][0][:-4], pw)
    bad = c["a"][0].astype(np.float32).copy()
    bad[0] = np.nan
    with pytest.raises(B.DataError):
        B.mpgemv(bad, pw)
    with pytest.raises(B.LayoutError):
        B.mpgemv(c["a"][0], pw, cfg=B.TileConfig(m_tile=16, k_tile=128))
    with pytest.raises(B.ParameterError):
        B.mpgemv(c["a"][0], pw, variant="vector-q8")


# ---------------------------------------------------------------- fp16 tables

def rel_maxnorm(y, ref):
    return float(np.abs(y - ref).max() / np.abs(ref).max())


def test_f16_small_vs_scalar_real(small_golden):
    """cuda-f16 vs the reference's fp32-table scalar-real: max|dy| <= 1e-3 max|y|
    (north-star tolerance; element-wise rtol is not meaningful)."""
    for name, c in small_golden.items():
        inst = small_inst(c)
        _, pw = make_pw(inst)
        y = B.mpgemm(c["a"], pw, variant="cuda-f16")
        if inst["zeros"] is None:
            ref = c["y_scalar_real"]
        else:
            ref = O.mpgemm_real(c["a"], c["q"], c["scales"].astype(np.float32), inst["bits"],
                                inst["group_size"], zeros=c["zeros"])
        assert rel_maxnorm(y, ref) <= 1e-3, (name, rel_maxnorm(y, ref))


def test_f16_config1_w4_asym_fp16_tables(config_golden):
    """BASELINE config 1 exactly: 4096x4096 W4 asymmetric zeros g128, fp16
    tables, compared against the reference (scalar-real + zero correction)."""
    inst = W.config1()
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw, variant="cuda-f16")[0]
    rs = O.row_sums(inst["a"].astype(np.float32), inst["group_size"])
    ref = (g["y_scalar-real"][0] + O.zero_correction(inst["scales"], inst["zeros"], 4, rs[0])).astype(np.float32)
    assert rel_maxnorm(y, ref) <= 1e-3, rel_maxnorm(y, ref)
    assert rel_maxnorm(y, g["y_dequant_ref"][0]) <= 1e-3


@pytest.mark.parametrize("si", [0, 1, 2])
@pytest.mark.parametrize("kind", ["sign", "ternary"])
def test_f16_config3(config_golden, si, kind):
    inst = W.config3(si, kind)
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw, variant="cuda-f16")[0]
    rs = O.row_sums(inst["a"].astype(np.float32), inst["group_size"])
    ref = (g["y_scalar-real"][0] + O.zero_correction(inst["scales"], inst["zeros"], inst["bits"], rs[0])).astype(np.float32)
    assert rel_maxnorm(y, ref) <= 1e-3, rel_maxnorm(y, ref)


@pytest.mark.parametrize("si", [0, 1, 2])
def test_f16_config2(config_golden, si):
    inst = W.config2(si)
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    y = B.mpgemm(inst["a"], pw, variant="cuda-f16")[0]
    assert rel_maxnorm(y, g["y_scalar-real"][0]) <= 1e-3


def test_f16_deterministic(small_golden):
    c = plain(small_golden, 3)
    _, pw = make_pw(small_inst(c))
    y0 = B.mpgemm(c["a"], pw, variant="cuda-f16")
    for _ in range(3):
        assert np.array_equal(B.mpgemm(c["a"], pw, variant="cuda-f16"), y0)


# ---------------------------------------------------------------- sharding

@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_slices_bitwise_on_one_gpu(world):
    """Every rank's shard, run through the CUDA kernel on one GPU and
    concatenated, equals the unsharded output bitwise (what the all-gather
    assembles on P GPUs; the gather itself is tested under gloo)."""
    from paper_2407_00088_b200 import parallel as PAR
    inst = W.config5(3, 2, 8)          # 1024 x 8192 W2, batch 8
    qw, pw = make_pw(inst)
    full = B.mpgemm(inst["a"], pw)
    parts = []
    for r in range(world):
        local = PAR.shard_quantized_weights(qw, r, world)
        parts.append(B.mpgemm(inst["a"], B.prepare_weights(local, B.TileConfig(m_tile=32, k_tile=128))))
    assert np.array_equal(np.concatenate(parts, axis=1), full)


def test_independent_launch_chain_matches():
    """k/v-style INDEPENDENT launches after a dependent one reading the same
    fresh table give the same (bitwise) results as fully dependent ones."""
    from paper_2407_00088_b200 import _native as N
    insts = [W.small_instance(40 + i, 512, 2048, 2, 64) for i in range(3)]
    pws = [make_pw(i)[1] for i in insts]
    a = torch.from_numpy(insts[0]["a"]).cuda()
    ref = [B.mpgemm(a, pw) for pw in pws]
    for _ in range(5):
        t, ts, rs = N.build_lut(a, 64, N.TABLE_Q8, N.FLAG_PDL)
        outs = []
        for j, pw in enumerate(pws):
            fl = N.FLAG_PDL | (N.FLAG_INDEPENDENT if j > 0 else 0)
            y, _ = N.lookup(pw.gpu, pw.scales, None, t, ts, rs, pw.m, pw.k, pw.bits, pw.group_size,
                            N.TABLE_Q8, fl, False)
            outs.append(y)
        for y, r in zip(outs, ref):
            assert torch.equal(y, r)


# ---------------------------------------------------------------- pipeline

@pytest.mark.parametrize("executor", ["graph", "graph-counters"])
def test_pipeline_matches_per_op_bitwise(executor):
    """Two decoder-like layers (shared-table q/k/v, dependent o, gate/up,
    down) through either pipeline executor == per-op mpgemm, bitwise."""
    from paper_2407_00088_b200.pipeline import Pipeline
    gs, bits = 64, 2
    shapes = {"q": (256, 512), "k": (256, 512), "v": (256, 512), "o": (256, 512),
              "gate": (352, 512), "up": (352, 512), "down": (256, 1024)}
    g = torch.Generator(device="cuda").manual_seed(3)
    layers = []
    for _ in range(2):
        L = {}
        for nm, (m, k) in shapes.items():
            q = torch.randint(0, 4, (m, k), dtype=torch.uint8, device="cuda", generator=g)
            sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
            L[nm] = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
        layers.append(L)
    xs = [{nm: torch.randn((1, k), device="cuda", generator=g).half() for nm, k in
           (("attn", 512), ("o", 512), ("mlp", 512), ("down", 1024))} for _ in layers]
    pl = Pipeline(executor="graph", sync="counters" if executor == "graph-counters" else "pdl")
    outs, prev = [], []
    for L, X in zip(layers, xs):
        t = pl.tables(X["attn"], gs, deps=prev)
        yq, yk, yv = pl.lookup(L["q"], t), pl.lookup(L["k"], t), pl.lookup(L["v"], t)
        t2 = pl.tables(X["o"], gs, deps=[pl.op_of(yq), pl.op_of(yk), pl.op_of(yv)])
        yo = pl.lookup(L["o"], t2)
        t3 = pl.tables(X["mlp"], gs, deps=[pl.op_of(yo)])
        yg, yu = pl.lookup(L["gate"], t3), pl.lookup(L["up"], t3)
        t4 = pl.tables(X["down"], gs, deps=[pl.op_of(yg), pl.op_of(yu)])
        yd = pl.lookup(L["down"], t4)
        prev = [pl.op_of(yd)]
        outs.append({"q": yq, "k": yk, "v": yv, "o": yo, "gate": yg, "up": yu, "down": yd})
    pl.compile()
    if True:
        F, I = B._native.FLAG_PDL, B._native.FLAG_PDL | B._native.FLAG_INDEPENDENT
        J = B._native.PLAN_JOINED          # q,k,v and gate,up share a launch
        assert pl.plan_flags()[:11] == [F, F, F | J, F | J, F, F, F, F, F | J, F, F]
    for _ in range(3):
        pl.run()
        torch.cuda.synchronize()
        for L, X, O in zip(layers, xs, outs):
            for nm, xk in (("q", "attn"), ("k", "attn"), ("v", "attn"), ("o", "o"), ("gate", "mlp"),
                           ("up", "mlp"), ("down", "down")):
                ref = B.mpgemm(X[xk], L[nm])
                assert torch.equal(O[nm], ref), nm


def test_fast_epilogue_exact_partials_and_tolerance(small_golden, config_golden):
    """Fast epilogue: same exact int32 partials; float output within 1e-5
    (max-norm) of the reference's vector-q8 output; deterministic."""
    for name, c in small_golden.items():
        inst = small_inst(c)
        _, pw = make_pw(inst)
        y, P = B.mpgemm(c["a"], pw, return_partials=True, exact_epilogue=False)
        assert np.array_equal(P.transpose(1, 0, 2, 3), c["partials"]), name
        ref = c["y_vector_q8"] if inst["zeros"] is None else O.mpgemm_q8(
            c["a"], c["q"], c["scales"].astype(np.float32), inst["bits"], inst["group_size"], zeros=c["zeros"])
        assert rel_maxnorm(y, ref) <= 1e-5, (name, rel_maxnorm(y, ref))
        # without partials: register epilogue (32-stream tiles), same bound, deterministic
        y2 = B.mpgemm(c["a"], pw, exact_epilogue=False)
        assert rel_maxnorm(y2, ref) <= 1e-5, (name, rel_maxnorm(y2, ref))
        assert np.array_equal(B.mpgemm(c["a"], pw, exact_epilogue=False), y2)
    for si in range(3):
        inst = W.config2(si)
        _, pw = make_pw(inst)
        y = B.mpgemm(inst["a"], pw, exact_epilogue=False)
        assert rel_maxnorm(y, config_golden[inst["name"]]["y_vector-q8"]) <= 1e-5
        yf = B.mpgemm(inst["a"], pw, variant="cuda-f16", exact_epilogue=False)
        assert rel_maxnorm(yf, config_golden[inst["name"]]["y_scalar-real"]) <= 1e-3


@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("gs", [16, 32, 64, 128, 256, 512])
@pytest.mark.parametrize("zeros", [False, True])
def test_group_sizes_exact_and_fast(bits, gs, zeros):
    """Every supported group size (1..16 units per group, R = 4 or 8) and
    width, with and without zero points: exact epilogue bitwise == oracle,
    fast epilogue within 1e-5 and deterministic."""
    m, k, n = 96 if bits == 3 else 64, 1024, 2
    inst = W.small_instance(1000 + bits * 10 + gs // 16, m, k, bits, gs, n=n, zeros=zeros)
    _, pw = make_pw(inst)
    ref = O.mpgemm_q8(inst["a"], inst["q"], inst["scales"].astype(np.float32), bits, gs,
                      zeros=inst.get("zeros"))
    y = B.mpgemm(inst["a"], pw)
    assert np.array_equal(y, ref)
    yf = B.mpgemm(inst["a"], pw, exact_epilogue=False)
    assert rel_maxnorm(yf, ref) <= 1e-5, rel_maxnorm(yf, ref)
    assert np.array_equal(B.mpgemm(inst["a"], pw, exact_epilogue=False), yf)


@pytest.mark.parametrize("bits", [1, 2, 4])
@pytest.mark.parametrize("gs", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("zeros", [False, True])
@pytest.mark.parametrize("k", [1024, 11008])
def test_batch1_fast_kernel(bits, gs, zeros, k):
    """Batch-1 fast path (csrc/gemv_b1.cu, persistent tiles, merged plane
    multipliers): within 1e-5 of the oracle's vector-q8 output and
    deterministic; k = 11008 exercises multi-round tiles with smem tables."""
    if k % gs:
        pytest.skip("k not a multiple of gs")
    m = 8 * 32 // bits * 3                     # several tiles per CTA pair
    inst = W.small_instance(2000 + bits * 100 + gs + k, m, k, bits, gs, n=1, zeros=zeros)
    _, pw = make_pw(inst)
    ref = O.mpgemm_q8(inst["a"], inst["q"], inst["scales"].astype(np.float32), bits, gs,
                      zeros=inst.get("zeros"))[0]
    y = B.mpgemv(inst["a"][0], pw, exact_epilogue=False)
    assert rel_maxnorm(y, ref) <= 1e-5, rel_maxnorm(y, ref)
    assert np.array_equal(B.mpgemv(inst["a"][0], pw, exact_epilogue=False), y)
    try:
        assert np.array_equal(B.mpgemv(inst["a"][0], pw), ref)      # exact path, same inputs
    except B.LayoutError:
        # the reference-order epilogue stages every partial of a tile in smem:
        # 688 groups (k=11008, gs=16) exceed 227 KB -- a documented limit
        assert gs == 16 and k == 11008


def test_fused_mpgemv_and_graph_fusion():
    """bitlut_mpgemv_fused (in-kernel cluster table build) == build_lut +
    batch-1 fast lookup, bitwise; the graph executor folds the table ops of
    fast lookups into them and matches per-op calls bitwise."""
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200.pipeline import Pipeline
    g = torch.Generator(device="cuda").manual_seed(5)
    for bits, gs, m, k, zeros in ((2, 64, 512, 4096, False), (4, 128, 256, 11008, True),
                                  (1, 32, 1024, 2048, False), (2, 256, 256, 4096, True),
                                  (4, 16, 128, 1024, False)):
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
        z = (torch.rand((m, k // gs), device="cuda", generator=g) * ((1 << bits) - 1)).half() if zeros else None
        pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc,
                                                  zeros=z))
        x = torch.randn((1, k), device="cuda", generator=g).half()
        fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE
        yf = N.mpgemv_fused(x, pw.gpu, pw.scales, pw.zeros, m, k, bits, gs, fl)
        t = N.build_lut(x, gs, N.TABLE_Q8)
        y2, _ = N.lookup(pw.gpu, pw.scales, pw.zeros, *t, m, k, bits, gs, N.TABLE_Q8, fl, False)
        assert torch.equal(yf, y2), (bits, gs, m, k)
        ref = O.mpgemm_q8(x.cpu().numpy(), q.cpu().numpy(), sc.float().cpu().numpy(), bits, gs,
                          zeros=None if z is None else z.cpu().numpy())
        assert rel_maxnorm(yf.cpu().numpy(), ref) <= 1e-5
    # graph executor: two layers of q,k,v / o / gate,up / down with fast lookups
    shapes = {"q": (256, 512), "k": (256, 512), "v": (256, 512), "o": (256, 512),
              "gate": (352, 512), "up": (352, 512), "down": (256, 1024)}
    layers = []
    for _ in range(2):
        L = {}
        for nm, (m, k) in shapes.items():
            q = torch.randint(0, 4, (m, k), dtype=torch.uint8, device="cuda", generator=g)
            sc = (torch.randn((m, k // 64), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
            L[nm] = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=2, group_size=64, qvalues=q, scales=sc))
        layers.append(L)
    xs = [{nm: torch.randn((1, k), device="cuda", generator=g).half() for nm, k in
           (("attn", 512), ("o", 512), ("mlp", 512), ("down", 1024))} for _ in layers]
    pl = Pipeline(executor="graph")
    outs, prev = [], []
    for L, X in zip(layers, xs):
        t = pl.tables(X["attn"], 64, deps=prev, fuse=True)
        ys = {nm: pl.lookup(L[nm], t, fast_epilogue=True) for nm in ("q", "k", "v")}
        t2 = pl.tables(X["o"], 64, deps=[pl.op_of(y) for y in ys.values()], fuse=True)
        ys["o"] = pl.lookup(L["o"], t2, fast_epilogue=True)
        t3 = pl.tables(X["mlp"], 64, deps=[pl.op_of(ys["o"])], fuse=True)
        ys["gate"], ys["up"] = (pl.lookup(L[nm], t3, fast_epilogue=True) for nm in ("gate", "up"))
        t4 = pl.tables(X["down"], 64, deps=[pl.op_of(ys["gate"]), pl.op_of(ys["up"])], fuse=True)
        ys["down"] = pl.lookup(L["down"], t4, fast_epilogue=True)
        prev = [pl.op_of(ys["down"])]
        outs.append(ys)
    plan = pl.plan_flags()
    assert plan.count(-1) == 8 and all(f & 8 for f in plan if f != -1)
    pl.compile()
    for _ in range(3):
        pl.run()
        torch.cuda.synchronize()
        for L, X, Y in zip(layers, xs, outs):
            for nm, xk in (("q", "attn"), ("k", "attn"), ("v", "attn"), ("o", "o"), ("gate", "mlp"),
                           ("up", "mlp"), ("down", "down")):
                assert torch.equal(Y[nm], B.mpgemm(X[xk], L[nm], exact_epilogue=False)), nm


@pytest.mark.parametrize("sync", ["counters", "pdl"])
@pytest.mark.parametrize("bits", [1, 2, 4])
def test_graph_grouped_launches_bitwise(bits, sync):
    """Layer-set op list (tables one layer ahead): the graph executor groups
    the table builds (bitlut_build_lut_multi) and the lookups over one table
    (bitlut_mpgemv_multi); every output == the per-op fast call, bitwise."""
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200.pipeline import Pipeline
    g = torch.Generator(device="cuda").manual_seed(11 + bits)
    gs = 64
    shapes = {"q": (256, 512), "k": (256, 512), "v": (128, 512), "o": (256, 512),
              "gate": (352, 512), "up": (352, 512), "down": (256, 2048)}
    groups = [("attn", 512, ["q", "k", "v"]), ("o", 512, ["o"]), ("mlp", 512, ["gate", "up"]),
              ("down", 2048, ["down"])]
    layers, xs = [], []
    for li in range(2):
        L = {}
        for nm, (m, k) in shapes.items():
            q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
            sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
            z = ((torch.rand((m, k // gs), device="cuda", generator=g) * ((1 << bits) - 1)).half()
                 if li == 1 else None)
            L[nm] = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q,
                                                         scales=sc, zeros=z))
        layers.append(L)
        xs.append({gn: torch.randn((1, k), device="cuda", generator=g).half() for gn, k, _ in groups})
    pl = Pipeline(executor="graph", sync=sync)
    tabs = [{gn: pl.tables(X[gn], gs) for gn, _, _ in groups} for X in xs]
    outs = []
    for L, T in zip(layers, tabs):
        outs.append({nm: pl.lookup(L[nm], T[gn], fast_epilogue=True) for gn, _, names in groups for nm in names})
    plan = pl.plan_flags()
    assert any(f & 16 for f in plan)                      # some launches are grouped
    pl.compile()
    for _ in range(2):
        pl.run()
        torch.cuda.synchronize()
        for L, X, Y in zip(layers, xs, outs):
            for gn, _, names in groups:
                t = N.build_lut(X[gn], gs, N.TABLE_Q8)
                for nm in names:
                    pw = L[nm]
                    ref, _ = N.lookup(pw.gpu, pw.scales, pw.zeros, *t, pw.m, pw.k, bits, gs, N.TABLE_Q8,
                                      N.FLAG_PDL | N.FLAG_FAST_EPILOGUE, False)
                    assert torch.equal(Y[nm], ref), (nm, bits)


def test_batch1_fast_integer_sums_exact(small_golden):
    """the fast batch-1 kernel's integer object -- the exact
    combination S = sum_p 2^p P_p per (channel, group) -- equals the one
    formed from the REFERENCE's int32 staging values, bitwise."""
    from paper_2407_00088_b200 import _native as N
    n_checked = 0
    for name, c in small_golden.items():
        inst = small_inst(c)
        if inst["bits"] == 3:
            continue
        _, pw = make_pw(inst)
        P = c["partials"].astype(np.int64)               # (bits, n, m, NQ), the reference's
        for row in range(inst["a"].shape[0]):
            x = torch.from_numpy(inst["a"][row:row + 1]).cuda()
            t = N.build_lut(x, inst["group_size"], N.TABLE_Q8)
            _, S = N.lookup(pw.gpu, pw.scales, pw.zeros, *t, pw.m, pw.k, pw.bits, pw.group_size, N.TABLE_Q8,
                            N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | N.FLAG_COMBINED_PARTIALS, True)
            want = sum((1 << p) * P[p, row] for p in range(inst["bits"]))
            assert np.array_equal(S[0, 0].cpu().numpy().astype(np.int64), want), name
            n_checked += 1
    assert n_checked >= 8


@pytest.mark.parametrize("bits,gs", [(2, 64), (4, 128)])
def test_long_k_batch1_fast(bits, gs):
    """K = 28672 (Llama-2-70B down projection): fast batch-1 calls (the
    split-K cluster kernel) within 1e-5 of the oracle; exact path bitwise;
    the combined integer sums (gemv_b1_kernel) equal those formed from the
    exact kernel's per-plane staging values."""
    from paper_2407_00088_b200 import _native as N
    m, k = 4800, 28672
    g = torch.Generator(device="cuda").manual_seed(28672 + bits)
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
    sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
    x = torch.randn((1, k), device="cuda", generator=g).half()
    ref = O.mpgemm_q8(x.cpu().numpy(), q.cpu().numpy(), sc.float().cpu().numpy(), bits, gs)[0]
    y = B.mpgemm(x, pw, exact_epilogue=False)
    assert rel_maxnorm(y[0].cpu().numpy(), ref) <= 1e-5
    assert np.array_equal(B.mpgemm(x, pw).cpu().numpy()[0], ref)          # exact path, bitwise
    t = N.build_lut(x, gs, N.TABLE_Q8)
    fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | N.FLAG_COMBINED_PARTIALS
    _, S1 = N.lookup(pw.gpu, pw.scales, None, *t, m, k, bits, gs, N.TABLE_Q8, fl, True)
    _, P = N.lookup(pw.gpu, pw.scales, None, *t, m, k, bits, gs, N.TABLE_Q8, N.FLAG_PDL, True)   # exact kernel
    want = sum((1 << p) * P[0, p].long() for p in range(bits))
    assert torch.equal(S1[0, 0].long(), want)


@pytest.mark.parametrize("world,bits,gs", [(2, 2, 64), (4, 2, 64), (8, 4, 128), (3, 1, 128)])
def test_fused_allgather_epilogue_emulated(world, bits, gs):
    """bitlut_mpgemv_gather with `world` ranks emulated on one GPU (every
    rank's gathered row and flag local; launches in rank order, so no rank
    waits on another): after each epoch every rank's row equals the
    single-GPU fast result bitwise, and the flags count world per epoch."""
    from paper_2407_00088_b200 import parallel as PP
    m, k = 1024, 4096
    g = torch.Generator(device="cuda").manual_seed(world * 10 + bits)
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
    sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    qw = B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc)
    full = B.prepare_weights(qw)
    shards = [B.prepare_weights(PP.shard_quantized_weights(qw, r, world)) for r in range(world)]
    fgs = PP.FusedGather.emulated(m, world, torch.device("cuda"))
    for epoch in range(1, 3):
        x = torch.randn((1, k), device="cuda", generator=g).half()
        from paper_2407_00088_b200 import _native as N
        t = N.build_lut(x, gs, N.TABLE_Q8)
        want, _ = N.lookup(full.gpu, full.scales, None, *t, m, k, bits, gs, N.TABLE_Q8,
                           N.FLAG_PDL | N.FLAG_FAST_EPILOGUE, False)
        locs = [fg.launch(x[0], pw) for fg, pw in zip(fgs, shards)]
        rows = [fg.wait() for fg in fgs]
        torch.cuda.synchronize()
        ref = O.mpgemm_q8(x.cpu().numpy(), q.cpu().numpy(), sc.float().cpu().numpy(), bits, gs)[0]
        assert rel_maxnorm(rows[0][0].cpu().numpy(), ref) <= 1e-5      # the gathered row vs the oracle
        for r in range(world):
            assert torch.equal(rows[r], want), (r, epoch)
            col, mr = PP.gather_plan(m, world)[r]
            assert torch.equal(locs[r], want[:, col:col + mr])
            assert int(fgs[r].flag.item()) == epoch * world
            assert int(fgs[r].ticket.item()) == 0


@pytest.mark.parametrize("bits,gs,n,m,k", [(2, 64, 8, 512, 4096), (4, 128, 40, 256, 4096), (1, 128, 33, 512, 2048),
                                          (2, 128, 128, 352, 4096), (4, 64, 16, 128, 11008)])
def test_fast_mpgemm_rows(bits, gs, n, m, k):
    """Fast-epilogue mpGEMM (weight-stationary rows, lean rows kernel where it
    applies): every row within 1e-5 of the oracle, deterministic."""
    g = torch.Generator(device="cuda").manual_seed(n * 100 + bits + k)
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
    sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
    x = torch.randn((n, k), device="cuda", generator=g).half()
    y = B.mpgemm(x, pw, exact_epilogue=False)
    assert torch.equal(y, B.mpgemm(x, pw, exact_epilogue=False))
    ref = O.mpgemm_q8(x.cpu().numpy(), q.cpu().numpy(), sc.float().cpu().numpy(), bits, gs)
    yn = y.cpu().numpy()
    for r in range(n):
        assert rel_maxnorm(yn[r], ref[r]) <= 1e-5, r


@pytest.mark.parametrize("bits,gs,m,zeros", [(2, 64, 1024, False), (4, 128, 512, True), (1, 128, 2048, False)])
def test_long_k_cluster_kernel(bits, gs, m, zeros):
    """K = 28672 shards below the streaming kernel's size threshold run the
    split-K cluster kernel (DSMEM partial sums): within 1e-5 of the oracle,
    deterministic, and its integer sums equal the exact kernel's."""
    from paper_2407_00088_b200 import _native as N
    k = 28672
    g = torch.Generator(device="cuda").manual_seed(bits * 7 + m)
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
    sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    z = (torch.rand((m, k // gs), device="cuda", generator=g) * ((1 << bits) - 1)).half() if zeros else None
    pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc, zeros=z))
    x = torch.randn((1, k), device="cuda", generator=g).half()
    t = N.build_lut(x, gs, N.TABLE_Q8)
    fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE
    y, _ = N.lookup(pw.gpu, pw.scales, pw.zeros, *t, m, k, bits, gs, N.TABLE_Q8, fl, False)
    y2, _ = N.lookup(pw.gpu, pw.scales, pw.zeros, *t, m, k, bits, gs, N.TABLE_Q8, fl | N.FLAG_INDEPENDENT, False)
    assert torch.equal(y, y2)
    ref = O.mpgemm_q8(x.cpu().numpy(), q.cpu().numpy(), sc.float().cpu().numpy(), bits, gs,
                      zeros=None if z is None else z.cpu().numpy())[0]
    assert rel_maxnorm(y[0].cpu().numpy(), ref) <= 1e-5


def test_f16_fast_batch1_lean(config_golden):
    """Variant cuda-f16, batch 1, fast epilogue (16-bit block-fixed-point
    tables, BITLUT_TABLE_X16, in the lean kernel): BASELINE config 1 within
    1e-3 of the reference (scalar-real + zero correction) and no further from
    it than the reference-order fp16-table path, which it matches within the
    fp16 tables' own rounding (1e-3); deterministic; plus W2 / W1 / W4 shapes
    against the fp16-table path."""
    inst = W.config1()
    g = config_golden[inst["name"]]
    _, pw = make_pw(inst)
    yf = B.mpgemm(inst["a"], pw, variant="cuda-f16", exact_epilogue=False)[0]
    ye = B.mpgemm(inst["a"], pw, variant="cuda-f16")[0]
    rs = O.row_sums(inst["a"].astype(np.float32), inst["group_size"])
    ref = (g["y_scalar-real"][0] + O.zero_correction(inst["scales"], inst["zeros"], 4, rs[0])).astype(np.float32)
    assert rel_maxnorm(yf, ref) <= 1e-3, rel_maxnorm(yf, ref)
    assert rel_maxnorm(yf, ref) <= rel_maxnorm(ye, ref) + 1e-5, (rel_maxnorm(yf, ref), rel_maxnorm(ye, ref))
    assert rel_maxnorm(yf, ye) <= 1e-3, rel_maxnorm(yf, ye)
    assert np.array_equal(yf, B.mpgemm(inst["a"], pw, variant="cuda-f16", exact_epilogue=False)[0])
    gen = torch.Generator(device="cuda").manual_seed(16)
    for bits, gs, m, k in ((2, 64, 512, 4096), (1, 128, 1024, 4096), (4, 64, 256, 11008), (2, 32, 352, 2048)):
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=gen)
        sc = (torch.randn((m, k // gs), device="cuda", generator=gen).abs() * 0.02 + 1e-3).half()
        pw2 = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
        x = torch.randn((1, k), device="cuda", generator=gen).half()
        a = B.mpgemm(x, pw2, variant="cuda-f16", exact_epilogue=False)
        b = B.mpgemm(x, pw2, variant="cuda-f16")
        assert rel_maxnorm(a.cpu().numpy(), b.cpu().numpy()) <= 1e-3, (bits, gs, m, k)
        # against float64 arithmetic on the dequantized weights: closer than the fp16 tables
        wd = (q.double() - float(1 << (bits - 1))) * sc.double().repeat_interleave(gs, dim=1)
        ref64 = (wd @ x[0].double()).cpu().numpy()
        ea = np.abs(a.cpu().numpy()[0] - ref64).max() / np.abs(ref64).max()
        eb = np.abs(b.cpu().numpy()[0] - ref64).max() / np.abs(ref64).max()
        assert ea <= 1e-3 and ea <= eb + 1e-5, (bits, gs, m, k, ea, eb)


@pytest.mark.parametrize("bits,gs", [(2, 64), (4, 128), (1, 128)])
def test_multi_tab_launch_bitwise(bits, gs):
    """bitlut_mpgemv_multi_tab (matrices with their own activation tables in
    one launch, CTAs partitioned among them): every output == the per-matrix
    fast call, bitwise; the graph executor groups q,k,v,o,gate,up of a layer
    set (different tables) into one launch and matches per-op calls."""
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200.pipeline import Pipeline
    g = torch.Generator(device="cuda").manual_seed(bits * 3 + gs)
    k = 4096
    ms = (4096, 1024, 1024, 4096, 11008 // 32 * 32, 2048)
    pws, tabs = [], []
    for m in ms:
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
        pws.append(B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc)))
        tabs.append(N.build_lut(torch.randn((1, k), device="cuda", generator=g).half(), gs, N.TABLE_Q8))
    fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE
    outs = N.mpgemv_multi_tab([(p.gpu, p.scales, None, p.m, *t) for p, t in zip(pws, tabs)], k, bits, gs, fl)
    for p, t, o in zip(pws, tabs, outs):
        ref, _ = N.lookup(p.gpu, p.scales, None, *t, p.m, k, bits, gs, N.TABLE_Q8, fl, False)
        assert torch.equal(o, ref)
    # graph executor: one layer set of two layers, tables first (lookahead)
    xs = [[torch.randn((1, k), device="cuda", generator=g).half() for _ in range(3)] for _ in range(2)]
    pl = Pipeline(executor="graph")
    ts = [[pl.tables(x, gs) for x in row] for row in xs]
    ys = []
    for L in range(2):
        names = ("q", "k", "v", "o", "gate", "up")
        tix = (0, 0, 0, 1, 2, 2)
        ys.append([pl.lookup(pws[i], ts[L][tix[i]], fast_epilogue=True) for i in range(6)])
    plan = pl.plan_flags()
    assert any(f & 16 for f in plan)
    pl.compile()
    pl.run()
    torch.cuda.synchronize()
    for L in range(2):
        for i, tx in enumerate((0, 0, 0, 1, 2, 2)):
            ref = B.mpgemm(xs[L][tx], pws[i], exact_epilogue=False)
            assert torch.equal(ys[L][i].reshape(ref.shape), ref), (L, i)


@pytest.mark.parametrize("bits,gs,scale_dtype", [(2, 64, torch.float16), (4, 128, torch.float32),
                                                 (1, 128, torch.float16)])
def test_batch_executor_bitwise(bits, gs, scale_dtype):
    """Pipeline(executor="batch"): every table build in one launch
    (bitlut_build_lut_batch), one bitlut_mpgemv_batch launch per K over
    device-resident descriptors; outputs == per-call mpgemm (fast epilogue)
    bitwise, tables == bitlut_build_lut bitwise; matrices of several sizes,
    two K values, more CTAs than tiles (tiny matrices); dependent op lists
    rejected."""
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200.pipeline import Pipeline
    g = torch.Generator(device="cuda").manual_seed(bits * 7 + gs)
    shapes = [(4096, 4096), (1024, 4096), (32, 4096), (2048, 2816), (64, 2816), (11008 // 32 * 32, 4096)]
    pws = []
    for m, k in shapes:
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).to(scale_dtype)
        pws.append(B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc)))
    xs = [torch.randn((1, k), device="cuda", generator=g).half() for _, k in shapes]
    pl = Pipeline(executor="batch")
    ts = [pl.tables(x, gs) for x in xs]
    ys = [pl.lookup(p, t, fast_epilogue=True) for p, t in zip(pws, ts)]
    ys.append(pl.lookup(pws[0], ts[1] if shapes[1][1] == shapes[0][1] else ts[0], fast_epilogue=True))
    for y in ys:
        y.fill_(float("nan"))
    pl.compile()
    assert pl.n_launches() == 3
    for _ in range(2):                                  # graph replay is repeatable
        pl.run()
        torch.cuda.synchronize()
        for i, (x, p) in enumerate(zip(xs, pws)):
            ref = B.mpgemm(x, p, exact_epilogue=False)
            assert torch.equal(ys[i].reshape(ref.shape), ref), i
            t_ref = N.build_lut(x, gs, N.TABLE_Q8)
            for a, b in zip(ts[i].tensors, t_ref):
                assert torch.equal(a, b), i
        ref = B.mpgemm(xs[1], pws[0], exact_epilogue=False)
        assert torch.equal(ys[-1].reshape(ref.shape), ref)
    # dependencies between ops: not a batch
    bad = Pipeline(executor="batch")
    t0 = bad.tables(xs[0], gs)
    y0 = bad.lookup(pws[0], t0, fast_epilogue=True)
    bad.tables(xs[0], gs, deps=[bad.op_of(y0)])
    with pytest.raises(B.ParameterError):
        bad.compile()
    exact = Pipeline(executor="batch")
    exact.lookup(pws[0], exact.tables(xs[0], gs))
    with pytest.raises(B.ParameterError):
        exact.compile()


# ---- layer-set layout conversion (bitlut_layer_set_weights / _scales) ----

def _perm_mask(lane, nidx):
    m, o, n = 0, 1, nidx >> 1
    while n >= 1:
        if lane & o:
            m |= n
        o, n = o << 1, n >> 1
    return m


@pytest.mark.parametrize("m,k,bits,gs", [(64, 1024, 2, 64), (32, 2048, 1, 128), (64, 512, 4, 128),
                                         (32, 1376, 2, 32), (32, 1024, 4, 512), (64, 2752, 2, 64)])
def test_layer_set_conversion(m, k, bits, gs):
    """The batch executor's operand format against a numpy restatement of
    csrc/layout.cuh: nibble pos of lane l's chunk = nibble pos ^ (bits *
    cmask(l)) of the v2 chunk (an involution), and the unit-major scales."""
    from paper_2407_00088_b200 import _native as N
    g = torch.Generator(device="cuda").manual_seed(m + k + bits)
    nbytes = m * bits * k // 8
    w = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda", generator=g)
    w3 = N.layer_set_weights(w, bits, m, k, gs)
    assert torch.equal(N.layer_set_weights(w3, bits, m, k, gs), w)
    tch, R = 32 // bits, (8 if (gs // 4) % 8 == 0 else 4)
    KG, U = k // 4, k // 4 // R
    wn, w3n = w.cpu().numpy(), w3.cpu().numpy()
    nib = lambda a: np.stack([a & 15, a >> 4], axis=-1).reshape(a.shape[0], -1)   # noqa: E731
    rng = np.random.default_rng(0)
    for _ in range(64):                      # sampled chunks
        tile, kg = int(rng.integers(m // tch)), int(rng.integers(KG))
        u, r = kg // R, kg % R
        ub, l = u >> 5, u & 31
        nu_b = min(32, U - 32 * ub)
        off = tile * KG * 16 + ub * (32 * R * 16) + (r * nu_b + l) * 16
        a, b = nib(wn[off:off + 16][None])[0], nib(w3n[off:off + 16][None])[0]
        pm = bits * _perm_mask(l, tch)
        assert np.array_equal(b, a[np.arange(32) ^ pm])
    # scales: unit u of a tile holds scale[(tile*tch + (j ^ cmask(u & 31))), u // Lg], j < NCH
    Lg = (gs // 4) // R
    nacc = 8 if bits == 4 else 16
    nch = max(1, nacc // Lg) * (2 if bits == 1 else 1)
    for dt in (torch.float16, torch.float32):
        sc = torch.randn((m, k // gs), device="cuda", generator=g).to(dt)
        s3 = N.layer_set_scales(sc, bits, m, k, gs).cpu().numpy().reshape(m // tch, U, nch)
        scn = sc.cpu().numpy()
        uu = np.arange(U)
        for j in range(nch):
            c = j ^ np.array([_perm_mask(int(x) & 31, tch) for x in uu])
            for tile in range(m // tch):
                assert np.array_equal(s3[tile, :, j], scn[tile * tch + c, uu // Lg])


@pytest.mark.parametrize("bits,gs", [(4, 256), (4, 512), (2, 512), (2, 256), (1, 512), (1, 64), (2, 32), (4, 32),
                                     (2, 16), (4, 16), (1, 32)])
@pytest.mark.parametrize("zeros", [False, True])
def test_batch_executor_group_sizes(bits, gs, zeros):
    """The batch executor over every lanes-per-group class of the layer-set
    layout -- a group narrower than a lane's unit (R = 4), one to sixteen
    lanes per group, and groups spanning more lanes than a lane has
    accumulators (the per-unit scale vectors then repeat: 4-bit gs >= 256,
    2-bit gs = 512) -- with fp16 and fp32 scales, with and without zero
    points, K with a partial unit block: outputs == the per-call fast
    lookups on the v2 operand, bitwise, and the exported integer sums equal
    the exact kernel's staging values combined."""
    from paper_2407_00088_b200.pipeline import Pipeline
    g = torch.Generator(device="cuda").manual_seed(bits * 1000 + gs + int(zeros))
    k = 1536 if gs <= 512 and 1536 % gs == 0 else 2048
    shapes = [(96, k), (32, k), (256, 2 * k)]
    items = []
    for i, (m, kk) in enumerate(shapes):
        q = torch.randint(0, 1 << bits, (m, kk), dtype=torch.uint8, device="cuda", generator=g)
        sdt = torch.float16 if i != 1 else torch.float32
        sc = (torch.randn((m, kk // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).to(sdt)
        z = (torch.rand((m, kk // gs), device="cuda", generator=g) * ((1 << bits) - 1)).to(sdt) if zeros else None
        pw = B.prepare_weights(B.QuantizedWeights(m=m, k=kk, bits=bits, group_size=gs, qvalues=q, scales=sc, zeros=z))
        items.append((pw, torch.randn((1, kk), device="cuda", generator=g).half()))
    # scale dtypes differ -> separate launches; run each dtype group as its own pipeline
    for grp in ([items[0], items[2]], [items[1]]):
        pl = Pipeline(executor="batch")
        outs, parts = [], []
        for pw, x in grp:
            t = pl.tables(x, gs)
            p = torch.full((pw.m, pw.k // gs), -(1 << 30), dtype=torch.int32, device="cuda")
            outs.append(pl.lookup(pw, t, fast_epilogue=True, partials=p))
            parts.append(p)
        for o in outs:
            o.fill_(float("nan"))
        pl.compile()
        pl.run()
        torch.cuda.synchronize()
        for (pw, x), o, p in zip(grp, outs, parts):
            ref = B.mpgemm(x, pw, exact_epilogue=False)
            assert torch.equal(o.reshape(ref.shape), ref), (pw.m, pw.k)
            _, P = B.mpgemm(x, pw, return_partials=True)
            want = sum((1 << b) * P[0, b].to(torch.int64) for b in range(bits))
            assert torch.equal(p.to(torch.int64), want), (pw.m, pw.k)


@pytest.mark.parametrize("bits,gs,k", [(2, 64, 4096), (1, 128, 4096), (4, 128, 2048), (2, 64, 11008), (4, 32, 1536),
                                       (2, 16, 1024)])
def test_lookup_layer_set_operand(bits, gs, k):
    """bitlut_mpgemm with BITLUT_FLAG_LAYER_SET (the layer-set operand in the
    lean batch-1 and mpGEMM rows kernels: select-free reductions, scale
    vectors): outputs bitwise those of the v2 operand at batch 1 (with and
    without zero points) and over row blocks with an odd tail; BITLUT_ELAYOUT
    where those kernels do not apply."""
    from paper_2407_00088_b200 import _native as N
    g = torch.Generator(device="cuda").manual_seed(bits * 31 + gs + k)
    m = 416
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
    sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    z = (torch.rand((m, k // gs), device="cuda", generator=g) * ((1 << bits) - 1)).half()
    F = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE
    for zeros in (None, z):
        pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc,
                                                  zeros=zeros))
        lw, lsc, lz = pw.layer_set_operand()
        for n in ((1, 9, 16) if zeros is None else (1,)):
            x = torch.randn((n, k), device="cuda", generator=g).half()
            tabs = N.build_lut(x, gs, N.TABLE_Q8)
            ref, _ = N.lookup(pw.gpu, pw.scales, pw.zeros, *tabs, m, k, bits, gs, N.TABLE_Q8, F, False)
            out, _ = N.lookup(lw, lsc, lz, *tabs, m, k, bits, gs, N.TABLE_Q8, F | N.FLAG_LAYER_SET, False)
            assert torch.equal(out, ref), (zeros is not None, n)
            if n == 1:                        # the 16-bit block-fixed-point tables of cuda-f16 fast
                t16 = N.build_lut(x, gs, N.TABLE_X16)
                r16, _ = N.lookup(pw.gpu, pw.scales, pw.zeros, *t16, m, k, bits, gs, N.TABLE_X16, F, False)
                o16, _ = N.lookup(lw, lsc, lz, *t16, m, k, bits, gs, N.TABLE_X16, F | N.FLAG_LAYER_SET, False)
                assert torch.equal(o16, r16), (zeros is not None, "x16")
    with pytest.raises(B.LayoutError):       # exact epilogue: v2 operand only
        N.lookup(lw, lsc, lz, *tabs, m, k, bits, gs, N.TABLE_Q8, N.FLAG_PDL | N.FLAG_LAYER_SET, False)
    # mpgemm picks the cached layer-set operand for fast multi-row calls: same bits as without it
    pw0 = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
    x = torch.randn((12, k), device="cuda", generator=g).half()
    ref = B.mpgemm(x, pw0, exact_epilogue=False)
    pw0.layer_set_operand()
    assert torch.equal(B.mpgemm(x, pw0, exact_epilogue=False), ref)


def test_graph_executor_layer_set_operand():
    """The graph executor with PackedWeights that carry the layer-set operand
    (pw.layer_set_operand()): grouped launches over one table (q,k,v), over
    different tables, a dependent chain and a zero-point matrix all run the
    lean kernel's layer-set path (plan flag 64) and give the bits of the v2
    operand; an exact-epilogue lookup in the same list keeps v2."""
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200.pipeline import Pipeline
    g = torch.Generator(device="cuda").manual_seed(99)
    k, gs, bits = 2048, 64, 2

    def mk(m, zeros=False):
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
        z = (torch.rand((m, k // gs), device="cuda", generator=g) * 3).half() if zeros else None
        return B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc, zeros=z)

    qws = [mk(512), mk(256), mk(256), mk(1024), mk(128, zeros=True)]
    xs = [torch.randn((1, k), device="cuda", generator=g).half() for _ in range(3)]

    def run(use_ls):
        pws = [B.prepare_weights(qw) for qw in qws]
        if use_ls:
            for p in pws:
                p.layer_set_operand()
        pl = Pipeline()
        t0 = pl.tables(xs[0], gs)
        ys = [pl.lookup(p, t0, fast_epilogue=True) for p in pws[:3]]          # one table: grouped
        t1 = pl.tables(xs[1], gs, deps=[pl.op_of(y) for y in ys])              # chain
        ys.append(pl.lookup(pws[3], t1, fast_epilogue=True))
        t2 = pl.tables(xs[2], gs)
        ys.append(pl.lookup(pws[4], t2, fast_epilogue=True))                   # zero points
        ys.append(pl.lookup(pws[0], t2))                                       # exact: v2 operand
        pl.compile()
        flags = [f for f in pl.plan_flags() if f != -1]
        pl.run()
        torch.cuda.synchronize()
        return ys, flags, pws

    ref, f0, _ = run(False)
    out, f1, keep = run(True)
    assert not any(f & N.FLAG_LAYER_SET for f in f0)
    assert sum(1 for f in f1 if f & N.FLAG_LAYER_SET) == 5
    for a, b in zip(ref, out):
        assert torch.equal(a, b)
