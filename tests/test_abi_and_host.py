"""CPU-side checks: the C ABI library loads and exports every symbol the
header declares; host-side validation mirrors the reference's errors."""
import os
import re

import numpy as np
import pytest

import paper_2407_00088_b200 as B
from paper_2407_00088_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "bitlut_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(bitlut_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for name in ("bitlut_decompose_bits", "bitlut_pack_v1", "bitlut_unpack_v1",
                 "bitlut_repack_gpu", "bitlut_build_lut", "bitlut_precompute_lut",
                 "bitlut_quantize_tables", "bitlut_row_sums", "bitlut_mpgemm"):
        assert name in syms


def test_library_loads_and_exports_every_header_symbol():
    lib = N.lib()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(N.exported_symbols())
    assert b"sm_100a" in lib.bitlut_version()


def test_layout_query_without_gpu():
    lay = N.layout_query(4096, 4096, 2, 64)
    assert lay.bytes == 2 * 4096 * 4096 // 8
    assert (lay.tile_channels, lay.stream_groups, lay.unit_kg, lay.lanes_per_group) == (16, 1, 8, 2)
    lay3 = N.layout_query(96, 512, 3, 64)
    assert (lay3.tile_channels, lay3.stream_groups) == (32, 3)
    with pytest.raises(B.LayoutError):
        N.layout_query(40, 4096, 2, 64)          # m not a multiple of 32
    with pytest.raises(B.ParameterError):
        N.layout_query(4096, 4096, 5, 64)        # bits
    with pytest.raises(B.ParameterError):
        N.layout_query(4096, 4096, 2, 1024)      # packed accumulator bound


def test_quantized_weights_validation():
    q = np.zeros((4, 8), np.uint8)
    s = np.ones((4, 2), np.float32)
    B.QuantizedWeights(m=4, k=8, bits=2, group_size=4, qvalues=q, scales=s)
    with pytest.raises(B.ParameterError):
        B.QuantizedWeights(m=4, k=8, bits=5, group_size=4, qvalues=q, scales=s)
    with pytest.raises(B.LayoutError):
        B.QuantizedWeights(m=4, k=8, bits=2, group_size=3, qvalues=q, scales=s)
    with pytest.raises(B.ShapeError):
        B.QuantizedWeights(m=4, k=8, bits=2, group_size=4, qvalues=q, scales=s[:, :1])
    with pytest.raises(B.DataError):
        B.QuantizedWeights(m=4, k=8, bits=1, group_size=4, qvalues=q + 3, scales=s)
    bad = s.copy()
    bad[0, 0] = np.inf
    with pytest.raises(B.DataError):
        B.QuantizedWeights(m=4, k=8, bits=2, group_size=4, qvalues=q, scales=bad)
    with pytest.raises(B.ShapeError):
        B.QuantizedWeights(m=4, k=8, bits=2, group_size=4, qvalues=q, scales=s, zeros=s[:, :1])


def test_sign_and_ternary_constructors():
    sq = np.array([[1, 0, 1, 0]], np.uint8)
    qw = B.QuantizedWeights.sign_planes(sq, np.full((1, 1), 0.25, np.float16), 4)
    assert qw.bits == 1 and float(qw.scales[0, 0]) == 0.5 and float(qw.zeros[0, 0]) == 0.5
    t = B.QuantizedWeights.ternary(np.array([[-1, 0, 1, 1]], np.int8), np.ones((1, 1), np.float32), 4)
    assert t.bits == 2 and t.qvalues.tolist() == [[0, 1, 2, 2]] and float(t.zeros[0, 0]) == 1.0


def test_tile_config_and_bit_serial():
    with pytest.raises(B.LayoutError):
        B.TileConfig(m_tile=24, lanes=16)
    with pytest.raises(B.ParameterError):
        B.TileConfig(g=9)
    p = B.bit_serial_params(3)
    for v in range(8):
        assert p.reconstruct(v) == v


def test_variant_and_config_validation():
    with pytest.raises(B.ParameterError):
        B.kernel._variant("vector-q8")
    with pytest.raises(B.ParameterError):
        B.kernel._variant("nope")
    assert B.kernel._variant("cuda-q8") is B.KernelVariant.CUDA_Q8
    cfg = B.TileConfig(m_tile=16, k_tile=8, g=4, lanes=16)
    with pytest.raises(B.OverflowConfigError):
        B.validate_kernel_config(cfg, bits=4, group_size=(2**25) * 32, m=16, k=(2**25) * 32)
    with pytest.raises(B.ParameterError):
        B.validate_kernel_config(B.TileConfig(g=2, k_tile=128), bits=2, group_size=64, m=64, k=128)
    with pytest.raises(B.ParameterError):
        B.validate_kernel_config(B.DEFAULT_TILE, bits=2, group_size=48 * 4, m=64, k=192 * 4)


def test_status_mapping():
    from paper_2407_00088_b200.errors import raise_for_status
    raise_for_status(0, "ok")
    for rc, cls in ((-1, B.ParameterError), (-2, B.DataError), (-3, B.ShapeError),
                    (-4, B.LayoutError), (-5, B.OverflowConfigError), (-100, B.BitLutError)):
        with pytest.raises(cls):
            raise_for_status(rc, "x")


def test_graph_executor_independence_plan():
    """bitlut_pipeline_plan_flags (no GPU needed): lookups that read a table
    already complete when they start skip the start-of-kernel wait."""
    import ctypes
    from paper_2407_00088_b200.pipeline import PipeOpSpec, _bind
    T, LK = 0, 1

    def op(t, deps=(), fast=False):
        s = PipeOpSpec()
        s.type = t
        s.dep[:] = list(deps) + [-1] * (3 - len(deps))
        s.flags = N.FLAG_FAST_EPILOGUE if fast else 0
        return s

    # layer: T0 q k v | T4(q,k,v) o | T6(o) gate up | T9(gate,up) down | T11(down) q'
    ops = [op(T), op(LK, [0]), op(LK, [0]), op(LK, [0]), op(T, [1, 2, 3]), op(LK, [4]),
           op(T, [5]), op(LK, [6], fast=True), op(LK, [6], fast=True), op(T, [7, 8]), op(LK, [9]),
           op(T, [10]), op(LK, [11]), op(LK, []), op(LK, [1])]
    arr = (PipeOpSpec * len(ops))(*ops)
    fl = (ctypes.c_int * len(ops))()
    assert _bind().bitlut_pipeline_plan_flags(arr, len(ops), fl) == 0
    P, I, F = N.FLAG_PDL, N.FLAG_INDEPENDENT, N.FLAG_FAST_EPILOGUE
    assert list(fl) == [P, P, P | I, P | I, P, P, P, P | F, P | I | F, P, P, P, P,
                        P | I,      # no deps: inputs from before the list, complete once a kernel waited
                        P | I]      # dep 1 < last dependent lookup (12)
    bad = (PipeOpSpec * 2)(op(T), op(LK, [1]))
    assert _bind().bitlut_pipeline_plan_flags(bad, 2, fl) == -1


def test_graph_executor_table_fusion_plan():
    """Batch-1 fp16 table ops marked fusable whose consumers are all
    fast-epilogue lookups are folded into them (BITLUT_PLAN_SKIP / BITLUT_FLAG_FUSED_TABLES); the
    fused lookups inherit the table op's dependencies."""
    import ctypes
    from paper_2407_00088_b200.pipeline import PipeOpSpec, _bind
    T, LK = 0, 1
    SKIP, FUSED = -1, 8

    def tab(deps=(), n=1, dt=N.DT_F16, k=4096):
        s = PipeOpSpec()
        s.type, s.n, s.k, s.group_size, s.a_dtype = T, n, k, 64, dt
        s.flags = N.FLAG_FUSED_TABLES
        s.dep[:] = list(deps) + [-1] * (3 - len(deps))
        return s

    def look(deps, m=4096, k=4096, bits=2, fast=True):
        s = PipeOpSpec()
        s.type, s.n, s.k, s.group_size, s.m, s.bits = LK, 1, k, 64, m, bits
        s.scale_dtype = N.DT_F16
        s.flags = N.FLAG_FAST_EPILOGUE if fast else 0
        s.dep[:] = list(deps) + [-1] * (3 - len(deps))
        return s

    ops = [tab([]), look([0]), look([0]), look([0]),            # qkv: fused, table skipped
           tab([1, 2, 3]), look([4], fast=False),               # exact consumer: not fused
           tab([5]), look([6], bits=3, m=4096),                 # 3-bit consumer: not fused
           tab([7]), look([8]), look([8])]                      # gate/up: fused
    arr = (PipeOpSpec * len(ops))(*ops)
    fl = (ctypes.c_int * len(ops))()
    assert _bind().bitlut_pipeline_plan_flags(arr, len(ops), fl) == 0
    P, I, F = N.FLAG_PDL, N.FLAG_INDEPENDENT, N.FLAG_FAST_EPILOGUE
    assert list(fl) == [SKIP, P | FUSED | F,            # first kernel of the list waits
                        P | FUSED | F | I, P | FUSED | F | I,   # inputs from before the list: complete
                        P, P,
                        P, P | F,
                        SKIP, P | FUSED | F, P | FUSED | F | I]


def test_graph_executor_launch_grouping_plan():
    """Consecutive table builds share one launch; consecutive batch-1 fast
    lookups with equal K share one launch (same tables, or their own tables
    through bitlut_mpgemv_multi_tab); a group is INDEPENDENT only if all its
    members' inputs are complete."""
    import ctypes
    from paper_2407_00088_b200.pipeline import PipeOpSpec, _bind
    T, LK, J = 0, 1, 16

    def tab(k=4096):
        s = PipeOpSpec()
        s.type, s.n, s.k, s.group_size, s.a_dtype = T, 1, k, 64, N.DT_F16
        s.dep[:] = [-1, -1, -1]
        return s

    def look(dep, m, k=4096, fast=True):
        s = PipeOpSpec()
        s.type, s.n, s.k, s.group_size, s.m, s.bits = LK, 1, k, 64, m, 2
        s.scale_dtype = N.DT_F16
        s.flags = N.FLAG_FAST_EPILOGUE if fast else 0
        s.dep[:] = [dep, -1, -1]
        return s

    # layer-set order: four table builds, then q,k,v | o | gate,up | down
    ops = [tab(), tab(), tab(), tab(11008),
           look(0, 4096), look(0, 4096), look(0, 4096), look(1, 4096),
           look(2, 11008), look(2, 11008), look(3, 4096, k=11008), look(3, 4096, k=11008, fast=False)]
    arr = (PipeOpSpec * len(ops))(*ops)
    fl = (ctypes.c_int * len(ops))()
    assert _bind().bitlut_pipeline_plan_flags(arr, len(ops), fl) == 0
    P, I, F = N.FLAG_PDL, N.FLAG_INDEPENDENT, N.FLAG_FAST_EPILOGUE
    assert list(fl) == [P, P | J, P | J, P | J,            # one table launch (first kernel: waits)
                        P | F, P | F | J, P | F | J,       # q,k,v,o,gate,up (K = 4096, fast, three
                        P | F | J,                         # different tables) in ONE launch, which
                        P | F | J, P | F | J,              # waits for the table launch
                        P | F | I,                         # down (K = 11008): tables complete
                        P | I]                             # exact epilogue: own launch
