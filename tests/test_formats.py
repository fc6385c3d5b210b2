"""Containers (paper_2407_00088_b200/formats.py) against files written by
the REAL reference (tests/golden/formats/, oracle/make_golden_formats.py):
byte-identical LMRM / LMQW / LMPW v1 writers, the reference's validation
errors, and (GPU) the LMPW v2 GPU-layout round trip and the CLI."""
import json
import os
import struct

import numpy as np
import pytest
import torch

import paper_2407_00088_b200 as B
from paper_2407_00088_b200 import formats as F
from paper_2407_00088_b200 import workloads as W
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")
CASES = json.load(open(os.path.join(GOLD, "index.json")))


def golden(name, ext):
    return open(os.path.join(GOLD, name + ext), "rb").read()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_lmqw_lmrm_byte_identical(tmp_path, case):
    qw = F.read_quantized(os.path.join(GOLD, case["name"] + ".lmqw"))
    inst = W.small_instance(case["seed"], case["m"], case["k"], case["bits"], case["group_size"])
    assert np.array_equal(np.asarray(qw.qvalues), inst["q"])
    F.write_quantized(tmp_path / "q.lmqw", qw)
    assert (tmp_path / "q.lmqw").read_bytes() == golden(case["name"], ".lmqw")
    mat = F.read_matrix(os.path.join(GOLD, case["name"] + "_a.lmrm"))
    F.write_matrix(tmp_path / "a.lmrm", mat)
    assert (tmp_path / "a.lmrm").read_bytes() == golden(case["name"], "_a.lmrm")


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_lmpw_v1_reference_stream(case):
    """Decode the reference's stream on the CPU (no GPU layout) and
    re-encode it byte for byte; the planes equal the oracle's v1 packing."""
    data = golden(case["name"], ".lmpw")
    pw = F.deserialize(data, device="cpu", gpu=False)
    assert F.serialize(pw) == data
    inst = W.small_instance(case["seed"], case["m"], case["k"], case["bits"], case["group_size"])
    planes = O.pack_v1(O.decompose_bits(inst["q"], case["bits"], case["g"]), 32, 128, case["g"], 16)
    assert np.array_equal(pw.planes.numpy(), planes)


def test_lmpw_errors():
    data = golden(CASES[0]["name"], ".lmpw")
    with pytest.raises(B.BitLutError) as e:
        F.deserialize(b"XXXX" + data[4:], device="cpu", gpu=False)
    assert e.value.code == "EMAGIC"
    with pytest.raises(B.BitLutError) as e:
        F.deserialize(data[:30], device="cpu", gpu=False)
    assert e.value.code == "ETRUNC"
    with pytest.raises(B.BitLutError) as e:
        F.deserialize(data[:4] + struct.pack("<I", 9) + data[8:], device="cpu", gpu=False)
    assert e.value.code == "EVERSION"
    with pytest.raises(B.BitLutError) as e:         # layout version
        F.deserialize(data[:8] + struct.pack("<I", 7) + data[12:], device="cpu", gpu=False)
    assert e.value.code == "EVERSION"
    with pytest.raises(B.BitLutError) as e:         # scale count disagrees
        F.deserialize(data[:48] + struct.pack("<I", 3) + data[52:], device="cpu", gpu=False)
    assert e.value.code == "ELENGTH"
    with pytest.raises(B.BitLutError) as e:
        F.deserialize(data[:-1], device="cpu", gpu=False)
    assert e.value.code == "ETRUNC"
    with pytest.raises(B.BitLutError) as e:
        F.deserialize(data + b"\0", device="cpu", gpu=False)
    assert e.value.code == "ELENGTH"
    import tempfile
    q = golden(CASES[0]["name"], ".lmqw")
    with tempfile.NamedTemporaryFile(suffix=".lmqw") as f:
        f.write(q[:-2])
        f.flush()
        with pytest.raises(B.BitLutError) as e:
            F.read_quantized(f.name)
    assert e.value.code == "ETRUNC"


def test_cli_parser_and_error_convention(capsys):
    from paper_2407_00088_b200 import cli
    assert cli.main(["nmse", "--shape", "12x"]) == 2
    assert "error:EPARAM:" in capsys.readouterr().err
    for cmd in ("quantize", "prepack", "bench", "nmse"):
        with pytest.raises(SystemExit):
            cli.build_parser().parse_args([cmd, "--help"])


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_lmpw_v1_from_gpu_pack(case):
    """prepare_weights on the GPU + serialize == the reference's file; the
    reference's file decodes to a usable GPU operand (g = 4)."""
    qw = F.read_quantized(os.path.join(GOLD, case["name"] + ".lmqw"))
    tile = B.TileConfig(n_tile=1, m_tile=32, k_tile=128, g=case["g"], lanes=16)
    pw = B.prepare_weights(qw, tile)
    data = golden(case["name"], ".lmpw")
    assert F.serialize(pw) == data
    back = F.deserialize(data)
    if case["g"] == 4:
        assert back.gpu is not None and torch.equal(back.gpu, pw.gpu)
        a = np.asarray(F.read_matrix(os.path.join(GOLD, case["name"] + "_a.lmrm")).to_array())
        assert np.array_equal(B.mpgemm(a, back), B.mpgemm(a, pw))


@pytest.mark.gpu
@pytest.mark.parametrize("bits,zeros,f16", [(2, False, True), (4, True, True), (1, False, False),
                                            (3, True, False)])
def test_lmpw_v2_gpu_round_trip(bits, zeros, f16):
    inst = W.small_instance(77 + bits, 128, 512, bits, 64, zeros=zeros)
    sc = inst["scales"] if f16 else inst["scales"].astype(np.float32)
    qw = B.QuantizedWeights(m=128, k=512, bits=bits, group_size=64, qvalues=inst["q"], scales=sc,
                            zeros=inst["zeros"])
    pw = B.prepare_weights(qw)
    data = F.serialize(pw, 2)
    back = F.deserialize(data)
    assert torch.equal(back.gpu, pw.gpu) and torch.equal(back.planes, pw.planes)
    assert back.scales.dtype == pw.scales.dtype and torch.equal(back.scales, pw.scales)
    assert (back.zeros is None) == (pw.zeros is None)
    a = inst["a"]
    assert np.array_equal(B.mpgemm(a, back), B.mpgemm(a, pw))
    with pytest.raises(B.BitLutError) as e:
        F.deserialize(data[:-3])
    assert e.value.code == "ETRUNC"


@pytest.mark.gpu
def test_cli_commands(tmp_path, capsys):
    """quantize -> prepack (both formats, --verify) -> bench (schema-valid) -> nmse."""
    import jsonschema
    from paper_2407_00088_b200 import cli
    rng = np.random.default_rng(3)
    F.write_matrix(tmp_path / "w.lmrm", rng.standard_normal((256, 1024)).astype(np.float32))
    assert cli.main(["quantize", str(tmp_path / "w.lmrm"), "-o", str(tmp_path / "w.lmqw"), "--bits", "4",
                     "--group-size", "128", "--json"]) == 0
    q = json.loads(capsys.readouterr().out)
    assert 0 < q["weight_nmse"] < 0.02
    for fmt in (1, 2):
        out = tmp_path / f"w{fmt}.lmpw"
        assert cli.main(["prepack", str(tmp_path / "w.lmqw"), "-o", str(out), "--format", str(fmt),
                         "--verify", "--json"]) == 0
        assert json.loads(capsys.readouterr().out)["verified"] is True
    assert cli.main(["bench", str(tmp_path / "w1.lmpw"), str(tmp_path / "w2.lmpw"), "--reps", "3",
                     "--json"]) == 0
    rep = json.loads(capsys.readouterr().out)
    schema = json.load(open(os.path.join(os.path.dirname(B.__file__), "schemas", "bench_report.schema.json")))
    jsonschema.validate(rep, schema)
    assert cli.main(["nmse", "--shape", "256x1024x2", "--bits", "4", "--group-size", "128", "--json"]) == 0
    nm = json.loads(capsys.readouterr().out)
    for r in nm["variants"]:                # the LUT paths add little error to the quantization's own
        assert r["nmse"] < nm["baseline_nmse"] * 1.5 + 1e-4, r
