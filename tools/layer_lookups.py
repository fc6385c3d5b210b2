"""The headline step's lookups alone (tables prebuilt), issued three ways
(diagnostic): 224 per-GEMV launches, 4 grouped launches per layer (same
tables), 2 grouped launches per layer (per-matrix tables).  CUDA graph,
overlapped (INDEPENDENT) launches, CUDA events; prints ms per step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

dev = torch.device("cuda", 0)
L = int(os.environ.get("LAYERS", "32"))
layers = bench.build_layers(L, 2, 64, 0, 1, dev)
acts, _ = bench.make_acts(L, dev)
tabs = [{g: N.build_lut(a[g], 64, N.TABLE_Q8) for g in a} for a in acts]
fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | N.FLAG_INDEPENDENT
grp = {"q": "attn", "k": "attn", "v": "attn", "o": "o", "gate": "mlp", "up": "mlp", "down": "down"}
st = torch.cuda.Stream()


def per_gemv():
    for Ly, T in zip(layers, tabs):
        for nm, pw in Ly.items():
            N.lookup(pw.gpu, pw.scales, None, *T[grp[nm]], pw.m, pw.k, 2, 64, N.TABLE_Q8, fl, False)


def grouped4():
    for Ly, T in zip(layers, tabs):
        N.mpgemv_multi([(Ly[n].gpu, Ly[n].scales, None, Ly[n].m) for n in ("q", "k", "v")], *T["attn"], 4096, 2,
                       64, fl)
        N.lookup(Ly["o"].gpu, Ly["o"].scales, None, *T["o"], Ly["o"].m, 4096, 2, 64, N.TABLE_Q8, fl, False)
        N.mpgemv_multi([(Ly[n].gpu, Ly[n].scales, None, Ly[n].m) for n in ("gate", "up")], *T["mlp"], 4096, 2,
                       64, fl)
        d = Ly["down"]
        N.lookup(d.gpu, d.scales, None, *T["down"], d.m, d.k, 2, 64, N.TABLE_Q8, fl, False)


def grouped2():
    for Ly, T in zip(layers, tabs):
        N.mpgemv_multi_tab([(Ly[n].gpu, Ly[n].scales, None, Ly[n].m, *T[grp[n]])
                            for n in ("q", "k", "v", "o", "gate", "up")], 4096, 2, 64, fl)
        d = Ly["down"]
        N.lookup(d.gpu, d.scales, None, *T["down"], d.m, d.k, 2, 64, N.TABLE_Q8, fl, False)


for name, fn in (("per_gemv", per_gemv), ("grouped4", grouped4), ("grouped2", grouped2)):
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name}: {ms:.4f} ms/step  {bench.packed_bytes_full(L, 2) / ms / 1e9:.1f} GB/s", flush=True)
