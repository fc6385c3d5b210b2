"""Fused table-build + lookup vs separate launches (diagnostic): CUDA graph
of PDL-chained batch-1 GEMVs rotating over weight copies > L2.
  sep    build_lut + lookup (dependent)           2 launches per GEMV
  fused  mpgemv_fused (dependent)                 1 launch
  fusedI mpgemv_fused (INDEPENDENT)               1 launch
  lookI  lookup only, tables prebuilt (INDEPENDENT)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
bits, gs = 2, 64
F = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE
for (m, k) in ((4096, 4096), (11008, 4096), (4096, 11008)):
    nbytes = bits * m * k // 8
    copies = max(8, (600 << 20) // nbytes)
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device=dev, generator=g)
    s = (torch.randn((m, k // gs), device=dev, generator=g).abs() * 0.02 + 1e-3).half()
    pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=s))
    ws = [pw.gpu.clone() for _ in range(copies)]
    x = torch.randn((1, k), device=dev, generator=g).half()
    tabs = N.build_lut(x, gs, N.TABLE_Q8)
    modes = {
        "sep": lambda w: N.lookup(w, pw.scales, None, *N.build_lut(x, gs, N.TABLE_Q8, N.FLAG_PDL), m, k, bits,
                                  gs, N.TABLE_Q8, F, False),
        "fused": lambda w: N.mpgemv_fused(x, w, pw.scales, None, m, k, bits, gs, F),
        "fusedI": lambda w: N.mpgemv_fused(x, w, pw.scales, None, m, k, bits, gs, F | N.FLAG_INDEPENDENT),
        "lookI": lambda w: N.lookup(w, pw.scales, None, *tabs, m, k, bits, gs, N.TABLE_Q8,
                                    F | N.FLAG_INDEPENDENT, False),
    }
    res = {}
    for name, fn in modes.items():
        def body():
            for w in ws:
                fn(w)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            body()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                body()
            for _ in range(3):
                gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                gr.replay()
            e1.record(st)
            torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) * 1e3 / 10 / len(ws)
    print(f"{m}x{k}: " + "  ".join(f"{n} {v:.3f} us" for n, v in res.items()), flush=True)
