"""Per-shape lookup latency (diagnostic, A/B between library builds via
BITLUT_B200_LIB): for each Llama-2-7B shape, a CUDA graph of PDL-chained
lookup launches rotating over enough weight copies to exceed L2, dependent
(wait at start) and INDEPENDENT; prints us per launch."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=2)
ap.add_argument("--gs", type=int, default=64)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--fast", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ls", type=int, default=0, help="1: layer-set operand (BITLUT_FLAG_LAYER_SET)")
ap.add_argument("--shapes", default="4096x4096,11008x4096,4096x11008")
args = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
print("lib", N.LIB_PATH)
for (m, k) in (tuple(int(v) for v in sh.split("x")) for sh in args.shapes.split(",")):
    nbytes = args.bits * m * k // 8
    copies = max(4, (600 << 20) // nbytes)
    q = torch.randint(0, 1 << args.bits, (m, k), dtype=torch.uint8, device=dev, generator=g)
    s = (torch.randn((m, k // args.gs), device=dev, generator=g).abs() * 0.02 + 1e-3).half()
    pw0 = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=args.bits, group_size=args.gs,
                                               qvalues=q, scales=s))
    w0, sc0 = pw0.gpu, pw0.scales
    if args.ls:
        w0, sc0, _ = pw0.layer_set_operand()
    ws = [w0.clone() for _ in range(copies)]
    x = torch.randn((args.n, k), device=dev, generator=g).half()
    tabs = N.build_lut(x, args.gs, N.TABLE_Q8)
    res = {}
    for mode, fl in (("dep", N.FLAG_PDL), ("indep", N.FLAG_PDL | N.FLAG_INDEPENDENT)):
        fl |= N.FLAG_FAST_EPILOGUE if args.fast else 0
        fl |= N.FLAG_LAYER_SET if args.ls else 0

        def body():
            for w in ws:
                N.lookup(w, sc0, None, *tabs, m, k, args.bits, args.gs, N.TABLE_Q8, fl, False)
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
            for _ in range(args.reps):
                gr.replay()
            e1.record(st)
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / args.reps / len(ws)
        res[mode] = us
    print(f"{m}x{k} n={args.n}: dep {res['dep']:.3f} us ({nbytes / res['dep'] / 1e3:.0f} GB/s)  "
          f"indep {res['indep']:.3f} us ({nbytes / res['indep'] / 1e3:.0f} GB/s)", flush=True)
