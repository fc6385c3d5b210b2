"""Per-CTA timeline of back-to-back lookup kernels (diagnostic).

Captures R traced lookups of one shape (rotating over distinct weight
buffers > L2) in a CUDA graph with PDL, replays it, and prints per-launch
phase timings from %globaltimer stamps (csrc/gemv.cu TRACE slots):
  0 start, 1 loads issued, 2 after griddepcontrol.wait, 3 tables staged,
  4 lookups done, 5 epilogue products, 6 end, 7 smid.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--bits", type=int, default=2)
ap.add_argument("--gs", type=int, default=64)
ap.add_argument("--bufs", type=int, default=64)
ap.add_argument("--reps", type=int, default=16)
ap.add_argument("--pdl", type=int, default=1)
ap.add_argument("--indep", type=int, default=0)
args = ap.parse_args()

g = torch.Generator(device="cuda").manual_seed(0)
pws = []
for _ in range(args.bufs):
    q = torch.randint(0, 1 << args.bits, (args.m, args.k), dtype=torch.uint8, device="cuda", generator=g)
    s = (torch.randn((args.m, args.k // args.gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    pws.append(B.prepare_weights(B.QuantizedWeights(m=args.m, k=args.k, bits=args.bits,
                                                    group_size=args.gs, qvalues=q, scales=s)))
a = torch.randn((1, args.k), device="cuda", generator=g).half()
t, ts, rs = N.build_lut(a, args.gs, N.TABLE_Q8)
lay = N.layout_query(args.m, args.k, args.bits, args.gs)
grid = args.m // lay.tile_channels
traces = torch.zeros((args.reps, grid, 8), dtype=torch.int64, device="cuda")
outs = torch.empty((args.reps, 1, args.m), dtype=torch.float32, device="cuda")
L = N.lib()
stream = torch.cuda.Stream()


def run():
    st = ctypes.c_void_p(stream.cuda_stream)
    for r in range(args.reps):
        pw = pws[r % len(pws)]
        rc = L.bitlut_mpgemm_traced(N.ptr(pw.gpu), pw.m, pw.k, pw.bits, pw.group_size, N.ptr(pw.scales),
                                    None, N.DT_F16, N.ptr(t), N.ptr(ts), N.ptr(rs), N.TABLE_Q8, 1,
                                    N.ptr(outs[r]), None, (N.FLAG_PDL if args.pdl else 0) | (N.FLAG_INDEPENDENT if args.indep and r > 0 else 0),
                                    N.ptr(traces[r]), st)
        assert rc == 0


with torch.cuda.stream(stream):
    run()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        run()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    gr.replay()
    e1.record(stream)
torch.cuda.synchronize()
print(f"shape {args.m}x{args.k} W{args.bits} g{args.gs}: grid {grid}, {args.reps} launches, "
      f"{e0.elapsed_time(e1) * 1e3 / args.reps:.2f} us/launch (graph, pdl={args.pdl})")
tr = traces.cpu().numpy().astype(np.int64)
t0 = tr[:, :, 0].min()
names = ["issue", "wait", "tables", "lookups", "terms", "chain+out"]
print("launch  first_start  last_start  first_end  last_end   med phase durations (ns): " + " ".join(names))
for r in range(args.reps):
    x = tr[r]
    d = [np.median(x[:, i + 1] - x[:, i]) for i in range(6)]
    print(f"{r:4d} {x[:, 0].min() - t0:11d} {x[:, 0].max() - t0:11d} {x[:, 6].min() - t0:10d} "
          f"{x[:, 6].max() - t0:9d}   " + " ".join(f"{v:7.0f}" for v in d))
sm = tr[:, :, 7]
print("CTAs per SM (launch 0): max", np.bincount(sm[0]).max(), "SMs used", len(np.unique(sm[0])))
