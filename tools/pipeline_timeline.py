"""Per-op timeline of the persistent pipeline (diagnostic).

Builds the bench step for --layers Llama-2-7B layers, runs the traced
pipeline and prints, per op: unit count, when its first unit started, when
its dependencies were met (first/last unit), when the last unit finished,
relative to the launch start (us)."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402
from paper_2407_00088_b200.pipeline import _bind  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--fast", type=int, default=0)
args = ap.parse_args()
dev = torch.device("cuda", 0)
layers = bench.build_layers(args.layers, 2, 64, 0, 1, dev)
acts, _ = bench.make_acts(args.layers, dev)
pl, _, _ = bench.build_pipeline(layers, acts, fast=bool(args.fast))
# per-op unit counts (mirror of bitlut_pipeline_encode)
units = []
for s in pl.specs:
    if s.type == 0:
        units.append(((s.k // 4 + 127) // 128) * s.n)
    else:
        lay = N.layout_query(s.m, s.k, s.bits, s.group_size)
        units.append((s.m // lay.tile_channels) * s.n)
base = np.concatenate([[0], np.cumsum(units)[:-1]]).astype(np.int32)
ub = torch.from_numpy(base).to(dev)
trace = torch.zeros((int(sum(units)), 4), dtype=torch.int64, device=dev)
L = _bind()
L.bitlut_pipeline_launch_traced.restype = ctypes.c_int
L.bitlut_pipeline_launch_traced.argtypes = [ctypes.c_void_p] * 6
for rep in range(3):
    trace.zero_()
    st = torch.cuda.current_stream()
    rc = L.bitlut_pipeline_launch_traced(ctypes.c_void_p(pl._host.data_ptr()), ctypes.c_void_p(pl._dev.data_ptr()),
                                         ctypes.c_void_p(pl._counters.data_ptr()), ctypes.c_void_p(trace.data_ptr()),
                                         ctypes.c_void_p(ub.data_ptr()), ctypes.c_void_p(st.cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
t = trace.cpu().numpy().astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
names = []
for L_ in range(args.layers):
    for g, _, nm in bench.LUT_GROUPS:
        names.append(f"L{L_}.lut_{g}")
        names += [f"L{L_}.{x}" for x in nm]
print(f"{'op':14s} {'units':>5s} {'start':>8s} {'dep_first':>9s} {'dep_last':>9s} {'stage_med':>9s} {'end_last':>9s}  (us)")
for i, (nm, b, n) in enumerate(zip(names, base, units)):
    x = t[b:b + n]
    print(f"{nm:14s} {n:5d} {(x[:,0].min()-t0)/1e3:8.2f} {(x[:,1].min()-t0)/1e3:9.2f} {(x[:,1].max()-t0)/1e3:9.2f} "
          f"{np.median(x[:,2]-x[:,1])/1e3:9.2f} {(x[:,3].max()-t0)/1e3:9.2f}   compute_med {np.median(x[:,3]-x[:,2])/1e3:6.2f}")
print("total us", (t[:, 3].max() - t0) / 1e3)
