"""Batch executor per K: the W2 g64 layer set's K = 4096 matrices (q,k,v,o,
gate,up) and K = 11008 matrices (down) as separate steps: lookups-only GB/s
and fraction of the HBM peak (diagnostic)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
st = torch.cuda.Stream(dev)
peak, _ = bench.load_peaks()
acts, _ = bench.make_acts(32, dev)
L = bench.build_layers(32, 2, 64, 0, 1, dev)
res = {}
for label, groups in (("k4096", [g[0] for g in bench.LUT_GROUPS if g[1] == 4096]),
                      ("k11008", [g[0] for g in bench.LUT_GROUPS if g[1] != 4096])):
    pl, _, _ = bench.build_pipeline(L, acts, fast=True, executor="batch", chain=False, groups=groups)
    pl.run(st)
    torch.cuda.synchronize()
    g = bench.capture(lambda: pl._launch_lookups(st), st)
    with torch.cuda.stream(st):
        ms = bench.time_graph(g, 30, 5)
    nb = sum(L[0][nm].packed_bytes for gr in bench.LUT_GROUPS if gr[0] in groups for nm in gr[2]) * 32
    res[label] = {"ms": round(ms, 4), "GBps": round(nb / ms / 1e6, 1), "frac": round(nb / ms / 1e6 / peak, 4)}
print(json.dumps(res))
