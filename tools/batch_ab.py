"""A/B of the batch executor on the 32-layer Llama-2-7B layer sets (W2 g64,
W4 g128, W1 g128, W1 sign, W2 ternary): lookup launches only (tables
prebuilt) and the whole step, ms and fraction of the HBM peak.

    BITLUT_BATCH_STAGES=2 python tools/batch_ab.py [label]
"""
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
res = {"label": sys.argv[1] if len(sys.argv) > 1 else os.environ.get("BITLUT_BATCH_STAGES", "default")}
sets = [("W2_g64", 2, 64, "offset"), ("W4_g128", 4, 128, "offset"), ("W1_g128", 1, 128, "offset"),
        ("W1_sign", 1, 128, "sign"), ("W2_ternary", 2, 128, "ternary")]
only = os.environ.get("SETS")
for label, b, gs, enc in sets:
    if only and label not in only.split(","):
        continue
    kw = {} if enc == "offset" else {"encoding": enc}
    L = bench.build_layers(32, b, gs, 0, 1, dev, seed=20251020 + b, **kw)
    pl, _, _ = bench.build_pipeline(L, acts, fast=True, executor="batch", chain=False)
    with torch.cuda.stream(st):
        for _ in range(5):
            pl.run(st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(30):
            pl.run(st)
        e1.record(st)
        torch.cuda.synchronize()
        ms_step = e0.elapsed_time(e1) / 30
    pl.run(st)
    torch.cuda.synchronize()
    g = bench.capture(lambda: pl._launch_lookups(st), st)
    with torch.cuda.stream(st):
        ms_look = bench.time_graph(g, 30, 5)
    nb = bench.packed_bytes_full(32, b)
    res[label] = {"step_frac": round(nb / (ms_step * 1e-3) / 1e9 / peak, 4),
                  "lookups_frac": round(nb / (ms_look * 1e-3) / 1e9 / peak, 4),
                  "step_ms": round(ms_step, 4), "lookups_ms": round(ms_look, 4)}
    del pl, L, g
    torch.cuda.empty_cache()
print(json.dumps(res))
