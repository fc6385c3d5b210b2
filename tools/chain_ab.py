"""Decode chain / graph-executor A/B (32 Llama-2-7B W2 g64 layers): ms per
step of the dependent decode chain (fast and exact epilogues) and of the
layer set through the graph executor.

    BITLUT_L2_PREFETCH=0 python tools/chain_ab.py [label]
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
L = bench.build_layers(32, 2, 64, 0, 1, dev)
acts, _ = bench.make_acts(32, dev)
if os.environ.get("CHAIN_LAYER_SET", "1") == "1":       # the lean kernels' layer-set operand (second weight copy)
    for layer in L:
        for pw in layer.values():
            pw.layer_set_operand()
res = {"label": sys.argv[1] if len(sys.argv) > 1 else os.environ.get("BITLUT_L2_PREFETCH", "1")}
nb = bench.packed_bytes_full(32, 2)
for name, fast, chain, ex in (("decode_chain_fast", True, True, "graph"),
                              ("decode_chain_exact", False, True, "graph"), ("layer_set_graph_fast", True, False, "graph")):
    pl, _, _ = bench.build_pipeline(L, acts, fast=fast, executor=ex, chain=chain)
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
    ms = e0.elapsed_time(e1) / 30
    res[name] = {"ms": round(ms, 4), "GBps": round(nb / (ms * 1e-3) / 1e9, 1)}
print(json.dumps(res))
