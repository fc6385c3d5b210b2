"""The headline step through the batch executor (diagnostic / profiling
target): LAYERS layers (default 32) of the Llama-2-7B layer set, BITS/GS
(default W2 g64),
int8 tables, fast epilogue; runs the step RUNS times (default 3) eagerly,
so ncu sees: table batch, lookup batch (K = 4096), lookup batch (K = 11008)
per run."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
L = int(os.environ.get("LAYERS", "32"))
BITS, GS = int(os.environ.get("BITS", "2")), int(os.environ.get("GS", "64"))
layers = bench.build_layers(L, BITS, GS, 0, 1, dev)
acts, _ = bench.make_acts(L, dev)
pl, outs, arena = bench.build_pipeline(layers, acts, fast=True, executor="batch", chain=False)
st = torch.cuda.Stream()
for _ in range(int(os.environ.get("RUNS", "3"))):
    pl.run_eager(st)
torch.cuda.synchronize()
print("algorithmic bytes per step:", bench.packed_bytes_full(L, BITS))
