"""The headline step (layer set, graph executor, fast epilogue) at several
table-build lookaheads D, plus the table builds alone (diagnostic: how much
of the step the table launches cost).  CUDA graph replays, CUDA events."""
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
st = torch.cuda.Stream()
total = bench.packed_bytes_full(L, 2)


def timed(fn, reps=30):
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for D in [int(x) for x in os.environ.get("DS", "1,2,4,8,16,32").split(",")]:
    pl, outs, arena = bench.build_pipeline(layers, acts, fast=True, executor="graph", chain=False, lookahead=D)
    ms = timed(pl.run)
    print(f"lookahead {D:2d}: {ms:.4f} ms/step  {total / ms / 1e6:.1f} GB/s  launches {pl.n_launches()}",
          flush=True)

# batch executor: one table launch + one lookup launch per K; bitwise check
ref, ref_arena = None, None
pl, outs, ref_arena = bench.build_pipeline(layers, acts, fast=True, executor="graph", chain=False, lookahead=8)
pl.run(st)
torch.cuda.synchronize()
ref = ref_arena.clone()
pb, outs_b, arena_b = bench.build_pipeline(layers, acts, fast=True, executor="batch", chain=False)
arena_b.fill_(float("nan"))
pb.run(st)
torch.cuda.synchronize()
print("batch == graph bitwise:", bool(torch.equal(arena_b, ref)), flush=True)
ms = timed(pb.run)
print(f"batch: {ms:.4f} ms/step  {total / ms / 1e6:.1f} GB/s  launches {pb.n_launches()}", flush=True)

# table builds alone (consecutive builds grouped, up to 8 per launch)
from paper_2407_00088_b200.pipeline import Pipeline  # noqa: E402
tp = Pipeline(executor="graph")
for a in acts:
    for g in a:
        tp.tables(a[g], 64)
tp.compile()
print(f"tables only ({tp.n_launches()} launches): {timed(tp.run):.4f} ms/step", flush=True)
