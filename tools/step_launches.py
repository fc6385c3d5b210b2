"""Driver for the ncu launch list of the headline step (diagnostic): the
layer-set op list (bench.py build_pipeline, chain=False, fast epilogue) for
--layers layers, replayed --reps times.  Only this executor runs, so the
launch list holds exactly the step's kernels (plus weight-prep setup)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--chain", type=int, default=0)
ap.add_argument("--fast", type=int, default=1)
args = ap.parse_args()
dev = torch.device("cuda", 0)
layers = bench.build_layers(args.layers, 2, 64, 0, 1, dev)
acts, _ = bench.make_acts(args.layers, dev)
pl, _, _ = bench.build_pipeline(layers, acts, fast=bool(args.fast), executor="graph", chain=bool(args.chain))
torch.cuda.synchronize()
for _ in range(args.reps):
    pl.run()
torch.cuda.synchronize()
print("ok")
