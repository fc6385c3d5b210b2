"""Minimal driver for ncu: one Llama-2-7B-shaped W2 GEMV (default 4096x4096),
table built once, lookup launched --reps times back to back."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=4096)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--bits", type=int, default=2)
ap.add_argument("--gs", type=int, default=64)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--fast", type=int, default=0)
ap.add_argument("--indep", type=int, default=0)
args = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randint(0, 1 << args.bits, (args.m, args.k), dtype=torch.uint8, device="cuda", generator=g)
s = (torch.randn((args.m, args.k // args.gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
pw = B.prepare_weights(B.QuantizedWeights(m=args.m, k=args.k, bits=args.bits, group_size=args.gs,
                                          qvalues=q, scales=s))
a = torch.randn((args.n, args.k), device="cuda", generator=g).half()
t, ts, rs = N.build_lut(a, args.gs, N.TABLE_Q8)
for _ in range(args.reps):
    N.lookup(pw.gpu, pw.scales, None, t, ts, rs, pw.m, pw.k, pw.bits, pw.gs if hasattr(pw, "gs") else pw.group_size,
             N.TABLE_Q8, N.FLAG_PDL | (N.FLAG_FAST_EPILOGUE if args.fast else 0)
             | (N.FLAG_INDEPENDENT if args.indep else 0), False)
torch.cuda.synchronize()
print("ok")
