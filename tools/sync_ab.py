"""Counter-synchronised vs PDL-synchronised op lists (diagnostic): one table
build + R lookups over rotating weight copies (4096x4096 W2, fast)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200.pipeline import Pipeline  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
m = k = 4096
q = torch.randint(0, 4, (m, k), dtype=torch.uint8, device=dev, generator=g)
s = (torch.randn((m, k // 64), device=dev, generator=g).abs() * 0.02 + 1e-3).half()
pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=2, group_size=64, qvalues=q, scales=s))
x = torch.randn((1, k), device=dev, generator=g).half()
copies = 128
import dataclasses  # noqa: E402
pws = [dataclasses.replace(pw, gpu=pw.gpu.clone()) for _ in range(copies)]
grouped = os.environ.get("BITLUT_PLAN_NOGROUP", "0") != "1"
if True:
    for sync in ("pdl", "counters"):
        pl = Pipeline(executor="graph", sync=sync)
        t = pl.tables(x, 64)
        for p2 in pws:
            pl.lookup(p2, t, fast_epilogue=True)
        pl.compile()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                pl.run(st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                pl.run(st)
            e1.record(st)
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 10
        print(f"grouped={grouped} sync={sync}: {us:.1f} us per list, {us / copies:.3f} us per lookup, "
              f"launches {pl.n_launches()}", flush=True)
