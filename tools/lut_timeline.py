"""Back-to-back table builds (PDL) for K=4096 / 11008 rows: us per launch,
dependent vs independent inputs (diagnostic for the table-build hop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_00088_b200 import _native as N  # noqa: E402

for k in (4096, 11008):
    xs = [torch.randn((1, k), device="cuda").half() for _ in range(64)]
    for gs in (64,):
        def run():
            for x in xs:
                N.build_lut(x, gs, N.TABLE_Q8, N.FLAG_PDL)
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                run()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"K={k} gs={gs}: {e0.elapsed_time(e1) * 1e3 / (10 * len(xs)):.2f} us per table build (graph, PDL chain)")
