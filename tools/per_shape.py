"""Per-shape batch-1 lookup timings (bench.py per_shape_table) as a compact
table: python tools/per_shape.py [bits,...]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

bits = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4").split(","))
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
peak = bench.load_peaks()[0]
res = bench.per_shape_table(dev, st, 10, 3, None, peak, 1, bits_list=bits)
for b, shapes in res.items():
    for name, e in shapes.items():
        f = e["fast"]
        print(f"{b} {name:11s} fast overlapped {f['overlapped_us']:7.3f} us {f['overlapped_GBps']:7.1f} GB/s "
              f"chained {f['chained_us']:7.3f} us  exact overlapped {e['exact']['overlapped_us']:7.3f}", flush=True)
