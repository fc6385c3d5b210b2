"""Steady-state lookup throughput on one large launch (diagnostic): M large
enough that launch ramp/tail are negligible; W1/W2/W4, K = 4096 / 11008.
Launches are captured in a CUDA graph (Python launch overhead excluded)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(8192, 8192, device="cuda")
for _ in range(200):          # clocks up before the first measurement
    x = x @ x * 1e-4
torch.cuda.synchronize()
bitsl = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4").split(",")]
epis = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
shapes = ((65536, 4096), (16384, 11008))
if len(sys.argv) > 3:
    shapes = tuple(tuple(int(v) for v in s.split("x")) for s in sys.argv[3].split(","))
st = torch.cuda.Stream()
for bits in bitsl:
    for (m, k) in shapes:
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        s = (torch.randn((m, k // 64), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
        pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=64, qvalues=q, scales=s))
        del q
        a = torch.randn((1, k), device="cuda", generator=g).half()
        t = N.build_lut(a, 64, N.TABLE_Q8)
        for fast in epis:
            fl = N.FLAG_PDL | (N.FLAG_FAST_EPILOGUE if fast else 0) | \
                (N.FLAG_INDEPENDENT if os.environ.get("BIGM_INDEP") == "1" else 0)
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                for _ in range(3):
                    N.lookup(pw.gpu, pw.scales, None, *t, m, k, bits, 64, N.TABLE_Q8, fl, False)
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=st):
                    for _ in range(10):
                        N.lookup(pw.gpu, pw.scales, None, *t, m, k, bits, 64, N.TABLE_Q8, fl, False)
                gr.replay()
                st.synchronize()
                best = 1e9
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    gr.replay()
                    e1.record(st)
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1) * 1e3 / 10)
            print(f"W{bits} {m}x{k} fast={fast}: {best:.2f} us  {bits * m * k / 8 / best / 1e3:.0f} GB/s", flush=True)
            del gr
        del pw
