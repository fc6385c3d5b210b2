"""Steady-state lookup throughput on one large launch (diagnostic): M large
enough that launch ramp/tail are negligible; W1/W2/W4, K = 4096 / 11008."""
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
for bits in bitsl:
    for (m, k) in ((65536, 4096), (16384, 11008)):
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        s = (torch.randn((m, k // 64), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
        pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=64, qvalues=q, scales=s))
        del q
        a = torch.randn((1, k), device="cuda", generator=g).half()
        t = N.build_lut(a, 64, N.TABLE_Q8)
        for fast in (0, 1):
            fl = N.FLAG_PDL | (N.FLAG_FAST_EPILOGUE if fast else 0)
            for _ in range(3):
                N.lookup(pw.gpu, pw.scales, None, *t, m, k, bits, 64, N.TABLE_Q8, fl, False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                N.lookup(pw.gpu, pw.scales, None, *t, m, k, bits, 64, N.TABLE_Q8, fl, False)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 20
            print(f"W{bits} {m}x{k} fast={fast}: {us:.2f} us  {bits * m * k / 8 / us / 1e3:.0f} GB/s", flush=True)
        del pw
