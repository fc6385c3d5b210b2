"""Prefill mpGEMM throughput (BASELINE config 4): N in {32,128,512} tokens,
W4/W2 at 4096x4096 and 11008x4096, gs=128, int8 tables.  Reports lookups/s,
equivalent TOPS (2*N*M*K/t) and packed-weight GB/s; table build included
(one build per token row, shared across all output tiles)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N  # noqa: E402

res = []
g = torch.Generator(device="cuda").manual_seed(0)
for (m, k) in ((4096, 4096), (11008, 4096)):
    for bits in (4, 2):
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
        s = (torch.randn((m, k // 128), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
        pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=128, qvalues=q, scales=s))
        for n in (32, 128, 512):
            a = torch.randn((n, k), device="cuda", generator=g).half()
            for fast in (False, True):
                fl = N.FLAG_FAST_EPILOGUE if fast else 0

                def step():
                    t, ts, rs = N.build_lut(a, 128, N.TABLE_Q8)
                    return N.lookup(pw.gpu, pw.scales, None, t, ts, rs, m, k, bits, 128, N.TABLE_Q8, fl, False)[0]
                for _ in range(3):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20 if n < 512 else 5
                e0.record()
                for _ in range(reps):
                    step()
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / reps * 1e-3
                lookups = bits * n * m * (k // 4)
                res.append({"shape": f"{m}x{k}", "bits": bits, "n": n, "epilogue": "fast" if fast else "exact",
                            "us": round(t * 1e6, 2), "lookups_per_s": lookups / t,
                            "equiv_TOPS": 2 * n * m * k / t / 1e12,
                            "packed_GBps": bits * m * k / 8 / t / 1e9})
                print(json.dumps(res[-1]), flush=True)
