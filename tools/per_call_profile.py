"""Where the per-call drop-in time goes (mpgemv(numpy) -> numpy): the whole
call, its Python parts, and the C host-buffer call alone, in microseconds.

    python tools/per_call_profile.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00088_b200 as B  # noqa: E402
from paper_2407_00088_b200 import _native as N, kernel as Kmod  # noqa: E402


def t_us(fn, n=200):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return round((time.perf_counter() - t0) / n * 1e6, 2)


res = {}
for (m, k, bits, gs) in ((4096, 4096, 2, 64), (11008, 4096, 2, 64), (4096, 11008, 2, 64)):
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device="cuda", generator=g)
    sc = (torch.randn((m, k // gs), device="cuda", generator=g).abs() * 0.02 + 1e-3).half()
    pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
    a = np.random.default_rng(0).standard_normal(k).astype(np.float16)
    rows = a.reshape(1, -1)
    r = {"mpgemv_exact": t_us(lambda: B.mpgemv(a, pw)),
         "mpgemv_fast": t_us(lambda: B.mpgemv(a, pw, exact_epilogue=False)),
         "host_rows_check": t_us(lambda: Kmod._host_rows(rows)),
         "validate": t_us(lambda: Kmod.validate_kernel_config(pw.tile, pw.bits, pw.group_size, pw.m, pw.k)),
         "c_call_exact": t_us(lambda: Kmod._host_call(rows, pw, N.TABLE_Q8, N.FLAG_PDL)),
         "c_call_fast": t_us(lambda: Kmod._host_call(rows, pw, N.TABLE_Q8, N.FLAG_PDL | N.FLAG_FAST_EPILOGUE))}
    res[f"{m}x{k}"] = r
print(json.dumps(res))
