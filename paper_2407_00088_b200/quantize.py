"""Group weight quantizer on the GPU (reference core.py:227-262 and
_kernels.py:18-82 `quantize_groups`), for the CLI's `quantize` / `nmse`.

Same algorithm: per group of `group_size` weights along K, the baseline
scale maps the signed extreme to exactly -2^(b-1); with `refine`, 19
candidate inverse scales (-half + 0.1 t) / smax, t in [-9, 9], are tried and
the rounding with the best least-squares score keeps its refit scale
sum(x l) / sum(l^2).  Rounding is round-half-to-even like the reference's
`round`.  The candidate sums are reduced in a different order than the
reference's sequential float32 loop, so a near-tie between candidates can
pick a different one: this is an offline tool, not the hot path, and it is
tested for error parity (NMSE), not bit parity.
"""
from __future__ import annotations

import numpy as np
import torch

from .core import DEFAULT_GROUP_SIZE, QuantizedWeights, as_tensor
from .errors import LayoutError, ParameterError


def quantize_weights(w, bits: int, group_size: int = DEFAULT_GROUP_SIZE, refine: bool = True,
                     device=None) -> QuantizedWeights:
    if not 1 <= bits <= 4:
        raise ParameterError(f"bits must be in [1, 4], got {bits}")
    x = as_tensor(w).float()
    if device is not None or not x.is_cuda:
        x = x.to(device if device is not None else "cuda")
    if x.dim() != 2:
        raise ParameterError("weights must be 2-D")
    m, k = x.shape
    if group_size < 1 or k % group_size != 0:
        raise LayoutError(f"k={k} not divisible by group_size={group_size}")
    half = 1 << (bits - 1)
    g = x.reshape(-1, group_size)                               # (ng, gs)
    idx = g.abs().argmax(dim=1, keepdim=True)                   # first max, like the reference's '>'
    smax = torch.gather(g, 1, idx)                              # signed extreme (ng, 1)
    zero = smax == 0
    safe = torch.where(zero, torch.ones_like(smax), smax)

    def levels(inv):                                            # inv (ng, c) -> (ng, c, gs)
        lv = torch.round(g[:, None, :] * inv[:, :, None])
        return lv.clamp_(-half, half - 1)

    if not refine:
        inv = (-float(half) / safe)
        lv = levels(inv)[:, 0, :]
        d = (safe / -float(half))[:, 0]
    else:
        t = torch.arange(-9, 10, device=x.device, dtype=torch.float32) * 0.1
        inv = (-float(half) + t)[None, :] / safe                # (ng, 19)
        lv = levels(inv)
        sumlx = (g[:, None, :] * lv).sum(-1)
        suml2 = (lv * lv).sum(-1)
        score = torch.where(suml2 > 0, sumlx * sumlx / suml2.clamp_min(1e-30), torch.full_like(suml2, -1.0))
        best = score.argmax(dim=1)                              # first best, like the reference's strict '>'
        lv = lv[torch.arange(lv.shape[0], device=x.device), best]
        sumlx = (g * lv).sum(-1)
        suml2 = (lv * lv).sum(-1)
        d = torch.where(suml2 > 0, sumlx / suml2.clamp_min(1e-30), torch.zeros_like(suml2))
    q = (lv + half).to(torch.uint8)
    q = torch.where(zero, torch.full_like(q, half), q)
    d = torch.where(zero[:, 0], torch.zeros_like(d), d)
    return QuantizedWeights(m=m, k=k, bits=bits, group_size=group_size, qvalues=q.reshape(m, k),
                            scales=d.reshape(m, k // group_size).float())


def dequantize(qw: QuantizedWeights) -> torch.Tensor:
    """scale[m][k / gs] * (q - z), z = zeros or the implicit 2^(b-1)
    (reference core.py:265-274)."""
    q = as_tensor(qw.qvalues).float().reshape(qw.m, qw.k // qw.group_size, qw.group_size)
    s = as_tensor(qw.scales).float().to(q.device)
    z = (as_tensor(qw.zeros).float().to(q.device) if qw.zeros is not None
         else torch.full_like(s, float(1 << (qw.bits - 1))))
    return ((q - z[:, :, None]) * s[:, :, None]).reshape(qw.m, qw.k)


def nmse(y, y_hat) -> float:
    y, y_hat = np.asarray(y, dtype=np.float64), np.asarray(y_hat, dtype=np.float64)
    return float(((y - y_hat) ** 2).sum() / (y ** 2).sum())
