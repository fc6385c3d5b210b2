#!/usr/bin/env python
"""Benchmark: LUT mpGEMV over the Llama-2-7B decode layer set at batch 1.

Workload (BASELINE.json configs[1]): per layer the 7 decode GEMVs
q,k,v,o (4096x4096), gate,up (11008x4096), down (4096x11008); 2-bit
weights in [0,4), group 64, fp16 scales, implicit zero 2, int8-quantized
tables (bit-exact vs the reference's vector-q8), fp16 activations ~N(0,1).
A STEP = one pass over L layers (default 32 = the whole 7B model, 1.62 GB of
packed weights > 126 MB L2, so no L2 flush is needed): per layer 4 table
builds (qkv / o / gate-up / down inputs) + 7 lookup GEMVs as independent
calls, through the package's batch executor (pipeline.Pipeline
executor="batch": every table build in one launch + one lookup launch per
K -- 3 launches per step).

value    = packed-weight bytes (bits*M*K/8, the reference's weight_bytes,
           cli.py:153) per step / device time, GB/s, all ranks aggregated.
e2e      = the same step through the Pipeline API with pinned HOST buffers on
           both sides (the table launch reads the activation rows, the lookup
           kernels write the results over the bus), inside the timed region.
roofline = the dominant kernel (gemv_batch_kernel) timed alone: the step's
           lookup launches (tables prebuilt), algorithmic bytes / time vs the
           measured HBM peak.
cpu_baseline = the C port of the reference's vector-q8 path on the host
           cores; --impl reference runs the real reference package
           (baseline/_ref) on the same host.
stdout: ONE compact JSON line (< 2 KB); the detail sections (--full: per
shape, configs[0], Llama-2-70B shards, prefill mpGEMM, every executor) go to
bench_details.json.

    python bench.py [--gpus N --steps K --warmup W] [--full] [--impl reference]
Multi-GPU (torchrun): output-channel sharding, one NCCL all-gather per step,
and the fused all-gather epilogue next to it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LUT mpGEMV packed-weight HBM GB/s, Llama-2-7B decode layer set, W2 g64 int8 tables, bs=1"
LAYER = [("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
         ("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]
# table-build inputs per layer and the GEMVs that share each table
LUT_GROUPS = [("attn", 4096, ["q", "k", "v"]), ("o", 4096, ["o"]),
              ("mlp", 4096, ["gate", "up"]), ("down", 11008, ["down"])]


def load_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"), "/root/repo/MEASURED_PEAKS.json"):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        time.sleep(0.1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------- workload

def build_layers(n_layers, bits, gs, rank, world, device, seed=20251020, encoding="offset"):
    """Packed weights for n_layers 7B layers; this rank's output-channel
    shard.  encoding "offset" (the reference's implicit zero), "sign" (1-bit
    sign planes w = +-s, per-group scale) or "ternary" ({-1,0,+1} in 2
    planes, one per-tensor scale): BASELINE configs[1] / configs[2]."""
    import torch
    import paper_2407_00088_b200 as B
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    tile = B.TileConfig(m_tile=32, k_tile=128)
    layers = []
    for _ in range(n_layers):
        mats = {}
        for name, m, k in LAYER:
            if encoding == "ternary":
                q = torch.randint(-1, 2, (m, k), dtype=torch.int8, device=device, generator=gen)
            else:
                q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device=device, generator=gen)
            s = (torch.randn((m, k // gs), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
            if world > 1:
                lo, hi = rank * m // world, (rank + 1) * m // world
                q, s = q[lo:hi].contiguous(), s[lo:hi].contiguous()
            if encoding == "sign":
                qw = B.QuantizedWeights.sign_planes(q, s, gs)
            elif encoding == "ternary":
                qw = B.QuantizedWeights.ternary(q, s[0, 0], gs)
            else:
                qw = B.QuantizedWeights(m=q.shape[0], k=k, bits=bits, group_size=gs, qvalues=q, scales=s)
            pw = B.prepare_weights(qw, tile)
            mats[name] = pw
            del q
        layers.append(mats)
    torch.cuda.synchronize()
    return layers


def make_acts(n_layers, device, seed=7, arena=None):
    """fp16 activation rows, one per table build, carved in order from one
    contiguous arena (so a step's inputs are one H2D copy); returns the
    list of per-layer dicts (the arena is the first row's base)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    per_layer = sum(k for _, k, _ in LUT_GROUPS)
    if arena is None:
        arena = torch.randn((n_layers * per_layer,), device=device, generator=gen).half()
    acts, off = [], 0
    for _ in range(n_layers):
        d = {}
        for g, k, _ in LUT_GROUPS:
            d[g] = arena[off:off + k].view(1, k)
            off += k
        acts.append(d)
    return acts, arena


def build_pipeline(layers, acts, fast=False, executor="graph", chain=True, sync="pdl", lookahead=None,
                   groups=None):
    """The step as a pipeline.Pipeline op list.  chain=True: the decode
    chain's dependencies -- a layer's qkv table build waits for the previous
    layer's down GEMV, o's for q,k,v, gate/up's for o, down's for gate,up.
    chain=False: the layer set as independent mpGEMV calls (activation rows
    are inputs; BASELINE configs[1]).  Either way every GEMV waits for its
    own table build.  All outputs are views of one f32 arena (one D2H per
    step).  groups: the LUT_GROUPS names to include (layer set only;
    default all).  Returns (pipeline, outputs, out_arena)."""
    import torch
    from paper_2407_00088_b200.pipeline import Pipeline
    lut_groups = [gr for gr in LUT_GROUPS if groups is None or gr[0] in groups]
    pl = Pipeline(executor=executor, sync=sync)
    per_layer = sum(layers[0][nm].m for _, _, names in lut_groups for nm in names)
    out_arena = torch.empty((len(layers) * per_layer,), dtype=torch.float32,
                            device=layers[0]["q"].gpu.device)
    prev, outs, off = [], [], 0
    if chain:
        for L, A in zip(layers, acts):
            for gname, k, names in lut_groups:
                t = pl.tables(A[gname], L[names[0]].group_size, deps=prev,
                              fuse=fast and os.environ.get("BENCH_CHAIN_FUSE", "0") == "1")
                ys = []
                for nm in names:
                    m = L[nm].m
                    ys.append(pl.lookup(L[nm], t, fast_epilogue=fast,
                                        out=out_arena[off:off + m].view(1, m)))
                    off += m
                outs += ys
                prev = [pl.op_of(y) for y in ys]
    else:
        # independent calls, software-pipelined: the table builds of layer
        # L+D are recorded before layer L's lookups (D = lookahead), so a
        # lookup finds its tables complete (INDEPENDENT launch) except right
        # after the planner's completed-prefix has to advance (every D+1 layers)
        D = int(os.environ.get("BENCH_LOOKAHEAD", "8")) if lookahead is None else lookahead
        D = max(1, min(D, len(layers)))

        def tables_of(i):
            return {g: pl.tables(acts[i][g], layers[i][names[0]].group_size)
                    for g, _, names in lut_groups}
        tabs = {}
        for i in range(D):
            tabs[i] = tables_of(i)
        for i, L in enumerate(layers):
            if i + D < len(layers):
                tabs[i + D] = tables_of(i + D)
            for gname, k, names in lut_groups:
                for nm in names:
                    m = L[nm].m
                    outs.append(pl.lookup(L[nm], tabs[i][gname], fast_epilogue=fast,
                                          out=out_arena[off:off + m].view(1, m)))
                    off += m
    pl.compile()
    return pl, outs, out_arena


def fast_operand(pw, tabs, n_rows=1):
    """(weights, scales, zeros, extra flag) for fast-epilogue int8-table
    lookups: the layer-set operand (BITLUT_FLAG_LAYER_SET: select-free lean
    kernels) where those kernels take the call, else the v2 operand."""
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200.errors import LayoutError
    try:
        lw, lsc, lz = pw.layer_set_operand()
        N.lookup(lw, lsc, lz, *tabs, pw.m, pw.k, pw.bits, pw.group_size, N.TABLE_Q8,
                 N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | N.FLAG_LAYER_SET, False)
        return lw, lsc, lz, N.FLAG_LAYER_SET
    except LayoutError:
        return pw.gpu, pw.scales, pw.zeros, 0


def capture(fn, stream):
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        fn()          # warm (allocations, NCCL comms)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            fn()
    torch.cuda.synchronize()
    return g


def time_graph(g, reps, warmup, barrier=None):
    import torch
    for _ in range(warmup):
        g.replay()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return e0.elapsed_time(e1) / reps     # ms per replay


def packed_bytes_full(n_layers, bits):
    return n_layers * sum(bits * m * k // 8 for _, m, k in LAYER)


SHAPES_7B = [("4096x4096", 4096, 4096), ("11008x4096", 11008, 4096), ("4096x11008", 4096, 11008)]
L2_BYTES = 126 * 1024 * 1024


# group size per bit width at batch 1: W2 g64 (BASELINE configs[1]), W1 g128
# (configs[2]: 1-bit sign planes), W4 g128 (configs[0] / configs[3])
GS_OF_BITS = {1: 128, 2: 64, 4: 128}


def per_shape_table(device, stream, reps, warmup, barrier, peak, world, bits_list=(1, 2, 4), gs_fixed=None):
    """Per-launch us and GB/s for every 7B shape at W1/W2/W4."""
    import torch
    import paper_2407_00088_b200 as B
    from paper_2407_00088_b200 import _native as N
    gen = torch.Generator(device=device)
    gen.manual_seed(99)
    flush = torch.ones(256 * 1024 * 1024, dtype=torch.uint8, device=device)
    flush_sum = torch.zeros((), dtype=torch.int64, device=device)
    out = {}
    for bits in bits_list:
        res = {}
        gs_b = gs_fixed or GS_OF_BITS[bits]
        for name, m, k in SHAPES_7B:
            gs = gs_b
            m_loc = m // world
            q = torch.randint(0, 1 << bits, (m_loc, k), dtype=torch.uint8, device=device, generator=gen)
            sc = (torch.randn((m_loc, k // gs), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
            pw = B.prepare_weights(B.QuantizedWeights(m=m_loc, k=k, bits=bits, group_size=gs, qvalues=q,
                                                      scales=sc))
            del q
            nbytes = pw.packed_bytes
            copies = max(8, -(-4 * L2_BYTES // nbytes))
            ws = [pw.gpu] + [pw.gpu.clone() for _ in range(copies - 1)]
            x = torch.randn((1, k), device=device, generator=gen).half()
            tabs = N.build_lut(x, gs, N.TABLE_Q8)
            entry = {"packed_bytes_per_gpu": nbytes, "launches_rotated": len(ws), "group_size": gs}
            for epi in ("fast", "exact"):
                e = {}
                base = N.FLAG_PDL | (N.FLAG_FAST_EPILOGUE if epi == "fast" else 0)
                wsel, scl = ws, pw.scales
                if epi == "fast":                      # the layer-set operand where the lean kernel takes it
                    lw, scl, _, lsf = fast_operand(pw, tabs)
                    if lsf:
                        wsel = [lw] + [lw.clone() for _ in range(copies - 1)]
                        base |= lsf
                    e["operand"] = "layer-set" if lsf else "v2"
                for mode, fl in (("overlapped", base | N.FLAG_INDEPENDENT), ("chained", base)):
                    def body(fl=fl, wsel=wsel, scl=scl):
                        for w in wsel:
                            N.lookup(w, scl, None, *tabs, pw.m, k, bits, gs, N.TABLE_Q8, fl, False)
                    g = capture(body, stream)
                    with torch.cuda.stream(stream):
                        ms = time_graph(g, reps, warmup, barrier)
                    del g
                    us = ms * 1e3 / len(ws)
                    e[mode + "_us"] = round(us, 3)
                    e[mode + "_GBps"] = round(nbytes / (us * 1e-6) / 1e9, 1)
                    e[mode + "_frac_of_peak"] = round(nbytes / (us * 1e-6) / 1e9 / peak, 4)
                # one launch after an L2 flush (tables prebuilt): a 256 MB read
                # evicts L2 without leaving dirty lines to write back
                ts_ = []
                with torch.cuda.stream(stream):
                    for _ in range(5):
                        flush_sum.copy_(flush.sum(dtype=torch.int64))
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        N.lookup(wsel[0], scl, None, *tabs, pw.m, k, bits, gs, N.TABLE_Q8, base, False)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ts_.append(e0.elapsed_time(e1) * 1e3)
                e["single_launch_l2_flushed_us"] = round(float(np.median(ts_)), 3)
                entry[epi] = e
                del wsel
            res[name] = entry
            del ws, pw
        out[f"W{bits}"] = res
    del flush
    torch.cuda.empty_cache()
    return out


def config1_table(device, stream, reps, warmup, barrier, peak):
    """BASELINE configs[0]: one 4096x4096 W4 mpGEMV, group 128, fp16 scales and
    asymmetric fp16 zeros, fp16 activation row -- per launch with the tables
    prebuilt (graph over rotating weight copies >= 4x L2, overlapped and
    chained) and per call (table build + lookup, chained), for the
    fp16-table variant (cuda-f16, the configuration the BASELINE names) and
    the int8-table ones (cuda-q8 exact / fast)."""
    import torch
    import paper_2407_00088_b200 as B
    from paper_2407_00088_b200 import _native as N
    gen = torch.Generator(device=device)
    gen.manual_seed(1)
    m = k = 4096
    bits, gs = 4, 128
    q = torch.randint(0, 16, (m, k), dtype=torch.uint8, device=device, generator=gen)
    sc = (torch.randn((m, k // gs), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
    z = (torch.rand((m, k // gs), device=device, generator=gen) * 15).half()
    pw = B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc, zeros=z))
    del q
    nbytes = pw.packed_bytes
    copies = max(8, -(-4 * L2_BYTES // nbytes))
    ws = [pw.gpu] + [pw.gpu.clone() for _ in range(copies - 1)]
    x = torch.randn((1, k), device=device, generator=gen).half()
    out = {"shape": "4096x4096", "bits": bits, "group_size": gs, "zeros": True, "packed_bytes": nbytes,
           "launches_rotated": len(ws)}
    # cuda-f16 fast at batch 1 = 16-bit block-fixed-point tables (what mpgemv picks)
    for name, mode, fast in (("cuda-f16", N.TABLE_F16, False), ("cuda-f16-fast", N.TABLE_X16, True),
                             ("cuda-q8-exact", N.TABLE_Q8, False), ("cuda-q8-fast", N.TABLE_Q8, True)):
        tabs = N.build_lut(x, gs, mode)
        base = N.FLAG_PDL | (N.FLAG_FAST_EPILOGUE if fast else 0)
        e = {}
        wsel, scl, zl = ws, pw.scales, pw.zeros
        if fast:                                   # the layer-set operand (the lean kernel takes both table formats)
            lw, lsc, lz = pw.layer_set_operand()
            try:
                N.lookup(lw, lsc, lz, *tabs, m, k, bits, gs, mode, base | N.FLAG_LAYER_SET, False)
                wsel, scl, zl = [lw] + [lw.clone() for _ in range(copies - 1)], lsc, lz
                base |= N.FLAG_LAYER_SET
            except B.LayoutError:
                pass
        for label, fl in (("overlapped", base | N.FLAG_INDEPENDENT), ("chained", base)):
            def body(fl=fl, tabs=tabs, mode=mode, wsel=wsel, scl=scl, zl=zl):
                for w in wsel:
                    N.lookup(w, scl, zl, *tabs, m, k, bits, gs, mode, fl, False)
            g = capture(body, stream)
            with torch.cuda.stream(stream):
                ms = time_graph(g, reps, warmup, barrier)
            del g
            us = ms * 1e3 / len(ws)
            e[label + "_us"] = round(us, 3)
            e[label + "_GBps"] = round(nbytes / (us * 1e-6) / 1e9, 1)
            e[label + "_frac_of_peak"] = round(nbytes / (us * 1e-6) / 1e9 / peak, 4)

        def call(mode=mode, base=base, wsel=wsel, scl=scl, zl=zl):     # the whole call: table build + lookup, chained
            for w in wsel:
                t = N.build_lut(x, gs, mode, N.FLAG_PDL)
                N.lookup(w, scl, zl, *t, m, k, bits, gs, mode, base, False)
        g = capture(call, stream)
        with torch.cuda.stream(stream):
            ms = time_graph(g, reps, warmup, barrier)
        del g
        e["call_us"] = round(ms * 1e3 / len(ws), 3)
        out[name] = e
    del ws, pw
    torch.cuda.empty_cache()
    return out


SHAPES_70B = [("q/o 8192x8192", 8192, 8192, 2), ("k/v 1024x8192", 1024, 8192, 2),
              ("gate/up 28672x8192", 28672, 8192, 2), ("down 8192x28672", 8192, 28672, 1)]


def llama70b_table(device, stream, reps, warmup, barrier, peak):
    """BASELINE configs[4] on ONE GPU: every Llama-2-70B layer matrix cut to
    the output-channel shard one rank of a P-GPU tensor-parallel group owns
    (P = 1, 2, 4, 8; M/P rows), W2/W4 g128, batch 1 (fast epilogue, launches
    overlapped as in a layer) and batch 8 (mpGEMM rows).  Per-GPU compute
    time; the all-gather of the output slices is not measurable with one GPU
    (parallel.py runs it; gloo tests cover it)."""
    import torch
    import paper_2407_00088_b200 as B
    from paper_2407_00088_b200 import _native as N
    gen = torch.Generator(device=device)
    gen.manual_seed(70)
    gs = 128
    out = {}
    for bits in (2, 4):
        for P in (1, 2, 4, 8):
            layer_us, layer_us8, layer_bytes = 0.0, 0.0, 0
            rows = {}
            for name, m, k, count in SHAPES_70B:
                m_loc = m // P
                q = torch.randint(0, 1 << bits, (m_loc, k), dtype=torch.uint8, device=device, generator=gen)
                sc = (torch.randn((m_loc, k // gs), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
                pw = B.prepare_weights(B.QuantizedWeights(m=m_loc, k=k, bits=bits, group_size=gs, qvalues=q,
                                                          scales=sc))
                del q
                nbytes = pw.packed_bytes
                copies = max(4, -(-4 * L2_BYTES // nbytes))
                ws = [pw.gpu] + [pw.gpu.clone() for _ in range(copies - 1)]
                scs = [pw.scales] + [pw.scales.clone() for _ in range(copies - 1)]
                e = {"m_per_gpu": m_loc, "k": k, "packed_bytes_per_gpu": nbytes}
                for nrow in (1, 8):
                    x = torch.randn((nrow, k), device=device, generator=gen).half()
                    tabs = N.build_lut(x, gs, N.TABLE_Q8)
                    fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | (N.FLAG_INDEPENDENT if nrow == 1 else 0)
                    wsel, ssel = ws, scs
                    lw, lsc, _, lsf = fast_operand(pw, tabs)     # layer-set operand where the lean kernels apply
                    if lsf:
                        wsel = [lw] + [lw.clone() for _ in range(copies - 1)]
                        ssel = [lsc] + [lsc.clone() for _ in range(copies - 1)]
                        fl |= lsf

                    def body(fl=fl, tabs=tabs, wsel=wsel, ssel=ssel):
                        for w, sc_ in zip(wsel, ssel):
                            N.lookup(w, sc_, None, *tabs, m_loc, k, bits, gs, N.TABLE_Q8, fl, False)
                    g = capture(body, stream)
                    with torch.cuda.stream(stream):
                        ms = time_graph(g, reps, warmup, barrier)
                    del g
                    del wsel, ssel
                    us = ms * 1e3 / len(ws)
                    e[f"n{nrow}_us"] = round(us, 3)
                    e[f"n{nrow}_GBps"] = round(nbytes / (us * 1e-6) / 1e9, 1)
                    if nrow == 1:
                        e["n1_frac_of_peak"] = round(nbytes / (us * 1e-6) / 1e9 / peak, 4)
                    else:
                        e["n8_equiv_TOPS"] = round(2 * nrow * m_loc * k / (us * 1e-6) / 1e12, 2)
                layer_us += count * e["n1_us"]
                layer_us8 += count * e["n8_us"]
                layer_bytes += count * nbytes
                rows[name] = e
                del ws, scs, pw
                torch.cuda.empty_cache()
            # the whole per-GPU layer as a decode step issues it: q,k,v in one
            # launch (one activation row), o, gate+up in one launch, down;
            # overlapped launches, rotating weight sets >= 4x L2
            lay = _llama70b_layer_graph(device, stream, reps, warmup, barrier, bits, gs, P, gen)
            out[f"W{bits}_tp{P}"] = {
                "shapes": rows,
                "layer_us_per_gpu_n1": round(layer_us, 2),
                "layer_GBps_per_gpu_n1": round(layer_bytes / (layer_us * 1e-6) / 1e9, 1),
                "layer_grouped_us_per_gpu_n1": lay["us"],
                "layer_grouped_GBps_per_gpu_n1": round(layer_bytes / (lay["us"] * 1e-6) / 1e9, 1),
                "layer_grouped_frac_of_peak": round(layer_bytes / (lay["us"] * 1e-6) / 1e9 / peak, 4),
                "layer_grouped_launches": lay["launches"],
                "layer_us_per_gpu_n8": round(layer_us8, 2),
                "layer_packed_bytes_per_gpu": layer_bytes}
    return out


def _llama70b_layer_graph(device, stream, reps, warmup, barrier, bits, gs, P, gen):
    """One 70B layer shard per GPU (tp P) as 4 grouped batch-1 launches."""
    import torch
    import paper_2407_00088_b200 as B
    from paper_2407_00088_b200 import _native as N

    def make(m, k):
        q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device=device, generator=gen)
        sc = (torch.randn((m, k // gs), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
        return B.prepare_weights(B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc))
    shapes = {"q": (8192, 8192), "k": (1024, 8192), "v": (1024, 8192), "o": (8192, 8192),
              "gate": (28672, 8192), "up": (28672, 8192), "down": (8192, 28672)}
    one = sum(bits * (m // P) * k // 8 for m, k in shapes.values())
    n_sets = max(2, -(-4 * L2_BYTES // one))
    sets = [{nm: make(m // P, k) for nm, (m, k) in shapes.items()} for _ in range(n_sets)]
    xs = {kk: torch.randn((1, kk), device=device, generator=gen).half() for kk in (8192, 28672)}
    tabs = {kk: N.build_lut(x, gs, N.TABLE_Q8) for kk, x in xs.items()}
    fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | N.FLAG_INDEPENDENT
    # layer-set operands for the K = 8192 launches where the lean kernel takes them
    # (the long-K down projection runs the split-K cluster kernel on layout v2)
    ops = []
    for L in sets:
        o = {}
        for nm, pw in L.items():
            w_, s_, _, f_ = fast_operand(pw, tabs[pw.k]) if nm != "down" else (pw.gpu, pw.scales, None, 0)
            o[nm] = (w_, s_, None, pw.m, f_)
        ops.append(o)
    ls8 = all(o[n][4] for o in ops for n in ("q", "k", "v", "o", "gate", "up"))
    f8 = fl | (N.FLAG_LAYER_SET if ls8 else 0)

    def body():
        for L, o in zip(sets, ops):
            sel = (lambda n: o[n][:4]) if ls8 else (lambda n: (L[n].gpu, L[n].scales, None, L[n].m))
            N.mpgemv_multi([sel(n) for n in ("q", "k", "v")], *tabs[8192], 8192, bits, gs, f8)
            wo = sel("o")
            N.lookup(wo[0], wo[1], None, *tabs[8192], L["o"].m, 8192, bits, gs, N.TABLE_Q8, f8, False)
            N.mpgemv_multi([sel(n) for n in ("gate", "up")], *tabs[8192], 8192, bits, gs, f8)
            N.lookup(L["down"].gpu, L["down"].scales, None, *tabs[28672], L["down"].m, 28672, bits, gs,
                     N.TABLE_Q8, fl, False)
    g = capture(body, stream)
    with torch.cuda.stream(stream):
        ms = time_graph(g, reps, warmup, barrier)
    del g, sets, ops
    torch.cuda.empty_cache()
    return {"us": round(ms * 1e3 / n_sets, 3), "launches": 4}


def gemm_table(device, stream, reps, warmup, barrier, world):
    """BASELINE configs[3] (prefill mpGEMM): N in {32, 128, 512} activation
    rows, W4/W2 at 4096x4096 and 11008x4096, gs = 128, int8 tables; one table
    build per row + the weight-stationary lookup kernel, in a CUDA graph.
    Work = lookups = b*N*M*K/4.  Bound: the lookups run on register-resident
    PRMT tables with one IDP.2A (dp2a) per lookup, so the INT pipe is the
    ceiling -- 64 lookups/clk/SM (IDP.2A measured at 63/clk/SM,
    tools/microbench/pipes.cu) x 148 SMs x 1.965 GHz = 18.6e12/s; SURVEY
    8(d)'s LSU figure (32/clk/SM, smem-gather lookups) is reported beside it.
    Equivalent TOPS = 2*N*M*K / t."""
    import torch
    import paper_2407_00088_b200 as B
    from paper_2407_00088_b200 import _native as N
    gen = torch.Generator(device=device)
    gen.manual_seed(5)
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    out = {"int_pipe_bound_lookups_per_s": sms * 64 * 1.965e9,
           "lsu_bound_lookups_per_s": sms * 32 * 1.965e9}
    for (m, k) in ((4096, 4096), (11008, 4096)):
        for bits in (4, 2):
            m_loc = m // world
            q = torch.randint(0, 1 << bits, (m_loc, k), dtype=torch.uint8, device=device, generator=gen)
            sc = (torch.randn((m_loc, k // 128), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
            pw = B.prepare_weights(B.QuantizedWeights(m=m_loc, k=k, bits=bits, group_size=128, qvalues=q,
                                                      scales=sc))
            del q
            for n in (32, 128, 512):
                a = torch.randn((n, k), device=device, generator=gen).half()
                for epi in ("exact", "fast"):
                    fl = N.FLAG_PDL | (N.FLAG_FAST_EPILOGUE if epi == "fast" else 0)
                    wsel, scl = pw.gpu, pw.scales
                    if epi == "fast":                  # the layer-set operand where the rows kernel takes it
                        wsel, scl, _, lsf = fast_operand(pw, N.build_lut(a, 128, N.TABLE_Q8))
                        fl |= lsf

                    def body(fl=fl, wsel=wsel, scl=scl):
                        t = N.build_lut(a, 128, N.TABLE_Q8, N.FLAG_PDL)
                        N.lookup(wsel, scl, None, *t, m_loc, k, bits, 128, N.TABLE_Q8, fl, False)
                    g = capture(body, stream)
                    with torch.cuda.stream(stream):
                        ms = time_graph(g, reps, warmup, barrier)
                    del g
                    t = ms * 1e-3
                    lookups = bits * n * m * (k // 4)
                    out[f"{m}x{k}_W{bits}_n{n}_{epi}"] = {
                        "us": round(t * 1e6, 2), "lookups_per_s": float(f"{lookups / t:.4g}"),
                        "frac_of_int_pipe_bound": round(lookups / t / out["int_pipe_bound_lookups_per_s"], 4),
                        "equiv_TOPS": round(2 * n * m * k / t / 1e12, 2)}
            del pw
    return out


# ----------------------------------------------------------------- CPU baseline

def cpu_baseline(layers_host, bits, gs, budget_s, threads):
    """C port of the reference's vector-q8 path (oracle/bitlut_oracle.c) on
    the host cores: one 7B layer (7 mpGEMV incl. table build) per sample."""
    from oracle import oracle as O
    reps, t_total, bytes_done = 0, 0.0, 0
    layer_bytes = sum(bits * m * k // 8 for _, m, k in LAYER)
    while t_total < budget_s or reps == 0:
        t0 = time.perf_counter()
        for name, m, k, planes, s, a in layers_host:
            O.c_mpgemm(a, planes, m, k, bits, gs, s, mode="vector-q8", threads=threads)
        t_total += time.perf_counter() - t0
        reps += 1
        bytes_done += layer_bytes
    return bytes_done / t_total / 1e9, reps, t_total


def host_layer(layer, acts, bits):
    import torch
    out = []
    for gname, k, names in LUT_GROUPS:
        a = acts[gname].float().cpu().numpy()
        for nm in names:
            pw = layer[nm]
            out.append((nm, pw.m, pw.k, pw.planes.cpu().numpy(), pw.scales.float().cpu().numpy(), a))
    return out


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


# ----------------------------------------------------------------- main

def details_path(arg):
    """Where the detail sections go: --details, else gpurun_out/ when it
    exists (it travels back from the GPU box), else next to bench.py."""
    if arg:
        return arg
    d = os.path.join(ROOT, "gpurun_out")
    return os.path.join(d if os.path.isdir(d) else ROOT, "bench_details.json")


def emit(line, details, path):
    """Detail sections to a side file; ONE compact JSON line (< 2 KB) last on
    stdout, so a driver that keeps only the tail of stdout parses it."""
    if details is not None:
        try:
            with open(path, "w") as f:
                json.dump(details, f, indent=1)
            line["details_file"] = os.path.relpath(path, ROOT)
        except OSError:
            pass
    s = json.dumps(line, separators=(",", ":"))
    for drop in ("summary", "details_file"):
        if len(s) <= 2000:
            break
        line.pop(drop, None)
        s = json.dumps(line, separators=(",", ":"))
    sys.stdout.flush()
    print(s, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--cpu-budget", type=float, default=6.0)
    ap.add_argument("--full", action="store_true",
                    help="also run the detail sections (per-shape, configs[0], 70B shards, prefill "
                         "mpGEMM, every executor) into the details file")
    ap.add_argument("--details", default=None, help="path of the details JSON (default gpurun_out/ or ./)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--ref-min-seconds", type=float, default=3.0,
                    help="reference arm: minimum timed region (s)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    bits, gs = 2, 64

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = {"workload": "llama2-7b decode layer set (q,k,v,o,gate,up,down) x "
                       f"{args.layers} layers, W2 g64, int8 tables, bs=1",
           "global_batch": 1, "bits": bits, "group_size": gs, "layers": args.layers,
           "parallelism": f"tp{world} (output-channel shard + all-gather)" if world > 1 else "single",
           "l2": f"weights {packed_bytes_full(args.layers, bits) / 1e9:.2f} GB/step > 126 MB L2; no flush"}

    if args.impl == "reference":
        return run_reference(args, bits, gs, rank, world, cfg)

    import torch
    import torch.distributed as dist
    from paper_2407_00088_b200 import _native as N
    import paper_2407_00088_b200 as B

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
        group = dist.group.WORLD
    barrier = (lambda: dist.barrier()) if world > 1 else None

    layers = build_layers(args.layers, bits, gs, rank, world, device)
    acts, act_arena = make_acts(args.layers, device)
    stream = torch.cuda.Stream(device)
    peak, peak_src = load_peaks()
    total_bytes = packed_bytes_full(args.layers, bits)
    details = {"config": cfg}
    summary = {}

    def time_runs(run, steps=None):
        steps = steps or args.steps
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                run()
            torch.cuda.synchronize()
            if barrier:
                barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                run()
            e1.record(stream)
            torch.cuda.synchronize()
            if barrier:
                barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:                                   # max over ranks
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---- the step through the package's op-list executors (pipeline.py).
    #      layer_set: the 7 GEMVs per layer as independent mpGEMV calls (the
    #      BASELINE metric); decode_chain: each table build also waits for the
    #      previous GEMVs, as in a real decode.  `value` = the batch executor
    #      (one table launch + one lookup launch per K). ----
    executors, pipes = {}, {}
    runs = [("layer_set_batch_fast", "batch", True, False, "pdl"),
            ("decode_chain_graph_fast", "graph", True, True, "pdl")]
    if args.full:
        runs += [("layer_set_graph_fast", "graph", True, False, "pdl"),
                 ("layer_set_graph_exact", "graph", False, False, "pdl"),
                 ("decode_chain_graph_exact", "graph", False, True, "pdl")]
    if world > 1:
        runs = [r for r in runs if not r[3]]            # the decode chain gathers per GEMV: details only
    gathered = {}
    with ClockSampler(local) as clk:
        for name, ex, fast, chain, sync in runs:
            pl, outs, out_arena = build_pipeline(layers, acts, fast=fast, executor=ex, chain=chain, sync=sync)
            pipes[name] = (pl, out_arena)
            if world == 1:
                executors[name] = {"ms": time_runs(lambda: pl.run(stream)), "launches": pl.n_launches()}
                continue
            # tensor parallel: the rank's shard of the layer set, then ONE
            # NCCL all-gather of the step's output arena (one collective per
            # step); compute-only and collective-only timed apart as well
            gat = torch.empty((world * out_arena.numel(),), dtype=out_arena.dtype, device=device)
            gathered[name] = gat

            def ls_step(pl=pl, out_arena=out_arena, gat=gat):
                pl.run(stream)
                dist.all_gather_into_tensor(gat, out_arena, group=group)

            def coll_only(out_arena=out_arena, gat=gat):
                dist.all_gather_into_tensor(gat, out_arena, group=group)
            executors[name] = {"ms": time_runs(ls_step), "launches": pl.n_launches(),
                               "compute_only_ms": time_runs(lambda pl=pl: pl.run(stream)),
                               "collective_only_ms": time_runs(coll_only),
                               "gather_bytes_per_rank": out_arena.numel() * out_arena.element_size()}
    best = "layer_set_batch_fast"
    ms_step = executors[best]["ms"]
    launches_per_step = executors[best]["launches"]
    value = total_bytes / (ms_step * 1e-3) / 1e9
    details["executors"] = {k: dict({kk: (round(vv, 5) if isinstance(vv, float) else vv)
                                     for kk, vv in v.items()},
                                    GBps=round(total_bytes / (v["ms"] * 1e-3) / 1e9, 2))
                            for k, v in executors.items()}
    if "decode_chain_graph_fast" in executors:
        summary["decode_chain_ms"] = round(executors["decode_chain_graph_fast"]["ms"], 4)
    if world > 1:
        summary["compute_only_ms"] = round(executors[best]["compute_only_ms"], 4)
        summary["collective_only_ms"] = round(executors[best]["collective_only_ms"], 4)

    # ---- N > 1: the all-gather fused into the lookup epilogue (peer stores
    #      over NVLink into torch symmetric memory + release flags), next to
    #      lookup + NCCL all-gather, on one 4096x4096 W2 GEMV ----
    if world > 1:
        try:
            fg_res = fused_gather_run(device, stream, world, group, rank, time_runs)
        except Exception as e:                         # report, never fake
            fg_res = {"error": f"{type(e).__name__}: {e}"[:300]}
        details["fused_gather"] = fg_res
        summary["fused_gather"] = {k: fg_res[k] for k in ("fused_us", "nccl_us", "bitwise_equal", "error")
                                   if k in fg_res}

    # ---- the dominant kernel alone: the batch executor's lookup launches
    #      (tables built by one eager run of the step), same flags ----
    pb = pipes[best][0]
    pb.run(stream)
    torch.cuda.synchronize()
    g_look = capture(lambda: pb._launch_lookups(stream), stream)
    n_look = len(pb._lbatches)
    ms_look = time_graph_max(g_look, args.steps, args.warmup, barrier, stream, world, device)
    del g_look
    local_bytes = sum(pw.packed_bytes for L in layers for pw in L.values())
    achieved = local_bytes / (ms_look * 1e-3) / 1e9
    kernel_name = "gemv_batch_kernel"
    details["roofline_how"] = (
        f"the step's {n_look} batched lookup launches (one per K; {args.layers} layers' q,k,v,o,gate,up and "
        f"down; tables prebuilt) per graph replay; algorithmic bytes = sum bits*M*K/8 = {local_bytes} per "
        f"replay per GPU; CUDA events on the launching stream over {args.steps} replays; peak {peak_src}")

    # ---- the same layer set at the other BASELINE widths (north star: >= 70 %
    #      of HBM peak at W4 / W2 / W1): batch executor, step and lookups only ----
    if not args.no_sweep and world == 1:
        sweep = {}
        with ClockSampler(local) as clk_sw:
            for label, b_, gs_, enc_ in (("W4_g128", 4, 128, "offset"), ("W1_g128", 1, 128, "offset"),
                                         ("W1_sign_g128", 1, 128, "sign"), ("W2_ternary", 2, 128, "ternary")):
                L_ = build_layers(args.layers, b_, gs_, rank, world, device, seed=20251020 + b_, encoding=enc_)
                pl_, _, _ = build_pipeline(L_, acts, fast=True, executor="batch", chain=False)
                ms_ = time_runs(lambda: pl_.run(stream))
                pl_.run(stream)
                torch.cuda.synchronize()
                g_ = capture(lambda: pl_._launch_lookups(stream), stream)
                msl_ = time_graph_max(g_, args.steps, args.warmup, barrier, stream, world, device)
                bytes_ = packed_bytes_full(args.layers, b_)
                sweep[label] = {
                    "packed_bytes_per_step": bytes_, "ms_per_step": round(ms_, 5),
                    "GBps": round(bytes_ / (ms_ * 1e-3) / 1e9, 1),
                    "frac_of_peak": round(bytes_ / (ms_ * 1e-3) / 1e9 / peak, 4),
                    "lookups_only_frac_of_peak": round(bytes_ / (msl_ * 1e-3) / 1e9 / peak, 4),
                    "launches_per_step": pl_.n_launches()}
                del g_, pl_, L_
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
        sweep["clocks"] = clk_sw.summary()
        details["layer_set_bits_sweep"] = sweep
        summary["layer_set_frac"] = {"W2_g64": round(value / peak, 4),
                                     **{k: v["frac_of_peak"] for k, v in sweep.items() if k != "clocks"}}

    # ---- e2e: the same step through the public API from HOST buffers: one
    #      H2D of the step's activation rows (pinned), the op list, one D2H of
    #      every GEMV output (pinned), all inside the timed region. ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, layers, acts, act_arena, stream, device, world, group, time_runs, total_bytes)
    per_call = None
    if not args.no_e2e and world == 1:
        per_call = per_call_run(layers, acts, bits, args)
        details["e2e_per_call_api"] = per_call
        summary["per_call_us"] = per_call["us_per_call"]

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_run(layers, acts, bits, gs, args)

    # ---- detail sections (--full): per-shape, configs[0], 70B shards, prefill ----
    if args.full:
        with ClockSampler(local) as clk_d:
            details["per_shape"] = per_shape_table(device, stream, max(5, args.steps // 4), args.warmup, barrier,
                                                   peak, world)
            if world == 1:
                details["config1_single_mpgemv"] = config1_table(device, stream, max(5, args.steps // 4),
                                                                 args.warmup, barrier, peak)
                details["llama70b_shards"] = llama70b_table(device, stream, max(3, args.steps // 5), args.warmup,
                                                            barrier, peak)
            details["mpgemm_prefill"] = gemm_table(device, stream, max(3, args.steps // 5), args.warmup, barrier,
                                                   world)
        details["detail_clocks"] = clk_d.summary()

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "u8 weights, i8 tables, i32 accumulate, f32 epilogue",
            "data": "synthetic (seeded torch RNG), random-init W2 weights of the Llama-2-7B shapes",
            "config": cfg,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": load_traffic(kernel_name),
                         "kernel": kernel_name},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "summary": summary,
        }
        details["line"] = dict(line)
        emit(line, details, details_path(args.details))
    if world > 1:
        dist.destroy_process_group()


def fused_gather_run(device, stream, world, group, rank, time_runs):
    """One 4096x4096 W2 g64 batch-1 GEMV sharded by output channel over the
    ranks: (a) FusedGather.symmetric -- the lookup kernel stores every output
    into every rank's gathered row over NVLink and releases the peers' flags;
    a bounded stream-ordered wait -- and (b) the lookup + NCCL
    all_gather_into_tensor.  Time per gathered GEMV (max over ranks) and a
    bitwise comparison of the two gathered rows."""
    import torch
    import torch.distributed as dist
    import paper_2407_00088_b200 as B
    from paper_2407_00088_b200 import _native as N
    from paper_2407_00088_b200 import parallel as PP
    m, k, bits, gs = 4096, 4096, 2, 64
    gen = torch.Generator(device=device)
    gen.manual_seed(4096)                                # identical weights / row on every rank
    q = torch.randint(0, 1 << bits, (m, k), dtype=torch.uint8, device=device, generator=gen)
    sc = (torch.randn((m, k // gs), device=device, generator=gen).abs() * 0.02 + 1e-3).half()
    x = torch.randn((1, k), device=device, generator=gen).half()
    qw = B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=q, scales=sc)
    shard = B.prepare_weights(PP.shard_quantized_weights(qw, rank, world))
    # every rank must be able to allocate symmetric memory before any enters
    # the (collective) rendezvous, else the others would wait there forever
    ok = torch.ones(1, device=device)
    try:
        import torch.distributed._symmetric_memory as symm_mem
        symm_mem.empty((1, 16), dtype=torch.float32, device=device)
    except Exception:
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if float(ok.item()) < 1:
        raise RuntimeError("torch symmetric memory unavailable on some rank")
    fg = PP.FusedGather.symmetric(m, group)
    with torch.cuda.stream(stream):
        fg.launch(x[0], shard)
        row = fg.wait().clone()
    torch.cuda.synchronize()
    if int(fg.timed_out.item()):
        raise RuntimeError("fused gather: a peer never arrived (bounded wait timed out)")
    gat = torch.empty((world, shard.m), dtype=torch.float32, device=device)
    fl = N.FLAG_PDL | N.FLAG_FAST_EPILOGUE

    def nccl_step():
        t = N.build_lut(x, gs, N.TABLE_Q8)
        y, _ = N.lookup(shard.gpu, shard.scales, None, *t, shard.m, k, bits, gs, N.TABLE_Q8, fl, False)
        dist.all_gather_into_tensor(gat, y.reshape(-1), group=group)

    def fused_step():
        fg.launch(x[0], shard)
        fg.wait()
    with torch.cuda.stream(stream):
        nccl_step()
    torch.cuda.synchronize()
    equal = bool(torch.equal(row.reshape(-1), gat.reshape(-1)))
    ms_f = time_runs(fused_step)
    ms_n = time_runs(nccl_step)
    if int(fg.timed_out.item()):
        raise RuntimeError("fused gather: a peer never arrived during timing")
    return {"shape": "4096x4096 W2 g64, channel shards", "world": world, "fused_us": round(ms_f * 1e3, 2),
            "nccl_us": round(ms_n * 1e3, 2), "bitwise_equal": equal}


def time_graph_max(g, reps, warmup, barrier, stream, world, device):
    import torch
    with torch.cuda.stream(stream):
        ms = time_graph(g, reps, warmup, barrier)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def e2e_run(args, layers, acts, act_arena, stream, device, world, group, time_runs, total_bytes):
    """The headline op list from pinned HOST buffers.  N = 1: the step cut
    into chunks of layers (one batch Pipeline each); the H2D of chunk c+1 and
    the D2H of chunk c-1 overlap chunk c.  N > 1: H2D of the (replicated)
    activations, the rank's shard, one all-gather, D2H of the gathered
    outputs."""
    import torch
    if world > 1:
        import torch.distributed as dist
        pl, _, out_arena = build_pipeline(layers, acts, fast=True, executor="batch", chain=False)
        gat = torch.empty((world * out_arena.numel(),), dtype=out_arena.dtype, device=device)
        host_in = act_arena.cpu().pin_memory()
        host_out = torch.empty(gat.shape, dtype=gat.dtype).pin_memory()

        def step():
            act_arena.copy_(host_in, non_blocking=True)
            pl.run(stream)
            dist.all_gather_into_tensor(gat, out_arena, group=group)
            host_out.copy_(gat, non_blocking=True)
        ms = time_runs(step)
        return {"value": round(total_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
                "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
                "ms_per_step": round(ms, 4)}
    if os.environ.get("BENCH_E2E_MODE", "zc") == "zc":
        return e2e_zero_copy(args, layers, acts, act_arena, stream, device, time_runs, total_bytes)
    split = [int(x) for x in os.environ.get("BENCH_E2E_SPLIT", "8,8,8,8").split(",") if x]
    if sum(split) != args.layers or min(split) < 1:
        split = [args.layers]
    bounds = [sum(split[:c]) for c in range(len(split) + 1)]
    n_chunks = len(split)
    chunks = [build_pipeline(layers[bounds[c]:bounds[c + 1]], acts[bounds[c]:bounds[c + 1]],
                             fast=True, executor="batch", chain=False) for c in range(n_chunks)]
    host_in = act_arena.cpu().pin_memory()
    per_layer_act = act_arena.numel() // args.layers
    host_outs = [torch.empty(ch[2].shape, dtype=ch[2].dtype).pin_memory() for ch in chunks]
    in_stream, out_stream = torch.cuda.Stream(device), torch.cuda.Stream(device)
    ev_start, ev_out = torch.cuda.Event(), torch.cuda.Event()
    ev_in = [torch.cuda.Event() for _ in chunks]
    ev_done = [torch.cuda.Event() for _ in chunks]

    def e2e_step():
        ev_start.record(stream)                              # time_runs' events are on `stream`
        in_stream.wait_event(ev_start)
        with torch.cuda.stream(in_stream):                   # H2D of chunk c+1 overlaps chunk c
            for c in range(n_chunks):
                lo, hi = bounds[c] * per_layer_act, bounds[c + 1] * per_layer_act
                act_arena[lo:hi].copy_(host_in[lo:hi], non_blocking=True)
                ev_in[c].record(in_stream)
        for c, (pl_c, _, arena_c) in enumerate(chunks):
            stream.wait_event(ev_in[c])
            pl_c.run(stream)
            ev_done[c].record(stream)
            out_stream.wait_event(ev_done[c])
            with torch.cuda.stream(out_stream):              # D2H of chunk c overlaps chunk c+1
                host_outs[c].copy_(arena_c, non_blocking=True)
        ev_out.record(out_stream)
        stream.wait_event(ev_out)                            # the step ends when the last D2H does
    ms = time_runs(e2e_step)
    for c, (_, _, arena_c) in enumerate(chunks):             # the bytes really arrived
        assert torch.equal(host_outs[c], arena_c.cpu())
    return {"value": round(total_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
            "d2h_bytes_per_step": int(sum(h.numel() * h.element_size() for h in host_outs)),
            "ms_per_step": round(ms, 4)}


def e2e_zero_copy(args, layers, acts, act_arena, stream, device, time_runs, total_bytes):
    """e2e through the public Pipeline API with HOST buffers on both sides:
    the batch table launch reads the step's activation rows from a pinned
    host arena and the lookup kernels write every result into a pinned host
    arena (UVA-mapped pages: the H2D / D2H transfers happen inside the
    kernels, over the bus, overlapped with the weight streaming).  The step
    ends when the last kernel (and so its host writes) completes; the host
    arena is checked bitwise against a device-resident run afterwards.
    (BENCH_E2E_ZC_IN=0: copy-engine H2D in chunks of layers instead, 6 %
    slower; BENCH_E2E_MODE=copy: the round-1 copy-engine path, 17 % slower.)"""
    import torch
    split = [int(x) for x in os.environ.get("BENCH_E2E_SPLIT", "8,8,8,8").split(",") if x]
    if sum(split) != args.layers or min(split) < 1:
        split = [args.layers]
    bounds = [sum(split[:c]) for c in range(len(split) + 1)]
    per_layer_out = sum(layers[0][nm].m for _, _, names in LUT_GROUPS for nm in names)
    host_out = torch.empty((args.layers * per_layer_out,), dtype=torch.float32).pin_memory()
    from paper_2407_00088_b200.pipeline import Pipeline
    chunks = []
    for c in range(len(split)):
        pl = Pipeline(executor="batch")
        off = bounds[c] * per_layer_out
        for L, A in zip(layers[bounds[c]:bounds[c + 1]], acts[bounds[c]:bounds[c + 1]]):
            for gname, _, names in LUT_GROUPS:
                t = pl.tables(A[gname], L[names[0]].group_size)
                for nm in names:
                    m = L[nm].m
                    pl.lookup(L[nm], t, fast_epilogue=True, out=host_out[off:off + m].view(1, m))
                    off += m
        pl.compile()
        chunks.append(pl)
    host_in = act_arena.cpu().pin_memory()
    per_layer_act = act_arena.numel() // args.layers
    in_stream = torch.cuda.Stream(device)
    ev_start = torch.cuda.Event()
    ev_in = [torch.cuda.Event() for _ in chunks]
    if os.environ.get("BENCH_E2E_ZC_IN", "1") == "1":
        # the table launch reads the rows from the pinned host arena itself
        host_acts, _ = make_acts(args.layers, device, arena=host_in)
        pl = Pipeline(executor="batch")
        off = 0
        for L, A in zip(layers, host_acts):
            for gname, _, names in LUT_GROUPS:
                t = pl.tables(A[gname], L[names[0]].group_size)
                for nm in names:
                    m = L[nm].m
                    pl.lookup(L[nm], t, fast_epilogue=True, out=host_out[off:off + m].view(1, m))
                    off += m
        pl.compile()
        chunks = [pl]
        ev_in = []

        def e2e_step():
            pl.run(stream)
        ms = time_runs(e2e_step)
        dev_pl, _, dev_arena = build_pipeline(layers, acts, fast=True, executor="batch", chain=False)
        dev_pl.run(stream)
        torch.cuda.synchronize()
        assert torch.equal(host_out, dev_arena.cpu())
        return {"value": round(total_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
                "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
                "ms_per_step": round(ms, 4),
                "h2d": "read by the table launch from pinned host memory",
                "d2h": "written by the lookup kernels into pinned host memory"}

    def e2e_step():
        ev_start.record(stream)
        in_stream.wait_event(ev_start)
        with torch.cuda.stream(in_stream):               # H2D of chunk c+1 overlaps chunk c
            for c in range(len(chunks)):
                lo, hi = bounds[c] * per_layer_act, bounds[c + 1] * per_layer_act
                act_arena[lo:hi].copy_(host_in[lo:hi], non_blocking=True)
                ev_in[c].record(in_stream)
        for c, pl in enumerate(chunks):
            stream.wait_event(ev_in[c])
            pl.run(stream)
    ms = time_runs(e2e_step)
    # the bytes really arrived: a device run of the same op list agrees bitwise
    dev_pl, _, dev_arena = build_pipeline(layers, acts, fast=True, executor="batch", chain=False)
    dev_pl.run(stream)
    torch.cuda.synchronize()
    assert torch.equal(host_out, dev_arena.cpu())
    return {"value": round(total_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(host_in.numel() * host_in.element_size()),
            "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
            "ms_per_step": round(ms, 4), "d2h": "written by the lookup kernels into pinned host memory"}


def per_call_run(layers, acts, bits, args):
    """The per-call drop-in API (reference kernel.py:374 mpgemv: numpy fp16
    row in, numpy f32 out), one call per GEMV, wall clock."""
    import paper_2407_00088_b200 as B
    n_pc = min(args.layers, 4)
    host_rows = [{g: A[g][0].cpu().numpy() for g in A} for A in acts[:n_pc]]

    def pc_step():
        for L, HA in zip(layers[:n_pc], host_rows):
            for gname, k, names in LUT_GROUPS:
                for nm in names:
                    B.mpgemv(HA[gname], L[nm])
    pc_step()
    reps, t0 = 5, time.perf_counter()
    for _ in range(reps):
        pc_step()
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(packed_bytes_full(n_pc, bits) / dt / 1e9, 2), "unit": "GB/s",
            "us_per_call": round(dt * 1e6 / (7 * n_pc), 1),
            "path": "mpgemv(numpy fp16 row, PackedWeights) -> numpy f32, one call per GEMV, wall clock"}


def cpu_baseline_run(layers, acts, bits, gs, args):
    try:
        from oracle import oracle as O
        threads = O.c_max_threads()
        hl = host_layer(layers[0], acts[0], bits)
        gbps, reps, secs = cpu_baseline(hl, bits, gs, args.cpu_budget, threads)
        model, ncpu = cpu_info()
        cpu = {"value": round(gbps, 4), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"1 7B W2 layer (7 vector-q8 mpGEMV + tables) x {reps} = {secs:.1f}s, "
                         f"{threads} threads, {model}"}
        g1, r1, s1 = cpu_baseline(hl, bits, gs, min(2.0, args.cpu_budget), 1)
        cpu["single_thread"] = round(g1, 4)
        return cpu
    except Exception as e:  # report, never fake
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "port", "sample": f"unavailable: {e}"}


def load_traffic(kernel="gemv_batch_kernel"):
    """ncu DRAM bytes (read + write) per launch of the headline's dominant
    kernel from one committed `ncu --set full` capture of the batch
    executor's lookup launches (mean per launch; roofline.achieved is per
    replay of the same launches)."""
    for name in ("r02d_batch_w2_full.json", "r02_batch_w2_full.json", "r01h_batch_full.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            tot = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in d["launches"])
            return round(tot / len(d["launches"]), 1)
    return None


# ----------------------------------------------------------------- reference arm

def _ref_module():
    """The UNMODIFIED reference package installed under baseline/_ref
    (pip --target), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "bitlut")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/bitlut_numba_cache")
    sys.path.insert(0, ref)
    try:
        import bitlut
        return bitlut
    except Exception:
        return None


def run_reference(args, bits, gs, rank, world, cfg):
    """--impl reference: the reference's own CPU implementation of the path
    on the host cores, same metric/config.  Preferred: the real reference
    package (baseline/_ref, numba) through its public API -- bitlut.mpgemv(a,
    pw, variant="vector-q8", threads=os.cpu_count()) -- on one Llama-2-7B W2
    layer (7 GEMVs incl. their table builds) per sample.  Fallback when it is
    not importable: the C port (oracle/, pinned bitwise to it).  A step is a
    bounded sample of the 32-layer workload: r layers, r chosen in warm-up
    so the K timed steps last >= --ref-min-seconds; median step time."""
    if rank != 0:
        return
    from paper_2407_00088_b200 import workloads as W
    bl = _ref_module()
    threads = os.cpu_count() or 1
    hl = []
    for name, m, k in LAYER:
        si = {(4096, 4096): 0, (11008, 4096): 1, (4096, 11008): 2}[(m, k)]
        hl.append((name, m, k, W.config2(si)))
    layer_bytes = sum(bits * m * k // 8 for _, m, k in LAYER)
    if bl is not None:
        kind = "reference"
        tile = bl.TileConfig(n_tile=1, m_tile=32, k_tile=128, g=4, lanes=16)
        prepared = {}
        for name, m, k, inst in hl:
            if (m, k) not in prepared:
                qw = bl.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=inst["q"],
                                         scales=inst["scales"].astype(np.float32))
                prepared[(m, k)] = (bl.prepare_weights(qw, tile), inst["a"][0].astype(np.float32))

        def layer():
            for name, m, k, _ in hl:
                pw, a = prepared[(m, k)]
                bl.mpgemv(a, pw, variant="vector-q8", threads=threads)
        impl = f"bitlut {getattr(bl, '__version__', '?')} (baseline/_ref, numba) mpgemv vector-q8 threads={threads}"
    else:
        kind = "port"
        from oracle import oracle as O
        threads = O.c_max_threads()
        ports = []
        for name, m, k, inst in hl:
            planes = O.pack_v1(O.decompose_bits(inst["q"], bits, 4), 32, 128, 4, 16)
            ports.append((m, k, planes, inst["scales"].astype(np.float32), inst["a"].astype(np.float32)))

        def layer():
            for m, k, planes, s, a in ports:
                O.c_mpgemm(a, planes, m, k, bits, gs, s, threads=threads)
        impl = f"C port of the reference vector-q8 kernel (oracle/), {threads} threads"
    t_layer = []
    for _ in range(max(2, args.warmup)):                     # includes numba JIT on the first call
        t0 = time.perf_counter()
        layer()
        t_layer.append(time.perf_counter() - t0)
    per_layer = min(t_layer[1:])
    # 25 % margin: the timed steps run faster than the warm-up estimate (caches, numba threads warm)
    reps = max(1, int(np.ceil(1.25 * args.ref_min_seconds / max(args.steps, 1) / per_layer)))
    samples = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for _ in range(reps):
            layer()
        samples.append(time.perf_counter() - t0)
    dt = float(np.median(samples))
    gbps = reps * layer_bytes / dt / 1e9
    model, ncpu = cpu_info()
    sample = (f"{reps} Llama-2-7B W2 g64 layer(s) (7 mpGEMV incl. table build) per step, {impl}, "
              f"{model}; median of {args.steps} steps, timed {sum(samples):.1f}s")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbps, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "u8 weights, i8 tables, i32 accumulate, f32 epilogue", "data": "synthetic (seeded numpy PCG64)",
        "config": cfg,
        "cpu_baseline": {"value": round(gbps, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(gbps, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_region_s": round(sum(samples), 2),
    }
    emit(line, None, None)


if __name__ == "__main__":
    main()
