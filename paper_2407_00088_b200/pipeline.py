"""Op-list executors (csrc/pipeline.cu): a list of table builds and lookup
GEMVs -- e.g. every projection of a batch-1 decode step -- recorded once and
replayed.  Two executors run the same list, bitwise identically to calling
``mpgemm`` op by op (same device code per tile):

* ``"graph"`` (default): per-op kernels chained with programmatic dependent
  launch (lookups whose inputs are already complete skip the start-of-kernel
  wait), captured into one CUDA graph; a replay is one graph launch.
* ``"batch"``: for op lists of INDEPENDENT batch-1 calls only (table builds
  without dependencies, each lookup reading one of them, fast epilogue, int8
  tables: a layer set): every table build in one launch
  (bitlut_build_lut_batch), then one lookup launch per (K, weight encoding)
  (bitlut_mpgemv_batch, csrc/gemv_batch.cu: each CTA one contiguous tile
  range over all the matrices; offset / zero-point / sign-plane / ternary
  weights); within 1e-5 of the reference, deterministic.

    pl = Pipeline()
    t = pl.tables(x, group_size=64)                     # op 0
    yq = pl.lookup(pw_q, t)                              # waits for op 0
    yk = pl.lookup(pw_k, t)                              # independent of yq
    t2 = pl.tables(x_o, 64, deps=[yq, yk])               # waits for q and k
    ...
    pl.compile(); pl.run()                               # stream-ordered
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _native as N
from .errors import ParameterError, raise_for_status

OP_TABLES, OP_LOOKUP = 0, 1


class PipeOpSpec(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("dep", ctypes.c_int * 3),
                ("a", ctypes.c_void_p), ("a_dtype", ctypes.c_int),
                ("n", ctypes.c_int), ("k", ctypes.c_int), ("group_size", ctypes.c_int),
                ("tables", ctypes.c_void_p), ("tscales", ctypes.c_void_p), ("rowsums", ctypes.c_void_p),
                ("wgpu", ctypes.c_void_p), ("wscales", ctypes.c_void_p), ("zeros", ctypes.c_void_p),
                ("scale_dtype", ctypes.c_int), ("m", ctypes.c_int), ("bits", ctypes.c_int),
                ("out", ctypes.c_void_p), ("flags", ctypes.c_int)]


def _bind():
    L = N.lib()
    L.bitlut_pipeline_plan_flags.restype = ctypes.c_int
    L.bitlut_pipeline_plan_flags.argtypes = [ctypes.POINTER(PipeOpSpec), ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int)]
    L.bitlut_pipeline_launch_ops.restype = ctypes.c_int
    L.bitlut_pipeline_launch_ops.argtypes = [ctypes.POINTER(PipeOpSpec), ctypes.c_int, ctypes.c_void_p]
    L.bitlut_pipeline_launch_ops_counted.restype = ctypes.c_int
    L.bitlut_pipeline_launch_ops_counted.argtypes = [ctypes.POINTER(PipeOpSpec), ctypes.c_int, ctypes.c_void_p,
                                                     ctypes.c_void_p]
    return L


@dataclass
class OpRef:
    index: int
    tensors: tuple = field(default=(), repr=False)


@dataclass
class TableRef(OpRef):
    n: int = 0
    k: int = 0
    group_size: int = 0


class Pipeline:
    """Records ops, then runs them as one CUDA graph replay."""

    EXECUTORS = ("graph", "batch")
    SYNCS = ("counters", "pdl")

    def __init__(self, device=None, executor: str = "graph", sync: str = "pdl"):
        """executor "graph": per-op launches captured in a CUDA graph; their
        inputs are tracked by programmatic-dependent-launch waits
        (sync="pdl", default) or by completion counters (sync="counters": no
        launch drains the stream, but measured slower on B200 -- DESIGN.md
        §4.6).  executor "batch": independent batch-1 calls, one lookup
        launch per (K, encoding)."""
        if executor not in self.EXECUTORS:
            raise ParameterError(f"executor must be one of {self.EXECUTORS}, got {executor!r}")
        if sync not in self.SYNCS:
            raise ParameterError(f"sync must be one of {self.SYNCS}, got {sync!r}")
        self.executor = executor
        self.sync = sync
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.specs: list[PipeOpSpec] = []
        self.keep: list = []           # tensors the device op table points into
        self.outputs: list[torch.Tensor] = []
        self._host = None
        self._dev = None
        self._counters = None
        self._arr = None
        self._graph = None
        self._wextra = {}              # lookup op index -> (PackedWeights, partials tensor or None)

    @staticmethod
    def _deps(deps) -> list[int]:
        idx = [d.index if isinstance(d, OpRef) else int(d) for d in (deps or [])]
        if len(idx) > 3:
            raise ParameterError("an op can name at most 3 dependencies")
        return idx + [-1] * (3 - len(idx))

    def tables(self, a: torch.Tensor, group_size: int, deps: Sequence = (), fuse: bool = False) -> TableRef:
        """Table build (kernel.py:226-251) for activations a (n, k) f16/f32
        on the device, or in pinned host memory (read over the bus).
        fuse=True lets the graph executor fold it into its consumers when they
        are all batch-1 fast-epilogue lookups (one launch per GEMV,
        bitlut_mpgemv_fused)."""
        if not (a.is_cuda or a.is_pinned()):          # pinned host rows: read over the bus (UVA)
            N.require_cuda(a, "activations")
        if a.dim() == 1:
            a = a.reshape(1, -1)
        a = a.contiguous()
        n, k = a.shape
        nq = k // group_size
        dev = a.device if a.is_cuda else self.device
        tables = torch.empty((n, k // 4, 8), dtype=torch.int8, device=dev)
        ts = torch.empty((n, nq), dtype=torch.float32, device=dev)
        rs = torch.empty((n, nq), dtype=torch.float32, device=dev)
        s = PipeOpSpec()
        s.type = OP_TABLES
        s.dep[:] = self._deps(deps)
        s.a, s.a_dtype, s.n, s.k, s.group_size = a.data_ptr(), N.dtype_code(a), n, k, group_size
        s.tables, s.tscales, s.rowsums = tables.data_ptr(), ts.data_ptr(), rs.data_ptr()
        s.flags = N.FLAG_FUSED_TABLES if fuse else 0
        self.specs.append(s)
        self.keep += [a, tables, ts, rs]
        return TableRef(index=len(self.specs) - 1, tensors=(tables, ts, rs), n=n, k=k,
                        group_size=group_size)

    def lookup(self, pw, t: TableRef, deps: Optional[Sequence] = None,
               fast_epilogue: bool = False, out: Optional[torch.Tensor] = None,
               partials: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Lookup GEMV with packed weights pw over table op t; returns the
        (n, m) float32 output tensor (filled when the pipeline runs; pass
        ``out`` to choose it, e.g. a view of one output arena).  By default
        the op depends on its table build only; ``out`` may also be a
        pinned host tensor (the kernel then writes the result over the bus,
        no copy operation).  ``partials`` (batch
        executor only): an (m, k/gs) int32 tensor that receives the exact
        integer sums S = sum_p 2^p P_p."""
        if pw.gpu is None:
            raise ParameterError("packed weights carry no GPU layout")
        if (pw.k, pw.group_size) != (t.k, t.group_size):
            raise ParameterError("table op does not match the weights' k / group_size")
        if out is None:
            out = torch.empty((t.n, pw.m), dtype=torch.float32, device=pw.gpu.device)
        elif (out.dtype != torch.float32 or not out.is_contiguous() or out.numel() != t.n * pw.m
              or not (out.device == pw.gpu.device or (out.device.type == "cpu" and out.is_pinned()))):
            # a PINNED host tensor is allowed: the kernel writes the result
            # over the bus into the UVA-mapped page (no D2H copy operation)
            raise ParameterError("out must be a contiguous float32 (n, m) tensor on the weights' device "
                                 "or in pinned host memory")
        tables, ts, rs = t.tensors
        s = PipeOpSpec()
        s.type = OP_LOOKUP
        s.dep[:] = self._deps([t] if deps is None else deps)
        s.n, s.k, s.group_size = t.n, pw.k, pw.group_size
        s.tables, s.tscales, s.rowsums = tables.data_ptr(), ts.data_ptr(), rs.data_ptr()
        s.wgpu, s.wscales = pw.gpu.data_ptr(), pw.scales.data_ptr()
        s.zeros = pw.zeros.data_ptr() if pw.zeros is not None else None
        s.scale_dtype, s.m, s.bits = N.dtype_code(pw.scales), pw.m, pw.bits
        s.out = out.data_ptr()
        s.flags = N.FLAG_FAST_EPILOGUE if fast_epilogue else 0
        ls = pw.__dict__.get("_layer_set")
        if (self.executor == "graph" and fast_epilogue and t.n == 1 and ls is not None
                and pw.encoding in ("offset", "zeros") and self._layer_set_ok(pw, ls, t, out)):
            # the cached layer-set operand (pw.layer_set_operand()) in the lean kernel: same bits
            s.wgpu, s.wscales = ls[0].data_ptr(), ls[1].data_ptr()
            s.zeros = ls[2].data_ptr() if ls[2] is not None else None
            s.flags |= N.FLAG_LAYER_SET
            self.keep += list(ls)
        self.specs.append(s)
        self.keep += [pw.gpu, pw.scales, pw.zeros, out, pw.native_scales, partials]
        self._wextra[len(self.specs) - 1] = (pw, partials)
        self.outputs.append(out)
        return out

    @staticmethod
    def _layer_set_ok(pw, ls, t: "TableRef", out: torch.Tensor) -> bool:
        """Probe launch: does bitlut_mpgemm take this call with the layer-set
        operand (BITLUT_ELAYOUT where the lean kernel does not apply)?  The
        op's own buffers are used; they are rewritten when the pipeline runs."""
        from .errors import LayoutError
        tables, ts, rs = t.tensors
        if not out.is_cuda:
            return False
        try:
            rc = N.lib().bitlut_mpgemm(ls[0].data_ptr(), pw.m, pw.k, pw.bits, pw.group_size, ls[1].data_ptr(),
                                       ls[2].data_ptr() if ls[2] is not None else None, N.dtype_code(ls[1]),
                                       tables.data_ptr(), ts.data_ptr(), rs.data_ptr(), N.TABLE_Q8, 1,
                                       out.data_ptr(), None, N.FLAG_FAST_EPILOGUE | N.FLAG_LAYER_SET,
                                       ctypes.c_void_p(torch.cuda.current_stream(out.device).cuda_stream))
            raise_for_status(rc, "bitlut_mpgemm")
            return True
        except LayoutError:
            return False

    def op_of(self, out: torch.Tensor) -> int:
        """Op index of a lookup output (to name it as a dependency)."""
        for i, s in enumerate(self.specs):
            if s.type == OP_LOOKUP and s.out == out.data_ptr():
                return i
        raise ParameterError("tensor is not an output of this pipeline")

    def plan_flags(self) -> list[int]:
        """Launch flags the graph executor gives each op (BITLUT_FLAG_*)."""
        n = len(self.specs)
        arr = (PipeOpSpec * n)(*self.specs)
        fl = (ctypes.c_int * n)()
        raise_for_status(_bind().bitlut_pipeline_plan_flags(arr, n, fl), "bitlut_pipeline_plan_flags")
        return list(fl)

    def compile(self) -> "Pipeline":
        L = _bind()
        n = len(self.specs)
        if n == 0:
            raise ParameterError("empty pipeline")
        self._arr = (PipeOpSpec * n)(*self.specs)
        if self.executor == "batch":
            self._compile_batch()
        else:
            self.plan_flags()                       # validates the list before capture
            if self.sync == "counters":
                self._counters = torch.zeros(n + 1, dtype=torch.int32, device=self.device)
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):           # one eager pass (module load, first-launch costs)
                self._launch_ops(side)
            side.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._launch_ops(side)
            self._graph = g
        return self

    def _compile_batch(self) -> None:
        """Validate an independent op list and encode the batched launches."""
        jobs, groups = [], {}
        for i, s in enumerate(self.specs):
            if s.type == OP_TABLES:
                if any(d >= 0 for d in s.dep):
                    raise ParameterError("batch executor: table builds must not depend on other ops")
                j = N.BitlutLutJob()
                j.a, j.a_dtype, j.n, j.k, j.group_size = s.a, s.a_dtype, s.n, s.k, s.group_size
                j.tables, j.tscales, j.rowsums = s.tables, s.tscales, s.rowsums
                jobs.append(j)
                continue
            if s.dep[0] < 0 or s.dep[1] >= 0 or s.dep[2] >= 0 or self.specs[s.dep[0]].type != OP_TABLES:
                raise ParameterError("batch executor: each lookup must depend on exactly its table build")
            if not (s.flags & N.FLAG_FAST_EPILOGUE) or s.n != 1:
                raise ParameterError("batch executor: batch-1 fast-epilogue lookups only")
            pw, partials = self._wextra[i]
            mode = N.W_MODES[pw.encoding]
            m = N.BitlutBatchMat()
            # the layer-set layout of the operand (converted once per PackedWeights);
            # sign: the native scale s of w = s (2q - 1); ternary: the one
            # per-tensor scale, no scale stream; zeros: + the zero points
            lw, lsc, lz = pw.layer_set_operand()
            self.keep += [lw, lsc, lz]
            m.wgpu, m.out, m.m = lw.data_ptr(), s.out, s.m
            m.wscales = pw.native_scales.data_ptr() if mode == N.W_TERNARY else lsc.data_ptr()
            m.zeros = lz.data_ptr() if mode == N.W_ZEROS else None
            m.partials = partials.data_ptr() if partials is not None else None
            m.tables, m.tscales, m.rowsums = s.tables, s.tscales, s.rowsums
            sd = N.dtype_code(pw.native_scales) if mode in (N.W_SIGN, N.W_TERNARY) else s.scale_dtype
            groups.setdefault((s.k, s.bits, s.group_size, sd, mode, partials is not None), []).append(m)
        if not jobs or len({j.a_dtype for j in jobs}) != 1:
            raise ParameterError("batch executor: table builds of one activation dtype")
        self._tbatch = N.TableBatch((N.BitlutLutJob * len(jobs))(*jobs), N.TABLE_Q8, self.device)
        self._lbatches = [N.LookupBatch((N.BitlutBatchMat * len(ms))(*ms), k, bits, gs, sd, self.device, mode)
                          for (k, bits, gs, sd, mode, _), ms in groups.items()]
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self._launch_batch(side)
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self._launch_batch(side)
        self._graph = g

    def _launch_batch(self, stream: torch.cuda.Stream) -> None:
        self._tbatch.launch(N.FLAG_PDL, stream)
        self._launch_lookups(stream)

    def _launch_lookups(self, stream: torch.cuda.Stream) -> None:
        """The batch executor's lookup launches only (diagnostic: the tables
        must be built already)."""
        for i, lb in enumerate(self._lbatches):
            # the first lookup launch waits for the tables; later ones start
            # after it passed that wait, so their tables are complete
            lb.launch(N.FLAG_PDL | N.FLAG_FAST_EPILOGUE | (N.FLAG_INDEPENDENT if i else 0), stream)

    def _launch_ops(self, stream: torch.cuda.Stream) -> None:
        if self.sync == "counters":
            if self._counters is None:
                self._counters = torch.zeros(len(self.specs) + 1, dtype=torch.int32, device=self.device)
            rc = _bind().bitlut_pipeline_launch_ops_counted(self._arr, len(self.specs),
                                                            ctypes.c_void_p(self._counters.data_ptr()),
                                                            ctypes.c_void_p(stream.cuda_stream))
            raise_for_status(rc, "bitlut_pipeline_launch_ops_counted")
            return
        rc = _bind().bitlut_pipeline_launch_ops(self._arr, len(self.specs),
                                                ctypes.c_void_p(stream.cuda_stream))
        raise_for_status(rc, "bitlut_pipeline_launch_ops")

    def n_launches(self) -> int:
        """Kernel launches per run (graph executor: launch units of the plan)."""
        if self.executor == "batch":
            if self._arr is None:
                self.compile()
            return 1 + len(self._lbatches)
        units = sum(1 for f in self.plan_flags() if f != -1 and not (f & N.PLAN_JOINED))
        return units + (1 if self.sync == "counters" else 0)      # + the join kernel

    def run(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Enqueue the whole op list on `stream` (default: current stream)."""
        if self._arr is None:
            self.compile()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            self._graph.replay()

    def run_eager(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Graph executor without the graph: launch the op list directly."""
        if self._arr is None:
            self._arr = (PipeOpSpec * len(self.specs))(*self.specs)
        if self.executor == "batch":
            if self._graph is None:
                self.compile()
            self._launch_batch(stream if stream is not None else torch.cuda.current_stream(self.device))
            return
        self._launch_ops(stream if stream is not None else torch.cuda.current_stream(self.device))

    @property
    def n_ops(self) -> int:
        return len(self.specs)
