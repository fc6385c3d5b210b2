"""Persistent pipeline executor (csrc/pipeline.cu): a list of table builds
and lookup GEMVs -- e.g. every projection of a batch-1 decode step -- runs
in ONE cooperative launch, with per-op dependencies resolved by completion
counters instead of kernel boundaries.  Results are bitwise identical to
calling ``mpgemm`` op by op (same device code per tile).

    pl = Pipeline()
    t = pl.tables(x, group_size=64)                     # op 0
    yq = pl.lookup(pw_q, t)                              # waits for op 0
    yk = pl.lookup(pw_k, t)                              # independent of yq
    t2 = pl.tables(x_o, 64, deps=[yq, yk])               # waits for q and k
    ...
    pl.compile(); pl.run()                               # stream-ordered, graph-capturable
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
    L.bitlut_pipeline_table_bytes.restype = ctypes.c_size_t
    L.bitlut_pipeline_table_bytes.argtypes = [ctypes.c_int]
    L.bitlut_pipeline_encode.restype = ctypes.c_int
    L.bitlut_pipeline_encode.argtypes = [ctypes.POINTER(PipeOpSpec), ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_size_t]
    L.bitlut_pipeline_launch.restype = ctypes.c_int
    L.bitlut_pipeline_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
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
    """Records ops, then runs them in one persistent launch."""

    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.specs: list[PipeOpSpec] = []
        self.keep: list = []           # tensors the device op table points into
        self.outputs: list[torch.Tensor] = []
        self._host = None
        self._dev = None
        self._counters = None

    @staticmethod
    def _deps(deps) -> list[int]:
        idx = [d.index if isinstance(d, OpRef) else int(d) for d in (deps or [])]
        if len(idx) > 3:
            raise ParameterError("an op can name at most 3 dependencies")
        return idx + [-1] * (3 - len(idx))

    def tables(self, a: torch.Tensor, group_size: int, deps: Sequence = ()) -> TableRef:
        """Table build (kernel.py:226-251) for activations a (n, k) f16/f32."""
        N.require_cuda(a, "activations")
        if a.dim() == 1:
            a = a.reshape(1, -1)
        a = a.contiguous()
        n, k = a.shape
        nq = k // group_size
        tables = torch.empty((n, k // 4, 8), dtype=torch.int8, device=a.device)
        ts = torch.empty((n, nq), dtype=torch.float32, device=a.device)
        rs = torch.empty((n, nq), dtype=torch.float32, device=a.device)
        s = PipeOpSpec()
        s.type = OP_TABLES
        s.dep[:] = self._deps(deps)
        s.a, s.a_dtype, s.n, s.k, s.group_size = a.data_ptr(), N.dtype_code(a), n, k, group_size
        s.tables, s.tscales, s.rowsums = tables.data_ptr(), ts.data_ptr(), rs.data_ptr()
        self.specs.append(s)
        self.keep += [a, tables, ts, rs]
        return TableRef(index=len(self.specs) - 1, tensors=(tables, ts, rs), n=n, k=k,
                        group_size=group_size)

    def lookup(self, pw, t: TableRef, deps: Optional[Sequence] = None,
               fast_epilogue: bool = False) -> torch.Tensor:
        """Lookup GEMV with packed weights pw over table op t; returns the
        (n, m) float32 output tensor (filled when the pipeline runs).  By
        default the op depends on its table build only."""
        if pw.gpu is None:
            raise ParameterError("packed weights carry no GPU layout")
        if (pw.k, pw.group_size) != (t.k, t.group_size):
            raise ParameterError("table op does not match the weights' k / group_size")
        out = torch.empty((t.n, pw.m), dtype=torch.float32, device=pw.gpu.device)
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
        self.specs.append(s)
        self.keep += [pw.gpu, pw.scales, pw.zeros, out]
        self.outputs.append(out)
        return out

    def op_of(self, out: torch.Tensor) -> int:
        """Op index of a lookup output (to name it as a dependency)."""
        for i, s in enumerate(self.specs):
            if s.type == OP_LOOKUP and s.out == out.data_ptr():
                return i
        raise ParameterError("tensor is not an output of this pipeline")

    def compile(self) -> "Pipeline":
        L = _bind()
        n = len(self.specs)
        nbytes = L.bitlut_pipeline_table_bytes(n)
        arr = (PipeOpSpec * n)(*self.specs)
        host = torch.empty(nbytes, dtype=torch.uint8)
        rc = L.bitlut_pipeline_encode(arr, n, ctypes.c_void_p(host.data_ptr()), nbytes)
        raise_for_status(rc, "bitlut_pipeline_encode")
        self._host = host
        self._dev = host.to(self.device)
        self._counters = torch.zeros(2 * n, dtype=torch.int32, device=self.device)
        return self

    def run(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        if self._dev is None:
            self.compile()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _bind().bitlut_pipeline_launch(ctypes.c_void_p(self._host.data_ptr()),
                                            ctypes.c_void_p(self._dev.data_ptr()),
                                            ctypes.c_void_p(self._counters.data_ptr()),
                                            ctypes.c_void_p(st.cuda_stream))
        raise_for_status(rc, "bitlut_pipeline_launch")

    @property
    def n_ops(self) -> int:
        return len(self.specs)
