"""Output-channel sharding across GPUs.

Rows of W (output channels) are independent -- the reference itself
partitions them across threads (kernel.py:254-263) with results identical
for any partition.  Rank r of P owns a contiguous block of channels (a
multiple of the 32-channel CUDA tile), builds its own tables for the
replicated activations, runs the lookup kernel on its shard, and the
slices are concatenated with one all-gather (NCCL over NVLink/NVSwitch in
production; gloo in the CPU tests).  No partial sums cross ranks, so the
result is bitwise identical to the single-GPU result for every P.

One process per GPU; the process group comes from torch.distributed.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

from .core import QuantizedWeights, TileConfig, as_tensor
from .errors import LayoutError, ParameterError

SHARD_ALIGN = 32      # CUDA tile granularity along M (layout.cuh)


def shard_bounds(m: int, rank: int, world: int, align: int = SHARD_ALIGN) -> tuple[int, int]:
    """Contiguous [lo, hi) channel range of `rank`: blocks of `align`
    channels dealt as evenly as possible (kernel.py:254-263 uses the same
    base/extra split over m-blocks)."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"bad rank/world {rank}/{world}")
    if m % align != 0:
        raise LayoutError(f"m={m} not divisible by the shard alignment {align}")
    blocks = m // align
    base, extra = divmod(blocks, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo * align, hi * align


def shard_sizes(m: int, world: int, align: int = SHARD_ALIGN) -> list[int]:
    return [b - a for a, b in (shard_bounds(m, r, world, align) for r in range(world))]


def shard_quantized_weights(qw: QuantizedWeights, rank: int, world: int) -> QuantizedWeights:
    """The rows of `qw` owned by `rank` (scales / zeros sliced alike)."""
    lo, hi = shard_bounds(qw.m, rank, world)
    q = as_tensor(qw.qvalues)[lo:hi]
    s = as_tensor(qw.scales)[lo:hi]
    z = None if qw.zeros is None else as_tensor(qw.zeros)[lo:hi]
    return QuantizedWeights(m=hi - lo, k=qw.k, bits=qw.bits, group_size=qw.group_size,
                            qvalues=q.contiguous(), scales=s.contiguous(),
                            zeros=None if z is None else z.contiguous())


@dataclass
class ShardedWeights:
    """This rank's PackedWeights plus the global row partition."""

    local: object            # PackedWeights (or any operand local_fn accepts)
    m_total: int
    rank: int
    world: int

    @property
    def sizes(self) -> list[int]:
        return shard_sizes(self.m_total, self.world)


def prepare_sharded(qw: QuantizedWeights, tile: TileConfig = None, rank: Optional[int] = None,
                    world: Optional[int] = None) -> ShardedWeights:
    """Shard then prepare (decompose / pack / repack on this rank's GPU)."""
    from .weight_prep import prepare_weights
    rank = dist.get_rank() if rank is None else rank
    world = dist.get_world_size() if world is None else world
    local = shard_quantized_weights(qw, rank, world)
    pw = prepare_weights(local, tile) if tile is not None else prepare_weights(local)
    return ShardedWeights(local=pw, m_total=qw.m, rank=rank, world=world)


def gather_rows(y_local: torch.Tensor, sizes: list[int], group=None) -> torch.Tensor:
    """All-gather (n, m_r) slices into (n, sum m_r), in rank order."""
    world = len(sizes)
    if world == 1:
        return y_local
    n = y_local.shape[0]
    if len(set(sizes)) == 1:
        # equal shards: one all_gather_into_tensor over a (world, n, m_r) buffer
        buf = torch.empty((world * n, sizes[0]), dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(buf, y_local.contiguous(), group=group)
        return buf.reshape(world, n, sizes[0]).permute(1, 0, 2).reshape(n, world * sizes[0])
    # uneven shards: pad to the largest slice, gather, drop the padding
    mx = max(sizes)
    pad = torch.zeros((n, mx), dtype=y_local.dtype, device=y_local.device)
    pad[:, :y_local.shape[1]] = y_local
    buf = torch.empty((world * n, mx), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(buf, pad, group=group)
    buf = buf.reshape(world, n, mx)
    return torch.cat([buf[r, :, :sizes[r]] for r in range(world)], dim=1)


def sharded_mpgemm(a, sw: ShardedWeights, group=None, variant="cuda-q8",
                   local_fn: Optional[Callable] = None, **kw) -> torch.Tensor:
    """Tensor-parallel mpGEMM: local lookup kernel on this rank's channels,
    then one all-gather of the output slices.  ``local_fn(a, local, **kw)``
    defaults to the CUDA ``mpgemm``; tests substitute a CPU oracle to check
    the partition/gather logic under gloo."""
    if local_fn is None:
        from .kernel import mpgemm

        def local_fn(x, pw, **k):
            return mpgemm(x, pw, variant=variant, **k)
    y = local_fn(a, sw.local, **kw)
    y = as_tensor(y)
    if y.dim() == 1:
        y = y.reshape(1, -1)
    return gather_rows(y, sw.sizes, group)


# ---------------------------------------------------------------------------
# Fused all-gather ("B200-native upgrade"): the lookup kernel's
# epilogue stores every output element straight into each rank's gathered
# row over peer memory and signals each rank's flag once per launch
# (bitlut_mpgemv_gather), so the step has no separate collective launch.
# A rank's row is complete when its flag reaches epoch * world
# (bitlut_gather_wait, stream-ordered).
# ---------------------------------------------------------------------------

def gather_plan(m_total: int, world: int) -> list[tuple[int, int]]:
    """(col_offset, m_r) of every rank in the gathered row (shard_bounds)."""
    return [(lo, hi - lo) for lo, hi in (shard_bounds(m_total, r, world) for r in range(world))]


class FusedGather:
    """Peer buffers of the fused all-gather for one rank: the gathered f32
    rows `row` (2, m_total) -- double-buffered by epoch parity -- and the u32
    `flag` of this rank, the device addresses of every rank's rows / flag, a
    launch ticket and the epoch counter.

    Reuse protocol (what makes the double buffer sufficient): a rank issues
    launch e+1 only after it consumed epoch e's row, in stream order
    (launch, wait, consume, launch, ...).  Launch e+2 on rank A writes the
    slot of epoch e; it is stream-ordered after A's wait for epoch e+1,
    which completes only when every rank B has issued launch e+1 -- and B
    issued that after consuming epoch e.  So no write of epoch e+2 can
    reach a slot a peer is still reading (the single-buffered version let a
    fast rank overwrite epoch e in a slow peer's row).

    `symmetric(m_total, group)`: production path, one process per GPU;
    buffers from torch symmetric memory (NVLink peer mappings via the
    rendezvous handle).  `emulated(m_total, world, device)`: all ranks' buffers
    on one GPU in one process (the kernel path is identical; used by the
    single-GPU tests and the CPU-side logic)."""

    def __init__(self, rank: int, world: int, m_total: int, row: torch.Tensor, flag: torch.Tensor,
                 out_ptrs: list, flag_ptrs: list, keep=None):
        self.rank, self.world, self.m_total = rank, world, m_total
        self.row, self.flag = row, flag
        self.out_ptrs, self.flag_ptrs = out_ptrs, flag_ptrs
        self.ticket = torch.zeros(1, dtype=torch.int32, device=row.device)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=row.device)   # set by a bounded wait
        self.epoch = 0
        self._keep = keep                      # keeps peer allocations / handles alive

    @classmethod
    def emulated(cls, m_total: int, world: int, device) -> list["FusedGather"]:
        rows = [torch.zeros((2, m_total), dtype=torch.float32, device=device) for _ in range(world)]
        flags = [torch.zeros(1, dtype=torch.int32, device=device) for _ in range(world)]
        out_ptrs = [r.data_ptr() for r in rows]
        flag_ptrs = [f.data_ptr() for f in flags]
        return [cls(r, world, m_total, rows[r], flags[r], out_ptrs, flag_ptrs, keep=(rows, flags))
                for r in range(world)]

    @classmethod
    def symmetric(cls, m_total: int, group=None) -> "FusedGather":
        import torch.distributed._symmetric_memory as symm_mem
        group = group or dist.group.WORLD
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        device = torch.device("cuda", torch.cuda.current_device())
        row = symm_mem.empty((2, m_total), dtype=torch.float32, device=device)
        flag = symm_mem.empty(1, dtype=torch.int32, device=device)
        row.zero_()
        flag.zero_()
        h_row = symm_mem.rendezvous(row, group.group_name)
        h_flag = symm_mem.rendezvous(flag, group.group_name)
        out_ptrs = [int(p) for p in h_row.buffer_ptrs]
        flag_ptrs = [int(p) for p in h_flag.buffer_ptrs]
        dist.barrier(group)
        return cls(rank, world, m_total, row, flag, out_ptrs, flag_ptrs, keep=(h_row, h_flag))

    def launch(self, a_row: torch.Tensor, pw, exact_epilogue: bool = False) -> torch.Tensor:
        """This rank's shard lookup (batch 1, fast epilogue) writing into
        every rank's row; returns the local (1, m_r) result.  Does not wait."""
        from . import _native as N
        if exact_epilogue:
            raise ParameterError("the fused all-gather runs the fast epilogue only")
        col, m_r = gather_plan(self.m_total, self.world)[self.rank]
        if pw.m != m_r:
            raise LayoutError(f"shard has {pw.m} channels, rank {self.rank} owns {m_r}")
        x = a_row.reshape(1, -1)
        t = N.build_lut(x, pw.group_size, N.TABLE_Q8)
        self.epoch += 1
        slot = (self.epoch & 1) * self.m_total * 4          # bytes: this epoch's row of every rank
        y = N.mpgemv_gather(pw.gpu, pw.scales, pw.zeros, *t, pw.m, pw.k, pw.bits, pw.group_size,
                            [p + slot for p in self.out_ptrs], self.flag_ptrs, self.ticket, col,
                            N.FLAG_PDL | N.FLAG_FAST_EPILOGUE)
        return y

    def wait(self) -> torch.Tensor:
        """Stream-ordered wait for every rank's slice of the current epoch;
        returns this epoch's gathered (1, m_total) row (valid until launch
        epoch + 2 -- see the reuse protocol above)."""
        from . import _native as N
        N.gather_wait(self.flag, self.epoch * self.world, self.timed_out)
        return self.row[self.epoch & 1:(self.epoch & 1) + 1]


def sharded_mpgemv_fused(a_row, sw: "ShardedWeights", fg: FusedGather) -> torch.Tensor:
    """Tensor-parallel batch-1 mpGEMV with the all-gather fused into the
    lookup epilogue: returns this rank's gathered (1, m_total) row."""
    fg.launch(a_row, sw.local)
    return fg.wait()
