"""Multi-process (world_size 2, gloo, CPU) tests of the output-channel
sharding path.  The per-rank compute is the CPU oracle (the CUDA kernel
needs a GPU); what is tested is the product's partition + gather logic and
the claim that sharding is bitwise transparent."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_00088_b200 import parallel as PAR
from paper_2407_00088_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover_and_align():
    for m in (1024, 4096, 8192, 11008, 28672, 96):
        for world in (1, 2, 3, 4, 8):
            if m // 32 < world:
                continue
            b = [PAR.shard_bounds(m, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == m
            for (lo, hi), (lo2, _) in zip(b, b[1:]):
                assert hi == lo2
            assert all((hi - lo) % 32 == 0 and hi > lo for lo, hi in b)
            sizes = PAR.shard_sizes(m, world)
            assert max(sizes) - min(sizes) <= 32


def _worker(rank, world, port, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    results = {"error": None}
    try:
        from oracle import oracle as O
        import paper_2407_00088_b200 as B
        for m, k, bits, gs in ((256, 512, 2, 64), (352, 256, 4, 128)):   # 352 = 11 tiles: uneven
            inst = W.small_instance(100 + m, m, k, bits, gs, n=3)
            qw = B.QuantizedWeights(m=m, k=k, bits=bits, group_size=gs, qvalues=inst["q"],
                                    scales=inst["scales"])
            local = PAR.shard_quantized_weights(qw, rank, world)
            sw = PAR.ShardedWeights(local=local, m_total=m, rank=rank, world=world)

            def oracle_fn(a, lw):
                return torch.from_numpy(O.mpgemm_q8(a, np.asarray(lw.qvalues),
                                                    np.asarray(lw.scales, np.float32),
                                                    lw.bits, lw.group_size))

            y = PAR.sharded_mpgemm(inst["a"], sw, local_fn=oracle_fn)
            full = O.mpgemm_q8(inst["a"], inst["q"], inst["scales"].astype(np.float32), bits, gs)
            results[(m, k)] = bool(np.array_equal(y.numpy(), full))
    except Exception as e:  # report instead of hanging the parent
        results["error"] = repr(e)
    finally:
        queue.put((rank, results))
        dist.destroy_process_group()


def test_sharded_mpgemm_world2_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out:
        assert res.pop("error") is None, res
        assert res and all(res.values()), (rank, res)


def test_gather_plan_matches_shard_bounds():
    """Fused all-gather host logic: each rank's column window in the gathered
    row is its shard_bounds range; windows tile [0, m) in rank order."""
    from paper_2407_00088_b200 import parallel as PP
    for m, world in ((4096, 1), (4096, 2), (11008, 4), (28672, 8), (1024, 3), (352, 8)):
        plan = PP.gather_plan(m, world)
        assert len(plan) == world
        pos = 0
        for r, (col, mr) in enumerate(plan):
            assert col == pos and (col, col + mr) == PP.shard_bounds(m, r, world)
            pos += mr
        assert pos == m
