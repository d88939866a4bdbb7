"""N>1 host logic on CPU: sharding + the counter all_reduce, world sizes 2 and 4 over gloo.

On the GPU box the same code path runs with NCCL (bench.py under torchrun);
here each rank computes its shard with the oracle (the CUDA path needs a
GPU), which is enough to prove the shard boundaries and the reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2112_03229_b200.dist import Dist, counters_to_u64, shard


def test_shard_tiles_exactly():
    for total in (0, 1, 7, 8, 1000, 8 << 30, (1 << 27) + 3):
        for world in (1, 2, 3, 4, 8):
            pieces = [shard(total, world, r) for r in range(world)]
            assert pieces[0][0] == 0
            for (o, c), (o2, _) in zip(pieces, pieces[1:]):
                assert o + c == o2
            assert sum(c for _, c in pieces) == total
            assert max(c for _, c in pieces) - min(c for _, c in pieces) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import datagen
    import oracle
    d = Dist().init("gloo")
    w = datagen.workload("cfg5", count=total)
    off, cnt = shard(total, world, rank)
    Y = w.targets.host_fill(off, cnt, w.table)
    idx = oracle.search(w.table, Y, threads=1)
    c = torch.from_numpy(oracle.counters(w.table, Y, idx, off).view(np.int64).copy())
    d.reduce_counters(c)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    d.allreduce(t, "max")
    d.barrier()
    if rank == 0:
        q.put((counters_to_u64(c.tolist()), float(t[0])))
    d.close()


@pytest.mark.parametrize("world", [2, 4])
def test_counters_allreduce_over_gloo_equals_global(world):
    import datagen
    import oracle
    total = (1 << 18) + 5
    w = datagen.workload("cfg5", count=total)
    Y = w.targets.host_fill(0, total, w.table)
    ref = counters_to_u64(oracle.counters(w.table, Y, oracle.search(w.table, Y), 0).tolist())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == ref
    assert tmax == float(world)
