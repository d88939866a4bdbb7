"""Multi-GPU plumbing of the hot path.

The target stream is embarrassingly parallel: rank r of G processes the
contiguous block [r*M/G, (r+1)*M/G) of the global stream (generated in place
by the counter-based generators, so every G sees the same dataset), with the
table replicated per device.  There is NO data-path collective; the only
exchange is one all_reduce(SUM) of the u64[8] validation counters (mod 2^64,
order independent) and one all_reduce(MAX) of per-rank device times.
"""
from __future__ import annotations

import os


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(global offset, count) of rank's contiguous block; blocks tile [0, total) exactly."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard request")
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


class Dist:
    """torch.distributed wrapper: NCCL on GPUs, gloo for the CPU tests."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None

    def init(self, backend: str = "nccl"):
        # world > 1, or launched by torchrun (exercises the NCCL path even at N = 1)
        if self.world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29500")
            dist.init_process_group(backend)
            self.pg = dist
            self.backend = backend
        return self

    def barrier(self):
        if self.pg:
            if self.backend == "nccl":
                import torch
                self.pg.barrier(device_ids=[torch.cuda.current_device()])
            else:
                self.pg.barrier()

    def allreduce(self, t, op: str = "max"):
        if self.pg:
            self.pg.all_reduce(t, op=getattr(self.pg.ReduceOp, op.upper()))
        return t

    def reduce_counters(self, c):
        """all_reduce(SUM) of an int64[8] counter tensor (wrapping = mod 2^64)."""
        return self.allreduce(c, "sum")

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()
            self.pg = None


def counters_to_u64(values) -> list[int]:
    return [int(v) & 0xFFFFFFFFFFFFFFFF for v in values]
