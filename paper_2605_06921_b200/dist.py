"""Multi-GPU plumbing for the solver engine: a torch.distributed adapter for
the engine's communicator (include/mqo_gpu.h `mqo_comm`).

One process per GPU; the engine shards the B chains over the ranks.
"Mode P" (solve_pooled): at every merge it all-gathers the per-chain records
and the candidate bodies -- tiny payloads (B x 32
bytes of records plus at most a few packed bodies).  "Mode R"
(solve_replicas): no exchange while solving, then one all-reduce (MAX) of
a packed (score, rank) key and a broadcast of the winning body.  NCCL over
NVLink on GPUs, gloo on CPU (tests).
"""
from __future__ import annotations

import numpy as np


class TorchComm:
    """Adapter: allgather(bytes) -> bytes of all ranks in rank order."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.torch = torch
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device())
                      if backend == "nccl" else torch.device("cpu"))
        self.device = device
        import os
        self.trace = bool(os.environ.get("MQO_COMM_TRACE"))
        self.calls = 0

    def allgather(self, data: bytes) -> bytes:
        torch = self.torch
        if self.trace:
            import sys
            import time
            self.calls += 1
            print(f"[comm rank{self.rank}] #{self.calls} {len(data)} B t={time.time():.3f}",
                  file=sys.stderr, flush=True)
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return b"".join(o.cpu().numpy().tobytes() for o in out)


    def allreduce_max(self, values):
        """Element-wise max over ranks of non-negative int64 keys."""
        torch = self.torch
        t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return [int(v) for v in t.cpu().tolist()]

    def broadcast(self, data: bytes, root: int) -> bytes:
        torch = self.torch
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(self.device)
        self.dist.broadcast(t, src=self.dist.get_global_rank(self.group, root)
                            if self.group is not None else root, group=self.group)
        return t.cpu().numpy().tobytes()


def nccl_comm(device: int | None = None, group=None):
    """The library's native NCCL communicator (include/mqo_gpu.h
    mqo_comm_nccl_create) for this torch.distributed rank: rank 0 creates
    the unique id, torch.distributed ships it to the others; afterwards the
    engine's collectives run inside libmqo_b200 without Python."""
    import torch
    import torch.distributed as dist
    from .api import NativeComm
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [NativeComm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    if device is None:
        device = torch.cuda.current_device()
    return NativeComm.nccl(rank, world, box[0], device)


def shard(b_global: int, world: int, rank: int) -> range:
    """Chains owned by `rank` (contiguous blocks of ceil(B/world)), the same
    split the engine uses."""
    per = (b_global + world - 1) // world
    lo = min(b_global, rank * per)
    return range(lo, min(b_global, lo + per))


def argmax_best(scores: np.ndarray) -> int:
    """Global best over ranks: highest score, ties to the lowest rank."""
    return int(np.argmax(scores))
