"""World-size-2 gloo tests of the multi-process plumbing on CPU: the
communicator adapter the engine's merges use, the chain sharding, and the
bench's max-over-ranks timing reduction."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_06921_b200.dist import TorchComm, shard
    c = TorchComm()
    got = c.allgather(bytes([rank + 1]) * 5)
    # records of the engine merge: 4 x int64 per owned chain, rank order
    import numpy as np
    B = 7
    mine = shard(B, world, rank)
    per = (B + world - 1) // world
    rec = np.zeros((per, 4), np.int64)
    for i, b in enumerate(mine):
        rec[i] = [100 + b, 1, 10 * b, b % 3]
    allrec = np.frombuffer(c.allgather(rec.tobytes()), np.int64).reshape(world * per, 4)
    order = [int(r[0]) - 100 for r in allrec if r[0] >= 100]
    t = torch.tensor([1.5 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # Mode R exchange: argmax key all-reduce + broadcast of the winner's body
    key = c.allreduce_max([(10 << 16) | (0xFFFF - rank), 7 * rank])
    body = c.broadcast(bytes([rank]) * 9 if rank == 1 else bytes(9), 1)
    q.put((rank, got, order, float(t.item()), list(mine), key, body))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, order, tmax, mine, key, body in res:
        assert key == [(10 << 16) | 0xFFFF, 7]  # ties -> the lowest rank
        assert body == b"\x01" * 9
        assert order == list(range(7))  # global chain order restored
        assert tmax == 2.5
    assert res[0][4] == [0, 1, 2, 3] and res[1][4] == [4, 5, 6]
