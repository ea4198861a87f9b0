"""World-size-2 (gloo, CPU) coverage of bench.py's multi-GPU path: each rank
owns an independent shard of adders (no data-path collective), records its
circuits, and only timings/counts are reduced (max / sum) across ranks."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2101_03403_b200 as P
    from conftest import fu
    ws, r, local = bench.dist_env()
    av, bv = bench.workload_operands(r)
    # record a slice of this rank's shard on the cleartext recorder
    b = P.Backend()
    ok = True
    for i in range(4):
        wa, wb = b.encrypt_word(int(av[i]), 16), b.encrypt_word(int(bv[i]), 16)
        out = fu(b, "add", wa, wb)
        ok &= b.decrypt_word(out) == int(av[i] + bv[i])
    gates = torch.tensor([b.stats()["bootstrapped"]], dtype=torch.float64)
    dist.all_reduce(gates, op=dist.ReduceOp.SUM)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)  # per-rank "device time"
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    first = torch.tensor([float(av[0])], dtype=torch.float64)
    gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, first)
    q.put((rank, ws, bool(ok), gates.item(), t.item(), [g.item() for g in gathered]))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, ws, ok, gates, tmax, firsts in res:
        assert ws == 2 and ok
        assert gates == 2 * 4 * 195          # weak scaling: per-rank work fixed
        assert tmax == 2.0                   # max over ranks
        assert firsts[0] != firsts[1]        # independent shards (seed + rank)
