"""Host-side logic of the multi-GPU path on CPU (gloo, world size 2): the NCCL unique-id bootstrap
through torch.distributed (what paper_2505_04846_b200.Comm does before hiper_comm_create) and the
library's own shard plan hiper_shard_range, which bench.py and tests/dist_topk_check.py use: every
rank's range is the one the library computes, the ranges tile the corpus exactly, and the sharded
id_base offsets reproduce the global ids."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import ctypes

    import torch

    import paper_2505_04846_b200 as H
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = (ctypes.c_uint8 * 128)()
    if rank == 0:
        assert H.lib().hiper_comm_unique_id(uid) == 0
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
    dist.broadcast(t, src=0)
    got = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(got, t)
    plans = {}
    for C in (0, 1, 7, 1_000_003, 3_600_000, 16_400_000):
        c0, c1 = H.hiper_shard_range(C, world, rank)      # the product's plan, on this rank
        ranges = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(ranges, torch.tensor([c0, c1]))
        plans[C] = [tuple(r.tolist()) for r in ranges]
    out[rank] = (bool(all(torch.equal(g, got[0]) for g in got)) and int(t.sum()) > 0, plans)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_unique_id_bootstrap_and_shard_plan(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        same, plans = out[r]
        assert same
        for C, ranges in plans.items():
            assert ranges == out[0][1][C]                      # every rank sees the same plan
            assert ranges[0][0] == 0 and ranges[-1][1] == C    # tiles [0, C) ...
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))  # ... contiguously
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1                # balanced within one chunk


def test_shard_range_errors():
    import paper_2505_04846_b200 as H
    for args in ((-1, 2, 0), (10, 0, 0), (10, 2, 2), (10, 2, -1)):
        with pytest.raises(H.HiperError):
            H.hiper_shard_range(*args)
