"""Host-side logic of the multi-GPU path on CPU (gloo, world size 2): the NCCL unique-id bootstrap
through torch.distributed and the shard plan (contiguous chunk ranges, id_base offsets)."""
import os
import socket

import numpy as np
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
    # shard plan used by bench.py / dist_topk_check.py
    C = 1_000_003
    c0, c1 = rank * C // world, (rank + 1) * C // world
    ranges = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ranges, torch.tensor([c0, c1]))
    out[rank] = (bool(all(torch.equal(g, got[0]) for g in got)) and int(t.sum()) > 0,
                 [tuple(r.tolist()) for r in ranges])
    dist.destroy_process_group()


def test_unique_id_bootstrap_and_shard_plan():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        same, ranges = out[r]
        assert same
        assert ranges[0][0] == 0 and ranges[-1][1] == 1_000_003
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
