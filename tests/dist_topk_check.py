"""Multi-GPU parity (P13): run under torchrun with N ranks, one GPU each.

Every rank scores the same queries against its contiguous shard of one corpus (id_base = shard
offset) and the shards are merged with hiper_maxsim_topk's ncclAllGather.  Rank 0 also scores the
whole corpus on its own GPU; the sharded result must be bitwise identical on every rank."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import paper_2505_04846_b200 as H
from synth import device, gen


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    C, L, Q, Lq, d = int(os.environ.get("DIST_C", 30011)), 256, 37, 32, 128
    seed, qseed = 5, 6
    comm = H.Comm()
    lens_all = gen.lengths(seed, C, L, True)
    q = torch.empty((Q, Lq, d), dtype=torch.bfloat16, device="cuda")
    device.queries_(q, qseed, corpus_seed=seed, n_chunks=C, L=L,
                    chunk_lens=torch.from_numpy(lens_all).cuda())
    qlen = gen.lengths(qseed, Q, Lq, True, stream=gen.QLEN)
    ok = True
    for k in (10, 100):
        c0, c1 = rank * C // world, (rank + 1) * C // world
        shard = torch.empty((c1 - c0, L, d), dtype=torch.bfloat16, device="cuda")
        device.corpus_(shard, seed, c0)
        idx = H.hiper_index_build(shard, lens_all[c0:c1], id_base=c0)
        s, i = H.hiper_maxsim_topk(idx, q, qlen, k, comm=comm)
        torch.cuda.synchronize()
        gs = [torch.empty_like(s) for _ in range(world)]
        gi = [torch.empty_like(i) for _ in range(world)]
        dist.all_gather(gs, s)
        dist.all_gather(gi, i)
        if rank == 0:
            full = torch.empty((C, L, d), dtype=torch.bfloat16, device="cuda")
            device.corpus_(full, seed, 0)
            fidx = H.hiper_index_build(full, lens_all)
            fs, fi = H.hiper_maxsim_topk(fidx, q, qlen, k)
            for r in range(world):
                same_i = torch.equal(gi[r], fi)
                same_s = torch.equal(gs[r].view(torch.int32), fs.view(torch.int32))
                print(f"k={k} rank{r}: ids equal {same_i}, scores bitwise {same_s}", flush=True)
                ok &= same_i and same_s
            del full, fidx
        del shard, idx
    flag = torch.tensor([int(ok)], device="cuda")
    dist.broadcast(flag, 0)
    comm.close()
    dist.destroy_process_group()
    if rank == 0:
        print("DIST_OK" if flag.item() else "DIST_FAIL", flush=True)
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
