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


def oracle_check(s, i, full, lens, q, qlen, k, what):
    """The sharded, all-gathered answer vs the ORACLE's exact top-k over the whole corpus, for
    sampled queries.  The oracle scores the bf16 operands of a dense layout of the full corpus,
    after sampled rows of it are checked bitwise against the oracle's own NORM of the raw inputs."""
    import oracle
    from tests._compare import assert_topk_ok
    C, L, d = full.shape
    bits = lambda t: t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    didx = H.hiper_index_build(full, lens)                 # dense layout (NORM'd in a copy)
    lay = bits(didx.layout())
    rows = [0, 1, C // 2, C - 1]
    raw = gen.corpus_tokens_f32(5, np.array(rows), L, d)
    for j, c in enumerate(rows):
        n = int(lens[c])
        assert np.array_equal(lay[c, :n], oracle.norm_rows(gen.f32_to_bf16_bits(raw[j, :n]))), c
    qlay, _ = H.hiper_prepare_queries(q, qlen)
    qlay = bits(qlay)
    sample = [0, len(qlen) - 1]
    S_o = oracle.maxsim_matrix(qlay[sample], qlen[sample], lay, lens)
    ids = np.arange(C, dtype=np.int64)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    try:
        for r, qq in enumerate(sample):
            assert_topk_ok(s[qq], i[qq], S_o[r], ids, k, qlen[qq], d, f"{what} query {qq}")
    except AssertionError as e:
        print(f"{what}: ORACLE MISMATCH {e}", flush=True)
        return False
    print(f"{what}: sharded top-{k} == oracle top-{k} over all {C} chunks (queries {sample})",
          flush=True)
    return True


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
    sem_all = gen.semantic_lengths(seed, C, L)  # N4: packed shards of a semantic-length corpus
    for k, packed in ((10, False), (100, False), (10, True)):
        lens_use = sem_all if packed else lens_all
        flags = H.HIPER_PACKED if packed else 0
        c0, c1 = H.hiper_shard_range(C, world, rank)
        shard = torch.empty((c1 - c0, L, d), dtype=torch.bfloat16, device="cuda")
        device.corpus_(shard, seed, c0)
        idx = H.hiper_index_build(shard, lens_use[c0:c1], id_base=c0, flags=flags)
        s, i = H.hiper_maxsim_topk(idx, q, qlen, k, comm=comm)
        torch.cuda.synchronize()
        gs = [torch.empty_like(s) for _ in range(world)]
        gi = [torch.empty_like(i) for _ in range(world)]
        dist.all_gather(gs, s)
        dist.all_gather(gi, i)
        if rank == 0:
            full = torch.empty((C, L, d), dtype=torch.bfloat16, device="cuda")
            device.corpus_(full, seed, 0)
            fidx = H.hiper_index_build(full, lens_use, flags=flags)
            fs, fi = H.hiper_maxsim_topk(fidx, q, qlen, k)
            for r in range(world):
                same_i = torch.equal(gi[r], fi)
                same_s = torch.equal(gs[r].view(torch.int32), fs.view(torch.int32))
                print(f"k={k} packed={packed} rank{r}: ids equal {same_i}, scores bitwise {same_s}",
                      flush=True)
                ok &= same_i and same_s
            ok &= oracle_check(gs[0], gi[0], full, lens_use, q, qlen, k, f"k={k} packed={packed}")
            del full, fidx
        del shard, idx
    # ---- NEXT N3 across ranks: global pooled top-k1, owner re-scoring, one more all-gather
    Ct, Lt, dp, k1, k = 4003, 128, 768, 100, 10
    tl_all = gen.lengths(81, Ct, Lt, True)
    c0, c1 = H.hiper_shard_range(Ct, world, rank)
    to_dev16 = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
    qt2 = gen.queries(83, 21, Lq, d, corpus_seed=81, n_chunks=Ct, L=Lt, chunk_lens_fn=lambda c: tl_all[c])
    ql2 = gen.lengths(83, 21, Lq, True, stream=gen.QLEN)
    qp2 = gen.queries(83, 21, 1, dp, corpus_seed=82, n_chunks=Ct, L=1, sigma_q=np.float32(8.0))
    pidx = H.hiper_index_build(to_dev16(gen.corpus(82, c0, c1 - c0, 1, dp)), np.ones(c1 - c0, np.int32),
                               id_base=c0, flags=H.HIPER_POOLED)
    tidx = H.hiper_index_build(to_dev16(gen.corpus(81, c0, c1 - c0, Lt, d)), tl_all[c0:c1], id_base=c0)
    s2, i2 = H.hiper_two_stage_topk(pidx, tidx, to_dev16(qp2), to_dev16(qt2), ql2, k1, k, comm=comm)
    torch.cuda.synchronize()
    gs = [torch.empty_like(s2) for _ in range(world)]
    gi = [torch.empty_like(i2) for _ in range(world)]
    dist.all_gather(gs, s2)
    dist.all_gather(gi, i2)
    if rank == 0:
        fp = H.hiper_index_build(to_dev16(gen.corpus(82, 0, Ct, 1, dp)), np.ones(Ct, np.int32),
                                flags=H.HIPER_POOLED)
        ft = H.hiper_index_build(to_dev16(gen.corpus(81, 0, Ct, Lt, d)), tl_all)
        fs, fi = H.hiper_two_stage_topk(fp, ft, to_dev16(qp2), to_dev16(qt2), ql2, k1, k)
        for r in range(world):
            same = torch.equal(gi[r], fi) and torch.equal(gs[r].view(torch.int32), fs.view(torch.int32))
            print(f"two-stage rank{r}: equal to 1-GPU bitwise {same}", flush=True)
            ok &= same
    del pidx, tidx
    # ---- the same with the LAST rank holding an empty shard (advisor round 1): it still takes part in
    # both all-gathers, and every rank gets the answer over the other ranks' chunks
    Ce = 1500
    ce0, ce1 = H.hiper_shard_range(Ce, world - 1, rank) if rank < world - 1 else (Ce, Ce)
    tle = gen.lengths(81, Ce, Lt, True)
    pidx = H.hiper_index_build(to_dev16(gen.corpus(82, ce0, ce1 - ce0, 1, dp)), np.ones(ce1 - ce0, np.int32),
                               id_base=ce0, flags=H.HIPER_POOLED)
    tidx = H.hiper_index_build(to_dev16(gen.corpus(81, ce0, ce1 - ce0, Lt, d)), tle[ce0:ce1], id_base=ce0)
    s2, i2 = H.hiper_two_stage_topk(pidx, tidx, to_dev16(qp2), to_dev16(qt2), ql2, k1, k, comm=comm)
    torch.cuda.synchronize()
    gs = [torch.empty_like(s2) for _ in range(world)]
    gi = [torch.empty_like(i2) for _ in range(world)]
    dist.all_gather(gs, s2)
    dist.all_gather(gi, i2)
    if rank == 0:
        fp = H.hiper_index_build(to_dev16(gen.corpus(82, 0, Ce, 1, dp)), np.ones(Ce, np.int32),
                                flags=H.HIPER_POOLED)
        ft = H.hiper_index_build(to_dev16(gen.corpus(81, 0, Ce, Lt, d)), tle)
        fs, fi = H.hiper_two_stage_topk(fp, ft, to_dev16(qp2), to_dev16(qt2), ql2, k1, k)
        for r in range(world):
            same = torch.equal(gi[r], fi) and torch.equal(gs[r].view(torch.int32), fs.view(torch.int32))
            print(f"two-stage, empty last shard, rank{r}: equal to 1-GPU bitwise {same}", flush=True)
            ok &= same
    del pidx, tidx
    # ---- NEXT N2: full ColTrast loss with the gathered pooled candidates (min(N, W) rule)
    import oracle
    b, dp, Lc = 24, 768, 128
    for n_max in (b * world, b + 5, b):
        dt = gen.corpus(30 + rank, 0, b, Lc, d)
        qt = gen.queries(40 + rank, b, Lq, d, corpus_seed=30 + rank, n_chunks=b, L=Lc, diagonal=True,
                         sigma_q=gen.SIGMA_Q_HARD)
        ones_q, ones_d = np.full(b, Lq, np.int32), np.full(b, Lc, np.int32)
        pools = [gen.corpus(50 + r, 0, b, 1, dp)[:, 0] for r in range(world)]   # every rank's passages
        qpool = gen.queries(60 + rank, b, 1, dp, corpus_seed=50 + rank, n_chunks=b, L=1,
                            diagonal=True, sigma_q=np.float32(4.0))[:, 0]
        to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
        losses, S, m = H.hiper_coltrast_loss(to_dev(qt), ones_q, to_dev(dt), ones_d, to_dev(qpool),
                                             to_dev(pools[rank]), n_max=n_max, tau_li=1.0,
                                             tau_c=0.05, comm=comm, want_scores=True)
        got = losses.cpu().numpy().astype(np.float64)
        cands = np.stack(oracle.gather_candidates([list(p) for p in pools], rank, n_max))
        S_li = oracle.maxsim_matrix(oracle.norm_rows(qt), ones_q, oracle.norm_rows(dt), ones_d)
        L_li = oracle.infonce(S_li, tau=1.0)
        S_c = oracle.maxsim_matrix(oracle.norm_rows(qpool)[:, None], np.ones(b, np.int32),
                                   oracle.norm_rows(cands)[:, None], np.ones(len(cands), np.int32))
        L_c = oracle.infonce(S_c, tau=0.05)
        exp = (L_li, L_c, oracle.coltrast_total(L_li, L_c))
        good = m == len(cands) and all(abs(g - o) <= max(1e-4 * abs(o), 1e-7) for g, o in zip(got, exp))
        print(f"rank{rank} N={n_max}: m={m} losses={got.tolist()} oracle={list(exp)} ok={good}", flush=True)
        ok &= bool(good)
    okt = torch.tensor([int(ok)], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    ok = bool(okt.item())
    flag = torch.tensor([int(ok)], device="cuda")
    dist.broadcast(flag, 0)
    comm.close()
    dist.destroy_process_group()
    if rank == 0:
        print("DIST_OK" if flag.item() else "DIST_FAIL", flush=True)
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
