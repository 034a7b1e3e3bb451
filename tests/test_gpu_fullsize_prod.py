"""Full-size parity for the production launch configurations bench.py times (BASELINE configs[2..3]).

test_gpu_fullsize.py covers config 3 at Q = 1024, top-10.  This file covers the other paths the
bench runs at size, each with the same four checks:
  (1) every query whose planted target chunk is in the index finds it at rank 1;
  (2) lists are sorted, duplicate-free, inside the id range;
  (3) for sampled queries the ORACLE re-scores every returned (query, chunk) pair one by one, on
      operands checked bitwise against its own NORM of the raw inputs (R8 tolerance);
  (4) for those queries an independent torch/cuBLAS reference over the WHOLE corpus confirms no
      unreturned chunk beats the k-th returned score beyond tolerance.
Cases:
  * config 3 at Q = 64 (the adaptive L2-lockstep window of small query batches);
  * the packed layout (N4, HIPER_PACKED) at 1M semantic-length chunks -- also bitwise equal to the
    dense layout of the same corpus at full size;
  * config 4's per-rank launch at W = 2: a 1.8M-chunk dense shard (id_base 1.8M), Q = 1024, top-100
    (KR = 4 register lists, ~300 L2-band partitions);
  * config 4v: the whole 3.6M-chunk semantic corpus packed in place on ONE GPU (96 GB), Q = 256,
    top-100 ("3.6 million indexed scientific papers").
Config 3 also reports (never gates) SURVEY §8(c)'s informational deviation from exact float64 cosine.
"""
import numpy as np
import pytest

import oracle
from synth import gen
from tests._compare import assert_scores_close, score_tol
from tests._fullsize import (bits, exact_cosine, record_info, torch_ref_dense, torch_ref_packed)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

L, LQ, D = 256, 32, 128
SEED, QSEED = 1, 2   # bench.py defaults


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_04846_b200 as H
    H.lib()
    return H


def need_free(gb):
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < gb * 1e9:
        pytest.skip(f"needs ~{gb} GB of free HBM")


def check_lists(s, i, lo, hi, k):
    assert ((i >= lo) & (i < hi)).all()
    assert all(len(set(r)) == k for r in i.tolist())
    assert (np.diff(s, axis=1) <= 0).all()


def rescore_sampled(H, q, qlen, s, i, sample, get_rows, raw_rows, n_chunks, lens, what):
    """(3): oracle re-scoring of returned pairs on bitwise-checked operands.  get_rows(ids) -> NORM'd
    layout rows [len(ids)][L][D] uint16 from the device; raw_rows(ids) -> raw bf16 input bits."""
    qlay, _ = H.hiper_prepare_queries(q, qlen)
    qlay = bits(qlay)
    for qq in sample:
        raw_q = gen.queries(QSEED, 1, LQ, D, corpus_seed=SEED, n_chunks=n_chunks, L=L,
                            chunk_lens_fn=(None if lens is None else (lambda c: lens[c])),
                            start=qq)[0]
        assert np.array_equal(qlay[qq], oracle.norm_rows(raw_q))
        ids = i[qq]
        rows = get_rows(ids)
        raw = raw_rows(ids)
        S_o = np.empty(len(ids))
        for j, c in enumerate(ids.tolist()):
            n = L if lens is None else int(lens[c])
            assert np.array_equal(rows[j][:n], oracle.norm_rows(raw[j][:n])), (what, qq, c)
            S_o[j] = oracle.maxsim(qlay[qq], rows[j][:n])
        assert_scores_close(s[qq][None], S_o[None], [LQ], D, f"{what} query {qq}")
    return qlay


def no_better_unreturned(ref, s, i, sample, lo, what):
    """(4): ref [len(sample)][C] over the whole index (ids lo..lo+C-1)."""
    C = ref.shape[1]
    for r, qq in enumerate(sample):
        kth = s[qq][-1]
        others = np.setdiff1d(np.arange(C), i[qq] - lo)
        tol = score_tol(np.array([kth]), LQ, D)[0]
        assert ref[r, others].max() <= kth + tol, f"{what} query {qq}: an unreturned chunk beats the k-th"
        # and the returned scores agree with the reference
        got = ref[r, i[qq] - lo]
        assert (np.abs(got - s[qq]) <= score_tol(got, LQ, D)).all(), f"{what} query {qq}"


def dense_layout_rows(idx):
    lay = idx.layout()
    return lambda ids: bits(lay[torch.from_numpy(np.asarray(ids)).cuda()])


def raw_dense_rows():
    return lambda ids: gen.f32_to_bf16_bits(gen.corpus_tokens_f32(SEED, np.asarray(ids), L, D))


# ------------------------------------------------------------------------------------------------
def test_config3_q64_full_size(H):
    """BASELINE configs[2] at its other query batch, Q = 64 (adaptive lockstep window)."""
    need_free(75)
    C, Q, K = 1_000_000, 64, 10
    from synth import device
    corpus = torch.empty((C, L, D), dtype=torch.bfloat16, device="cuda")
    device.corpus_(corpus, SEED, 0)
    idx = H.hiper_index_build(corpus, np.full(C, L, np.int32), flags=H.HIPER_BORROW_TOKENS)
    q = torch.empty((Q, LQ, D), dtype=torch.bfloat16, device="cuda")
    device.queries_(q, QSEED, corpus_seed=SEED, n_chunks=C, L=L)
    qlen = np.full(Q, LQ, np.int32)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, q, qlen, K)]
    tgt = gen.query_targets(QSEED, Q, C, False)
    assert (i[:, 0] == tgt).all()
    check_lists(s, i, 0, C, K)
    # Q = 64 is a prefix of bench's Q = 1024 batch: batch invariance (P14) -- same scores bitwise
    q2 = torch.empty((1024, LQ, D), dtype=torch.bfloat16, device="cuda")
    device.queries_(q2, QSEED, corpus_seed=SEED, n_chunks=C, L=L)
    s2, i2 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, q2, np.full(1024, LQ, np.int32), K)]
    assert np.array_equal(i2[:Q], i) and np.array_equal(s2[:Q].view(np.uint32), s.view(np.uint32))
    sample = [0, 1, 33, 63]
    qlay = rescore_sampled(H, q, qlen, s, i, sample, dense_layout_rows(idx), raw_dense_rows(), C,
                           None, "config3 Q=64")
    lay = idx.layout()
    qrows = torch.from_numpy(qlay[sample].reshape(-1, D).view(np.int16)).cuda().view(torch.bfloat16).float()
    ref = torch_ref_dense(lay, torch.full((C,), L, dtype=torch.int32, device="cuda"), qrows, LQ)
    no_better_unreturned(ref, s, i, sample, 0, "config3 Q=64")
    # informational: deviation of the returned scores from exact float64 cosine on the raw inputs
    dev = []
    for qq in sample:
        raw_q = gen.queries(QSEED, 1, LQ, D, corpus_seed=SEED, n_chunks=C, L=L, start=qq)[0]
        raw_c = gen.f32_to_bf16_bits(gen.corpus_tokens_f32(SEED, i[qq], L, D))
        for j in range(K):
            ex = exact_cosine(gen.bf16_bits_to_f32(raw_q), gen.bf16_bits_to_f32(raw_c[j]))
            dev.append((abs(s[qq][j] - ex), abs(s[qq][j] - ex) / abs(ex)))
    dev = np.array(dev)
    record_info("config3_q64_vs_exact_cosine", {
        "pairs": len(dev), "max_abs": float(dev[:, 0].max()), "max_rel": float(dev[:, 1].max()),
        "mean_abs": float(dev[:, 0].mean()), "bound_2^-7*len_q": LQ * 2.0 ** -7})
    del corpus, idx, lay, ref


def test_packed_1m_semantic_full_size(H):
    """N4 at 1M semantic-length chunks (bench --workload config3v): packed == dense bitwise, and
    parity with the oracle."""
    need_free(100)
    C, Q, K = 1_000_000, 1024, 10
    from synth import device
    lens = gen.semantic_lengths(SEED, C, L)
    corpus = torch.empty((C, L, D), dtype=torch.bfloat16, device="cuda")
    device.corpus_(corpus, SEED, 0)
    pidx = H.hiper_index_build(corpus, lens, flags=H.HIPER_PACKED)        # a packed copy
    torch.cuda.synchronize()
    didx = H.hiper_index_build(corpus, lens, flags=H.HIPER_BORROW_TOKENS)  # dense, NORM'd in place
    q = torch.empty((Q, LQ, D), dtype=torch.bfloat16, device="cuda")
    lens_dev = torch.from_numpy(lens).cuda()
    device.queries_(q, QSEED, corpus_seed=SEED, n_chunks=C, L=L, chunk_lens=lens_dev)
    qlen = np.full(Q, LQ, np.int32)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(pidx, q, qlen, K)]
    sd, id_ = [t.cpu().numpy() for t in H.hiper_maxsim_topk(didx, q, qlen, K)]
    assert np.array_equal(i, id_) and np.array_equal(s.view(np.uint32), sd.view(np.uint32))
    tgt = gen.query_targets(QSEED, Q, C, False)
    assert (i[:, 0] == tgt).all()
    check_lists(s, i, 0, C, K)
    sample = [0, 5, 700, 1023]
    qlay = rescore_sampled(H, q, qlen, s, i, sample, dense_layout_rows(didx), raw_dense_rows(), C,
                           lens, "config3v packed")
    qrows = torch.from_numpy(qlay[sample].reshape(-1, D).view(np.int16)).cuda().view(torch.bfloat16).float()
    ref = torch_ref_dense(didx.layout(), lens_dev, qrows, LQ)
    no_better_unreturned(ref, s, i, sample, 0, "config3v packed")
    del corpus, pidx, didx, ref


def test_config4_shard_top100_full_size(H):
    """Config 4's per-rank launch at W = 2: rank 1's 1.8M-chunk shard of the 3.6M corpus (118 GB,
    id_base = 1.8M), Q = 1024, top-100 -- the bench's k = 100 path (KR = 4, banded partitions)."""
    need_free(125)
    CT, W, Q, K = 3_600_000, 2, 1024, 100
    c0, c1 = CT // W, CT
    C = c1 - c0
    from synth import device
    corpus = torch.empty((C, L, D), dtype=torch.bfloat16, device="cuda")
    device.corpus_(corpus, SEED, c0)
    idx = H.hiper_index_build(corpus, np.full(C, L, np.int32), id_base=c0, flags=H.HIPER_BORROW_TOKENS)
    q = torch.empty((Q, LQ, D), dtype=torch.bfloat16, device="cuda")
    device.queries_(q, QSEED, corpus_seed=SEED, n_chunks=CT, L=L)
    qlen = np.full(Q, LQ, np.int32)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, q, qlen, K)]
    tgt = gen.query_targets(QSEED, Q, CT, False)
    mine = (tgt >= c0) & (tgt < c1)
    assert mine.sum() > 400 and (i[mine, 0] == tgt[mine]).all()
    check_lists(s, i, c0, c1, K)
    lay = idx.layout()
    sample = [int(np.flatnonzero(mine)[0]), int(np.flatnonzero(~mine)[0]), 512, 1023]
    get_rows = lambda ids: bits(lay[torch.from_numpy(np.asarray(ids) - c0).cuda()])
    qlay = rescore_sampled(H, q, qlen, s, i, sample, get_rows, raw_dense_rows(), CT, None,
                           "config4 shard")
    qrows = torch.from_numpy(qlay[sample].reshape(-1, D).view(np.int16)).cuda().view(torch.bfloat16).float()
    ref = torch_ref_dense(lay, torch.full((C,), L, dtype=torch.int32, device="cuda"), qrows, LQ)
    no_better_unreturned(ref, s, i, sample, c0, "config4 shard")
    del corpus, idx, lay, ref


def test_config4v_3p6m_packed_one_gpu_top100(H):
    """The paper-scale 3.6M-chunk corpus (semantic lengths) packed in place on one GPU (bench
    --workload config4v at N = 1), Q = 256, top-100."""
    need_free(115)
    C, Q, K = 3_600_000, 256, 100
    from synth import device
    lens = gen.semantic_lengths(SEED, C, L)
    dst, n_rows = H.hiper_pack_dst_rows(lens)
    corpus = torch.empty((n_rows, D), dtype=torch.bfloat16, device="cuda")
    dst_dev, lens_dev = torch.from_numpy(dst).cuda(), torch.from_numpy(lens).cuda()
    device.corpus_packed_(corpus, SEED, 0, dst_dev, lens_dev, L)
    idx = H.hiper_index_build(corpus, lens, flags=H.HIPER_PACKED | H.HIPER_BORROW_TOKENS)
    q = torch.empty((Q, LQ, D), dtype=torch.bfloat16, device="cuda")
    device.queries_(q, QSEED, corpus_seed=SEED, n_chunks=C, L=L, chunk_lens=lens_dev)
    qlen = np.full(Q, LQ, np.int32)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, q, qlen, K)]
    tgt = gen.query_targets(QSEED, Q, C, False)
    assert (i[:, 0] == tgt).all()
    check_lists(s, i, 0, C, K)
    lay = idx.layout()                                                   # [n_rows][D]

    def get_rows(ids):
        out = np.zeros((len(ids), L, D), np.uint16)
        for j, c in enumerate(np.asarray(ids).tolist()):
            out[j, :lens[c]] = bits(lay[int(dst[c]):int(dst[c]) + int(lens[c])])
        return out

    sample = [0, 100, 255]
    qlay = rescore_sampled(H, q, qlen, s, i, sample, get_rows, raw_dense_rows(), C, lens,
                           "config4v packed 3.6M")
    # packed row -> chunk map (real token rows only), then the whole-corpus reference
    cid = torch.repeat_interleave(torch.arange(C, device="cuda"), lens_dev.long())
    starts = torch.cumsum(lens_dev.long(), 0) - lens_dev.long()
    off = torch.arange(cid.numel(), device="cuda") - starts[cid]
    row_chunk = torch.full((n_rows,), -1, dtype=torch.int64, device="cuda")
    row_chunk[dst_dev[cid] + off] = cid
    del cid, starts, off
    qrows = torch.from_numpy(qlay[sample].reshape(-1, D).view(np.int16)).cuda().view(torch.bfloat16).float()
    ref = torch_ref_packed(lay, row_chunk, C, qrows, LQ)
    no_better_unreturned(ref, s, i, sample, 0, "config4v packed 3.6M")
    del corpus, idx, lay, ref, row_chunk


def test_two_stage_3p6m_full_size(H):
    """bench.py --workload two_stage at size: 3.6M pooled (768-d) + the same chunks' packed token rows,
    Q = 1024, k1 = 100, k = 10.  Stage 1 is checked against a torch/cuBLAS pooled-cosine reference over
    the whole pooled index (its top-100 set, up to near-ties); stage 2 against the oracle's exact MaxSim
    of every candidate of the sampled queries (SPEC.md:268-276 rerank)."""
    need_free(115)
    C, Q, K1, K, DP = 3_600_000, 1024, 100, 10, 768
    from synth import device
    lens = gen.semantic_lengths(SEED, C, L)
    dst, n_rows = H.hiper_pack_dst_rows(lens)
    tok = torch.empty((n_rows, D), dtype=torch.bfloat16, device="cuda")
    lens_dev = torch.from_numpy(lens).cuda()
    device.corpus_packed_(tok, SEED, 0, torch.from_numpy(dst).cuda(), lens_dev, L)
    tidx = H.hiper_index_build(tok, lens, flags=H.HIPER_PACKED | H.HIPER_BORROW_TOKENS)
    PSEED = SEED + 1000                       # bench.py's pooled corpus seed
    pool = torch.empty((C, 1, DP), dtype=torch.bfloat16, device="cuda")
    device.corpus_(pool, PSEED, 0)
    pidx = H.hiper_index_build(pool, np.ones(C, np.int32), flags=H.HIPER_POOLED | H.HIPER_BORROW_TOKENS)
    qt = torch.empty((Q, LQ, D), dtype=torch.bfloat16, device="cuda")
    device.queries_(qt, QSEED, corpus_seed=SEED, n_chunks=C, L=L, chunk_lens=lens_dev)
    qp = torch.empty((Q, 1, DP), dtype=torch.bfloat16, device="cuda")
    device.queries_(qp, QSEED, corpus_seed=PSEED, n_chunks=C, L=1)
    qlen = np.full(Q, LQ, np.int32)
    s, i = [t.cpu().numpy() for t in H.hiper_two_stage_topk(pidx, tidx, qp, qt, qlen, K1, K)]
    tgt = gen.query_targets(QSEED, Q, C, False)
    assert (i[:, 0] == tgt).all()
    check_lists(s, i, 0, C, K)
    # stage 1 vs a cuBLAS reference over all 3.6M pooled rows (the exact top-100 set up to near-ties)
    s1, i1 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(pidx, qp, np.ones(Q, np.int32), K1)]
    sample = [0, 511, 1023]
    # (the pooled query rows: the oracle's NORM of the raw inputs, which the pooled tests show the
    # library reproduces bitwise)
    qpb = np.stack([oracle.norm_rows(gen.queries(QSEED, 1, 1, DP, corpus_seed=PSEED, n_chunks=C, L=1,
                                                 start=qq)[0, 0]) for qq in sample])
    torch.backends.cuda.matmul.allow_tf32 = False
    qrow = torch.from_numpy(qpb.view(np.int16)).cuda().view(torch.bfloat16).float()
    ref = (qrow @ pidx.layout()[:, 0].float().T).cpu().numpy().astype(np.float64)   # [3][C]
    for r, qq in enumerate(sample):
        kth = np.sort(ref[r])[::-1][K1 - 1]
        tol = 2e-3 * abs(kth) + DP * 2.0 ** -24
        got = ref[r][i1[qq]]
        assert (got >= kth - tol).all(), f"stage 1 query {qq}: a returned candidate below the 100th"
        others = np.setdiff1d(np.arange(C), i1[qq])
        assert ref[r][others].max() <= s1[qq][-1] + tol, f"stage 1 query {qq}: a better unreturned chunk"
    # stage 2: the oracle's exact MaxSim of each sampled query's 100 candidates, re-sorted
    qlay, _ = H.hiper_prepare_queries(qt, qlen)
    qlay = bits(qlay)
    lay = tidx.layout()
    for qq in sample:
        cands = i1[qq]
        S2 = np.empty(len(cands))
        for jx, c in enumerate(cands.tolist()):
            rows = bits(lay[int(dst[c]):int(dst[c]) + int(lens[c])])
            raw = gen.f32_to_bf16_bits(gen.corpus_tokens_f32(SEED, [c], L, D))[0][:lens[c]]
            assert np.array_equal(rows, oracle.norm_rows(raw))
            S2[jx] = oracle.maxsim(qlay[qq], rows)
        o_s, o_i = oracle.topk(S2, cands.astype(np.int64), K)
        tol = score_tol(o_s, LQ, D)
        assert (np.abs(s[qq] - o_s) <= tol).all(), (qq, s[qq], o_s)
        for r_ in range(K):   # ids equal except inside near-tie runs
            if i[qq][r_] != o_i[r_]:
                assert abs(S2[list(cands).index(i[qq][r_])] - o_s[r_]) <= tol[r_]
    del tok, tidx, pool, pidx, lay
