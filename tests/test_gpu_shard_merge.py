"""a8 on ONE GPU, through the C ABI: the cross-GPU merge without NCCL.

hiper_maxsim_topk(comm != NULL) is: each rank's local top-k keys (hiper_maxsim_topk_keys) -> one
ncclAllGather into [W][n_q][k] -> the merge + decode kernel on every rank (hiper_topk_merge_keys).
Here W shard indexes (contiguous chunk ranges, id_base = shard offset, as bench.py shards) live on
one GPU; their key lists are stacked [W][n_q][k] exactly as ncclAllGather lays them out and merged
by the library's own kernel.  The result must be
  * the oracle's exact top-k over the WHOLE corpus (R8 near-tie rule; §2.3 "nearest
    neighbors" over the whole store), and
  * bitwise the unsharded single-index call (sharding invariance P13).
Covers dense, packed (N4) and pooled (a12) shards, k = 10 / 100, W = 2 / 3 / 4, and an empty shard.
"""
import functools

import numpy as np
import pytest

import oracle
from synth import gen
from tests._compare import assert_topk_ok

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_04846_b200 as H
    H.lib()
    return H


def bits(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def shard_bounds(C, W, empty=False):
    """bench.py's plan (rank r owns [r*C//W, (r+1)*C//W)); `empty` makes shard 1 empty."""
    b = [r * C // W for r in range(W + 1)]
    if empty:
        b[1] = b[0]
    return b


@functools.lru_cache(maxsize=None)
def _oracle_scores(packed, C, L, Q, Lq, d):
    """Oracle S over the whole corpus from the raw inputs (its own NORM; cached per corpus)."""
    corp = gen.corpus(21, 0, C, L, d)
    clen = gen.semantic_lengths(21, C, L) if packed else gen.lengths(21, C, L, True)
    q = gen.queries(22, Q, Lq, d, corpus_seed=21, n_chunks=C, L=L, chunk_lens_fn=lambda c: clen[c])
    qlen = gen.lengths(22, Q, Lq, True, stream=gen.QLEN)
    cn = np.zeros((C, L, d), np.uint16)
    for c in range(C):
        cn[c, :clen[c]] = oracle.norm_rows(corp[c, :clen[c]])
    qn = np.zeros((Q, Lq, d), np.uint16)
    for r in range(Q):
        qn[r, :qlen[r]] = oracle.norm_rows(q[r, :qlen[r]])
    return oracle.maxsim_matrix(qn, qlen, cn, clen)


def merged_via_keys(H, make_index, q, qlen, k, bounds):
    keys = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        ix = make_index(a, b)
        keys.append(H.hiper_maxsim_topk_keys(ix, q, qlen, k))
        # one list alone decodes to the shard's own hiper_maxsim_topk answer
        s1, i1 = H.hiper_topk_merge_keys(keys[-1][None].contiguous(), k)
        s0, i0 = H.hiper_maxsim_topk(ix, q, qlen, k)
        assert torch.equal(i1, i0) and torch.equal(s1.view(torch.int32), s0.view(torch.int32))
    lists = torch.stack(keys).contiguous()       # [W][n_q][k], the all-gather layout
    return [t.cpu().numpy() for t in H.hiper_topk_merge_keys(lists, k)]


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("W,k,empty", [(2, 10, False), (3, 100, False), (4, 10, True)])
def test_token_shards_merge_vs_oracle(H, packed, W, k, empty):
    C, L, Q, Lq, d = 2003, 128, 13, 32, 128
    corp = gen.corpus(21, 0, C, L, d)
    clen = gen.semantic_lengths(21, C, L) if packed else gen.lengths(21, C, L, True)
    q = gen.queries(22, Q, Lq, d, corpus_seed=21, n_chunks=C, L=L, chunk_lens_fn=lambda c: clen[c])
    qlen = gen.lengths(22, Q, Lq, True, stream=gen.QLEN)
    flags = H.HIPER_PACKED if packed else 0
    qd = to_dev(q)

    def make_index(a, b):
        return H.hiper_index_build(to_dev(corp[a:b]), clen[a:b], id_base=a, flags=flags)

    full = H.hiper_index_build(to_dev(corp), clen, flags=flags)
    s_ref, i_ref = [t.cpu().numpy() for t in H.hiper_maxsim_topk(full, qd, qlen, k)]
    s, i = merged_via_keys(H, make_index, qd, qlen, k, shard_bounds(C, W, empty))
    assert np.array_equal(i, i_ref)
    assert np.array_equal(s.view(np.uint32), s_ref.view(np.uint32))
    # the oracle over the whole corpus, on the exact operands (layouts checked bitwise)
    qlay, _ = H.hiper_prepare_queries(qd, qlen)
    qlay = bits(qlay)[:Q]
    for r in range(Q):
        assert np.array_equal(qlay[r, :qlen[r]], oracle.norm_rows(q[r, :qlen[r]]))
    S_o = _oracle_scores(packed, C, L, Q, Lq, d)
    ids = np.arange(C, dtype=np.int64)
    for r in range(Q):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, qlen[r], d, f"W={W} k={k} query {r}")


@pytest.mark.parametrize("W,k", [(2, 10), (4, 16), (3, 100)])
def test_pooled_shards_merge_vs_oracle(H, W, k):
    C, Q, dp = 3001, 21, 768
    corp = gen.corpus(31, 0, C, 1, dp)
    q = gen.queries(32, Q, 1, dp, corpus_seed=31, n_chunks=C, L=1, sigma_q=np.float32(8.0))
    ones_c, ones_q = np.ones(C, np.int32), np.ones(Q, np.int32)
    qd = to_dev(q)

    def make_index(a, b):
        return H.hiper_index_build(to_dev(corp[a:b]), ones_c[a:b], id_base=a, flags=H.HIPER_POOLED)

    full = make_index(0, C)
    s_ref, i_ref = [t.cpu().numpy() for t in H.hiper_maxsim_topk(full, qd, ones_q, k)]
    s, i = merged_via_keys(H, make_index, qd, ones_q, k, shard_bounds(C, W))
    assert np.array_equal(i, i_ref)
    assert np.array_equal(s.view(np.uint32), s_ref.view(np.uint32))
    S_o = oracle.maxsim_matrix(oracle.norm_rows(q), ones_q, oracle.norm_rows(corp), ones_c)
    ids = np.arange(C, dtype=np.int64)
    for r in range(Q):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, 1, dp, f"pooled W={W} query {r}")


def test_merge_keys_edge_cases(H):
    # zero lists -> all padding; k > every list's real entries -> padding tail
    out = H.hiper_topk_merge_keys(torch.empty((0, 3, 5), dtype=torch.int64, device="cuda"), 5)
    assert (out[1].cpu().numpy() == -1).all() and np.isneginf(out[0].cpu().numpy()).all()
    with pytest.raises(H.HiperError):
        H.hiper_topk_merge_keys(torch.zeros((1, 2, 129), dtype=torch.int64, device="cuda"), 129)
