"""The supported domain of SURVEY §8(b) through the C ABI: token dim % 16 == 0 (<= 256), q_max_len
<= 128, chunk max_len <= 512, any k <= 128 -- every shape against the oracle on the exact operands.

Kernel paths exercised: query slots of 32 / 64 / 128 rows (a query spanning 1, 2 or 4 warps of TMEM
lanes, their sums added through shared memory), chunks of up to 512 tokens (two MMA halves per chunk,
the running max carried across the two accumulators), dims that are not a multiple of 64 (TMA
zero-fill of the last 64-wide box), single-token chunks scored by the token kernel (a
32-token query against a one-token doc is the dot of the summed query rows with it).
"""
import numpy as np
import pytest

import oracle
from synth import gen
from tests._compare import assert_loss_close, assert_scores_close, assert_topk_ok

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
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def case(C, L, Q, Lq, d, seed, kind="planted", var=True, dtype="bf16"):
    corp = gen.corpus(seed, 0, C, L, d, kind=kind, dtype=dtype)
    clen = gen.lengths(seed, C, L, var)
    q = gen.queries(seed + 1, Q, Lq, d, corpus_seed=seed, n_chunks=C, L=L,
                    chunk_lens_fn=lambda c: clen[c], kind=kind, corpus_kind=kind, dtype=dtype)
    qlen = gen.lengths(seed + 1, Q, Lq, var, stream=gen.QLEN)
    return corp, clen, q, qlen


def oracle_S(H, idx, q, qlen, Lq):
    """Oracle scores on the device layouts (checked bitwise against the oracle's own NORM)."""
    lay = bits(idx.layout().clone())
    ql, _ = H.hiper_prepare_queries(to_dev(q), qlen)
    ql = bits(ql)
    qs = 32 if Lq <= 32 else (64 if Lq <= 64 else 128)
    assert ql.shape[1] == qs
    for r in range(len(qlen)):
        assert np.array_equal(ql[r, :qlen[r]], oracle.norm_rows(q[r, :qlen[r]]))
        assert not ql[r, qlen[r]:].any()
    return ql[:len(qlen)], lay


SHAPES = [  # (Lq, L, d)
    (64, 128, 128), (128, 256, 128), (32, 384, 128), (100, 512, 128), (32, 128, 192),
    (32, 128, 256), (64, 200, 80), (128, 512, 256), (48, 48, 48), (32, 1, 128), (17, 257, 64),
]


@pytest.mark.parametrize("Lq,L,d", SHAPES)
def test_dense_scores_domain(H, Lq, L, d):
    C, Q = 61, 13
    corp, clen, q, qlen = case(C, L, Q, Lq, d, seed=5 + L + d)
    idx = H.hiper_index_build(to_dev(corp), clen)
    ql, lay = oracle_S(H, idx, q, qlen, Lq)
    for c in range(C):
        assert np.array_equal(lay[c, :clen[c]], oracle.norm_rows(corp[c, :clen[c]]))
    S = H.hiper_maxsim_scores(idx, to_dev(q), qlen).cpu().numpy()
    S_o = oracle.maxsim_matrix(ql, qlen, lay, clen)
    assert_scores_close(S, S_o, qlen, d, f"Lq={Lq} L={L} d={d}")
    assert np.abs(S - S_o).max() <= 1e-5 * max(1.0, np.abs(S_o).max()) * Lq  # diagnostic tier


@pytest.mark.parametrize("Lq,L,d,k", [(64, 256, 128, 10), (128, 512, 128, 100), (32, 384, 192, 16),
                                      (100, 128, 256, 128), (32, 1, 128, 5)])
def test_topk_domain(H, Lq, L, d, k):
    C, Q = 400, 11
    corp, clen, q, qlen = case(C, L, Q, Lq, d, seed=7 + L, var=True)
    idx = H.hiper_index_build(to_dev(corp), clen, id_base=500)
    ql, lay = oracle_S(H, idx, q, qlen, Lq)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), qlen, k)]
    S_o = oracle.maxsim_matrix(ql, qlen, lay, clen)
    ids = np.arange(C, dtype=np.int64) + 500
    for r in range(Q):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, qlen[r], d, f"Lq={Lq} L={L} d={d} q{r}")


def test_single_token_docs_closed_form(H):
    """SURVEY P3 through the kernel: a 32-token query vs one-token chunks (a TOKEN index with
    max_len 1, not HIPER_POOLED) is S = <sum_i q_i, d> on the NORM'd rows."""
    C, Q, d = 300, 7, 128
    corp, clen, q, qlen = case(C, 1, Q, 32, d, seed=41, var=False)
    idx = H.hiper_index_build(to_dev(corp), clen)
    ql, lay = oracle_S(H, idx, q, qlen, 32)
    S = H.hiper_maxsim_scores(idx, to_dev(q), qlen).cpu().numpy()
    qsum = oracle.bf16_bits_to_f64(ql).sum(axis=1)                    # [Q][d]
    closed = qsum @ oracle.bf16_bits_to_f64(lay[:, 0]).T              # [Q][C]
    assert_scores_close(S, closed, qlen, d, "P3 closed form")


@pytest.mark.parametrize("Lq", [64, 128])
def test_batch_invariance_multiwarp_queries(H, Lq):
    """P14 with queries spanning 2 / 4 warps: a query scored alone is bitwise the same query inside a
    batch (fixed cross-warp summation order)."""
    corp, clen, q, qlen = case(90, 256, 9, Lq, 128, seed=61)
    idx = H.hiper_index_build(to_dev(corp), clen)
    S = H.hiper_maxsim_scores(idx, to_dev(q), qlen).cpu().numpy()
    for r in (0, 4, 8):
        S1 = H.hiper_maxsim_scores(idx, to_dev(q[r:r + 1]), qlen[r:r + 1]).cpu().numpy()
        assert np.array_equal(S1[0].view(np.uint32), S[r].view(np.uint32))


@pytest.mark.parametrize("Lq", [64, 128])
def test_packed_equals_dense_multiwarp_queries(H, Lq):
    """N4 packed layout with long queries: bitwise the dense layout (top-k and dense scores)."""
    C, Q, L, d = 700, 10, 256, 128
    corp = gen.corpus(71, 0, C, L, d)
    clen = gen.semantic_lengths(71, C, L)
    q = gen.queries(72, Q, Lq, d, corpus_seed=71, n_chunks=C, L=L, chunk_lens_fn=lambda c: clen[c])
    qlen = gen.lengths(72, Q, Lq, True, stream=gen.QLEN)
    dense = H.hiper_index_build(to_dev(corp), clen)
    packed = H.hiper_index_build(to_dev(corp), clen, flags=H.HIPER_PACKED)
    for k in (10, 100):
        s0, i0 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(dense, to_dev(q), qlen, k)]
        s1, i1 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(packed, to_dev(q), qlen, k)]
        assert np.array_equal(i0, i1) and np.array_equal(s0.view(np.uint32), s1.view(np.uint32))
    S0 = H.hiper_maxsim_scores(dense, to_dev(q), qlen).cpu().numpy()
    S1 = H.hiper_maxsim_scores(packed, to_dev(q), qlen).cpu().numpy()
    assert np.array_equal(S0.view(np.uint32), S1.view(np.uint32))


@pytest.mark.parametrize("Lq,Ld,d", [(64, 384, 128), (128, 512, 256), (40, 100, 96)])
def test_coltrast_loss_domain(H, Lq, Ld, d):
    B = 24
    corp, clen, q, qlen = case(B, Ld, B, Lq, d, seed=81, var=True)
    q = gen.queries(82, B, Lq, d, corpus_seed=81, n_chunks=B, L=Ld, chunk_lens_fn=lambda c: clen[c],
                    diagonal=True, sigma_q=gen.SIGMA_Q_HARD)
    S, L = H.hiper_coltrast_scores_loss(to_dev(q), qlen, to_dev(corp), clen, temperature=0.5)
    S, L = S.cpu().numpy(), float(L.item())
    qn = np.zeros_like(q)
    for r in range(B):
        qn[r, :qlen[r]] = oracle.norm_rows(q[r, :qlen[r]])
    cn = np.zeros_like(corp)
    for c in range(B):
        cn[c, :clen[c]] = oracle.norm_rows(corp[c, :clen[c]])
    S_o = oracle.maxsim_matrix(qn, qlen, cn, clen)
    assert_scores_close(S, S_o, qlen, d, "coltrast domain S")
    assert_loss_close(L, oracle.infonce(S_o, tau=0.5), "coltrast domain loss")


def test_domain_errors(H):
    z = lambda *s: torch.zeros(s, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(H.HiperError) as e:          # dim not a multiple of 16
        H.hiper_index_build(z(4, 16, 72), np.full(4, 16, np.int32))
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"
    with pytest.raises(H.HiperError) as e:          # dim > 256 on token rows
        H.hiper_index_build(z(4, 16, 320), np.full(4, 16, np.int32))
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"
    with pytest.raises(H.HiperError) as e:          # max_len > 512
        H.hiper_index_build(z(2, 528, 64), np.full(2, 528, np.int32))
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"
    idx = H.hiper_index_build(z(4, 16, 64) + 1, np.full(4, 16, np.int32))
    with pytest.raises(H.HiperError) as e:          # q_max_len > 128
        H.hiper_maxsim_topk(idx, z(2, 129, 64) + 1, np.full(2, 129, np.int32), 3)
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"
    with pytest.raises(H.HiperError) as e:          # HIPER_POOLED needs max_len 1
        H.hiper_index_build(z(4, 2, 64) + 1, np.full(4, 2, np.int32), flags=H.HIPER_POOLED)
    assert e.value.name == "HIPER_ERR_INVALID_ARG"
