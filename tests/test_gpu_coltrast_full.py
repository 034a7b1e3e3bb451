"""NEXT N2 on one GPU: the full ColTrast loss L = (L_LI + L_C)/2 vs the oracle.
(The gathered multi-rank case runs in tests/dist_topk_check.py under torchrun.)"""
import numpy as np
import pytest

import oracle
from synth import gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_04846_b200 as H
    return H


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def oracle_full(q, ql, d, dl, qp, dpool_cands, tau_li, tau_c):
    S_li = oracle.maxsim_matrix(oracle.norm_rows(q), ql, oracle.norm_rows(d), dl)
    L_li = oracle.infonce(S_li, tau=tau_li)
    qn = oracle.norm_rows(qp)[:, None]
    cn = oracle.norm_rows(dpool_cands)[:, None]
    S_c = oracle.maxsim_matrix(qn, np.ones(len(qn), np.int32), cn, np.ones(len(cn), np.int32))
    L_c = oracle.infonce(S_c, tau=tau_c)
    return L_li, L_c, oracle.coltrast_total(L_li, L_c), S_c


@pytest.mark.parametrize("b,dp,tau_c", [(24, 4096, 0.05), (37, 768, 0.05), (64, 128, 1.0)])
def test_full_coltrast_loss_single_rank(H, b, dp, tau_c):
    L, Lq = 128, 32
    d = gen.corpus(7, 0, b, L, 128)
    q = gen.queries(8, b, Lq, 128, corpus_seed=7, n_chunks=b, L=L, diagonal=True,
                    sigma_q=gen.SIGMA_Q_HARD)
    dl = gen.lengths(7, b, L, True)
    ql = gen.lengths(8, b, Lq, True, stream=gen.QLEN)
    # pooled embeddings: a planted pair structure (query i near passage i) at dimension dp
    dpool = gen.corpus(9, 0, b, 1, dp)[:, 0]
    qpool = gen.queries(10, b, 1, dp, corpus_seed=9, n_chunks=b, L=1, diagonal=True,
                        sigma_q=np.float32(4.0))[:, 0]
    losses, S, m = H.hiper_coltrast_loss(to_dev(q), ql, to_dev(d), dl, to_dev(qpool), to_dev(dpool),
                                         n_max=4 * b, tau_li=1.0, tau_c=tau_c, want_scores=True)
    assert m == b
    got = losses.cpu().numpy().astype(np.float64)
    L_li, L_c, L_tot, S_c = oracle_full(q, ql, d, dl, qpool, dpool, 1.0, tau_c)
    for g, o, name in zip(got, (L_li, L_c, L_tot), ("L_LI", "L_C", "L")):
        assert abs(g - o) <= max(1e-4 * abs(o), 1e-7), (name, g, o)
    assert np.all(np.abs(S.cpu().numpy() - S_c) <= np.maximum(2e-3 * np.abs(S_c), dp * 2.0 ** -24))
    assert got[2] == np.float32(0.5) * (np.float32(got[0]) + np.float32(got[1]))


def test_full_coltrast_errors(H):
    b = 8
    z = np.zeros((b, 4, 128), np.uint16)
    zp = np.zeros((b, 64), np.uint16)
    with pytest.raises(H.HiperError) as e:
        H.hiper_coltrast_loss(to_dev(z), np.ones(b), to_dev(z), np.ones(b), to_dev(zp), to_dev(zp),
                              n_max=4)
    assert e.value.name == "HIPER_ERR_INVALID_ARG"   # SPEC NTooSmall
    with pytest.raises(H.HiperError) as e:
        H.hiper_coltrast_loss(to_dev(z), np.ones(b), to_dev(z), np.ones(b), to_dev(zp), to_dev(zp),
                              n_max=8, tau_c=0.0)
    assert e.value.name == "HIPER_ERR_BAD_TEMPERATURE"


@pytest.mark.parametrize("world,b,dp,n_max", [(3, 24, 768, 72), (3, 24, 768, 29), (4, 17, 80, 40),
                                              (2, 33, 4096, 66), (5, 8, 768, 8)])
def test_full_coltrast_loss_simulated_ranks(H, world, b, dp, n_max):
    """N2 with `world` simulated ranks on ONE GPU: every rank's pooled passages live in one buffer and
    the library's candidate gather (the kernel that reads the peers' windows over NVLink on a real
    node) builds each rank's min(N, W) candidates in (local first, then rank, position) order; the
    losses equal the oracle's (SPEC.md:321-329 gather_candidates)."""
    L, Lq = 64, 32
    pools = [gen.corpus(50 + r, 0, b, 1, dp)[:, 0] for r in range(world)]
    allp = np.stack(pools)                                           # [world][b][dp]
    for rank in range(world):
        d = gen.corpus(30 + rank, 0, b, L, 128)
        q = gen.queries(40 + rank, b, Lq, 128, corpus_seed=30 + rank, n_chunks=b, L=L,
                        diagonal=True, sigma_q=gen.SIGMA_Q_HARD)
        dl = gen.lengths(30 + rank, b, L, True)
        ql = gen.lengths(40 + rank, b, Lq, True, stream=gen.QLEN)
        qpool = gen.queries(60 + rank, b, 1, dp, corpus_seed=50 + rank, n_chunks=b, L=1,
                            diagonal=True, sigma_q=np.float32(4.0))[:, 0]
        losses, S, m = H.hiper_coltrast_loss_simulated(
            to_dev(q), ql, to_dev(d), dl, to_dev(qpool), to_dev(allp), world=world, rank=rank,
            n_max=n_max, tau_li=1.0, tau_c=0.05, want_scores=True)
        cands = np.stack(oracle.gather_candidates([list(p) for p in pools], rank, n_max))
        assert m == len(cands) == min(n_max, world * b)
        L_li, L_c, L_tot, S_c = oracle_full(q, ql, d, dl, qpool, cands, 1.0, 0.05)
        got = losses.cpu().numpy().astype(np.float64)
        for g, o, name in zip(got, (L_li, L_c, L_tot), ("L_LI", "L_C", "L")):
            assert abs(g - o) <= max(1e-4 * abs(o), 1e-7), (rank, name, g, o)
        assert np.all(np.abs(S.cpu().numpy() - S_c) <= np.maximum(2e-3 * np.abs(S_c), dp * 2.0 ** -24))
