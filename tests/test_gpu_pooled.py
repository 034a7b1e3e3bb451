"""Pooled single-vector limit case (a12, BASELINE.json configs[4]): Lq = Ld = 1, dim 768.

MaxSim with one token per side is the dot of NORM'd vectors (cosine); the
kernel is a K-pipelined pair GEMM with a fused per-query top-k."""
import numpy as np
import pytest

import oracle
from synth import gen
from tests._compare import assert_scores_close, assert_topk_ok, score_tol

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
D = 768


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_04846_b200 as H
    return H


def to_dev(a):
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def case(C, Q, kind="planted", dtype="bf16", seed=11, qseed=12):
    corp = gen.corpus(seed, 0, C, 1, D, kind=kind, dtype=dtype)                    # [C][1][D]
    q = gen.queries(qseed, Q, 1, D, corpus_seed=seed, n_chunks=C, L=1, kind=kind,
                    corpus_kind=kind, dtype=dtype)                                  # [Q][1][D]
    return corp, q


@pytest.mark.parametrize("C,Q,dtype", [(1000, 8, "f32"), (777, 300, "bf16"), (256, 256, "bf16")])
def test_pooled_dense_scores(H, C, Q, dtype):
    corp, q = case(C, Q, kind="iid", dtype=dtype)
    idx = H.hiper_index_build(to_dev(corp), np.ones(C, np.int32), flags=H.HIPER_POOLED)
    assert idx.ld_pad == 1
    lay = bits(idx.layout().clone())
    assert np.array_equal(lay[:, 0], oracle.norm_rows(corp[:, 0]))     # layout bitwise (a1)
    S = H.hiper_maxsim_scores(idx, to_dev(q), np.ones(Q, np.int32)).cpu().numpy()
    qn = oracle.norm_rows(q[:, 0])
    S_o = oracle.maxsim_matrix(qn[:, None], np.ones(Q, np.int32), lay, np.ones(C, np.int32))
    assert_scores_close(S, S_o, np.ones(Q), D, "pooled dense")
    assert np.all(np.abs(S) <= 1 + 2.0 ** -6)


@pytest.mark.parametrize("k,kind", [(10, "planted"), (16, "iid"), (1, "iid"), (17, "iid"),
                                    (100, "planted"), (128, "iid")])
def test_pooled_topk(H, k, kind):
    C, Q = 5000, 300
    corp, q = case(C, Q, kind=kind)
    idx = H.hiper_index_build(to_dev(corp), np.ones(C, np.int32), id_base=77,
                              flags=H.HIPER_POOLED)
    s, i = H.hiper_maxsim_topk(idx, to_dev(q), np.ones(Q, np.int32), k)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    lay = bits(idx.layout().clone())
    qn = oracle.norm_rows(q[:, 0])
    S_o = oracle.maxsim_matrix(qn[:, None], np.ones(Q, np.int32), lay, np.ones(C, np.int32))
    ids = np.arange(C, dtype=np.int64) + 77
    for r in range(Q):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, 1, D, f"pooled q{r}")
    if kind == "planted":
        assert (i[:, 0] == gen.query_targets(12, Q, C, False) + 77).all()


def test_pooled_topk_append_overflow_falls_back(H, monkeypatch):
    """k > 16 on a corpus >= 32 k chunks takes the APPEND path (sample bound + candidate buffers);
    a buffer too small for the candidates must trigger the heap-path rerun, with the same answer."""
    C, Q, k = 6000, 40, 100
    corp, q = case(C, Q, kind="iid")
    idx = H.hiper_index_build(to_dev(corp), np.ones(C, np.int32), flags=H.HIPER_POOLED)
    s0, i0 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), np.ones(Q, np.int32), k)]
    monkeypatch.setenv("HIPER_POOLED_APPEND_CAP", "1")   # one slot per segment: overflows
    s1, i1 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), np.ones(Q, np.int32), k)]
    assert np.array_equal(i0, i1) and np.array_equal(s0.view(np.uint32), s1.view(np.uint32))
    lay = bits(idx.layout().clone())
    S_o = oracle.maxsim_matrix(oracle.norm_rows(q[:, 0])[:, None], np.ones(Q, np.int32), lay,
                               np.ones(C, np.int32))
    ids = np.arange(C, dtype=np.int64)
    for r in range(Q):
        assert_topk_ok(s1[r], i1[r], S_o[r], ids, k, 1, D, f"append overflow q{r}")


def test_pooled_edge_cases(H):
    corp, q = case(3, 5)
    idx = H.hiper_index_build(to_dev(corp), np.ones(3, np.int32), flags=H.HIPER_POOLED)
    s, i = H.hiper_maxsim_topk(idx, to_dev(q), np.ones(5, np.int32), 6)
    assert (i.cpu().numpy()[:, 3:] == -1).all()
    s, i = H.hiper_maxsim_topk(idx, to_dev(q), np.ones(5, np.int32), 40)   # warp-list path, k > n
    assert (i.cpu().numpy()[:, 3:] == -1).all() and (i.cpu().numpy()[:, :3] >= 0).all()
    with pytest.raises(H.HiperError) as e:
        H.hiper_maxsim_topk(idx, to_dev(q), np.ones(5, np.int32), 129)
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"
    qq = np.zeros((5, 2, D), np.uint16)
    with pytest.raises(H.HiperError) as e:
        H.hiper_maxsim_topk(idx, to_dev(qq), np.ones(5, np.int32), 3)
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"


def test_config5_full_size(H):
    """BASELINE configs[4] on one GPU: 3.6M pooled chunks x 768 bf16, Q = 4096, top-10."""
    from synth import device
    C, Q, k = 3_600_000, 4096, 10
    corpus = torch.empty((C, 1, D), dtype=torch.bfloat16, device="cuda")
    device.corpus_(corpus, 21, 0)
    idx = H.hiper_index_build(corpus, np.ones(C, np.int32), flags=H.HIPER_BORROW_TOKENS | H.HIPER_POOLED)
    q = torch.empty((Q, 1, D), dtype=torch.bfloat16, device="cuda")
    device.queries_(q, 22, corpus_seed=21, n_chunks=C, L=1)
    s, i = H.hiper_maxsim_topk(idx, q, np.ones(Q, np.int32), k)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    assert (i[:, 0] == gen.query_targets(22, Q, C, False)).all()
    assert (np.diff(s, axis=1) <= 0).all() and all(len(set(r)) == k for r in i.tolist())
    lay = idx.layout()
    sample = [0, 2047, 4095]
    torch.backends.cuda.matmul.allow_tf32 = False
    raw_q = np.stack([gen.queries(22, 1, 1, D, corpus_seed=21, n_chunks=C, L=1, start=r)[0, 0]
                      for r in sample])
    qn = oracle.norm_rows(raw_q)
    full = (torch.from_numpy(qn.view(np.int16)).cuda().view(torch.bfloat16).float()
            @ lay[:, 0].float().T).cpu().numpy()                                # fp32 GEMM reference
    for j, r in enumerate(sample):
        rows = bits(lay[torch.from_numpy(i[r]).cuda()])[:, 0]
        S_o = np.array([oracle.maxsim(qn[j:j + 1], rows[m:m + 1]) for m in range(k)])
        assert_scores_close(s[r][None], S_o[None], [1], D, f"config5 q{r}")
        others = np.setdiff1d(np.arange(C), i[r])
        assert full[j, others].max() <= s[r][-1] + score_tol(np.array([s[r][-1]]), 1, D)[0]
    del corpus, idx, lay
