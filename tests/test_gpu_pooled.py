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


def _kernels_launched(fn):
    """Names of the CUDA kernels fn() launches (CUPTI via torch.profiler)."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        out = fn()
        torch.cuda.synchronize()
    return out, {e.name for e in prof.events() if e.device_type.name == "CUDA"}


@pytest.mark.parametrize("C,Q,k,dim,mode,tn", [
    (3, 5, 7, 768, "1", None),          # one ragged chunk tile on one pair, k > n
    (1000, 8, 10, 768, "1", None),      # 4 tiles (ragged) on 4 pairs, one query tile: two list slots
    (5000, 300, 16, 768, "1", None),    # 2 query tiles: one list slot per (pair, query)
    (40_123, 40, 10, 768, "2", None),   # auto selection (>= 2 tiles per pair), ragged tail
    (39_000, 600, 1, 256, "2", None),   # 3 query tiles, dim 256: 4 resident K-blocks, 12 query stages
    (38_500, 100, 10, 720, "2", None),  # dim % 64 != 0: zero-filled K tail in both operands
    (5000, 300, 10, 768, "1", "256"),   # 256-chunk tiles (MMA N = 256, 128 rows per CTA, 2 stages)
    (41_000, 513, 16, 768, "2", "240"), # 240-chunk tiles, 3 query tiles
    (9_999, 70, 5, 768, "1", "192"),    # 192-chunk tiles
])
def test_pooled_chunk_stationary(H, monkeypatch, C, Q, k, dim, mode, tn):
    """a12 on the chunk-stationary kernel (pooled_cs_sm100.cuh) vs the oracle, and bitwise vs the
    streaming kernel (same K order of the same MMAs)."""
    corp = gen.corpus(31, 0, C, 1, dim, kind="planted", dtype="bf16")
    q = gen.queries(32, Q, 1, dim, corpus_seed=31, n_chunks=C, L=1, kind="planted", dtype="bf16")
    if mode:
        monkeypatch.setenv("HIPER_POOLED_CS", mode)
    if tn:
        monkeypatch.setenv("HIPER_POOLED_CS_N", tn)
    if C == 1000:
        monkeypatch.setenv("HIPER_POOLED_CS_A", "32")   # 32-dim query stages (64-B swizzle)
    idx = H.hiper_index_build(to_dev(corp), np.ones(C, np.int32), id_base=5, flags=H.HIPER_POOLED)
    qd = to_dev(q)
    (s, i), names = _kernels_launched(lambda: H.hiper_maxsim_topk(idx, qd, np.ones(Q, np.int32), k))
    assert any("pooled_cs_sm100_kernel" in n for n in names), names
    s, i = s.cpu().numpy(), i.cpu().numpy()
    lay = bits(idx.layout().clone())
    qn = oracle.norm_rows(q[:, 0])
    S_o = oracle.maxsim_matrix(qn[:, None], np.ones(Q, np.int32), lay, np.ones(C, np.int32))
    ids = np.arange(C, dtype=np.int64) + 5
    for r in range(Q):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, 1, dim, f"pooled_cs q{r}")
    assert (i[:, 0] == gen.query_targets(32, Q, C, False) + 5).all()
    monkeypatch.setenv("HIPER_POOLED_CS", "0")
    (s0, i0), names0 = _kernels_launched(lambda: H.hiper_maxsim_topk(idx, qd, np.ones(Q, np.int32), k))
    assert not any("pooled_cs_sm100_kernel" in n for n in names0)
    s0, i0 = s0.cpu().numpy(), i0.cpu().numpy()
    assert np.array_equal(i, i0) and np.array_equal(s.view(np.uint32), s0.view(np.uint32))


@pytest.mark.parametrize("k", [1, 8, 9])
def test_pooled_short_register_list(H, k):
    """k <= 8 runs the 8-slot register-list instantiation (k = 9: the 16-slot one), checked by the
    kernel names CUPTI records; both against the oracle's exact top-k."""
    C, Q = 7000, 260
    corp, q = case(C, Q, kind="iid")
    idx = H.hiper_index_build(to_dev(corp), np.ones(C, np.int32), id_base=3, flags=H.HIPER_POOLED)
    qd = to_dev(q)
    (s, i), names = _kernels_launched(lambda: H.hiper_maxsim_topk(idx, qd, np.ones(Q, np.int32), k))
    want = "pooled_sm100_pair_kernel<1, 8," if k <= 8 else "pooled_sm100_pair_kernel<1, 16,"
    assert any(want in n for n in names), names
    s, i = s.cpu().numpy(), i.cpu().numpy()
    lay = bits(idx.layout().clone())
    S_o = oracle.maxsim_matrix(oracle.norm_rows(q[:, 0])[:, None], np.ones(Q, np.int32), lay,
                               np.ones(C, np.int32))
    ids = np.arange(C, dtype=np.int64) + 3
    for r in range(Q):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, 1, D, f"pooled k={k} q{r}")


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
