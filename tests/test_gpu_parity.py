"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on the same seeded inputs.

Every comparison feeds the oracle the exact bf16 operands the kernels consumed (layouts read back
from the device), after checking those layouts bitwise against the oracle's own NORM of the raw
inputs.
"""
import numpy as np
import pytest

import oracle
from synth import gen
from tests._compare import (assert_loss_close, assert_scores_close, assert_topk_ok)

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
    """torch bf16 tensor -> numpy uint16 bit patterns."""
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def to_dev(a):
    """numpy float32 -> cuda f32; numpy uint16 (bf16 bits) -> cuda bf16."""
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make_case(C, L, Q, Lq, d, *, dtype="bf16", kind="planted", var_len=False, seed=1, qseed=2,
              diagonal=False, sigma_q=gen.SIGMA_Q_EASY):
    corp = gen.corpus(seed, 0, C, L, d, kind=kind, dtype=dtype)
    clen = gen.lengths(seed, C, L, var_len)
    q = gen.queries(qseed, Q, Lq, d, corpus_seed=seed, n_chunks=C, L=L,
                    chunk_lens_fn=lambda c: clen[c], kind=kind, corpus_kind=kind, dtype=dtype,
                    diagonal=diagonal, sigma_q=sigma_q)
    qlen = gen.lengths(qseed, Q, Lq, var_len, stream=gen.QLEN)
    return corp, clen, q, qlen


def expected_layout(raw, lens, rows_out):
    """Oracle NORM of the real rows, zero rows elsewhere (the layout contract of hiper.h)."""
    n, rows_in, d = raw.shape
    out = np.zeros((n, rows_out, d), dtype=np.uint16)
    for i in range(n):
        if lens[i]:
            out[i, :lens[i]] = oracle.norm_rows(raw[i, :lens[i]])
    return out


def index_and_layout(H, corp, clen, id_base=0, flags=0):
    idx = H.hiper_index_build(to_dev(corp), clen, id_base=id_base, flags=flags)
    lay = bits(idx.layout().clone())
    return idx, lay


def query_layout(H, q, qlen):
    lay, status = H.hiper_prepare_queries(to_dev(q), qlen)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    return bits(lay)


# ------------------------------------------------------------------------------------------ generator
def test_synth_device_matches_numpy(H):
    from synth import device
    for kind in ("planted", "iid"):
        for dt in (torch.float32, torch.bfloat16):
            out = torch.empty((5, 48, 64), dtype=dt, device="cuda")
            device.corpus_(out, 9, 17, kind=kind)
            ref = gen.corpus(9, 17, 5, 48, 64, kind=kind, dtype="f32" if dt == torch.float32 else "bf16")
            got = out.cpu().numpy() if dt == torch.float32 else bits(out)
            assert np.array_equal(got.view(np.uint32) if dt == torch.float32 else got,
                                  ref.view(np.uint32) if dt == torch.float32 else ref), (kind, dt)
    clen = gen.lengths(9, 40, 48, True)
    qo = torch.empty((6, 32, 64), dtype=torch.bfloat16, device="cuda")
    device.queries_(qo, 4, corpus_seed=9, n_chunks=40, L=48,
                    chunk_lens=torch.from_numpy(clen).cuda(), start=3)
    ref = gen.queries(4, 6, 32, 64, corpus_seed=9, n_chunks=40, L=48,
                      chunk_lens_fn=lambda c: clen[c], start=3)
    assert np.array_equal(bits(qo), ref)


# ------------------------------------------------------------------------------------------ a1 / a2
@pytest.mark.parametrize("dtype,var_len,L", [("f32", True, 128), ("bf16", False, 256),
                                             ("bf16", True, 100)])
def test_layout_bitwise(H, dtype, var_len, L):
    corp, clen, q, qlen = make_case(37, L, 9, 32, 128, dtype=dtype, var_len=var_len)
    idx, lay = index_and_layout(H, corp, clen)
    ld_pad = (L + 15) // 16 * 16
    assert lay.shape == (37, ld_pad, 128)
    assert np.array_equal(lay, expected_layout(corp, clen, ld_pad))
    ql = query_layout(H, q, qlen)
    exp_q = np.zeros((16, 32, 128), dtype=np.uint16)
    exp_q[:9] = expected_layout(q, qlen, 32)
    assert np.array_equal(ql, exp_q)


def test_layout_borrow_in_place(H):
    corp, clen, _, _ = make_case(20, 64, 1, 8, 128, var_len=True)
    t = to_dev(corp)
    idx = H.hiper_index_build(t, clen, flags=H.HIPER_BORROW_TOKENS)
    assert idx.layout_ptr == t.data_ptr()
    assert np.array_equal(bits(t), expected_layout(corp, clen, 64))


def test_layout_assume_normalized_and_scale_invariance(H):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((6, 32, 64)).astype(np.float32)
    lens = np.full(6, 32, np.int32)
    _, lay = index_and_layout(H, x, lens)
    _, lay2 = index_and_layout(H, (x * np.float32(2.0 ** 7)).astype(np.float32), lens)
    assert np.array_equal(lay, lay2)   # P11
    _, lay3 = index_and_layout(H, x, lens, flags=H.HIPER_ASSUME_NORMALIZED)
    assert np.array_equal(lay3, gen.f32_to_bf16_bits(x))


# ------------------------------------------------------------------------------------------ a3-a5
def run_scores(H, corp, clen, q, qlen, d):
    idx, lay = index_and_layout(H, corp, clen)
    ql = query_layout(H, q, qlen)
    S = H.hiper_maxsim_scores(idx, to_dev(q), qlen).cpu().numpy()
    S_o = oracle.maxsim_matrix(ql[:len(qlen)], qlen, lay, clen)
    return S, S_o


@pytest.mark.parametrize("kind,var_len", [("planted", False), ("iid", True), ("planted", True)])
def test_scores_config1(H, kind, var_len):
    """Config 1 (BASELINE.json configs[0]): 8 queries x 32 tokens vs 1,000 chunks x 128, d=128, fp32."""
    corp, clen, q, qlen = make_case(1000, 128, 8, 32, 128, dtype="f32", kind=kind, var_len=var_len)
    S, S_o = run_scores(H, corp, clen, q, qlen, 128)
    assert_scores_close(S, S_o, qlen, 128, "config1")
    # diagnostic tier: identical operands -> ~1e-6 relative
    assert np.all(np.abs(S - S_o) <= np.maximum(1e-5 * np.abs(S_o), 1e-5))


@pytest.mark.parametrize("n_q,C,L,d", [(1, 1, 16, 64), (5, 7, 48, 128), (13, 300, 256, 64),
                                       (37, 45, 112, 128)])
def test_scores_ragged_shapes(H, n_q, C, L, d):
    corp, clen, q, qlen = make_case(C, L, n_q, 32, d, var_len=True, kind="iid")
    S, S_o = run_scores(H, corp, clen, q, qlen, d)
    assert_scores_close(S, S_o, qlen, d, f"ragged {n_q},{C},{L},{d}")


def test_masking_adversary(H):
    """P10: real doc tokens all have negative dot with the query token; padding must not be 0-scored."""
    d = 128
    qv = np.zeros((4, 32, d), np.float32)
    qv[:, 0, 0] = 1.0
    qlen = np.ones(4, np.int32)
    rng = np.random.default_rng(3)
    docs = np.zeros((9, 64, d), np.float32)
    docs[:, :, 0] = -np.abs(rng.standard_normal((9, 64))) - 0.1
    docs[:, :, 1:] = rng.standard_normal((9, 64, d - 1)) * 0.1
    clen = np.array([1, 2, 5, 31, 32, 33, 63, 64, 17], np.int32)
    S, S_o = run_scores(H, docs, clen, qv, qlen, d)
    assert (S_o < 0).all() and (S < 0).all()
    assert_scores_close(S, S_o, qlen, d, "masking")


def test_batch_invariance_bitwise(H):
    """P14: S(q, c) does not depend on the other queries in the batch."""
    corp, clen, q, qlen = make_case(200, 256, 11, 32, 128, var_len=True)
    idx = H.hiper_index_build(to_dev(corp), clen)
    S_all = H.hiper_maxsim_scores(idx, to_dev(q), qlen).cpu().numpy()
    for i in (0, 5, 10):
        S_one = H.hiper_maxsim_scores(idx, to_dev(q[i:i + 1]), qlen[i:i + 1]).cpu().numpy()
        assert np.array_equal(S_one[0].view(np.uint32), S_all[i].view(np.uint32))


def test_spec_examples_on_gpu(H):
    """SPEC.md:265-266 / north-star invariants through the kernel: {e1,e2} vs {e1} = 1.0; exactly
    unit query rows contained in the doc -> len_q (P4); single-token doc closed form (P3)."""
    d = 64
    q = np.zeros((2, 32, d), np.float32)
    q[0, 0, 0] = q[0, 1, 1] = 1.0
    rng = np.random.default_rng(4)
    qrows = np.zeros((32, d), np.float32)
    for r in range(32):
        qrows[r, rng.choice(d, 64, replace=False)] = rng.choice([-0.125, 0.125], 64)
    q[1] = qrows
    docs = np.zeros((2, 64, d), np.float32)
    docs[0, 0, 0] = 1.0
    docs[1, :32] = qrows[rng.permutation(32)]
    docs[1, 32:] = rng.standard_normal((32, d))
    S, _ = run_scores(H, docs, np.array([1, 64], np.int32), q, np.array([2, 32], np.int32), d)
    assert S[0, 0] == 1.0
    assert S[1, 1] == 32.0


# ------------------------------------------------------------------------------------------ a6-a9
def run_topk_vs_oracle(H, corp, clen, q, qlen, k, d, id_base=0):
    idx, lay = index_and_layout(H, corp, clen, id_base=id_base)
    ql = query_layout(H, q, qlen)
    s, i = H.hiper_maxsim_topk(idx, to_dev(q), qlen, k)
    s, i = s.cpu().numpy(), i.cpu().numpy()
    S_o = oracle.maxsim_matrix(ql[:len(qlen)], qlen, lay, clen)
    ids = np.arange(len(clen), dtype=np.int64) + id_base
    diffs = 0
    for r in range(len(qlen)):
        diffs += assert_topk_ok(s[r], i[r], S_o[r], ids, k, qlen[r], d, f"query {r}")
    return s, i, diffs


@pytest.mark.parametrize("kind,k", [("planted", 10), ("iid", 10), ("planted", 100), ("iid", 128)])
def test_topk_config1(H, kind, k):
    corp, clen, q, qlen = make_case(1000, 128, 8, 32, 128, dtype="f32", kind=kind,
                                    var_len=(kind == "iid"))
    s, i, _ = run_topk_vs_oracle(H, corp, clen, q, qlen, k, 128, id_base=12345)
    if kind == "planted":
        tgt = gen.query_targets(2, 8, 1000, False) + 12345
        assert (i[:, 0] == tgt).all()


def test_topk_edge_cases(H):
    # k > n: padding; n_q not a multiple of 4; chunk count below the partition count
    corp, clen, q, qlen = make_case(3, 40, 6, 20, 64, var_len=True)
    s, i, _ = run_topk_vs_oracle(H, corp, clen, q, qlen, 7, 64)
    assert (i[:, 3:] == -1).all()
    # empty index
    idx = H.hiper_index_build(torch.empty((0, 16, 64), dtype=torch.bfloat16, device="cuda"), [])
    s, i = H.hiper_maxsim_topk(idx, to_dev(q), qlen, 5)
    assert (i.cpu().numpy() == -1).all() and np.isneginf(s.cpu().numpy()).all()


def test_topk_duplicate_chunks_tie_order(H):
    """P9: duplicated chunks give bitwise-equal scores; they must come out in ascending id order."""
    corp, clen, q, qlen = make_case(50, 64, 5, 32, 128)
    corp = np.concatenate([corp, corp[::-1], corp])
    clen = np.concatenate([clen, clen[::-1], clen])
    s, i, _ = run_topk_vs_oracle(H, corp, clen, q, qlen, 30, 128)


def test_fake_sharding_bitwise(H):
    """P13 on one GPU: shards with id_base offsets, merged on the host == unsharded, bitwise."""
    corp, clen, q, qlen = make_case(600, 128, 9, 32, 128, var_len=True, kind="iid")
    k = 16
    idx = H.hiper_index_build(to_dev(corp), clen)
    s_ref, i_ref = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), qlen, k)]
    bounds = [0, 101, 350, 600]
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        ix = H.hiper_index_build(to_dev(corp[a:b]), clen[a:b], id_base=a)
        parts.append([t.cpu().numpy() for t in H.hiper_maxsim_topk(ix, to_dev(q), qlen, k)])
    for r in range(9):
        cand = [(float(s), int(i)) for ps, pi in parts for s, i in zip(ps[r], pi[r]) if i >= 0]
        cand.sort(key=lambda t: (-t[0], t[1]))
        assert [c[1] for c in cand[:k]] == i_ref[r].tolist()
        assert np.array_equal(np.array([c[0] for c in cand[:k]], np.float32).view(np.uint32),
                              s_ref[r].view(np.uint32))


# ------------------------------------------------------------------------------------------ a10-a11
@pytest.mark.parametrize("B,M,tau,kind", [(64, 64, 1.0, "planted"), (37, 45, 1.0, "planted"),
                                          (64, 64, 0.05, "iid")])
def test_coltrast_scores_loss(H, B, M, tau, kind):
    """Config 2 shape at oracle-friendly size (full 256 x 256 in test_coltrast_config2_full)."""
    n = max(B, M)
    corp, clen, q, qlen = make_case(n, 256, n, 32, 128, kind=kind, diagonal=True,
                                    sigma_q=gen.SIGMA_Q_HARD, var_len=(B != M), seed=3, qseed=4)
    corp, clen, q, qlen = corp[:M], clen[:M], q[:B], qlen[:B]
    S, L = H.hiper_coltrast_scores_loss(to_dev(q), qlen, to_dev(corp), clen, temperature=tau)
    S, L = S.cpu().numpy(), float(L.item())
    _, dlay = index_and_layout(H, corp, clen)
    ql = query_layout(H, q, qlen)
    S_o = oracle.maxsim_matrix(ql[:B], qlen, dlay, clen)
    assert_scores_close(S, S_o, qlen, 128, "coltrast S")
    L_o = oracle.infonce(S_o, tau=tau)
    assert_loss_close(L, L_o, "coltrast L")
    # diagnostic: the loss kernel alone on the GPU's own S vs float64 on that S
    L_own = float(H.hiper_infonce_loss(torch.from_numpy(S).cuda(), temperature=tau).item())
    assert abs(L_own - oracle.infonce(S.astype(np.float64), tau=tau)) <= max(1e-6 * abs(L_o), 1e-7)


def test_loss_kernel_pins(H):
    """a11 alone: B=1 -> 0; equal scores -> ln M; explicit positives; log1p regime (tiny loss)."""
    one = H.hiper_infonce_loss(torch.tensor([[7.0]], device="cuda")).item()
    assert one == 0.0
    eq = H.hiper_infonce_loss(torch.full((3, 50), 0.3, device="cuda"), pos_idx=[0, 49, 7],
                              temperature=0.05).item()
    assert abs(eq - np.log(50)) <= 1e-6 * np.log(50)
    S = np.array([[30.0, 1.0, 2.0], [0.5, 29.0, 0.1]], np.float32)
    L = H.hiper_infonce_loss(torch.from_numpy(S).cuda(), pos_idx=[0, 1], temperature=1.0).item()
    L_o = oracle.infonce(S.astype(np.float64), pos=[0, 1], tau=1.0)
    assert L_o < 1e-10 and abs(L - L_o) <= max(1e-4 * L_o, 1e-7)


# ------------------------------------------------------------------------------------------ ABI errors
def test_abi_errors(H):
    corp, clen, q, qlen = make_case(10, 32, 4, 8, 64)
    idx = H.hiper_index_build(to_dev(corp), clen)
    with pytest.raises(H.HiperError) as e:
        H.hiper_maxsim_topk(idx, to_dev(np.zeros((2, 8, 128), np.float32)), [1, 1], 5)
    assert e.value.name == "HIPER_ERR_DIM_MISMATCH"
    with pytest.raises(H.HiperError) as e:
        H.hiper_maxsim_topk(idx, to_dev(q), [1, 0, 1, 1], 5)
    assert e.value.name == "HIPER_ERR_EMPTY_TOKENS"
    with pytest.raises(H.HiperError) as e:
        H.hiper_index_build(to_dev(corp), np.zeros(10, np.int32))
    assert e.value.name == "HIPER_ERR_EMPTY_TOKENS"
    z = np.zeros((2, 8, 64), np.float32)
    z[0, 0, 0] = 1.0
    with pytest.raises(H.HiperError) as e:
        H.hiper_index_build(to_dev(z), [1, 2])
    assert e.value.name == "HIPER_ERR_ZERO_VECTOR"
    bad = np.ones((2, 8, 64), np.float32)
    bad[1, 3, 3] = np.nan
    with pytest.raises(H.HiperError) as e:
        H.hiper_index_build(to_dev(bad), [8, 8])
    assert e.value.name == "HIPER_ERR_NONFINITE"
    with pytest.raises(H.HiperError) as e:
        H.hiper_maxsim_topk(idx, to_dev(z), [2, 1], 5, flags=H.HIPER_VALIDATE_SYNC)
    assert e.value.name == "HIPER_ERR_ZERO_VECTOR"
    with pytest.raises(H.HiperError) as e:
        H.hiper_coltrast_scores_loss(to_dev(q), qlen, to_dev(corp), clen, temperature=0.0)
    assert e.value.name == "HIPER_ERR_BAD_TEMPERATURE"
    with pytest.raises(H.HiperError) as e:
        H.hiper_coltrast_scores_loss(to_dev(q), qlen, to_dev(corp), clen, pos_idx=[0, 1, 2, 10])
    assert e.value.name == "HIPER_ERR_BAD_POSITIVE"
    with pytest.raises(H.HiperError) as e:
        H.hiper_coltrast_scores_loss(to_dev(q[:0]), [], to_dev(corp), clen)
    assert e.value.name == "HIPER_ERR_EMPTY_BATCH"
    with pytest.raises(H.HiperError) as e:
        H.hiper_maxsim_topk(idx, to_dev(q), qlen, 129)
    assert e.value.name == "HIPER_ERR_UNSUPPORTED"
