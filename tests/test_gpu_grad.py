"""NEXT N1: the L_LI backward on the GPU vs the oracle's chain-rule gradient (itself pinned by
float64 finite differences in tests/test_oracle_pins.py).

Argmax decisions are taken in fp32 on the GPU and in float64 by the oracle; (query token, doc) pairs
whose best and second-best dot differ by less than 1e-4 may legitimately pick different tokens, so
gradient rows touched by such near-ties are excluded (and must be rare)."""
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
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def widen(a):
    return gen.bf16_bits_to_f32(a).astype(np.float64) if a.dtype == np.uint16 else a.astype(np.float64)


@pytest.mark.parametrize("n_q,n_d,Lq,Ld,d,dtype,tau,kind", [
    (32, 48, 32, 96, 128, "f32", 1.0, "planted"),
    (16, 40, 20, 64, 64, "bf16", 0.1, "iid"),
    (37, 37, 32, 128, 128, "bf16", 0.5, "planted"),
    (64, 80, 32, 256, 128, "bf16", 1.0, "planted"),   # 8 query tiles x full-length docs (streamed paths)
    # ld_pad 144 and 208 (not multiples of 64: the argmax epilogue's last 64-column block is
    # partial), ragged lengths
    (24, 30, 32, 144, 64, "bf16", 1.0, "iid"),
    (33, 40, 17, 200, 128, "f32", 0.3, "planted"),
])
def test_li_backward_matches_oracle(H, n_q, n_d, Lq, Ld, d, dtype, tau, kind):
    corp = gen.corpus(71, 0, n_d, Ld, d, kind=kind, dtype=dtype)
    dl = gen.lengths(71, n_d, Ld, True)
    q = gen.queries(72, n_q, Lq, d, corpus_seed=71, n_chunks=n_d, L=Ld, kind=kind, corpus_kind=kind,
                    chunk_lens_fn=lambda c: dl[c], dtype=dtype, diagonal=True,
                    sigma_q=gen.SIGMA_Q_HARD)
    ql = gen.lengths(72, n_q, Lq, True, stream=gen.QLEN)
    S, L, gq, gd = H.hiper_coltrast_scores_loss_grad(to_dev(q), ql, to_dev(corp), dl, temperature=tau)
    gq, gd, L = gq.cpu().numpy().astype(np.float64), gd.cpu().numpy().astype(np.float64), float(L.item())
    L_o, gq_o, gd_o, am, gap, am2 = oracle.li_loss_grad(widen(q), ql, widen(corp), dl, tau=tau)
    assert abs(L - L_o) <= max(1e-4 * abs(L_o), 1e-7)
    # fp32-vs-float64 argmax ambiguity: both dots within 2e-5 (> the fp32 accumulation error bound
    # d * 2^-24 * sum|products| ~ 7.6e-6 for unit rows, doubled)
    amb = np.zeros((n_q, n_d, Lq), bool)
    for i in range(n_q):
        amb[i, :, :ql[i]] = gap[i, :, :ql[i]] < 2e-5
    bad_q = amb.any(axis=1)                      # grad_q rows touched by an ambiguous argmax
    bad_d = np.zeros((n_d, Ld), bool)            # grad_d rows that may receive or lose that term
    for i, j, t in zip(*np.nonzero(amb)):
        bad_d[j, am[i, j, t]] = bad_d[j, am2[i, j, t]] = True
    assert bad_q.mean() < 0.05 and bad_d.mean() < 0.05, (bad_q.mean(), bad_d.mean())
    for got, ref, mask in ((gq, gq_o, ~bad_q[:, :, None]), (gd, gd_o, ~bad_d[:, :, None])):
        m = np.broadcast_to(mask, got.shape)
        scale = np.abs(ref).max()
        err = np.abs(got - ref)
        tol = 2e-3 * np.abs(ref) + 1e-4 * scale
        assert (err[m] <= tol[m]).all(), (err[m].max(), scale)
    # padding rows are exactly zero
    for i in range(n_q):
        assert (gq[i, ql[i]:] == 0).all()
    for j in range(n_d):
        assert (gd[j, dl[j]:] == 0).all()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_li_backward_zero_padding_rows(H, dtype):
    """Raw inputs whose padding rows are ZERO (norm 0: NORM's Jacobian would divide by 0 there):
    both gradients stay finite, padding rows exactly 0, real rows equal to the run with non-zero
    padding (padding never enters the forward)."""
    n_q, n_d, Lq, Ld, d = 20, 24, 32, 160, 128
    corp = gen.corpus(73, 0, n_d, Ld, d, dtype=dtype)
    dl = gen.lengths(73, n_d, Ld, True)
    q = gen.queries(74, n_q, Lq, d, corpus_seed=73, n_chunks=n_d, L=Ld, chunk_lens_fn=lambda c: dl[c],
                    dtype=dtype, diagonal=True)
    ql = gen.lengths(74, n_q, Lq, True, stream=gen.QLEN)
    ref = H.hiper_coltrast_scores_loss_grad(to_dev(q), ql, to_dev(corp), dl)
    qz, cz = q.copy(), corp.copy()
    for i in range(n_q):
        qz[i, ql[i]:] = 0
    for j in range(n_d):
        cz[j, dl[j]:] = 0
    got = H.hiper_coltrast_scores_loss_grad(to_dev(qz), ql, to_dev(cz), dl)
    for a, b in zip(ref, got):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.isfinite(b).all()
        assert np.array_equal(a, b)
