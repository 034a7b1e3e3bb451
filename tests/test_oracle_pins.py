"""Pins of the CPU oracle against things other than itself (CPU only, -m "not gpu").

Each test names the passage / property it pins (SPEC.md examples) and the
plausible oracle mistake it would catch.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from synth import gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def bf(x):
    """float -> bf16 bits (exact for the small dyadic values used here)."""
    return gen.f32_to_bf16_bits(np.asarray(x, dtype=np.float32))


def unit_rows_exact(rng, n, d, nnz=64):
    """Rows with `nnz` entries of +-1/8 (nnz = 64 -> squared norm exactly 1): NORM maps them to
    themselves, and their dot products are exact dyadic rationals."""
    assert nnz == 64 and d >= 64
    out = np.zeros((n, d), dtype=np.float32)
    for r in range(n):
        idx = rng.choice(d, nnz, replace=False)
        out[r, idx] = rng.choice([-0.125, 0.125], nnz)
    return out


# ----------------------------------------------------------------------------------- NORM (R1)
def _round_frac(x: Fraction, mant_bits: int) -> Fraction:
    """Exact round-to-nearest-even of a rational to a binary float with `mant_bits` significand
    bits (normal range only)."""
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    # a in [2^e, 2^(e+1)); quantum = 2^(e - mant_bits + 1)
    q = Fraction(2) ** (e - mant_bits + 1)
    m = a / q
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * fl * q


def _f32(x: Fraction) -> Fraction:
    return _round_frac(x, 24)


def _sqrt_f32(a: Fraction) -> Fraction:
    """Correctly rounded fp32 sqrt of a positive fp32 value, decided exactly."""
    y = Fraction(float(np.float32(math.sqrt(float(a)))))
    e = y.numerator.bit_length() - y.denominator.bit_length()
    if Fraction(2) ** e > y:
        e -= 1
    ulp = Fraction(2) ** (e - 23)
    for cand in (y - ulp, y, y + ulp):
        # cand is the nearest iff sqrt(a) lies within half an ulp of it
        lo, hi = cand - ulp / 2, cand + ulp / 2
        if lo * lo <= a <= hi * hi:
            return cand
    raise AssertionError("sqrt bracket")


def norm_row_exact(x) -> list:
    """NORM (reading R1) in exact rational arithmetic: fmaf = round(exact a*b + c)."""
    xs = [Fraction(float(v)) for v in x]
    acc = Fraction(0)
    for v in xs:
        acc = _f32(v * v + acc)
    inv = _f32(Fraction(1) / _sqrt_f32(acc))
    return [_round_frac(_f32(v * inv), 8) for v in xs]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_norm_matches_exact_rational(dtype):
    """Pins NORM bit for bit against exact arithmetic (catches a wrong rounding step, an FMA vs
    mul+add mix-up, a dropped element of the sum, rsqrt instead of 1/sqrt)."""
    rng = np.random.default_rng(7)
    d = 128
    x = (rng.standard_normal((6, d)) * rng.choice([0.01, 1.0, 37.0], (6, 1))).astype(np.float32)
    x[5, :] = 0.0
    x[5, 3] = 3.0                   # single nonzero entry -> exact +-1 after NORM
    if dtype == "bf16":
        x = gen.bf16_bits_to_f32(bf(x))
        y = oracle.norm_rows(bf(x))
    else:
        y = oracle.norm_rows(x)
    got = oracle.bf16_bits_to_f64(y)
    for r in range(x.shape[0]):
        ref = [float(v) for v in norm_row_exact(x[r])]
        assert got[r].tolist() == ref, f"row {r}"
    assert got[5, 3] == 1.0 and np.count_nonzero(got[5]) == 1


def test_norm_identity_on_exact_unit_rows():
    """Rows that are exactly unit (entries +-1/8 x 64, and +-e_k) are fixed points of NORM."""
    rng = np.random.default_rng(1)
    x = unit_rows_exact(rng, 10, 128)
    e = np.zeros((4, 128), dtype=np.float32)
    e[0, 0], e[1, 77], e[2, 127], e[3, 5] = 1.0, -1.0, 1.0, -1.0
    for rows in (x, e):
        y = oracle.norm_rows(rows)
        assert np.array_equal(y, bf(rows))


def test_norm_power_of_two_scale_invariance():
    """P11: x * 2^k normalises to bitwise the same bf16 row (every NORM step is exact under 2^k)."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((32, 128)).astype(np.float32)
    y0 = oracle.norm_rows(x)
    for k in (-20, -3, 1, 9, 30):
        assert np.array_equal(oracle.norm_rows((x * np.float32(2.0 ** k)).astype(np.float32)), y0)


def test_norm_unit_length_within_bf16_rounding():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 128)).astype(np.float32) * 5
    y = oracle.bf16_bits_to_f64(oracle.norm_rows(x))
    n = np.sqrt((y * y).sum(1))
    assert np.all(np.abs(n - 1) < 2.0 ** -7)


def test_norm_errors():
    x = np.ones((3, 16), dtype=np.float32)
    x[1] = 0
    with pytest.raises(oracle.OracleError) as e:
        oracle.norm_rows(x)
    assert e.value.args == ("zero", 1)
    x[1] = 1
    x[2, 4] = np.inf
    with pytest.raises(oracle.OracleError) as e:
        oracle.norm_rows(x)
    assert e.value.args == ("nonfinite", 2)


# ----------------------------------------------------------------------------------- MaxSim
def test_spec_golden_maxsim():
    """SPEC.md:265, 266, 275 worked examples (tests/golden/spec_examples.json)."""
    for ex in json.load(open(GOLDEN))["maxsim"]:
        q = oracle.norm_rows(np.asarray(ex["query"], dtype=np.float32))
        dd = oracle.norm_rows(np.asarray(ex["doc"], dtype=np.float32))
        assert oracle.maxsim(q, dd) == ex["expected"], ex["cite"]


def test_p1_brute_force_tiny():
    """P1 (acceptance #2): 100 random pairs T <= 16, d = 32 vs a numpy all-pairs
    matrix -> row max -> sum, within 1e-9."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        lq, ld, d = rng.integers(1, 17), rng.integers(1, 17), 32
        q = oracle.norm_rows(rng.standard_normal((lq, d)).astype(np.float32))
        dd = oracle.norm_rows(rng.standard_normal((ld, d)).astype(np.float32))
        Q, D = oracle.bf16_bits_to_f64(q), oracle.bf16_bits_to_f64(dd)
        ref = (Q @ D.T).max(axis=1).sum()
        assert abs(oracle.maxsim(q, dd) - ref) <= 1e-9


def test_p2_permutation_invariance():
    """P2: doc-row permutation -> bitwise equal; query-row permutation -> 1e-12."""
    rng = np.random.default_rng(12)
    q = oracle.norm_rows(rng.standard_normal((32, 128)).astype(np.float32))
    dd = oracle.norm_rows(rng.standard_normal((200, 128)).astype(np.float32))
    s = oracle.maxsim(q, dd)
    assert oracle.maxsim(q, dd[rng.permutation(200)]) == s
    assert abs(oracle.maxsim(q[rng.permutation(32)], dd) - s) <= 1e-12


def test_p3_single_token_doc_closed_form():
    """P3: a one-token doc d gives S = <sum_i q_i, d> (the max is over one element).  Catches a
    transposed max (over query tokens) and a sign error."""
    rng = np.random.default_rng(13)
    for lq in (1, 5, 32):
        q = oracle.norm_rows(rng.standard_normal((lq, 64)).astype(np.float32))
        dd = oracle.norm_rows(rng.standard_normal((1, 64)).astype(np.float32))
        Q, D = oracle.bf16_bits_to_f64(q), oracle.bf16_bits_to_f64(dd)
        closed = float(np.dot(Q.sum(axis=0), D[0]))
        assert abs(oracle.maxsim(q, dd) - closed) <= 1e-12


def test_p4_query_contained_in_doc_gives_len_q():
    """P4 (north star): exactly-unit query rows, all present in the doc
    among random others -> S == len_q exactly.  Catches a dropped query term, a mean instead of a
    sum (reading R4), a max over the wrong axis."""
    rng = np.random.default_rng(14)
    for lq in (1, 7, 32):
        qf = unit_rows_exact(rng, lq, 128)
        other = unit_rows_exact(rng, 100, 128)
        docf = np.concatenate([other, qf])[rng.permutation(100 + lq)]
        s = oracle.maxsim(oracle.norm_rows(qf), oracle.norm_rows(docf))
        assert s == float(lq)


def test_p5_bound_and_monotone():
    """P5: S <= len_q (up to NORM's bf16 norm error); appending doc rows never
    decreases S."""
    rng = np.random.default_rng(15)
    q = oracle.norm_rows(rng.standard_normal((32, 128)).astype(np.float32))
    dd = oracle.norm_rows(rng.standard_normal((64, 128)).astype(np.float32))
    s_prev = -np.inf
    for ld in range(1, 65, 7):
        s = oracle.maxsim(q, dd, len_d=ld)
        assert s >= s_prev
        assert s <= 32 * (1 + 2.0 ** -7)
        s_prev = s


def test_p10_masking_adversary():
    """P10 (reading R2): a doc whose real tokens all have negative dot with every query token,
    stored zero-padded: the padded rows must not take part in the max (zero-padding bug -> 0)."""
    q = oracle.norm_rows(np.eye(1, 64, dtype=np.float32))                 # e_0
    real = -np.abs(np.random.default_rng(16).standard_normal((5, 64))).astype(np.float32)
    padded = np.concatenate([oracle.norm_rows(real), np.zeros((11, 64), np.uint16)])
    s_pad = oracle.maxsim(q, padded, len_d=5)
    assert s_pad == oracle.maxsim(q, oracle.norm_rows(real))
    assert s_pad < 0
    # query padding (reading R3): rows >= len_q are excluded from the sum
    q2 = np.concatenate([q, oracle.norm_rows(np.ones((3, 64), np.float32))])
    assert oracle.maxsim(q2, padded, len_q=1, len_d=5) == s_pad


def test_matrix_equals_pairs_and_lengths():
    rng = np.random.default_rng(17)
    qt = oracle.norm_rows(rng.standard_normal((3, 8, 32)).astype(np.float32))
    dt = oracle.norm_rows(rng.standard_normal((5, 12, 32)).astype(np.float32))
    ql, dl = [8, 1, 5], [12, 3, 1, 7, 9]
    S = oracle.maxsim_matrix(qt, ql, dt, dl)
    for i in range(3):
        for j in range(5):
            assert S[i, j] == oracle.maxsim(qt[i], dt[j], ql[i], dl[j])
    with pytest.raises(oracle.OracleError):
        oracle.maxsim_matrix(qt, [8, 0, 5], dt, dl)


def test_pooled_limit_case_is_cosine():
    """P12 / config 5: with Lq = Ld = 1 MaxSim reduces to the dot of NORM'd vectors (cosine)."""
    rng = np.random.default_rng(18)
    a = rng.standard_normal((1, 768)).astype(np.float32)
    b = rng.standard_normal((1, 768)).astype(np.float32)
    qa, qb = oracle.norm_rows(a), oracle.norm_rows(b)
    A, B = oracle.bf16_bits_to_f64(qa)[0], oracle.bf16_bits_to_f64(qb)[0]
    assert abs(oracle.maxsim(qa, qb) - float(A @ B)) <= 1e-12
    cos = float(a[0].astype(np.float64) @ b[0] / np.linalg.norm(a[0]) / np.linalg.norm(b[0]))
    assert abs(oracle.maxsim(qa, qb) - cos) <= 2.0 ** -6


# ----------------------------------------------------------------------------------- top-k
def test_spec_golden_search():
    for ex in json.load(open(GOLDEN))["search"]:
        s, i = oracle.topk(np.asarray(ex["scores"]), np.asarray(ex["ids"]), ex["k"])
        assert i.tolist() == ex["expected_ids"], ex["cite"]
        assert s.tolist() == [float(v) for v in ex["expected_scores"]], ex["cite"]


def test_p9_topk_vs_full_sort_with_duplicates():
    """P9: equals a full sort with ascending-id ties, incl. duplicated chunks."""
    rng = np.random.default_rng(19)
    for n, k in ((500, 10), (50, 100), (1000, 128), (1, 1)):
        sc = np.round(rng.standard_normal(n), 1)          # many exact ties
        ids = rng.permutation(10 * n)[:n].astype(np.int64)
        s, i = oracle.topk(sc, ids, k)
        ref = sorted(zip(sc.tolist(), ids.tolist()), key=lambda t: (-t[0], t[1]))[:k]
        m = min(k, n)
        assert i[:m].tolist() == [t[1] for t in ref]
        assert s[:m].tolist() == [t[0] for t in ref]
        assert (i[m:] == -1).all() and np.isneginf(s[m:]).all()


# ----------------------------------------------------------------------------------- InfoNCE
def test_spec_golden_li_loss():
    for ex in json.load(open(GOLDEN))["li_loss"]:
        L = oracle.infonce(np.asarray(ex["S"]), tau=ex["tau"])
        assert abs(L - ex["expected"]) <= 1e-12, ex["cite"]


def test_p7_closed_forms():
    """P7: B = 1 -> 0; equal scores -> ln M; two-way closed form
    log(1 + e^{(b-a)/tau}) -- catches a wrong sign, a missing /tau, a dropped term."""
    assert oracle.infonce(np.array([[5.0]]), tau=0.05) == 0.0
    for M in (2, 7, 256):
        assert abs(oracle.infonce(np.full((3, M), 1.7), pos=[0, M - 1, 0], tau=0.3) - math.log(M)) <= 1e-12
    for a, b, tau in ((3.0, 1.0, 1.0), (0.2, 0.9, 0.05), (-1.0, -1.5, 2.0)):
        ref = math.log1p(math.exp((b - a) / tau))
        assert abs(oracle.infonce(np.array([[a, b]]), tau=tau) - ref) <= 1e-12
    S = np.array([[1.0, 2.0, 3.0], [0.5, 0.1, 0.2]])
    ref = (math.log(sum(math.exp(v) for v in S[0])) - 2.0
           + math.log(sum(math.exp(v) for v in S[1])) - 0.2) / 2
    assert abs(oracle.infonce(S, pos=[1, 2]) - ref) <= 1e-12


def test_p8_vs_torch_cross_entropy():
    """P8: library routine (torch.nn.functional.cross_entropy, float64) on random S."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(20)
    for B, M, tau in ((4, 4, 1.0), (64, 64, 0.05), (16, 40, 0.7)):
        S = rng.standard_normal((B, M)) * 5
        pos = rng.integers(0, M, B)
        ref = torch.nn.functional.cross_entropy(torch.tensor(S / tau), torch.tensor(pos)).item()
        assert abs(oracle.infonce(S, pos, tau) - ref) <= 1e-10 * max(1, abs(ref))


def test_infonce_errors():
    with pytest.raises(oracle.OracleError):
        oracle.infonce(np.zeros((0, 3)))
    with pytest.raises(oracle.OracleError):
        oracle.infonce(np.zeros((2, 3)), tau=0.0)
    with pytest.raises(oracle.OracleError):
        oracle.infonce(np.zeros((2, 3)), pos=[0, 3])


# ----------------------------------------------------------------------------------- N2 gather / total
def test_gather_candidates_spec_examples():
    """SPEC.md:327-329 examples of the min(N, W) rule."""
    ranks = [[(r, i) for i in range(12)] for r in range(4)]
    assert len(oracle.gather_candidates(ranks, 0, 100)) == 48          # min(100, 48)
    with pytest.raises(oracle.OracleError):
        oracle.gather_candidates(ranks, 0, 10)                          # NTooSmall
    c = oracle.gather_candidates(ranks, 0, 16)
    assert c == ranks[0] + ranks[1][:4]                                 # 12 local + first 4 of rank 1
    c = oracle.gather_candidates(ranks, 2, 30)
    assert c == ranks[2] + ranks[0] + ranks[1][:6]                      # local first, then rank order
    assert oracle.gather_candidates([[1, 2, 3]], 0, 5) == [1, 2, 3]     # one rank: the local batch


def test_contrastive_and_total_spec_examples():
    """SPEC.md:336-337 (uniform cosines -> ln m; single positive candidate -> 0) and SPEC.md:354
    (L_C = 0.6, L_LI = 0.4 -> L = 0.5)."""
    assert abs(oracle.infonce(np.full((5, 9), 0.3), pos=[0] * 5, tau=0.05) - math.log(9)) <= 1e-12
    assert oracle.infonce(np.array([[0.7]]), tau=0.05) == 0.0
    assert oracle.coltrast_total(0.4, 0.6) == 0.5


# ----------------------------------------------------------------------------------- N1 gradient
def _li_loss_exact(xq, ql, xd, dl, tau):
    return oracle.li_loss_grad(xq, ql, xd, dl, tau=tau, exact_norm=True)[0]


@pytest.mark.parametrize("tau", [1.0, 0.3])
def test_li_grad_central_finite_differences(tau):
    """SPEC.md:357-365 grad_check: analytic gradient (chain rule through argmax and normalisation)
    vs central finite differences in float64, max relative error <= 1e-4."""
    rng = np.random.default_rng(31)
    B, Lq, M, Ld, d = 3, 4, 3, 5, 6
    xq = rng.standard_normal((B, Lq, d))
    xd = rng.standard_normal((M, Ld, d))
    ql = np.array([4, 2, 3], np.int32)
    dl = np.array([5, 1, 3], np.int32)
    L, gq, gd, _, gap, _ = oracle.li_loss_grad(xq, ql, xd, dl, tau=tau, exact_norm=True)
    assert gap[gap > 0].min() > 1e-3  # no near-ties: the max is differentiable here
    eps = 1e-6
    for x, g, lens in ((xq, gq, ql), (xd, gd, dl)):
        for idx in np.ndindex(*x.shape):
            if idx[1] >= lens[idx[0]]:
                assert g[idx] == 0.0
                continue
            x[idx] += eps
            lp = _li_loss_exact(xq, ql, xd, dl, tau)
            x[idx] -= 2 * eps
            lm = _li_loss_exact(xq, ql, xd, dl, tau)
            x[idx] += eps
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - g[idx]) / max(1e-8, abs(fd) + abs(g[idx])) <= 1e-4 or abs(fd - g[idx]) < 1e-9, idx


def test_li_grad_matches_loss_and_structure():
    """The oracle's loss equals infonce(maxsim_matrix) on the same NORM'd operands; gradients sum
    structure: sum over docs of dL/dS is 0 per row (softmax - onehot), so with B = 1 and one doc the
    gradient vanishes."""
    rng = np.random.default_rng(32)
    xq = rng.standard_normal((4, 8, 64)).astype(np.float32)
    xd = rng.standard_normal((5, 16, 64)).astype(np.float32)
    ql, dl = np.array([8, 3, 1, 5], np.int32), np.array([16, 2, 9, 1, 7], np.int32)
    L, gq, gd, am, _, _ = oracle.li_loss_grad(xq, ql, xd, dl, pos=[0, 1, 2, 3], tau=0.5)
    S = oracle.maxsim_matrix(oracle.norm_rows(xq), ql, oracle.norm_rows(xd), dl)
    assert abs(L - oracle.infonce(S, pos=[0, 1, 2, 3], tau=0.5)) <= 1e-12
    assert (am < dl[None, :, None]).all()
    L1, g1, g2, _, _, _ = oracle.li_loss_grad(xq[:1], ql[:1], xd[:1], dl[:1])
    assert L1 == 0.0 and np.abs(g1).max() == 0.0 and np.abs(g2).max() == 0.0


def _fixed_point_rows(rng, shape, d):
    """Rows of exactly unit norm whose entries are 0 or +-1/8 (64 nonzeros, d >= 64): NORM maps them to
    themselves bit for bit (acc = 64 * 2^-6 = 1 exactly, inv = 1), and so does x / ||x|| in float64."""
    out = np.zeros(shape + (d,), np.float64)
    for idx in np.ndindex(*shape):
        nz = rng.choice(d, 64, replace=False)
        out[idx + (nz,)] = rng.choice([-0.125, 0.125], 64)
    return out


@pytest.mark.parametrize("scale", [1.0, 4.0])
def test_li_grad_straight_through_branch_on_norm_fixed_points(scale):
    """Reading R19: with exact_norm = 0 the oracle takes the forward, the argmax and the
    G.d sums on the bf16 NORM'd operands (the GPU's), but the Jacobian of the normalisation on the
    float64 x/||x|| (a straight-through view of the bf16 rounding).  On NORM fixed points the two
    operand sets coincide exactly, so this branch must equal the finite-difference-pinned
    exact_norm = 1 branch to rounding (a power-of-two scale keeps both exact and exercises 1/||x||)."""
    rng = np.random.default_rng(33)
    B, Lq, M, Ld, d = 3, 5, 4, 7, 128
    xq = _fixed_point_rows(rng, (B, Lq), d) * scale
    xd = _fixed_point_rows(rng, (M, Ld), d) * scale
    ql = np.array([5, 2, 4], np.int32)
    dl = np.array([7, 1, 3, 6], np.int32)
    ex = oracle.li_loss_grad(xq, ql, xd, dl, tau=0.5, exact_norm=True)
    st = oracle.li_loss_grad(xq, ql, xd, dl, tau=0.5, exact_norm=False)
    assert abs(ex[0] - st[0]) <= 1e-12 * max(1.0, abs(ex[0]))
    assert np.array_equal(ex[3], st[3])                    # same argmax (same tie rule, same values)
    for a, b in ((ex[1], st[1]), (ex[2], st[2])):
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(a).max())
    assert np.abs(ex[1]).max() > 0 and np.abs(ex[2]).max() > 0
    # and away from fixed points the branches differ by the bf16 rounding only (~2^-8 relative)
    xq2 = rng.standard_normal((B, Lq, d))
    xd2 = rng.standard_normal((M, Ld, d))
    e2 = oracle.li_loss_grad(xq2, ql, xd2, dl, tau=0.5, exact_norm=True)
    s2 = oracle.li_loss_grad(xq2, ql, xd2, dl, tau=0.5, exact_norm=False)
    assert abs(e2[0] - s2[0]) <= 2e-2 * abs(e2[0])
