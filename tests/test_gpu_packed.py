"""NEXT N4 on the GPU: the length-bucketed packed corpus (HIPER_PACKED) against the oracle.

The packed layout changes where rows live and the MMA N per tile; it must not change any result:
* layout: every chunk's packed rows are bitwise the oracle's NORM of its raw rows, padding rows of its
  16-row slot repeat its last real row (R1, R2: a repeated column cannot change the max);
* scores / top-k: within the R8 tolerance of the float64 oracle on the same bf16 operands, on
  semantic-chunk, tiny-chunk (16 per tile), full-length and mixed corpora;
* packed == dense index bitwise (scores and top-k): per (query, chunk) the same K order and epilogue.
"""
import numpy as np
import pytest

import oracle
from synth import gen
from tests._compare import assert_scores_close, assert_topk_ok
from tests.test_gpu_parity import bits, expected_layout, query_layout, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_04846_b200 as H
    H.lib()
    return H


def semantic_case(C, L, Q, d, *, lens=None, kind="planted", dtype="bf16", seed=11, qseed=12):
    corp = gen.corpus(seed, 0, C, L, d, kind=kind, dtype=dtype)
    clen = gen.semantic_lengths(seed, C, L) if lens is None else np.asarray(lens, np.int32)
    q = gen.queries(qseed, Q, 32, d, corpus_seed=seed, n_chunks=C, L=L,
                    chunk_lens_fn=lambda c: clen[c], kind=kind, corpus_kind=kind, dtype=dtype)
    qlen = gen.lengths(qseed, Q, 32, True, stream=gen.QLEN)
    return corp, clen, q, qlen


def packed_index(H, corp, clen, id_base=0):
    idx = H.hiper_index_build(to_dev(corp), clen, id_base=id_base, flags=H.HIPER_PACKED)
    assert idx.packed
    return idx


def unpack(H, idx, clen, rows_out):
    """Test-side view of the packed layout as [n][rows_out][d] (+ the padding rows of each slot)."""
    lay = bits(idx.layout().clone())
    tiles, ents = idx.pack_tables()
    t_tiles, t_ents, t_rows = H.hiper_pack_plan(clen)
    assert np.array_equal(tiles, t_tiles) and np.array_equal(ents, t_ents) and idx.n_rows == t_rows
    n, d = len(clen), lay.shape[1]
    dense = np.zeros((n, rows_out, d), np.uint16)
    pad_ok = True
    for t0, nr, e0, e1 in tiles.tolist():
        for c, cl in ents[e0:e1].tolist():
            r0, ln = t0 + (cl >> 16), cl & 0xFFFF
            dense[c, :ln] = lay[r0:r0 + ln]
            w = (ln + 15) // 16 * 16
            # padding rows of the chunk's last 16-row group repeat its last real row
            pad_ok &= bool((lay[r0 + ln:r0 + w] == lay[r0 + ln - 1]).all())
    return dense, pad_ok


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_packed_layout_bitwise(H, dtype):
    corp, clen, _, _ = semantic_case(300, 256, 1, 128, dtype=dtype)
    idx = packed_index(H, corp, clen)
    dense, pad_ok = unpack(H, idx, clen, 256)
    assert pad_ok
    assert np.array_equal(dense, expected_layout(corp, clen, 256))


CASES = {
    "semantic": dict(C=700, L=256, lens=None),
    "tiny": dict(C=333, L=16, lens="tiny"),            # lengths 1..16: 16 chunks per tile
    "full": dict(C=90, L=256, lens="full"),             # one chunk per tile (= dense layout)
    "mixed": dict(C=500, L=256, lens="mixed"),          # every width bucket, ragged tails
}


def case_lens(name, C, L):
    rng = np.random.default_rng(len(name))
    if name == "tiny":
        return rng.integers(1, 17, C).astype(np.int32)
    if name == "full":
        return np.full(C, L, np.int32)
    if name == "mixed":
        return rng.integers(1, L + 1, C).astype(np.int32)
    return None


@pytest.mark.parametrize("name,kind", [("semantic", "planted"), ("tiny", "iid"), ("full", "iid"),
                                       ("mixed", "iid"), ("mixed", "planted")])
def test_packed_scores_vs_oracle_and_dense(H, name, kind):
    c = CASES[name]
    corp, clen, q, qlen = semantic_case(c["C"], c["L"], 13, 128, lens=case_lens(name, c["C"], c["L"]),
                                        kind=kind)
    idx = packed_index(H, corp, clen)
    S = H.hiper_maxsim_scores(idx, to_dev(q), qlen).cpu().numpy()
    ql = query_layout(H, q, qlen)
    lay = expected_layout(corp, clen, (c["L"] + 15) // 16 * 16)
    S_o = oracle.maxsim_matrix(ql[:len(qlen)], qlen, lay, clen)
    assert_scores_close(S, S_o, qlen, 128, f"packed {name}")
    dense = H.hiper_index_build(to_dev(corp), clen)
    S_d = H.hiper_maxsim_scores(dense, to_dev(q), qlen).cpu().numpy()
    assert np.array_equal(S.view(np.uint32), S_d.view(np.uint32))


@pytest.mark.parametrize("name,kind,k", [("semantic", "planted", 10), ("semantic", "iid", 100),
                                         ("tiny", "iid", 10), ("mixed", "iid", 128)])
def test_packed_topk_vs_oracle(H, name, kind, k):
    c = CASES[name]
    corp, clen, q, qlen = semantic_case(c["C"], c["L"], 21, 128, lens=case_lens(name, c["C"], c["L"]),
                                        kind=kind)
    idx = packed_index(H, corp, clen, id_base=777)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), qlen, k)]
    ql = query_layout(H, q, qlen)
    lay = expected_layout(corp, clen, (c["L"] + 15) // 16 * 16)
    S_o = oracle.maxsim_matrix(ql[:len(qlen)], qlen, lay, clen)
    ids = np.arange(len(clen), dtype=np.int64) + 777
    for r in range(len(qlen)):
        assert_topk_ok(s[r], i[r], S_o[r], ids, k, qlen[r], 128, f"packed {name} q{r}")
    if kind == "planted":
        tgt = gen.query_targets(12, 21, c["C"], False) + 777
        assert (i[:, 0] == tgt).all()
    dense = H.hiper_index_build(to_dev(corp), clen, id_base=777)
    s_d, i_d = [t.cpu().numpy() for t in H.hiper_maxsim_topk(dense, to_dev(q), qlen, k)]
    assert np.array_equal(i, i_d) and np.array_equal(s.view(np.uint32), s_d.view(np.uint32))


def test_packed_edge_cases(H):
    # k > n, one chunk, empty index
    corp, clen, q, qlen = semantic_case(3, 64, 5, 64, lens=[1, 64, 17])
    idx = packed_index(H, corp, clen)
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), qlen, 7)]
    assert (i[:, 3:] == -1).all() and np.isneginf(s[:, 3:]).all()
    assert sorted(i[0, :3].tolist()) == [0, 1, 2]
    e = H.hiper_index_build(torch.empty((0, 16, 64), dtype=torch.bfloat16, device="cuda"), [],
                            flags=H.HIPER_PACKED)
    s, i = H.hiper_maxsim_topk(e, to_dev(q), qlen, 5)
    assert (i.cpu().numpy() == -1).all()
    # masking adversary (P10) inside shared tiles: all real dots negative
    d = 128
    qv = np.zeros((4, 32, d), np.float32)
    qv[:, 0, 0] = 1.0
    rng = np.random.default_rng(3)
    docs = np.zeros((40, 64, d), np.float32)
    docs[:, :, 0] = -np.abs(rng.standard_normal((40, 64))) - 0.1
    docs[:, :, 1:] = rng.standard_normal((40, 64, d - 1)) * 0.1
    dl = rng.integers(1, 65, 40).astype(np.int32)
    idx = packed_index(H, docs, dl)
    S = H.hiper_maxsim_scores(idx, to_dev(qv), np.ones(4, np.int32)).cpu().numpy()
    assert (S < 0).all()
    with pytest.raises(H.HiperError) as ex:  # a borrowed packed buffer must be bf16
        H.hiper_index_build(to_dev(docs.astype(np.float32)), dl,
                            flags=H.HIPER_PACKED | H.HIPER_BORROW_TOKENS)
    assert ex.value.name == "HIPER_ERR_INVALID_ARG"


def test_packed_fake_sharding_bitwise(H):
    """P13 with packed shards: per-shard packing differs, results do not."""
    corp, clen, q, qlen = semantic_case(900, 256, 9, 128, kind="iid")
    k = 16
    idx = packed_index(H, corp, clen)
    s_ref, i_ref = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), qlen, k)]
    bounds = [0, 250, 251, 900]
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        ix = packed_index(H, corp[a:b], clen[a:b], id_base=a)
        parts.append([t.cpu().numpy() for t in H.hiper_maxsim_topk(ix, to_dev(q), qlen, k)])
    for r in range(9):
        cand = [(float(s), int(i)) for ps, pi in parts for s, i in zip(ps[r], pi[r]) if i >= 0]
        cand.sort(key=lambda t: (-t[0], t[1]))
        assert [c[1] for c in cand[:k]] == i_ref[r].tolist()


def test_packed_borrow_in_place(H):
    """HIPER_PACKED | HIPER_BORROW_TOKENS: a corpus generated straight into the packed layout and
    NORM'd in place gives the same layout and results as packing a padded tensor."""
    from synth import device
    C, L, d = 500, 256, 128
    corp, clen, q, qlen = semantic_case(C, L, 9, d)
    ref = packed_index(H, corp, clen)
    dst, n_rows = H.hiper_pack_dst_rows(clen)
    buf = torch.full((n_rows, d), 7.0, dtype=torch.bfloat16, device="cuda")  # junk must not matter
    device.corpus_packed_(buf, 11, 0, torch.from_numpy(dst).cuda(), torch.from_numpy(clen).cuda(), L)
    idx = H.hiper_index_build(buf, clen, flags=H.HIPER_PACKED | H.HIPER_BORROW_TOKENS)
    assert idx.packed and idx.layout_ptr == buf.data_ptr() and idx.n_rows == n_rows
    got = bits(idx.layout().clone())
    assert np.array_equal(got, bits(ref.layout().clone()))
    s1, i1 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(q), qlen, 10)]
    s0, i0 = [t.cpu().numpy() for t in H.hiper_maxsim_topk(ref, to_dev(q), qlen, 10)]
    assert np.array_equal(i1, i0) and np.array_equal(s1.view(np.uint32), s0.view(np.uint32))


def test_packed_masking_adversary(H):
    """P10 on the packed layout: every real doc token has a negative dot with the query token, and no
    length is a multiple of 16, so a zero padding row would win the max.  The padding rows repeat
    each chunk's last real row, so the packed scores equal the oracle's (negative) masked scores and
    the dense index's bitwise, through both the dense-score and the top-k epilogues."""
    d = 128
    qv = np.zeros((4, 32, d), np.float32)
    qv[:, 0, 0] = 1.0
    qlen = np.ones(4, np.int32)
    rng = np.random.default_rng(5)
    C, L = 40, 64
    docs = np.zeros((C, L, d), np.float32)
    docs[:, :, 0] = -np.abs(rng.standard_normal((C, L))) - 0.1
    docs[:, :, 1:] = rng.standard_normal((C, L, d - 1)) * 0.1
    clen = np.array([(1 + 3 * c) % 63 + 1 for c in range(C)], np.int32)
    clen[clen % 16 == 0] += 1
    idx = packed_index(H, docs, clen)
    S = H.hiper_maxsim_scores(idx, to_dev(qv), qlen).cpu().numpy()
    ql = query_layout(H, qv, qlen)
    lay = expected_layout(docs, clen, L)
    S_o = oracle.maxsim_matrix(ql[:len(qlen)], qlen, lay, clen)
    assert (S_o < 0).all() and (S < 0).all()
    assert_scores_close(S, S_o, qlen, d, "packed masking")
    dense = H.hiper_index_build(to_dev(docs), clen)
    S_d = H.hiper_maxsim_scores(dense, to_dev(qv), qlen).cpu().numpy()
    assert np.array_equal(S.view(np.uint32), S_d.view(np.uint32))
    s, i = [t.cpu().numpy() for t in H.hiper_maxsim_topk(idx, to_dev(qv), qlen, 5)]
    s_d, i_d = [t.cpu().numpy() for t in H.hiper_maxsim_topk(dense, to_dev(qv), qlen, 5)]
    assert np.array_equal(i, i_d) and np.array_equal(s.view(np.uint32), s_d.view(np.uint32))
    assert (s < 0).all()
