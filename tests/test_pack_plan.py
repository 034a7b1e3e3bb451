"""NEXT N4 host logic (no GPU): the packing plan behind HIPER_PACKED, and the semantic-chunk length
recipe of the variable-length workload (DESIGN.md §7.5 / §5)."""
import numpy as np
import pytest

from synth import gen


@pytest.fixture(scope="module")
def H():
    import paper_2505_04846_b200 as H
    try:
        H.lib()
    except Exception as e:  # the library is built by __graft_entry__.build()
        pytest.skip(f"libhiper.so not built: {e}")
    return H


def check_plan(lens, tiles, ents, n_rows):
    """Every invariant hiper.h states for hiper_pack_plan."""
    lens = np.asarray(lens)
    n = len(lens)
    w = (lens + 15) // 16 * 16
    assert ents.shape == (n, 2)
    # every chunk exactly once, with its own length
    assert np.array_equal(np.sort(ents[:, 0]), np.arange(n))
    assert np.array_equal(ents[:, 1] & 0xFFFF, lens[ents[:, 0]])
    row = 0
    e_next = 0
    for t0, nr, e0, e1 in tiles.tolist():
        assert t0 == row and 0 < nr <= 256 and nr % 16 == 0
        assert e0 == e_next and e1 > e0 and e1 - e0 <= 16
        col = 0
        for e in range(e0, e1):               # segments tile [0, n_rows) in order, no gaps
            c, cl = ents[e]
            assert (cl >> 16) == col and col % 16 == 0
            col += w[c]
        assert col == nr
        row += nr
        e_next = e1
    assert e_next == n and row == n_rows == int(w.sum())


def test_pack_plan_invariants(H):
    rng = np.random.default_rng(7)
    for lens in (rng.integers(1, 257, 3000), np.ones(100, np.int64), np.full(40, 256),
                 rng.integers(1, 17, 500), np.array([256, 1, 255, 16, 17, 240, 15]),
                 gen.semantic_lengths(3, 5000, 256)):
        tiles, ents, n_rows = H.hiper_pack_plan(lens)
        check_plan(lens, tiles, ents, n_rows)


def test_pack_plan_fill_and_special_cases(H):
    # full-length chunks: one per tile (the dense layout, tile = chunk)
    tiles, ents, _ = H.hiper_pack_plan(np.full(10, 256))
    assert len(tiles) == 10 and (tiles[:, 1] == 256).all()
    assert np.array_equal(ents[:, 0], np.arange(10))
    # single-token chunks: 16 per tile
    tiles, _, _ = H.hiper_pack_plan(np.ones(64, np.int64))
    assert len(tiles) == 4 and (tiles[:, 3] - tiles[:, 2] == 16).all()
    # the semantic-chunking workload packs tiles almost full (greedy largest-first fill)
    lens = gen.semantic_lengths(1, 20000, 256)
    tiles, _, n_rows = H.hiper_pack_plan(lens)
    assert n_rows / (256 * len(tiles)) > 0.99
    # empty corpus; deterministic
    tiles, ents, n_rows = H.hiper_pack_plan(np.zeros(0, np.int32))
    assert len(tiles) == 0 and n_rows == 0
    a = H.hiper_pack_plan(lens[:999])
    b = H.hiper_pack_plan(lens[:999])
    assert all(np.array_equal(x, y) for x, y in zip(a[:2], b[:2]))


def test_pack_plan_errors(H):
    for bad in ([3, 0, 5], [257], [-1]):
        with pytest.raises(H.HiperError) as e:
            H.hiper_pack_plan(np.array(bad))
        assert e.value.name == "HIPER_ERR_INVALID_ARG"


def test_semantic_lengths_recipe():
    lens = gen.semantic_lengths(1, 100000, 256)
    assert lens.dtype == np.int32 and lens.min() >= gen.SEM_SENT_MIN and lens.max() == 256
    # 1 + Geometric(1 - p) sentences of mean 26 tokens: mean ~ 26 / (1 - 0.75) = 104 before truncation
    assert 90 < lens.mean() < 105
    # a single sentence (prob 1 - p = 0.25) lies in [12, 40]
    assert 0.22 < (lens <= gen.SEM_SENT_MAX).mean() < 0.30
    # counter-based: any slice regenerates the same lengths; other seeds differ
    assert np.array_equal(gen.semantic_lengths(1, 500, 256, start=700), lens[700:1200])
    assert not np.array_equal(gen.semantic_lengths(2, 500, 256), lens[:500])
    assert (gen.semantic_lengths(1, 1000, 64) == np.minimum(lens[:1000], 64)).all()
