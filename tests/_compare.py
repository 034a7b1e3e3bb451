"""Comparison rules between the CUDA path and the oracle.

* scores: |S_gpu - S_o| <= tol(S_o) = max(2e-3 * |S_o|, d * len_q * 2^-24)   (north star 2e-3
  relative, bf16 in / fp32 accumulate; the floor is the fp32 accumulation bound for unit rows, R8)
* top-k (R8/g8): no duplicate ids; every returned score within tol of the oracle score of its id;
  position r holds an item whose oracle score is within tol of the true r-th score (so ids may
  differ only inside near-tie runs); bitwise-equal GPU scores come in ascending id order.
* loss: |L_gpu - L_o| <= max(1e-4 * |L_o|, 1e-7)
"""
from __future__ import annotations

import numpy as np

import oracle


def score_tol(s_oracle, len_q, d):
    return np.maximum(2e-3 * np.abs(s_oracle), d * np.asarray(len_q, dtype=np.float64) * 2.0 ** -24)


def assert_scores_close(S_gpu, S_o, q_lens, d, what=""):
    S_gpu = np.asarray(S_gpu, dtype=np.float64)
    tol = score_tol(S_o, np.asarray(q_lens).reshape(-1, 1), d)
    err = np.abs(S_gpu - S_o)
    bad = err > tol
    assert not bad.any(), (f"{what}: {bad.sum()} scores outside tolerance; worst "
                           f"{np.unravel_index(np.argmax(err - tol), err.shape)} "
                           f"gpu={S_gpu.flat[np.argmax(err - tol)]} oracle={S_o.flat[np.argmax(err - tol)]}")
    return float(np.max(err / np.maximum(np.abs(S_o), 1e-30))) if S_o.size else 0.0


def assert_topk_ok(gpu_scores, gpu_ids, oracle_scores_all, ids_all, k, len_q, d, what=""):
    """One query.  oracle_scores_all / ids_all: every candidate's oracle score and global id."""
    gpu_scores = np.asarray(gpu_scores, dtype=np.float64)
    gpu_ids = np.asarray(gpu_ids, dtype=np.int64)
    n = len(ids_all)
    m = min(k, n)
    o_s, o_i = oracle.topk(oracle_scores_all, ids_all, k)
    # padding
    assert (gpu_ids[m:] == -1).all() and np.isneginf(gpu_scores[m:]).all(), f"{what}: padding"
    g_i = gpu_ids[:m]
    assert len(set(g_i.tolist())) == m, f"{what}: duplicate ids {g_i}"
    pos = {int(i): j for j, i in enumerate(ids_all.tolist())}
    assert all(int(i) in pos for i in g_i), f"{what}: unknown ids"
    s_of = np.array([oracle_scores_all[pos[int(i)]] for i in g_i])
    tol = score_tol(s_of, len_q, d)
    assert (np.abs(gpu_scores[:m] - s_of) <= tol).all(), f"{what}: returned score vs oracle"
    tol_r = score_tol(o_s[:m], len_q, d)
    assert (np.abs(s_of - o_s[:m]) <= tol_r).all(), (
        f"{what}: rank mismatch outside near-ties gpu={g_i.tolist()} oracle={o_i[:m].tolist()}")
    # exact ties in fp32: ascending ids
    for r in range(m - 1):
        if gpu_scores[r] == gpu_scores[r + 1]:
            assert g_i[r] < g_i[r + 1], f"{what}: tie order at {r}"
        assert gpu_scores[r] >= gpu_scores[r + 1], f"{what}: not sorted at {r}"
    return int((g_i != o_i[:m]).sum())


def assert_loss_close(L_gpu, L_o, what=""):
    assert abs(L_gpu - L_o) <= max(1e-4 * abs(L_o), 1e-7), f"{what}: gpu {L_gpu} oracle {L_o}"
