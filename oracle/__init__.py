"""CPU oracle for the ColTrast MaxSim hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import this package.  The product package ``paper_2505_04846_b200``
never imports it and shares no code with it (see the header of ``oracle/oracle.c``).

The arithmetic lives in ``oracle/oracle.c`` (plain float64 loops; NORM in IEEE fp32 op by op);
this module only marshals numpy arrays into it.  Each wrapper names the passage it follows:

* :func:`norm_rows`      NORM, row normalisation on entry (reading R1)
* :func:`maxsim`         S(q,d) = sum_i max_j <q_i,d_j>  (§2.2, Fig. 3B,
                         SPEC.md:259-267)
* :func:`maxsim_matrix`  every (query, doc) pair of the above
* :func:`topk`           exact top-k, score desc then id asc, padded (-inf,-1) (§2.3,
                         SPEC.md:193-201)
* :func:`infonce`        mean_i logsumexp_j(S_ij/tau) - S_{i,pos_i}/tau  ("L_LI is
                         maxsim loss"; also L_C's SimCSE form)
* :func:`gather_candidates`  min(N, W) candidates, local positives first, then (rank, position)
                         order -- plain list logic
* :func:`coltrast_total` L = (L_LI + L_C) / 2
* :func:`li_loss_grad`   gradient of L_LI w.r.t. the raw token rows, chain rule through the argmax
                         and the normalisation (NEXT N1; SPEC.md:357-365 grad_check pins it by
                         central finite differences in float64)

Parity status: every function above is pinned by ``tests/test_oracle_pins.py`` (no "parity
unpinned" function).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
             "-fopenmp"]


def build(force: bool = False) -> str:
    """Compile oracle/oracle.c -> oracle/liboracle.so with gcc (no GPU involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        _lib.oracle_norm_rows.argtypes = [P, i32, i64, i32, i32, P, P]
        _lib.oracle_norm_rows.restype = i64
        _lib.oracle_maxsim.argtypes = [P, i32, P, i32, i32]
        _lib.oracle_maxsim.restype = ctypes.c_double
        _lib.oracle_maxsim_matrix.argtypes = [P, P, i64, i32, P, P, i64, i32, i32, P, i32]
        _lib.oracle_maxsim_matrix.restype = None
        _lib.oracle_topk.argtypes = [P, P, i64, i32, P, P]
        _lib.oracle_topk.restype = None
        _lib.oracle_infonce.argtypes = [P, i32, i32, P, ctypes.c_double]
        _lib.oracle_infonce.restype = ctypes.c_double
        _lib.oracle_maxsim_infonce_grad.argtypes = [P, P, i32, i32, P, P, i32, i32, i32, P,
                                                    ctypes.c_double, i32, P, P, P, P, P]
        _lib.oracle_maxsim_infonce_grad.restype = ctypes.c_double
        _lib.oracle_max_threads.argtypes = []
        _lib.oracle_max_threads.restype = i32
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(ValueError):
    pass


def norm_rows(x: np.ndarray, assume_normalized: bool = False) -> np.ndarray:
    """NORM every row of ``x`` ([..., d], float32 or bf16 bit patterns as uint16) -> uint16 bf16.

    Raises OracleError('zero', row) / OracleError('nonfinite', row) like SPEC ZeroVector."""
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        dt = 0
    elif x.dtype == np.uint16:
        dt = 1
    else:
        raise TypeError(x.dtype)
    d = x.shape[-1]
    n = int(np.prod(x.shape[:-1])) if x.ndim > 1 else 1
    y = np.zeros(x.shape, dtype=np.uint16)
    st = np.zeros(1, dtype=np.int32)
    r = lib().oracle_norm_rows(_ptr(x), dt, n, d, int(bool(assume_normalized)), _ptr(y), _ptr(st))
    if r >= 0:
        raise OracleError({1: "zero", 2: "nonfinite"}.get(int(st[0]), "bad"), int(r))
    return y


def maxsim(q: np.ndarray, doc: np.ndarray, len_q: int | None = None,
           len_d: int | None = None) -> float:
    """S(q,d) over NORM'd bf16 rows (uint16 [Lq][d], [Ld][d]); only the first len rows count."""
    q = np.ascontiguousarray(q, dtype=np.uint16)
    doc = np.ascontiguousarray(doc, dtype=np.uint16)
    lq = q.shape[0] if len_q is None else len_q
    ld = doc.shape[0] if len_d is None else len_d
    if lq < 1 or ld < 1:
        raise OracleError("empty", 0)
    return float(lib().oracle_maxsim(_ptr(q), lq, _ptr(doc), ld, q.shape[1]))


def maxsim_matrix(q_tokens: np.ndarray, q_lens, d_tokens: np.ndarray, d_lens,
                  n_threads: int = 0) -> np.ndarray:
    """All-pairs MaxSim: q_tokens [n_q][Lq][d], d_tokens [n_d][Ld][d] (uint16 bf16) -> [n_q][n_d] f64."""
    q_tokens = np.ascontiguousarray(q_tokens, dtype=np.uint16)
    d_tokens = np.ascontiguousarray(d_tokens, dtype=np.uint16)
    ql = np.ascontiguousarray(q_lens, dtype=np.int32)
    dl = np.ascontiguousarray(d_lens, dtype=np.int32)
    nq, lq, d = q_tokens.shape
    nd, ld, d2 = d_tokens.shape
    assert d == d2 and ql.shape == (nq,) and dl.shape == (nd,)
    if (ql < 1).any() or (dl < 1).any():
        raise OracleError("empty", 0)
    out = np.empty((nq, nd), dtype=np.float64)
    lib().oracle_maxsim_matrix(_ptr(q_tokens), _ptr(ql), nq, lq, _ptr(d_tokens), _ptr(dl), nd, ld,
                               d, _ptr(out), int(n_threads))
    return out


def topk(scores: np.ndarray, ids: np.ndarray, k: int):
    """Exact top-k of one query's scores: (scores desc, ids asc), padded with (-inf, -1)."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    i = np.ascontiguousarray(ids, dtype=np.int64)
    os_ = np.empty(k, dtype=np.float64)
    oi = np.empty(k, dtype=np.int64)
    lib().oracle_topk(_ptr(s), _ptr(i), s.shape[0], k, _ptr(os_), _ptr(oi))
    return os_, oi


def infonce(S: np.ndarray, pos=None, tau: float = 1.0) -> float:
    """mean_i [logsumexp_j(S_ij/tau) - S_{i,pos_i}/tau] in float64 (pos default: diagonal)."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    B, M = S.shape
    if B < 1:
        raise OracleError("empty_batch", 0)
    if not tau > 0:
        raise OracleError("temperature", 0)
    p = np.arange(B, dtype=np.int32) if pos is None else np.ascontiguousarray(pos, dtype=np.int32)
    if (p < 0).any() or (p >= M).any():
        raise OracleError("positive", 0)
    return float(lib().oracle_infonce(_ptr(S), B, M, _ptr(p), float(tau)))


def gather_candidates(batches, local_rank: int, N: int):
    """PAPER.md:252 "loss is calculated with the local rank compared to min(N, W) samples, where N is
    the maximum to consider and W is the total samples across all ranks"; SPEC.md:321-329 fill order:
    the local rank's positives first, then the other ranks' rows in (rank, position) order."""
    b = len(batches[local_rank])
    W = sum(len(x) for x in batches)
    if N < b:
        raise OracleError("NTooSmall", N)
    m = min(N, W)
    out = list(batches[local_rank])
    for r, batch in enumerate(batches):
        if r == local_rank:
            continue
        for row in batch:
            if len(out) == m:
                return out
            out.append(row)
    return out[:m]


def coltrast_total(l_li: float, l_c: float) -> float:
    """"The total loss per iteration is L = (L_LI + L_C) / 2"."""
    return (l_li + l_c) / 2.0


def li_loss_grad(x_q, q_lens, x_d, d_lens, pos=None, tau: float = 1.0, exact_norm: bool = False):
    """(loss, grad_q, grad_d, argmax, gap, second_argmax) for L_LI over raw rows x_q [B][Lq][d],
    x_d [M][Ld][d].

    exact_norm=True normalises in float64 (differentiable; finite-difference pin); False uses the
    library's NORM (bf16 operands, as the GPU) for the forward/argmax."""
    xq = np.ascontiguousarray(x_q, dtype=np.float64)
    xd = np.ascontiguousarray(x_d, dtype=np.float64)
    B, Lq, d = xq.shape
    M, Ld, _ = xd.shape
    ql = np.ascontiguousarray(q_lens, dtype=np.int32)
    dl = np.ascontiguousarray(d_lens, dtype=np.int32)
    p = np.arange(B, dtype=np.int32) if pos is None else np.ascontiguousarray(pos, dtype=np.int32)
    gq = np.zeros_like(xq)
    gd = np.zeros_like(xd)
    am = np.zeros((B, M, Lq), dtype=np.int32)
    gap = np.zeros((B, M, Lq), dtype=np.float64)
    am2 = np.zeros((B, M, Lq), dtype=np.int32)
    loss = lib().oracle_maxsim_infonce_grad(_ptr(xq), _ptr(ql), B, Lq, _ptr(xd), _ptr(dl), M, Ld, d,
                                            _ptr(p), float(tau), int(bool(exact_norm)), _ptr(gq),
                                            _ptr(gd), _ptr(am), _ptr(gap), _ptr(am2))
    return float(loss), gq, gd, am, gap, am2


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ---------------------------------------------------------------- bf16 helpers (test plumbing)
def bf16_bits_to_f64(u: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to float64."""
    return (np.asarray(u, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)
