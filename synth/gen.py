"""Seeded synthetic inputs shared by the oracle side and the CUDA side (numpy implementation).

This module holds NONE of the method's arithmetic (no normalisation, no dot products, no max/sum,
no top-k, no loss): it only draws token embeddings.  It is a counter-based generator, so any
(chunk, token, dim) element can be produced independently and identically here and on the device
(``synth/csrc/synth.cu`` implements the same integer recipe; ``tests/test_gpu_parity.py::test_synth_device_matches_numpy`` checks the
two bitwise).

Recipe:
* ``h(seed, stream, i) = splitmix64(key(seed, stream) + i)``, ``key = splitmix64(seed ^ (stream << 48))``
* ``g(h)`` = Irwin-Hall(4) of the four 16-bit lanes of ``h``, centred, times 2**-15: an exactly
  representable float32 in (-4, 4) with std ~1.155 -- no libm, so host and device agree bit for bit.
* iid corpus: ``x[c,j,k] = g(h(seed, TOK, (c*L + j)*d + k))``.
* planted-topic corpus (the paper's query->chunk pairing: "a high-level question that
  uses the chunk as a reference"): chunk ``c`` has topic ``t(c)``; 25% of its tokens take a second
  topic; ``x = cent[t][k] + sigma*g(...)`` in float32 (one RN multiply, one RN add).
* planted queries: query ``q`` copies tokens of a target chunk ``c*(q)`` and adds
  ``sigma_q * g(...)`` noise; ``c*(q) = h(qseed, QTARGET, q) % C`` or ``q`` (diagonal, for the
  in-batch ColTrast step where query i's positive is chunk i).
* lengths: fixed, or ``1 + h(seed, LEN, c) % L`` (variable, for masking parity), or the
  semantic-chunking recipe ``semantic_lengths`` (NEXT N4 workload).
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# stream ids
TOK, CENT, TOPIC, TOPIC2, MIX, LEN, QTARGET, QPOS, QTOK, QLEN, SEMLEN = range(1, 12)

N_TOPICS = 4096
SIGMA_TOKEN = np.float32(0.75)      # token noise around the topic centroid
SIGMA_Q_EASY = np.float32(0.125)     # retrieval configs: target chunk is top-1 by a wide margin
SIGMA_Q_HARD = np.float32(6.0)       # ColTrast step: InfoNCE stays O(1) at tau = 1


def splitmix64(x):
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def key(seed: int, stream: int) -> np.uint64:
    return splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream) << np.uint64(48)))


def h(seed: int, stream: int, idx) -> np.ndarray:
    with np.errstate(over="ignore"):
        return splitmix64(key(seed, stream) + np.asarray(idx, dtype=np.uint64))


def g_of(hv: np.ndarray) -> np.ndarray:
    """Irwin-Hall(4) of the 16-bit lanes, centred, * 2**-15 -> float32 (exact)."""
    m = np.uint64(0xFFFF)
    s = ((hv & m) + ((hv >> np.uint64(16)) & m) + ((hv >> np.uint64(32)) & m)
         + (hv >> np.uint64(48))).astype(np.int64) - 131070
    return (s.astype(np.float32) * np.float32(2.0 ** -15)).astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """IEEE round-to-nearest-even float32 -> bf16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return (u >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(u: np.ndarray) -> np.ndarray:
    return (np.asarray(u, dtype=np.uint32) << 16).view(np.float32)


# ---------------------------------------------------------------- lengths
def lengths(seed: int, n: int, max_len: int, variable: bool, start: int = 0,
            stream: int = LEN) -> np.ndarray:
    if not variable:
        return np.full(n, max_len, dtype=np.int32)
    idx = np.arange(start, start + n, dtype=np.uint64)
    return (np.uint64(1) + h(seed, stream, idx) % np.uint64(max_len)).astype(np.int32)


# Semantic-chunk lengths (NEXT N4 workload).  The paper's chunker keeps "adding to a segment as long
# as the cosine similarity between consecutive sentences remains above a predetermined threshold"
# (PAPER.md:274), so the sentence count of a chunk is 1 + Geometric: each next sentence joins with a
# fixed probability P_CONT.  Sentence lengths are U[SENT_MIN, SENT_MAX] tokens; the encoder truncates
# at max_len.  Paper silent on both numbers -- DESIGN.md records the reading (mean ~104 tokens).
SEM_P_CONT = 0.75
SEM_SENT_MIN, SEM_SENT_MAX = 12, 40
SEM_MAX_SENT = 64


def semantic_lengths(seed: int, n: int, max_len: int, start: int = 0) -> np.ndarray:
    """int32 [n] chunk lengths of chunks start..start+n-1 (counter-based: any slice regenerates).

    u_s = h(seed, SEMLEN, c*64 + s); sentence s has 12 + (u_s >> 16) % 29 tokens; sentence s+1 joins
    iff (u_{s+1} & 0xFFFF) < 0.75 * 65536 (and every earlier one joined)."""
    out = np.empty(n, dtype=np.int32)
    thr = np.uint64(int(SEM_P_CONT * 65536))
    span = np.uint64(SEM_SENT_MAX - SEM_SENT_MIN + 1)
    for b0 in range(0, n, 1 << 16):
        c = np.arange(start + b0, start + min(n, b0 + (1 << 16)), dtype=np.uint64)
        s = np.arange(SEM_MAX_SENT, dtype=np.uint64)
        with np.errstate(over="ignore"):
            u = h(seed, SEMLEN, c.reshape(-1, 1) * np.uint64(SEM_MAX_SENT) + s.reshape(1, -1))
        slen = (np.uint64(SEM_SENT_MIN) + (u >> np.uint64(16)) % span).astype(np.int64)
        join = (u & np.uint64(0xFFFF)) < thr
        join[:, 0] = True                                   # the first sentence always starts it
        alive = np.cumprod(join, axis=1).astype(bool)       # stops at the first failed join
        tot = (slen * alive).sum(axis=1)
        out[b0:b0 + len(c)] = np.minimum(tot, max_len).astype(np.int32)
    return out


# ---------------------------------------------------------------- corpus
def corpus_tokens_f32(seed: int, chunks, L: int, d: int, kind: str = "planted") -> np.ndarray:
    """float32 [len(chunks)][L][d] raw (un-normalised) token embeddings of the given chunk ids."""
    c = np.asarray(chunks, dtype=np.uint64).reshape(-1, 1, 1)
    j = np.arange(L, dtype=np.uint64).reshape(1, -1, 1)
    k = np.arange(d, dtype=np.uint64).reshape(1, 1, -1)
    with np.errstate(over="ignore"):
        tok_idx = (c * np.uint64(L) + j) * np.uint64(d) + k
    noise = g_of(h(seed, TOK, tok_idx))
    if kind == "iid":
        return noise
    assert kind == "planted", kind
    t1 = h(seed, TOPIC, c) % np.uint64(N_TOPICS)
    t2 = h(seed, TOPIC2, c) % np.uint64(N_TOPICS)
    with np.errstate(over="ignore"):
        mix = (h(seed, MIX, c * np.uint64(L) + j) & np.uint64(3)) == 0
    t = np.where(mix, t2, t1)
    cent = g_of(h(seed, CENT, t * np.uint64(d) + k))
    return (cent + (SIGMA_TOKEN * noise).astype(np.float32)).astype(np.float32)


def corpus(seed: int, chunk_start: int, n: int, L: int, d: int, kind: str = "planted",
           dtype: str = "bf16") -> np.ndarray:
    x = corpus_tokens_f32(seed, np.arange(chunk_start, chunk_start + n), L, d, kind)
    return f32_to_bf16_bits(x) if dtype == "bf16" else x


# ---------------------------------------------------------------- queries
def query_targets(qseed: int, n_q: int, n_chunks: int, diagonal: bool, start: int = 0):
    qi = np.arange(start, start + n_q, dtype=np.uint64)
    if diagonal:
        return qi.astype(np.int64) % n_chunks
    return (h(qseed, QTARGET, qi) % np.uint64(n_chunks)).astype(np.int64)


def queries(qseed: int, n_q: int, Lq: int, d: int, *, corpus_seed: int, n_chunks: int, L: int,
            chunk_lens_fn=None, kind: str = "planted", corpus_kind: str = "planted",
            sigma_q=SIGMA_Q_EASY,
            diagonal: bool = False, dtype: str = "bf16", start: int = 0) -> np.ndarray:
    """[n_q][Lq][d] query token embeddings.

    planted: token i of query q = corpus token (c*(q), j_i) + sigma_q * g, j_i = h(QPOS) % len(c*).
    chunk_lens_fn(c) -> lengths of chunks c (default: all L)."""
    qi = np.arange(start, start + n_q, dtype=np.uint64)
    i = np.arange(Lq, dtype=np.uint64)
    k = np.arange(d, dtype=np.uint64)
    with np.errstate(over="ignore"):
        tok_idx = ((qi.reshape(-1, 1, 1) * np.uint64(Lq) + i.reshape(1, -1, 1)) * np.uint64(d)
                   + k.reshape(1, 1, -1))
    noise = g_of(h(qseed, QTOK, tok_idx))
    if kind == "iid":
        x = noise
    else:
        tgt = query_targets(qseed, n_q, n_chunks, diagonal, start)
        tl = (np.full(n_q, L, dtype=np.int64) if chunk_lens_fn is None
              else np.asarray(chunk_lens_fn(tgt), dtype=np.int64))
        with np.errstate(over="ignore"):
            pos = h(qseed, QPOS, qi.reshape(-1, 1) * np.uint64(Lq) + i.reshape(1, -1))
        j = (pos % tl.reshape(-1, 1).astype(np.uint64)).astype(np.int64)   # [n_q][Lq]
        base = np.empty((n_q, Lq, d), dtype=np.float32)
        for qq in range(n_q):
            toks = corpus_tokens_f32(corpus_seed, [tgt[qq]], L, d, corpus_kind)[0]
            base[qq] = toks[j[qq]]
        x = (base + (np.float32(sigma_q) * noise).astype(np.float32)).astype(np.float32)
    return f32_to_bf16_bits(x) if dtype == "bf16" else x
