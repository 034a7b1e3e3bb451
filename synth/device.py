"""Device side of the seeded generator (synth/csrc/synth.cu -> synth/libsynth.so).

Same counter-based recipe as synth/gen.py, bit for bit; used to materialise large corpora (e.g. the
65.5 GB 1M-chunk corpus) directly in HBM.  No method arithmetic here."""
from __future__ import annotations

import ctypes
import os

from . import gen

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB)
        P, i32, i64, u64, f32 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                 ctypes.c_float)
        L.synth_corpus.argtypes = [P, i32, i64, i64, i32, i32, u64, i32, f32, P]
        L.synth_corpus.restype = i32
        L.synth_queries.argtypes = [P, i32, i64, i64, i32, i32, u64, i32, i32, i64, i32, P, u64,
                                    i32, f32, f32, P]
        L.synth_queries.restype = i32
        L.synth_corpus_packed.argtypes = [P, i64, i64, i32, i32, u64, i32, f32, P, P, P]
        L.synth_corpus_packed.restype = i32
        _lib = L
    return _lib


def _stream(stream):
    import torch
    return ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)


def corpus_(out, seed: int, chunk_start: int, kind: str = "planted", stream=None):
    """Fill CUDA tensor out [n][L][d] (float32 or bfloat16) with corpus chunks chunk_start.."""
    import torch
    n, L, d = out.shape
    r = lib().synth_corpus(ctypes.c_void_p(out.data_ptr()), int(out.dtype == torch.bfloat16),
                           chunk_start, n, L, d, seed & (2**64 - 1), int(kind == "planted"),
                           float(gen.SIGMA_TOKEN), _stream(stream))
    if r != 0:
        raise RuntimeError(f"synth_corpus CUDA error {r}")
    return out


def queries_(out, qseed: int, *, corpus_seed: int, n_chunks: int, L: int, chunk_lens=None,
             kind: str = "planted", corpus_kind: str = "planted", sigma_q=gen.SIGMA_Q_EASY,
             diagonal: bool = False, start: int = 0, stream=None):
    """Fill CUDA tensor out [n_q][Lq][d] with queries (see gen.queries); chunk_lens: CUDA int32 [C]."""
    import torch
    n_q, Lq, d = out.shape
    r = lib().synth_queries(ctypes.c_void_p(out.data_ptr()), int(out.dtype == torch.bfloat16),
                            start, n_q, Lq, d, qseed & (2**64 - 1), int(diagonal),
                            int(kind == "planted"), n_chunks, L,
                            ctypes.c_void_p(chunk_lens.data_ptr()) if chunk_lens is not None else None,
                            corpus_seed & (2**64 - 1), int(corpus_kind == "planted"),
                            float(gen.SIGMA_TOKEN), float(sigma_q), _stream(stream))
    if r != 0:
        raise RuntimeError(f"synth_queries CUDA error {r}")
    return out


def corpus_packed_(out, seed: int, chunk_start: int, dst_row, lens, L: int, kind: str = "planted",
                   stream=None):
    """Fill the packed bf16 CUDA tensor out [rows][d] with chunks chunk_start.. (count = len(lens)):
    chunk c's token j at row dst_row[c] + j (dst_row: CUDA int64, lens: CUDA int32), zero padding up
    to the chunk's 16-row slot; token values as corpus_() with token stride L."""
    n = lens.shape[0]
    d = out.shape[-1]
    r = lib().synth_corpus_packed(ctypes.c_void_p(out.data_ptr()), chunk_start, n, L, d,
                                  seed & (2**64 - 1), int(kind == "planted"), float(gen.SIGMA_TOKEN),
                                  ctypes.c_void_p(dst_row.data_ptr()), ctypes.c_void_p(lens.data_ptr()),
                                  _stream(stream))
    if r != 0:
        raise RuntimeError(f"synth_corpus_packed CUDA error {r}")
    return out
