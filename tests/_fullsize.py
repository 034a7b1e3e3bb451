"""Helpers of the full-size parity tests (test infrastructure; -m gpu only).

* torch_ref_dense / torch_ref_packed: an independent library-routine reference over a WHOLE corpus
  for a few queries -- fp32 GEMM of the bf16 operands (exact products, cuBLAS / torch), masked amax
  over each chunk's real tokens, sum over query tokens.  Shares no code with the kernels.
* exact_cosine: the informational deviation of SURVEY §8(c): MaxSim on float64-normalised RAW input
  rows (no bf16 rounding of the normalised rows), i.e. what reading R1's bf16 NORM costs against
  the paper's cosine definition ("cosine(q_i, d_j)").  Reported, never gated.
"""
from __future__ import annotations

import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(t):
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def torch_ref_dense(lay, lens_dev, qrows, lq, step=4096):
    """lay: CUDA bf16 [C][ld][d] (rows >= len ignored); qrows: CUDA f32 [nq*lq][d] NORM'd query rows
    (all lq rows real); lens_dev: CUDA int32 [C] -> float64 numpy [nq][C]."""
    import torch
    C, ld, d = lay.shape
    nq = qrows.shape[0] // lq
    ref = torch.empty((nq, C), dtype=torch.float32, device="cuda")
    col = torch.arange(ld, device="cuda")
    for c0 in range(0, C, step):
        c1 = min(C, c0 + step)
        blk = lay[c0:c1].reshape(-1, d).float()
        sim = (qrows @ blk.T).view(nq, lq, c1 - c0, ld)
        pad = (col[None, :] >= lens_dev[c0:c1, None])           # [n][ld] padding rows
        sim.masked_fill_(pad[None, None], float("-inf"))
        ref[:, c0:c1] = sim.amax(dim=3).sum(dim=1)
    return ref.cpu().numpy().astype(np.float64)


def torch_ref_packed(lay, row_chunk, n_chunks, qrows, lq, step=1 << 22):
    """lay: CUDA bf16 [n_rows][d] packed layout; row_chunk: CUDA int64 [n_rows] chunk of each packed
    row, -1 for rows that are not a real token (padding / tile slack) -> float64 numpy [nq][C]."""
    import torch
    nq = qrows.shape[0] // lq
    m = torch.full((nq * lq, n_chunks), float("-inf"), dtype=torch.float32, device="cuda")
    for r0 in range(0, lay.shape[0], step):
        r1 = min(lay.shape[0], r0 + step)
        sim = qrows @ lay[r0:r1].float().T                        # [nq*lq][rows]
        rc = row_chunk[r0:r1]
        real = rc >= 0
        m.scatter_reduce_(1, rc[real][None].expand(nq * lq, -1), sim[:, real], reduce="amax")
    return m.view(nq, lq, n_chunks).sum(dim=1).cpu().numpy().astype(np.float64)


def exact_cosine(q_in, c_in):
    """Sum_i max_j cos(q_i, d_j) in float64 on raw input rows (float32 arrays, real rows only)."""
    qn = q_in.astype(np.float64)
    qn /= np.linalg.norm(qn, axis=-1, keepdims=True)
    cn = c_in.astype(np.float64)
    cn /= np.linalg.norm(cn, axis=-1, keepdims=True)
    return float((qn @ cn.T).max(axis=1).sum())


def record_info(name: str, values: dict):
    """Append an informational (ungated) measurement to gpurun_out/informational.jsonl."""
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "informational.jsonl"), "a") as f:
        f.write(json.dumps({"test": name, **values}) + "\n")
    print(name, values)
