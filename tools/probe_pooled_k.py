"""Probe: pooled top-k time vs k on the 3.6M x 768 pooled corpus (bench's config5 data), Q queries.
Prints ms per call for each k (CUDA events, 5 calls after 2 warm-ups); run with HIPER_PIPE_STATS=1
for the kernel's pipeline counters."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_04846_b200 as H
from synth import device

C, D = int(os.environ.get("C", 3_600_000)), 768
Q = int(os.environ.get("Q", 1024))
ks = [int(x) for x in os.environ.get("KS", "10,16,17,64,100").split(",")]
corpus = torch.empty((C, 1, D), dtype=torch.bfloat16, device="cuda")
device.corpus_(corpus, 1001, 0)
idx = H.hiper_index_build(corpus, np.ones(C, np.int32), flags=H.HIPER_BORROW_TOKENS | H.HIPER_POOLED)
q = torch.empty((Q, 1, D), dtype=torch.bfloat16, device="cuda")
device.queries_(q, 2, corpus_seed=1001, n_chunks=C, L=1)
ones = np.ones(Q, np.int32)
for k in ks:
    ws = H.TopkWorkspace(idx, Q, k)
    for _ in range(2):
        H.hiper_maxsim_topk(idx, q, ones, k, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 5
    for _ in range(n):
        s, i = H.hiper_maxsim_topk(idx, q, ones, k, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"k={k}: {ms:.3f} ms per call ({2 * D * Q * C / ms / 1e9:.0f} TF/s)", flush=True)
