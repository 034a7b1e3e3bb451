"""config2 e2e feeding variants (dev probe): serial H2D + step, H2D on a copy stream double-buffered,
copies alone, steps alone.  Prints ms per step for each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_04846_b200 as H
from synth import gen

B, L, Lq, d = 256, 256, 32, 128
to_dev = lambda x: torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
docs = to_dev(gen.corpus(3, 0, B, L, d))
qs = to_dev(gen.queries(4, B, Lq, d, corpus_seed=3, n_chunks=B, L=L, diagonal=True, sigma_q=gen.SIGMA_Q_HARD))
ql, dl = np.full(B, Lq, np.int32), np.full(B, L, np.int32)
ws = H.ColtrastWorkspace(B, B, L, d)
out = (torch.empty((B, B), dtype=torch.float32, device="cuda"), torch.empty(1, dtype=torch.float32, device="cuda"))
stream = torch.cuda.current_stream()
step = lambda q, dd: H.hiper_coltrast_scores_loss(q, ql, dd, dl, temperature=1.0, workspace=ws, out=out, stream=stream)
qh, dh = qs.cpu().pin_memory(), docs.cpu().pin_memory()
qd = [torch.empty_like(qs) for _ in range(2)]
dd = [torch.empty_like(docs) for _ in range(2)]
lh = torch.empty(1, dtype=torch.float32).pin_memory()
cs = torch.cuda.Stream()
N = 100

def timed(fn):
    for _ in range(3):
        fn(5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn(N)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / N

def serial(n):
    for i in range(n):
        qd[0].copy_(qh, non_blocking=True); dd[0].copy_(dh, non_blocking=True)
        step(qd[0], dd[0]); lh.copy_(out[1], non_blocking=True)

def piped(n):
    cp = [torch.cuda.Event() for _ in range(2)]; rl = [torch.cuda.Event() for _ in range(2)]
    cs.wait_stream(stream)
    for i in range(n):
        b = i & 1
        with torch.cuda.stream(cs):
            if i >= 2: cs.wait_event(rl[b])
            qd[b].copy_(qh, non_blocking=True); dd[b].copy_(dh, non_blocking=True)
            cp[b].record(cs)
        stream.wait_event(cp[b])
        step(qd[b], dd[b]); lh.copy_(out[1], non_blocking=True)
        rl[b].record(stream)
    stream.wait_stream(cs)

ds = torch.cuda.Stream()
def piped_ds(n):
    cp = [torch.cuda.Event() for _ in range(2)]; rl = [torch.cuda.Event() for _ in range(2)]
    cs.wait_stream(stream)
    for i in range(n):
        b = i & 1
        with torch.cuda.stream(cs):
            if i >= 2: cs.wait_event(rl[b])
            qd[b].copy_(qh, non_blocking=True); dd[b].copy_(dh, non_blocking=True)
            cp[b].record(cs)
        stream.wait_event(cp[b])
        step(qd[b], dd[b])
        rl[b].record(stream)
        ds.wait_event(rl[b])
        with torch.cuda.stream(ds):
            lh.copy_(out[1], non_blocking=True)
    stream.wait_stream(cs); stream.wait_stream(ds)

def piped_nod2h(n):
    cp = [torch.cuda.Event() for _ in range(2)]; rl = [torch.cuda.Event() for _ in range(2)]
    cs.wait_stream(stream)
    for i in range(n):
        b = i & 1
        with torch.cuda.stream(cs):
            if i >= 2: cs.wait_event(rl[b])
            qd[b].copy_(qh, non_blocking=True); dd[b].copy_(dh, non_blocking=True)
            cp[b].record(cs)
        stream.wait_event(cp[b])
        step(qd[b], dd[b])
        rl[b].record(stream)
    stream.wait_stream(cs)

def copies_cs(n):
    cs.wait_stream(stream)
    with torch.cuda.stream(cs):
        for i in range(n):
            qd[i & 1].copy_(qh, non_blocking=True); dd[i & 1].copy_(dh, non_blocking=True)
    stream.wait_stream(cs)

def copies_main(n):
    for i in range(n):
        qd[i & 1].copy_(qh, non_blocking=True); dd[i & 1].copy_(dh, non_blocking=True)

def steps_only(n):
    for i in range(n):
        step(qs, docs)

import ctypes
nbg = H.lib().hiper_coltrast_grad_workspace_size(B, B, L, d)
gws, gwp, gwn = H._workspace(nbg, "cuda")
gq = torch.empty((B, Lq, d), dtype=torch.float32, device="cuda")
gdd = torch.empty((B, L, d), dtype=torch.float32, device="cuda")
def grad_step(q, dd_):
    H._check(H.lib().hiper_coltrast_scores_loss_grad(
        H._dev_ptr(q), H._ptr(ql), B, Lq, H._dev_ptr(dd_), H._ptr(dl), B, L, d,
        H._dtype_code(q), 0, None, ctypes.c_float(1.0), ctypes.c_void_p(gwp), gwn,
        H._dev_ptr(out[0]), H._dev_ptr(out[1]), H._dev_ptr(gq), H._dev_ptr(gdd), H._stream_ptr(stream)))
fwd_step = step
for name, st in (("fwd", fwd_step), ("grad", grad_step)):
  step = st
  for f in (steps_only, copies_cs, serial, piped, piped_ds, piped_nod2h):
    print(name, f.__name__, round(timed(f) * 1000, 1), "us/step")
import sys; sys.exit(0)
for f in (steps_only, copies_main, copies_cs, serial, piped):
    print(f.__name__, round(timed(f) * 1000, 1), "us/step")
