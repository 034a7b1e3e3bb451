"""Host enqueue cost per call of the C-ABI entry points (dev probe): wall time of N enqueues without
synchronising, against the device time of the same N steps."""
import os, sys, time, ctypes
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
nbg = H.lib().hiper_coltrast_grad_workspace_size(B, B, L, d)
gws, gwp, gwn = H._workspace(nbg, "cuda")
gq = torch.empty((B, Lq, d), dtype=torch.float32, device="cuda")
gd = torch.empty((B, L, d), dtype=torch.float32, device="cuda")
fwd = lambda: H.hiper_coltrast_scores_loss(qs, ql, docs, dl, temperature=1.0, workspace=ws, out=out, stream=stream)
def grad():
    H._check(H.lib().hiper_coltrast_scores_loss_grad(
        H._dev_ptr(qs), H._ptr(ql), B, Lq, H._dev_ptr(docs), H._ptr(dl), B, L, d,
        H._dtype_code(qs), 0, None, ctypes.c_float(1.0), ctypes.c_void_p(gwp), gwn,
        H._dev_ptr(out[0]), H._dev_ptr(out[1]), H._dev_ptr(gq), H._dev_ptr(gd), H._stream_ptr(stream)))
for name, fn in (("forward", fwd), ("grad", grad)):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    N = 12
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(stream)
    for _ in range(N): fn()
    e1.record(stream); t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, "host enqueue", round((t1 - t0) / N * 1e6, 1), "us/call; device", round(e0.elapsed_time(e1) / N * 1e3, 1), "us/step")
