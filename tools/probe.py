"""Quick perf probe: device-generated corpus, timed hiper_maxsim_topk / scores (dev tool)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_04846_b200 as H
from synth import device, gen

C = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
Qs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "64,256,1024").split(",")]
L, Lq, d, k = 256, 32, 128, 10
t = torch.empty((C, L, d), dtype=torch.bfloat16, device="cuda")
device.corpus_(t, 1, 0)
clen = np.full(C, L, np.int32)
torch.cuda.synchronize(); t0 = time.time()
idx = H.hiper_index_build(t, clen, flags=H.HIPER_BORROW_TOKENS)
torch.cuda.synchronize(); print("build s", time.time() - t0, flush=True)
for Q in Qs:
    q = torch.empty((Q, Lq, d), dtype=torch.bfloat16, device="cuda")
    device.queries_(q, 2, corpus_seed=1, n_chunks=C, L=L)
    qlen = np.full(Q, Lq, np.int32)
    ws = H.TopkWorkspace(idx, Q, k)
    out = None
    for _ in range(2):
        out = H.hiper_maxsim_topk(idx, q, qlen, k, workspace=ws, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record()
    for _ in range(n):
        out = H.hiper_maxsim_topk(idx, q, qlen, k, workspace=ws, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flops = 2.0 * Q * C * Lq * L * d
    tgt = gen.query_targets(2, Q, C, False)
    hit = (out[1][:, 0].cpu().numpy() == tgt).mean()
    print(json.dumps({"C": C, "Q": Q, "ms": ms, "tflops": flops / ms / 1e9, "qps": Q / ms * 1e3,
                      "top1_hit": float(hit), "launches": H.last_launch_count()}), flush=True)
