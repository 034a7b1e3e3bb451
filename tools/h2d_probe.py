import torch, time
torch.cuda.init()
n = 16 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
s0 = torch.cuda.current_stream(); cs = torch.cuda.Stream()
def timeit(fn, reps=50):
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(s0); fn(reps); e1.record(s0); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps
def serial(r):
    for i in range(r): d[i&1].copy_(h, non_blocking=True)
def side(r):
    cs.wait_stream(s0)
    with torch.cuda.stream(cs):
        for i in range(r): d[i&1].copy_(h, non_blocking=True)
    s0.wait_stream(cs)
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
def side_with_gemm(r):
    cs.wait_stream(s0)
    with torch.cuda.stream(cs):
        for i in range(r): d[i&1].copy_(h, non_blocking=True)
    for i in range(r): a @ a
    s0.wait_stream(cs)
for f in (serial, side, side_with_gemm):
    ms = timeit(f)
    print(f.__name__, round(ms*1000,1), "us/copy", round(n/ms/1e6,1), "GB/s")
h2 = torch.empty(n, dtype=torch.uint8)  # pageable
print("pinned", h.is_pinned())
