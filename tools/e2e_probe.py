import time, torch, json, sys, os
sys.path.insert(0, os.getcwd())
m, n = 131072, 1024
h = torch.empty((n, m), dtype=torch.float64).pin_memory()
h.normal_()
d = torch.empty((n, m), dtype=torch.float64, device="cuda")
hq = torch.empty((n, m), dtype=torch.float64).pin_memory()
s = torch.cuda.current_stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(h, non_blocking=True); e1.record(); e1.synchronize()
h2d = e0.elapsed_time(e1)
e0.record(); hq.copy_(d, non_blocking=True); e1.record(); e1.synchronize()
d2h = e0.elapsed_time(e1)
# both directions at once on two streams
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s2):
    hq.copy_(d, non_blocking=True)
d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
both = (time.perf_counter() - t0) * 1e3
gb = m * n * 8 / 1e9
print(json.dumps({"h2d_ms": h2d, "h2d_GBs": gb / h2d * 1e3, "d2h_ms": d2h, "d2h_GBs": gb / d2h * 1e3, "both_directions_ms": both}))
# D2H split over k concurrent streams
for k in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cols = n // k
    for i, st in enumerate(ss):
        with torch.cuda.stream(st):
            hq[i * cols:(i + 1) * cols].copy_(d[i * cols:(i + 1) * cols], non_blocking=True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"d2h_streams": k, "ms": ms, "GBs": gb / ms * 1e3}))
# 64-column blocks on one copy stream (the library's pattern)
torch.cuda.synchronize()
t0 = time.perf_counter()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for c0 in range(0, n, 64):
        hq[c0:c0 + 64].copy_(d[c0:c0 + 64], non_blocking=True)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) * 1e3
print(json.dumps({"d2h_64col_blocks_ms": ms, "GBs": gb / ms * 1e3}))
