import time, torch, numpy as np, os
n = 134217728
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, f in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, "GB/s", n / min(ts) / 1e9, "median", n / sorted(ts)[2] / 1e9)
# host memory bandwidth: numpy copy of 268 MB (pageable)
a = np.ones(n // 4, np.int64); b = np.empty_like(a)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); np.copyto(b, a); ts.append(time.perf_counter() - t0)
print("host memcpy 1thr GB/s (r+w)", 2 * a.nbytes / min(ts) / 1e9)
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
