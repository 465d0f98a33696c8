import torch, time
n = 818 * (1 << 20) // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    ch = n // ns
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(ns, "streams:", round(n * 4 / (t1 - t0) / 1e9, 1), "GB/s")
