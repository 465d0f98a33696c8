import torch
x = torch.empty(1 << 29, dtype=torch.float32, device="cuda")  # 2 GiB
y = torch.empty_like(x)
for name, fn, nbytes in [("memset(write)", lambda: x.zero_(), x.numel() * 4),
                         ("fill(write)", lambda: x.fill_(1.0), x.numel() * 4),
                         ("copy(r+w)", lambda: y.copy_(x), 2 * x.numel() * 4)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(name, round(nbytes / ms / 1e6, 1), "GB/s")
