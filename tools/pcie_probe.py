import torch, time
n = 795_110_784
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hi = torch.empty(33_177_600, dtype=torch.uint8, pin_memory=True)
di = torch.empty(33_177_600, dtype=torch.uint8, device="cuda")
for chunk in (n, 64 << 20, 16 << 20, 4 << 20):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for o in range(0, n, chunk):
            h[o:o + chunk].copy_(d[o:o + chunk], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"D2H chunk {chunk >> 20} MiB: {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms)")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): di.copy_(hi, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print(f"H2D 33 MB: {33_177_600 / dt / 1e9:.1f} GB/s")
