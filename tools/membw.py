"""HBM microbenchmarks: copy (R+W), write-only, read-only, for the roofline."""
import torch
def t(fn, n=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
N = 800 * 2**20
a = torch.empty(N // 4, dtype=torch.int32, device="cuda")
b = torch.empty(N // 4, dtype=torch.int32, device="cuda")
ms = t(lambda: b.copy_(a)); print(f"copy 800MiB: {2*N/ms/1e6:.0f} GB/s (r+w)")
ms = t(lambda: a.fill_(7)); print(f"fill 800MiB: {N/ms/1e6:.0f} GB/s (write)")
ms = t(lambda: a.zero_()); print(f"memset 800MiB: {N/ms/1e6:.0f} GB/s (write)")
ms = t(lambda: a.sum()); print(f"sum 800MiB: {N/ms/1e6:.0f} GB/s (read)")
big = torch.empty(2**30, dtype=torch.bfloat16, device="cuda"); big2 = torch.empty_like(big)
ms = t(lambda: big2.copy_(big)); print(f"copy 2GiB bf16: {2*2**31/ms/1e6:.0f} GB/s (r+w)")
