"""Pinned host -> device copy ceiling on this box (the bound of bench.py's e2e)."""
import torch

for mib in (64, 256, 1024):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"H2D {mib} MiB: {10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
    e0.record()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"D2H {mib} MiB: {10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
