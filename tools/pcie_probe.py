"""Probe (not product): pinned host -> device copy bandwidth, the roof of bench.py's e2e numbers."""
import torch
dev = torch.device("cuda:0")
for mb in (32, 256, 1024, 4096):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"H2D pinned {mb:5d} MB: {n / best / 1e6:7.1f} GB/s")
