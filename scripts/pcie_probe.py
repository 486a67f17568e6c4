"""Pinned host<->device copy bandwidth on this box (C2's e2e bytes)."""
import torch

dev = torch.device("cuda", 0)
for mb in (3.1, 18.9, 28.3):
    n = int(mb * 1e6 / 8)
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    for direction in ("H2D", "D2H"):
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if direction == "H2D":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[5]
        print(f"{direction} {mb:5.1f} MB: {ms:.3f} ms = {mb / ms:.1f} GB/s", flush=True)
