"""Pinned host <-> device copy bandwidth (the e2e path's PCIe ceiling)."""
import torch

n = 1 << 27  # 1 GiB of float64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        fn()
    e1.record()
    e1.synchronize()
    print(f"{name}: {4 * 8 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
