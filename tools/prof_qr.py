"""Blocked QR timing (and one call for an ncu launch list): m n bs [reps]."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import ControlNode  # noqa: E402

args = [int(x) for x in sys.argv[1:]]
m, n, bs = args[:3] if len(args) >= 3 else (8192, 4096, 128)
reps = args[3] if len(args) > 3 else 1
a0 = np.random.default_rng(0).uniform(-1, 1, (m, n))
tree = ControlNode("qr", "blocked", bs=bs, child=ControlNode("qr", "unblocked"))
v = bf.make_view(m, n, fill=a0)
src = v.storage.clone()
for r in range(reps):
    v.storage.copy_(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.qr_householder(v, tree)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"qr {m}x{n} bs{bs} ms {ms:.2f}  {(2 * m * n * n - 2 * n ** 3 / 3) / ms / 1e9:.2f} TF/s")
