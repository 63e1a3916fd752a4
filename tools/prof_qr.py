"""One blocked QR (for an ncu launch list): m n bs."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import ControlNode  # noqa: E402

m, n, bs = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 4096, 128)))
a0 = np.random.default_rng(0).uniform(-1, 1, (m, n))
v = bf.make_view(m, n, fill=a0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bf.qr_householder(v, ControlNode("qr", "blocked", bs=bs, child=ControlNode("qr", "unblocked")))
e1.record()
e1.synchronize()
print("qr ms", e0.elapsed_time(e1))
