"""Pivoted LTL^T timing: n bs [reps] (bs 0 = unblocked)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import ControlNode  # noqa: E402

args = [int(x) for x in sys.argv[1:]]
n, bs = (args + [4096, 128][len(args):])[:2] if len(args) < 2 else args[:2]
reps = args[2] if len(args) > 2 else 1
rng = np.random.default_rng(0)
m = rng.uniform(-1, 1, (n, n))
x0 = np.tril(m - m.T)
tree = ControlNode("ltlt", "unblocked") if bs == 0 else ControlNode("ltlt", "blocked", bs=bs,
                                                                     child=ControlNode("ltlt", "unblocked"))
if len(args) > 3:
    from paper_2604_07311_b200.engine import _lib
    _lib.lib().bf_set_option(b"ltlt_grid", args[3])
v = bf.make_view(n, n, fill=x0)
src = v.storage.clone()
for _ in range(reps):
    v.storage.copy_(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.ltlt_pivoted(v, tree)
    e1.record()
    e1.synchronize()
    print(f"ltlt n={n} bs={bs} grid_cap={args[3] if len(args) > 3 else 0} ms {e0.elapsed_time(e1):.2f}")
