"""Single-rank timing of the distributed driver against the single-GPU
driver on the same tree (1x1 grid: no communication, so the difference is the
schedule), plus the same run with the lookahead off.

    python tools/prof_dist.py [n] [nb]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.dist import BlockCyclic2D, cholesky_distributed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
tree = parse_tree(json.dumps({"op": "cholesky", "variant": 3, "bs": nb, "kernel": {"kc": nb},
                              "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                                        "child": {"op": "cholesky", "variant": "unblocked3"}}}))


class Solo:
    rank, world = 0, 1

    def bcast(self, t, root):
        pass


g = torch.Generator(device="cuda")
g.manual_seed(1)
m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
a0 = m @ m.T
a0.diagonal().add_(float(n))
del m
work = torch.empty_like(a0)
layout = BlockCyclic2D(n, nb, 1, 1)


def timed(fn):
    out = []
    for _ in range(3):
        work.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return round(min(out), 2)


res = {"n": n, "nb": nb,
       "single_gpu_driver_ms": timed(lambda: bf.cholesky(bf.from_torch(work), "lower", tree)),
       "dist_lookahead_ms": timed(lambda: cholesky_distributed(work, layout, tree, Solo(), lookahead=True)),
       "dist_no_lookahead_ms": timed(lambda: cholesky_distributed(work, layout, tree, Solo(), lookahead=False))}
print(json.dumps(res))
