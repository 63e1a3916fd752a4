"""Mixed solve n=32768: diagonal-block tree sweep (the FP64 diag chain is the
critical path of the bf16 factorization)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.mixed import MixedWorkspace, cholesky_mixed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
g = torch.Generator(device="cuda").manual_seed(7)
m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
a = m @ m.T
a.diagonal().add_(float(n))
del m
ws = MixedWorkspace(n, bs)


def tree(levels):
    doc = {"op": "cholesky", "variant": "unblocked3"}
    for b in reversed(levels):
        doc = {"op": "cholesky", "variant": 3, "bs": b, "kernel": {"kc": b}, "child": doc}
    return parse_tree(json.dumps(doc))


for lv in ([128], [64], [256, 64], [256, 128], [512, 128], [128, 32], [256, 32]):
    t = tree(lv)
    ms = []
    for _ in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cholesky_mixed(a, bs, diag_tree=t, ws=ws)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(json.dumps({"n": n, "bs": bs, "diag_tree": lv, "factor_ms": [round(x, 2) for x in ms[1:]]}), flush=True)
