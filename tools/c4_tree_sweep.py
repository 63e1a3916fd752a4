"""C4 (mixed solve, n=32768, bs=1024): factor time for several FP64 diagonal-
block trees (the mixed factor's diagonal blocks are not bound to the
reference's bits: refinement makes the solve exact), plus posv time with the
bench's step_tol.   python tools/c4_tree_sweep.py [n] [bs]"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
import os  # noqa: E402

for _kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # library options for sweeps
    _k, _v = _kv.split("=")
    assert _lib.lib().bf_set_option(_k.encode(), int(_v)) == 0, _kv
from paper_2604_07311_b200.mixed import MixedWorkspace, cholesky_mixed, posv_mixed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
U3 = {"op": "cholesky", "variant": "unblocked3"}


def v3(b, child, kc=None):
    return {"op": "cholesky", "variant": 3, "bs": b, "kernel": {"kc": kc or b}, "child": child}


TREES = {
    "v3/128>u3 (default)": v3(128, U3),
    "v3/64>u3": v3(64, U3),
    "v3/256>v3/64>u3": v3(256, v3(64, U3)),
    "v3/256>v3/128>u3": v3(256, v3(128, U3)),
    "v3/512>v3/128>u3": v3(512, v3(128, U3)),
    "v3/32>u3": v3(32, U3),
    "v3/256>v3/32>u3": v3(256, v3(32, U3)),
}
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
a = a0 + a0.T
a.diagonal().sub_(a0.diagonal())
del a0
g = torch.Generator(device="cuda")
g.manual_seed(3)
b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
ws = MixedWorkspace(n, bs)
for name, doc in TREES.items():
    tree = parse_tree(json.dumps(doc))
    cholesky_mixed(a, bs, diag_tree=tree, ws=ws)
    fms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cholesky_mixed(a, bs, diag_tree=tree, ws=ws)
        e1.record()
        e1.synchronize()
        fms.append(e0.elapsed_time(e1))
    print(f"{name:24s} factor ms {statistics.median(fms):8.2f}  {[round(x, 2) for x in fms]}", flush=True)
