"""A/B of the TMA GEMM's fold: load/add/store (red_fold=0) vs L2 reductions
(red_fold=1) on the C5 contraction (d=128, 64 folds per tile) and the C2
Cholesky (bench tree).  Prints times and whether both modes give identical bits.

    python tools/ab_redfold.py [d] [n]
"""
import hashlib
import os
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.tensor import ContractionSpec, contract, make_tensor  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
dev = torch.device("cuda")
modes = [int(x) for x in os.environ.get("MODES", "0,1").split(",")] * 2


def sha(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts


out = {}
spec = ContractionSpec.parse("abij,cdij->abcd")
g = torch.Generator(device="cuda")
g.manual_seed(42)


def rand():
    t = make_tensor([d] * 4)
    t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device=dev, generator=g) * 2 - 1)
    return t


ta, tb, tc = rand(), rand(), make_tensor([d] * 4)
for mode in modes:
    _lib.lib().bf_set_option(b"red_fold", mode)
    contract(1.0, ta, tb, 0.0, tc, spec)
    ts = timed(lambda: contract(1.0, ta, tb, 0.0, tc, spec))
    out.setdefault(f"c5_d{d}_red{mode}", []).append({"ms": [round(t, 2) for t in ts], "gflops": round(2 * d**6 / (min(ts) * 1e6), 1), "sha": sha(tc.storage)})
del ta, tb, tc
torch.cuda.empty_cache()

tree = parse_tree(json.dumps(bench.GPU_TREE))
a0 = bench.make_spd(bf, torch, n, dev)
a = torch.empty_like(a0)
for mode in modes:
    _lib.lib().bf_set_option(b"red_fold", mode)
    ts = []
    for _ in range(3):
        a.copy_(a0)
        v = bf.from_torch(a)
        ts += timed(lambda: bf.cholesky(v, "lower", tree), reps=1)
    out.setdefault(f"chol_n{n}_red{mode}", []).append({"ms": [round(t, 2) for t in ts], "sha": sha(a.tril())})
print(json.dumps(out))
