"""BASELINE configs[2] size on ONE B200: FP64 Cholesky n=131072 (137 GB in
HBM), factored in place with the bench tree; backward check A x = L L^T x on a
random x with A regenerated block-row by block-row.

A: lower triangle U(-1,1) (seeded per 2048-row block), diagonal + n, so A is
SPD by diagonal dominance (forming M M^T would need a second 137 GB).

    python tools/bench_c3_single.py [n] [bs_root]
"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
RB = 2048
dev = torch.device("cuda:0")
import os  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # e.g. BF_OPTS=tail_reserve=0
    k, v = kv.split("=")
    assert _lib.lib().bf_set_option(k.encode(), int(v)) == 0, kv
tree_doc = {"op": "cholesky", "variant": 3, "bs": bs, "kernel": {"kc": bs},
            "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                      "child": {"op": "cholesky", "variant": "unblocked3"}}}
tree = parse_tree(json.dumps(tree_doc))


def block(r0):
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + r0)
    r1 = min(n, r0 + RB)
    blk = torch.rand(r1 - r0, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
    idx = torch.arange(r0, r1, device=dev)
    blk[idx - r0, idx] += float(n)
    return blk


t0 = time.time()
a = torch.empty(n, n, dtype=torch.float64, device=dev)
for r0 in range(0, n, RB):
    a[r0:r0 + RB] = block(r0)
torch.cuda.synchronize()
gen_s = time.time() - t0
v = bf.from_torch(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
info = bf.cholesky_async(v, "lower", tree)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1)
bad = int(info.item()) if hasattr(info, "item") else info
# backward check: y = A x (A symmetric from its lower triangle), z = L (L^T x)
g = torch.Generator(device=dev)
g.manual_seed(7)
x = torch.rand(n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
y = torch.zeros(n, dtype=torch.float64, device=dev)
w = torch.zeros(n, dtype=torch.float64, device=dev)
for r0 in range(0, n, RB):
    r1 = min(n, r0 + RB)
    blk = block(r0)[:, :r1]
    low = torch.tril(blk, diagonal=r0)
    y[r0:r1] += low @ x[:r1]
    y[:r1] += torch.tril(blk, diagonal=r0 - 1).T @ x[r0:r1]
    lf = torch.tril(a[r0:r1, :r1], diagonal=r0)
    w[:r1] += lf.T @ x[r0:r1]
z = torch.zeros(n, dtype=torch.float64, device=dev)
for r0 in range(0, n, RB):
    r1 = min(n, r0 + RB)
    z[r0:r1] = torch.tril(a[r0:r1, :r1], diagonal=r0) @ w[:r1]
rel = float(torch.linalg.vector_norm(y - z) / torch.linalg.vector_norm(y))
print(json.dumps({"n": n, "tree": tree_doc, "ms": round(ms, 1), "tflops": round(n ** 3 / 3 / ms / 1e9, 2),
                  "pct_fp64_peak": round(100 * n ** 3 / 3 / ms / 1e9 / 37.1, 1), "info": bad,
                  "rel_residual_Ax_vs_LLtx": rel, "gen_s": round(gen_s, 1),
                  "hbm_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)}))
