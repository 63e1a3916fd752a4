"""Profiling driver (run under ncu on a GPU box): one factorization and/or one
standalone trailing SYRK, with an NVTX-free, minimal launch sequence.

    python tools/prof_chol.py chol  N      # one factorization (bench tree)
    python tools/prof_chol.py syrk  NK BS  # one GEMMT: C(NK x NK) -= A(NK x BS) A^T
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402

what = sys.argv[1]
dev = torch.device("cuda")
from paper_2604_07311_b200.engine import _lib  # noqa: E402

for opt in sys.argv[2:]:
    if "=" in opt:
        k, v = opt.split("=")
        _lib.lib().bf_set_option(k.encode(), int(v))
sys.argv = [a for a in sys.argv if "=" not in a]
if what == "chol":
    n = int(sys.argv[2])
    tree = parse_tree(sys.argv[3]) if len(sys.argv) > 3 else parse_tree(json.dumps(bench.GPU_TREE))
    a0 = bench.make_spd(bf, torch, n, dev)
    torch.cuda.synchronize()
    v = bf.from_torch(a0)
    bf.cholesky(v, "lower", tree)
    torch.cuda.synchronize()
else:
    nk, bs = int(sys.argv[2]), int(sys.argv[3])
    a = torch.rand(nk, bs, dtype=torch.float64, device=dev)
    c = torch.rand(nk, nk, dtype=torch.float64, device=dev)
    cfg = bf.KernelConfig(8, 6, 64, bs, 2048, bf.DType.F64, bf.DType.F64)
    for _ in range(2):
        bf.syrk_lower(-1.0, bf.from_torch(a), 1.0, bf.from_torch(c), cfg=cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.syrk_lower(-1.0, bf.from_torch(a), 1.0, bf.from_torch(c), cfg=cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"syrk nk={nk} bs={bs}: {ms:.3f} ms, {nk * (nk + 1) * bs / ms / 1e9:.2f} TF/s")
