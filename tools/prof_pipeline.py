"""FP64 Cholesky n=32768 bench tree, first-step pipelining on/off (CUDA events)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
tree = parse_tree(json.dumps(bench.GPU_TREE))
a0 = bench.make_spd(bf, torch, n, torch.device("cuda:0"))
a = torch.empty_like(a0)
lib = _lib.lib()
out = {}
for pipe in (0, 2, 3, 4, 6, 8, 15, 0):
    lib.bf_set_option(b"pipeline_first", pipe)
    ms = []
    for _ in range(3):
        a.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bf.cholesky_async(bf.from_torch(a), "lower", tree)
        e1.record()
        e1.synchronize()
        ms.append(round(e0.elapsed_time(e1), 2))
    out.setdefault(f"pipeline_{pipe}", []).extend(ms)
lib.bf_set_option(b"pipeline_first", 0)
print(json.dumps(out))
