"""The diagonal-block factor alone: bs x bs block (default 2048) with the bench
tree's child (v3 bs 128 kc 128 -> unblocked3), device ms.
python tools/prof_diag.py [bs] [reps]"""
import json
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

bs = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
child = bench.GPU_TREE["child"]
tree = parse_tree(json.dumps(child))
a0 = bench.make_spd(bf, torch, bs, torch.device("cuda"))
work = a0.clone()
ms = []
for _ in range(reps):
    work.copy_(a0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.cholesky(bf.from_torch(work), "lower", tree)
    e1.record()
    e1.synchronize()
    ms.append(round(e0.elapsed_time(e1), 3))
print(f"diag factor bs={bs} tree={json.dumps(child)}: ms {ms}")
if os.environ.get("BF_OPTS", "").find("fused_diag=0") < 0:
    import ctypes

    st = (ctypes.c_int64 * 12)()
    lib = _lib.lib()
    if lib.bf_fused_diag_stats(st) == 0:
        for k, name in enumerate(("leaf", "trsm", "update")):
            cnt = max(st[3 * k], 1)
            print(f"  {name:6s} tasks {st[3 * k]:5d}  wait {st[3 * k + 1] / cnt / 1.9e3:8.2f} us  "
                  f"run {st[3 * k + 2] / cnt / 1.9e3:8.2f} us  (sum run {st[3 * k + 2] / 1.9e6:7.3f} ms)")
        cnt = max(st[6], 1)
        print(f"  update phases per task: stage {st[9] / cnt / 1.9e3:.2f} us, compute {st[10] / cnt / 1.9e3:.2f} us, "
              f"fold {st[11] / cnt / 1.9e3:.2f} us")
