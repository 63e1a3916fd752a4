"""C5 contraction (abij,cdij->abcd, d=128, FP64) with the C tile in TMEM across
the kc folds (tmem_fold=1) vs folded through L2 (tmem_fold=0): device time and
bit equality.   python tools/c5_tmem.py [d] [reps]"""
import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1"]
spec = ContractionSpec.parse("abij,cdij->abcd")
g = torch.Generator(device="cuda")
g.manual_seed(42)


def rand():
    t = make_tensor([d] * 4)
    t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    return t


a, b, c = rand(), rand(), make_tensor([d] * 4)
lib = _lib.lib()
import os

for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # e.g. BF_OPTS=group=16,persist=1
    k, v = kv.split("=")
    assert lib.bf_set_option(k.encode(), int(v)) == 0, kv
out = {}
for mode in modes:
    lib.bf_set_option(b"tmem_fold", int(mode))
    bf.contract(1.0, a, b, 0.0, c, spec)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bf.contract(1.0, a, b, 0.0, c, spec)
        e1.record()
        e1.synchronize()
        ms.append(round(e0.elapsed_time(e1), 2))
    h = hashlib.sha256(c.storage.cpu().numpy().tobytes()).hexdigest()[:16]
    out[f"tmem_fold={mode}"] = {"ms": ms, "tflops": round(2 * d ** 6 / (min(ms) / 1e3) / 1e12, 2), "sha": h}
print(json.dumps({"opts": os.environ.get("BF_OPTS", ""), **out}))
