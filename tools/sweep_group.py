"""C5 contraction (abij,cdij->abcd, d) time vs the TMA GEMM's raster group
height (bf_set_option("group", g)) with and without the strided persistent
grid (bf_set_option("persist", 1)); bits must not change with g.

    python tools/sweep_group.py [d] [g ...]
"""
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
groups = [int(x) for x in sys.argv[2:]] or [8, 4, 16, 32, 64]
spec = ContractionSpec.parse("abij,cdij->abcd")
g = torch.Generator(device="cuda")
g.manual_seed(42)
ts = []
for _ in range(2):
    t = make_tensor([d] * 4)
    t.storage.copy_(torch.rand(t.storage.numel(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    ts.append(t)
c = make_tensor([d] * 4)
out = {}
for persist, grp in [(pp, gg) for pp in (0, 1) for gg in groups]:
    _lib.lib().bf_set_option(b"group", grp)
    _lib.lib().bf_set_option(b"persist", persist)
    bf.contract(1.0, ts[0], ts[1], 0.0, c, spec)
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        bf.contract(1.0, ts[0], ts[1], 0.0, c, spec)
        e1.record()
        e1.synchronize()
        ms.append(round(e0.elapsed_time(e1), 2))
    out[f"persist{persist}_group{grp}"] = {"ms": ms, "tflops": round(2 * d**6 / min(ms) / 1e9, 2),
                "sha": hashlib.sha256(c.storage.cpu().numpy().tobytes()).hexdigest()[:16]}
print(json.dumps(out))
