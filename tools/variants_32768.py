"""All three blocked variants and both triangles at n=32768 (BASELINE configs[1]
size), the bench tree shape (bs 2048 kc 2048 -> bs 128 kc 128 -> unblocked3),
plain device ms x3 each."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
a0 = a0 + torch.tril(a0, -1).T  # dense symmetric: the upper factorization reads the upper triangle
work = torch.empty_like(a0)
for variant in (3, 2, 1):
    for uplo in ("lower", "upper"):
        doc = json.loads(json.dumps(bench.GPU_TREE))
        doc["variant"] = variant
        tree = parse_tree(json.dumps(doc))
        ms = []
        for i in range(3):
            work.copy_(a0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bf.cholesky(bf.from_torch(work), uplo, tree)
            e1.record()
            e1.synchronize()
            ms.append(round(e0.elapsed_time(e1), 2))
        print(json.dumps({"n": n, "variant": variant, "uplo": uplo, "ms": ms,
                          "tflops": round(n ** 3 / 3 / (min(ms) / 1e3) / 1e12, 2)}), flush=True)
