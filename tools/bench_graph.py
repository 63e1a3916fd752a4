"""Direct native driver vs CUDA-graph replay (CholeskyGraph), FP64 Cholesky,
several orders with the bench-shaped tree scaled down (bs = n/8, inner 128):
median ms over reps, CUDA events, input restored outside the events."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402

for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "1024,2048,4096,8192".split(","))]:
    bs = max(128, n // 8)
    tree = parse_tree(json.dumps({"op": "cholesky", "variant": 3, "bs": bs, "kernel": {"kc": bs},
                                  "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                                            "child": {"op": "cholesky", "variant": "unblocked3"}}}))
    m = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
    a0 = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    a = a0.clone()
    v = bf.from_torch(a)
    g = bf.CholeskyGraph(v, "lower", tree)
    out = {"n": n, "bs": bs}
    for name, fn in (("direct", lambda: bf.cholesky_async(v, "lower", tree)), ("graph", g.run)):
        ts = []
        for _ in range(7):
            a.copy_(a0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = round(statistics.median(ts[2:]), 3)
    out["speedup"] = round(out["direct_ms"] / out["graph_ms"], 2)
    print(json.dumps(out), flush=True)
