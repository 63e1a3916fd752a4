"""One LU factorization (for an ncu launch list): n and tree levels from argv."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
levels = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "512,64,16").split(",")]
kc = int(sys.argv[3]) if len(sys.argv) > 3 else 0
doc = {"op": "lu", "variant": "unblocked"}
for bs in reversed(levels):
    doc = {"op": "lu", "variant": "blocked", "bs": bs, "child": doc}
if kc:
    doc["kernel"] = {"kc": kc}
rng = np.random.default_rng(42)
a0 = rng.uniform(-1, 1, (n, n)) + n * np.eye(n)
for rep in range(2):
    v = bf.make_view(n, n, fill=a0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.lu_partial(v, parse_tree(json.dumps(doc)))
    e1.record()
    e1.synchronize()
    print(json.dumps({"n": n, "tree": levels, "kc": kc or None, "ms": round(e0.elapsed_time(e1), 2),
                      "tflops": round(2 * n ** 3 / 3 / e0.elapsed_time(e1) / 1e9, 2)}))
