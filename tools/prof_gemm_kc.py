"""FP64 GEMM C -= A B^T (M=N=K=n, NT, all k-contiguous: the TMA kernel) at
several kc: the cost of the reference's kc-segment folds."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.engine.config import default_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda")
g.manual_seed(0)
a = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g)
b = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g)
c = torch.zeros(n, n, dtype=torch.float64, device="cuda")
va, vb, vc = bf.from_torch(a), bf.from_torch(b).transposed(), bf.from_torch(c)
for kc in (256, 512, 1024, 4096, n):
    cfg = default_config().with_overrides({"kc": kc})
    bf.gemm(-1.0, va, vb, 1.0, vc, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.gemm(-1.0, va, vb, 1.0, vc, cfg)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"n": n, "kc": kc, "ms": round(ms, 2), "tflops": round(2 * n ** 3 / ms / 1e9, 2)}), flush=True)
