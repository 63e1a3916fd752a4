"""The first panel's TRSM alone: X * L^T = B, B 30720 x 2048, L 2048 lower,
kc 2048 (the bench tree's root), device ms; run under an ncu launch list to
split subtree kernels from folds.   python tools/prof_trsm.py [m] [n] [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30720
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = torch.Generator(device="cuda")
g.manual_seed(0)
lt = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g)
lt = torch.tril(lt) + n * torch.eye(n, dtype=torch.float64, device="cuda")
b0 = torch.rand(m, n, dtype=torch.float64, device="cuda", generator=g)
b = b0.clone()
cfg = bf.KernelConfig(8, 6, 64, n, 2048, bf.DType.F64, bf.DType.F64)
ms = []
for _ in range(reps):
    b.copy_(b0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf.trsm(bf.engine.RIGHT_LOWER_TRANS_NONUNIT, 1.0, bf.from_torch(lt), bf.from_torch(b), cfg=cfg)
    e1.record()
    e1.synchronize()
    ms.append(round(e0.elapsed_time(e1), 3))
print(f"trsm m={m} n={n}: ms {ms}, {m * n * n / (min(ms) / 1e3) / 1e12:.2f} TF/s")
