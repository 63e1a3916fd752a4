"""C4 mixed solve at n=32768 for several block sizes: factor ms, whole solve
ms (posv, its own factorization included, step_tol 1e-11 as in bench.py),
iterations, forward error against a torch FP64 solve."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.mixed import MixedWorkspace, cholesky_mixed, posv_mixed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
sizes = [int(x) for x in sys.argv[2:]] or [1024, 2048]
import os  # noqa: E402
step_tols = [float(x) for x in os.environ.get("STEP_TOLS", "1e-11").split(",")]
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
a = a0 + a0.T
a.diagonal().sub_(a0.diagonal())
g = torch.Generator(device="cuda")
g.manual_seed(3)
b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
lo = torch.tril(a0)
del a0
y = torch.linalg.solve_triangular(torch.linalg.cholesky(a), b[:, None], upper=False)
xref = torch.linalg.solve_triangular(torch.linalg.cholesky(a).T, y, upper=True)[:, 0]
del y, lo
for bs, step_tol in [(b_, t_) for b_ in sizes for t_ in step_tols]:
    ws = MixedWorkspace(n, bs)
    posv_mixed(a, b, bs=bs, ws=ws, step_tol=step_tol)
    fms, ms = [], []
    for _ in range(3):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        cholesky_mixed(a, bs, ws=ws)
        e1.record()
        res = posv_mixed(a, b, bs=bs, ws=ws, step_tol=step_tol)
        e2.record()
        e2.synchronize()
        fms.append(e0.elapsed_time(e1))
        ms.append(e1.elapsed_time(e2))
    fwd = float((res.x - xref).norm() / xref.norm())
    print(f"bs={bs} step_tol={step_tol:g}: factor {statistics.median(fms):.2f} ms, solve {statistics.median(ms):.2f} ms, "
          f"iterations {res.iterations}, backward {res.backward_error:.2e}, forward {fwd:.2e}", flush=True)
    del ws
