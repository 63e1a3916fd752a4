"""FP32 Cholesky on the tensor cores (3xTF32, mixed.cholesky_f32_tc) at
n=32768 for several block sizes: ms and the relative residual."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.mixed import F32TcWorkspace, cholesky_f32_tc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
sizes = [int(x) for x in sys.argv[2:]] or [1024, 2048]
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
a32 = a0.float()
w32 = torch.empty_like(a32)
for bs in sizes:
    ws32 = F32TcWorkspace(n, bs)
    ms = []
    for i in range(4):
        w32.copy_(a32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cholesky_f32_tc(w32, bs=bs, ws=ws32)
        e1.record()
        e1.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
    xv = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    lf = torch.tril(w32).double()
    ax = a0 @ xv + a0.T @ xv - a0.diagonal() * xv
    rr = float(torch.linalg.vector_norm(ax - lf @ (lf.T @ xv)) / torch.linalg.vector_norm(ax))
    print(f"bs={bs}: {statistics.median(ms):.2f} ms, residual {rr:.2e}", flush=True)
    del ws32, lf, ax
