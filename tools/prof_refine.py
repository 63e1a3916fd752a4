"""C4 refinement pieces at n=32768 (after one mixed factorization): device ms
of the row sums, one blocked fp32 solve, one FP64 residual, and one whole
refinement iteration as posv_mixed runs it (three host reads)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.mixed import MixedWorkspace, cholesky_mixed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
a0 = bench.make_spd(bf, torch, n, torch.device("cuda"))
a = a0 + a0.T
a.diagonal().sub_(a0.diagonal())
del a0
b = torch.rand(n, dtype=torch.float64, device="cuda")
ws = MixedWorkspace(n, bs)
f = cholesky_mixed(a, bs, ws=ws)
lib = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
x, r, d = ws.x, ws.r, ws.d


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return round(e0.elapsed_time(e1) / reps, 3)


x.zero_()
r.copy_(b)
rows = lambda: lib.bf_row_abs_sum_d(a.data_ptr(), n, ws.rows.data_ptr(), n, st)  # noqa: E731
potrs = lambda: lib.bf_potrs_blocked_f32_d(f.w.data_ptr(), n, f.xinv.data_ptr(), bs, d.data_ptr(), n,  # noqa: E731
                                           ws.work.data_ptr(), st)
resid = lambda: lib.bf_residual_d(a.data_ptr(), n, x.data_ptr(), b.data_ptr(), r.data_ptr(), n, st)  # noqa: E731


def it():
    d.copy_(r)
    potrs()
    x.add_(d)
    resid()
    xmax = float(x.abs().max())
    _ = float(r.abs().max()) / xmax
    _ = float(d.abs().max())


import os  # noqa: E402
for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):
    k_, v_ = kv.split("=")
    lib.bf_set_option(k_.encode(), int(v_))
print({"opts": os.environ.get("BF_OPTS", ""), "n": n, "row_sums_ms": t(rows), "potrs_ms": t(potrs),
       "residual_ms": t(resid), "iteration_ms": t(it)})
