"""tcgen05 bf16 GEMM throughput: C(fp32) -= A B^T, full and lower (GEMMT),
at the mixed Cholesky's trailing-update shapes (k = bs) and a square 8192^3."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.views import from_torch  # noqa: E402

lib = _lib.lib()
import os  # noqa: E402
for _kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):
    _k, _v = _kv.split("=")
    assert lib.bf_set_option(_k.encode(), int(_v)) == 0, _kv
for m, k, lower in ((8192, 8192, 0), (31744, 1024, 1), (30720, 2048, 1), (16384, 1024, 1), (31744, 1024, 0)):
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    c = torch.randn(m, m, device="cuda")
    v = _lib.as_bfview(from_torch(c))
    s = torch.cuda.current_stream().cuda_stream
    call = lambda: lib.bf_gemm_bf16(-1.0, a.data_ptr(), k, a.data_ptr(), k, 1.0, ctypes.byref(v), k, lower, s)  # noqa
    assert call() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * m * m * k * (0.5 if lower else 1.0)
    ref = torch.matmul(a, a.T)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        torch.matmul(a, a.T, out=ref)
    e1.record()
    e1.synchronize()
    ms_ref = e0.elapsed_time(e1) / reps
    print(json.dumps({"m": m, "k": k, "lower": lower, "ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1),
                      "cublas_full_bf16out_ms": round(ms_ref, 3)}), flush=True)
    del a, c, ref
