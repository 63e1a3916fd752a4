"""tcgen05 kind::tf32 GEMM throughput: the raw tf32 GEMM (C -= A B^T, fp32
operands) and the 3xTF32 FP32 GEMM (bf_gemm_f32_tc: split + one K = 3k GEMM)
at a square 8192^3 and the FP32 Cholesky trailing shape (k = 3*1024)."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.views import from_torch  # noqa: E402

lib = _lib.lib()
s = torch.cuda.current_stream().cuda_stream


def timed(call, reps=5):
    assert call() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for m, k, lower in ((8192, 8192, 0), (31744, 3072, 1)):
    a = torch.randn(m, k, device="cuda")
    c = torch.randn(m, m, device="cuda")
    v = _lib.as_bfview(from_torch(c))
    ms = timed(lambda: lib.bf_gemm_tf32(-1.0, a.data_ptr(), k, a.data_ptr(), k, 1.0, ctypes.byref(v), k, lower, s))
    flops = 2.0 * m * m * k * (0.5 if lower else 1.0)
    print(json.dumps({"kernel": "tf32", "m": m, "k": k, "lower": lower, "ms": round(ms, 3),
                      "tflops": round(flops / ms / 1e9, 1)}), flush=True)
m = k = 8192
a = torch.randn(m, k, device="cuda")
c = torch.randn(m, m, device="cuda")
va, vc = _lib.as_bfview(from_torch(a)), _lib.as_bfview(from_torch(c))
ms = timed(lambda: lib.bf_gemm_f32_tc(1.0, ctypes.byref(va), ctypes.byref(va), 0.0, ctypes.byref(vc), 0, s))
print(json.dumps({"kernel": "3xtf32 (split + K=3k tf32 GEMM)", "m": m, "k": k, "ms": round(ms, 3),
                  "fp32_equiv_tflops": round(2.0 * m * m * k / ms / 1e9, 1)}), flush=True)
