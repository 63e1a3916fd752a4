"""Phase breakdown of the mixed factorization (synchronous event timing per
call; adds launch gaps, so use only for shares): diag factor, inverse,
conversions, panel GEMM, trailing GEMMT, and one blocked solve + residual."""
import ctypes
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200.mixed as M  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
lib = _lib.lib()
acc = defaultdict(float)
cnt = defaultdict(int)
names = {"bf_cholesky_d": "diag", "bf_trsm_rltn_d": "inverse", "bf_convert_f32_bf16": "convert",
         "bf_convert_f32_f64": "convert", "bf_convert_f64_bf16": "convert",
         "bf_convert_f64_f32": "convert64", "bf_gemm_bf16": "gemm", "bf_potrs_blocked_f32_d": "potrs",
         "bf_residual_d": "residual"}


class Timed:
    def __init__(self, inner):
        self._inner = inner

    def __getattr__(self, name):
        fn = getattr(self._inner, name)
        if name not in names:
            return fn

        def wrap(*args):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn(*args)
            e1.record()
            e1.synchronize()
            key = names[name]
            if name == "bf_gemm_bf16":
                key = "gemm_lower" if args[8] else "gemm_panel"
            acc[key] += e0.elapsed_time(e1)
            cnt[key] += 1
            return rc
        return wrap


M._lib = type("L", (), {"lib": staticmethod(lambda: Timed(lib)), "check": staticmethod(_lib.check),
                        "as_bfview": staticmethod(_lib.as_bfview), "BfCholLevel": _lib.BfCholLevel})
g = torch.Generator(device="cuda")
g.manual_seed(7)
m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
a = torch.mm(m, m.T)
a.diagonal().add_(float(n))
del m
b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
M.posv_mixed(a, b, bs=bs, lookahead=False)
acc.clear()
cnt.clear()
res = M.posv_mixed(a, b, bs=bs, lookahead=False)  # one stream: per-call events are meaningful
print(json.dumps({"n": n, "bs": bs, "iterations": res.iterations,
                  "ms": {k: round(v, 2) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])},
                  "calls": dict(cnt)}))
