"""Panel pieces of the bench tree, timed alone: the 2048 diagonal factor (inner
tree v3 128 -> unblocked3, no lookahead inside) and the panel TRSM
(m x 2048 against it, kc 2048) at several m."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_07311_b200.control import flatten_cholesky, parse_tree, resolve_config  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.views import DType, from_torch  # noqa: E402

bs = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
lib = _lib.lib()
tree = parse_tree(json.dumps({"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                              "child": {"op": "cholesky", "variant": "unblocked3"}}))
levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, b, kc) for v, b, kc in levels])
g = torch.Generator(device="cuda")
g.manual_seed(1)
m = torch.rand(bs, bs, dtype=torch.float64, device="cuda", generator=g)
a0 = m @ m.T + bs * torch.eye(bs, dtype=torch.float64, device="cuda")
info = torch.full((1,), -1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return round(best, 3)


a = a0.clone()
out = {"bs": bs}
# (leaves `a` factored for the TRSMs)
out["diag_factor_ms"] = t(lambda: (a.copy_(a0), lib.bf_cholesky_ex_d(ctypes.byref(_lib.as_bfview(from_torch(a))), arr,
                                                                     len(levels), 0, info.data_ptr(), s)))
assert int(info.item()) == -1
for mm in [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ('30720', '16384', '8192', '2048'))]:
    b0 = torch.rand(mm, bs, dtype=torch.float64, device="cuda", generator=g)
    b = b0.clone()
    out[f"trsm_{mm}_ms"] = t(lambda: (b.copy_(b0), lib.bf_trsm_rltn_ex_d(1.0, ctypes.byref(_lib.as_bfview(from_torch(a))),
                                                                        ctypes.byref(_lib.as_bfview(from_torch(b))), bs,
                                                                        None, info.data_ptr(), s)))
print(json.dumps(out))
