"""Cost of one block of the mixed solve's side chain (n=32768, bs=1024), each
piece timed alone with CUDA events: FP64 diagonal factor, inverse TRSM,
conversions, the bf16 panel GEMM."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_07311_b200.control import flatten_cholesky, parse_tree, resolve_config  # noqa: E402
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.mixed import DIAG_TREE  # noqa: E402
from paper_2604_07311_b200.views import DType, from_torch  # noqa: E402

n, bs = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (32768, 1024)
tree = parse_tree(sys.argv[3]) if len(sys.argv) > 3 else parse_tree(json.dumps(DIAG_TREE))
lib = _lib.lib()
levels = flatten_cholesky(tree, resolve_config(tree, DType.F64))
arr = (_lib.BfCholLevel * len(levels))(*[_lib.BfCholLevel(v, 0, b, kc) for v, b, kc in levels])
s = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda")
g.manual_seed(1)
m = torch.rand(bs, bs, dtype=torch.float64, device="cuda", generator=g)
spd = m @ m.T + bs * torch.eye(bs, dtype=torch.float64, device="cuda")
d = spd.clone()
x = torch.empty_like(d)
a21 = torch.rand(n - bs, bs, device="cuda", generator=g)
p = torch.empty(n - bs, bs, dtype=torch.bfloat16, device="cuda")
xt = torch.empty(bs, bs, dtype=torch.bfloat16, device="cuda")
info = torch.full((1,), -1, dtype=torch.int32, device="cuda")
V = lambda t: ctypes.byref(_lib.as_bfview(from_torch(t)))  # noqa: E731


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


def diag():
    d.copy_(spd)
    lib.bf_cholesky_ex_d(V(d), arr, len(levels), 0, info.data_ptr(), s)


def copy_only():
    d.copy_(spd)


def inverse():
    x.zero_()
    x.diagonal().fill_(1.0)
    lib.bf_trsm_rltn_d(1.0, V(torch.tril(spd)), V(x), 512, None, s)


def panel():
    lib.bf_gemm_bf16(1.0, p.data_ptr(), bs, xt.data_ptr(), bs, 0.0, V(a21), bs, 0, s)


def conv():
    lib.bf_convert_f32_bf16(V(a21), p.data_ptr(), bs, 0, s)


out = {"n": n, "bs": bs, "diag_ms": round(timed(diag) - timed(copy_only), 4), "inverse_ms": timed(inverse),
       "panel_gemm_ms": timed(panel), "convert_a21_ms": timed(conv)}
print(json.dumps(out))
