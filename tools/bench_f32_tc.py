"""FP32 Cholesky n (default 32768): 3xTF32 tensor-core factorization
(mixed.cholesky_f32_tc) against the bitwise-reference FP32 engine path
(bf.cholesky on an f32 view: f32 storage, reference semantics), CUDA events.

    python tools/bench_f32_tc.py [n] [bs]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_07311_b200 as bf  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.mixed import F32TcWorkspace, cholesky_f32_tc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(42)
m = torch.rand(n, n, dtype=torch.float32, device=dev, generator=g) * 2 - 1
a0 = torch.zeros(n, n, dtype=torch.float32, device=dev)
bf.syrk_lower(1.0, bf.from_torch(m), 0.0, bf.from_torch(a0))
del m
a0.diagonal().add_(float(n))
a = torch.empty_like(a0)
ws = F32TcWorkspace(n, bs, dev)


def timed(fn):
    a.copy_(a0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1)


out = {"n": n, "bs": bs}
tc = [timed(lambda: cholesky_f32_tc(a, bs=bs, ws=ws)) for _ in range(3)]
out["tc_ms"] = [round(t, 2) for t in tc]
out["tc_tflops"] = round(n ** 3 / 3 / min(tc) / 1e9, 2)
# backward check on a random vector: A x vs L (L^T x), A symmetric from its lower triangle
x = torch.rand(n, device=dev, dtype=torch.float64) * 2 - 1
low = torch.tril(a0).double()
ax = low @ x + torch.tril(a0, -1).double().T @ x
lf = torch.tril(a).double()
out["tc_rel_residual"] = float(torch.linalg.vector_norm(ax - lf @ (lf.T @ x)) / torch.linalg.vector_norm(ax))
del low, lf
tree = parse_tree(json.dumps({"op": "cholesky", "variant": 3, "bs": 2048, "kernel": {"kc": 2048},
                              "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                                        "child": {"op": "cholesky", "variant": "unblocked3"}}}))
ref = [timed(lambda: bf.cholesky_async(bf.from_torch(a), "lower", tree)) for _ in range(2)]
out["engine_f32_ms"] = [round(t, 2) for t in ref]
out["engine_f32_tflops"] = round(n ** 3 / 3 / min(ref) / 1e9, 2)
print(json.dumps(out))
