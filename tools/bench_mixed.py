"""Mixed-precision SPD solve benchmark (BASELINE configs[3]): n=32768,
bf16/fp32 factorization + FP64 iterative refinement.

    python tools/bench_mixed.py [n] [bs] [bf16|tf32]

Prints one JSON line: factor / refine ms (CUDA events, inputs resident),
iterations, backward error, and FP64-equivalent GFLOP/s = (n^3/3) / total.
Two matrices: well conditioned (M M^T + n I) and harder (M M^T / n + 1e-2 I).
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_07311_b200.engine import _lib  # noqa: E402
from paper_2604_07311_b200.mixed import MixedWorkspace, cholesky_mixed, posv_mixed  # noqa: E402


def main():
    import os

    for kv in filter(None, os.environ.get("BF_OPTS", "").split(",")):  # e.g. BF_OPTS=mixed_reserve=48
        k, v = kv.split("=")
        assert _lib.lib().bf_set_option(k.encode(), int(v)) == 0, kv
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    bs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    ws = MixedWorkspace(n, bs, precision=prec)
    for name, scale, shift in (("mmt_plus_nI", 1.0, float(n)), ("mmt_over_n_plus_1e-2I", 1.0 / n, 1e-2)):
        a = torch.mm(m, m.T).mul_(scale)
        a.diagonal().add_(shift)
        b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        posv_mixed(a, b, bs=bs, ws=ws)  # warm
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        cholesky_mixed(a, bs, ws=ws)
        e[1].record()
        res = posv_mixed(a, b, bs=bs, ws=ws, step_tol=float(os.environ.get("STEP_TOL", "0")) or None)
        e[2].record()
        e[2].synchronize()
        fac = e[0].elapsed_time(e[1])
        tot = e[1].elapsed_time(e[2])  # factor + refinement inside posv_mixed
        # forward error against the FP64 solution (bitwise-reference FP64 factor + triangular solves)
        import paper_2604_07311_b200 as bfp

        l64 = a.clone()
        bfp.cholesky(bfp.from_torch(l64), "lower", None if n < 2048 else bfp.parse_tree(json.dumps(
            {"op": "cholesky", "variant": 3, "bs": 2048, "kernel": {"kc": 2048},
             "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                       "child": {"op": "cholesky", "variant": "unblocked3"}}})))
        l64 = torch.tril(l64)
        y = torch.linalg.solve_triangular(l64, b[:, None], upper=False)
        xref = torch.linalg.solve_triangular(l64.T, y, upper=True)[:, 0]
        fwd = float((res.x - xref).norm() / xref.norm())
        del l64, y
        print(json.dumps({"fwd_err_vs_fp64": fwd, "opts": os.environ.get("BF_OPTS", ""), "n": n, "bs": bs, "precision": prec, "matrix": name, "factor_ms": round(fac, 2), "posv_ms": round(tot, 2),
                          "refine_ms": round(tot - fac, 2), "iterations": res.iterations,
                          "backward_error": res.backward_error, "converged": res.converged,
                          "fp64_equiv_gflops": round(n ** 3 / 3 / (tot / 1e3) / 1e9, 1),
                          "launches": _lib.lib().bf_launch_count()}), flush=True)
        del a


if __name__ == "__main__":
    main()
