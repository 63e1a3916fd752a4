"""Small invocations of every hand-written kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) on the box:

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases: tma_gemm (TMA/mbarrier DMMA SYRK, red.global fold on and off),
cpasync_gemm (cp.async DMMA kernel, mn-major operands), chol (leaf +
fused TRSM + lookahead streams), bf16 (tcgen05/TMEM GEMM and GEMMT),
tf32 (3xTF32 tcgen05 path), lu (cluster leaf + grid leaf), qr (cooperative
panel), ltlt, contract (scatter gather), dist (NCCL driver on one rank).
Each case checks its own result loosely so a silent corruption also fails.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2604_07311_b200 as bf  # noqa: E402
from golden_inputs import spd_int  # noqa: E402
from paper_2604_07311_b200.control import parse_tree  # noqa: E402
from paper_2604_07311_b200.engine import KernelConfig, _lib  # noqa: E402
from paper_2604_07311_b200.views import DType  # noqa: E402

dev = torch.device("cuda")
F64 = DType.F64


def tma_gemm():
    lib = _lib.lib()
    rng = np.random.default_rng(1)
    n, k = 300, 96
    a = rng.uniform(-1, 1, (n, k))
    for red in (1, 0):
        lib.bf_set_option(b"red_fold", red)
        c = bf.make_view(n, n, fill=np.eye(n), device=dev)
        bf.syrk_lower(-1.0, bf.make_view(n, k, fill=a, device=dev), 1.0, c, cfg=KernelConfig(8, 6, 64, 32, 2048, F64, F64))
        ref = np.tril(np.eye(n) - a @ a.T)
        assert np.abs(np.tril(c.to_numpy()) - ref).max() < 1e-12
    lib.bf_set_option(b"red_fold", 1)


def cpasync_gemm():
    rng = np.random.default_rng(2)
    m, n, k = 150, 130, 70
    a, b = rng.uniform(-1, 1, (m, k)), rng.uniform(-1, 1, (k, n))
    va = bf.make_view(m, k, fill=a, layout="col-major", device=dev)
    vb = bf.make_view(k, n, fill=b, layout="row-major", device=dev)
    c = bf.make_view(m, n, device=dev)
    bf.gemm(1.0, va, vb, 0.0, c)
    assert np.abs(c.to_numpy() - a @ b).max() < 1e-12


def chol():
    n = 700
    a0 = spd_int(5, n)
    v = bf.make_view(n, n, fill=a0, device=dev)
    tree = parse_tree('{"op":"cholesky","variant":3,"bs":256,"kernel":{"kc":256},"child":{"op":"cholesky",'
                      '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}')
    bf.cholesky(v, "lower", tree)
    L = np.tril(v.to_numpy())
    assert np.abs(L @ L.T - a0).max() / np.abs(a0).max() < 1e-13


def bf16():
    from paper_2604_07311_b200 import mixed

    n = 512
    a = spd_int(6, n) / n
    res = mixed.posv_mixed(torch.tensor(a, device=dev), torch.ones(n, dtype=torch.float64, device=dev), bs=256)
    r = a @ res.x.cpu().numpy().reshape(-1) - 1.0
    assert np.abs(r).max() < 1e-10


def tf32():
    from paper_2604_07311_b200 import mixed

    n = 512
    a = torch.tensor(spd_int(7, n), dtype=torch.float32, device=dev)
    l = a.clone()
    mixed.cholesky_f32_tc(l, bs=256)
    L = torch.tril(l).double()
    assert ((L @ L.T - a.double()).abs().max() / a.abs().max()).item() < 1e-5


def lu():
    rng = np.random.default_rng(8)
    for m, n in ((256, 256), (600, 200)):
        a0 = rng.uniform(-1, 1, (m, n))
        v = bf.make_view(m, n, fill=a0, device=dev)
        bf.lu_partial(v, None)


def qr():
    rng = np.random.default_rng(9)
    a0 = rng.uniform(-1, 1, (400, 160))
    v = bf.make_view(400, 160, fill=a0, device=dev)
    bf.qr_householder(v)


def ltlt():
    rng = np.random.default_rng(10)
    x = rng.uniform(-1, 1, (200, 200))
    x = x - x.T
    bf.ltlt_pivoted(bf.make_view(200, 200, fill=x, device=dev))


def contract():
    from paper_2604_07311_b200.tensor import ContractionSpec

    rng = np.random.default_rng(11)
    d = 12
    a0, b0 = rng.uniform(-1, 1, (d,) * 4), rng.uniform(-1, 1, (d,) * 4)
    ta, tb = bf.make_tensor((d,) * 4, fill=a0, device=dev), bf.make_tensor((d,) * 4, fill=b0, device=dev)
    tc = bf.make_tensor((d,) * 4, device=dev)
    bf.contract(1.0, ta, tb, 0.0, tc, ContractionSpec.parse("aibj,cjdi->abcd"))
    ref = np.einsum("aibj,cjdi->abcd", a0, b0)
    assert np.abs(tc.storage.cpu().numpy().reshape((d,) * 4) - ref).max() < 1e-12


def dist():
    from paper_2604_07311_b200.dist import native

    native.selftest_single_rank(n=640, nb=128)


CASES = {f.__name__: f for f in (tma_gemm, cpasync_gemm, chol, bf16, tf32, lu, qr, ltlt, contract, dist)}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        torch.cuda.synchronize()
        print(f"case {name} ok", flush=True)
    print(json.dumps({"cases": names}))
