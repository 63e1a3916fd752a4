"""Mixed precision (BASELINE configs[3]): the tcgen05 bf16 GEMM against a
torch fp32 reference of the same bf16-rounded operands, and the bf16/fp32
factorization + FP64 refinement pinned to the FP64 solution (no reference
oracle exists for this mode: SPEC.md:360 makes refinement a non-goal)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from paper_2604_07311_b200.engine import _lib
from paper_2604_07311_b200.mixed import posv_mixed
from paper_2604_07311_b200.views import from_torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k,lower", [(256, 256, 128, False), (300, 200, 504, False), (1000, 1000, 320, True),
                                         (129, 129, 64, True), (2048, 1024, 2048, False)])
def test_bf16_tcgen05_gemm_vs_torch_fp32(cuda, m, n, k, lower):
    g = torch.Generator(device="cuda")
    g.manual_seed(m + n + k)
    a = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    c0 = torch.rand(m, n, device="cuda", generator=g)
    c = c0.clone()
    lib = _lib.lib()
    vc = _lib.as_bfview(from_torch(c))
    rc = lib.bf_gemm_bf16(-1.0, a.data_ptr(), k, b.data_ptr(), k, 1.0, ctypes.byref(vc), k, int(lower),
                          torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    ref = c0 - (a.float() @ b.float().T)
    tol = 1e-6 * k + 1e-6
    if lower:
        mask = torch.tril(torch.ones(m, n, dtype=torch.bool, device="cuda"))
        assert torch.equal(c[~mask], c0[~mask])  # strict upper untouched
        assert (c - ref)[mask].abs().max().item() <= tol
    else:
        assert (c - ref).abs().max().item() <= tol


def test_bf16_gemm_rejects_unaligned_leading_dim(cuda):
    a = torch.zeros(64, 500, dtype=torch.bfloat16, device="cuda")  # 1000-byte rows: not a TMA stride
    c = torch.zeros(64, 64, device="cuda")
    lib = _lib.lib()
    rc = lib.bf_gemm_bf16(1.0, a.data_ptr(), 500, a.data_ptr(), 500, 0.0, ctypes.byref(_lib.as_bfview(from_torch(c))),
                          500, 0, torch.cuda.current_stream().cuda_stream)
    assert rc != 0 and b"aligned" in lib.bf_last_error()


@pytest.mark.parametrize("n,bs", [(1000, 256), (3000, 1024)])
def test_mixed_solve_reaches_fp64_accuracy(cuda, n, bs):
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    res = posv_mixed(a, b, bs=bs)
    assert res.converged and res.iterations <= 30
    eps = np.finfo(np.float64).eps
    x = res.x.cpu().numpy()
    an, bn = a.cpu().numpy(), b.cpu().numpy()
    back = np.abs(bn - an @ x).max() / (np.abs(an).sum(1).max() * np.abs(x).max() + np.abs(bn).max())
    assert back <= 10 * n * eps
    x_ref = np.linalg.solve(an, bn)
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-12
