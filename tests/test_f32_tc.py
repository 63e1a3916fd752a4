"""FP32 on the tensor cores (3xTF32 tcgen05 GEMM and the FP32 Cholesky built
on it).  No reference counterpart bit for bit (the reference's f32 GEMM
accumulates in f32/f64 scalar FMAs, engine/gemm.py:179-201), so the bar is
the reference's own FP32 tolerance: backward error <= 10*n*eps32
(tests/test_cholesky.py:78-86 of the reference) and GEMM error at the fp32
level."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

EPS32 = float(np.finfo(np.float32).eps)


def _gemm_f32_tc(alpha, a, b, beta, c, lower=0):
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    _lib.check(lib.bf_gemm_f32_tc(alpha, ctypes.byref(_lib.as_bfview(a)), ctypes.byref(_lib.as_bfview(b)), beta,
                                  ctypes.byref(_lib.as_bfview(c)), lower, _lib.stream_ptr(a.device)), "f32 tc gemm")


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k,beta,lower", [(256, 256, 1024, 0.0, 0), (300, 200, 77, 1.0, 0), (1000, 1000, 512, -0.5, 1),
                                              (129, 4, 3, 0.0, 0), (512, 384, 4096, 1.0, 0)])
def test_cuda_gemm_f32_tc_fp32_accuracy(cuda, m, n, k, beta, lower):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.views import DType

    rng = np.random.default_rng(m + 7 * n + k)
    a0, b0, c0 = (rng.uniform(-1, 1, s).astype(np.float32) for s in ((m, k), (k, n), (m, n)))
    va, vb, vc = (bf.make_view(*x.shape, DType.F32, fill=x) for x in (a0, b0, c0))
    _gemm_f32_tc(-1.25, va, vb, beta, vc, lower)
    got = vc.to_numpy().astype(np.float64)
    ref = -1.25 * (a0.astype(np.float64) @ b0.astype(np.float64)) + beta * c0.astype(np.float64)
    scale = 1.25 * (np.abs(a0).astype(np.float64) @ np.abs(b0).astype(np.float64)) + abs(beta) * np.abs(c0)
    if lower:
        il = np.tril_indices(m)
        iu = np.triu_indices(m, 1)
        assert np.array_equal(got[iu], c0.astype(np.float64)[iu])  # strict upper untouched
        got, ref, scale = got[il], ref[il], scale[il]
    # 3xTF32: ~2^-21 per product, then fp32 accumulation over K = 3k terms
    # (the error of any fp32 GEMM); a single tf32 pass would be ~2^-11
    assert np.max(np.abs(got - ref) / (scale + 1e-30)) <= 4 * (3 * k) ** 0.5 * EPS32


@pytest.mark.gpu
def test_cuda_gemm_tf32_single_pass_is_tf32(cuda):
    """The raw kind::tf32 GEMM on unsplit fp32 operands: tf32-level error
    (catches a wrong instruction descriptor, which would give garbage)."""
    import torch

    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import _lib
    from paper_2604_07311_b200.views import from_torch

    m, n, k = 256, 128, 512
    g = torch.Generator().manual_seed(1)
    a = (torch.rand(m, k, generator=g) * 2 - 1).cuda()
    b = (torch.rand(n, k, generator=g) * 2 - 1).cuda()
    c = torch.zeros(m, n, device="cuda")
    lib = _lib.lib()
    _lib.check(lib.bf_gemm_tf32(1.0, a.data_ptr(), k, b.data_ptr(), k, 0.0, ctypes.byref(_lib.as_bfview(from_torch(c))),
                                k, 0, _lib.stream_ptr(a.device)), "tf32")
    ref = a.double() @ b.double().T
    err = float(((c.double() - ref).abs() / (a.abs().double() @ b.abs().double().T)).max())
    assert 1e-6 < err < 2e-3
    assert bf is not None


@pytest.mark.gpu
@pytest.mark.parametrize("n,bs,lookahead", [(3000, 1024, True), (2048, 512, False), (700, 1024, True),
                                            (4100, 1024, True)])
def test_cuda_cholesky_f32_tc_backward_error(cuda, n, bs, lookahead):
    import torch

    from paper_2604_07311_b200.mixed import cholesky_f32_tc

    g = torch.Generator(device="cuda").manual_seed(n)
    m = torch.rand(n, n, device="cuda", generator=g, dtype=torch.float64) * 2 - 1
    a64 = m @ m.T + n * torch.eye(n, device="cuda", dtype=torch.float64)
    a = a64.float()
    canary = torch.triu(a, 1).clone()
    cholesky_f32_tc(a, bs=bs, lookahead=lookahead)
    assert torch.equal(torch.triu(a, 1), canary)
    l = torch.tril(a).double()
    be = float(torch.linalg.matrix_norm(a64 - l @ l.T) / torch.linalg.matrix_norm(a64))
    assert be <= 10 * n * EPS32
    assert be <= 4 * n ** 0.5 * EPS32  # in practice fp32 rounding growth, far inside the bound


@pytest.mark.gpu
def test_cuda_cholesky_f32_tc_not_pd_global_index(cuda):
    import torch

    from paper_2604_07311_b200.errors import NotPositiveDefiniteError
    from paper_2604_07311_b200.mixed import cholesky_f32_tc

    n = 1500
    a = torch.eye(n, device="cuda") * 4.0
    a[1100, 1100] = -1.0
    with pytest.raises(NotPositiveDefiniteError) as ei:
        cholesky_f32_tc(a, bs=512)
    assert ei.value.index == 1100
