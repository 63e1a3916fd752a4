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


@pytest.mark.parametrize("tma_c", [1, 0])
@pytest.mark.parametrize("c_off", [0, 1])
@pytest.mark.parametrize("m", [333, 336])
def test_bf16_gemm_epilogues_on_views(cuda, tma_c, c_off, m):
    """TMA C-tile epilogue and the per-element fallback (forced, or picked for a
    misaligned C view) give the same values, and leave the strict upper
    triangle and the rest of the storage untouched."""
    k = 192  # m=336 with c_off=0 takes the TMA path; 333 has a ragged 16-byte row end
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    a = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    store = torch.rand(m + 2, 340, device="cuda", generator=g)  # 1360-byte rows
    c = store[1:1 + m, c_off:c_off + m]
    before = store.clone()
    lib = _lib.lib()
    assert lib.bf_set_option(b"bf16_tma_c", tma_c) == 0
    try:
        rc = lib.bf_gemm_bf16(-0.5, a.data_ptr(), k, a.data_ptr(), k, 2.0, ctypes.byref(_lib.as_bfview(from_torch(c))), k,
                              1, torch.cuda.current_stream().cuda_stream)
    finally:
        lib.bf_set_option(b"bf16_tma_c", 1)
    assert rc == 0
    c0 = before[1:1 + m, c_off:c_off + m]
    ref = 2.0 * c0 - 0.5 * (a.float() @ a.float().T)
    mask = torch.tril(torch.ones(m, m, dtype=torch.bool, device="cuda"))
    assert (c - ref)[mask].abs().max().item() <= 1e-4
    assert torch.equal(c[~mask], c0[~mask])
    outside = torch.ones_like(store, dtype=torch.bool)
    outside[1:1 + m, c_off:c_off + m] = False
    assert torch.equal(store[outside], before[outside])


def test_bf16_gemm_rejects_unaligned_leading_dim(cuda):
    a = torch.zeros(64, 500, dtype=torch.bfloat16, device="cuda")  # 1000-byte rows: not a TMA stride
    c = torch.zeros(64, 64, device="cuda")
    lib = _lib.lib()
    rc = lib.bf_gemm_bf16(1.0, a.data_ptr(), 500, a.data_ptr(), 500, 0.0, ctypes.byref(_lib.as_bfview(from_torch(c))),
                          500, 0, torch.cuda.current_stream().cuda_stream)
    assert rc != 0 and b"aligned" in lib.bf_last_error()


@pytest.mark.parametrize("symv", [1, 0])
@pytest.mark.parametrize("n", [1000, 258, 4096])
def test_residual_and_row_sums_vs_torch(cuda, n, symv):
    """The refinement's residual r = b - A x and |A| row sums: from the lower
    triangle of the symmetric A (per-tile partials, option "symv") or row by
    row, both against a torch fp64 reference to rounding."""
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m + m.T
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    r = torch.empty_like(b)
    rows = torch.empty_like(b)
    lib = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    try:
        lib.bf_set_option(b"symv", symv)
        _lib.check(lib.bf_residual_d(a.data_ptr(), n, x.data_ptr(), b.data_ptr(), r.data_ptr(), n, st), "residual")
        _lib.check(lib.bf_row_abs_sum_d(a.data_ptr(), n, rows.data_ptr(), n, st), "row sums")
    finally:
        lib.bf_set_option(b"symv", 1)
    ref_r = b - a @ x
    scale = (a.abs() @ x.abs()).max().item()
    assert (r - ref_r).abs().max().item() <= 8 * n * 2.0 ** -53 * scale
    ref_rows = a.abs().sum(1)
    assert (rows - ref_rows).abs().max().item() <= 8 * n * 2.0 ** -53 * ref_rows.max().item()


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
@pytest.mark.parametrize("n,bs,lookahead", [(1000, 256, True), (3000, 1024, True), (2100, 512, False),
                                             (4500, 2048, True)])
def test_mixed_solve_reaches_fp64_accuracy(cuda, n, bs, lookahead, precision):
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    res = posv_mixed(a, b, bs=bs, lookahead=lookahead, precision=precision)
    assert res.converged and res.iterations <= (30 if precision == "bf16" else 8)
    eps = np.finfo(np.float64).eps
    x = res.x.cpu().numpy()
    an, bn = a.cpu().numpy(), b.cpu().numpy()
    back = np.abs(bn - an @ x).max() / (np.abs(an).sum(1).max() * np.abs(x).max() + np.abs(bn).max())
    assert back <= 10 * n * eps
    x_ref = np.linalg.solve(an, bn)
    # forward error <= cond(A) * backward error; cond(M M^T + n I) is ~2-3
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 100 * n * eps


@pytest.mark.parametrize("opts", [{}, {"potrs_vec": 0}, {"potrs_coop": 0}], ids=["vec", "scalar", "launches"])
@pytest.mark.parametrize("n,bs", [(700, 256), (702, 256), (4100, 2048), (2048, 1024)])
def test_blocked_potrs_matches_direct_solve(cuda, n, bs, opts):
    """ragged last blocks; n % 4 != 0 (702) takes the cooperative kernel's
    scalar form even with potrs_vec = 1"""
    from paper_2604_07311_b200.mixed import cholesky_mixed

    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    f = cholesky_mixed(a, bs)
    rhs = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    lib = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    x1, x2 = rhs.clone(), rhs.clone()
    work = torch.empty(129 * bs, dtype=torch.float64, device="cuda")
    assert lib.bf_potrs_f32_d(f.w.data_ptr(), n, x1.data_ptr(), n, s) == 0
    try:
        for k, v in opts.items():
            assert lib.bf_set_option(k.encode(), v) == 0
        assert lib.bf_potrs_blocked_f32_d(f.w.data_ptr(), n, f.xinv.data_ptr(), bs, x2.data_ptr(), n,
                                          work.data_ptr(), s) == 0
    finally:
        for k in opts:
            lib.bf_set_option(k.encode(), 1)
    lw = torch.tril(f.w).double().cpu().numpy()
    ref = np.linalg.solve(lw @ lw.T, rhs.cpu().numpy())
    for x in (x1, x2):  # fp64 arithmetic on the fp32 factor; the blocked one uses fp32 inverses
        assert np.linalg.norm(x.cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-5


@pytest.mark.parametrize("fused", [1, 2])
@pytest.mark.parametrize("n,bs,bad", [(900, 256, 613), (3000, 1024, 1500), (3000, 1024, 5)])
def test_mixed_factor_reports_npd_pivot(cuda, n, bs, bad, fused):
    """fused = 2: the FP64 diagonal blocks as one fused launch each, the inverse
    released per tile column by stream memory waits — also after a failure
    (the later blocks' launches publish their columns and exit)."""
    from paper_2604_07311_b200.errors import NotPositiveDefiniteError
    from paper_2604_07311_b200.mixed import cholesky_mixed

    a = torch.eye(n, dtype=torch.float64, device="cuda") * 4
    a[bad, bad] = -1.0
    lib = _lib.lib()
    try:
        assert lib.bf_set_option(b"fused_diag", fused) == 0
        with pytest.raises(NotPositiveDefiniteError) as e:
            cholesky_mixed(a, bs)
        torch.cuda.synchronize()
    finally:
        lib.bf_set_option(b"fused_diag", 1)
    assert e.value.index == bad


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_mixed_solve_forward_error_vs_fp64_solution(cuda, precision):
    """after refinement ||x - x_ref|| / ||x_ref|| <= 1e-12,
    x_ref from the FP64 factor (the bitwise-reference tree) and triangular
    solves; step_tol is the forward-error stopping criterion."""
    import paper_2604_07311_b200 as bf

    n = 3000
    g = torch.Generator(device="cuda")
    g.manual_seed(99)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    res = posv_mixed(a, b, bs=512, precision=precision, step_tol=1e-11)
    assert res.converged
    l64 = a.clone()
    bf.cholesky(bf.from_torch(l64), "lower")
    lo = torch.tril(l64)
    xref = torch.linalg.solve_triangular(lo.T, torch.linalg.solve_triangular(lo, b[:, None], upper=False),
                                         upper=True)[:, 0]
    assert float((res.x - xref).norm() / xref.norm()) <= 1e-12


@pytest.mark.parametrize("inverse", [0, 1])
@pytest.mark.parametrize("n,bs", [(3000, 1024), (2600, 2048), (1000, 384), (4104, 2048)])
def test_mixed_diagonal_inverses(cuda, n, bs, inverse):
    """xinv[k] = L_kk^-T for every diagonal block, from the trailing right
    solve (mixed_inverse = 0) or the recursive-doubling inverse (1: 128-wide
    tile inverses in one launch, X12 = -X11 B^T X22 per split; ragged last
    tiles): X L_kk^T = I to fp32 storage accuracy, strict lower part zero."""
    from paper_2604_07311_b200.mixed import cholesky_mixed

    g = torch.Generator(device="cuda")
    g.manual_seed(n + bs)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    lib = _lib.lib()
    try:
        assert lib.bf_set_option(b"mixed_inverse", inverse) == 0
        f = cholesky_mixed(a, bs)
        torch.cuda.synchronize()
    finally:
        lib.bf_set_option(b"mixed_inverse", 0)
    for k in range(-(-n // bs)):
        k0, b = k * bs, min(bs, n - k * bs)
        lkk = torch.tril(f.w[k0:k0 + b, k0:k0 + b].double())
        x = f.xinv[k, :b, :b].double()
        err = (x @ lkk.T - torch.eye(b, dtype=torch.float64, device="cuda")).abs().max().item()
        assert err <= 1e-5, (k, err)
        assert not torch.tril(x, -1).any()


@pytest.mark.parametrize("n,bs", [(3000, 1024), (4500, 2048)])
def test_mixed_solve_with_doubling_inverse(cuda, n, bs):
    """mixed_inverse = 1 end to end: FP64 accuracy after refinement."""
    g = torch.Generator(device="cuda")
    g.manual_seed(7 + n)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    lib = _lib.lib()
    try:
        assert lib.bf_set_option(b"mixed_inverse", 1) == 0
        res = posv_mixed(a, b, bs=bs, step_tol=1e-13)
        torch.cuda.synchronize()
    finally:
        lib.bf_set_option(b"mixed_inverse", 0)
    assert res.converged
    x_ref = torch.linalg.solve(a, b)
    assert ((res.x - x_ref).norm() / x_ref.norm()).item() <= 1e-12
