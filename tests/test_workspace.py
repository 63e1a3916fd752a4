"""Device scratch accounting (reference engine/workspace.py:18-56 and its
bound test tests/test_engine_sandwich.py:63-72)."""
from __future__ import annotations

import numpy as np
import pytest
import torch


def test_pool_live_peak_and_reuse_cpu():
    from paper_2604_07311_b200.engine.workspace import Workspace

    ws = Workspace()
    a = ws.checkout(100, torch.float64, "cpu", stream=7)
    b = ws.checkout(50, torch.float64, "cpu", stream=7)
    assert ws.live_elements == 150 and ws.peak_elements == 150
    ws.checkin(a)
    assert ws.live_elements == 50
    c = ws.checkout(100, torch.float64, "cpu", stream=7)
    assert c.data_ptr() == a.data_ptr()  # recycled on the same stream
    d = ws.checkout(100, torch.float64, "cpu", stream=8)
    assert d.data_ptr() != a.data_ptr()  # never across streams
    ws.checkin(b), ws.checkin(c), ws.checkin(d)
    assert ws.live_elements == 0 and ws.peak_elements == 250
    ws.reset_peak()
    assert ws.peak_elements == 0


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_sandwich_needs_no_scratch(cuda, dt):
    """The fused skew sandwich forms T*A^T while staging B: neither the host
    pool nor the library allocates a k x n intermediate (f64 and f32)."""
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine.gemm import sandwich_skew
    from paper_2604_07311_b200.engine.workspace import workspace
    from paper_2604_07311_b200.views import DType

    rng = np.random.default_rng(9)
    n, k = 300, 260
    D = DType.parse(dt)
    c = bf.make_view(n, n, D, fill=rng.uniform(-1, 1, (n, n)))
    a = bf.make_view(n, k, D, fill=rng.uniform(-1, 1, (n, k)))
    workspace.reset_peak()
    live0, _ = workspace.device_bytes()
    before = torch.cuda.memory_allocated()
    sandwich_skew(c, a, rng.uniform(-1, 1, k - 1))
    torch.cuda.synchronize()
    assert workspace.peak_elements == 0 and workspace.live_elements == 0
    assert workspace.device_bytes()[1] == live0  # no library scratch either
    assert torch.cuda.memory_allocated() - before < n * k * 4  # only the (k-1)-vector t went to the device


@pytest.mark.gpu
def test_contraction_scratch_accounting(cuda):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine.workspace import workspace
    from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor

    d = 32
    rng = np.random.default_rng(1)
    for spec, staged in (("aibj,cidj->abcd", 0), ("aibj,cjdi->abcd", d ** 4)):
        ta = make_tensor((d,) * 4, fill=rng.uniform(-1, 1, (d,) * 4))
        tb = make_tensor((d,) * 4, fill=rng.uniform(-1, 1, (d,) * 4))
        tc = make_tensor((d,) * 4)
        workspace.reset_peak()
        bf.contract(1.0, ta, tb, 0.0, tc, ContractionSpec.parse(spec), stage="always")
        torch.cuda.synchronize()
        assert workspace.peak_elements == staged, spec  # mode-group TMA: no copy; k-transposed B: one k x n copy
        assert workspace.live_elements == 0


@pytest.mark.gpu
def test_upper_copy_is_accounted(cuda):
    import paper_2604_07311_b200 as bf
    from golden_inputs import spd_int
    from paper_2604_07311_b200.engine.workspace import workspace

    n = 1536
    workspace.release()
    workspace.reset_peak()
    v = bf.make_view(n, n, fill=spd_int(3, n))
    bf.cholesky(v, "upper")
    torch.cuda.synchronize()
    live, peak = workspace.device_bytes()
    assert peak >= n * n * 8 and live >= n * n * 8  # the row-major copy stays cached
    workspace.release()
    assert workspace.device_bytes()[0] == 0
