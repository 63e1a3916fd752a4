"""The native multi-GPU Cholesky (csrc/dist_schedule.h + dist.cu), checked on
a CPU.

tests/dist_harness.cpp instantiates the SAME schedule template the NCCL
driver runs, with the oracle as the compute and an in-process broadcast per
row / column communicator as the transport, P threads standing for the P
ranks.  The distributed factor must be bit-identical to the oracle's
single-process factorization with the same tree (every element receives the
same fold sequence), for the 1x1 / 1x2 / 2x2 / 2x4 grids the bench uses and
for odd grids and ragged last tiles; a pivot failure must give every rank the
same global index.  The layout queries exported by the product library
(host-only functions, no GPU) must agree with the Python mirror
(dist/layout.py LowerPanels).
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from conftest import ROOT
from golden_inputs import spd_int

HARNESS_SRC = ROOT / "tests" / "dist_harness.cpp"
HARNESS = ROOT / "tests" / "_build" / "libdist_harness.so"


class _Level(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("pad_", ctypes.c_int32), ("bs", ctypes.c_int64), ("kc", ctypes.c_int64)]


@pytest.fixture(scope="module")
def harness():
    O.build()
    deps = [HARNESS_SRC, *(ROOT / "paper_2604_07311_b200" / "csrc").glob("dist_*.h")]
    if not HARNESS.exists() or any(d.stat().st_mtime > HARNESS.stat().st_mtime for d in deps):
        HARNESS.parent.mkdir(exist_ok=True)
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-ffp-contract=off",
                        "-I", str(ROOT / "include"), "-I", str(ROOT / "paper_2604_07311_b200" / "csrc"),
                        str(HARNESS_SRC), str(O.LIB), f"-Wl,-rpath,{O.LIB.parent}", "-o", str(HARNESS)], check=True)
    lib = ctypes.CDLL(str(HARNESS))
    lib.harness_chol_dist.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(_Level), ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int64)]
    lib.harness_chol_dist.restype = ctypes.c_int64
    lib.harness_set_grouped.argtypes = [ctypes.c_int]
    return lib


def _tree(nb: int, inner: int | None):
    doc = {"op": "cholesky", "variant": 3, "bs": nb, "kernel": {"kc": nb}}
    if inner:
        doc["child"] = {"op": "cholesky", "variant": 3, "bs": inner, "kernel": {"kc": inner},
                        "child": {"op": "cholesky", "variant": "unblocked3"}}
    else:
        doc["child"] = {"op": "cholesky", "variant": "unblocked3"}
    return doc


def _run(harness, a0, pr, pc, doc, lookahead=True, grouped=False):
    n = a0.shape[0]
    harness.harness_set_grouped(int(grouped))
    lv = O.levels_from_tree(doc, n, "f64")
    arr = (_Level * len(lv))(*[_Level(v, 0, bs, kc) for v, bs, kc in lv])
    full = np.ascontiguousarray(a0, dtype=np.float64).copy()
    calls = ctypes.c_int64(0)
    info = harness.harness_chol_dist(full.ctypes.data, n, pr, pc, arr, len(lv), int(lookahead), ctypes.byref(calls))
    return full, int(info), calls.value


def _oracle(a0, doc):
    n = a0.shape[0]
    st = np.ascontiguousarray(a0, dtype=np.float64).reshape(-1).copy()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}, O.levels_from_tree(doc, n, "f64"))
    return st.reshape(n, n), bad


@pytest.mark.parametrize("grouped", [False, True], ids=["per_panel", "grouped"])
@pytest.mark.parametrize("pr,pc", [(1, 1), (1, 2), (2, 2), (2, 4), (2, 3), (3, 2), (4, 1)])
@pytest.mark.parametrize("n,nb,inner", [(512, 64, 16), (450, 64, None), (300, 96, 32)])
def test_dist_schedule_bitwise_vs_oracle(harness, pr, pc, n, nb, inner, grouped):
    """grouped: the update's panels go to the executor as one group list (the
    one-launch path of dist.cu), each panel one GEMM over its trapezoid."""
    a0 = spd_int(900 + n + 10 * pr + pc, n)
    doc = _tree(nb, inner)
    got, info, calls = _run(harness, a0, pr, pc, doc, grouped=grouped)
    ref, bad = _oracle(a0, doc)
    assert info == -1 and bad == -1
    assert calls > 0
    low = np.tril_indices(n)
    assert got[low].tobytes() == ref[low].tobytes(), "distributed factor differs from the oracle"


@pytest.mark.parametrize("lookahead", [True, False])
def test_dist_schedule_lookahead_same_bits(harness, lookahead):
    a0 = spd_int(4711, 384)
    doc = _tree(64, 16)
    got, info, _ = _run(harness, a0, 2, 2, doc, lookahead)
    ref, _ = _oracle(a0, doc)
    assert info == -1
    low = np.tril_indices(384)
    assert got[low].tobytes() == ref[low].tobytes()


@pytest.mark.parametrize("grouped", [False, True], ids=["per_panel", "grouped"])
@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 2), (2, 4)])
def test_dist_schedule_pivot_failure_index(harness, pr, pc, grouped):
    n = 320
    a0 = spd_int(77, n)
    a0[200, 200] = -1e6  # fails at global pivot 200 (tile 3 of nb=64)
    doc = _tree(64, 16)
    _, info, _ = _run(harness, a0, pr, pc, doc, grouped=grouped)
    _, bad = _oracle(a0, doc)
    assert bad == 200 and info == 200


@pytest.mark.parametrize("pr,pc", [(1, 1), (1, 2), (2, 2), (2, 4), (3, 2)])
@pytest.mark.parametrize("n,nb", [(1000, 128), (1024, 128), (131072, 1024), (5, 8)])
def test_layout_queries_match_python_mirror(pr, pc, n, nb):
    from paper_2604_07311_b200.dist.layout import LowerPanels
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    total = 0
    for r in range(pr * pc):
        lp = LowerPanels(n, nb, pr, pc, r)
        assert lib.bf_dist_local_elems(n, nb, pr, pc, r) == lp.local_elems()
        for q, (_, _, _, _, off) in enumerate(lp.panels()):
            assert lib.bf_dist_panel_offset(n, nb, pr, pc, r, q) == off
        total += lp.local_elems()
    t = -(-n // nb)
    # the ranks together hold exactly the lower tiles
    full_tiles = sum(min(nb, n - i * nb) * min(nb, n - j * nb) for i in range(t) for j in range(i + 1))
    assert total == full_tiles


def test_python_scatter_gather_roundtrip():
    from paper_2604_07311_b200.dist.layout import LowerPanels

    n, nb, pr, pc = 700, 128, 2, 4
    rng = np.random.default_rng(3)
    full = rng.uniform(-1, 1, (n, n))
    out = np.zeros_like(full)
    for r in range(pr * pc):
        lp = LowerPanels(n, nb, pr, pc, r)
        lp.gather_into(lp.scatter(full), out)
    t = np.arange(n) // nb
    lower_tiles = t[:, None] >= t[None, :]
    assert np.array_equal(out[lower_tiles], full[lower_tiles])
    assert not out[~lower_tiles].any()


# ---- GPU: the NCCL driver itself (one rank per GPU; the box has one GPU) -------


@pytest.mark.gpu
@pytest.mark.parametrize("grouped", [0, 1], ids=["per_panel", "grouped"])
@pytest.mark.parametrize("lookahead", [0, 1])
@pytest.mark.parametrize("n,nb,kc", [(640, 128, None), (1000, 256, None), (3000, 512, None), (2900, 512, 128),
                                     (4100, 1024, 256)])
def test_nccl_driver_single_rank_bitwise(cuda, n, nb, kc, grouped, lookahead):
    """grouped=1: every update part is one grouped TMA launch over the column
    panels (ragged last tiles, kc < nb segments); 0: one GEMM per panel."""
    from paper_2604_07311_b200.dist import native

    native.selftest_single_rank(n=n, nb=nb, seed=n, kc=kc, options={"grouped": grouped, "lookahead": lookahead})


@pytest.mark.gpu
@pytest.mark.parametrize("grouped", [0, 1], ids=["per_panel", "grouped"])
@pytest.mark.parametrize("lookahead", [0, 1])
def test_nccl_driver_pivot_failure(cuda, lookahead, grouped):
    import torch

    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree_dict
    from paper_2604_07311_b200.dist import native

    n, nb = 700, 128
    tree = parse_tree_dict({"op": "cholesky", "variant": 3, "bs": nb, "kernel": {"kc": nb},
                            "child": {"op": "cholesky", "variant": "unblocked3"}})
    ctx = native.DistContext.single()
    try:
        ctx.set_option("lookahead", lookahead)
        ctx.set_option("grouped", grouped)
        lp = ctx.layout(n, nb)
        full = torch.empty(n, n, dtype=torch.float64, device=cuda)
        native.fill_synthetic_full(full, 5)
        full[300, 300] = -1e9
        local = native.scatter_local(lp, full)
        with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
            native.cholesky_dist(ctx, local, n, tree)
        assert e.value.index == 300
    finally:
        ctx.close()


@pytest.mark.gpu
def test_nccl_driver_synthetic_is_spd_and_residual(cuda):
    """fill_synthetic gives each rank its tiles of S + nI; the factor's
    randomized backward error is at rounding level."""
    import torch

    from paper_2604_07311_b200.control import parse_tree_dict
    from paper_2604_07311_b200.dist import native

    n, nb = 4096, 512
    tree = parse_tree_dict({"op": "cholesky", "variant": 3, "bs": nb, "kernel": {"kc": nb},
                            "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                                      "child": {"op": "cholesky", "variant": "unblocked3"}}})
    ctx = native.DistContext.single()
    try:
        lp = ctx.layout(n, nb)
        local = torch.empty(lp.local_elems(), dtype=torch.float64, device=cuda)
        native.fill_synthetic(ctx, local, n, nb, 11)
        native.cholesky_dist(ctx, local, n, tree)
        a0 = torch.empty(n, n, dtype=torch.float64, device=cuda)
        native.fill_synthetic_full(a0, 11)
        assert torch.equal(a0, a0.T)
        L = torch.zeros_like(a0)
        native.gather_local(lp, local, L)
        L = torch.tril(L)
        x = torch.randn(n, 3, dtype=torch.float64, device=cuda)
        rel = ((a0 @ x - L @ (L.T @ x)).norm() / (a0.norm() * x.norm())).item()
        assert rel < 1e-15
    finally:
        ctx.close()
