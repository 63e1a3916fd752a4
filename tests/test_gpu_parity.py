"""GPU parity beyond the golden fixtures: larger sizes against the (golden-
pinned) oracle on identical bytes, the reference's bitwise contracts, its
edge semantics, and size-independent properties at bench sizes."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
import paper_2604_07311_b200 as bf
from golden_inputs import digest, spd_int
from paper_2604_07311_b200.control import parse_tree
from paper_2604_07311_b200.engine import KernelConfig
from paper_2604_07311_b200.views import DType, Range, make_view

pytestmark = pytest.mark.gpu

F64 = DType.F64


def chol_gpu(a0: np.ndarray, tree_doc, uplo="lower"):
    n = a0.shape[0]
    v = make_view(n, n, fill=a0)
    bf.cholesky(v, uplo, parse_tree(tree_doc) if tree_doc else None)
    return v.storage.cpu().numpy()


def chol_oracle(a0: np.ndarray, tree_doc, uplo="lower"):
    import json

    n = a0.shape[0]
    st = a0.reshape(-1).copy()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                     O.levels_from_tree(json.loads(tree_doc) if tree_doc else None, n, "f64"), uplo=uplo,
                     nthreads=O.host_threads())
    assert bad == -1
    return st


TREES = [
    '{"op":"cholesky","variant":3,"bs":128,"child":{"op":"cholesky","variant":"unblocked3"}}',
    '{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky","variant":3,"bs":64,'
    '"child":{"op":"cholesky","variant":"unblocked3"}}}',
    '{"op":"cholesky","variant":2,"bs":256,"child":{"op":"cholesky","variant":"unblocked2"}}',
    '{"op":"cholesky","variant":1,"bs":192,"kernel":{"kc":96},"child":{"op":"cholesky","variant":"unblocked1"}}',
]


@pytest.mark.parametrize("tree", TREES)
def test_cholesky_2000_bitwise_vs_oracle(cuda, tree):
    a0 = spd_int(777, 2000)
    assert digest(chol_gpu(a0, tree)) == digest(chol_oracle(a0, tree))


def test_upper_is_bitwise_transpose_of_lower(cuda):
    a0 = spd_int(5, 700)
    t = TREES[1]
    lo = chol_gpu(a0, t, "lower").reshape(700, 700)
    up = chol_gpu(a0, t, "upper").reshape(700, 700)
    assert np.tril(lo).tobytes() == np.tril(up.T).tobytes()
    assert np.triu(lo, 1).tobytes() == np.triu(a0, 1).tobytes()  # other triangle untouched


def test_npd_reports_global_index_and_stops(cuda):
    a0 = spd_int(9, 300)
    a0[211, 211] = -1e6
    v = make_view(300, 300, fill=a0)
    with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
        bf.cholesky(v, tree=parse_tree(TREES[1]))
    assert e.value.index == 211
    st = a0.reshape(-1).copy()
    import json

    bad = O.cholesky(st, {"off": 0, "m": 300, "n": 300, "rs": 300, "cs": 1},
                     O.levels_from_tree(json.loads(TREES[1]), 300, "f64"))
    assert bad == 211
    assert digest(v.storage.cpu().numpy()) == digest(st)  # same partial state as the reference stops in


@pytest.mark.parametrize("pipeline", [2, 4, 15])
@pytest.mark.parametrize("tree", TREES[:2])
def test_pipelined_first_step_bitwise_vs_oracle(cuda, tree, pipeline):
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    a0 = spd_int(778, 2000)
    assert lib.bf_set_option(b"pipeline_first", pipeline) == 0
    try:
        got = chol_gpu(a0, tree)
    finally:
        lib.bf_set_option(b"pipeline_first", 0)
    assert digest(got) == digest(chol_oracle(a0, tree))


@pytest.mark.parametrize("npd_at", [100, 700, 1300])
@pytest.mark.parametrize("pipeline", [4, 0, 15, 2])
def test_lookahead_pipelined_first_step_npd_partial_state(cuda, npd_at, pipeline):
    """The row-chunked first step (panel TRSM chunks on the panel stream, the
    chunk's block-column and rest updates on two more streams) stops in the
    reference's partial state for a failure in step 0's diagonal block, in
    panel 1, and later."""
    import json

    from paper_2604_07311_b200.engine import _lib

    n = 2000
    a0 = spd_int(31, n)
    a0[npd_at, npd_at] = -1e9
    lib = _lib.lib()
    assert lib.bf_set_option(b"pipeline_first", pipeline) == 0
    try:
        v = make_view(n, n, fill=a0)
        with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
            bf.cholesky(v, tree=parse_tree(TREES[1]))
    finally:
        lib.bf_set_option(b"pipeline_first", 0)
    assert e.value.index == npd_at
    st = a0.reshape(-1).copy()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                     O.levels_from_tree(json.loads(TREES[1]), n, "f64"), nthreads=O.host_threads())
    assert bad == npd_at
    assert digest(v.storage.cpu().numpy()) == digest(st)


RESERVE_TREE = ('{"op": "cholesky", "variant": 3, "bs": 256, "kernel": {"kc": 256}, "child": {"op": "cholesky", '
                '"variant": 3, "bs": 64, "kernel": {"kc": 64}, "child": {"op": "cholesky", "variant": "unblocked3"}}}')


@pytest.mark.parametrize("overlap", [1, 0, 3, 4])  # 3: 3 row chunks on their own streams; 4: no early panels
@pytest.mark.parametrize("npd_at", [None, 10, 300, 1000, 1290, 2200])
def test_panel_overlap_bitwise(cuda, overlap, npd_at):
    """Overlapped panels (option "panel_overlap"): the TRSM of the rows below
    trails the diagonal factor's inner steps on a second stream, on a copy that
    is written back only when no pivot failure was flagged.  Same bits as the
    oracle, and after a failure the same partial state — failures in the first
    panel's first and later inner blocks, in a later panel, in the last one."""
    import json

    from paper_2604_07311_b200.engine import _lib

    n = 2304
    a0 = spd_int(4343, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    lib = _lib.lib()
    try:
        assert lib.bf_set_option(b"panel_overlap", 1 if overlap else 0) == 0
        assert lib.bf_set_option(b"panel_chunks", 3 if overlap == 3 else 2) == 0
        assert lib.bf_set_option(b"panel_chunk_rows", 256 if overlap == 3 else 6144) == 0
        assert lib.bf_set_option(b"early_panel", 0 if overlap == 4 else 1) == 0
        v = make_view(n, n, fill=a0)
        bad = int(bf.cholesky_async(v, "lower", parse_tree(RESERVE_TREE)).item())
    finally:
        lib.bf_set_option(b"panel_overlap", 1)
        lib.bf_set_option(b"panel_chunks", 2)
        lib.bf_set_option(b"panel_chunk_rows", 6144)
        lib.bf_set_option(b"early_panel", 1)
    st = a0.reshape(-1).copy()
    ref_bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                         O.levels_from_tree(json.loads(RESERVE_TREE), n, "f64"), nthreads=O.host_threads())
    assert ref_bad == (-1 if npd_at is None else npd_at)
    assert bad == ref_bad
    assert digest(v.storage.cpu().numpy()) == digest(st)


FUSED_TREE = ('{"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128}, '
              '"child": {"op": "cholesky", "variant": "unblocked3"}}')


@pytest.mark.parametrize("ctas", [0, 1, 5])
@pytest.mark.parametrize("n,npd_at", [(129, None), (200, None), (256, None), (700, None), (1000, None), (2048, None),
                                      (2048, 5), (2048, 130), (2048, 1000), (2048, 2047), (777, 700), (300, 150)])
def test_fused_diag_factor_bitwise(cuda, n, npd_at, ctas):
    """The one-launch diagonal factor (potrf_diag_fused_kernel: leaf, TRSM and
    update tasks claimed by ticket, any grid size) against the oracle running
    the same tree: same bits, same pivot index and, after a failure, the same
    partial state (updates of earlier steps complete, later steps skipped).
    fused_diag = 0 (the launch sequence) must agree too."""
    import json

    from paper_2604_07311_b200.engine import _lib

    a0 = spd_int(5150 + n, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    st = a0.reshape(-1).copy()
    ref_bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                         O.levels_from_tree(json.loads(FUSED_TREE), n, "f64"), nthreads=O.host_threads())
    assert ref_bad == (-1 if npd_at is None else npd_at)
    lib = _lib.lib()
    launches = {}
    for fused in (1, 0):
        try:
            assert lib.bf_set_option(b"fused_diag", fused) == 0
            assert lib.bf_set_option(b"fused_diag_ctas", ctas) == 0
            v = make_view(n, n, fill=a0)
            before = lib.bf_launch_count()
            bad = int(bf.cholesky_async(v, "lower", parse_tree(FUSED_TREE)).item())
            launches[fused] = lib.bf_launch_count() - before
        finally:
            lib.bf_set_option(b"fused_diag", 1)
            lib.bf_set_option(b"fused_diag_ctas", 0)
        assert bad == ref_bad, f"fused={fused}"
        assert digest(v.storage.cpu().numpy()) == digest(st), f"fused={fused}"
    assert launches[1] == 1 and launches[0] > 3


OVERLAP_FUSED_TREE = ('{"op": "cholesky", "variant": 3, "bs": 1024, "kernel": {"kc": 1024}, "child": ' + FUSED_TREE + '}')


@pytest.mark.parametrize("fused", [2, 1])
@pytest.mark.parametrize("npd_at", [None, 10, 700, 1100, 2500])
def test_fused_diag_in_overlapped_panels_bitwise(cuda, fused, npd_at):
    """fused_diag = 2: the overlapped panels' diagonal factors run as one
    launch whose per-column flags release the trailing TRSM through stream
    memory waits.  Same bits as the oracle and the same partial state after a
    failure in the first panel, a later one and the last one."""
    import json

    from paper_2604_07311_b200.engine import _lib

    n = 2600
    a0 = spd_int(6161, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    lib = _lib.lib()
    try:
        assert lib.bf_set_option(b"fused_diag", fused) == 0
        v = make_view(n, n, fill=a0)
        bad = int(bf.cholesky_async(v, "lower", parse_tree(OVERLAP_FUSED_TREE)).item())
    finally:
        lib.bf_set_option(b"fused_diag", 1)
    st = a0.reshape(-1).copy()
    ref_bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                         O.levels_from_tree(json.loads(OVERLAP_FUSED_TREE), n, "f64"), nthreads=O.host_threads())
    assert ref_bad == (-1 if npd_at is None else npd_at)
    assert bad == ref_bad
    assert digest(v.storage.cpu().numpy()) == digest(st)


@pytest.mark.parametrize("kc", [320, 64])
@pytest.mark.parametrize("npd_at", [None, 700, 1650])
def test_panel_overlap_ragged_inner_blocks_bitwise(cuda, kc, npd_at):
    """Overlapped and early panels when the inner block (96) does not divide
    the panel (320) and the order (1700) is not a multiple of either: the
    TRSM pieces wait for the right inner step, ragged last blocks, kc below
    the panel width, and the partial state after a failure."""
    import json

    n = 1700
    tree = json.dumps({"op": "cholesky", "variant": 3, "bs": 320, "kernel": {"kc": kc},
                       "child": {"op": "cholesky", "variant": 3, "bs": 96, "kernel": {"kc": 96},
                                 "child": {"op": "cholesky", "variant": "unblocked3"}}})
    a0 = spd_int(5252 + kc, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    v = make_view(n, n, fill=a0)
    bad = int(bf.cholesky_async(v, "lower", parse_tree(tree)).item())
    st = a0.reshape(-1).copy()
    ref_bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                         O.levels_from_tree(json.loads(tree), n, "f64"), nthreads=O.host_threads())
    assert ref_bad == (-1 if npd_at is None else npd_at)
    assert bad == ref_bad
    assert digest(v.storage.cpu().numpy()) == digest(st)


@pytest.mark.parametrize("opts", [
    {"tail_reserve": 0},                                     # 1-tile CTAs on the whole GPU
    {"tail_reserve": 16, "tail_rows": 1 << 40},              # default grid shape on every step
    {"tail_reserve": 40, "tail_rows": 1 << 40, "reserve_strided": 1},
    {"tail_reserve": 0, "diag_reserve": 24, "diag_rows": 700},  # two-phase rest update
    {"tail_reserve": 16, "tail_rows": 1024, "diag_reserve": 8, "diag_rows": 384},
])
@pytest.mark.parametrize("npd_at", [None, 1500])
def test_lookahead_sm_reservation_bitwise(cuda, opts, npd_at):
    """The SM-reservation options of the lookahead schedule (persistent grid
    leaving SMs to the panel stream, strided tile order, the two-phase rest
    update) only change grid shapes and launch splits: the factor, and the
    partial state after a pivot failure, stay the reference's bits.  n=2304
    with bs=256 puts up to 28 tile rows (406 tiles > one per SM) in the rest
    update, so the persistent grid really holds several tiles per CTA."""
    import json

    from paper_2604_07311_b200.engine import _lib

    n = 2304
    a0 = spd_int(4242, n)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e9
    lib = _lib.lib()
    defaults = {"tail_reserve": 16, "tail_rows": 32768, "diag_reserve": 0, "diag_rows": 0, "reserve_strided": 0}
    try:
        for key, val in opts.items():
            assert lib.bf_set_option(key.encode(), int(val)) == 0
        v = make_view(n, n, fill=a0)
        bad = int(bf.cholesky_async(v, "lower", parse_tree(RESERVE_TREE)).item())
    finally:
        for key, val in defaults.items():
            lib.bf_set_option(key.encode(), val)
    st = a0.reshape(-1).copy()
    ref_bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1},
                         O.levels_from_tree(json.loads(RESERVE_TREE), n, "f64"), nthreads=O.host_threads())
    assert ref_bad == (-1 if npd_at is None else npd_at)
    assert bad == ref_bad
    assert digest(v.storage.cpu().numpy()) == digest(st)


@pytest.mark.parametrize("leaf_blocked,leaf_pipe", [(1, 1), (1, 0), (0, 0)])
@pytest.mark.parametrize("dt,npd_at", [("f64", None), ("f64", 77), ("f64", 100), ("f32", None), ("f32", 45)])
def test_leaf_kernels_bitwise_and_partial_state(cuda, leaf_blocked, leaf_pipe, dt, npd_at):
    """Both variant-3 leaf kernels (blocked lane-per-row v4 — with the next
    diagonal chain overlapping the previous block's trailing update or not —
    and column-parallel v3) give the oracle's bits, and on a failing pivot —
    inside the first column block, or mid-block past it — the oracle's
    partial state and index."""
    import json

    from paper_2604_07311_b200.engine import _lib

    n = 123  # ragged last 32-column block
    doc = '{"op":"cholesky","variant":"unblocked3"}'
    a0 = spd_int(31, n, dt)
    if npd_at is not None:
        a0[npd_at, npd_at] = -1e6
    st = a0.reshape(-1).copy()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}, O.levels_from_tree(json.loads(doc), n, dt))
    lib = _lib.lib()
    lib.bf_set_option(b"leaf_blocked", leaf_blocked)
    lib.bf_set_option(b"leaf_pipe", leaf_pipe)
    try:
        v = make_view(n, n, DType.parse(dt), fill=a0)
        if npd_at is None:
            bf.cholesky(v, "lower", parse_tree(doc))
        else:
            with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
                bf.cholesky(v, "lower", parse_tree(doc))
            assert e.value.index == bad == npd_at
    finally:
        lib.bf_set_option(b"leaf_blocked", 1)  # the defaults
        lib.bf_set_option(b"leaf_pipe", 1)
    assert digest(v.storage.cpu().numpy()) == digest(st)


def test_gemmt_lower_equals_gemm_lower_bitwise(cuda):
    rng = np.random.default_rng(13)
    n, k = 777, 513
    a = make_view(n, k, fill=rng.uniform(-1, 1, (n, k)))
    b = make_view(k, n, fill=rng.uniform(-1, 1, (k, n)))
    c0 = rng.uniform(-1, 1, (n, n))
    ct, cf = make_view(n, n, fill=c0), make_view(n, n, fill=c0)
    bf.gemmt_lower(-1.0, a, b, 1.0, ct)
    bf.gemm(-1.0, a, b, 1.0, cf)
    assert np.tril(ct.to_numpy()).tobytes() == np.tril(cf.to_numpy()).tobytes()
    assert np.triu(ct.to_numpy(), 1).tobytes() == np.triu(c0, 1).tobytes()


@pytest.mark.parametrize("kind", ["contiguous", "transposed", "padded"])
def test_gemm_layouts_bitwise_vs_oracle(cuda, kind):
    from golden_inputs import gemm_inputs

    for seed, (m, n, k), kc in [(1, (300, 200, 700), 256), (2, (129, 1000, 64), 33), (3, (1000, 40, 500), 500)]:
        a, b, c = gemm_inputs(seed, "gemm", "f64", m, n, k, (kind, kind, kind))
        cst = c[0].copy()
        O.gemm(0.75, a, b, -1.5, (cst, c[1]), kc=kc)
        cfg = KernelConfig(8, 6, 64, kc, 2048, F64, F64)
        dv = lambda s, meta: bf.MatrixView(torch.as_tensor(s).cuda(), meta["off"], meta["m"], meta["n"],
                                           meta["rs"], meta["cs"], F64)
        vc = dv(*c)
        bf.gemm(0.75, dv(*a), dv(*b), -1.5, vc, cfg=cfg)
        assert digest(vc.storage.cpu().numpy()) == digest(cst)


def test_edge_semantics(cuda):
    nan = float("nan")
    c = make_view(3, 3, fill=np.full((3, 3), nan))
    bf.gemm(1.0, make_view(3, 2, fill=np.ones((3, 2))), make_view(2, 3, fill=np.ones((2, 3))), 0.0, c)
    assert np.array_equal(c.to_numpy(), np.full((3, 3), 2.0))  # beta=0 never reads C
    c0 = np.array([[0.25, -0.0], [np.pi, 7.0]])
    c = make_view(2, 2, fill=c0)
    bf.gemm(0.0, make_view(2, 2, fill=np.full((2, 2), nan)), make_view(2, 2), 1.0, c)
    assert c.to_numpy().tobytes() == c0.tobytes()  # alpha=0, beta=1: exact no-op
    c = make_view(2, 2, fill=[[1, 2], [3, 4]])
    bf.gemm(1.0, make_view(2, 0), make_view(0, 2), 0.0, c)
    assert c.to_numpy().tolist() == [[0, 0], [0, 0]]
    c = make_view(3, 3, fill=np.arange(9.0).reshape(3, 3))
    bf.gemmt_lower(1.0, make_view(3, 2), make_view(2, 3), 0.5, c)
    cn = c.to_numpy()
    assert np.array_equal(np.tril(cn), 0.5 * np.tril(np.arange(9.0).reshape(3, 3)))
    assert np.array_equal(np.triu(cn, 1), np.triu(np.arange(9.0).reshape(3, 3), 1))


def test_trsm_singular_and_hand(cuda):
    tri = make_view(2, 2, fill=[[2, 0], [1, 2]])
    b = make_view(1, 2, fill=[[2, 5]])
    bf.trsm(bf.engine.RIGHT_LOWER_TRANS_NONUNIT, 1.0, tri, b)
    assert b.to_numpy().tolist() == [[1, 2]]
    with pytest.raises(bf.errors.SingularMatrixError):
        bf.trsm(bf.engine.RIGHT_LOWER_TRANS_NONUNIT, 1.0, make_view(2, 2, fill=[[1, 0], [1, 0]]),
                make_view(1, 2, fill=[[1, 1]]))


def test_cholesky_bench_size_residual(cuda):
    """n=8192 with the bench tree: randomized backward error on device."""
    n = 8192
    torch.manual_seed(0)
    m = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
    a0 = m @ m.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    a = bf.from_torch(a0.clone())
    tree = parse_tree('{"op":"cholesky","variant":3,"bs":1024,"kernel":{"kc":1024},"child":{"op":"cholesky",'
                      '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}')
    bf.cholesky(a, tree=tree)
    L = torch.tril(a.to_torch())
    x = torch.randn(n, 4, dtype=torch.float64, device="cuda")
    r = a0 @ x - L @ (L.T @ x)
    rel = (r.norm() / (a0.norm() * x.norm())).item()
    assert rel <= 10 * n * np.finfo(np.float64).eps / n  # far inside 10*n*eps


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_tma_kernel_variants_bitwise(cuda, variant):
    """Every TMA mainloop variant (m8n8k4 / m16n8k8, 1 or 2 k boxes per stage)
    must give the oracle's bits on SYRK and on a full factorization."""
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    lib.bf_set_option(b"tma_variant", variant)
    try:
        a0 = spd_int(4242 + variant, 1500)
        tree = ('{"op":"cholesky","variant":3,"bs":384,"kernel":{"kc":128},"child":{"op":"cholesky",'
                '"variant":3,"bs":64,"child":{"op":"cholesky","variant":"unblocked3"}}}')
        assert digest(chol_gpu(a0, tree)) == digest(chol_oracle(a0, tree))
        rng = np.random.default_rng(variant)
        n, k = 1000, 512
        a = rng.uniform(-1, 1, (n, k))
        c0 = rng.uniform(-1, 1, (n, n))
        va, vc = make_view(n, k, fill=a), make_view(n, n, fill=c0)
        cfg = KernelConfig(8, 6, 64, 256, 2048, F64, F64)
        bf.syrk_lower(-0.5, va, 2.0, vc, cfg=cfg)
        cst = c0.reshape(-1).copy()
        O.syrk(-0.5, (a.reshape(-1).copy(), {"off": 0, "m": n, "n": k, "rs": k, "cs": 1}), 2.0,
               (cst, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}), kc=256)
        assert digest(vc.storage.cpu().numpy()) == digest(cst)
    finally:
        lib.bf_set_option(b"tma_variant", 2)


@pytest.mark.parametrize("beta", [0.0, 1.0, -0.75])
@pytest.mark.parametrize("lower", [False, True])
def test_tma_red_fold_bitwise(cuda, beta, lower):
    """The TMA kernel folds every segment with beta_eff == 1 as L2 reductions
    (red.global.add.f64): same bits as the load/add/store fold and the oracle,
    over many segments (kc=64 -> 12 folds), ragged edges, and lower-only C."""
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    rng = np.random.default_rng(77 + int(lower))
    m, n, k, kc = 700, 650, 768, 64
    if lower:
        n = m
    a = rng.uniform(-1, 1, (m, k))
    bt = rng.uniform(-1, 1, (n, k))
    c0 = rng.uniform(-1, 1, (m, n))
    cst = c0.reshape(-1).copy()
    O.gemm(-1.25, (a.reshape(-1).copy(), {"off": 0, "m": m, "n": k, "rs": k, "cs": 1}),
           (bt.reshape(-1).copy(), {"off": 0, "m": k, "n": n, "rs": 1, "cs": k}), beta,
           (cst, {"off": 0, "m": m, "n": n, "rs": n, "cs": 1}), kc=kc, lower_only=lower)
    cfg = KernelConfig(8, 6, 64, kc, 2048, F64, F64)
    outs = []
    try:
        for mode in (1, 0):
            lib.bf_set_option(b"red_fold", mode)
            va, vb, vc = make_view(m, k, fill=a), make_view(n, k, fill=bt), make_view(m, n, fill=c0)
            fn = bf.gemmt_lower if lower else bf.gemm
            fn(-1.25, va, vb.transposed(), beta, vc, cfg=cfg)
            outs.append(digest(vc.storage.cpu().numpy()))
    finally:
        lib.bf_set_option(b"red_fold", 1)
    assert outs[0] == outs[1] == digest(cst)


@pytest.mark.parametrize("bn", [64, 128, "64tmc"])
@pytest.mark.parametrize("lower", [False, True])
def test_tma_half_width_tiles_bitwise(cuda, bn, lower):
    """Both TMA tile shapes (option "tma_bn": 64 = two 8-warp groups on
    128 x 64 tiles, the default; 128 = one 16-warp 128 x 128 tile): same
    per-element fma chains and folds, so the oracle's bits — ragged edges,
    lower-only C split into tile halves, many kc segments (TMEM fold off so
    the 64-wide path runs them), and a whole factorization."""
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    tmc = bn == "64tmc"  # the TMEM-fold instantiation on the two-group tiles (option "tmc_bn64")
    bn = 64 if tmc else bn
    rng = np.random.default_rng(91 + int(lower) + bn)
    m, n, k, kc = 700, 650, 768, 64
    if lower:
        n = m
    a = rng.uniform(-1, 1, (m, k))
    bt = rng.uniform(-1, 1, (n, k))
    c0 = rng.uniform(-1, 1, (m, n))
    cst = c0.reshape(-1).copy()
    O.gemm(-1.25, (a.reshape(-1).copy(), {"off": 0, "m": m, "n": k, "rs": k, "cs": 1}),
           (bt.reshape(-1).copy(), {"off": 0, "m": k, "n": n, "rs": 1, "cs": k}), 0.5,
           (cst, {"off": 0, "m": m, "n": n, "rs": n, "cs": 1}), kc=kc, lower_only=lower)
    cfg = KernelConfig(8, 6, 64, kc, 2048, F64, F64)
    try:
        lib.bf_set_option(b"tma_bn", bn)
        lib.bf_set_option(b"tmem_fold", 1 if tmc else 0)
        lib.bf_set_option(b"tmc_bn64", 1 if tmc else 0)
        va, vb, vc = make_view(m, k, fill=a), make_view(n, k, fill=bt), make_view(m, n, fill=c0)
        fn = bf.gemmt_lower if lower else bf.gemm
        fn(-1.25, va, vb.transposed(), 0.5, vc, cfg=cfg)
        got = digest(vc.storage.cpu().numpy())
        a0 = spd_int(5150 + bn, 1700)
        tree = ('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":256},"child":{"op":"cholesky",'
                '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}')
        chol_ok = digest(chol_gpu(a0, tree)) == digest(chol_oracle(a0, tree))
    finally:
        lib.bf_set_option(b"tma_bn", 64)
        lib.bf_set_option(b"tmem_fold", 1)
        lib.bf_set_option(b"tmc_bn64", 0)
    assert got == digest(cst)
    assert chol_ok


def test_tma_persist_grid_bitwise(cuda):
    """The strided persistent grid (option "persist", long-K GEMMs with at
    least 4 tiles per SM) only reorders tiles: same bits as the default grid."""
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    torch.manual_seed(5)
    m, n, k, kc = 3200, 3072, 4096, 1024
    a = torch.rand(m, k, dtype=torch.float64, device="cuda") - 0.5
    bt = torch.rand(n, k, dtype=torch.float64, device="cuda") - 0.5
    c0 = torch.rand(m, n, dtype=torch.float64, device="cuda") - 0.5
    cfg = KernelConfig(8, 6, 64, kc, 2048, F64, F64)
    outs = []
    try:
        for persist in (0, 1):
            lib.bf_set_option(b"persist", persist)
            c = c0.clone()
            bf.gemm(0.5, bf.from_torch(a), bf.from_torch(bt).transposed(), 1.0, bf.from_torch(c), cfg=cfg)
            torch.cuda.synchronize()
            outs.append(c)
    finally:
        lib.bf_set_option(b"persist", 0)
    assert torch.equal(outs[0], outs[1])
    assert not torch.equal(outs[0], c0)


@pytest.mark.parametrize("dt,kc,bs,n", [("f64", 40, 128, 700), ("f64", 1024, 96, 700), ("f32", 20, 96, 700),
                                        ("f32", 512, 100, 700), ("f64", 128, 128, 5000), ("f32", 64, 128, 5000)])
def test_fused_trsm_subtree_bitwise(cuda, dt, kc, bs, n):
    """Panels of width <= 128 take a fused TRSM kernel (warp per 32 rows, one
    or two warps per CTA — n=5000 reaches the paired grid — or the 64-row CTA
    kernel); multi-segment kc and f32 must still give the oracle's bits (and
    the unfused launches' bits)."""
    import json

    from paper_2604_07311_b200.engine import _lib

    doc = json.dumps({"op": "cholesky", "variant": 3, "bs": bs, "kernel": {"kc": kc},
                      "child": {"op": "cholesky", "variant": "unblocked3"}})
    a0 = spd_int(99, n, dt)
    st = a0.reshape(-1).copy()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}, O.levels_from_tree(json.loads(doc), n, dt))
    assert bad == -1
    outs = []
    lib = _lib.lib()
    for fused, warp in ((1, 1), (1, 0), (0, 1)):
        lib.bf_set_option(b"fused_trsm", fused)
        lib.bf_set_option(b"trsm_warp", warp)
        try:
            v = make_view(n, n, DType.parse(dt), fill=a0)
            bf.cholesky(v, "lower", parse_tree(doc))
            outs.append(digest(v.storage.cpu().numpy()))
        finally:
            lib.bf_set_option(b"fused_trsm", 1)
            lib.bf_set_option(b"trsm_warp", 1)
    assert outs[0] == outs[1] == outs[2] == digest(st)


@pytest.mark.parametrize("n,uplo", [(1000, "lower"), (5000, "lower"), (777, "upper")])
def test_cholesky_host_streams_back_same_bits(cuda, n, uplo):
    """The host entry point (lower triangle in by block columns, finished
    block columns streamed back under the remaining steps) gives exactly
    bf.cholesky's bits and leaves the other host triangle untouched."""
    t = TREES[1] if n < 2000 else ('{"op":"cholesky","variant":3,"bs":1024,"kernel":{"kc":1024},"child":'
                                   '{"op":"cholesky","variant":3,"bs":128,"child":{"op":"cholesky","variant":"unblocked3"}}}')
    a0 = spd_int(17, n)
    host = torch.from_numpy(a0.copy()).pin_memory()
    bf.cholesky_host(host, uplo, parse_tree(t))
    ref = chol_gpu(a0, t, uplo).reshape(n, n)
    got = host.numpy()
    tri, other = (np.tril, np.triu) if uplo == "lower" else (np.triu, np.tril)
    assert tri(got).tobytes() == tri(ref).tobytes()
    assert other(got, 1 if uplo == "lower" else -1).tobytes() == other(a0, 1 if uplo == "lower" else -1).tobytes()


@pytest.mark.parametrize("npd_at", [2211, 100, 1100])
def test_cholesky_host_npd_partial_state(cuda, npd_at):
    """Failures after, inside and during the overlapped host load (step 0
    consumes block columns as they land) leave the reference's partial state."""
    a0 = spd_int(9, 3000)
    a0[npd_at, npd_at] = -1e6
    t = ('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":'
         '{"op":"cholesky","variant":3,"bs":128,"child":{"op":"cholesky","variant":"unblocked3"}}}')
    host = torch.from_numpy(a0.copy()).pin_memory()
    with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
        bf.cholesky_host(host, "lower", parse_tree(t))
    assert e.value.index == npd_at
    v = make_view(3000, 3000, fill=a0)
    with pytest.raises(bf.errors.NotPositiveDefiniteError):
        bf.cholesky(v, tree=parse_tree(t))
    assert np.tril(host.numpy()).tobytes() == np.tril(v.to_numpy()).tobytes()


@pytest.mark.parametrize("spec", ["aibj,cjdi->abcd", "iabj,jcid->abcd", "abij,cdij->abcd", "ajbi,ijcd->abcd",
                                  "aibj,jcid->acbd"])
@pytest.mark.parametrize("kc", [16, 40, 256])
@pytest.mark.parametrize("fold", [True, False])
def test_contraction_staged_bitwise_vs_oracle(cuda, spec, kc, fold):
    """Permuted contractions with the operands staged k-contiguous by the pack
    kernel (bf_pack_scatter_d) and run on the strided/TMA GEMM give the
    oracle's bits, as the element-gathering GEMM does (stage="never")."""
    from golden_inputs import tensor_inputs

    from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor

    dims = {"a": 24, "b": 20, "c": 16, "d": 12, "i": 8, "j": 10}
    lhs, lc = spec.split("->")
    la, lb = lhs.split(",")
    ad, bd, cd = [dims[x] for x in la], [dims[x] for x in lb], [dims[x] for x in lc]
    a0, b0, c0 = tensor_inputs(5150, ad, bd, cd)
    alpha, beta = -0.75, 0.5
    ref = np.asarray(c0, dtype=np.float64).reshape(-1).copy()
    O.contract(alpha, np.asarray(a0, np.float64).reshape(-1).copy(), ad, np.asarray(b0, np.float64).reshape(-1).copy(),
               bd, beta, ref, cd, spec, kc=kc, fold=fold)
    cfg = KernelConfig(8, 6, 64, kc, 2048, F64, F64)
    for stage in ("always", "never"):
        ta, tb, tc = make_tensor(ad, fill=a0), make_tensor(bd, fill=b0), make_tensor(cd, fill=c0)
        bf.contract(alpha, ta, tb, beta, tc, ContractionSpec.parse(spec), cfg=cfg, fold=fold, stage=stage)
        assert digest(tc.storage.cpu().numpy()) == digest(ref), stage


def test_pack_scatter_exact(cuda):
    """bf_pack_scatter_d copies facade elements exactly, plain and transposed."""
    import ctypes

    from paper_2604_07311_b200.engine import _lib

    src = torch.arange(5000, dtype=torch.float64, device="cuda") * 1.0000001
    rs = torch.tensor([7, 300, 11, 4000, 0], dtype=torch.int64, device="cuda")
    cs = torch.tensor([0, 3, 1, 900, 2, 5, 44], dtype=torch.int64, device="cuda")
    want = src[rs[:, None] + cs[None, :]]
    for tr in (0, 1):
        out = torch.full((35,), float("nan"), dtype=torch.float64, device="cuda")
        sv = _lib.BfScatterView(src.data_ptr(), 5, 7, rs.data_ptr(), cs.data_ptr())
        _lib.check(_lib.lib().bf_pack_scatter_d(ctypes.byref(sv), tr, out.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream), "pack")
        got = out.reshape(7, 5) if tr else out.reshape(5, 7)
        assert torch.equal(got, want.T if tr else want)


@pytest.mark.parametrize("npd", [False, True])
def test_upper_on_row_major_copy_bitwise(cuda, npd):
    """uplo="upper" at n >= upper_transpose runs on a row-major copy (the TMA
    kernel) — same bits as the in-place run on the mn-contiguous view,
    including the partial state after a pivot failure."""
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    n = 2000
    a0 = spd_int(777, n)
    if npd:
        a0[1500, 1500] = -1e9
    tree = parse_tree('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky",'
                      '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}')
    outs = []
    for thr in (0, 1024):
        lib.bf_set_option(b"upper_transpose", thr)
        v = make_view(n, n, fill=a0)
        err = None
        try:
            bf.cholesky(v, "upper", tree)
        except bf.errors.NotPositiveDefiniteError as e:
            err = e.index
        outs.append((v.to_numpy().tobytes(), err))
    lib.bf_set_option(b"upper_transpose", 1024)
    assert outs[0] == outs[1]
    assert outs[0][1] == (1500 if npd else None)


def test_two_host_threads_two_streams_bitwise(cuda):
    """Factorizations enqueued from two host threads on two streams (each with
    its own library side streams) give the sequential bits."""
    import threading

    n = 2600
    tree = parse_tree('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky",'
                      '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}')
    inputs = [spd_int(31 + i, n) for i in range(2)]
    expect = []
    for a0 in inputs:
        v = make_view(n, n, fill=a0)
        bf.cholesky(v, "lower", tree)
        expect.append(v.to_numpy().tobytes())
    views = [make_view(n, n, fill=a0) for a0 in inputs]
    torch.cuda.synchronize()
    errors = []

    def work(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(3):
                    views[i].storage.copy_(torch.as_tensor(inputs[i].reshape(-1), device="cuda"))
                    bf.cholesky(views[i], "lower", tree)
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    for i in range(2):
        assert views[i].to_numpy().tobytes() == expect[i]


@pytest.mark.parametrize("variant", [1, 2])
def test_segment_split_deep_k_bitwise(cuda, variant):
    """V1/V2's deep-K narrow updates (A11 -= A10 A10^T, A21 -= A20 A10^T) run
    their kc segments in parallel and fold them in order: the oracle's bits,
    with the split on and off."""
    from paper_2604_07311_b200.engine import _lib

    lib = _lib.lib()
    n = 4096
    a0 = spd_int(800 + variant, n)
    tree = ('{"op":"cholesky","variant":%d,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky",'
            '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}' % variant)
    ref = digest(chol_oracle(a0, tree))
    for split in (1, 0):
        lib.bf_set_option(b"segsplit", split)
        try:
            assert digest(chol_gpu(a0, tree)) == ref, f"segsplit={split}"
        finally:
            lib.bf_set_option(b"segsplit", 1)


def test_upper_copy_on_offset_subview_bitwise(cuda):
    """uplo="upper" on a submatrix view (offset, leading dimension > n) through
    the row-major copy: the oracle's bits, the rest of the storage untouched."""
    N, n, r0 = 2100, 1600, 250
    rng = np.random.default_rng(5)
    big = rng.uniform(-1, 1, (N, N))
    a0 = spd_int(91, n)
    big[r0:r0 + n, r0:r0 + n] = a0
    st = torch.tensor(big.reshape(-1), device="cuda")
    from paper_2604_07311_b200.views import MatrixView

    v = MatrixView(st, r0 * N + r0, n, n, N, 1, DType.F64)
    tree = ('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky",'
            '"variant":3,"bs":128,"kernel":{"kc":128},"child":{"op":"cholesky","variant":"unblocked3"}}}')
    bf.cholesky(v, "upper", parse_tree(tree))
    got = st.cpu().numpy().reshape(N, N)
    ref = chol_oracle(a0, tree, "upper").reshape(n, n)
    assert got[r0:r0 + n, r0:r0 + n].tobytes() == ref.tobytes()
    mask = np.ones((N, N), bool)
    mask[r0:r0 + n, r0:r0 + n] = False
    assert got[mask].tobytes() == big[mask].tobytes()
