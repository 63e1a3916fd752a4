"""CUDA-graph replay of the native Cholesky driver: the same bits as the
direct call (lookahead fork/join captured as graph edges), repeatable,
and the pivot flag of a failing matrix."""
from __future__ import annotations

import json

import numpy as np
import pytest

from golden_inputs import digest, spd_int

pytestmark = pytest.mark.gpu

TREE = ('{"op":"cholesky","variant":3,"bs":512,"kernel":{"kc":512},"child":{"op":"cholesky","variant":3,"bs":64,'
        '"child":{"op":"cholesky","variant":"unblocked3"}}}')


@pytest.mark.parametrize("n,uplo", [(3000, "lower"), (1700, "upper"), (300, "lower")])
def test_graph_replay_bitwise_equals_direct(cuda, n, uplo):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree

    a0 = spd_int(41, n)
    tree = parse_tree(TREE)
    ref = bf.make_view(n, n, fill=a0)
    bf.cholesky(ref, uplo, tree)
    v = bf.make_view(n, n, fill=a0)
    g = bf.CholeskyGraph(v, uplo, tree)
    for _ in range(2):  # replays on refilled storage
        v.copy_from(a0)
        g()
        assert digest(v.to_numpy()) == digest(ref.to_numpy())


def test_graph_replay_reports_npd(cuda):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree

    n = 2000
    a0 = spd_int(43, n)
    v = bf.make_view(n, n, fill=a0)
    g = bf.CholeskyGraph(v, "lower", parse_tree(TREE))
    bad = a0.copy()
    bad[1234, 1234] = -1e9
    v.copy_from(bad)
    with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
        g()
    assert e.value.index == 1234
    v.copy_from(a0)
    g()  # the flag resets on every replay
    assert np.isfinite(np.tril(v.to_numpy())).all()
    assert json.loads(TREE)["bs"] == 512


FUSED_CHILD = {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
               "child": {"op": "cholesky", "variant": "unblocked3"}}


@pytest.mark.parametrize("fused", [1, 2])
@pytest.mark.parametrize("n,root", [(2600, 1024), (2000, None)])
def test_graph_replay_with_fused_diagonal_factor(cuda, n, root, fused):
    """Captured: the one-launch diagonal factor (its counters reset by a
    captured memset, scratch owned by the graph); fused = 2 under capture
    records the inner-step events after the whole kernel.  Same bits as the
    direct call; a failure still reports its pivot."""
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.control import parse_tree
    from paper_2604_07311_b200.engine import _lib

    doc = FUSED_CHILD if root is None else {"op": "cholesky", "variant": 3, "bs": root, "kernel": {"kc": root},
                                            "child": FUSED_CHILD}
    tree = parse_tree(json.dumps(doc))
    lib = _lib.lib()
    a0 = spd_int(47 + n, n)
    try:
        assert lib.bf_set_option(b"fused_diag", fused) == 0
        ref = bf.make_view(n, n, fill=a0)
        bf.cholesky(ref, "lower", tree)
        v = bf.make_view(n, n, fill=a0)
        g = bf.CholeskyGraph(v, "lower", tree)
        for _ in range(2):
            v.copy_from(a0)
            g()
            assert digest(v.to_numpy()) == digest(ref.to_numpy())
        bad = a0.copy()
        bad[n - 300, n - 300] = -1e9
        v.copy_from(bad)
        with pytest.raises(bf.errors.NotPositiveDefiniteError) as e:
            g()
        assert e.value.index == n - 300
    finally:
        lib.bf_set_option(b"fused_diag", 1)
