"""Host-side logic on CPU: views, partitioning, control trees, the C-ABI
library's exports, and the no-fallback guarantee.  Mirrors the reference's
tests/test_views.py and tests/test_control.py for the hot-path API."""
from __future__ import annotations

import ctypes
import json

import numpy as np
import pytest
import torch

import paper_2604_07311_b200 as bf
from paper_2604_07311_b200.control import (
    ControlNode,
    default_tree,
    enumerate_trees,
    flatten_cholesky,
    parse_tree,
    resolve_config,
    tree_descriptor,
    tree_to_json,
    validate,
)
from paper_2604_07311_b200.engine import _lib
from paper_2604_07311_b200.errors import DeviceError, ShapeError, TreeParseError, TreeValidationError  # noqa: F401
from paper_2604_07311_b200.views import DType, Range, make_view, partition_steps, views_overlap

CPU = "cpu"


class TestViews:
    def test_sequence_logical_for_col_major(self):
        v = make_view(2, 3, layout="col-major", fill="sequence", device=CPU)
        assert v.to_numpy().tolist() == [[1, 2, 3], [4, 5, 6]]
        assert (v.rs, v.cs) == (1, 2)

    def test_offset_arithmetic_and_transpose(self):
        v = make_view(6, 7, fill="sequence", device=CPU)
        s = v.subview(Range(2, 3), Range(1, 4))
        assert s.offset == 2 * 7 + 1 and s.shape == (3, 4)
        assert np.array_equal(s.transposed().to_numpy(), s.to_numpy().T)
        assert s.transposed().transposed().to_numpy().tobytes() == s.to_numpy().tobytes()

    def test_out_of_bounds(self):
        with pytest.raises(ShapeError):
            make_view(3, 3, device=CPU).subview(Range(2, 2), Range(0, 1))
        with pytest.raises(ShapeError):
            make_view(-1, 2, device=CPU)

    def test_copy_from_writes_through(self):
        parent = make_view(5, 6, device=CPU)
        sub = parent.subview(Range(1, 2), Range(2, 3))
        sub.copy_from([[1, 2, 3], [4, 5, 6]])
        assert parent.to_numpy()[1:3, 2:5].tolist() == [[1, 2, 3], [4, 5, 6]]

    @pytest.mark.parametrize("n,bs", [(0, 3), (5, 2), (7, 7), (64, 5), (10, 100)])
    def test_partition_r1_tiles_exactly(self, n, bs):
        seen = []
        for st in partition_steps(n, bs):
            assert st.r0.end == st.r1.start and st.r1.end == st.r2.start and st.r2.end == n
            seen.extend(range(st.r1.start, st.r1.end))
        assert seen == list(range(n))

    def test_lookahead_slice(self):
        steps = list(partition_steps(10, 4, lookahead=2))
        assert steps[0].r1b == Range(4, 2) and steps[-1].r1b == Range(10, 0)
        with pytest.raises(ValueError):
            list(partition_steps(4, 0))

    def test_overlap(self):
        v = make_view(8, 8, device=CPU)
        left = v.subview(Range(0, 8), Range(0, 4))
        right = v.subview(Range(0, 8), Range(4, 4))
        assert not views_overlap(left, right)
        assert views_overlap(left, v.subview(Range(2, 2), Range(3, 2)))
        assert views_overlap(v, v.transposed())
        assert not views_overlap(v, make_view(8, 8, device=CPU))

    def test_from_torch_aliases(self):
        t = torch.arange(12, dtype=torch.float64).reshape(3, 4)
        v = bf.from_torch(t[1:, 1:])
        assert v.to_numpy().tolist() == [[5, 6, 7], [9, 10, 11]]
        v.copy_from(np.zeros((2, 3)))
        assert t[1:, 1:].sum().item() == 0.0


class TestControl:
    def test_depth_two_document(self):
        node = parse_tree('{"op":"cholesky","variant":3,"bs":128,"child":{"op":"cholesky","variant":"unblocked1"}}')
        assert node.depth() == 2 and node.child.variant == "unblocked1"

    def test_errors(self):
        with pytest.raises(TreeValidationError) as e:
            parse_tree('{"op":"cholesky","variant":"unblocked1","bs":8}')
        assert any("bs" in p for p, _ in e.value.violations)
        with pytest.raises(TreeParseError) as e2:
            parse_tree('{"op": "cholesky",')
        assert "line 1" in str(e2.value)
        with pytest.raises(TreeValidationError):
            parse_tree('{"op":"cholesky","variant":3,"bs":8,"bogus":1}')
        with pytest.raises(TreeValidationError):
            parse_tree('{"op":"gemm","variant":"blocked","kernel":{"zz":4}}')

    def test_round_trip(self):
        rng = np.random.default_rng(2)
        for _ in range(25):
            node = ControlNode("cholesky", "unblocked2")
            for _ in range(int(rng.integers(0, 3))):
                node = ControlNode("cholesky", int(rng.integers(1, 4)), bs=int(rng.integers(1, 200)),
                                   ways=int(rng.integers(1, 5)),
                                   kernel={"kc": int(rng.integers(8, 64))} if rng.random() < 0.5 else None, child=node)
            assert parse_tree(tree_to_json(node)) == node

    def test_validate(self):
        assert validate(default_tree("cholesky", 500), op="cholesky") == []
        bad = ControlNode("cholesky", 3, bs=8, child=ControlNode("lu", "unblocked"))
        assert any(p.endswith("child.op") for p, _ in validate(bad))
        deep = ControlNode("cholesky", "unblocked3")
        for _ in range(16):
            deep = ControlNode("cholesky", 3, bs=4, child=deep)
        assert any("depth" in r for _, r in validate(deep))

    def test_enumerate_counts(self):
        assert len(list(enumerate_trees("cholesky", [1, 2, 3], [64, 128], depth=1))) == 18
        assert len(list(enumerate_trees("cholesky", [1, 2], [64, 128], depth=2))) == (2 * 2) ** 2 * 3
        assert [t.kernel for t in enumerate_trees("gemm", [], [64, 128])] == [{"kc": 64}, {"kc": 128}]

    def test_defaults_and_descriptor(self):
        assert default_tree("cholesky", 128).variant == "unblocked3"
        t = default_tree("cholesky", 129)
        assert (t.variant, t.bs, t.child.variant) == (3, 128, "unblocked3")
        assert tree_descriptor(t) == "v3:bs128/unblocked3"

    def test_flatten_nests_kc(self):
        doc = {"op": "cholesky", "variant": 2, "bs": 48, "kernel": {"kc": 20},
               "child": {"op": "cholesky", "variant": 1, "bs": 16,
                         "child": {"op": "cholesky", "variant": "unblocked2"}}}
        t = parse_tree(json.dumps(doc))
        assert flatten_cholesky(t, resolve_config(t, DType.F64)) == [(2, 48, 20), (1, 16, 20), (12, 0, 20)]
        t2 = default_tree("cholesky", 1000)
        assert flatten_cholesky(t2, resolve_config(t2, DType.F32)) == [(3, 128, 512), (13, 0, 512)]


class TestLibrary:
    def test_loads_and_exports_every_declared_symbol(self):
        lib = _lib.lib()
        declared = _lib.declared_symbols()
        assert len(declared) >= 18
        for name in declared:
            assert hasattr(lib, name), name
        assert lib.bf_abi_version() == 1

    def test_header_structs_match_ctypes(self):
        assert ctypes.sizeof(_lib.BfView) == 48
        assert ctypes.sizeof(_lib.BfCholLevel) == 24
        assert ctypes.sizeof(_lib.BfScatterView) == 40

    def test_no_cpu_fallback(self):
        a = make_view(4, 4, fill=np.eye(4), device=CPU)
        with pytest.raises(DeviceError):
            bf.cholesky(a)
        with pytest.raises(DeviceError):
            bf.gemm(1.0, make_view(2, 2, device=CPU), make_view(2, 2, device=CPU), 0.0, make_view(2, 2, device=CPU))

    def test_shape_and_alias_checks_before_launch(self):
        with pytest.raises(ShapeError):
            bf.gemm(1.0, make_view(2, 3, device=CPU), make_view(2, 2, device=CPU), 0.0, make_view(2, 2, device=CPU))
        v = make_view(4, 4, fill="sequence", device=CPU)
        with pytest.raises(bf.errors.AliasingError):
            bf.gemm(1.0, v, make_view(4, 4, device=CPU), 0.0, v)
        with pytest.raises(ShapeError):
            bf.gemmt_lower(1.0, make_view(2, 2, device=CPU), make_view(2, 3, device=CPU), 0.0, make_view(2, 3, device=CPU))
        with pytest.raises(ShapeError):
            bf.cholesky(make_view(2, 3, device=CPU))
