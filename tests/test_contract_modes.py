"""Permuted contractions on the mode-group TMA path (bf_contract_modes_d):
operand mode groups go straight into TMA-staged tiles through 4-D tensor
maps.  Every path — mode-group TMA, TMA with one operand staged k-contiguous,
the element-gathering GEMM — must give the oracle's bits (the k order is the
reference's on every path: tensor/contract.py:58-83)."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle as O
from golden_inputs import tensor_inputs

pytestmark = pytest.mark.gpu


def _run(spec, dims, seed, fold, stage, kc=256, alpha=1.25, beta=-0.5):
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.engine import KernelConfig
    from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor
    from paper_2604_07311_b200.views import DType

    lhs, lc = spec.split("->")
    la, lb = lhs.split(",")
    ad, bd, cd = [dims[x] for x in la], [dims[x] for x in lb], [dims[x] for x in lc]
    a0, b0, c0 = tensor_inputs(seed, ad, bd, cd)
    ta, tb, tc = make_tensor(ad, fill=a0), make_tensor(bd, fill=b0), make_tensor(cd, fill=c0)
    bf.contract(alpha, ta, tb, beta, tc, ContractionSpec.parse(spec), cfg=KernelConfig(8, 6, 64, kc, 2048, DType.F64,
                                                                                         DType.F64),
                fold=fold, stage=stage)
    got = tc.storage.cpu().numpy()
    ref = np.asarray(c0, dtype=np.float64).reshape(-1).copy()
    O.contract(alpha, np.asarray(a0).reshape(-1).copy(), ad, np.asarray(b0).reshape(-1).copy(), bd, beta, ref, cd,
               spec, kc=kc, fold=fold, nthreads=O.host_threads())
    return got, ref


CASES = [
    ("aibj,cidj->abcd", {"a": 32, "b": 128, "c": 16, "d": 128, "i": 8, "j": 64}),   # both operands TMA, no copy
    ("aibj,cidj->abcd", {"a": 4, "b": 32, "c": 8, "d": 64, "i": 4, "j": 32}),       # inner M/N groups < 128
    ("aibj,cjdi->abcd", {"a": 32, "b": 64, "c": 32, "d": 64, "i": 16, "j": 32}),    # B's k order transposed: staged
    ("ijab,ijcd->abcd", {"a": 64, "b": 64, "c": 32, "d": 64, "i": 4, "j": 16}),     # K slowest (folds)
    ("abij,cdij->acbd", {"a": 16, "b": 128, "c": 8, "d": 256, "i": 8, "j": 32}),    # permuted C
]


@pytest.mark.parametrize("stage", ["auto", "always", "never", "gather"])
@pytest.mark.parametrize("fold", [True, False])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_mode_group_paths_bitwise_vs_oracle(cuda, case, fold, stage):
    spec, dims = case
    got, ref = _run(spec, dims, 61_000 + len(spec), fold, stage)
    assert hashlib.sha256(got.tobytes()).hexdigest() == hashlib.sha256(ref.tobytes()).hexdigest()


def test_mode_group_path_is_taken(cuda):
    """aibj,cidj->abcd runs on the mode-group TMA kernel with no staging copy."""
    import sys

    from paper_2604_07311_b200.engine import _lib

    C = sys.modules["paper_2604_07311_b200.tensor.contract"]  # the package re-exports the function

    calls = {"stage": 0}
    orig = C._stage

    def counting(*a, **k):
        calls["stage"] += 1
        return orig(*a, **k)

    C._stage = counting
    try:
        l0 = _lib.lib().bf_launch_count()
        _run("aibj,cidj->abcd", {"a": 16, "b": 128, "c": 16, "d": 128, "i": 8, "j": 64}, 5, True, "auto")
        assert calls["stage"] == 0
        assert _lib.lib().bf_launch_count() - l0 == 1  # one GEMM launch, nothing else
    finally:
        C._stage = orig


@pytest.mark.parametrize("spec,dims", [("abij,cdij->abcd", {"a": 16, "b": 24, "c": 16, "d": 32, "i": 12, "j": 20}),
                                       ("aibj,cjdi->abcd", {"a": 8, "b": 16, "c": 16, "d": 8, "i": 32, "j": 8})])
def test_bf16_contraction_within_bf16_bound(cuda, spec, dims):
    """precision='bf16' (tcgen05, fp32 accumulation): each product carries at
    most ~2^-8 relative error from the bf16 roundings, so |C - C64| stays under
    2^-7 * (|A| |B|) elementwise (plus the beta*C term exactly in FP64)."""
    import paper_2604_07311_b200 as bf
    from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor

    lhs, lc = spec.split("->")
    la, lb = lhs.split(",")
    ad, bd, cd = [dims[x] for x in la], [dims[x] for x in lb], [dims[x] for x in lc]
    a0, b0, c0 = tensor_inputs(77, ad, bd, cd)
    ta, tb, tc = make_tensor(ad, fill=a0), make_tensor(bd, fill=b0), make_tensor(cd, fill=c0)
    bf.contract(1.5, ta, tb, 0.5, tc, ContractionSpec.parse(spec), precision="bf16")
    got = tc.storage.cpu().numpy().reshape(cd)
    ref = 1.5 * np.einsum(spec, a0, b0) + 0.5 * c0
    bound = 1.5 * np.einsum(spec, np.abs(a0), np.abs(b0)) * 2.0 ** -7
    assert np.all(np.abs(got - ref) <= bound + 1e-12)
    assert np.abs(got - ref).max() > 0  # it really ran in reduced precision
