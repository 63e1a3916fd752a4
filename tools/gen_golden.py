"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    python tools/gen_golden.py
It imports the reference package `blockfam` from /root/reference/pkg/src,
runs its hot-path entry points on inputs from tests/golden_inputs.py (seeded,
platform independent) and writes tests/golden/golden.json: per case the
parameters, the input seed, the SHA-256 of every output buffer and, for
small cases, the output values themselves.  The tests regenerate the inputs,
run the oracle (CPU) or the CUDA path (GPU) and compare digests, i.e. they
demand bit-identical results.  Nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT / "tests"))

from blockfam.control import ControlNode, parse_tree, serialize_tree  # noqa: E402
from blockfam.engine import RIGHT_LOWER_TRANS_NONUNIT, KernelConfig, gemm, gemmt_lower, syrk_lower, trsm  # noqa: E402
from blockfam.errors import NotPositiveDefiniteError, SingularMatrixError  # noqa: E402
from blockfam.factor import cholesky  # noqa: E402
from blockfam.oracle import gemm_naive  # noqa: E402
from blockfam.tensor import ContractionSpec, contract, make_tensor  # noqa: E402
from blockfam.views import DType, MatrixView, make_view  # noqa: E402

from golden_inputs import digest, gemm_inputs, spd_float, spd_int, tensor_inputs, trsm_inputs  # noqa: E402

cases: list[dict] = []
SMALL = 64  # outputs with at most this many elements are stored inline


def add(kind: str, **params) -> None:
    params = {"id": f"c{len(cases):03d}", "kind": kind, **params}
    cases.append(params)


def ref_view(storage: np.ndarray, meta: dict, dt: DType) -> MatrixView:
    return MatrixView(storage=storage, offset=meta["off"], m=meta["m"], n=meta["n"], rs=meta["rs"], cs=meta["cs"], dtype=dt)


def out_record(arr: np.ndarray) -> dict:
    rec = {"sha256": digest(arr), "size": int(arr.size)}
    if arr.size <= SMALL:
        rec["values"] = [float(x) for x in arr.reshape(-1)]
    return rec


def gen_gemm():
    shapes = [(1, 1, 1), (2, 3, 4), (9, 7, 5), (33, 17, 40), (65, 49, 33), (40, 40, 300), (130, 70, 600)]
    kinds = ("contiguous", "transposed", "padded")
    seed = 10_000
    for dt, acc in (("f64", "f64"), ("f32", "f32"), ("f32", "f64")):
        for op in ("gemm", "gemmt", "syrk"):
            for kc in (256, 8, 7, 64):
                for m, n, k in shapes:
                    seed += 1
                    kk = (kinds[seed % 3], kinds[(seed + 1) % 3], kinds[(seed + 2) % 3])
                    (ast, am), b, (cst, cm) = gemm_inputs(seed, op, dt, m, n, k, kk)
                    rng = np.random.default_rng(seed + 7)
                    alpha = float(rng.choice([1.0, -1.0, 1.25, 0.3]))
                    beta = float(rng.choice([0.0, 1.0, -0.5]))
                    D = DType.parse(dt)
                    cfg = KernelConfig(mr=8, nr=6, mc=64, kc=kc, nc=2048, dtype=D, acc_dtype=DType.parse(acc))
                    a = ref_view(ast.copy(), am, D)
                    c = ref_view(cst.copy(), cm, D)
                    if op == "gemm":
                        gemm(alpha, a, ref_view(b[0].copy(), b[1], D), beta, c, cfg=cfg)
                    elif op == "gemmt":
                        gemmt_lower(alpha, a, ref_view(b[0].copy(), b[1], D), beta, c, cfg=cfg)
                    else:
                        syrk_lower(alpha, a, beta, c, cfg=cfg)
                    add("gemm", op=op, dtype=dt, acc=acc, kc=kc, alpha=alpha, beta=beta, seed=seed, shape=[m, n, k],
                        kinds=list(kk), c_out=out_record(c.storage))
    # hand examples (reference tests/test_engine_gemm.py:87-92, 176-183, 153-160)
    add("hand_gemm", name="gemm_2x2", expect=[[19.0, 22.0], [43.0, 50.0]])
    cfg = KernelConfig(mr=4, nr=4, mc=8, kc=8, nc=8, dtype=DType.F32, acc_dtype=DType.F64)
    a = make_view(1, 3, DType.F32, fill=[[1e8, 1.0, -1e8]])
    b = make_view(3, 1, DType.F32, fill=[[1.0], [1.0], [1.0]])
    c = make_view(1, 1, DType.F32)
    gemm(1.0, a, b, 0.0, c, cfg=cfg)
    add("hand_gemm", name="mixed_1e8", expect=[[float(c.item(0, 0))]])


def gen_naive():
    for seed, (m, n, k) in ((20_001, (5, 4, 3)), (20_002, (17, 9, 31))):
        (ast, am), (bst, bm), (cst, cm) = gemm_inputs(seed, "gemm", "f64", m, n, k, ("contiguous",) * 3)
        c = ref_view(cst.copy(), cm, DType.F64)
        gemm_naive(1.5, ref_view(ast, am, DType.F64), ref_view(bst, bm, DType.F64), -0.25, c)
        add("gemm_naive", seed=seed, shape=[m, n, k], alpha=1.5, beta=-0.25, c_out=out_record(c.storage))


def run_chol(kind: str, a0: np.ndarray, dt: str, tree_doc, uplo: str, **extra):
    D = DType.parse(dt)
    a = make_view(a0.shape[0], a0.shape[0], D, fill=a0)
    tree = parse_tree(json.dumps(tree_doc)) if tree_doc is not None else None
    err = None
    try:
        cholesky(a, uplo, tree)
    except NotPositiveDefiniteError as e:
        err = e.index
    add("chol", input=kind, dtype=dt, uplo=uplo, tree=tree_doc, n=int(a0.shape[0]), error=err,
        a_out=out_record(a.storage), **extra)


def tree_doc(variant, bs, leaf="unblocked3", kc=None):
    node = ControlNode("cholesky", variant, bs=bs, kernel={"kc": kc} if kc else None, child=ControlNode("cholesky", leaf))
    return serialize_tree(node)


def gen_chol():
    # leaves alone
    seed = 30_000
    for dt in ("f64", "f32"):
        for n in (1, 2, 5, 37, 64, 100):
            for leaf in ("unblocked1", "unblocked2", "unblocked3"):
                seed += 1
                run_chol("spd_int", spd_int(seed, n, dt), dt, {"op": "cholesky", "variant": leaf}, "lower", seed=seed)
    # the family: 3 variants x block sizes (reference tests/test_cholesky.py:52-63)
    for variant in (1, 2, 3):
        for bs in (1, 7, 32, 100):
            seed += 1
            run_chol("spd_int", spd_int(seed, 100), "f64", tree_doc(variant, bs), "lower", seed=seed)
    for leaf in ("unblocked1", "unblocked2", "unblocked3"):
        seed += 1
        run_chol("spd_int", spd_int(seed, 64), "f64", tree_doc(3, 16, leaf), "lower", seed=seed)
    docs = [
        ({"op": "cholesky", "variant": 2, "bs": 48, "kernel": {"kc": 20},
          "child": {"op": "cholesky", "variant": 1, "bs": 16, "kernel": {"kc": 8},
                    "child": {"op": "cholesky", "variant": "unblocked2"}}}, 150, "f64", "lower"),
        (tree_doc(3, 16), 75, "f64", "upper"),
        (tree_doc(3, 16), 75, "f64", "lower"),
        (tree_doc(3, 16), 60, "f32", "lower"),
        (tree_doc(1, 24, "unblocked1"), 90, "f32", "lower"),
        (tree_doc(2, 24, "unblocked2"), 90, "f32", "lower"),
        (None, 200, "f64", "lower"),
        (tree_doc(3, 512), 300, "f64", "lower"),
        (tree_doc(3, 64, kc=64), 256, "f64", "lower"),
        ({"op": "cholesky", "variant": 3, "bs": 96, "kernel": {"kc": 96},
          "child": {"op": "cholesky", "variant": 3, "bs": 32,
                    "child": {"op": "cholesky", "variant": "unblocked3"}}}, 333, "f64", "lower"),
        (tree_doc(2, 64, kc=128), 256, "f64", "upper"),
        (tree_doc(1, 40), 130, "f64", "lower"),
    ]
    for doc, n, dt, uplo in docs:
        seed += 1
        run_chol("spd_int", spd_int(seed, n, dt), dt, doc, uplo, seed=seed)
    # not positive definite -> global index 7 (tests/test_cholesky.py:43-49)
    seed += 1
    a0 = spd_int(seed, 12)
    a0[7, 7] = -50.0
    run_chol("spd_int_npd7", a0, "f64", tree_doc(3, 4), "lower", seed=seed)
    seed += 1
    a0 = spd_int(seed, 40)
    a0[33, 33] = float("nan")
    run_chol("spd_int_nan33", a0, "f64", tree_doc(2, 8), "lower", seed=seed)
    # hand example [[4,2],[2,5]] -> [[2,2],[1,2]]
    add("hand_chol", expect=[[2.0, 2.0], [1.0, 2.0]])


def gen_trsm():
    seed = 40_000
    for dt in ("f64", "f32"):
        for n, m, alpha, kc in [(2, 1, 1.0, 256), (5, 3, 1.5, 256), (33, 10, 1.5, 256), (70, 64, 1.5, 8),
                                (129, 40, -0.75, 256), (100, 77, 1.0, 7), (256, 300, 1.0, 256)]:
            seed += 1
            tn, b0 = trsm_inputs(seed, dt, n, m)
            D = DType.parse(dt)
            tri = make_view(n, n, D, fill=tn)
            b = make_view(m, n, D, fill=b0)
            cfg = KernelConfig(mr=8, nr=6, mc=64, kc=kc, nc=2048, dtype=D, acc_dtype=D)
            trsm(RIGHT_LOWER_TRANS_NONUNIT, alpha, tri, b, cfg=cfg)
            add("trsm", dtype=dt, n=n, m=m, alpha=alpha, kc=kc, seed=seed, b_out=out_record(b.storage))
    tri = make_view(2, 2, fill=[[1, 0], [1, 0]])
    b = make_view(1, 2, fill=[[1, 1]])
    try:
        trsm(RIGHT_LOWER_TRANS_NONUNIT, 1.0, tri, b)
        err = None
    except SingularMatrixError as e:
        err = e.index
    add("hand_trsm_singular", error=err, b_out=out_record(b.storage))


def gen_contract():
    specs = [
        ("abij,cdij->abcd", {"a": 5, "b": 4, "c": 3, "d": 6, "i": 4, "j": 5}),
        ("aibj,cjdi->abcd", {"a": 4, "b": 5, "c": 3, "d": 4, "i": 3, "j": 6}),
        ("ik,kj->ij", {"i": 7, "j": 9, "k": 5}),
        ("abc,cd->abd", {"a": 4, "b": 5, "c": 6, "d": 3}),
        ("ij,j->i", {"i": 6, "j": 7}),
        ("a,b->ab", {"a": 5, "b": 4}),
        ("ab,ab->", {"a": 5, "b": 6}),
        ("abij,cdij->abcd", {"a": 12, "b": 12, "c": 12, "d": 12, "i": 12, "j": 12}),
    ]
    seed = 50_000
    for text, dims in specs:
        spec = ContractionSpec.parse(text)
        ad = [dims[l] for l in spec.labels_a]
        bd = [dims[l] for l in spec.labels_b]
        cd = [dims[l] for l in spec.labels_c]
        for fold in (True, False):
            for kc in (256, 5):
                seed += 1
                a0, b0, c0 = tensor_inputs(seed, ad, bd, cd)
                a, b, c = make_tensor(ad, fill=a0), make_tensor(bd, fill=b0), make_tensor(cd, fill=c0)
                cfg = KernelConfig(mr=8, nr=6, mc=64, kc=kc, nc=2048, dtype=DType.F64, acc_dtype=DType.F64)
                contract(1.7, a, b, -0.3, c, spec, cfg=cfg, fold=fold)
                add("contract", spec=text, dims=dims, fold=fold, kc=kc, alpha=1.7, beta=-0.3, seed=seed,
                    c_out=out_record(c.storage))


def gen_c1():
    """Config C1 (BASELINE.json configs[0]) through the reference CLI generator
    (cli.py:55-64): n=1024, seed 42, v3/bs128 -> unblocked3.  Its input bits
    depend on the host BLAS (M @ M.T), so the input digest is recorded too."""
    from blockfam.cli import gen_matrix

    a0 = gen_matrix("cholesky", 1024, 1024, 1024, DType.F64, 42)["a"]
    run_chol("cli_gen_matrix_seed42", a0, "f64", tree_doc(3, 128), "lower", input_sha256=digest(a0))
    a1 = spd_float(7, 512)
    run_chol("spd_float_seed7", a1, "f64", tree_doc(3, 128), "lower", input_sha256=digest(a1))


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    gen_gemm()
    gen_naive()
    gen_chol()
    gen_trsm()
    gen_contract()
    gen_c1()
    doc = {"generator": "tools/gen_golden.py", "reference": str(REF), "inputs": "tests/golden_inputs.py", "cases": cases}
    (OUT / "golden.json").write_text(json.dumps(doc, indent=0))
    print(f"{len(cases)} cases")
