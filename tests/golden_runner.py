"""Replay golden cases (tests/golden/golden.json) through an implementation.

`run_case(case, impl)` regenerates the case's inputs (tests/golden_inputs.py),
executes it through `impl` ("oracle" = the CPU restatement, "cuda" = the
product package on the GPU) and returns {output name: ndarray} plus the error
index, so the caller can compare SHA-256 digests with the reference's.
"""
from __future__ import annotations

import numpy as np

from golden_inputs import NP, digest, gemm_inputs, spd_float, spd_int, tensor_inputs, trsm_inputs


def chol_input(case: dict) -> np.ndarray | None:
    kind, n, dt = case["input"], case["n"], case["dtype"]
    if kind == "spd_int":
        return spd_int(case["seed"], n, dt)
    if kind == "spd_int_npd7":
        a = spd_int(case["seed"], n, dt)
        a[7, 7] = -50.0
        return a
    if kind == "spd_int_nan33":
        a = spd_int(case["seed"], n, dt)
        a[33, 33] = float("nan")
        return a
    if kind == "cli_gen_matrix_seed42":  # cli.py:55-64 with seed 42
        rng = np.random.default_rng(42)
        m = rng.uniform(-1, 1, (n, n))
        a = m @ m.T + n * np.eye(n)
    elif kind == "spd_float_seed7":
        a = spd_float(7, n)
    else:
        raise KeyError(kind)
    if digest(a) != case["input_sha256"]:
        return None  # host BLAS formed M @ M.T with different bits than the reference host
    return a


def run_case(case: dict, impl: str) -> tuple[dict, object]:
    kind = case["kind"]
    if impl == "oracle":
        import oracle as O
    else:
        import torch

        import paper_2604_07311_b200 as bf
        from paper_2604_07311_b200.engine import KernelConfig
        from paper_2604_07311_b200.views import DType, MatrixView

        dev = torch.device("cuda")

        def dview(storage: np.ndarray, meta: dict):
            t = torch.as_tensor(storage).to(dev)
            return MatrixView(t, meta["off"], meta["m"], meta["n"], meta["rs"], meta["cs"], DType.parse(
                "f64" if storage.dtype == np.float64 else "f32"))

    if kind == "gemm":
        m, n, k = case["shape"]
        op, dt = case["op"], case["dtype"]
        a, b, c = gemm_inputs(case["seed"], op, dt, m, n, k, tuple(case["kinds"]))
        if impl == "oracle":
            cst = c[0].copy()
            if op == "syrk":
                O.syrk(case["alpha"], a, case["beta"], (cst, c[1]), kc=case["kc"], acc=case["acc"])
            else:
                O.gemm(case["alpha"], a, b, case["beta"], (cst, c[1]), kc=case["kc"], lower_only=(op == "gemmt"),
                       acc=case["acc"])
            return {"c_out": cst}, None
        cfg = KernelConfig(8, 6, 64, case["kc"], 2048, DType.parse(dt), DType.parse(case["acc"]))
        va, vc = dview(*a), dview(*c)
        if op == "gemm":
            bf.gemm(case["alpha"], va, dview(*b), case["beta"], vc, cfg=cfg)
        elif op == "gemmt":
            bf.gemmt_lower(case["alpha"], va, dview(*b), case["beta"], vc, cfg=cfg)
        else:
            bf.syrk_lower(case["alpha"], va, case["beta"], vc, cfg=cfg)
        return {"c_out": vc.storage.cpu().numpy()}, None

    if kind == "gemm_naive":
        m, n, k = case["shape"]
        a, b, c = gemm_inputs(case["seed"], "gemm", "f64", m, n, k, ("contiguous",) * 3)
        cst = c[0].copy()
        if impl != "oracle":
            raise NotImplementedError("gemm_naive is an oracle-only routine")
        O.gemm_naive(case["alpha"], a, b, case["beta"], (cst, c[1]))
        return {"c_out": cst}, None

    if kind == "chol":
        a0 = chol_input(case)
        if a0 is None:
            return None, "input-mismatch"
        n, dt = case["n"], case["dtype"]
        st = np.ascontiguousarray(a0, dtype=NP[dt]).reshape(-1).copy()
        meta = {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}
        if impl == "oracle":
            bad = O.cholesky(st, meta, O.levels_from_tree(case["tree"], n, dt), uplo=case["uplo"])
            return {"a_out": st}, (bad if bad >= 0 else None)
        va = dview(st, meta)
        tree = bf.control.parse_tree_dict(case["tree"]) if case["tree"] is not None else None
        err = None
        try:
            bf.cholesky(va, case["uplo"], tree, engine=case.get("engine", "native"))
        except bf.errors.NotPositiveDefiniteError as e:
            err = e.index
        return {"a_out": va.storage.cpu().numpy()}, err

    if kind == "trsm":
        n, m, dt = case["n"], case["m"], case["dtype"]
        tn, b0 = trsm_inputs(case["seed"], dt, n, m)
        tst, bst = tn.reshape(-1).copy(), b0.reshape(-1).copy()
        tm = {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}
        bm = {"off": 0, "m": m, "n": n, "rs": n, "cs": 1}
        if impl == "oracle":
            bad = O.trsm_rltn(case["alpha"], (tst, tm), (bst, bm), kc=case["kc"])
            return {"b_out": bst}, (bad if bad >= 0 else None)
        cfg = KernelConfig(8, 6, 64, case["kc"], 2048, DType.parse(dt), DType.parse(dt))
        vb = dview(bst, bm)
        bf.trsm(bf.engine.RIGHT_LOWER_TRANS_NONUNIT, case["alpha"], dview(tst, tm), vb, cfg=cfg)
        return {"b_out": vb.storage.cpu().numpy()}, None

    if kind == "contract":
        from golden_inputs import NP as _NP  # noqa: F401

        lhs, lc = case["spec"].split("->")
        la, lb = lhs.split(",")
        dims = case["dims"]
        ad, bd, cd = [dims[l] for l in la], [dims[l] for l in lb], [dims[l] for l in lc]
        a0, b0, c0 = tensor_inputs(case["seed"], ad, bd, cd)
        ast, bst, cst = (np.asarray(x, dtype=np.float64).reshape(-1).copy() for x in (a0, b0, c0))
        if impl == "oracle":
            O.contract(case["alpha"], ast, ad, bst, bd, case["beta"], cst, cd, case["spec"], kc=case["kc"],
                       fold=case["fold"])
            return {"c_out": cst}, None
        from paper_2604_07311_b200.tensor import ContractionSpec, make_tensor

        ta, tb, tc = make_tensor(ad, fill=a0), make_tensor(bd, fill=b0), make_tensor(cd, fill=c0)
        cfg = KernelConfig(8, 6, 64, case["kc"], 2048, DType.F64, DType.F64)
        bf.contract(case["alpha"], ta, tb, case["beta"], tc, ContractionSpec.parse(case["spec"]), cfg=cfg,
                    fold=case["fold"])
        return {"c_out": tc.storage.cpu().numpy()}, None

    raise KeyError(kind)
