"""Golden fixtures for the LU family, from the REFERENCE implementation.

    python tools/gen_golden_lu.py      (build container only: imports /root/reference)

Runs the reference's lu_partial (factor/lu.py:56-130) and its left-lower-unit
TRSM (engine/trsm.py:71-88,114-125) on the seeded inputs of
tests/golden_inputs.py and writes tests/golden/golden_lu.json: per case the
parameters, the SHA-256 of the factored matrix, the pivot vector and the
first exactly-zero pivot column the reference warned about.
"""
from __future__ import annotations

import json
import sys
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "tests"))

from blockfam.control import parse_tree  # noqa: E402
from blockfam.engine import LEFT_LOWER_NOTRANS_UNIT, KernelConfig, trsm  # noqa: E402
from blockfam.errors import SingularFactorWarning  # noqa: E402
from blockfam.factor import lu_partial  # noqa: E402
from blockfam.views import DType, make_view  # noqa: E402

from golden_inputs import digest, left_trsm_inputs, lu_input  # noqa: E402

cases: list[dict] = []


def lu_tree(*levels, kc=None):
    """levels: block sizes root -> leaf parent; e.g. lu_tree(64, 16)."""
    node = {"op": "lu", "variant": "unblocked"}
    for i, bs in enumerate(reversed(levels)):
        node = {"op": "lu", "variant": "blocked", "bs": bs, "child": node}
        if kc is not None and i == len(levels) - 1:
            node["kernel"] = {"kc": kc}
    return node


def run_lu(seed, m, n, kind, dt, doc):
    a0 = lu_input(seed, m, n, kind, dt)
    v = make_view(m, n, DType.parse(dt), fill=a0)
    sing = -1
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        piv = lu_partial(v, parse_tree(json.dumps(doc)) if doc else None)
        for x in w:
            if issubclass(x.category, SingularFactorWarning):
                sing = int(str(x.message).split("column ")[1].split(":")[0])
    out = v.to_numpy()
    cases.append({"id": f"lu{len(cases):03d}", "kind": "lu", "seed": seed, "m": m, "n": n, "input": kind, "dtype": dt,
                  "tree": doc, "sha256": digest(out), "piv": [int(p) for p in piv.piv], "sing": sing})


def run_trsm_left(seed, n, ncols, dt, alpha, kc):
    tri, b = left_trsm_inputs(seed, n, ncols, dt)
    vt = make_view(n, n, DType.parse(dt), fill=tri)
    vb = make_view(n, ncols, DType.parse(dt), fill=b)
    cfg = KernelConfig(mr=8, nr=6, mc=64, kc=kc, nc=2048, dtype=DType.parse(dt), acc_dtype=DType.parse(dt))
    trsm(LEFT_LOWER_NOTRANS_UNIT, alpha, vt, vb, cfg=cfg)
    cases.append({"id": f"lu{len(cases):03d}", "kind": "trsm_left", "seed": seed, "n": n, "ncols": ncols,
                  "dtype": dt, "alpha": alpha, "kc": kc, "sha256": digest(vb.to_numpy())})


def main():
    seed = 50_000
    # the unblocked leaf alone, square / tall / wide, all input kinds
    for dt in ("f64", "f32"):
        for (m, n) in ((1, 1), (5, 5), (37, 37), (64, 40), (40, 64), (100, 100)):
            for kind in ("uniform", "ties", "diag", "zerocol"):
                seed += 1
                run_lu(seed, m, n, kind, dt, {"op": "lu", "variant": "unblocked"})
    # one blocked level over block sizes (reference tests/test_lu.py style)
    for bs in (1, 7, 32, 100):
        for kind in ("uniform", "ties", "zerocol"):
            seed += 1
            run_lu(seed, 100, 100, kind, "f64", lu_tree(bs))
    # nested trees, kc overrides, tall and wide panels, f32
    docs = [
        (lu_tree(48, 16), 150, 150, "uniform", "f64"),
        (lu_tree(64, 16, kc=20), 130, 130, "uniform", "f64"),
        (lu_tree(96, 32), 333, 333, "uniform", "f64"),
        (lu_tree(128, 32), 300, 200, "uniform", "f64"),
        (lu_tree(64, 32), 200, 300, "uniform", "f64"),
        (lu_tree(64, 16), 160, 160, "ties", "f64"),
        (lu_tree(40, 8), 120, 120, "zerocol", "f64"),
        (lu_tree(48, 16), 150, 150, "uniform", "f32"),
        (lu_tree(32), 90, 90, "diag", "f32"),
        (None, 200, 200, "uniform", "f64"),
        (lu_tree(256, 64, 16), 512, 512, "uniform", "f64"),
    ]
    for doc, m, n, kind, dt in docs:
        seed += 1
        run_lu(seed, m, n, kind, dt, doc)
    # the left-lower-unit TRSM alone (base 32, recursion, kc folds, alpha)
    for dt in ("f64", "f32"):
        for n, ncols, alpha, kc in ((1, 3, 1.0, 256), (20, 7, 1.0, 256), (33, 10, -2.5, 256), (100, 64, 1.0, 16),
                                    (150, 200, 0.5, 256), (300, 40, 1.0, 33)):
            seed += 1
            run_trsm_left(seed, n, ncols, dt, alpha, kc)
    out = ROOT / "tests" / "golden" / "golden_lu.json"
    out.write_text(json.dumps({"generator": "tools/gen_golden_lu.py", "reference": "blockfam (/root/reference/pkg)",
                               "cases": cases}, indent=1))
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()
