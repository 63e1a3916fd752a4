"""Golden fixtures for the skew family, from the
REFERENCE implementation (build container only: imports /root/reference).

    python tools/gen_golden_ltlt.py

sandwich_skew (engine/gemm.py:245-280): digests of lower(C) after the fused
product — bitwise targets.  ltlt_pivoted unblocked (factor/ltlt.py:157-182,
compiled scalar loops): digests of the factor and T, pivots — bitwise.
ltlt_pivoted blocked (its in-panel column updates are NumPy/BLAS products):
pivots and T values stored for tolerance checks.  pfaffian values.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "tests"))

from blockfam.control import ControlNode  # noqa: E402
from blockfam.engine import KernelConfig, sandwich_skew  # noqa: E402
from blockfam.factor import ltlt_pivoted, pfaffian  # noqa: E402
from blockfam.views import DType, make_view  # noqa: E402

from golden_inputs import digest, sandwich_inputs, skew_input  # noqa: E402

cases: list[dict] = []


def add(**kw):
    cases.append({"id": f"sk{len(cases):03d}", **kw})


def main():
    seed = 70_000
    for dt in ("f64", "f32"):
        for n, k, kc in ((1, 1, 256), (2, 2, 256), (8, 6, 256), (31, 17, 256), (64, 40, 16), (100, 257, 256),
                         (130, 129, 64), (200, 33, 256)):
            seed += 1
            c0, a, t = sandwich_inputs(seed, n, k, dt)
            c = make_view(n, n, DType.parse(dt), fill=c0)
            av = make_view(n, k, DType.parse(dt), fill=a)
            cfg = KernelConfig(mr=8, nr=6, mc=64, kc=kc, nc=2048, dtype=DType.parse(dt), acc_dtype=DType.parse(dt))
            sandwich_skew(c, av, t, cfg=cfg)
            add(kind="sandwich", seed=seed, n=n, k=k, kc=kc, dtype=dt, sha256=digest(c.to_numpy()))
    for dt in ("f64", "f32"):
        for n, kind in ((2, "uniform"), (3, "uniform"), (10, "uniform"), (33, "uniform"), (64, "ties"), (100, "uniform")):
            seed += 1
            x0 = skew_input(seed, n, kind, dt)
            v = make_view(n, n, DType.parse(dt), fill=x0)
            piv, tri = ltlt_pivoted(v, ControlNode("ltlt", "unblocked"))
            add(kind="ltlt_unblocked", seed=seed, n=n, input=kind, dtype=dt, sha256=digest(v.to_numpy()),
                t_sha256=digest(np.asarray(tri.t)), piv=[int(p) for p in piv.piv])
    for n, bs in ((40, 8), (100, 16), (130, 32), (257, 64)):
        seed += 1
        x0 = skew_input(seed, n)
        v = make_view(n, n, fill=x0)
        piv, tri = ltlt_pivoted(v, ControlNode("ltlt", "blocked", bs=bs, child=ControlNode("ltlt", "unblocked")))
        add(kind="ltlt_blocked", seed=seed, n=n, bs=bs, dtype="f64", piv=[int(p) for p in piv.piv],
            t=[float(x) for x in tri.t])
    for n in (2, 4, 10, 31, 64):
        seed += 1
        x0 = skew_input(seed, n)
        add(kind="pfaffian", seed=seed, n=n, value=float(pfaffian(make_view(n, n, fill=x0))))
    out = ROOT / "tests" / "golden" / "golden_ltlt.json"
    out.write_text(json.dumps({"generator": "tools/gen_golden_ltlt.py", "reference": "blockfam (/root/reference/pkg)",
                               "cases": cases}, indent=1))
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()
