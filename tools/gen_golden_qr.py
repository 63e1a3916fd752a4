"""Golden fixtures for Householder QR from the
REFERENCE implementation (build container only).  The reference's panel
operations are NumPy/BLAS products, so these are value fixtures for
tolerance comparisons: the factored matrix (R and reflectors) and taus.

    python tools/gen_golden_qr.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
from blockfam.control import ControlNode  # noqa: E402
from blockfam.factor import qr_householder  # noqa: E402
from blockfam.views import DType, make_view  # noqa: E402

cases = []
seed = 90_000
for m, n, bs, dt in ((2, 1, None, "f64"), (4, 4, None, "f64"), (30, 20, None, "f64"), (50, 50, 16, "f64"),
                     (80, 60, 24, "f64"), (64, 64, 8, "f32"), (120, 40, None, "f32")):
    seed += 1
    rng = np.random.default_rng(seed)
    a0 = rng.uniform(-1, 1, (m, n)).astype(np.float64 if dt == "f64" else np.float32)
    v = make_view(m, n, DType.parse(dt), fill=a0)
    tree = ControlNode("qr", "unblocked") if bs is None else ControlNode("qr", "blocked", bs=bs,
                                                                          child=ControlNode("qr", "unblocked"))
    refl = qr_householder(v, tree)
    cases.append({"id": f"qr{len(cases):02d}", "seed": seed, "m": m, "n": n, "bs": bs, "dtype": dt,
                  "factored": [float(x) for x in v.to_numpy().reshape(-1)], "taus": [float(x) for x in refl.taus]})
out = ROOT / "tests" / "golden" / "golden_qr.json"
out.write_text(json.dumps({"generator": "tools/gen_golden_qr.py", "cases": cases}))
print(f"wrote {len(cases)} cases to {out}")
