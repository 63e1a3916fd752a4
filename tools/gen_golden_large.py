"""Golden digests at the HEADLINE configurations, produced by the reference
itself and cross-checked by the oracle.

Run in the build container (where /root/reference exists), e.g.
    nohup python tools/gen_golden_large.py > /tmp/gen_large.log 2>&1 &
It takes about an hour on 8 cores (the n=32768 case dominates: ~18 min for
the reference at ways=8 plus ~27 min for the oracle).

Cases (tests/golden/golden_large.json, consumed by tests/test_headline_parity.py):
  * the bench tree of BASELINE configs[1] (v3 bs=2048 kc=2048 -> v3 bs=128
    kc=128 -> unblocked3) at n = 8192, 16384 and 32768 on spd_int inputs
    (small-integer M, exact in any order, platform independent);
  * the other variants and the upper triangle at n = 8192 (V1, V2, upper);
  * the C5 contraction abij,cdij->abcd (folded) at d = 64 and 128, and the
    permuted aibj,cjdi->abcd at d = 64 (fold on and off).
For every case the reference's output SHA-256 is recorded and the oracle must
reproduce it before the case is written.  The reference runs with the root
node's `ways` = 8 (results are identical for every ways: SPEC.md:180); the
recorded tree omits `ways`.
"""
from __future__ import annotations

import copy
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden" / "golden_large.json"
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "oracle"))

from blockfam.control import parse_tree  # noqa: E402
from blockfam.engine import KernelConfig  # noqa: E402
from blockfam.factor import cholesky  # noqa: E402
from blockfam.tensor import ContractionSpec, contract, make_tensor  # noqa: E402
from blockfam.views import DType, MatrixView  # noqa: E402

import oracle as O  # noqa: E402
from golden_inputs import digest, spd_int, tensor_inputs  # noqa: E402

WAYS = 8
BENCH_TREE = {"op": "cholesky", "variant": 3, "bs": 2048, "kernel": {"kc": 2048},
              "child": {"op": "cholesky", "variant": 3, "bs": 128, "kernel": {"kc": 128},
                        "child": {"op": "cholesky", "variant": "unblocked3"}}}


def two_level(variant: int, bs: int = 2048, inner: int = 128) -> dict:
    t = copy.deepcopy(BENCH_TREE)
    t["variant"], t["bs"], t["kernel"]["kc"] = variant, bs, bs
    t["child"]["bs"], t["child"]["kernel"]["kc"] = inner, inner
    return t


def load() -> dict:
    if OUT.exists():
        return json.loads(OUT.read_text())
    return {"generator": "tools/gen_golden_large.py", "cases": []}


def save(doc: dict) -> None:
    OUT.write_text(json.dumps(doc, indent=1) + "\n")


def have(doc: dict, cid: str) -> bool:
    return any(c["id"] == cid for c in doc["cases"])


def run_chol(doc: dict, cid: str, n: int, seed: int, tree: dict, uplo: str = "lower") -> None:
    if have(doc, cid):
        return
    a0 = spd_int(seed, n)
    in_sha = digest(a0)
    # reference
    st = a0.reshape(-1).copy()
    ref_tree = dict(tree, ways=WAYS)
    t0 = time.time()
    cholesky(MatrixView(storage=st, offset=0, m=n, n=n, rs=n, cs=1, dtype=DType.F64), uplo,
             parse_tree(json.dumps(ref_tree)))
    t_ref = time.time() - t0
    ref_sha = digest(st)
    del st
    print(f"{cid}: reference {t_ref:.1f} s {ref_sha[:16]}", flush=True)
    # oracle cross-check
    st = a0.reshape(-1).copy()
    del a0
    t0 = time.time()
    bad = O.cholesky(st, {"off": 0, "m": n, "n": n, "rs": n, "cs": 1}, O.levels_from_tree(tree, n, "f64"),
                     uplo=uplo, nthreads=O.host_threads())
    t_orc = time.time() - t0
    orc_sha = digest(st)
    print(f"{cid}: oracle {t_orc:.1f} s {orc_sha[:16]}", flush=True)
    assert bad < 0 and orc_sha == ref_sha, f"{cid}: oracle disagrees with the reference"
    doc["cases"].append({"id": cid, "kind": "chol", "input": "spd_int", "seed": seed, "n": n, "dtype": "f64",
                         "uplo": uplo, "tree": tree, "error": None, "input_sha256": in_sha,
                         "a_out": {"sha256": ref_sha, "size": n * n},
                         "ref_seconds_ways8": round(t_ref, 1), "oracle_seconds": round(t_orc, 1)})
    save(doc)


def run_contract(doc: dict, cid: str, spec_text: str, d: int, fold: bool, seed: int, kc: int = 256) -> None:
    if have(doc, cid):
        return
    spec = ContractionSpec.parse(spec_text)
    dims = {l: d for l in set(spec_text) if l.isalpha()}
    ad = [dims[l] for l in spec.labels_a]
    bd = [dims[l] for l in spec.labels_b]
    cd = [dims[l] for l in spec.labels_c]
    a0, b0, c0 = tensor_inputs(seed, ad, bd, cd)
    alpha, beta = 1.0, 0.0
    a, b, c = make_tensor(ad, fill=a0), make_tensor(bd, fill=b0), make_tensor(cd, fill=c0)
    cfg = KernelConfig(mr=8, nr=6, mc=64, kc=kc, nc=2048, dtype=DType.F64, acc_dtype=DType.F64)
    t0 = time.time()
    contract(alpha, a, b, beta, c, spec, cfg=cfg, ways=WAYS, fold=fold)
    t_ref = time.time() - t0
    ref_sha = digest(c.storage)
    del a, b, c
    print(f"{cid}: reference {t_ref:.1f} s {ref_sha[:16]}", flush=True)
    cst = np.asarray(c0, dtype=np.float64).reshape(-1).copy()
    t0 = time.time()
    O.contract(alpha, np.asarray(a0).reshape(-1).copy(), ad, np.asarray(b0).reshape(-1).copy(), bd, beta, cst, cd,
               spec_text, kc=kc, fold=fold, nthreads=O.host_threads())
    t_orc = time.time() - t0
    orc_sha = digest(cst)
    print(f"{cid}: oracle {t_orc:.1f} s {orc_sha[:16]}", flush=True)
    assert orc_sha == ref_sha, f"{cid}: oracle disagrees with the reference"
    doc["cases"].append({"id": cid, "kind": "contract", "spec": spec_text, "dims": dims, "fold": fold, "kc": kc,
                         "alpha": alpha, "beta": beta, "seed": seed, "c_out": {"sha256": ref_sha, "size": int(cst.size)},
                         "ref_seconds_ways8": round(t_ref, 1), "oracle_seconds": round(t_orc, 1)})
    save(doc)


def main(which: list[str]) -> None:
    doc = load()
    plan = [
        ("L8192", lambda: run_chol(doc, "L8192", 8192, 70_001, BENCH_TREE)),
        ("K64f", lambda: run_contract(doc, "K64f", "abij,cdij->abcd", 64, True, 71_001)),
        ("K64p", lambda: run_contract(doc, "K64p", "aibj,cjdi->abcd", 64, True, 71_002)),
        ("K64u", lambda: run_contract(doc, "K64u", "aibj,cjdi->abcd", 64, False, 71_003)),
        ("V1_8192", lambda: run_chol(doc, "V1_8192", 8192, 70_002, two_level(1))),
        ("V2_8192", lambda: run_chol(doc, "V2_8192", 8192, 70_003, two_level(2))),
        ("U8192", lambda: run_chol(doc, "U8192", 8192, 70_004, BENCH_TREE, "upper")),
        ("L16384", lambda: run_chol(doc, "L16384", 16384, 70_005, BENCH_TREE)),
        ("L32768", lambda: run_chol(doc, "L32768", 32768, 70_006, BENCH_TREE)),
        ("K128f", lambda: run_contract(doc, "K128f", "abij,cdij->abcd", 128, True, 71_004)),
    ]
    for name, fn in plan:
        if not which or name in which:
            fn()


if __name__ == "__main__":
    main(sys.argv[1:])
