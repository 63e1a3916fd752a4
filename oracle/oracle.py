"""ORACLE (test infrastructure) — ctypes front end of the CPU restatement in
oracle/blockfam_oracle.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline and
--impl reference legs) may use this module, as the checker or as the timed
CPU baseline.  It never imports the product package: control-tree handling
is restated here from the reference (control.py:287-291,
factor/cholesky.py:115,154-158) so the checker stays independent.

Parity pinned: tests/test_oracle_golden.py demands bit-identical agreement
with the reference's own outputs (tests/golden/golden.json).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

_lib: Optional[ctypes.CDLL] = None


class _ViewD(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("off", ctypes.c_int64), ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("rs", ctypes.c_int64), ("cs", ctypes.c_int64)]


class _Level(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("pad_", ctypes.c_int32), ("bs", ctypes.c_int64), ("kc", ctypes.c_int64)]


def build() -> Path:
    """Compile the oracle (make) if it is missing or stale."""
    src = HERE / "blockfam_oracle.cpp"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(LIB))
        P = ctypes.POINTER(_ViewD)
        for name in ("orc_gemm_d", "orc_gemm_s", "orc_gemm_sd"):
            fn = getattr(_lib, name)
            fn.argtypes = [ctypes.c_double, P, P, ctypes.c_double, P, ctypes.c_int, ctypes.c_int64, ctypes.c_int]
            fn.restype = ctypes.c_int
        for name in ("orc_potrf_leaf_d", "orc_potrf_leaf_s"):
            getattr(_lib, name).argtypes = [P, ctypes.c_int]
            getattr(_lib, name).restype = ctypes.c_int
        for name in ("orc_trsm_rltn_d", "orc_trsm_rltn_s"):
            getattr(_lib, name).argtypes = [ctypes.c_double, P, P, ctypes.c_int64, ctypes.c_int]
            getattr(_lib, name).restype = ctypes.c_int
        for name in ("orc_cholesky_d", "orc_cholesky_s"):
            getattr(_lib, name).argtypes = [P, ctypes.POINTER(_Level), ctypes.c_int, ctypes.c_int]
            getattr(_lib, name).restype = ctypes.c_int64
        for name in ("orc_lu_d", "orc_lu_s"):
            getattr(_lib, name).argtypes = [P, ctypes.POINTER(_Level), ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
            getattr(_lib, name).restype = ctypes.c_int64
        for name in ("orc_trsm_llnu_d", "orc_trsm_llnu_s"):
            getattr(_lib, name).argtypes = [ctypes.c_double, P, P, ctypes.c_int64, ctypes.c_int]
            getattr(_lib, name).restype = None
        for name in ("orc_sandwich_d", "orc_sandwich_s"):
            getattr(_lib, name).argtypes = [P, P, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
            getattr(_lib, name).restype = None
        for name in ("orc_ltlt_unblocked_d", "orc_ltlt_unblocked_s"):
            getattr(_lib, name).argtypes = [P, ctypes.c_void_p, ctypes.c_void_p]
            getattr(_lib, name).restype = None
        _lib.orc_gemm_naive_d.argtypes = [ctypes.c_double, P, P, ctypes.c_double, P]
        _lib.orc_gemm_naive_d.restype = None
        VP, L = ctypes.c_void_p, ctypes.c_int64
        _lib.orc_gemm_scatter_d.argtypes = [ctypes.c_double, VP, VP, VP, VP, VP, VP, ctypes.c_double, VP, VP, VP,
                                            L, L, L, L, ctypes.c_int]
        _lib.orc_gemm_scatter_d.restype = ctypes.c_int
    return _lib


def _suffix(storage: np.ndarray) -> str:
    if storage.dtype == np.float64:
        return "d"
    if storage.dtype == np.float32:
        return "s"
    raise TypeError(storage.dtype)


def _view(storage: np.ndarray, meta: dict) -> _ViewD:
    assert storage.flags.c_contiguous and storage.ndim == 1
    return _ViewD(storage.ctypes.data, meta["off"], meta["m"], meta["n"], meta["rs"], meta["cs"])


def transposed(meta: dict) -> dict:
    return {"off": meta["off"], "m": meta["n"], "n": meta["m"], "rs": meta["cs"], "cs": meta["rs"]}


def gemm(alpha, a, b, beta, c, *, kc: int, lower_only: bool = False, acc: Optional[str] = None, nthreads: int = 1):
    """c := beta*c + alpha*a*b in place; a/b/c are (storage, meta) pairs."""
    sfx = _suffix(c[0])
    if sfx == "s" and acc == "f64":
        sfx = "sd"
    rc = getattr(lib(), "orc_gemm_" + sfx)(alpha, _view(*a), _view(*b), beta, _view(*c), int(lower_only), kc, nthreads)
    if rc:
        raise ValueError("oracle gemm: dims mismatch")


def syrk(alpha, a, beta, c, *, kc: int, acc: Optional[str] = None, nthreads: int = 1):
    gemm(alpha, a, (a[0], transposed(a[1])), beta, c, kc=kc, lower_only=True, acc=acc, nthreads=nthreads)


def gemm_naive(alpha, a, b, beta, c):
    lib().orc_gemm_naive_d(alpha, _view(*a), _view(*b), beta, _view(*c))


def gemm_scatter(alpha, abuf, ar, ac, bbuf, br, bc, beta, cbuf, cr, cc, *, kc: int, nthreads: int = 1):
    vecs = [np.ascontiguousarray(v, dtype=np.int64) for v in (ar, ac, br, bc, cr, cc)]
    m, n, k = len(vecs[0]), len(vecs[3]), len(vecs[1])
    rc = lib().orc_gemm_scatter_d(alpha, abuf.ctypes.data, vecs[0].ctypes.data, vecs[1].ctypes.data, bbuf.ctypes.data,
                                  vecs[2].ctypes.data, vecs[3].ctypes.data, beta, cbuf.ctypes.data,
                                  vecs[4].ctypes.data, vecs[5].ctypes.data, m, n, k, kc, nthreads)
    if rc:
        raise ValueError("oracle gemm_scatter failed")


def potrf_leaf(storage: np.ndarray, meta: dict, variant: int) -> int:
    return getattr(lib(), "orc_potrf_leaf_" + _suffix(storage))(_view(storage, meta), variant)


def trsm_rltn(alpha: float, tri, b, *, kc: int, nthreads: int = 1) -> int:
    return getattr(lib(), "orc_trsm_rltn_" + _suffix(b[0]))(alpha, _view(*tri), _view(*b), kc, nthreads)


# ---- control trees, restated from the reference --------------------------
_DEFAULT_KC = {"f64": 256, "f32": 512}


def levels_from_tree(doc: Optional[dict], n: int, dtype: str) -> list[tuple[int, int, int]]:
    """Tree document -> [(variant_code, bs, effective kc)]: blocked variants
    keep their number, unblockedK becomes 10+K; None means the reference
    default tree (control.py:212-223)."""
    if doc is None:
        doc = {"op": "cholesky", "variant": "unblocked3"} if n <= 128 else {
            "op": "cholesky", "variant": 3, "bs": 128, "child": {"op": "cholesky", "variant": "unblocked3"}}
    kc = _DEFAULT_KC[dtype]
    out = []
    node = doc
    while node is not None:
        kc = int((node.get("kernel") or {}).get("kc", kc))
        v = node["variant"]
        if isinstance(v, int):
            out.append((v, int(node["bs"]), kc))
        else:
            out.append((10 + int(str(v)[-1]), 0, kc))
        node = node.get("child")
    return out


def cholesky(storage: np.ndarray, meta: dict, levels, *, uplo: str = "lower", nthreads: int = 1) -> int:
    """In-place blocked Cholesky; returns the global failing index or -1."""
    if uplo == "upper":
        meta = transposed(meta)
    arr = (_Level * len(levels))(*[_Level(v, 0, bs, kc) for v, bs, kc in levels])
    return int(getattr(lib(), "orc_cholesky_" + _suffix(storage))(_view(storage, meta), arr, len(levels), nthreads))


def levels_from_tree_lu(doc: Optional[dict], n: int, dtype: str) -> list[tuple[int, int, int]]:
    """LU tree document -> [(20 blocked | 21 leaf, bs, effective kc)]; None is
    the reference default (control.py:212-223: unblocked up to 128, else one
    blocked level of 128)."""
    if doc is None:
        doc = {"op": "lu", "variant": "unblocked"} if n <= 128 else {
            "op": "lu", "variant": "blocked", "bs": 128, "child": {"op": "lu", "variant": "unblocked"}}
    kc = _DEFAULT_KC[dtype]
    out = []
    node = doc
    while node is not None:
        kc = int((node.get("kernel") or {}).get("kc", kc))
        out.append((20, int(node["bs"]), kc) if node["variant"] == "blocked" else (21, 0, kc))
        node = node.get("child")
    return out


def lu(storage: np.ndarray, meta: dict, levels, *, nthreads: int = 1) -> tuple[int, np.ndarray]:
    """In-place LU with partial pivoting (factor/lu.py:56-103): returns the
    first exactly-zero pivot column (or -1) and the LAPACK-style swap list."""
    steps = min(meta["m"], meta["n"])
    piv = np.arange(max(steps, 1), dtype=np.int64)
    arr = (_Level * len(levels))(*[_Level(v, 0, bs, kc) for v, bs, kc in levels])
    sing = int(getattr(lib(), "orc_lu_" + _suffix(storage))(_view(storage, meta), arr, len(levels),
                                                               piv.ctypes.data, nthreads))
    return sing, piv[:steps]


def trsm_llnu(alpha: float, tri, b, *, kc: int, nthreads: int = 1) -> None:
    """unit_tril(tri) X = alpha b, b := X (engine/trsm.py:71-88,114-125)."""
    (ts, tm), (bs_, bm) = tri, b
    getattr(lib(), "orc_trsm_llnu_" + _suffix(bs_))(float(alpha), _view(ts, tm), _view(bs_, bm), int(kc), nthreads)


def sandwich(c, a, t: np.ndarray, *, kc: int, nthreads: int = 1) -> None:
    """lower(C) -= A T A^T, T skew tridiagonal (engine/gemm.py:245-280): W = T A^T
    formed with the reference's packing arithmetic, then the kc-segmented GEMMT."""
    (cs_, cm), (as_, am) = c, a
    tt = np.ascontiguousarray(t, dtype=cs_.dtype) if len(t) else np.zeros(1, dtype=cs_.dtype)
    getattr(lib(), "orc_sandwich_" + _suffix(cs_))(_view(cs_, cm), _view(as_, am), tt.ctypes.data, int(kc), nthreads)


def ltlt_unblocked(storage: np.ndarray, meta: dict) -> tuple[np.ndarray, np.ndarray]:
    """factor/ltlt.py:157-182 in place; returns (piv, t)."""
    n = meta["n"]
    piv = np.arange(n, dtype=np.int64)
    t = np.zeros(max(n - 1, 1), dtype=storage.dtype)
    if n > 1:
        getattr(lib(), "orc_ltlt_unblocked_" + _suffix(storage))(_view(storage, meta), piv.ctypes.data, t.ctypes.data)
    return piv, t[: max(n - 1, 0)]


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---- contraction planner, restated from tensor/contract.py:39-152 ----------
def _row_major_strides(dims) -> list[int]:
    out, acc = [], 1
    for d in reversed(dims):
        out.append(acc)
        acc *= d
    return list(reversed(out))


def _axis(start, dims, strides) -> np.ndarray:
    off = np.array([start], dtype=np.int64)
    for d, s in zip(dims, strides):
        off = (off[:, None] + np.arange(d, dtype=np.int64)[None, :] * s).reshape(-1)
    return off


def contract(alpha, a_st, a_dims, b_st, b_dims, beta, c_st, c_dims, spec: str, *, kc: int, fold: bool = True,
             nthreads: int = 1) -> None:
    """c := beta*c + alpha*contraction for row-major tensors (in place)."""
    lhs, lc = spec.replace(" ", "").split("->")
    la, lb = lhs.split(",")
    tabs = {}
    for labels, dims in ((la, a_dims), (lb, b_dims), (lc, c_dims)):
        st = _row_major_strides(dims)
        tabs[labels] = {l: (int(d), int(s)) for l, d, s in zip(labels, dims, st)}
    ta, tb, tc = tabs[la], tabs[lb], tabs[lc]
    sa, sb, sc = set(la), set(lb), set(lc)

    def order(labels, owner, table):
        pos = {l: i for i, l in enumerate(owner)}
        return sorted(labels, key=lambda l: (-abs(table[l][1]), pos[l]))

    def groups(ordered, tables):
        out = []
        for l in ordered:
            if out and fold and all(t[out[-1][-1]][1] == t[l][1] * t[l][0] for t in tables):
                out[-1].append(l)
            else:
                out.append([l])
        return out

    mg = groups(order(sa & sc, lc, tc), [ta, tc])
    ng = groups(order(sb & sc, lc, tc), [tb, tc])
    kg = groups(order((sa & sb) - sc, la, ta), [ta, tb])

    def vec(gs, table, start):
        dims = [int(np.prod([table[l][0] for l in g])) for g in gs]
        strides = [table[g[-1]][1] for g in gs]
        return _axis(start, dims, strides)

    gemm_scatter(alpha, a_st, vec(mg, ta, 0), vec(kg, ta, 0), b_st, vec(kg, tb, 0), vec(ng, tb, 0), beta, c_st,
                 vec(mg, tc, 0), vec(ng, tc, 0), kc=kc, nthreads=nthreads)
