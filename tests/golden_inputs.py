"""Seeded, platform-independent input generators for the golden fixtures.

Shared by tools/gen_golden.py (which feeds them to the reference) and the
tests (which feed them to the oracle and the CUDA path), so the fixture file
only needs output digests.  numpy's PCG64 streams are platform independent;
SPD matrices are built from small integers so M @ M.T is exact whatever BLAS
kernel forms it.
"""
from __future__ import annotations

import hashlib

import numpy as np

NP = {"f64": np.float64, "f32": np.float32}


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def strided_operand(rng: np.random.Generator, m: int, n: int, dt: str, kind: str):
    """(storage, meta) of an m x n operand laid out as kind."""
    vals = rng.uniform(-1, 1, (m, n)).astype(NP[dt])
    if kind == "contiguous":
        return vals.reshape(-1).copy(), {"off": 0, "m": m, "n": n, "rs": n, "cs": 1}
    if kind == "transposed":
        return np.ascontiguousarray(vals.T).reshape(-1), {"off": 0, "m": m, "n": n, "rs": 1, "cs": m}
    parent = rng.uniform(-1, 1, (m + 3, n + 5)).astype(NP[dt])
    parent[2 : 2 + m, 3 : 3 + n] = vals
    return parent.reshape(-1).copy(), {"off": 2 * (n + 5) + 3, "m": m, "n": n, "rs": n + 5, "cs": 1}


def gemm_inputs(seed: int, op: str, dt: str, m: int, n: int, k: int, kinds: tuple[str, str, str]):
    rng = np.random.default_rng(seed)
    n_eff = m if op in ("syrk", "gemmt") else n
    a = strided_operand(rng, m, k, dt, kinds[0])
    b = strided_operand(rng, k, n_eff, dt, kinds[1]) if op != "syrk" else None
    c = strided_operand(rng, m, n_eff, dt, kinds[2])
    return a, b, c


def spd_int(seed: int, n: int, dt: str = "f64") -> np.ndarray:
    """A = M M^T + n I with small-integer M: exact in any summation order."""
    if n > 4096:
        return spd_int_large(seed, n).astype(NP[dt], copy=False)
    rng = np.random.default_rng(seed)
    m = rng.integers(-4, 5, (n, n)).astype(np.float64)
    return (m @ m.T + n * np.eye(n)).astype(NP[dt])


def spd_int_large(seed: int, n: int, block: int = 4096) -> np.ndarray:
    """spd_int for large n, bit-identical to the small-n formula.

    Every entry of M M^T is a sum of n integer products in [-16, 16], so its
    magnitude stays below 16 n < 2^24 for n < 2^20: float32 arithmetic forms
    it exactly, in any order.  Row blocks avoid OpenBLAS's n=32768 fp64 SYRK
    crash."""
    assert 16 * n < 2**24
    rng = np.random.default_rng(seed)
    m = rng.integers(-4, 5, (n, n)).astype(np.float32)
    mt = np.ascontiguousarray(m.T)
    out = np.empty((n, n), dtype=np.float64)
    for i in range(0, n, block):
        out[i : i + block] = m[i : i + block] @ mt
    del mt, m
    out[np.diag_indices(n)] += n
    return out


def spd_int_torch(seed: int, n: int, device="cuda"):
    """spd_int(seed, n) as a float64 torch tensor formed on `device` (same bits:
    the integer products are exact in any summation order)."""
    import torch

    rng = np.random.default_rng(seed)
    m = torch.from_numpy(rng.integers(-4, 5, (n, n)).astype(np.float32)).to(device).double()
    a = m @ m.T
    del m
    a.diagonal().add_(n)
    return a


def spd_float(seed: int, n: int) -> np.ndarray:
    """The reference's own generator (tests/util.py:7-10); BLAS-dependent bits."""
    rng = np.random.default_rng(seed)
    m = rng.uniform(-1, 1, (n, n))
    return m @ m.T + n * np.eye(n)


def trsm_inputs(seed: int, dt: str, n: int, m: int):
    rng = np.random.default_rng(seed)
    tri = (np.tril(rng.uniform(-1, 1, (n, n))) + n * np.eye(n)).astype(NP[dt])
    b = rng.uniform(-1, 1, (m, n)).astype(NP[dt])
    return tri, b


def tensor_inputs(seed: int, a_dims, b_dims, c_dims):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, a_dims), rng.uniform(-1, 1, b_dims), rng.uniform(-1, 1, c_dims))


def lu_input(seed: int, m: int, n: int, kind: str, dt: str = "f64") -> np.ndarray:
    """Platform-independent LU inputs (numpy default_rng values):
    uniform  U(-1,1): real pivoting everywhere;
    ties     small integers: equal-magnitude pivot candidates (smallest row wins);
    diag     U(-1,1) + n I (the reference CLI's generator, cli.py:66-67): no swaps;
    zerocol  uniform with column n//3 zeroed below the diagonal: an exactly-zero pivot."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        a = rng.uniform(-1, 1, (m, n))
    elif kind == "ties":
        a = rng.integers(-2, 3, (m, n)).astype(np.float64)
    elif kind == "diag":
        a = rng.uniform(-1, 1, (m, n)) + max(m, n) * np.eye(m, n)
    elif kind == "zerocol":
        a = rng.uniform(-1, 1, (m, n))
        j = n // 3
        a[:, j] = 0.0
    else:
        raise KeyError(kind)
    return a.astype(NP[dt])


def left_trsm_inputs(seed: int, n: int, ncols: int, dt: str = "f64"):
    """(tri, b): unit-lower triangle (strict lower U(-1,1)/n, diagonal and
    upper garbage that must be ignored) and a right-hand side block."""
    rng = np.random.default_rng(seed)
    tri = rng.uniform(-1, 1, (n, n)) / max(n, 1)
    tri[np.triu_indices(n)] = 7.0  # never read: unit diagonal, lower only
    b = rng.uniform(-1, 1, (n, ncols))
    return tri.astype(NP[dt]), b.astype(NP[dt])


def sandwich_inputs(seed: int, n: int, k: int, dt: str = "f64", a_layout: str = "row"):
    """(c0, a, t) for lower(C) -= A T A^T: U(-1,1) values; a stored row-major
    or as the transpose of a row-major (k x n) block."""
    rng = np.random.default_rng(seed)
    c0 = rng.uniform(-1, 1, (n, n)).astype(NP[dt])
    a = rng.uniform(-1, 1, (n, k)).astype(NP[dt])
    t = rng.uniform(-1, 1, max(k - 1, 0))
    return c0, a, t


def skew_input(seed: int, n: int, kind: str = "uniform", dt: str = "f64") -> np.ndarray:
    """Skew-symmetric X = M - M^T (the reference CLI's ltlt generator)."""
    rng = np.random.default_rng(seed)
    if kind == "ties":
        m = rng.integers(-2, 3, (n, n)).astype(np.float64)
    else:
        m = rng.uniform(-1, 1, (n, n))
    return (m - m.T).astype(NP[dt])
