"""Seeded synthetic inputs (shared by oracle tests, GPU tests and bench.py).

Input generators only: nothing here computes any part of the method (no SpMV,
no dot, no recurrence).  Shapes follow BASELINE.json ``configs`` as specified in
SURVEY.md §8(d); they stand in for the paper's SuiteSparse matrices
(§3 l.103), which are not available offline.

The right-hand side ``b = A*ones`` used by the stencil configs is *not* built
here: each side (oracle, GPU) computes it with its own SpMV.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-std=gnu11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lquadmath", "-lm"])
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, u64, i32, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        lib.gen_stencil_nnz.restype = i64
        lib.gen_stencil_nnz.argtypes = [i32, i64]
        lib.gen_stencil.argtypes = [i32, i64, dbl, vp, vp, vp]
        lib.gen_random_rowlens.argtypes = [i64, u64, dbl, i32, i32, i64, vp]
        lib.gen_random_fill.argtypes = [i64, u64, dbl, i32, i32, i64, dbl, vp, vp, vp]
        lib.gen_uniform.argtypes = [i64, u64, dbl, dbl, vp]
        lib.gen_ill.argtypes = [i64, u64, dbl, i32, i64, vp, vp]
        lib.gen_loguniform.argtypes = [i64, u64, dbl, dbl, vp]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class CSR:
    n: int
    row_ptr: np.ndarray  # int32 [n+1]
    col: np.ndarray      # int32 [nnz], strictly increasing per row
    val: np.ndarray      # float64 [nnz]
    name: str = ""
    rhs: str = "Aones"   # "Aones" -> b = A*ones (computed by each side); "given" -> see b
    b: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def rows(self, r0: int, r1: int) -> "CSR":
        """Contiguous row block [r0,r1) with global column ids (one rank's share)."""
        s, e = int(self.row_ptr[r0]), int(self.row_ptr[r1])
        return CSR(n=self.n, row_ptr=(self.row_ptr[r0:r1 + 1] - s).astype(np.int32),
                   col=self.col[s:e], val=self.val[s:e], name=self.name, rhs=self.rhs,
                   b=None if self.b is None else self.b[r0:r1])


def stencil(d: int, N: int, Pe: float) -> CSR:
    L = _L()
    n = N ** d
    nnz = L.gen_stencil_nnz(d, N)
    rp = np.empty(n + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    rc = L.gen_stencil(d, N, float(Pe), _p(rp), _p(col), _p(val))
    assert rc == 0 and rp[-1] == nnz
    return CSR(n, rp, col, val, name=f"cd{d}d_{N}_pe{Pe:g}")


def random_banded(n: int, seed: int = 42, lam: float = 27.0, lmin: int = 5, lmax: int = 200,
                  band: int = 5000, diag_scale: float = 1.2, b_seed: int = 43) -> CSR:
    L = _L()
    rp = np.empty(n + 1, np.int32)
    rc = L.gen_random_rowlens(n, seed, lam, lmin, lmax, band, _p(rp))
    assert rc == 0, rc
    nnz = int(rp[-1])
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    rc = L.gen_random_fill(n, seed, lam, lmin, lmax, band, diag_scale, _p(rp), _p(col), _p(val))
    assert rc == 0, rc
    b = uniform(n, b_seed, 0.0, 1.0)
    return CSR(n, rp, col, val, name=f"rand_{n}_s{seed}", rhs="given", b=b)


def uniform(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    v = np.empty(n, np.float64)
    _L().gen_uniform(n, seed, lo, hi, _p(v))
    return v


def ill_pair(n: int, seed: int = 3, b: float = 100.0, spread: int = 175, block: int = 1 << 20):
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    rc = _L().gen_ill(n, seed, b, spread, block, _p(x), _p(y))
    assert rc == 0
    return x, y


def loguniform(n: int, seed: int, emin: float, emax: float) -> np.ndarray:
    v = np.empty(n, np.float64)
    _L().gen_loguniform(n, seed, emin, emax, _p(v))
    return v


def dense_as_sparse(n: int, seed: int, density: float = 1.0, diag_boost: float = 2.0) -> CSR:
    """Small random unsymmetric, diagonally dominant system (tests only)."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (n, n))
    if density < 1.0:
        A *= rng.uniform(0, 1, (n, n)) < density
    A[np.arange(n), np.arange(n)] = diag_boost * (np.abs(A).sum(1) + 1.0)
    return from_dense(A, name=f"dense{n}_s{seed}")


def from_dense(A: np.ndarray, name: str = "dense") -> CSR:
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    rp = [0]
    cols, vals = [], []
    for i in range(n):
        nzc = np.nonzero(A[i])[0]
        cols.extend(nzc.tolist())
        vals.extend(A[i, nzc].tolist())
        rp.append(len(cols))
    return CSR(n, np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals, np.float64), name=name)


# BASELINE.json configs (SURVEY.md §8(d) recipe)
CONFIGS = {
    "c1_2d64": dict(kind="stencil", d=2, N=64, Pe=10.0, tol=1e-10, max_iter=500),
    "c3_3d128": dict(kind="stencil", d=3, N=128, Pe=100.0, tol=1e-10, max_iter=10000),
    "c4_rand4m": dict(kind="random", n=1 << 22, seed=42, tol=1e-10, max_iter=10000),
    "c5_3d256": dict(kind="stencil", d=3, N=256, Pe=200.0, tol=1e-10, max_iter=10000),
}


def make_config(name: str, **over) -> CSR:
    c = dict(CONFIGS[name])
    c.update(over)
    if c["kind"] == "stencil":
        A = stencil(c["d"], c["N"], c["Pe"])
    else:
        A = random_banded(c["n"], seed=c.get("seed", 42))
    A.name = name
    return A
