"""CPU oracle for the p-BiCGStab + ExBLAS hot path (arXiv 2404.13216).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2404_13216_b200``) never imports it and
shares no code with it.

This module is argument marshalling around ``oracle.c`` (plain C99, built with
``-ffp-contract=off``); every computation and its citation lives there:

* ``exdot``        EXDOT = RN-even(exact sum x_k y_k)   SPEC.md l.83/92/111
* ``spmv``         fixed-order per-row FMA chain          SPEC.md l.164 (reading R-6)
* ``PBiCGStab``    Algorithm 2 step by step
* ``bicgstab``     Algorithm 1 in plain fp64
* ``true_relres``  NORM(b - A x)/NORM(b)

Parity status: every function above is pinned by ``tests/test_oracle_*.py``
against brute force (``fractions.Fraction``), closed forms, invariants and a
dense direct solve; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

F_RANGE = 1
F_NONFINITE = 2
F_OVERFLOW = 4

CONVERGED, MAXITER, BREAKDOWN_INIT, BREAKDOWN_RHO, BREAKDOWN_OMEGA, BREAKDOWN_ALPHA, RANGE = range(7)
RUNNING = -1
STATUS_NAMES = {0: "converged", 1: "maxiter", 2: "breakdown_init", 3: "breakdown_rho",
                4: "breakdown_omega", 5: "breakdown_alpha", 6: "range", -1: "running"}
# history columns (one row per iteration; row 0 = initialisation)
H_THETA, H_ETA, H_SIGMA, H_ZETA, H_OMEGA, H_RHO, H_DELTA, H_RR, H_RELRES, H_BETA, H_ALPHA = range(11)
H_COLS = 12
VEC = dict(b=0, x=1, r=2, rh=3, p=4, s=5, z=6, q=7, y=8, w=9, t=10, v=11)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        lib.orc_exdot.restype = dbl
        lib.orc_exdot.argtypes = [i64, vp, vp, vp]
        lib.orc_exdot_parts.restype = dbl
        lib.orc_exdot_parts.argtypes = [i64, vp, vp, i32, vp, vp]
        lib.orc_acc_size.restype = i32
        lib.orc_acc_clear.argtypes = [vp]
        lib.orc_acc_add_product.argtypes = [vp, dbl, dbl]
        lib.orc_acc_add_double.argtypes = [vp, dbl]
        lib.orc_acc_merge.argtypes = [vp, vp]
        lib.orc_acc_round.restype = dbl
        lib.orc_acc_round.argtypes = [vp]
        lib.orc_acc_flags.restype = i32
        lib.orc_acc_flags.argtypes = [vp]
        lib.orc_spmv.argtypes = [i64, vp, vp, vp, vp, vp]
        lib.orc_dot_seq.restype = dbl
        lib.orc_dot_seq.argtypes = [i64, vp, vp]
        lib.orc_pbcg_size.restype = i32
        lib.orc_pbcg_init.restype = i32
        lib.orc_pbcg_init.argtypes = [vp, i64, vp, vp, vp, vp, vp, dbl, dbl, i32, vp, i32, vp]
        lib.orc_bj_apply.argtypes = [i64, vp, vp, vp]
        lib.orc_bj_blocks.restype = i32
        lib.orc_bj_blocks.argtypes = [i64, vp, vp, vp, vp, vp]
        lib.orc_pbcg_step.restype = i32
        lib.orc_pbcg_step.argtypes = [vp]
        lib.orc_pbcg_run.restype = i32
        lib.orc_pbcg_run.argtypes = [vp, i32]
        lib.orc_pbcg_iterations.restype = i32
        lib.orc_pbcg_iterations.argtypes = [vp]
        lib.orc_pbcg_status.restype = i32
        lib.orc_pbcg_status.argtypes = [vp]
        lib.orc_pbcg_loop_seconds.restype = dbl
        lib.orc_pbcg_loop_seconds.argtypes = [vp]
        lib.orc_pbcg_scalar.restype = dbl
        lib.orc_pbcg_scalar.argtypes = [vp, i32]
        lib.orc_pbcg_vec.restype = ctypes.POINTER(ctypes.c_double)
        lib.orc_pbcg_vec.argtypes = [vp, i32]
        lib.orc_pbcg_free.argtypes = [vp]
        lib.orc_true_relres.restype = dbl
        lib.orc_true_relres.argtypes = [i64, vp, vp, vp, vp, vp, vp]
        lib.orc_bicgstab.restype = i32
        lib.orc_bicgstab.argtypes = [i64, vp, vp, vp, vp, vp, dbl, i32, vp, vp]
        lib.orc_pbcg_replace.restype = i32
        lib.orc_pbcg_replace.argtypes = [vp]
        lib.orc_pbcg_set_rr.restype = None
        lib.orc_pbcg_set_rr.argtypes = [vp, i32]
        lib.orc_pbcg_replacements.restype = i32
        lib.orc_pbcg_replacements.argtypes = [vp]
        lib.orc_bicgstab_dots.restype = i32
        lib.orc_bicgstab_dots.argtypes = [i64, vp, vp, vp, vp, vp, dbl, i32, i32, vp, vp]
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def exdot(x, y) -> tuple[float, int]:
    """(EXDOT(x,y), flags)."""
    x, y = _f64(x), _f64(y)
    assert x.shape == y.shape
    f = ctypes.c_int(0)
    r = _L().orc_exdot(x.size, _p(x), _p(y), ctypes.byref(f))
    return r, f.value


def exdot_parts(x, y, nparts: int, order=None) -> tuple[float, int]:
    x, y = _f64(x), _f64(y)
    f = ctypes.c_int(0)
    o = None
    if order is not None:
        o = np.ascontiguousarray(order, dtype=np.int32)
    r = _L().orc_exdot_parts(x.size, _p(x), _p(y), nparts, None if o is None else _p(o), ctypes.byref(f))
    return r, f.value


class Acc:
    """The oracle's exact long accumulator (for merge/round tests)."""

    def __init__(self):
        self._buf = ctypes.create_string_buffer(_L().orc_acc_size())
        _L().orc_acc_clear(self._buf)

    def add_product(self, x: float, y: float):
        _L().orc_acc_add_product(self._buf, float(x), float(y))
        return self

    def add(self, x: float):
        _L().orc_acc_add_double(self._buf, float(x))
        return self

    def merge(self, other: "Acc"):
        _L().orc_acc_merge(self._buf, other._buf)
        return self

    def round(self) -> float:
        return _L().orc_acc_round(self._buf)

    @property
    def flags(self) -> int:
        return _L().orc_acc_flags(self._buf)


def spmv(A, x) -> np.ndarray:
    """y = A x for all rows of A (A.col are indices into x)."""
    x = _f64(x)
    nrows = A.row_ptr.size - 1
    y = np.empty(nrows, np.float64)
    rp = np.ascontiguousarray(A.row_ptr, np.int32)
    col = np.ascontiguousarray(A.col, np.int32)
    val = _f64(A.val)
    _L().orc_spmv(nrows, _p(rp), _p(col), _p(val), _p(x), _p(y))
    return y


def dot_seq(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return _L().orc_dot_seq(x.size, _p(x), _p(y))


class PBiCGStab:
    """Algorithm 2 state machine.  ``b=None`` means b := A*ones (each side
    computes it with its own SpMV); ``x0=None`` means x0 := 0."""

    def __init__(self, A, b=None, x0=None, tol=1e-10, eps=1e-30, max_iter=10000, history=True, rr_period=0,
                 range_mode="full", minv=None):
        """range_mode "full" (R-24): dots exact over the whole
        binary64 range, only NaN/Inf or an overflowing exact sum stops the
        solve; "fast" (R-9): any product outside the fast zone stops it.
        minv: [nb, 4] M^-1 blocks (block_jacobi_right): the pipelined right
        2x2 block Jacobi of R-25 -- every product of the iteration is
        A (M^-1 u); x0 is then y0 = M x0 and vec("x") the final y."""
        L = _L()
        self.A = A
        self._rp = np.ascontiguousarray(A.row_ptr, np.int32)
        self._col = np.ascontiguousarray(A.col, np.int32)
        self._val = _f64(A.val)
        self._b = None if b is None else _f64(b)
        self._x0 = None if x0 is None else _f64(x0)
        self._minv = None if minv is None else np.ascontiguousarray(minv, np.float64).reshape(-1)
        self.max_iter = max_iter
        self.hist = np.zeros((max_iter + 1, H_COLS), np.float64) if history else None
        self._S = ctypes.create_string_buffer(L.orc_pbcg_size())
        self.rc = L.orc_pbcg_init(self._S, A.n, _p(self._rp), _p(self._col), _p(self._val),
                                  None if self._b is None else _p(self._b),
                                  None if self._x0 is None else _p(self._x0),
                                  float(tol), float(eps), int(max_iter),
                                  None if self.hist is None else _p(self.hist),
                                  {"full": 1, "fast": 0}[range_mode],
                                  None if self._minv is None else _p(self._minv))
        if rr_period:  # residual replacement every rr_period iterations (NEXT-2, R-21)
            L.orc_pbcg_set_rr(self._S, int(rr_period))

    def replace(self) -> None:
        """One residual replacement now: r := b - A x; w := A r; s := A p; z := A s; t := A w."""
        _L().orc_pbcg_replace(self._S)

    @property
    def replacements(self) -> int:
        return _L().orc_pbcg_replacements(self._S)

    def step(self) -> int:
        return _L().orc_pbcg_step(self._S)

    def run(self, max_steps: int | None = None) -> int:
        return _L().orc_pbcg_run(self._S, self.max_iter + 1 if max_steps is None else max_steps)

    @property
    def status(self) -> int:
        return _L().orc_pbcg_status(self._S)

    @property
    def iterations(self) -> int:
        return _L().orc_pbcg_iterations(self._S)

    @property
    def loop_seconds(self) -> float:
        return _L().orc_pbcg_loop_seconds(self._S)

    def scalar(self, name: str) -> float:
        return _L().orc_pbcg_scalar(self._S, ["alpha", "beta", "omega", "rho", "nb", "epsn"].index(name))

    def vec(self, name: str) -> np.ndarray:
        p = _L().orc_pbcg_vec(self._S, VEC[name])
        return np.ctypeslib.as_array(p, shape=(self.A.n,)).copy()

    def history(self) -> np.ndarray:
        return self.hist[: self.iterations + 1].copy()

    def true_relres(self) -> float:
        return true_relres(self.A, self.vec("b"), self.vec("x"))[0]

    def close(self):
        if self._S is not None:
            _L().orc_pbcg_free(self._S)
            self._S = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def true_relres(A, b, x) -> tuple[float, int]:
    b, x = _f64(b), _f64(x)
    rp = np.ascontiguousarray(A.row_ptr, np.int32)
    col = np.ascontiguousarray(A.col, np.int32)
    val = _f64(A.val)
    f = ctypes.c_int(0)
    r = _L().orc_true_relres(A.n, _p(rp), _p(col), _p(val), _p(b), _p(x), ctypes.byref(f))
    return r, f.value


def bicgstab(A, b, x0=None, tol=1e-10, max_iter=10000, exact_dots=False):
    """Algorithm 1.  exact_dots=False: sequential plain
    double dots (the textbook routine); True: EXDOT (the arithmetic of the
    GPU's Alg. 1 arm).  Returns (status, iterations, x, relres history)."""
    b = _f64(b)
    x = np.zeros(A.n) if x0 is None else _f64(x0).copy()
    rp = np.ascontiguousarray(A.row_ptr, np.int32)
    col = np.ascontiguousarray(A.col, np.int32)
    val = _f64(A.val)
    it = ctypes.c_int(0)
    hist = np.zeros(max_iter + 1)
    st = _L().orc_bicgstab_dots(A.n, _p(rp), _p(col), _p(val), _p(b), _p(x), float(tol), int(max_iter),
                                int(bool(exact_dots)), ctypes.byref(it), _p(hist))
    return st, it.value, x, hist[: it.value + 1]


def jacobi_right(A):
    """Right Jacobi preconditioning as a column scaling (SURVEY §8(f) NEXT-3,
    DESIGN.md R-22): A' = A D^-1 with D = diag(A), one RN division per stored
    entry.  Solve A' y = b with Algorithm 2 (y0 = D x0), then x = D^-1 y (one
    RN division per entry).  Returns (A', d); A' has the attributes
    PBiCGStab and spmv use (n, row_ptr, col, val, rhs, b)."""
    import types
    rp = np.asarray(A.row_ptr, np.int64)
    col = np.asarray(A.col, np.int64)
    val = _f64(A.val)
    rows = np.repeat(np.arange(A.n), np.diff(rp))
    d = np.zeros(A.n)
    on = col == rows
    d[rows[on]] = val[on]
    if np.any(d == 0.0):
        raise ValueError("jacobi: zero or missing diagonal entry")
    As = types.SimpleNamespace(n=A.n, row_ptr=A.row_ptr, col=A.col, val=val / d[col],
                               rhs=getattr(A, "rhs", "given"), b=getattr(A, "b", None))
    return As, d


def _fma(a: float, b: float, c: float) -> float:
    """fl(a*b + c), one rounding (RN-even), from exact rationals; an exact
    zero takes IEEE 754's sign (-0 only for (-0) + (-0))."""
    import math
    from fractions import Fraction
    r = Fraction(a) * Fraction(b) + Fraction(c)
    if r == 0:
        neg_p = (a == 0.0 or b == 0.0) and math.copysign(1.0, a) * math.copysign(1.0, b) < 0
        return -0.0 if (neg_p and c == 0.0 and math.copysign(1.0, c) < 0) else 0.0
    try:
        return float(r)
    except OverflowError:  # beyond the binary64 range: RN gives +-inf
        return math.inf if r > 0 else -math.inf


def block_jacobi_right(A):
    """Right 2x2 point-block Jacobi (R-23).
    M = the 2x2 diagonal blocks of A (rows 2m, 2m+1; 1x1 for the last row when
    n is odd).  Per block (a b; c d): det = fma(a, d, -(b c)),
    M^-1 = (d -b; -c a) / det, one RN division per entry.  B = A M^-1 stored
    explicitly: row i's pattern widened to whole column blocks, A's values at
    A's columns and 0 at the added ones, then per block
    B_i,2m = fma(A_i,2m, m00, A_i,2m+1 m10), B_i,2m+1 = fma(A_i,2m, m01, A_i,2m+1 m11).
    Returns (B, M, Minv): M and Minv as [nblocks, 4] row-major blocks.
    Solve B y = b with Algorithm 2 (y0 = M x0), then x = M^-1 y (bj_apply)."""
    import types
    n = A.n
    rp = np.asarray(A.row_ptr, np.int64)
    col = np.asarray(A.col, np.int64)
    val = _f64(A.val)
    nb = (n + 1) // 2

    def at(r, c):
        s, e = rp[r], rp[r + 1]
        k = np.searchsorted(col[s:e], c)
        return float(val[s + k]) if k < e - s and col[s + k] == c else 0.0

    M = np.zeros((nb, 4))
    Mi = np.zeros((nb, 4))
    for m in range(nb):
        r0 = 2 * m
        if r0 + 1 < n:
            a, b, c, d = at(r0, r0), at(r0, r0 + 1), at(r0 + 1, r0), at(r0 + 1, r0 + 1)
            det = _fma(a, d, -(b * c))
            if det == 0.0:
                raise ValueError("block jacobi: singular 2x2 diagonal block")
            M[m] = (a, b, c, d)
            Mi[m] = (d / det, -(b / det), -(c / det), a / det)
        else:
            a = at(r0, r0)
            if a == 0.0:
                raise ValueError("block jacobi: singular 1x1 tail block")
            M[m] = (a, 0.0, 0.0, 0.0)
            Mi[m] = (1.0 / a, 0.0, 0.0, 0.0)
    if not np.all(np.isfinite(Mi)):
        raise ValueError("block jacobi: non-finite inverse block")
    brp, bcol, bval = [0], [], []
    for i in range(n):
        s, e = rp[i], rp[i + 1]
        k = s
        while k < e:
            m = int(col[k]) >> 1
            v0 = v1 = 0.0
            while k < e and (int(col[k]) >> 1) == m:
                if col[k] & 1:
                    v1 = float(val[k])
                else:
                    v0 = float(val[k])
                k += 1
            m00, m01, m10, m11 = Mi[m]
            if 2 * m + 1 < n:
                bcol += [2 * m, 2 * m + 1]
                bval += [_fma(v0, m00, v1 * m10), _fma(v0, m01, v1 * m11)]
            else:
                bcol.append(2 * m)
                bval.append(v0 * m00)
        brp.append(len(bcol))
    B = types.SimpleNamespace(n=n, row_ptr=np.array(brp, np.int32), col=np.array(bcol, np.int32),
                              val=np.array(bval, np.float64), rhs=getattr(A, "rhs", "given"),
                              b=getattr(A, "b", None), nnz=len(bcol))
    return B, M, Mi


def bj_blocks_c(A):
    """(M, M^-1) of A's 2x2 diagonal blocks by orc_bj_blocks (the C twin of
    block_jacobi_right's blocks, for full-size systems); ValueError if a
    block is singular or its inverse not finite."""
    nb = (A.n + 1) // 2
    M = np.zeros((nb, 4))
    Mi = np.zeros((nb, 4))
    rp = np.ascontiguousarray(A.row_ptr, np.int32)
    col = np.ascontiguousarray(A.col, np.int32)
    val = _f64(A.val)
    if _L().orc_bj_blocks(A.n, _p(rp), _p(col), _p(val), _p(M), _p(Mi)):
        raise ValueError("block jacobi: singular or non-finite 2x2 diagonal block")
    return M, Mi


def bj_apply_c(Q, x) -> np.ndarray:
    """orc_bj_apply (the C twin used inside the pipelined preconditioner)."""
    x = _f64(x)
    Q = np.ascontiguousarray(Q, np.float64)
    y = np.empty_like(x)
    _L().orc_bj_apply(x.size, _p(Q), _p(x), _p(y))
    return y


def bj_apply(Q, x):
    """y = Q x per 2x2 block (Q: M or M^-1 from block_jacobi_right):
    y_2m = fma(q00, x_2m, q01 x_2m+1), y_2m+1 = fma(q10, x_2m, q11 x_2m+1);
    1x1 tail: y = q00 x."""
    x = _f64(x)
    n = x.size
    y = np.empty(n)
    for m in range(Q.shape[0]):
        r0 = 2 * m
        q00, q01, q10, q11 = Q[m]
        if r0 + 1 < n:
            y[r0] = _fma(q00, x[r0], q01 * x[r0 + 1])
            y[r0 + 1] = _fma(q10, x[r0], q11 * x[r0 + 1])
        else:
            y[r0] = q00 * x[r0]
    return y
