"""B200-native p-BiCGStab with ExBLAS-style exactly rounded dots (arXiv 2404.13216).

Thin Python binding over the C ABI in ``include/pbicgstab.h`` (library
``libpbicgstab.so``, sm_100a).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels of ``csrc/``.  There is no CPU fallback:
importing this package without the built library, or calling it without a
CUDA device, raises.

PyTorch provides device memory (the caller-owned workspace, vectors), streams
and process groups; nothing else.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = _build.LIB

CONVERGED, MAXITER, BREAKDOWN_INIT, BREAKDOWN_RHO, BREAKDOWN_OMEGA, BREAKDOWN_ALPHA, RANGE = range(7)
STATUS_NAMES = {0: "converged", 1: "maxiter", 2: "breakdown_init", 3: "breakdown_rho",
                4: "breakdown_omega", 5: "breakdown_alpha", 6: "range", -1: "running"}
RC_NAMES = {0: "OK", 1: "EINVAL", 2: "ECUDA", 3: "ENCCL", 4: "ENOMEM", 5: "ENONFINITE", 6: "ERANGE"}
H_COLS = 12
FLAG_RANGE, FLAG_NONFINITE = 1, 2


class PbcgError(RuntimeError):
    def __init__(self, rc: int, msg: str):
        super().__init__(f"{RC_NAMES.get(rc, rc)}: {msg}")
        self.rc = rc


class _Csr(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("nnz_local", ctypes.c_int64), ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
                ("values", ctypes.c_void_p)]


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("nccl_uid", ctypes.c_void_p),
                ("virtual_ranks", ctypes.c_int32), ("history_capacity", ctypes.c_int32), ("comm_mode", ctypes.c_int32),
                ("precond", ctypes.c_int32)]


# pbcg_opts.dot_mode: "exact" = ExBLAS dots (reproducible), "plain" = fp64 dots (NEXT-1 comparison arm)
DOT_MODES = {"exact": 0, "plain": 1}
# pbcg_opts.method: "pbicgstab" = Algorithm 2 (the hot path), "bicgstab" = Algorithm 1 with exact dots
METHODS = {"pbicgstab": 0, "bicgstab": 1}
# pbcg_dist.precond: "bjacobi2" = B = A M^-1 stored (R-23); "bjacobi2_pipe" = M^-1 applied inside K2/K3 (R-25)
PRECONDS = {"none": 0, "jacobi": 1, "bjacobi2": 2, "bjacobi2_pipe": 3}
# pbcg_opts.range_mode: "full" = dots exact over the whole binary64 range (R-24), "fast" = R-9 zone stops
RANGE_MODES = {"full": 0, "fast": 1}


class _Opts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int32), ("breakdown_eps", ctypes.c_double),
                ("poll_every", ctypes.c_int32), ("use_graphs", ctypes.c_int32), ("dot_mode", ctypes.c_int32),
                ("method", ctypes.c_int32), ("rr_period", ctypes.c_int32), ("x0_zero", ctypes.c_int32),
                ("range_mode", ctypes.c_int32)]


class _Result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32), ("relres_recursive", ctypes.c_double),
                ("relres_true", ctypes.c_double), ("loop_seconds", ctypes.c_double),
                ("history_rows", ctypes.c_int32), ("reserved", ctypes.c_int32), ("digest", ctypes.c_uint64)]


_lib = None


def lib(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load the in-tree CUDA library (building it with nvcc if it is missing)."""
    global _lib
    if _lib is None:
        if build_if_missing and not os.environ.get("PBCG_LIB") and _build.needs_build():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2404_13216_b200/build.py (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        P = ctypes.POINTER
        L.pbicgstab_workspace_size.argtypes = [P(_Csr), P(_Dist), P(ctypes.c_size_t)]
        L.pbicgstab_setup.argtypes = [P(_Csr), P(_Dist), vp, vp, ctypes.c_size_t, P(vp)]
        L.pbicgstab_solve.argtypes = [vp, vp, vp, P(_Opts), P(_Result)]
        L.pbicgstab_start.argtypes = [vp, vp, vp, P(_Opts)]
        L.pbicgstab_iterate.argtypes = [vp, i32]
        L.pbicgstab_finish.argtypes = [vp, vp, P(_Result)]
        L.pbicgstab_history.argtypes = [vp, vp, i32, P(i32)]
        L.pbicgstab_spmv.argtypes = [vp, vp, vp]
        L.exdot.argtypes = [vp, i64, vp, vp, vp, vp, ctypes.c_int, vp]
        L.pbcg_dot_plain.argtypes = [i64, vp, vp, vp, vp]
        L.pbicgstab_destroy.argtypes = [vp]
        L.pbicgstab_destroy.restype = None
        L.pbicgstab_last_error.restype = ctypes.c_char_p
        L.pbcg_nccl_unique_id.argtypes = [vp]
        L.pbcg_plan_partition.argtypes = [i64, i32, vp]
        L.pbcg_plan_halo.argtypes = [i32, i32, vp, vp, vp, vp, vp, P(i64), P(i64)]
        L.pbcg_sacc_accumulate.argtypes = [i64, vp, vp, vp]
        L.pbcg_sacc_round.argtypes = [vp, vp]
        L.pbcg_set_chunk.argtypes = [i32]
        L.pbcg_profile_iterations.argtypes = [vp, i32, vp]
        L.pbcg_debug_counters.argtypes = [vp, i32]
        L.pbcg_spmv_format.argtypes = [vp, vp]
        L.pbcg_exec_mode.argtypes = [vp, vp]
        L.pbcg_get_vector.argtypes = [vp, i32, vp]
        L.pbcg_config_hash.argtypes = [P(_Csr), P(_Dist), P(ctypes.c_uint64)]
        L.pbcg_check_ranks.argtypes = [i32, vp, i64, i32]
        L.pbcg_history_digest.argtypes = [vp, i32, P(ctypes.c_uint64)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise PbcgError(rc, lib().pbicgstab_last_error().decode())


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2404_13216_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _dev_f64(t, torch, n=None):
    if isinstance(t, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(t, np.float64))
    t = t.to(device="cuda", dtype=torch.float64).contiguous()
    if n is not None:
        assert t.numel() == n, (t.numel(), n)
    return t


def _dev_i32(t, torch):
    if isinstance(t, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(t, np.int32))
    return t.to(device="cuda", dtype=torch.int32).contiguous()


@dataclass
class Result:
    status: int
    iterations: int
    relres_recursive: float
    relres_true: float
    loop_seconds: float
    history_rows: int
    digest: int = 0  # fingerprint of the scalar trajectory (pbcg_result.digest)

    @property
    def status_name(self) -> str:
        return STATUS_NAMES.get(self.status, str(self.status))


class Solver:
    """p-BiCGStab handle over one rank's rows (or the full matrix with
    ``virtual_ranks``).  ``row_ptr``/``col``/``val`` may be numpy arrays or
    torch tensors; they are converted into the workspace at setup."""

    def __init__(self, row_ptr, col, val, n_global: int, row_begin: int = 0, row_end: int | None = None,
                 rank: int = 0, nranks: int = 1, nccl_uid: bytes | None = None, virtual_ranks: int = 1,
                 history_capacity: int = 0, stream=None, force_nccl: bool = False, precond: str = "none"):
        torch = _torch()
        L = lib()
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.Stream()
        rp = _dev_i32(row_ptr, torch)
        ci = _dev_i32(col, torch)
        va = _dev_f64(val, torch)
        row_end = n_global if row_end is None else row_end
        self.n_global, self.row_begin, self.row_end = n_global, row_begin, row_end
        self.n_local = row_end - row_begin
        self._csr = _Csr(n_global, row_begin, row_end, int(ci.numel()), rp.data_ptr(), ci.data_ptr(), va.data_ptr())
        self._uid = None
        if nccl_uid is not None:
            self._uid = ctypes.create_string_buffer(bytes(nccl_uid), 128)
        self._dist = _Dist(rank, nranks, ctypes.cast(self._uid, ctypes.c_void_p) if self._uid is not None else None,
                           virtual_ranks, history_capacity, 1 if force_nccl else 0,
                           PRECONDS[precond])
        nbytes = ctypes.c_size_t(0)
        torch.cuda.synchronize()
        _check(L.pbicgstab_workspace_size(ctypes.byref(self._csr), ctypes.byref(self._dist), ctypes.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device="cuda")
        h = ctypes.c_void_p()
        _check(L.pbicgstab_setup(ctypes.byref(self._csr), ctypes.byref(self._dist),
                                 ctypes.c_void_p(self.stream.cuda_stream), ctypes.c_void_p(self.workspace.data_ptr()),
                                 ctypes.c_size_t(self.workspace.numel()), ctypes.byref(h)))
        self._h = h
        self.workspace_bytes = int(nbytes.value)
        del rp, ci, va

    # -- helpers ------------------------------------------------------------
    def _opts(self, tol, max_iter, eps, poll_every, use_graphs, dot_mode="exact", method="pbicgstab", rr_period=0,
              x0_zero=False, range_mode="full"):
        return _Opts(float(tol), int(max_iter), float(eps), int(poll_every), int(use_graphs), DOT_MODES[dot_mode],
                     METHODS[method], int(rr_period), int(bool(x0_zero)), RANGE_MODES[range_mode])

    def _vec(self, v, allow_host: bool):
        torch = self.torch
        if isinstance(v, np.ndarray):
            v = np.ascontiguousarray(v, np.float64)
            if allow_host:
                return v, v.ctypes.data
            v = torch.from_numpy(v)
        if v.device.type == "cpu":
            v = v.to(torch.float64).contiguous()
            if allow_host:
                return v, v.data_ptr()
            v = v.cuda()
        v = v.to(torch.float64).contiguous()
        return v, v.data_ptr()

    def _check_out(self, out, on_host: bool):
        """`out` receives x in place: it must be float64, contiguous, on the
        same side as b and hold n_local_vec elements (no silent copies)."""
        n = self.n_local_vec
        if isinstance(out, np.ndarray):
            ok = out.dtype == np.float64 and out.flags.c_contiguous and on_host and out.size == n
        else:
            ok = (out.dtype == self.torch.float64 and out.is_contiguous() and out.numel() == n
                  and (out.device.type == "cpu") == on_host)
        if not ok:
            raise ValueError(f"solve(out=): need a contiguous float64 buffer of {n} elements on the "
                             f"{'host' if on_host else 'device'} (the side of b)")

    def _sync_in(self):
        self.stream.wait_stream(self.torch.cuda.current_stream())

    def _sync_out(self):
        self.torch.cuda.current_stream().wait_stream(self.stream)

    # -- API ------------------------------------------------------------------
    def solve(self, b, x0=None, tol=1e-10, max_iter=10000, eps=1e-30, poll_every=16, use_graphs=True,
              dot_mode="exact", method="pbicgstab", rr_period=0, out=None, range_mode="full"):
        """Solve; b/x0 may be CUDA tensors or host arrays/tensors (host buffers
        go through the library's staging path).  Returns (x, Result) with x on
        the same side as b.  x0=None starts from 0 without copying an initial
        guess; `out` (optional, same side as b, e.g. a pinned host tensor)
        receives x instead of a newly allocated buffer."""
        torch = self.torch
        self._sync_in()
        keep_b, bp = self._vec(b, allow_host=True)
        on_host = not (isinstance(keep_b, torch.Tensor) and keep_b.is_cuda)
        if out is not None:
            self._check_out(out, on_host)
            x = out
            if x0 is not None:
                src, _ = self._vec(x0, allow_host=on_host)
                if isinstance(x, np.ndarray):
                    np.copyto(x, src)
                else:
                    x.copy_(torch.as_tensor(src))
        elif x0 is None:
            x = np.zeros(self.n_local_vec, np.float64) if on_host else torch.zeros(self.n_local_vec, dtype=torch.float64, device="cuda")
        else:
            x, _ = self._vec(x0, allow_host=on_host)
            x = x.copy() if isinstance(x, np.ndarray) else x.clone()
        xp = x.ctypes.data if isinstance(x, np.ndarray) else x.data_ptr()
        res = _Result()
        opts = self._opts(tol, max_iter, eps, poll_every, use_graphs, dot_mode, method, rr_period, x0 is None, range_mode)
        _check(lib().pbicgstab_solve(self._h, ctypes.c_void_p(bp), ctypes.c_void_p(xp), ctypes.byref(opts), ctypes.byref(res)))
        self._sync_out()
        return x, self._result(res)

    @property
    def n_local_vec(self) -> int:
        return self.n_global if self._dist.virtual_ranks > 1 else self.n_local

    def start(self, b, x0=None, tol=1e-10, max_iter=10000, eps=1e-30, poll_every=16, use_graphs=True,
              dot_mode="exact", method="pbicgstab", rr_period=0, range_mode="full"):
        torch = self.torch
        self._sync_in()
        self._b, bp = self._vec(b, allow_host=True)
        if x0 is None:  # x0 = 0 on the device, nothing copied (pbcg_opts.x0_zero)
            self._x0, xp = None, None
        else:
            self._x0, xp = self._vec(x0, allow_host=True)
        opts = self._opts(tol, max_iter, eps, poll_every, use_graphs, dot_mode, method, rr_period, x0 is None, range_mode)
        _check(lib().pbicgstab_start(self._h, ctypes.c_void_p(bp), ctypes.c_void_p(xp), ctypes.byref(opts)))

    def iterate(self, k: int):
        _check(lib().pbicgstab_iterate(self._h, int(k)))

    def finish(self, x_out=None):
        res = _Result()
        xp = None
        if x_out is not None:
            xp = x_out.ctypes.data if isinstance(x_out, np.ndarray) else x_out.data_ptr()
        _check(lib().pbicgstab_finish(self._h, ctypes.c_void_p(xp) if xp else None, ctypes.byref(res)))
        self._sync_out()
        return self._result(res)

    def profile(self, k: int) -> np.ndarray:
        """Summed ms of [K2, finalize A, SpMV v=Az, K3, finalize B, SpMV t=Aw]
        over k more iterations (direct launches serialised and bracketed by
        CUDA events on the solver stream)."""
        ms = np.zeros(6, np.float64)
        _check(lib().pbcg_profile_iterations(self._h, int(k), ctypes.c_void_p(ms.ctypes.data)))
        return ms

    def spmv_format(self) -> dict:
        """The stored SpMV format (include/pbicgstab.h pbcg_spmv_format)."""
        out = np.zeros(8, np.int64)
        _check(lib().pbcg_spmv_format(self._h, ctypes.c_void_p(out.ctypes.data)))
        keys = ("rows", "nnz", "sell_entries", "explicit_cols", "slot_records", "bytes_per_spmv", "max_row_len",
                "sigma_sorted")
        return {k: int(v) for k, v in zip(keys, out)}

    def exec_mode(self) -> int:
        """0: six kernels per iteration (CUDA graphs); 1: the fused small-system
        kernel, one launch per iterate call (include/pbicgstab.h pbcg_exec_mode)."""
        m = ctypes.c_int32(0)
        _check(lib().pbcg_exec_mode(self._h, ctypes.byref(m)))
        return int(m.value)

    VEC = dict(b=0, x=1, r=2, rh=3, p=4, s=5, z=6, q=7, y=8, w=9, t=10, v=11)

    def vec(self, name: str) -> np.ndarray:
        """Host copy of an internal vector (the oracle's names)."""
        out = np.empty(self.n_local_vec, np.float64)
        _check(lib().pbcg_get_vector(self._h, self.VEC[name], ctypes.c_void_p(out.ctypes.data)))
        return out

    def history(self, max_rows: int = 1 << 20) -> np.ndarray:
        buf = np.zeros((max_rows, H_COLS), np.float64)
        rows = ctypes.c_int32(0)
        _check(lib().pbicgstab_history(self._h, ctypes.c_void_p(buf.ctypes.data), max_rows, ctypes.byref(rows)))
        return buf[: rows.value].copy()

    def spmv(self, x):
        torch = self.torch
        self._sync_in()
        x = _dev_f64(x, torch, self.n_local_vec)
        y = torch.empty_like(x)
        _check(lib().pbicgstab_spmv(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
        self._sync_out()
        return y

    def exdot(self, x, y) -> tuple[float, int]:
        return exdot(x, y, handle=self)

    @staticmethod
    def _result(r: _Result) -> Result:
        return Result(r.status, r.iterations, r.relres_recursive, r.relres_true, r.loop_seconds, r.history_rows,
                      r.digest)

    def close(self):
        if getattr(self, "_h", None):
            self.torch.cuda.synchronize()
            lib().pbicgstab_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exdot(x, y, handle: Solver | None = None, on_device: bool = False, stream=None, out=None, flags_out=None):
    """EXDOT(x, y) on the GPU.  on_device=False: returns (float, flags);
    on_device=True: writes `out` (float64 CUDA tensor of >=1 element) and
    `flags_out` (int32 CUDA tensor or None) stream-ordered on `stream`."""
    torch = _torch()
    x = _dev_f64(x, torch)
    y = _dev_f64(y, torch, x.numel())
    st = stream if stream is not None else torch.cuda.current_stream()
    h = handle._h if handle is not None else None
    L = lib()
    if on_device:
        _check(L.exdot(h, x.numel(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                       ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(flags_out.data_ptr()) if flags_out is not None else None,
                       1, ctypes.c_void_p(st.cuda_stream)))
        return out, flags_out
    res = ctypes.c_double(0.0)
    fl = ctypes.c_int32(0)
    rc = L.exdot(h, x.numel(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.byref(res),
                 ctypes.byref(fl), 0, ctypes.c_void_p(st.cuda_stream))
    if rc not in (0, 5, 6):
        _check(rc)
    return res.value, fl.value


def dot_plain(x, y, out=None, stream=None):
    """Plain (non-reproducible) fp64 dot: the measurement baseline."""
    torch = _torch()
    st = stream if stream is not None else torch.cuda.current_stream()
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device="cuda")
    _check(lib().pbcg_dot_plain(x.numel(), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    return out


class Comm:
    """Comm-only handle (pbicgstab_setup with A = NULL; include/pbicgstab.h):
    the distributed EXDOT of SURVEY §8(b)/(e).  Every rank passes its own
    contiguous slice of x and y; the superaccumulators are allreduced as
    int64 over NCCL and rounded once, identically on every rank."""

    def __init__(self, rank: int = 0, nranks: int = 1, nccl_uid: bytes | None = None, stream=None,
                 force_nccl: bool = False):
        torch = _torch()
        L = lib()
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self._uid = ctypes.create_string_buffer(bytes(nccl_uid), 128) if nccl_uid is not None else None
        self._dist = _Dist(rank, nranks, ctypes.cast(self._uid, ctypes.c_void_p) if self._uid is not None else None,
                           1, 0, 1 if force_nccl else 0, 0)
        nbytes = ctypes.c_size_t(0)
        _check(L.pbicgstab_workspace_size(None, ctypes.byref(self._dist), ctypes.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device="cuda")
        h = ctypes.c_void_p()
        torch.cuda.synchronize()
        _check(L.pbicgstab_setup(None, ctypes.byref(self._dist), ctypes.c_void_p(self.stream.cuda_stream),
                                 ctypes.c_void_p(self.workspace.data_ptr()), ctypes.c_size_t(self.workspace.numel()),
                                 ctypes.byref(h)))
        self._h = h

    def exdot(self, x, y, on_device: bool = False, out=None, flags_out=None):
        return exdot(x, y, handle=self, on_device=on_device, stream=self.stream, out=out, flags_out=flags_out)

    def close(self):
        if getattr(self, "_h", None):
            self.torch.cuda.synchronize()
            lib().pbicgstab_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def config_hash(n_global: int | None, nranks: int = 1, virtual_ranks: int = 1, precond: str = "none",
                comm_mode: int = 0) -> int:
    """pbcg_config_hash of these setup arguments (n_global None: comm-only)."""
    csr = _Csr(n_global or 0, 0, n_global or 0, 0, None, None, None)
    d = _Dist(0, nranks, None, virtual_ranks, 0, comm_mode, PRECONDS[precond])
    out = ctypes.c_uint64(0)
    _check(lib().pbcg_config_hash(ctypes.byref(csr) if n_global is not None else None, ctypes.byref(d),
                                  ctypes.byref(out)))
    return int(out.value)


def history_digest(history) -> int:
    """pbcg_history_digest of a (rows, 12) float64 history in host memory:
    the pbcg_result.digest a solve with that trajectory reports."""
    h = np.ascontiguousarray(np.asarray(history, dtype=np.float64).reshape(-1, 12))
    out = ctypes.c_uint64(0)
    _check(lib().pbcg_history_digest(ctypes.c_void_p(h.ctypes.data), h.shape[0], ctypes.byref(out)))
    return int(out.value)


def check_ranks(records, n_global: int, has_matrix: bool = True) -> tuple[int, str]:
    """pbcg_check_ranks on allgathered records [(row_begin, row_end, cmin,
    cmax, hash), ...]: (rc, message)."""
    rec = np.ascontiguousarray(np.asarray(records, dtype=np.uint64).view(np.int64), np.int64)
    rc = lib().pbcg_check_ranks(rec.shape[0], ctypes.c_void_p(rec.ctypes.data), int(n_global), int(bool(has_matrix)))
    return rc, (lib().pbicgstab_last_error().decode() if rc else "")


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().pbcg_nccl_unique_id(buf))
    return buf.raw


# -- host-only helpers (no GPU needed) -----------------------------------------
def plan_partition(n: int, p: int) -> np.ndarray:
    b = np.zeros(p + 1, np.int64)
    _check(lib().pbcg_plan_partition(n, p, ctypes.c_void_p(b.ctypes.data)))
    return b


def plan_halo(ranges: np.ndarray, me: int):
    """ranges: int64 [p,4] rows (row_begin, row_end, cmin, cmax)."""
    ranges = np.ascontiguousarray(ranges, np.int64)
    p = ranges.shape[0]
    outs = [np.zeros(p, np.int64) for _ in range(4)]
    blo, bhi = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib().pbcg_plan_halo(p, me, ctypes.c_void_p(ranges.ctypes.data),
                                *[ctypes.c_void_p(o.ctypes.data) for o in outs], ctypes.byref(blo), ctypes.byref(bhi)))
    return dict(recv_lo=outs[0], recv_hi=outs[1], send_lo=outs[2], send_hi=outs[3], buf_lo=blo.value, buf_hi=bhi.value)


def sacc_words() -> int:
    return int(lib().pbcg_sacc_words())


def sacc_accumulate(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Host twin of the device superaccumulator: normalised int64 words of
    sum x_k*y_k (products split exactly by TwoProd; R-9 zone)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    w = np.zeros(sacc_words(), np.int64)
    _check(lib().pbcg_sacc_accumulate(x.size, ctypes.c_void_p(x.ctypes.data), ctypes.c_void_p(y.ctypes.data),
                                      ctypes.c_void_p(w.ctypes.data)))
    return w


def sacc_round(words: np.ndarray) -> float:
    words = np.ascontiguousarray(words, np.int64)
    out = ctypes.c_double(0.0)
    rc = lib().pbcg_sacc_round(ctypes.c_void_p(words.ctypes.data), ctypes.byref(out))
    if rc not in (0, 6):
        _check(rc)
    return out.value


def debug_counters(reset: bool = True) -> np.ndarray:
    """Spill counters of a -DPBCG_DEBUG_COUNTERS build (zeros otherwise):
    [1] warp spill votes taken (K2/K3), [2] lane overflow() calls, [3] deposits."""
    out = np.zeros(16, np.uint64)
    _check(lib().pbcg_debug_counters(ctypes.c_void_p(out.ctypes.data), int(reset)))
    return out
