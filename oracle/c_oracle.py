"""ctypes wrapper of the C/OpenMP oracle (TEST INFRASTRUCTURE ONLY).

Same call shapes as ``oracle.mdp_oracle`` (greedy / solve / inner_solve /
spmv) plus the locality generator used to build the CPU baseline's sample.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build_oracle
from .mdp_oracle import OracleResult, InnerReport

_lib = None
_p = C.c_void_p


class _Rep(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("pad", C.c_int32), ("final_resid", C.c_double), ("eff", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("status", C.c_int32), ("outer", C.c_int32), ("inner", C.c_int64)]


def lib():
    global _lib
    if _lib is None:
        path = build_oracle.OUT
        if not path.exists():
            path = build_oracle.build()
        L = C.CDLL(str(path))
        L.orc_greedy.restype = C.c_double
        L.orc_greedy.argtypes = [C.c_int64, C.c_int32, _p, _p, _p, _p, C.c_double, C.c_int, _p,
                                 C.c_int64, _p, _p, C.c_int]
        L.orc_spmv.argtypes = [_p, _p, _p, C.c_int64, _p, _p, C.c_int]
        L.orc_inner_solve.argtypes = [_p, _p, _p, C.c_int64, C.c_double, _p, _p, C.c_double,
                                      C.c_int32, C.c_int32, C.c_double, C.POINTER(_Rep), C.c_int]
        L.orc_solve.argtypes = [C.c_int64, C.c_int32, _p, _p, _p, _p, C.c_double, C.c_int,
                                C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_double, _p, _p, _p, C.c_int32, C.POINTER(_Stats), C.c_int]
        L.orc_gen_locality.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_uint64,
                                       C.c_int64, C.c_int64, _p, _p, _p, C.c_int]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def threads(n: int | None = None) -> int:
    return n if n else (os.cpu_count() or 1)


def _a(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


def spmv(row_ptr, col, val, x, nthreads=None):
    rp, ci, va, xv = _a(row_ptr, np.int64), _a(col, np.int32), _a(val, np.float64), _a(x, np.float64)
    y = np.empty(rp.shape[0] - 1)
    lib().orc_spmv(rp.ctypes.data, ci.ctypes.data, va.ctypes.data, y.shape[0], xv.ctypes.data,
                   y.ctypes.data, threads(nthreads))
    return y


def greedy(row_ptr, col, val, cost, gamma, v, maximize=False, state0=0, nthreads=None):
    """Returns (policy int64, applied, max |v[state0+s] - applied[s]|)."""
    cost = _a(cost, np.float64)
    n, m = cost.shape
    rp, ci, va, vv = _a(row_ptr, np.int64), _a(col, np.int32), _a(val, np.float64), _a(v, np.float64)
    pi = np.empty(n, np.int64)
    ap = np.empty(n)
    res = lib().orc_greedy(n, m, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, cost.ctypes.data,
                           gamma, int(maximize), vv.ctypes.data, state0, pi.ctypes.data,
                           ap.ctypes.data, threads(nthreads))
    return pi, ap, res


def inner_solve(rp, col, val, gamma, b, theta0, target, max_it, kind="gmres", scale=1.0,
                nthreads=None):
    rp, ci, va, bb = _a(rp, np.int64), _a(col, np.int32), _a(val, np.float64), _a(b, np.float64)
    x = np.array(theta0, dtype=np.float64, copy=True)
    rep = _Rep()
    lib().orc_inner_solve(rp.ctypes.data, ci.ctypes.data, va.ctypes.data, x.shape[0], gamma,
                          bb.ctypes.data, x.ctypes.data, target, max_it,
                          {"richardson": 0, "gmres": 1}[kind], scale, C.byref(rep),
                          threads(nthreads))
    return x, InnerReport(rep.iterations, rep.final_resid, bool(rep.converged), False, rep.eff)


def solve(row_ptr, col, val, cost, gamma, *, maximize=False, tol=1e-8, alpha=1e-4,
          max_outer=1000, max_inner=1000, kind="gmres", ksp_max_it=None, richardson_scale=1.0,
          v0=None, nthreads=None) -> OracleResult:
    cost = _a(cost, np.float64)
    n, m = cost.shape
    rp, ci, va = _a(row_ptr, np.int64), _a(col, np.int32), _a(val, np.float64)
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=np.float64, copy=True)
    pi = np.zeros(n, np.int64)
    hist = np.zeros(max_outer + 2)
    st = _Stats()
    lib().orc_solve(n, m, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, cost.ctypes.data, gamma,
                    int(maximize), tol, alpha, max_outer, max_inner,
                    {"richardson": 0, "gmres": 1}[kind], ksp_max_it or 0, richardson_scale,
                    v.ctypes.data, pi.ctypes.data, hist.ctypes.data, hist.shape[0], C.byref(st),
                    threads(nthreads))
    status = {0: "converged", 1: "outer_cap", 2: "stalled"}[st.status]
    return OracleResult(values=v, policy=pi, outer_iterations=st.outer,
                        inner_iterations_total=int(st.inner),
                        residual_history=[float(x) for x in hist[: st.outer + 1]], status=status)


def gen_locality(n, m, K, W, seed=0, state0=0, n_states=None, nthreads=None):
    ns = n - state0 if n_states is None else n_states
    col = np.empty(ns * m * K, np.int32)
    val = np.empty(ns * m * K)
    cost = np.empty(ns * m)
    lib().orc_gen_locality(n, m, K, W, seed, state0, ns, col.ctypes.data, val.ctypes.data,
                           cost.ctypes.data, threads(nthreads))
    return np.arange(ns * m + 1, dtype=np.int64) * K, col, val, cost.reshape(ns, m)
