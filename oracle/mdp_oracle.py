"""CPU oracle for the iPI hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference's algorithm for the
Bellman backup -> policy gather -> Krylov policy evaluation -> outer iPI loop
(``/root/reference/pkg/src/mdpsolve``).  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it.  The product path
(``paper_2507_22538_b200``) never calls into ``oracle/`` and fails loudly when
its CUDA library is missing.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (importable
in the build container only) on seeded fixtures and commits inputs + outputs
under ``tests/golden/``; ``tests/test_oracle_golden.py`` asserts that every
function here reproduces those outputs **bitwise** (same numpy primitives in
the same order as the reference), so the oracle is pinned, not assumed.

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/mdpsolve``).  Arrays use the reference's layout:
row-stacked ``(n*m, n)`` CSR with row ``s*m + a`` (``model.py:112-131``),
int64 row pointers, fp64 values; column indices may be int32 or int64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GMRES_RESTART = 30          # inner.py:40
TARGET_FLOOR_SCALE = 1e-14  # inner.py:41
STALL_WINDOW = 50           # driver.py:38
ROW_SUM_TOL = 1e-12         # model.py:21

CONVERGED, OUTER_CAP, STALLED = "converged", "outer_cap", "stalled"  # driver.py:41-44


# ----------------------------------------------------------------------------
# L1: CSR kernels (sparse.py)
# ----------------------------------------------------------------------------

def segment_sums(data: np.ndarray, ptr: np.ndarray) -> np.ndarray:
    """Per-segment sums, empty segments -> 0 (sparse.py:126-139)."""
    nseg = len(ptr) - 1
    out = np.zeros(nseg)
    if data.size == 0 or nseg == 0:
        return out
    lengths = np.diff(ptr)
    nonempty = lengths > 0
    if nonempty.any():
        out[nonempty] = np.add.reduceat(data, np.asarray(ptr[:-1])[nonempty])
    return out


def spmv(row_ptr: np.ndarray, col: np.ndarray, val: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y = A x, gather-multiply then segment sums (sparse.py:189-215, block 206-209)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    prod = val * x[np.asarray(col, dtype=np.int64)]
    return segment_sums(prod, rp)


def dot(x: np.ndarray, y: np.ndarray) -> float:
    """Inner product, single block (sparse.py:218-226, workers=None branch)."""
    return float(np.dot(x, y))


def norm2(x: np.ndarray) -> float:
    """Euclidean norm = sqrt(dot(x, x)) (sparse.py:238-239)."""
    return math.sqrt(dot(x, x))


def norm_inf(x: np.ndarray) -> float:
    """Max-abs norm, 0 for empty (sparse.py:232-234)."""
    return float(np.max(np.abs(x))) if x.size else 0.0


# ----------------------------------------------------------------------------
# L2: Bellman backup and policy gather (bellman.py, sparse.py)
# ----------------------------------------------------------------------------

def greedy(row_ptr, col, val, cost, gamma: float, v: np.ndarray, maximize: bool = False):
    """Greedy policy + applied Bellman operator (bellman.py:44-68).

    q = stage_cost + gamma * (P V).reshape(n, m)   -- gamma applied to PV first
    pi = first argmin (argmax for MAX), applied = q[s, pi[s]].
    Returns (policy int64[n], applied f64[n]).
    """
    cost = np.asarray(cost, dtype=np.float64)
    n, m = cost.shape
    pv = spmv(row_ptr, col, val, v)
    q = cost + gamma * pv.reshape(n, m)
    pi = q.argmax(axis=1) if maximize else q.argmin(axis=1)
    applied = q[np.arange(n), pi]
    return pi.astype(np.int64), applied


def gather_policy(row_ptr, col, val, cost, pi):
    """P_pi rows s*m+pi[s] copied into fresh CSR, plus g_pi (sparse.py:243-269)."""
    cost = np.asarray(cost, dtype=np.float64)
    n, m = cost.shape
    rp = np.asarray(row_ptr, dtype=np.int64)
    pi = np.asarray(pi, dtype=np.int64)
    src = np.arange(n, dtype=np.int64) * m + pi
    starts = rp[src]
    lengths = rp[src + 1] - starts
    rp_pi = np.concatenate(([0], np.cumsum(lengths))).astype(np.int64)
    total = int(rp_pi[-1])
    take = np.repeat(starts - rp_pi[:-1], lengths) + np.arange(total, dtype=np.int64)
    g_pi = cost[np.arange(n), pi].copy()
    return rp_pi, np.asarray(col)[take], np.asarray(val)[take], g_pi


def apply_J(rp_pi, col_pi, val_pi, gamma: float, x: np.ndarray) -> np.ndarray:
    """x - gamma * (P_pi x), two-step rounding (sparse.py:294-295)."""
    return np.asarray(x, dtype=np.float64) - gamma * spmv(rp_pi, col_pi, val_pi, x)


# ----------------------------------------------------------------------------
# L3: inner solvers (inner.py)
# ----------------------------------------------------------------------------

@dataclass
class InnerReport:
    iterations: int
    final_linear_residual_2norm: float
    converged: bool
    breakdown: bool
    target_2norm: float


def _identity(r):
    return r


def jacobi(rp_pi, col_pi, val_pi, gamma):
    """Jacobi preconditioner of I - gamma P_pi (inner.py:115-118; diagonal as
    CsrMatrix.diagonal, sparse.py:102-109)."""
    rp = np.asarray(rp_pi, dtype=np.int64)
    n = rp.shape[0] - 1
    d = np.zeros(n)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    col = np.asarray(col_pi, dtype=np.int64)
    mask = rows == col
    d[col[mask]] = np.asarray(val_pi)[mask]
    inv_diag = 1.0 / (1.0 - gamma * d)
    return lambda r: r * inv_diag


def _richardson(apply_a, b, theta0, eff, max_it, scale, pc=_identity):
    """inner.py:216-226."""
    theta = theta0.copy()
    it = 0
    while True:
        r = b - apply_a(theta)
        rn = norm2(r)
        if rn <= eff or it >= max_it or not math.isfinite(rn):
            break
        theta = theta + scale * pc(r)
        it += 1
    return theta, it, rn, False


def _back_substitute(r_mat, rhs):
    """Upper-triangular solve, zero pivot -> 0 (inner.py:286-292)."""
    k = rhs.shape[0]
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        acc = rhs[i] - np.dot(r_mat[i, i + 1:], y[i + 1:])
        y[i] = acc / r_mat[i, i] if r_mat[i, i] != 0.0 else 0.0
    return y


def _gmres(apply_a, b, theta0, eff, max_it, pc=_identity):
    """Restarted GMRES(30), MGS, Givens, estimate-then-verify (inner.py:229-283)."""
    x = theta0.copy()
    it = 0
    r = b - apply_a(x)
    rn = norm2(r)
    est_target = eff
    n = x.shape[0]
    R = GMRES_RESTART
    while rn > eff and it < max_it:
        z = pc(r)
        beta = norm2(z)
        if beta == 0.0 or not math.isfinite(beta):
            break
        V = np.empty((R + 1, n))
        V[0] = z / beta
        H = np.zeros((R + 1, R))
        cs = np.zeros(R)
        sn = np.zeros(R)
        g = np.zeros(R + 1)
        g[0] = beta
        j = 0
        while j < R and it < max_it:
            w = pc(apply_a(V[j]))
            it += 1
            for l in range(j + 1):
                H[l, j] = dot(V[l], w)
                w = w - H[l, j] * V[l]
            hnorm = norm2(w)
            H[j + 1, j] = hnorm
            for l in range(j):
                t = cs[l] * H[l, j] + sn[l] * H[l + 1, j]
                H[l + 1, j] = -sn[l] * H[l, j] + cs[l] * H[l + 1, j]
                H[l, j] = t
            denom = math.hypot(H[j, j], H[j + 1, j])
            if denom == 0.0:
                break
            cs[j], sn[j] = H[j, j] / denom, H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j += 1
            if abs(g[j]) <= est_target or hnorm == 0.0:
                break
            V[j] = w / hnorm
        if j == 0:
            break
        y = _back_substitute(H[:j, :j], g[:j])
        x = x + V[:j].T @ y
        r = b - apply_a(x)
        rn = norm2(r)
        if rn > eff and abs(g[j]) <= est_target:
            if abs(g[j]) == 0.0:
                break
            est_target = abs(g[j]) * (eff / rn) * 0.5
    return x, it, rn, False


def _tighten(est, eff, rn, current):
    """inner.py:453-455."""
    return min(current, est * (eff / rn) * 0.5)


def _bicgstab(apply_a, b, theta0, eff, max_it, pc=_identity):
    """BiCGStab with estimate-then-verify stopping (inner.py:295-373), pc = identity."""
    x = theta0.copy()
    r_true = b - apply_a(x)
    rn = norm2(r_true)
    it = 0
    breakdown = False
    if rn <= eff:
        return x, it, rn, breakdown
    r = np.array(pc(r_true), dtype=np.float64, copy=True)
    rtilde = r.copy()
    rtilde_norm = norm2(rtilde)
    rho = dot(rtilde, r)
    p = r.copy()
    est = norm2(r)
    est_target = eff
    stale = False
    while it < max_it:
        if abs(rho) <= 1e-14 * rtilde_norm * est:
            breakdown = True
            break
        v = pc(apply_a(p))
        sigma = dot(rtilde, v)
        if abs(sigma) <= 1e-14 * rtilde_norm * norm2(v):
            breakdown = True
            break
        alpha = rho / sigma
        s = r - alpha * v
        s_norm = norm2(s)
        if s_norm <= est_target:
            x = x + alpha * p
            it += 1
            r_true = b - apply_a(x)
            rn = norm2(r_true)
            stale = False
            if rn <= eff:
                break
            est_target = _tighten(s_norm, eff, rn, est_target)
            r = np.array(pc(r_true), dtype=np.float64, copy=True)
            rtilde = r.copy()
            rtilde_norm = norm2(rtilde)
            rho = dot(rtilde, r)
            p = r.copy()
            est = norm2(r)
            continue
        t = pc(apply_a(s))
        tt = dot(t, t)
        if tt == 0.0:
            breakdown = True
            break
        omega = dot(t, s) / tt
        if omega == 0.0 or not math.isfinite(omega):
            breakdown = True
            break
        x = x + alpha * p + omega * s
        r = s - omega * t
        it += 1
        stale = True
        est = norm2(r)
        if est <= est_target:
            r_true = b - apply_a(x)
            rn = norm2(r_true)
            stale = False
            if rn <= eff:
                break
            if est == 0.0:
                break
            est_target = _tighten(est, eff, rn, est_target)
        rho_new = dot(rtilde, r)
        beta = (rho_new / rho) * (alpha / omega)
        if not math.isfinite(beta):
            breakdown = True
            break
        rho = rho_new
        p = r + beta * (p - omega * v)
    if stale or breakdown:
        r_true = b - apply_a(x)
        rn = norm2(r_true)
    return x, it, rn, breakdown


def _tfqmr(apply_a, b, theta0, eff, max_it, pc=_identity):
    """Transpose-free QMR with estimate-then-verify stopping (inner.py:376-450)."""
    x = theta0.copy()
    r_true = b - apply_a(x)
    rn = norm2(r_true)
    it = 0
    breakdown = False
    if rn <= eff:
        return x, it, rn, breakdown
    r0 = np.array(pc(r_true), dtype=np.float64, copy=True)
    w = r0.copy()
    y = r0.copy()
    d = np.zeros_like(r0)
    u = pc(apply_a(y))
    v = u.copy()
    tau = norm2(r0)
    r0_norm = tau
    theta_q = 0.0
    eta = 0.0
    rho = dot(r0, r0)
    est_target = eff
    stale = False
    while it < max_it:
        sigma = dot(r0, v)
        if abs(sigma) <= 1e-14 * r0_norm * norm2(v):
            breakdown = True
            break
        alpha = rho / sigma
        if alpha == 0.0 or not math.isfinite(alpha):
            breakdown = True
            break
        converged = False
        for half in (1, 2):
            if half == 2:
                y = y - alpha * v
                u = pc(apply_a(y))
            w = w - alpha * u
            d = y + (theta_q * theta_q * eta / alpha) * d
            if tau == 0.0:
                breakdown = True
                break
            theta_q = norm2(w) / tau
            c = 1.0 / math.sqrt(1.0 + theta_q * theta_q)
            tau = tau * theta_q * c
            eta = c * c * alpha
            x = x + eta * d
            stale = True
            est = tau * math.sqrt(2.0 * it + half + 1.0)
            if est <= est_target:
                r_true = b - apply_a(x)
                rn = norm2(r_true)
                stale = False
                if rn <= eff:
                    converged = True
                    break
                if est == 0.0:
                    breakdown = True
                    break
                est_target = _tighten(est, eff, rn, est_target)
        it += 1
        if converged or breakdown:
            break
        rho_new = dot(r0, w)
        if abs(rho_new) <= 1e-14 * r0_norm * norm2(w):
            breakdown = True
            break
        beta = rho_new / rho
        rho = rho_new
        y = w + beta * y
        v = beta * u + beta * beta * v
        u = pc(apply_a(y))
        v = v + u
    if stale or breakdown:
        r_true = b - apply_a(x)
        rn = norm2(r_true)
    return x, it, rn, breakdown


def inner_solve(rp_pi, col_pi, val_pi, gamma, b, theta0, target, max_it,
                kind="gmres", richardson_scale=1.0, pc="none"):
    """Floor the target, dispatch, report (inner.py:163-213); pc none | jacobi."""
    b = np.asarray(b, dtype=np.float64)
    theta0 = np.asarray(theta0, dtype=np.float64)
    if max_it < 1:
        raise ValueError(f"iteration cap must be >= 1, got {max_it}")
    if target < 0.0:
        raise ValueError(f"residual target must be >= 0, got {target}")
    eff = max(target, TARGET_FLOOR_SCALE * max(1.0, norm2(b)))
    apply_a = lambda x: apply_J(rp_pi, col_pi, val_pi, gamma, x)  # noqa: E731
    P = jacobi(rp_pi, col_pi, val_pi, gamma) if pc == "jacobi" else _identity
    if kind == "richardson":
        theta, its, rn, broke = _richardson(apply_a, b, theta0, eff, max_it, richardson_scale, P)
    elif kind == "gmres":
        theta, its, rn, broke = _gmres(apply_a, b, theta0, eff, max_it, P)
    elif kind == "tfqmr":
        theta, its, rn, broke = _tfqmr(apply_a, b, theta0, eff, max_it, P)
    elif kind == "bicgstab":
        theta, its, rn, broke = _bicgstab(apply_a, b, theta0, eff, max_it, P)
    else:
        raise ValueError(f"oracle has no inner solver {kind!r}")
    return theta, InnerReport(its, rn, bool(rn <= eff) and not broke, broke, eff)


# ----------------------------------------------------------------------------
# L4: outer iPI loop (driver.py:109-209)
# ----------------------------------------------------------------------------

@dataclass
class OracleResult:
    values: np.ndarray
    policy: np.ndarray
    outer_iterations: int
    inner_iterations_total: int
    residual_history: list = field(default_factory=list)
    status: str = CONVERGED


def solve(row_ptr, col, val, cost, gamma, *, maximize=False, tol=1e-8, alpha=1e-4,
          max_outer=1000, max_inner=1000, kind="gmres", ksp_max_it=None,
          richardson_scale=1.0, v0=None, pc="none") -> OracleResult:
    """Algorithm 1: greedy -> inf-norm residual -> tests -> gather -> inner solve.

    Mirrors driver.py:117-209: history appended before the tests; CONVERGED,
    then OUTER_CAP, then the 50-step stall rule; inner target alpha*residual
    (or 0 with cap ksp_max_it); breakdown -> one evaluation sweep.
    """
    cost = np.asarray(cost, dtype=np.float64)
    n = cost.shape[0]
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=np.float64, copy=True)
    history: list[float] = []
    inner_total = 0
    stall = 0
    k = 0
    while True:
        pi, applied = greedy(row_ptr, col, val, cost, gamma, v, maximize)
        res = norm_inf(v - applied)
        history.append(res)
        if res <= tol:
            status = CONVERGED
            break
        if k >= max_outer:
            status = OUTER_CAP
            break
        if k > 0 and res >= history[k - 1]:
            stall += 1
            if stall >= STALL_WINDOW:
                status = STALLED
                break
        else:
            stall = 0
        rp_pi, col_pi, val_pi, g_pi = gather_policy(row_ptr, col, val, cost, pi)
        if ksp_max_it is not None:
            target, cap = 0.0, ksp_max_it
        else:
            target, cap = alpha * res, max_inner
        theta, rep = inner_solve(rp_pi, col_pi, val_pi, gamma, g_pi, v, target, cap,
                                 kind, richardson_scale, pc)
        inner_total += rep.iterations
        if rep.breakdown:
            theta = g_pi + gamma * spmv(rp_pi, col_pi, val_pi, v)
            inner_total += 1
        v = theta
        k += 1
    return OracleResult(values=v, policy=pi, outer_iterations=k,
                        inner_iterations_total=inner_total, residual_history=history,
                        status=status)


def q_gap(row_ptr, col, val, cost, gamma, v, maximize=False) -> np.ndarray:
    """Per-state gap between best and second-best Q (parity tie exemption)."""
    cost = np.asarray(cost, dtype=np.float64)
    n, m = cost.shape
    q = cost + gamma * spmv(row_ptr, col, val, v).reshape(n, m)
    if m == 1:
        return np.full(n, np.inf)
    qs = np.sort(-q if maximize else q, axis=1)
    return qs[:, 1] - qs[:, 0]
