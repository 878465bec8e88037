"""Seeded instance generators for the five BASELINE configs.

The reference's own generators (``problems.py:56-488``) do not produce the
BASELINE.json configs, so these recipes are new and pinned here
(Appendix-B decisions):

* C1 ``random_dirichlet``: host numpy, ``default_rng(seed)``; cost first, then
  per row ``sort(choice(n, K, replace=False))`` and Exp(1) weights normalised
  (Dirichlet(1)).  Small enough to build on the host and upload.
* C2 / C5 ``random_locality``: counter-based Philox4x32-10 keyed by
  ``(seed, global row)`` so every shard can build its own rows and the
  instance does not depend on the rank count.  Candidates are local with
  probability 0.9 (uniform in the window ``[s-W, s+W]`` clipped to
  ``[0, n)``) else uniform over ``[0, n)``; the first ``K`` distinct
  candidates are kept and sorted; weights are normalised Exp(1).
  Built on the device (``ipi_gen_locality``); a host restatement of the same
  counter recipe exists for small cross-checks.
* C3 ``pendulum``: angle-major state index ``i_theta * N + j_omega``,
  theta_i = -pi + i*2pi/N (periodic), omega_j = linspace(-10, 10, N),
  torque linspace(-3, 3, n_a); omega' = omega + dt*(9.81 sin theta + u),
  theta' = theta + dt*omega' wrapped into [-pi, pi); omega' clipped to
  [-10, 10] only for the grid mapping; bilinear weights over the 4
  surrounding nodes, exactly 4 sorted distinct columns per row (explicit zero
  weights kept).  Cost theta^2 + 0.1 omega^2 + 0.01 u^2.
* C4 ``sis``: s = number infected; s' = s - Bin(s, 0.1) +
  Bin(N-s, 1-exp(-beta_a s/N)); exact fp64 convolution of the two pmfs,
  entries < 1e-14 dropped, row renormalised; cost s/N + w_a.

Host builders return numpy arrays ``(row_ptr int64, col int32, val f64,
cost f64 (n, m))``; device builders return torch CUDA tensors in the same
layout.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ----------------------------------------------------------------------------
# config registry (BASELINE.json "configs")
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    kind: str          # dirichlet | locality | pendulum | sis
    n: int
    m: int
    K: int             # nnz per row (0 = variable)
    gamma: float
    window: int = 0    # locality half-window W
    grid: int = 0      # pendulum grid points per dimension
    population: int = 0
    alpha: float = 1e-4
    atol: float = 1e-8


CONFIGS = {
    1: ConfigSpec("c1_random_dirichlet", "dirichlet", 10_000, 20, 50, 0.99),
    2: ConfigSpec("c2_random_locality", "locality", 1_048_576, 32, 64, 0.999, window=4096),
    3: ConfigSpec("c3_pendulum", "pendulum", 2048 * 2048, 21, 4, 0.9999, grid=2048),
    4: ConfigSpec("c4_sis", "sis", 20_001, 5, 0, 0.9999, population=20_000),
    5: ConfigSpec("c5_random_locality_sharded", "locality", 16_777_216, 16, 64, 0.999,
                  window=65_536),
}

SIS_BETAS = (0.5, 0.35, 0.25, 0.15, 0.05)
SIS_WEIGHTS = (0.0, 0.2, 0.5, 1.0, 2.0)
SIS_RECOVERY = 0.1
SIS_TRUNCATION = 1e-14
LOCAL_PROB_NUM = 3865470566  # floor(0.9 * 2**32): candidate is local iff x0 < this

# Philox stream tags (4th counter word) so the three uses never overlap.
TAG_CAND = 0xC2C5
TAG_WEIGHT = 0xD1D1
TAG_COST = 0xC057


# ----------------------------------------------------------------------------
# Philox4x32-10 (Salmon et al., SC'11) — vectorised numpy restatement
# ----------------------------------------------------------------------------

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x32 rounds over broadcastable uint32 counters."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = (x.copy() for x in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = _M0 * c0.astype(np.uint64)
            p1 = _M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def _u53_open0(x0, x1):
    """53-bit uniform in (0, 1] from two words."""
    bits = (x1.astype(np.uint64) << np.uint64(21)) | (x0.astype(np.uint64) >> np.uint64(11))
    return (bits.astype(np.float64) + 1.0) * (2.0 ** -53)


def _u53_closed0(x0, x1):
    """53-bit uniform in [0, 1) from two words."""
    bits = (x1.astype(np.uint64) << np.uint64(21)) | (x0.astype(np.uint64) >> np.uint64(11))
    return bits.astype(np.float64) * (2.0 ** -53)


def _umulhi64(a: int, b: int) -> int:
    return (a * b) >> 64


# ----------------------------------------------------------------------------
# C1: Dirichlet random (host)
# ----------------------------------------------------------------------------

def random_dirichlet(n: int, m: int, K: int, seed: int = 0):
    """BASELINE config 1 recipe; host numpy, deterministic."""
    if not (1 <= K <= n):
        raise ValueError(f"K must lie in [1, {n}]")
    rng = np.random.default_rng(seed)
    cost = rng.random((n, m))
    rows = n * m
    col = np.empty(rows * K, dtype=np.int32)
    val = np.empty(rows * K, dtype=np.float64)
    for r in range(rows):
        c = np.sort(rng.choice(n, K, replace=False))
        e = rng.standard_exponential(K)
        col[r * K:(r + 1) * K] = c
        val[r * K:(r + 1) * K] = e / e.sum()
    row_ptr = np.arange(rows + 1, dtype=np.int64) * K
    return row_ptr, col, val, cost


# ----------------------------------------------------------------------------
# C2 / C5: locality random (host restatement of the device counter recipe)
# ----------------------------------------------------------------------------

def locality_row_host(s: int, a: int, n: int, m: int, K: int, W: int, seed: int):
    """One row of the locality recipe; identical integer stream to the kernel."""
    r = s * m + a
    r_lo, r_hi = r & 0xFFFFFFFF, r >> 32
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    lo = max(0, s - W)
    hi = min(n - 1, s + W)
    chosen: list[int] = []
    seen: set[int] = set()
    t = 0
    while len(chosen) < K:
        batch = np.arange(t, t + 64, dtype=np.uint32)
        x0, x1, x2, _ = philox4x32(batch, r_lo, r_hi, TAG_CAND, k0, k1)
        for i in range(64):
            pos = (int(x2[i]) << 32) | int(x1[i])
            if int(x0[i]) < LOCAL_PROB_NUM:
                c = lo + _umulhi64(pos, hi - lo + 1)
            else:
                c = _umulhi64(pos, n)
            if c not in seen:
                seen.add(c)
                chosen.append(c)
                if len(chosen) == K:
                    break
        t += 64
    cols = np.array(sorted(chosen), dtype=np.int32)
    w0, w1, _, _ = philox4x32(np.arange(K, dtype=np.uint32), r_lo, r_hi, TAG_WEIGHT, k0, k1)
    e = -np.log(_u53_open0(w0, w1))
    total = 0.0
    for x in e:          # sequential sum, same order as the kernel
        total += float(x)
    vals = e / total
    c0, c1, _, _ = philox4x32(np.zeros(1, np.uint32), r_lo, r_hi, TAG_COST, k0, k1)
    cost = float(_u53_closed0(c0, c1)[0])
    return cols, vals, cost


def random_locality_host(n: int, m: int, K: int, W: int, seed: int = 0):
    """Whole instance on the host (small n only; the kernel builds full sizes)."""
    rows = n * m
    col = np.empty(rows * K, dtype=np.int32)
    val = np.empty(rows * K, dtype=np.float64)
    cost = np.empty((n, m))
    for s in range(n):
        for a in range(m):
            r = s * m + a
            c, v, g = locality_row_host(s, a, n, m, K, W, seed)
            col[r * K:(r + 1) * K] = c
            val[r * K:(r + 1) * K] = v
            cost[s, a] = g
    return np.arange(rows + 1, dtype=np.int64) * K, col, val, cost


# ----------------------------------------------------------------------------
# C3: pendulum (host, vectorised)
# ----------------------------------------------------------------------------

PEND_DT = 0.01
PEND_G = 9.81
PEND_OMEGA = 10.0
PEND_TORQUE = 3.0


def pendulum_host(N: int, n_actions: int = 21):
    """BASELINE config 3 recipe on the host (bit-for-bit the kernel's formula
    up to libm differences in sin)."""
    n = N * N
    h_t = 2.0 * math.pi / N
    h_o = 2.0 * PEND_OMEGA / (N - 1)
    i_t, j_o = np.divmod(np.arange(n, dtype=np.int64), N)
    theta = -math.pi + i_t * h_t
    omega = -PEND_OMEGA + j_o * h_o
    if n_actions == 1:
        u = np.zeros(1)
    else:
        u = -PEND_TORQUE + np.arange(n_actions) * (2.0 * PEND_TORQUE / (n_actions - 1))
    cost = (theta * theta + 0.1 * (omega * omega))[:, None] + (0.01 * (u * u))[None, :]
    th = np.repeat(theta, n_actions)
    om = np.repeat(omega, n_actions)
    uu = np.tile(u, n)
    om_next = om + PEND_DT * (PEND_G * np.sin(th) + uu)
    th_next = th + PEND_DT * om_next
    a = (th_next + math.pi) / h_t          # fractional angle index, may leave [0, N)
    fa = np.floor(a)
    ft = a - fa
    i0 = np.mod(fa.astype(np.int64), N)
    i1 = (i0 + 1) % N
    oc = np.clip(om_next, -PEND_OMEGA, PEND_OMEGA)
    t = (oc + PEND_OMEGA) / h_o
    j0 = np.clip(np.floor(t).astype(np.int64), 0, N - 2)
    fo = t - j0
    j1 = j0 + 1
    ca = np.stack([i0 * N + j0, i0 * N + j1, i1 * N + j0, i1 * N + j1], axis=1)
    wa = np.stack([(1.0 - ft) * (1.0 - fo), (1.0 - ft) * fo, ft * (1.0 - fo), ft * fo], axis=1)
    # wrap (i0 = N-1, i1 = 0) puts the i1 block first in ascending order
    wrap = i1 < i0
    ca[wrap] = ca[wrap][:, [2, 3, 0, 1]]
    wa[wrap] = wa[wrap][:, [2, 3, 0, 1]]
    rows = n * n_actions
    return (np.arange(rows + 1, dtype=np.int64) * 4, ca.ravel().astype(np.int32),
            wa.ravel().copy(), cost)


# ----------------------------------------------------------------------------
# C4: SIS epidemic (host; small populations — the kernel builds N = 20,000)
# ----------------------------------------------------------------------------

PMF_FLOOR = 1e-300


def _binom_pmf(k_max: int, p: float) -> np.ndarray:
    """Binomial(k_max, p) pmf over 0..k_max in log space (lgamma)."""
    if p <= 0.0 or k_max == 0:
        out = np.zeros(k_max + 1)
        out[0] = 1.0
        return out
    if p >= 1.0:
        out = np.zeros(k_max + 1)
        out[k_max] = 1.0
        return out
    k = np.arange(k_max + 1)
    lg = np.array([math.lgamma(x + 1.0) for x in range(k_max + 1)])
    logp = lg[k_max] - lg[k] - lg[k_max - k] + k * math.log(p) + (k_max - k) * math.log1p(-p)
    return np.exp(logp)


def sis_row_host(s: int, a: int, N: int):
    """One convolution row: successor distribution of s' = s - X + Y."""
    px = _binom_pmf(s, SIS_RECOVERY)                              # X recoveries
    py = _binom_pmf(N - s, -math.expm1(-SIS_BETAS[a] * s / N))    # Y infections
    conv = np.convolve(px[::-1], py)   # index k <-> s' = k  (s - x + y, x reversed)
    keep = np.flatnonzero(conv >= SIS_TRUNCATION)
    vals = conv[keep]
    return keep.astype(np.int32), vals / vals.sum()


def sis_host(N: int):
    n, m = N + 1, len(SIS_BETAS)
    cols, vals, lens = [], [], []
    for s in range(n):
        for a in range(m):
            c, v = sis_row_host(s, a, N)
            cols.append(c)
            vals.append(v)
            lens.append(c.size)
    row_ptr = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    cost = (np.arange(n) / N)[:, None] + np.array(SIS_WEIGHTS)[None, :]
    return row_ptr, np.concatenate(cols), np.concatenate(vals), cost


def build_host(cfg: int | ConfigSpec, *, n: int | None = None, grid: int | None = None,
               population: int | None = None, seed: int = 0):
    """Host arrays for a (possibly scaled) config: (row_ptr, col, val, cost, spec)."""
    spec = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if spec.kind == "dirichlet":
        nn = n or spec.n
        return (*random_dirichlet(nn, spec.m, spec.K, seed), spec)
    if spec.kind == "locality":
        nn = n or spec.n
        return (*random_locality_host(nn, spec.m, spec.K, spec.window, seed), spec)
    if spec.kind == "pendulum":
        return (*pendulum_host(grid or spec.grid, spec.m), spec)
    if spec.kind == "sis":
        return (*sis_host(population or spec.population), spec)
    raise ValueError(spec.kind)
