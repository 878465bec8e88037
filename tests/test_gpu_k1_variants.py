"""K1 variants against the oracle on identical inputs.

The planner picks one K1 kernel per instance (``plan()["k1_variant"]``); the
environment switches below force the alternatives so every variant is checked
on the same arrays.  Flat rows (K <= 4) sum each row left to right from 0.0
exactly like numpy's reduceat on a segment shorter than 8 (first element, then
sequential adds), so their Q values are asserted **bitwise** against the
oracle (`bellman.py:44-68` via `oracle.mdp_oracle.greedy`).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import mdp_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402


def uniform_instance(n, m, K, seed):
    """K distinct sorted columns per row inside a 100-state band around s."""
    rng = np.random.default_rng(seed)
    rows = n * m
    s = np.arange(rows) // m
    lo = np.clip(s - 50, 0, n - 100)
    off = np.sort(rng.random((rows, 100)).argsort(axis=1)[:, :K], axis=1)
    col = (lo[:, None] + off).astype(np.int64)
    e = rng.standard_exponential((rows, K))
    val = e / e.sum(axis=1, keepdims=True)
    cost = rng.random((n, m))
    rp = np.arange(rows + 1, dtype=np.int64) * K
    return rp, col.reshape(-1), val.reshape(-1), cost


VARIANTS = {
    "ring6x12": {"IPI_K1_RING": "1", "IPI_RING_STAGES": "6", "IPI_RING_WARPS": "12"},
    "ring5x12": {"IPI_K1_RING": "1", "IPI_RING_STAGES": "5", "IPI_RING_WARPS": "12"},
    "ring4x16": {"IPI_K1_RING": "1", "IPI_RING_STAGES": "4", "IPI_RING_WARPS": "16"},
    "ring8x8": {"IPI_K1_RING": "1", "IPI_RING_STAGES": "8", "IPI_RING_WARPS": "8"},
    "ring4x18": {"IPI_K1_RING": "1", "IPI_RING_STAGES": "4", "IPI_RING_WARPS": "18"},
    "registers": {"IPI_K1_RING": "0"},
}


def expected_variant(variant, K, m):
    """4 (cp.async ring) when the forced shape fits one CTA per SM, else 5."""
    if not variant.startswith("ring"):
        return 5
    S, NW = (int(x) for x in variant[4:].split("x"))
    stage = 32 * K * 12 + 17 * 16
    return 4 if NW * (S * stage + 32 * m * 8) <= 227 * 1024 - 256 else 5


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("K,m,n", [(4, 21, 3000), (4, 1, 20000), (4, 3, 7001), (2, 21, 3000),
                                   (2, 33, 2500), (4, 40, 1500), (2, 5, 9001)])
@pytest.mark.parametrize("maximize", [False, True])
def test_flat_rows_bitwise(monkeypatch, variant, K, m, n, maximize):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    rp, col, val, cost = uniform_instance(n, m, K, seed=K * 1000 + m)
    gamma = 0.97
    mode = ipi.Mode.MAX if maximize else ipi.Mode.MIN
    csr = ipi.CsrMatrix(n * m, n, rp, col, val)
    mdp = ipi.MdpInstance(n=n, m=m, gamma=gamma, stage_cost=cost, transitions=csr, mode=mode)
    plan = mdp.plan()
    assert plan["k1_variant"] == expected_variant(variant, K, m), plan
    v = np.random.default_rng(7).random(n) * 10
    res = ipi.greedy_policy(mdp, v)
    pi_ref, ap_ref = orc.greedy(rp, col, val, cost, gamma, v, maximize)
    np.testing.assert_array_equal(res.policy, pi_ref)
    np.testing.assert_array_equal(res.applied, ap_ref)  # bitwise
    # the fused residual equals the host max |v - TV|
    vd = torch.as_tensor(v, device="cuda")
    _, ap, rb = greedy_device(mdp, vd, mode, with_residual=True)
    assert float(rb.view(torch.float64)[0]) == float(np.max(np.abs(v - ap_ref)))


@pytest.mark.parametrize("variant", ["ring6x12", "ring8x8", "registers"])
def test_flat_rows_ties_first_index(monkeypatch, variant):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    n, m, K = 4000, 6, 4
    rp, col, val, cost = uniform_instance(n, m, K, seed=5)
    # make actions 0, 2, 4 and 1, 3, 5 identical rows: exact ties everywhere
    col2 = col.reshape(n, m, K)
    val2 = val.reshape(n, m, K)
    col2[:, 2] = col2[:, 4] = col2[:, 0]
    val2[:, 2] = val2[:, 4] = val2[:, 0]
    col2[:, 3] = col2[:, 5] = col2[:, 1]
    val2[:, 3] = val2[:, 5] = val2[:, 1]
    cost[:, 2] = cost[:, 4] = cost[:, 0]
    cost[:, 3] = cost[:, 5] = cost[:, 1]
    col, val = col2.reshape(-1), val2.reshape(-1)
    csr = ipi.CsrMatrix(n * m, n, rp, col, val)
    mdp = ipi.MdpInstance(n=n, m=m, gamma=0.9, stage_cost=cost, transitions=csr)
    v = np.random.default_rng(3).random(n)
    res = ipi.greedy_policy(mdp, v)
    pi_ref, ap_ref = orc.greedy(rp, col, val, cost, 0.9, v, False)
    np.testing.assert_array_equal(res.policy, pi_ref)
    assert set(np.unique(res.policy)) <= {0, 1}
    np.testing.assert_array_equal(res.applied, ap_ref)


def test_flat_ring_matches_registers_on_c3_slice(monkeypatch):
    """Pendulum rows (explicit zero weights, periodic wrap) through both flat kernels."""
    from paper_2507_22538_b200 import devgen
    outs = []
    for variant in ("ring6x12", "registers"):
        for k, v in VARIANTS[variant].items():
            monkeypatch.setenv(k, v)
        rp, col, val, cost, spec, nn = devgen.build_arrays(3, grid=256)
        csr = ipi.CsrMatrix(nn * spec.m, nn, rp, col, val)
        mdp = ipi.MdpInstance(nn, spec.m, spec.gamma, cost, csr)
        v = torch.linspace(0, 10, nn, dtype=torch.float64, device="cuda")
        pi, ap, rb = greedy_device(mdp, v, ipi.Mode.MIN, with_residual=True)
        torch.cuda.synchronize()
        outs.append((pi.cpu(), ap.cpu(), int(rb[0])))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


# ---------------------------------------------------------------------------
# uniform rows, K = 64 (C2/C5 shape): cp.async ring (variant 6) vs registers
# ---------------------------------------------------------------------------
def wide_instance(n, m, K, seed, band):
    """K distinct sorted columns per row; band=None -> uniform over [0, n)."""
    rng = np.random.default_rng(seed)
    rows = n * m
    s = np.arange(rows) // m
    if band is None:
        col = np.sort(np.stack([rng.choice(n, K, replace=False) for _ in range(rows)]), axis=1)
    else:
        lo = np.clip(s - band // 2, 0, n - band)
        off = np.sort(rng.random((rows, band)).argsort(axis=1)[:, :K], axis=1)
        col = lo[:, None] + off
    e = rng.standard_exponential((rows, K))
    val = e / e.sum(axis=1, keepdims=True)
    cost = rng.random((n, m))
    rp = np.arange(rows + 1, dtype=np.int64) * K
    return rp, col.astype(np.int64).reshape(-1), val.reshape(-1), cost


UVARIANTS = {
    "uring8x4": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "8", "IPI_URING_STAGES": "4",
                 "IPI_URING_WAVES": "1"},
    "uring10x3": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "10", "IPI_URING_STAGES": "3",
                  "IPI_URING_WAVES": "1"},
    "uring8x4w2": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "8", "IPI_URING_STAGES": "4",
                   "IPI_URING_WAVES": "2"},
    "uring8x4w2d2": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "8", "IPI_URING_STAGES": "4",
                     "IPI_URING_WAVES": "2", "IPI_URING_AHEAD": "2"},
    "uring12x4w4d2": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "12", "IPI_URING_STAGES": "4",
                      "IPI_URING_WAVES": "4", "IPI_URING_AHEAD": "2"},
    "uring12x4w8": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "12", "IPI_URING_STAGES": "4",
                    "IPI_URING_WAVES": "8"},
    "uring11x4w8d2": {"IPI_K1_URING": "1", "IPI_URING_WARPS": "11", "IPI_URING_STAGES": "4",
                      "IPI_URING_WAVES": "8", "IPI_URING_AHEAD": "2"},
    "registers": {"IPI_K1_URING": "0", "IPI_K1_DEEP": "0"},
    "deep": {"IPI_K1_URING": "0", "IPI_K1_DEEP": "1"},
}


@pytest.mark.parametrize("variant", sorted(UVARIANTS))
@pytest.mark.parametrize("m,n,band", [(32, 3000, 400), (4, 20000, 300), (8, 5000, None),
                                      (32, 700, None)])
@pytest.mark.parametrize("maximize", [False, True])
def test_uniform_rows_k64(monkeypatch, variant, m, n, band, maximize):
    for k, v in UVARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    K = 64
    rp, col, val, cost = wide_instance(n, m, K, seed=m * 7 + n, band=band)
    gamma = 0.999
    mode = ipi.Mode.MAX if maximize else ipi.Mode.MIN
    csr = ipi.CsrMatrix(n * m, n, rp, col, val)
    mdp = ipi.MdpInstance(n=n, m=m, gamma=gamma, stage_cost=cost, transitions=csr, mode=mode)
    plan = mdp.plan()
    ring = variant.startswith("uring")
    if ring and plan["k1_variant"] != 6:  # forced shape + resident V window exceed smem
        assert plan["halo"] >= 0, plan
        ring = False
    assert plan["k1_variant"] == (6 if ring else (3 if variant == "deep" else 1)), plan
    v = np.random.default_rng(11).random(n) * 100
    res = ipi.greedy_policy(mdp, v)
    pi_ref, ap_ref = orc.greedy(rp, col, val, cost, gamma, v, maximize)
    if ring:  # numpy reduceat order restated exactly: bitwise
        np.testing.assert_array_equal(res.policy, pi_ref)
        np.testing.assert_array_equal(res.applied, ap_ref)
    else:
        gap = orc.q_gap(rp, col, val, cost, gamma, v, maximize)
        bad = np.flatnonzero(res.policy != pi_ref)
        assert np.all(gap[bad] < 1e-10)
        np.testing.assert_allclose(res.applied, ap_ref, rtol=1e-13, atol=1e-13)
    vd = torch.as_tensor(v, device="cuda")
    pi_d, ap_d, rb = greedy_device(mdp, vd, mode, with_residual=True)
    want = float(np.max(np.abs(v - ap_d.cpu().numpy())))
    assert float(rb.view(torch.float64)[0]) == want


def test_uring_misaligned_v_is_realigned():
    """The ring's V window is staged in 16-byte cp.async chunks: a V view at an
    odd offset goes through an aligned copy and gives the same backup."""
    n, m, K = 6000, 32, 64
    rp, col, val, cost = wide_instance(n, m, K, seed=5, band=400)
    mdp = ipi.MdpInstance(n=n, m=m, gamma=0.999, stage_cost=cost,
                          transitions=ipi.CsrMatrix(n * m, n, rp, col, val))
    plan = mdp.plan()
    assert plan["k1_variant"] == 6 and plan["halo"] >= 0, plan
    v = np.random.default_rng(3).random(n)
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.as_tensor(v, device="cuda")
    pi_a, ap_a, _ = greedy_device(mdp, buf[1:], ipi.Mode.MIN)
    pi_b, ap_b, _ = greedy_device(mdp, torch.as_tensor(v, device="cuda"), ipi.Mode.MIN)
    assert torch.equal(pi_a, pi_b) and torch.equal(ap_a, ap_b)
    pi_ref, ap_ref = orc.greedy(rp, col, val, cost, 0.999, v)
    np.testing.assert_array_equal(ap_a.cpu().numpy(), ap_ref)


def ragged_instance(n, m, seed, lo=0, hi=120):
    """Variable row lengths in [lo, hi) (empty rows included when lo == 0),
    sorted distinct columns, Dirichlet weights."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.integers(lo, hi, size=n * m), n)
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    cols, vals = [], []
    for L in lens:
        c = np.sort(rng.choice(n, size=min(L, n), replace=False))
        e = rng.standard_exponential(len(c))
        cols.append(c)
        vals.append(e / e.sum() if len(c) else e)
    cost = rng.random((n, m))
    return rp, np.concatenate(cols).astype(np.int64), np.concatenate(vals), cost


@pytest.mark.parametrize("m,n,lo,hi", [(5, 3000, 0, 120), (8, 700, 1, 900), (1, 4000, 16, 64),
                                       (3, 257, 0, 40)])
@pytest.mark.parametrize("maximize", [False, True])
def test_variable_rows_generic(m, n, lo, hi, maximize):
    """Generic per-row kernel on ragged rows (empty rows included) vs the oracle."""
    rp, col, val, cost = ragged_instance(n, m, seed=m * 100 + n, lo=lo, hi=hi)
    gamma = 0.99
    mode = ipi.Mode.MAX if maximize else ipi.Mode.MIN
    mdp = ipi.MdpInstance(n=n, m=m, gamma=gamma, stage_cost=cost,
                          transitions=ipi.CsrMatrix(n * m, n, rp, col, val), mode=mode)
    assert mdp.plan()["k1_variant"] == 0
    v = np.random.default_rng(2).random(n) * 50
    res = ipi.greedy_policy(mdp, v)
    pi_ref, ap_ref = orc.greedy(rp, col, val, cost, gamma, v, maximize)
    gap = orc.q_gap(rp, col, val, cost, gamma, v, maximize)
    bad = np.flatnonzero(res.policy != pi_ref)
    assert np.all(gap[bad] < 1e-10)
    np.testing.assert_allclose(res.applied, ap_ref, rtol=1e-13, atol=1e-13)
    vd = torch.as_tensor(v, device="cuda")
    pi_d, ap_d, rb = greedy_device(mdp, vd, mode, with_residual=True)
    assert float(rb.view(torch.float64)[0]) == float(np.max(np.abs(v - ap_d.cpu().numpy())))
    pi2, ap2, _ = greedy_device(mdp, vd, mode)  # reruns are bit-identical
    assert torch.equal(pi_d, pi2) and torch.equal(ap_d, ap2)


def test_no_window_uniform_rows_pick_deep_kernel():
    """Uniform K = 64 rows whose columns span more than a window can hold (C5's
    +-65536 locality) plan the register-deep kernel (all gathers are L2)."""
    from paper_2507_22538_b200 import devgen
    from paper_2507_22538_b200.generators import CONFIGS
    spec = CONFIGS[5]
    n = 1 << 20  # C5's generator and window on a 1M-state slice
    rp, col, val, cost = devgen.locality(n, 8, spec.K, spec.window, 0, 0, 20000)
    from paper_2507_22538_b200.parallel import MdpShard
    sh = MdpShard(n, 8, spec.gamma, 0, cost, ipi.CsrMatrix(20000 * 8, n, rp, col, val))
    plan = sh.plan()
    assert plan["halo"] < 0 and plan["k1_variant"] == 3, plan
    v = torch.rand(n, dtype=torch.float64, device="cuda")
    pol, app, _ = sh.bellman(v)
    rph, colh, valh = (t.cpu().numpy() for t in (rp, col, val))
    pi_ref, ap_ref = orc.greedy(rph, colh, valh, cost.cpu().numpy(), spec.gamma, v.cpu().numpy())
    np.testing.assert_allclose(app.cpu().numpy(), ap_ref, rtol=1e-13, atol=1e-13)
