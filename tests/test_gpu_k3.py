"""K3 (planned policy operator, ``ipi_op_*``) against the oracle.

The ring kernels restate numpy's reduceat row sums, so ``spmv`` is asserted
**bitwise** equal to the reference's ``spmv`` (sparse.py:189-215, restated by
``oracle.mdp_oracle.spmv``) and ``apply`` bitwise equal to
``x - gamma*spmv(x)`` (sparse.py:294-295; the identity the reference itself
asserts in test_sparse.py:191-196) — for uniform rows of length 64 (C2/C5's
P_pi), 4 (C3) and 2, ragged tails (row counts not multiples of 4/32), row
shards (state0 > 0), with and without the shared-memory window, and every
forced ring shape.  Variable-length rows (C4) take the generic kernel
(1e-13 relative: row sums in lane order).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import mdp_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.sparse import DeviceOperator  # noqa: E402


def band_rows(n, K, seed, band=300, far=0.1):
    """n x n P with K distinct sorted columns per row: mostly inside a band
    around the row's state, a fraction `far` uniform (C2's locality shape)."""
    assert n >= K
    rng = np.random.default_rng(seed)
    width = min(n, max(2 * band + 1, K))
    lo = np.clip(np.arange(n) - band, 0, n - width)
    band_cols = lo[:, None] + np.argsort(rng.random((n, width)), axis=1)[:, :K]
    cols = np.where(rng.random((n, K)) < far, rng.integers(0, n, size=(n, K)), band_cols)
    cols.sort(axis=1)
    dup = (cols[:, 1:] == cols[:, :-1]).any(axis=1)
    cols[dup] = np.sort(band_cols[dup], axis=1)
    e = rng.standard_exponential((n, K))
    val = e / e.sum(axis=1, keepdims=True)
    rp = np.arange(n + 1, dtype=np.int64) * K
    return rp, cols.reshape(-1), val.reshape(-1)


def dev(rp, col, val):
    return (torch.as_tensor(rp, device="cuda"), torch.as_tensor(col, dtype=torch.int32, device="cuda"),
            torch.as_tensor(val, device="cuda"))


def host(t):
    return t.cpu().numpy()


@pytest.fixture
def env_guard():
    keys = ("IPI_K3_RING", "IPI_K3_WARPS", "IPI_K3_STAGES", "IPI_K3_WAVES", "IPI_K3_HALO",
            "IPI_K3_INTERLEAVE")
    saved = {k: os.environ.get(k) for k in keys}
    yield os.environ
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def check_bitwise(rp, col, val, gamma, *, n_local=None, state0=0, expect=None, seed=0):
    n_glob = len(rp) - 1
    rng = np.random.default_rng(seed)
    x = rng.random(n_glob)
    b = rng.random(n_glob)
    if n_local is None:
        n_local, state0 = n_glob, 0
    sub_rp = rp[state0:state0 + n_local + 1] - rp[state0]
    sl = slice(rp[state0], rp[state0 + n_local])
    sub_col, sub_val = col[sl], val[sl]
    R, Cc, Vv = dev(sub_rp, sub_col, sub_val)
    op = DeviceOperator(R, Cc, Vv, n_local, n_glob, state0, gamma)
    if expect is not None:
        assert op.plan()["variant"] == expect, op.plan()
    xt = torch.as_tensor(x, device="cuda")
    bt = torch.as_tensor(b[state0:state0 + n_local].copy(), device="cuda")
    px = orc.spmv(sub_rp, sub_col, sub_val, x)
    ref_apply = x[state0:state0 + n_local] - gamma * px
    ref_res = b[state0:state0 + n_local] - ref_apply
    got_spmv = host(op.spmv(xt))
    got_apply = host(op.apply(xt))
    got_res = host(op.apply(xt, bt))
    if op.plan()["variant"] == 0:  # generic rows: lane-order row sums
        for g, r in ((got_spmv, px), (got_apply, ref_apply), (got_res, ref_res)):
            np.testing.assert_allclose(g, r, rtol=1e-13, atol=1e-15)
        return op
    assert np.array_equal(got_spmv, px), np.abs(got_spmv - px).max()
    assert np.array_equal(got_apply, ref_apply), np.abs(got_apply - ref_apply).max()
    assert np.array_equal(got_res, ref_res), np.abs(got_res - ref_res).max()
    return op


@pytest.mark.parametrize("n", [64, 65, 67, 1001, 20003])
def test_uring_k64_bitwise(n):
    rp, col, val = band_rows(n, 64, seed=n)
    check_bitwise(rp, col, val, 0.999, expect=1)


@pytest.mark.parametrize("n", [1, 3, 5, 37])
def test_tiny_dense_systems(n):
    rng = np.random.default_rng(n)
    rp = np.arange(n + 1, dtype=np.int64) * n
    col = np.tile(np.arange(n), n)
    e = rng.standard_exponential((n, n))
    check_bitwise(rp, col, (e / e.sum(axis=1, keepdims=True)).reshape(-1), 0.99)


@pytest.mark.parametrize("shape", [(12, 3, 4), (16, 3, 2), (8, 4, 4), (10, 3, 4), (14, 3, 4), (15, 3, 4), (11, 3, 1)])
def test_uring_forced_shapes(shape, env_guard):
    env_guard["IPI_K3_WARPS"], env_guard["IPI_K3_STAGES"], env_guard["IPI_K3_WAVES"] = map(str, shape)
    rp, col, val = band_rows(30001, 64, seed=7)
    op = check_bitwise(rp, col, val, 0.999, expect=1)
    p = op.plan()
    assert (p["threads"] // 32, p["stages"]) == shape[:2]


@pytest.mark.parametrize("shape", [(12, 3, 1), (10, 3, 2), (10, 4, 1), (12, 4, 1), (13, 4, 1)])
@pytest.mark.parametrize("halo,ilv", [(-1, 1), (-1, 0), (100, 1), (300, 0)])
@pytest.mark.parametrize("n", [4099, 30001])
def test_uring_window_and_interleave(shape, halo, ilv, n, env_guard):
    """No-window / capped-window rings with contiguous or interleaved warp rows
    (the autotuner's candidates): still bitwise, shards included."""
    env_guard["IPI_K3_WARPS"], env_guard["IPI_K3_STAGES"], env_guard["IPI_K3_WAVES"] = map(str, shape)
    env_guard["IPI_K3_HALO"], env_guard["IPI_K3_INTERLEAVE"] = str(halo), str(ilv)
    rp, col, val = band_rows(n, 64, seed=n + halo)
    op = check_bitwise(rp, col, val, 0.999, expect=1)
    p = op.plan()
    assert p["interleave"] == ilv and (p["halo"] == -1) == (halo == -1), p
    check_bitwise(rp, col, val, 0.999, n_local=n // 3 + 1, state0=n // 3, expect=1)


def test_uring_shard_rows(env_guard):
    rp, col, val = band_rows(24001, 64, seed=11)
    for state0, n_local in [(0, 8000), (8001, 7999), (16001, 8000), (5, 3)]:
        check_bitwise(rp, col, val, 0.999, n_local=n_local, state0=state0)


@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("n", [7, 33, 4099, 100001])
def test_flat_bitwise(K, n):
    rp, col, val = band_rows(n, K, seed=K * n, band=40)
    check_bitwise(rp, col, val, 0.9999, expect=2)


@pytest.mark.parametrize("shape", [(16, 4, 1), (24, 4, 1), (8, 6, 2), (28, 4, 1), (20, 5, 1)])
def test_flat_forced_shapes(shape, env_guard):
    env_guard["IPI_K3_WARPS"], env_guard["IPI_K3_STAGES"], env_guard["IPI_K3_WAVES"] = map(str, shape)
    rp, col, val = band_rows(70001, 4, seed=3, band=2048)
    check_bitwise(rp, col, val, 0.9999, expect=2)
    check_bitwise(rp, col, val, 0.9999, n_local=30000, state0=20001, expect=2)


def test_generic_forced_equals_ring(env_guard):
    rp, col, val = band_rows(9001, 64, seed=5)
    env_guard["IPI_K3_RING"] = "0"
    R, Cc, Vv = dev(rp, col, val)
    op_g = DeviceOperator(R, Cc, Vv, 9001, 9001, 0, 0.99)
    assert op_g.plan()["variant"] == 0
    env_guard.pop("IPI_K3_RING")
    op_r = DeviceOperator(R, Cc, Vv, 9001, 9001, 0, 0.99)
    assert op_r.plan()["variant"] == 1
    x = torch.rand(9001, dtype=torch.float64, device="cuda")
    a, b = host(op_g.apply(x)), host(op_r.apply(x))
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-15)


def test_variable_rows_generic_c4():
    rp, col, val, cost, spec, n = devgen.build_arrays(4, n=3000)
    mdp = ipi.MdpInstance(n, spec.m, spec.gamma, cost, ipi.CsrMatrix(n * spec.m, n, rp, col, val))
    pi, _, _ = greedy_device(mdp, torch.zeros(n, dtype=torch.float64, device="cuda"), ipi.Mode.MIN)
    P = ipi.gather_policy_matrix(mdp, pi.long())
    op = ipi.PolicyOperator(P, spec.gamma)
    assert op.device_operator().plan()["variant"] == 0
    x = np.random.default_rng(0).random(n)
    ref = orc.apply_J(host(P.row_ptr), host(P.col_idx), host(P.values), spec.gamma, x)
    np.testing.assert_allclose(op.apply(x), ref, rtol=1e-13, atol=1e-14)


def test_unaligned_b_falls_back():
    rp, col, val = band_rows(4001, 64, seed=9)
    R, Cc, Vv = dev(rp, col, val)
    op = DeviceOperator(R, Cc, Vv, 4001, 4001, 0, 0.99)
    x = torch.rand(4001, dtype=torch.float64, device="cuda")
    bb = torch.rand(4002, dtype=torch.float64, device="cuda")[1:]  # 8-byte aligned only
    got = host(op.apply(x, bb))
    ref = host(bb) - (host(x) - 0.99 * orc.spmv(rp, col, val, host(x)))
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15)


def test_empty_operator():
    R = torch.zeros(1, dtype=torch.int64, device="cuda")
    Cc = torch.zeros(1, dtype=torch.int32, device="cuda")
    Vv = torch.zeros(1, dtype=torch.float64, device="cuda")
    op = DeviceOperator(R, Cc, Vv, 0, 5, 5, 0.9)
    x = torch.rand(5, dtype=torch.float64, device="cuda")
    assert op.apply(x).numel() == 0


def test_policy_operator_matches_reference_apply():
    """PolicyOperator.apply (the Python mirror) routes through the ring kernel."""
    rp, col, val = band_rows(5003, 64, seed=1)
    P = ipi.CsrMatrix(5003, 5003, rp, col, val)
    op = ipi.PolicyOperator(P, 0.95)
    x = np.random.default_rng(2).random(5003)
    assert np.array_equal(op.apply(x), orc.apply_J(rp, col, val, 0.95, x))
    assert op.device_operator().plan()["variant"] == 1


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_policy_matrix_bitwise(cfg):
    """BASELINE C2 / C3 at full size: P_pi of the greedy policy of a random V."""
    mdp, spec = devgen.build_instance(cfg)
    v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
    pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
    P = ipi.gather_policy_matrix(mdp, pi.long())
    del mdp
    torch.cuda.empty_cache()
    op = ipi.PolicyOperator(P, spec.gamma)
    plan = op.device_operator().plan()
    assert plan["variant"] == (1 if cfg == 2 else 2), plan
    x = torch.rand(P.rows, dtype=torch.float64, device="cuda")
    got = host(op.apply(x))
    ref = orc.apply_J(host(P.row_ptr), host(P.col_idx), host(P.values), spec.gamma, host(x))
    assert np.array_equal(got, ref)


def test_unaligned_x_falls_back():
    rp, col, val = band_rows(4001, 64, seed=13)
    R, Cc, Vv = dev(rp, col, val)
    op = DeviceOperator(R, Cc, Vv, 4001, 4001, 0, 0.99)
    assert op.plan()["halo"] >= 0  # windowed ring: x chunks need 16-byte alignment
    x = torch.rand(4002, dtype=torch.float64, device="cuda")[1:]
    got = host(op.apply(x))
    ref = host(x) - 0.99 * orc.spmv(rp, col, val, host(x))
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15)


def test_operator_plan_does_not_shrink_k1_smem():
    """Kernel smem limits are process-wide: planning an m = 1 operator view of
    P_pi (smaller rings) must not break the instance's own K1 launches."""
    mdp, spec = devgen.build_instance(3, grid=256)
    v = torch.zeros(mdp.n, dtype=torch.float64, device="cuda")
    pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
    P = ipi.gather_policy_matrix(mdp, pi.long())
    ipi.PolicyOperator(P, spec.gamma).device_operator()
    pi2, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
    torch.cuda.synchronize()
    assert torch.equal(pi, pi2)
    res = ipi.solve(mdp, ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol, max_outer=2))
    assert res.outer_iterations <= 2
