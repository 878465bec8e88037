"""Row-sharded iPI with the real device kernels at world size 2.

Two processes share the one GPU of the box and talk over gloo (collectives
staged through the host), so no kernel ever waits on another rank's kernel:
this checks the sharded device path (K1 on row blocks with global columns,
K2 on local rows, the planned K3 operator on row blocks with state0 > 0,
the device-resident MGS passes) end to end against the single-process
persistent solver on the same instance.  Also the MGS kernels against torch.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_22538_b200 as ipi  # noqa: E402
from conftest import assert_outer_count  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, kind, q, overlap="1", ortho="cgs2"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), IPI_SHARD_OVERLAP=overlap, IPI_SHARD_ORTHO=ortho)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.parallel import MdpShard, RankContext, ShardOps, solve_sharded
        from paper_2507_22538_b200.generators import CONFIGS
        spec = CONFIGS[2]
        ctx = RankContext.from_env(n)
        lo, hi = ctx.block
        rp, col, val, cost = devgen.locality(n, spec.m, spec.K, spec.window, 0, lo, hi - lo)
        shard = MdpShard(n, spec.m, spec.gamma, lo, cost,
                         ipi.CsrMatrix((hi - lo) * spec.m, n, rp, col, val))
        opts = ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol,
                                inner=ipi.InnerSolver.from_name(kind), max_outer=200)
        res = solve_sharded(ShardOps(shard, ctx), opts, n)
        q.put((rank, res.status.value, res.outer_iterations, res.values.tolist(),
               res.policy.tolist(), res.residual_history))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,overlap,ortho", [("gmres", 8191, "1", "cgs2"),
                                                  ("richardson", 8191, "1", "cgs2"),
                                                  ("gmres", 8192, "1", "cgs2"),
                                                  ("gmres", 8192, "0", "mgs")])
def test_two_ranks_on_device_match_persistent_solver(kind, n, overlap, ortho):
    """n = 8191: unequal blocks (blocking gather); n = 8192: equal blocks, the
    split operator's all-gather runs async (overlap) or the unsplit path."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, kind, q, overlap, ortho))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, st0, k0, v0, p0, h0), (_, st1, k1, v1, p1, h1) = out
    assert (st0, k0, p0, h0) == (st1, k1, p1, h1) and v0 == v1  # ranks agree exactly
    mdp, spec = devgen.build_instance(2, n=n)
    ref = ipi.solve(mdp, ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol,
                                          inner=ipi.InnerSolver.from_name(kind), max_outer=200))
    assert st0 == ref.status.value
    assert_outer_count(type("R", (), {"outer_iterations": k0, "residual_history": h0})(), ref,
                       spec.atol, spec.alpha)
    np.testing.assert_allclose(v0, ref.values, rtol=1e-8, atol=1e-8)
    np.testing.assert_array_equal(p0, ref.policy)


@pytest.mark.parametrize("n", [1, 1000, 1_000_003])
def test_mgs_kernels_match_torch(n):
    from paper_2507_22538_b200.parallel import ShardVectorOps, ShardOps
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    v2 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    dev_ops = ShardOps.__new__(ShardOps)
    ref_ops = ShardVectorOps()
    d = dev_ops.dot_partial(a, b)
    np.testing.assert_allclose(d.item(), torch.dot(a, b).item(), rtol=1e-13)
    parts = torch.tensor([0.25, -0.5, 0.125], dtype=torch.float64, device="cuda")
    w1, w2 = a.clone(), a.clone()
    h1, nx1 = dev_ops.mgs_pass(parts, w1, b, v2)
    h2, nx2 = ref_ops.mgs_pass(parts, w2, b, v2)
    assert h1.item() == h2.item()
    assert torch.equal(w1, w2)  # same elementwise roundings
    np.testing.assert_allclose(nx1.item(), nx2.item(), rtol=1e-13)
    _, nn = dev_ops.mgs_pass(parts[:1], w1, b, None)
    np.testing.assert_allclose(nn.item(), torch.dot(w1, w1).item(), rtol=1e-13)
    # deterministic: rerun bit-identical
    assert dev_ops.dot_partial(a, b).item() == d.item()


@pytest.mark.parametrize("state0,n_local", [(0, 3000), (3000, 2000), (7000, 1192)])
def test_split_operator_halves_equal_unsplit(state0, n_local):
    """Local-column / remote-column split of a rank's P_pi rows: the two halves
    (ipi_csr_split_local, ipi_op_apply_partial) reproduce the unsplit apply to
    1e-13 (only the row-sum association differs)."""
    from paper_2507_22538_b200.parallel import SplitShardOperator
    from paper_2507_22538_b200.sparse import DeviceOperator
    from paper_2507_22538_b200.generators import CONFIGS
    spec = CONFIGS[2]
    n = 8192
    rp, col, val, cost = devgen.locality(n, 1, spec.K, 600, 0, state0, n_local)
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n_local, dtype=torch.float64, device="cuda")
    whole = DeviceOperator(rp, col, val, n_local, n, state0, 0.99)
    sp = SplitShardOperator(rp, col, val, n_local, n, state0, 0.99)
    plan = sp.plan()
    assert plan["nnz_local"] + plan["nnz_remote"] == n_local * spec.K
    assert plan["nnz_remote"] > 0 or n_local == n
    for bb in (None, b):
        y_loc = sp.local.spmv(x[state0:state0 + n_local].contiguous())
        got = sp.remote.apply_partial(x, y_loc, bb)
        ref = whole.apply(x, bb)
        torch.testing.assert_close(got, ref, rtol=1e-13, atol=1e-14)



def _sis_worker(rank, world, port, q, halo_frac):
    """C4-shaped (SIS, variable rows with banded columns) sharded solve; with
    IPI_HALO_FRAC = 1 the V exchange is point-to-point halos, not all-gathers."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), IPI_HALO_FRAC=halo_frac)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.parallel import MdpShard, RankContext, ShardOps, solve_sharded
        mdp, spec = devgen.build_instance(4, population=2000)
        n, m = mdp.n, mdp.m
        ctx = RankContext.from_env(n)
        lo, hi = ctx.block
        rp, col, val = mdp.transitions.row_ptr, mdp.transitions.col_idx, mdp.transitions.values
        a, b = int(rp[lo * m]), int(rp[hi * m])
        sub = ipi.CsrMatrix((hi - lo) * m, n, (rp[lo * m:hi * m + 1] - a).clone(),
                            col[a:b].clone(), val[a:b].clone())
        shard = MdpShard(n, m, spec.gamma, lo, mdp.stage_cost[lo:hi].clone(), sub)
        ops = ShardOps(shard, ctx)
        res = solve_sharded(ops, ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol), n)
        q.put((rank, ops.halo.enabled, ops.halo.bytes_received(), res.status.value,
               res.outer_iterations, res.values.tolist(), res.policy.tolist(),
               res.residual_history))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("halo_frac", ["1.0", "0.0"])
def test_two_ranks_sis_halo_exchange(halo_frac):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sis_worker, args=(r, 2, port, q, halo_frac)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, en0, b0, st0, k0, v0, p0, h0), (_, en1, b1, st1, k1, v1, p1, _) = out
    assert en0 == en1 == (halo_frac == "1.0")
    if en0:  # a halo, not the other rank's whole block
        assert 0 < b0 < 8 * 1001 and 0 < b1 < 8 * 1001
    assert (st0, k0, p0) == (st1, k1, p1) and v0 == v1
    mdp, spec = devgen.build_instance(4, population=2000)
    ref = ipi.solve(mdp, ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol))
    assert st0 == ref.status.value
    assert_outer_count(type("R", (), {"outer_iterations": k0, "residual_history": h0})(), ref,
                       spec.atol, spec.alpha)
    np.testing.assert_allclose(v0, ref.values, rtol=1e-8, atol=1e-8 * np.abs(ref.values).max())
    np.testing.assert_array_equal(p0, ref.policy)
