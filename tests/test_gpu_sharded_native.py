"""The native row-sharded iPI driver (ipi_solve_sharded) against the C oracle.

Ranks are processes sharing the box's one GPU and talking over gloo (the
driver's two collectives staged through the host by NativeComm's callbacks),
so no kernel ever waits on another rank's kernel; with NCCL (one process per
GPU) the same driver runs the collectives as NCCL kernels.  The instance is
C5-shaped: the locality recipe with a window much narrower than n, so each
rank's rows read mostly their own block plus ~10% uniform columns from every
other rank (the local/remote mix of the sharded-only config at reduced n).

Bars (north star): status and outer count equal to the oracle's; V within
1e-8 relative; the greedy policy equal outside Q ties (gap < 1e-10); the
returned V's Bellman residual (recomputed by the oracle) <= atol; every rank
returns bit-identical results.
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
from paper_2507_22538_b200 import devgen  # noqa: E402

TIE_GAP = 1e-10
# C5's recipe (64 nnz per row, 0.9 local probability, Dirichlet(1), gamma 0.999)
# at n = 32768 with a +-512 window: window << block at every world size tested
N, M, K, W, GAMMA = 32768, 16, 64, 512, 0.999


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, n, kind, mode, pc, v0_seed, ksp=None):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.parallel import MdpShard, RankContext, solve_sharded_native
        ctx = RankContext.from_env(n)
        lo, hi = ctx.block
        rp, col, val, cost = devgen.locality(n, M, K, W, 0, lo, hi - lo)
        shard = MdpShard(n, M, GAMMA, lo, cost, ipi.CsrMatrix((hi - lo) * M, n, rp, col, val))
        v0 = None if v0_seed is None else np.random.default_rng(v0_seed).random(n) * 100
        opts = ipi.SolveOptions(alpha=1e-4, tol=1e-8, inner=ipi.InnerSolver.from_name(kind),
                                pc=ipi.Preconditioner.from_name(pc),
                                mode=ipi.Mode.from_name(mode), max_outer=300, v0=v0, ksp_max_it=ksp)
        res = solve_sharded_native(shard, ctx, opts)
        q.put((rank, res.status.value, res.outer_iterations, res.values.tolist(),
               res.policy.tolist(), res.residual_history, res.inner_iterations_total))
    except Exception as exc:  # pragma: no cover - reported by the parent
        q.put((rank, "error", repr(exc), None, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, n=N, kind="gmres", mode="min", pc="none", v0_seed=None, ksp=None):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, kind, mode, pc, v0_seed, ksp))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=900) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    assert all(o[1] != "error" for o in out), out
    for p in procs:
        assert p.exitcode == 0
    first = out[0]
    for o in out[1:]:  # every rank holds bit-identical scalars and results
        assert o[1:] == first[1:]
    return first


def _oracle(n, mode, pc, kind, v0_seed):
    from oracle import c_oracle as co
    rp, col, val, cost = (t.cpu().numpy() for t in devgen.locality(n, M, K, W, 0, 0, n))
    v0 = None if v0_seed is None else np.random.default_rng(v0_seed).random(n) * 100
    ref = co.solve(rp, col, val, cost, GAMMA, maximize=mode == "max", tol=1e-8, alpha=1e-4,
                   kind=kind, v0=v0, max_outer=300)
    return ref, (rp, col, val, cost)


def _assert_parity(got, ref, arrays, mode):
    from oracle import c_oracle as co
    _, status, outer, values, policy, history, _ = got
    rp, col, val, cost = arrays
    assert status == ref.status
    assert outer == ref.outer_iterations
    assert len(history) == len(ref.residual_history)
    values = np.asarray(values)
    scale = max(1.0, np.abs(ref.values).max())
    np.testing.assert_allclose(values, ref.values, rtol=1e-8, atol=1e-8 * scale)
    diff = np.flatnonzero(np.asarray(policy) != ref.policy)
    if diff.size:
        pv = co.spmv(rp, col, val, ref.values).reshape(-1, M)
        q = np.sort(cost[diff] + GAMMA * pv[diff], axis=1)
        gap = q[:, 1] - q[:, 0] if mode == "min" else q[:, -1] - q[:, -2]
        assert np.all(gap < TIE_GAP), diff[:10]
    _, _, r = co.greedy(rp, col, val, cost, GAMMA, values, maximize=mode == "max")
    assert r <= 1e-8 * 1.0001
    # a-posteriori certificate ||V - V*||_inf <= ||r(V)||_inf / (1 - gamma)
    assert np.max(np.abs(values - ref.values)) <= (r + 1e-8) / (1 - GAMMA) + 1e-12


@pytest.mark.parametrize("world", [1, 2, 4])
def test_c5_shaped_sharded_solve_matches_c_oracle(world):
    got = _run(world)
    ref, arrays = _oracle(N, "min", "none", "gmres", None)
    _assert_parity(got, ref, arrays, "min")


def test_unequal_blocks_richardson_jacobi():
    """n mod R != 0 (NCCL would use per-rank broadcasts), Richardson with the
    Jacobi preconditioner across 3 ranks vs the oracle's MIN solution (the
    Richardson path changes the iterates, not the fixed point)."""
    from oracle import c_oracle as co
    n = 3 * 4096 + 1
    got = _run(3, n=n, kind="richardson", pc="jacobi")
    ref, (rp, col, val, cost) = _oracle(n, "min", "none", "gmres", None)
    _, status, _, values, _, _, _ = got
    assert status == "converged"
    # another inner solver stops at other iterates: both are certified within
    # ||r(V)||_inf / (1 - gamma) of V*, so they agree to twice that bound
    _, _, r = co.greedy(rp, col, val, cost, GAMMA, np.asarray(values))
    assert r <= 1e-8 * 1.0001
    assert np.max(np.abs(np.asarray(values) - ref.values)) <= 2e-8 / (1 - GAMMA)


def test_mode_override_and_warm_start():
    """opts.mode = MAX on MIN-built shards and a seeded v0 (the reference's
    driver.py:117-123): both honoured, against the oracle's MAX solve from the
    same v0."""
    n = 2 * 4096
    got = _run(2, n=n, mode="max", v0_seed=11)
    ref, arrays = _oracle(n, "max", "none", "gmres", 11)
    _assert_parity(got, ref, arrays, "max")


def test_gmres_jacobi_two_ranks():
    from oracle import c_oracle as co
    n = 2 * 4096
    got = _run(2, n=n, pc="jacobi")
    ref, (rp, col, val, cost) = _oracle(n, "min", "none", "gmres", None)
    _, status, _, values, policy, _, _ = got
    assert status == "converged"
    _, _, r = co.greedy(rp, col, val, cost, GAMMA, np.asarray(values))
    assert r <= 1e-8 * 1.0001
    assert np.max(np.abs(np.asarray(values) - ref.values)) <= 2e-8 / (1 - GAMMA)


@pytest.mark.parametrize("ksp", [5, 33])
def test_fixed_inner_iterations_two_ranks(ksp):
    """ksp_max_it (driver.py:170-175): exactly that many GMRES iterations per
    outer step, the cap falling inside a cycle (5) or after a restart (33) —
    with the host enqueueing one step ahead, the device must stop on the cap
    and the step enqueued past it must be a no-op."""
    from oracle import c_oracle as co
    n = 2 * 4096
    got = _run(2, n=n, ksp=ksp)
    rp, col, val, cost = (t.cpu().numpy() for t in devgen.locality(n, M, K, W, 0, 0, n))
    ref = co.solve(rp, col, val, cost, GAMMA, tol=1e-8, alpha=1e-4, kind="gmres", max_outer=300,
                   ksp_max_it=ksp)
    _, status, outer, values, _, history, inner = got
    assert status == ref.status
    assert outer == ref.outer_iterations
    assert inner == ksp * outer == ref.inner_iterations_total
    scale = max(1.0, np.abs(ref.values).max())
    np.testing.assert_allclose(np.asarray(values), ref.values, rtol=1e-8, atol=1e-8 * scale)


def test_unsupported_kinds_raise():
    from paper_2507_22538_b200.parallel import MdpShard, RankContext, solve_sharded_native
    n = 1024
    rp, col, val, cost = devgen.locality(n, M, K, W, 0, 0, n)
    shard = MdpShard(n, M, GAMMA, 0, cost, ipi.CsrMatrix(n * M, n, rp, col, val))
    ctx = RankContext.from_env(n)
    for kind in ("tfqmr", "bicgstab"):
        with pytest.raises(NotImplementedError):
            solve_sharded_native(shard, ctx, ipi.SolveOptions(inner=ipi.InnerSolver.from_name(kind)))
    with pytest.raises(NotImplementedError):
        solve_sharded_native(shard, ctx, ipi.SolveOptions(pc=ipi.Preconditioner.SOR_FORWARD))


def _cb_trans(s, a):
    rng = np.random.default_rng(1000 * s + a)
    k = 1 + (s * 7 + a) % 9
    cols = rng.choice(300, size=k, replace=False)
    p = rng.random(k) + 0.1
    return cols.tolist(), (p / p.sum()).tolist()


def _cb_cost(s, a):
    return ((s * 13 + a * 7) % 17) / 17.0


def _callback_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.frontend import build_shard_from_callbacks
        from paper_2507_22538_b200.parallel import RankContext, solve_sharded_native
        ctx = RankContext.from_env(300)
        shard = build_shard_from_callbacks(300, 3, 0.95, _cb_cost, _cb_trans, ctx)
        res = solve_sharded_native(shard, ctx, ipi.SolveOptions(max_outer=300))
        q.put((rank, res.status.value, res.outer_iterations, res.values.tolist(),
               res.policy.tolist(), res.residual_history, res.inner_iterations_total))
    finally:
        dist.destroy_process_group()


def test_per_rank_callback_construction_solves_like_one_process():
    """build_shard_from_callbacks at world 2 (each rank evaluates only its
    block, problems.py:419-488) -> the native sharded solve reproduces the
    one-process solve of createTransitionProbabilityTensor's instance."""
    import paper_2507_22538_b200.frontend as mf
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_callback_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=600) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0][1:] == out[1][1:]
    P = mf.createTransitionProbabilityTensor(300, 3, _cb_trans)
    cost = mf.createStageCostMatrix(300, 3, _cb_cost)
    mdp = ipi.MdpInstance(n=300, m=3, gamma=0.95, stage_cost=cost.data, transitions=P.data)
    ref = ipi.solve(mdp, ipi.SolveOptions(max_outer=300))
    _, status, outer, values, policy, _, _ = out[0]
    assert status == ref.status.value and outer == ref.outer_iterations
    np.testing.assert_allclose(values, ref.values, rtol=1e-8, atol=1e-8)
    np.testing.assert_array_equal(policy, ref.policy)


def _nccl_world1_worker(q, force):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1",
                      IPI_COMM_FORCE_NCCL=force)
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        dist.barrier()
    except Exception as exc:  # no usable NCCL bootstrap on this box: nothing to exercise
        q.put(("skip", repr(exc), None, None, None, None))
        return
    try:
        from paper_2507_22538_b200.parallel import MdpShard, NativeComm, RankContext, solve_sharded_native
        n = 8191  # odd: the last 16-byte chunk of every vector is half-filled
        ctx = RankContext.from_env(n)
        lo, hi = ctx.block
        rp, col, val, cost = devgen.locality(n, M, K, W, 0, lo, hi - lo)
        shard = MdpShard(n, M, GAMMA, lo, cost, ipi.CsrMatrix((hi - lo) * M, n, rp, col, val))
        comm = NativeComm(ctx)
        res = solve_sharded_native(shard, ctx, ipi.SolveOptions(alpha=1e-4, tol=1e-8, max_outer=300),
                                   comm=comm)
        q.put((comm.kind, res.status.value, res.outer_iterations, res.inner_iterations_total,
               res.values.tolist(), res.policy.tolist()))
    except Exception as exc:  # pragma: no cover - reported by the parent
        q.put(("error", repr(exc), None, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_nccl_binding_on_a_one_rank_communicator():
    """The NCCL path of ipi_comm (comm_nccl.cu: dlopen'd ncclAllGather and the
    grouped ncclBroadcast all-gather-v, torch's own communicator through
    ProcessGroupNCCL._comm_ptr) exercised on the one GPU there is: a one-rank
    communicator, with IPI_COMM_FORCE_NCCL sending the driver's exchanges
    through NCCL instead of the one-rank device copies.  Results must be
    bitwise those of the copy path (a one-rank all-gather / broadcast is a
    copy): this checks symbol resolution, argument order, the dtype enum and
    stream ordering, not multi-GPU behaviour."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    outs = {}
    for force in ("0", "1", "2"):  # copies / ncclAllGather / grouped ncclBroadcast
        q = ctx.Queue()
        p = ctx.Process(target=_nccl_world1_worker, args=(q, force))
        p.start()
        outs[force] = q.get(timeout=600)
        p.join(timeout=120)
        if outs[force][0] == "skip":
            pytest.skip(f"NCCL process group unavailable here: {outs[force][1]}")
        assert outs[force][0] != "error", outs[force]
        assert p.exitcode == 0
    assert outs["0"][0] == "local" and outs["1"][0] == "nccl" and outs["2"][0] == "nccl"
    assert outs["1"][1:] == outs["0"][1:]
    assert outs["2"][1:] == outs["0"][1:]
    assert outs["0"][1] == "converged"
