"""CPU-only tests: C ABI surface, host logic of the reference-facing API,
generators, and the row-block sharding plumbing (gloo, world size 2)."""

from __future__ import annotations

import math
import os
import re
import socket
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2507_22538_b200 as ipi
from paper_2507_22538_b200 import _lib, frontend as mf, generators as gen
from paper_2507_22538_b200.model import make_partition

REPO = Path(__file__).resolve().parents[1]


# ----------------------------------------------------------------------------
# C ABI
# ----------------------------------------------------------------------------

def header_symbols():
    text = (REPO / "include" / "ipi_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(ipi_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/ipi_b200.h but not exported"
    assert set(declared) == set(_lib.exported_symbols())
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                        text=True).stdout
    exported = set(re.findall(r" T (ipi_\w+)", nm))
    assert set(declared) <= exported


@pytest.mark.parametrize("cname,pyname", [
    ("ipi_inner_report", "InnerReport"), ("ipi_opts", "Opts"), ("ipi_stats", "Stats"),
    ("ipi_plan", "Plan"), ("ipi_op_plan", "OpPlan"), ("ipi_validation", "Validation"),
    ("ipi_csr_report", "CsrReport")])
def test_ctypes_structs_match_the_header(cname, pyname, tmp_path):
    """The ctypes mirrors in _lib.py have the C header's size and field offsets
    (compiled with gcc against include/ipi_b200.h)."""
    cls = getattr(_lib, pyname)
    fields = [f[0] for f in cls._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", '#include "ipi_b200.h"', "int main(void) {",
            f'  printf("%zu\\n", sizeof({cname}));']
    prog += [f'  printf("%zu\\n", offsetof({cname}, {f}));' for f in fields]
    prog += ["  return 0;", "}"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(prog) + "\n")
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", str(REPO / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got[0] == __import__("ctypes").sizeof(cls), (cname, got[0])
    assert got[1:] == [getattr(cls, f).offset for f in fields], cname


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_no_device_here():
    lib = _lib.load()
    assert b"sm_100a" in lib.ipi_version()
    if not __import__("torch").cuda.is_available():
        assert lib.ipi_device_count() == 0


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ipi.CsrMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])


# ----------------------------------------------------------------------------
# host API logic (mirrors the reference's frontend tests without a device)
# ----------------------------------------------------------------------------

def test_options_table_and_aliases():
    mdp = mf.MDP()
    mdp.setOption("-max_iter_pi", "7")
    mdp.setOption("max_iter_ksp", 9)
    mdp.setOption("-atol_pi", "1e-9")
    mdp.setOption("-alpha", "0.001")
    mdp.setOption("-ksp_type", "richardson")
    mdp.setOption("-ksp_max_it", "3")
    mdp.setOption("-ksp_richardson_scale", "0.5")
    mdp.setOption("-pc_sor_forward", "true")
    mdp.setOption("-pc_sor_omega", "1.2")
    mdp.setOption("-workers", "2")
    mdp.setOption("-mode", "MAXREWARD")
    mdp.SetOption("-discount_factor", "0.95")
    o = mdp.solverOptions()
    assert (o.max_outer, o.max_inner, o.tol, o.alpha) == (7, 9, 1e-9, 0.001)
    assert o.inner is ipi.InnerSolver.RICHARDSON and o.ksp_max_it == 3
    assert o.richardson_scale == 0.5 and o.sor_omega == 1.2 and o.workers == 2
    assert o.mode is ipi.Mode.MAX
    assert mdp._discount == 0.95
    mdp.setOption("-discount", "0.5")
    assert mdp._discount == 0.5
    mdp.setOption("-mode", "MINCOST")
    assert mdp.solverOptions().mode is ipi.Mode.MIN
    mdp.setOption("-mode", "max")
    assert mdp.solverOptions().mode is ipi.Mode.MAX


def test_defaults_match_reference_table():
    o = mf.MDP().solverOptions()
    assert (o.tol, o.alpha, o.max_outer, o.max_inner) == (1e-8, 1e-4, 1000, 1000)
    assert o.inner is ipi.InnerSolver.GMRES and o.pc is ipi.Preconditioner.NONE


@pytest.mark.parametrize("name,value,pattern", [
    ("-bogus", "1", "valid options"),
    ("-max_iter_pi", "abc", "cannot parse"),
    ("-ksp_type", "cg", "cannot parse"),
    ("-mode", "sideways", "cannot parse"),
])
def test_option_errors(name, value, pattern):
    with pytest.raises(ipi.ValidationError, match=pattern):
        mf.MDP().setOption(name, value)


def test_instance_errors_before_device_use():
    mdp = mf.MDP()
    with pytest.raises(ipi.ValidationError, match="setStageCostMatrix"):
        mdp.instance()
    mdp.setStageCostMatrix(np.zeros((2, 3)))
    with pytest.raises(ipi.ValidationError, match="setTransitionProbabilityTensor"):
        mdp.instance()
    with pytest.raises(ipi.ValidationError, match="dense"):
        mf.MDP().setStageCostMatrix(object.__new__(ipi.CsrMatrix))
    with pytest.raises(ipi.ValidationError, match="2-D"):
        mf.MDP().setStageCostMatrix(np.zeros(3))
    with pytest.raises(ipi.ValidationError, match="CSR"):
        mf.MDP().setTransitionProbabilityTensor(np.eye(2))


@pytest.mark.parametrize("kw,pattern", [
    (dict(tol=0.0), "tolerance"), (dict(alpha=1.0), "alpha"), (dict(max_outer=0), "max_outer"),
    (dict(ksp_max_it=0), "ksp_max_it"), (dict(workers=0), "worker"),
    (dict(richardson_scale=0.0), "richardson_scale"), (dict(sor_omega=2.0), "sor_omega"),
    (dict(pc=ipi.Preconditioner.EXACT), "svd"),
])
def test_solve_options_check(kw, pattern):
    with pytest.raises(ipi.ValidationError, match=pattern):
        ipi.SolveOptions(**kw).check()


def test_partition_formula():
    p = make_partition(10, 4)
    assert p.block_starts == (0, 3, 6, 8, 10)
    assert make_partition(3, 5).block_sizes() == [1, 1, 1, 0, 0]
    with pytest.raises(ipi.ValidationError):
        make_partition(5, 0)


def test_flatten_index_and_mode_names():
    assert ipi.flatten_index(3, 2, 5) == 17
    with pytest.raises(ipi.ValidationError):
        ipi.flatten_index(0, 5, 5)
    assert ipi.Mode.from_name("MINCOST") is ipi.Mode.MIN
    assert ipi.Mode.from_name(" maxreward ") is ipi.Mode.MAX


def test_presets():
    assert ipi.preset("VI").ksp_max_it == 1
    assert ipi.preset("OPI", w=4).ksp_max_it == 4
    assert ipi.preset("beta-vi", beta=0.5).richardson_scale == 0.5
    with pytest.raises(ipi.ValidationError):
        ipi.preset("OPI")


# ----------------------------------------------------------------------------
# generators (host restatements)
# ----------------------------------------------------------------------------

def test_philox_known_answers():
    """Random123 philox4x32-10 known-answer vectors."""
    cases = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
             ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
             ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
              (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]
    for ctr, key, want in cases:
        got = gen.philox4x32(np.array([ctr[0]], np.uint32), ctr[1], ctr[2], ctr[3], *key)
        assert tuple(int(x[0]) for x in got) == want


def _row_invariants(rp, col, val, n):
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0)
    for r in range(len(rp) - 1):
        c = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < n
    sums = np.add.reduceat(val, rp[:-1])
    assert np.all(np.abs(sums - 1.0) <= 1e-12)
    assert np.all((val >= 0) & (val <= 1))


def test_dirichlet_recipe_deterministic():
    a = gen.random_dirichlet(50, 4, 7, seed=3)
    b = gen.random_dirichlet(50, 4, 7, seed=3)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    _row_invariants(a[0], a[1], a[2], 50)


def test_locality_recipe_invariants():
    n, m, K, W = 4096, 2, 16, 64
    rp, col, val, cost = gen.random_locality_host(n, m, K, W, seed=0)
    _row_invariants(rp, col, val, n)
    s = np.repeat(np.arange(n), m * K)
    local = np.abs(col.astype(np.int64) - s) <= W
    assert 0.85 < local.mean() < 0.95
    assert np.all((cost >= 0) & (cost < 1))


def test_pendulum_recipe_invariants():
    rp, col, val, cost = gen.pendulum_host(16, 21)
    _row_invariants(rp, col, val, 256)
    assert np.all(np.diff(rp) == 4)
    i_t, j_o = np.divmod(np.arange(256), 16)
    theta = -math.pi + i_t * 2 * math.pi / 16
    assert np.allclose(cost[:, 10], theta ** 2 + 0.1 * (-10 + j_o * 20 / 15) ** 2)


def test_sis_recipe_invariants():
    rp, col, val, cost = gen.sis_host(40)
    _row_invariants(rp, col, val, 41)
    assert np.all(val >= 1e-14 / 1.0001)
    # s = 0 is absorbing for every action
    for a in range(5):
        assert list(col[rp[a]:rp[a + 1]]) == [0]
    np.testing.assert_allclose(cost[:, 0], np.arange(41) / 40)


# ----------------------------------------------------------------------------
# row-block sharding plumbing over gloo (world size 2), oracle as the stand-in
# ----------------------------------------------------------------------------

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mdp_oracle as orc
        from paper_2507_22538_b200.parallel import (RankContext, allgather_blocks, rank_max,
                                                    rank_ordered_sum)
        rp, col, val, cost = gen.random_locality_host(37, 3, 5, 6, seed=1)  # n mod R != 0
        n, m = cost.shape
        ctx = RankContext.from_env(n)
        lo, hi = ctx.block
        v_full = torch.zeros(n, dtype=torch.float64)
        v_local = torch.arange(lo, hi, dtype=torch.float64) * 0.25
        allgather_blocks(v_local, v_full, ctx.partition)
        # local backup on this rank's rows with the gathered V (oracle stands in for K1)
        r0, r1 = lo * m, hi * m
        rpl = rp[r0:r1 + 1] - rp[r0]
        pi, applied = orc.greedy(rpl, col[rp[r0]:rp[r1]], val[rp[r0]:rp[r1]], cost[lo:hi], 0.9,
                                 v_full.numpy())
        res = rank_max(torch.tensor([float(np.max(np.abs(v_full.numpy()[lo:hi] - applied)))], dtype=torch.float64))
        tot = rank_ordered_sum(torch.tensor([float(applied.sum())], dtype=torch.float64), world)
        pis = [torch.zeros(b, dtype=torch.int64) for b in ctx.partition.block_sizes()]
        dist.all_gather_object(pis, pi.tolist())
        q.put((rank, v_full.numpy().tolist(), float(res[0]), float(tot[0]), pis))
    finally:
        dist.destroy_process_group()


def test_rowblock_sharding_gloo_world2():
    import torch.multiprocessing as mp
    from oracle import mdp_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rp, col, val, cost = gen.random_locality_host(37, 3, 5, 6, seed=1)
    v = np.arange(37) * 0.25
    pi, applied = orc.greedy(rp, col, val, cost, 0.9, v)
    for rank, vfull, res, tot, pis in out:
        np.testing.assert_array_equal(vfull, v)
        assert res == float(np.max(np.abs(v - applied)))
        assert np.isclose(tot, applied.sum(), rtol=1e-14)
        np.testing.assert_array_equal(np.concatenate([np.asarray(p) for p in pis]), pi)


# ----------------------------------------------------------------------------
# sharded iPI control flow over gloo (world size 2) with oracle stand-ins for
# the device kernels; must reproduce the single-process oracle solve
# ----------------------------------------------------------------------------

from paper_2507_22538_b200.parallel import ShardVectorOps  # noqa: E402


class _CpuShardOps(ShardVectorOps):
    """Test stand-in for parallel.ShardOps: same interface, numpy oracle math
    (the device-resident MGS primitives are the torch defaults)."""

    def __init__(self, arrays, gamma, ctx):
        import torch
        from oracle import mdp_oracle as orc
        self.orc = orc
        rp, col, val, cost = arrays
        self.ctx = ctx
        self.gamma = gamma
        lo, hi = ctx.block
        m = cost.shape[1]
        r0, r1 = lo * m, hi * m
        self.rp = rp[r0:r1 + 1] - rp[r0]
        self.col = col[rp[r0]:rp[r1]]
        self.val = val[rp[r0]:rp[r1]]
        self.cost = cost[lo:hi]
        self.lo = lo
        self.full = torch.zeros(cost.shape[0], dtype=torch.float64)

    def allgather(self, local):
        from paper_2507_22538_b200.parallel import allgather_blocks
        return allgather_blocks(local, self.full, self.ctx.partition)

    def dot(self, a, b):
        import torch
        from paper_2507_22538_b200.parallel import rank_ordered_sum
        return float(rank_ordered_sum(torch.dot(a, b).reshape(1), self.ctx.world)[0])

    def greedy(self, v_local):
        import torch
        from paper_2507_22538_b200.parallel import rank_max
        vf = self.allgather(v_local).numpy()
        pi, applied = self.orc.greedy(self.rp, self.col, self.val, self.cost, self.gamma, vf)
        res = float(np.max(np.abs(v_local.numpy() - applied)))
        return (torch.as_tensor(pi.astype(np.int32)), torch.as_tensor(applied),
                float(rank_max(torch.tensor([res], dtype=torch.float64))[0]))

    def gather_policy(self, pol):
        import torch
        rpp, cp, vp, g = self.orc.gather_policy(self.rp, self.col, self.val, self.cost,
                                                pol.numpy().astype(np.int64))
        return (rpp, cp, vp), torch.as_tensor(g)

    def apply(self, P, x_local, b_local=None):
        import torch
        xf = self.allgather(x_local).numpy()
        rpp, cp, vp = P
        n_loc = x_local.shape[0]
        y = xf[self.lo:self.lo + n_loc] - self.gamma * self.orc.spmv(rpp, cp, vp, xf)
        y = torch.as_tensor(y)
        return b_local - y if b_local is not None else y


def _sharded_solve_worker(rank, world, port, kind, q, ortho=None):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.parallel import RankContext, solve_sharded
        arrays = gen.random_locality_host(61, 4, 6, 8, seed=2)
        ctx = RankContext.from_env(61)
        ops = _CpuShardOps(arrays, 0.95, ctx)
        lo, hi = ctx.block
        res = solve_sharded(ops, ipi.SolveOptions(inner=ipi.InnerSolver.from_name(kind)), 61,
                            torch.zeros(hi - lo, dtype=torch.float64), ortho=ortho)
        q.put((rank, res.status.value, res.outer_iterations, res.values.tolist(),
               res.policy.tolist(), res.residual_history))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,ortho", [("gmres", "mgs"), ("gmres", "cgs2"), ("richardson", None)])
def test_sharded_ipi_gloo_world2_matches_oracle(kind, ortho):
    import torch.multiprocessing as mp
    from oracle import mdp_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_solve_worker, args=(r, 2, port, kind, q, ortho))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rp, col, val, cost = gen.random_locality_host(61, 4, 6, 8, seed=2)
    ref = orc.solve(rp, col, val, cost, 0.95, kind=kind)
    (_, st0, k0, v0, p0, h0), (_, st1, k1, v1, p1, h1) = out
    assert (st0, k0, p0, h0) == (st1, k1, p1, h1) and v0 == v1   # ranks agree exactly
    assert st0 == ref.status and k0 == ref.outer_iterations
    np.testing.assert_allclose(v0, ref.values, rtol=1e-10, atol=1e-10)
    np.testing.assert_array_equal(p0, ref.policy)
    np.testing.assert_allclose(h0, ref.residual_history, rtol=1e-6, atol=1e-12)


def test_fromfile_errors_carry_offsets(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"WRONGMAG" + b"\x00" * 40)
    with pytest.raises(ipi.FileFormatError) as err:
        mf.Matrix.fromFile(bad)
    assert err.value.offset == 0
    short = tmp_path / "short.bin"
    short.write_bytes(b"MDPMAT01")
    with pytest.raises(ipi.FileFormatError, match="shorter than the header"):
        mf.Matrix.fromFile(short)


def test_dense_file_round_trip_host(tmp_path):
    a = np.arange(12, dtype=np.float64).reshape(3, 4)
    ipi.write_matrix(tmp_path / "d.bin", a)
    np.testing.assert_array_equal(mf.Matrix.fromFile(tmp_path / "d.bin").data, a)


def test_creator_argument_errors_before_device():
    with pytest.raises(ipi.ValidationError, match="empty distribution"):
        mf.createTransitionProbabilityTensor(2, 1, lambda s, a: ([], []))
    with pytest.raises(ipi.ValidationError, match="outside"):
        mf.createTransitionProbabilityTensor(2, 1, lambda s, a: ([5], [1.0]))
    with pytest.raises(ipi.ValidationError, match="twice"):
        mf.createTransitionProbabilityTensor(2, 1, lambda s, a: ([0, 0], [0.5, 0.5]))
    with pytest.raises(ipi.ValidationError, match="negative"):
        mf.createTransitionProbabilityTensor(2, 1, lambda s, a: ([0, 1], [1.5, -0.5]))


# ----------------------------------------------------------------------------
# halo (point-to-point) V exchange over gloo, world size 3, CPU tensors
# ----------------------------------------------------------------------------

def _halo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.model import make_partition
        from paper_2507_22538_b200.parallel import HaloExchange
        n = 100
        part = make_partition(n, world)
        lo, hi = part.block(rank)
        need = (max(0, lo - 7), min(n - 1, hi - 1 + 11))  # asymmetric halo
        os.environ["IPI_HALO_FRAC"] = "0.9"
        hx = HaloExchange(part, rank, world, need, n, torch.device("cpu"))
        ref = torch.arange(n, dtype=torch.float64) * 1.5 + 2.0
        full = torch.full((n,), float("nan"), dtype=torch.float64)
        hx.exchange_async(ref[lo:hi].clone(), full).wait()
        ok = bool(torch.equal(full[need[0]:need[1] + 1], ref[need[0]:need[1] + 1]))
        q.put((rank, hx.enabled, ok, hx.bytes_received()))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_gloo_world3():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(enabled and ok for _, enabled, ok, _ in out), out
    # the middle rank receives both halos (7 + 11 entries), the outer ranks one each
    assert [b // 8 for *_, b in out] == [11, 18, 7]


# ----------------------------------------------------------------------------
# per-rank callback construction (problems.py:419-488 with workers = ranks):
# each rank evaluates only its partition block; the blocks concatenate to the
# one-process build bit for bit
# ----------------------------------------------------------------------------

def _cb_trans(s, a):
    rng = np.random.default_rng(1000 * s + a)
    k = 1 + (s * 7 + a) % 9                       # ragged rows, 1..9 successors
    cols = rng.choice(53, size=k, replace=False)
    p = rng.random(k) + 0.1
    return cols.tolist(), (p / p.sum()).tolist()


def _cb_cost(s, a):
    return 0.5 * s - 0.25 * a


def _callback_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_22538_b200.frontend import callback_block
        from paper_2507_22538_b200.parallel import RankContext
        ctx = RankContext.from_env(53)
        lo, hi = ctx.block
        rp, cols, vals, cost = callback_block(53, 3, lo, hi, _cb_trans, _cb_cost)
        got = [None] * world
        dist.all_gather_object(got, (rank, lo, hi, rp.tolist(), cols.tolist(), vals.tolist(),
                                     cost.tolist()))
        q.put(got)
    finally:
        dist.destroy_process_group()


def test_callback_construction_per_rank_gloo_world2():
    import torch.multiprocessing as mp
    from paper_2507_22538_b200.frontend import callback_block
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_callback_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rp, cols, vals, cost = callback_block(53, 3, 0, 53, _cb_trans, _cb_cost)
    blocks = sorted(outs[0])
    assert blocks == sorted(outs[1])  # every rank saw the same gathered blocks
    # concatenating the ranks' blocks reproduces the sequential build exactly
    assert [b[1] for b in blocks] == [0, 27] and blocks[-1][2] == 53
    off = 0
    rp_cat = [0]
    for _, lo, hi, brp, bcols, bvals, bcost in blocks:
        rp_cat += [off + x for x in brp[1:]]
        off += brp[-1]
    np.testing.assert_array_equal(rp_cat, rp)
    np.testing.assert_array_equal(np.concatenate([b[4] for b in blocks]), cols)
    assert np.concatenate([b[5] for b in blocks]).tobytes() == vals.tobytes()
    assert np.concatenate([b[6] for b in blocks]).tobytes() == cost.tobytes()


def test_callback_block_errors_name_the_pair():
    from paper_2507_22538_b200.frontend import callback_block
    with pytest.raises(ipi.ValidationError, match=r"trans_fn\(s=4, a=1\).*pre-allocation"):
        callback_block(10, 2, 3, 6, lambda s, a: (([0, 1, 2], [0.2, 0.3, 0.5]) if (s, a) == (4, 1)
                                                  else ([0], [1.0])), prealloc=2)
    with pytest.raises(ipi.ValidationError, match="sum to"):
        callback_block(10, 2, 0, 1, lambda s, a: ([0, 1], [0.2, 0.3]))
