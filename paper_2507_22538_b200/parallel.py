"""Row-block data parallelism across GPUs (one process per GPU).

The reference's only parallel strategy is contiguous state blocks
(``Workers`` over ``make_partition``, parallel.py:36-79; model.py:95-109),
the in-process stand-in for the paper's MPI row distribution
(PAPER.md:150-158).  Here rank r owns states ``make_partition(n, R).block(r)``
and all their (s, a) rows in HBM; K1 and K2 are purely local.  The one data
exchange per SpMV is the value vector: every rank needs V at the columns its
rows touch, so V blocks are all-gathered (NCCL over NVLink; gloo in the CPU
tests) into a full-length V on every rank before the backup.  Scalar
reductions gather the R per-rank partials and combine them in rank order, so
a run at fixed R is bit-reproducible like ``tree_reduce`` (parallel.py:21-33).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from .model import Mode, Partition, make_partition
from .sparse import CsrMatrix, DeviceOperator

__all__ = ["MdpShard", "NativeComm", "RankContext", "ShardOps", "allgather_blocks", "host_gmres",
           "host_richardson", "rank_max", "rank_ordered_sum", "solve_sharded",
           "solve_sharded_native"]


@dataclass
class RankContext:
    """Who am I in the job: rank, world size and the state partition."""

    rank: int
    world: int
    partition: Partition

    @classmethod
    def from_env(cls, n: int) -> "RankContext":
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            r, w = dist.get_rank(), dist.get_world_size()
        else:
            r, w = 0, 1
        return cls(r, w, make_partition(n, w))

    @property
    def block(self) -> tuple[int, int]:
        return self.partition.block(self.rank)


def _nccl() -> bool:
    """NCCL takes the flat *_into_tensor collectives; gloo (CPU tests, or CUDA
    tensors staged through the host) takes tensor lists."""
    import torch.distributed as dist
    return dist.get_backend() == "nccl"


def gather_partials(part: torch.Tensor, world: int) -> torch.Tensor:
    """(1,) per-rank partial -> (R,) partials of every rank, in rank order."""
    import torch.distributed as dist
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return part.reshape(1)
    parts = torch.empty(world, dtype=part.dtype, device=part.device)
    if _nccl():
        dist.all_gather_into_tensor(parts, part.reshape(1).contiguous())
    else:
        dist.all_gather(list(parts.split(1)), part.reshape(1).contiguous())
    return parts


def ordered_sum(parts: torch.Tensor) -> torch.Tensor:
    """parts[0] + parts[1] + ... in rank order (deterministic like tree_reduce)."""
    out = parts[0:1].clone()
    for r in range(1, parts.numel()):
        out = out + parts[r:r + 1]
    return out


def allgather_blocks(local: torch.Tensor, full: torch.Tensor, partition: Partition) -> torch.Tensor:
    """Fill ``full`` (n) with every rank's block; ``local`` is this rank's.

    Equal blocks use one ``all_gather_into_tensor``; unequal ones (n mod R != 0)
    pad to the largest block and compact.  Works with NCCL (CUDA tensors) and
    gloo (CPU tensors)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or partition.worker_count == 1:
        if full.data_ptr() != local.data_ptr():
            full.copy_(local)
        return full
    sizes = partition.block_sizes()
    R = partition.worker_count
    if len(set(sizes)) == 1:
        if _nccl():
            dist.all_gather_into_tensor(full, local.contiguous())
        else:
            parts = list(full.split(sizes))
            dist.all_gather(parts, local.contiguous())
        return full
    mx = max(sizes)
    pad = torch.zeros(mx, dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    buf = torch.empty(mx * R, dtype=local.dtype, device=local.device)
    if _nccl():
        dist.all_gather_into_tensor(buf, pad)
    else:
        dist.all_gather(list(buf.split(mx)), pad)
    for r in range(R):
        lo, hi = partition.block(r)
        full[lo:hi] = buf[r * mx: r * mx + (hi - lo)]
    return full


class _Done:
    def wait(self):
        return None


def allgather_blocks_async(local: torch.Tensor, full: torch.Tensor, partition: Partition):
    """Start the all-gather of ``local`` into ``full``; returns a waitable.  With
    NCCL the collective runs on its own stream while the caller keeps launching
    work that does not read ``full``; ``wait()`` orders later work after it.
    Unequal blocks fall back to the blocking path."""
    import torch.distributed as dist
    if (not (dist.is_available() and dist.is_initialized()) or partition.worker_count == 1
            or len(set(partition.block_sizes())) != 1):
        allgather_blocks(local, full, partition)
        return _Done()
    if _nccl():
        return dist.all_gather_into_tensor(full, local.contiguous(), async_op=True)
    return dist.all_gather(list(full.split(partition.block_sizes())), local.contiguous(),
                           async_op=True)


class _Staged:
    """Waitable for gloo P2P on device tensors: receives land in host buffers
    and are copied into place after the waits."""

    def __init__(self, works, copies):
        self.works, self.copies = works, copies

    def wait(self):
        for w in self.works:
            w.wait()
        for dst, src in self.copies:
            dst.copy_(src)


class HaloExchange:
    """Point-to-point V exchange for row blocks whose columns stay near the
    block (north star (5): "or by halo exchange when column locality allows").

    Every rank publishes the global column range its rows read
    (``ipi_col_range``); rank r then receives from each rank q the part of q's
    block inside r's range and sends q the part of its own block inside q's
    range.  Enabled when every rank's range spans at most ``frac`` of the
    states (``IPI_HALO_FRAC``, default 0.5); otherwise the all-gather is the
    cheaper exchange (C2 / C5: 10% uniform columns make every range full).
    Entries of ``full`` outside the rank's range are never read by its kernels."""

    def __init__(self, partition: Partition, rank: int, world: int, need: tuple[int, int],
                 n_global: int, device):
        import torch.distributed as dist
        self.partition, self.rank, self.world = partition, rank, world
        mine = torch.tensor([int(need[0]), int(need[1])], dtype=torch.int64, device=device)
        if world > 1 and dist.is_available() and dist.is_initialized():
            allr = torch.empty((world, 2), dtype=torch.int64, device=device)
            if _nccl():
                dist.all_gather_into_tensor(allr, mine)
            else:
                dist.all_gather(list(allr.unbind(0)), mine)
            self.ranges = [tuple(r) for r in allr.cpu().tolist()]
        else:
            self.ranges = [(int(need[0]), int(need[1]))]
        frac = float(os.environ.get("IPI_HALO_FRAC", "0.5"))
        widest = max(max(0, hi - lo + 1) for lo, hi in self.ranges)
        self.enabled = world > 1 and widest <= frac * n_global
        lo_me, hi_me = partition.block(rank)
        self.lo, self.hi = lo_me, hi_me
        self.recv, self.send = [], []  # (peer, a, b): global slice [a, b)
        for q in range(world if self.enabled else 0):
            if q == rank:
                continue
            lq, hq = partition.block(q)
            nlo, nhi = self.ranges[rank]
            a, b = max(lq, nlo), min(hq, nhi + 1)
            if a < b:
                self.recv.append((q, a, b))
            qlo, qhi = self.ranges[q]
            a, b = max(lo_me, qlo), min(hi_me, qhi + 1)
            if a < b:
                self.send.append((q, a, b))

    def bytes_received(self) -> int:
        return 8 * sum(b - a for _, a, b in self.recv)

    def exchange_async(self, local: torch.Tensor, full: torch.Tensor):
        import torch.distributed as dist
        full[self.lo:self.hi].copy_(local)
        if _nccl():
            ops = [dist.P2POp(dist.isend, local[a - self.lo:b - self.lo].contiguous(), q)
                   for q, a, b in self.send]
            ops += [dist.P2POp(dist.irecv, full[a:b], q) for q, a, b in self.recv]
            works = dist.batch_isend_irecv(ops) if ops else []
            return _Staged(works, [])
        # gloo: host-staged point-to-point
        works, copies = [], []
        for q, a, b in self.send:
            works.append(dist.isend(local[a - self.lo:b - self.lo].detach().cpu().contiguous(), q))
        for q, a, b in self.recv:
            buf = torch.empty(b - a, dtype=full.dtype)
            works.append(dist.irecv(buf, q))
            copies.append((full[a:b], buf))
        return _Staged(works, copies)


class SplitShardOperator:
    """J_pi on a rank's rows with the V exchange overlapped (north star (5)):
    the rank's P_pi rows are split into local columns (its own state block,
    re-indexed) and remote columns (``ipi_csr_split_local``).  ``apply`` starts
    the all-gather of x, runs the local-column SpMV on x_local while it is in
    flight, waits, then the remote half adds its sum and forms
    x - gamma*(P_loc x + P_rem x) (``ipi_op_apply_partial``).  Row sums are
    (local part) + (remote part): deterministic, within 1e-13 of the unsplit
    order."""

    def __init__(self, rp, col, val, n_local: int, n_global: int, state0: int, gamma: float):
        from .sparse import DeviceOperator
        dev = rp.device
        L = _lib.lib()
        rp_loc = torch.zeros(n_local + 1, dtype=torch.int64, device=dev)
        rp_rem = torch.zeros(n_local + 1, dtype=torch.int64, device=dev)
        lo, hi = state0, state0 + n_local
        _lib.check(L.ipi_csr_split_local(_lib.ptr(rp), _lib.ptr(col), _lib.ptr(val), n_local, lo, hi,
                                         _lib.ptr(rp_loc), None, None, _lib.ptr(rp_rem), None, None,
                                         _lib.stream_ptr()), "ipi_csr_split_local")
        rp_loc[1:] = torch.cumsum(rp_loc[1:], 0)
        rp_rem[1:] = torch.cumsum(rp_rem[1:], 0)
        nl, nr = (int(x) for x in torch.stack([rp_loc[-1], rp_rem[-1]]).tolist())
        col_loc = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
        val_loc = torch.empty(max(nl, 1), dtype=torch.float64, device=dev)
        col_rem = torch.empty(max(nr, 1), dtype=torch.int32, device=dev)
        val_rem = torch.empty(max(nr, 1), dtype=torch.float64, device=dev)
        _lib.check(L.ipi_csr_split_local(_lib.ptr(rp), _lib.ptr(col), _lib.ptr(val), n_local, lo, hi,
                                         _lib.ptr(rp_loc), _lib.ptr(col_loc), _lib.ptr(val_loc),
                                         _lib.ptr(rp_rem), _lib.ptr(col_rem), _lib.ptr(val_rem),
                                         _lib.stream_ptr()), "ipi_csr_split_local")
        self.local = DeviceOperator(rp_loc, col_loc[:nl], val_loc[:nl], n_local, n_local, 0, gamma)
        self.remote = DeviceOperator(rp_rem, col_rem[:nr], val_rem[:nr], n_local, n_global, state0,
                                     gamma)
        self.n_local, self.nnz_local, self.nnz_remote = n_local, nl, nr

    def plan(self) -> dict:
        return {"split": True, "nnz_local": self.nnz_local, "nnz_remote": self.nnz_remote,
                "local": self.local.plan(), "remote": self.remote.plan()}

    def apply_overlapped(self, x_local: torch.Tensor, full: torch.Tensor, partition: Partition,
                         b: torch.Tensor | None = None, exchange_async=None) -> torch.Tensor:
        work = (exchange_async(x_local, full) if exchange_async is not None
                else allgather_blocks_async(x_local, full, partition))
        y_loc = self.local.spmv(x_local)          # overlaps the all-gather
        work.wait()
        return self.remote.apply_partial(full, y_loc, b)


def rank_ordered_sum(partial: torch.Tensor, world: int) -> torch.Tensor:
    """Deterministic all-reduce: gather the R partials, add them in rank order."""
    import torch.distributed as dist
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return partial.clone()
    parts = torch.empty((world,) + tuple(partial.shape), dtype=partial.dtype, device=partial.device)
    if _nccl():
        dist.all_gather_into_tensor(parts, partial.contiguous())
    else:
        dist.all_gather(list(parts.unbind(0)), partial.contiguous())
    out = parts[0].clone()
    for r in range(1, world):
        out = out + parts[r]
    return out


def rank_max(x: torch.Tensor) -> torch.Tensor:
    """Max over ranks (exact and order-independent)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        x = x.clone()
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return x


class MdpShard:
    """This rank's rows of an (n*m) x n instance: states [state0, state0+n_local).

    ``transitions`` is the local (n_local*m) x n_global CSR (global column
    indices), ``stage_cost`` the local (n_local, m) block.  The device handle
    plans K1 for the shard (nnz-balanced CTA ranges, V window in global
    coordinates)."""

    def __init__(self, n_global: int, m: int, gamma: float, state0: int, stage_cost: torch.Tensor,
                 transitions: CsrMatrix, mode: Mode = Mode.MIN):
        self.n_global, self.m, self.gamma, self.mode = int(n_global), int(m), float(gamma), mode
        self.state0 = int(state0)
        self.n_local = int(stage_cost.shape[0])
        if transitions.shape != (self.n_local * self.m, self.n_global):
            raise ValueError("shard CSR shape does not match (n_local*m, n_global)")
        self.stage_cost = stage_cost.contiguous()
        self.transitions = transitions
        out = _lib.C.c_void_p()
        t = transitions
        _lib.check(_lib.lib().ipi_mdp_create(
            _lib.ptr(t.row_ptr), _lib.ptr(t.col_idx), _lib.ptr(t.values), _lib.ptr(self.stage_cost),
            self.n_local, self.n_global, self.m, self.state0, self.gamma,
            _lib.MODE_MAX if mode is Mode.MAX else _lib.MODE_MIN, _lib.stream_ptr(),
            _lib.C.byref(out)), "ipi_mdp_create")
        self._handle = out
        dev = stage_cost.device
        self.policy = torch.empty(self.n_local, dtype=torch.int32, device=dev)
        self.applied = torch.empty(self.n_local, dtype=torch.float64, device=dev)
        self.res_bits = torch.zeros(1, dtype=torch.int64, device=dev)

    def handle(self):
        return self._handle

    def plan(self) -> dict:
        p = _lib.Plan()
        _lib.check(_lib.lib().ipi_mdp_plan(self._handle, _lib.C.byref(p)), "ipi_mdp_plan")
        return p.as_dict()

    def bellman(self, v_full: torch.Tensor, *, residual: bool = True, stream=None):
        """K1 over the local rows with the full V; returns (policy, applied, res_bits)."""
        _lib.check(_lib.lib().ipi_bellman(
            self._handle, _lib.ptr(v_full), _lib.MODE_MAX if self.mode is Mode.MAX else _lib.MODE_MIN,
            _lib.ptr(self.policy), _lib.ptr(self.applied), None, None,
            _lib.ptr(self.res_bits) if residual else None, _lib.stream_ptr(stream)), "ipi_bellman")
        return self.policy, self.applied, self.res_bits

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                torch.cuda.synchronize()
                _lib.lib().ipi_mdp_destroy(h)
            except Exception:
                pass
            self._handle = None


# ----------------------------------------------------------------------------
# Sharded iPI (host-driven phases, collectives between them)
# ----------------------------------------------------------------------------
#
# Every rank runs the same control flow on bit-identical scalars (all scalar
# reductions go through rank_ordered_sum / rank_max), so decisions (stopping
# tests, Givens, est_target) agree across ranks without broadcasts.  The
# numeric phases are the rank-local kernels: K1 on the shard with the
# all-gathered V, K2 on the local rows, and the sharded J_pi apply
# (DeviceOperator: ipi_op_apply) on the all-gathered Krylov vector.  The GMRES /
# Richardson control logic below restates inner.py:216-292 exactly; it is
# written against a tiny vector-ops interface so the CPU tests can drive it
# with gloo and numpy stand-ins.

GMRES_RESTART = 30


class ShardVectorOps:
    """Device-resident scalar primitives of the sharded inner solve.

    Scalars stay tensors until ``to_host`` (one host sync per Arnoldi step):
    ``dot_partial`` is this rank's share of a dot, ``gather_partials`` the
    all-gather of the R shares, ``mgs_pass`` one modified Gram-Schmidt pass
    (inner.py:251-253) on the gathered shares.  These defaults are torch ops
    (CPU tests over gloo); ``ShardOps`` overrides them with CUDA kernels."""

    ctx: RankContext

    def dot_partial(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        return torch.dot(a, b).reshape(1)

    def gather_partials(self, part: torch.Tensor) -> torch.Tensor:
        return gather_partials(part, self.ctx.world)

    def ordered_sum(self, parts: torch.Tensor) -> torch.Tensor:
        return ordered_sum(parts)

    def mgs_pass(self, parts, w, v, v_next):
        """h = ordered_sum(parts); w -= h*v (in place); next share <v_next, w> (or <w, w>)."""
        h = ordered_sum(parts)
        w.sub_(h * v)
        return h, self.dot_partial(v_next if v_next is not None else w, w)

    def gather_sum(self, part: torch.Tensor) -> torch.Tensor:
        """Per-rank shares (k,) -> their rank-ordered sum (k,), on every rank."""
        return rank_ordered_sum(part.reshape(-1), self.ctx.world)

    def to_host(self, scalars) -> list[float]:
        return torch.cat([t.reshape(-1) for t in scalars]).cpu().tolist()


class ShardOps(ShardVectorOps):
    """Device implementation of the sharded-iPI vector interface for one rank."""

    def __init__(self, shard: "MdpShard", ctx: RankContext):
        self.shard = shard
        self.ctx = ctx
        dev = shard.stage_cost.device
        self.full = torch.empty(shard.n_global, dtype=torch.float64, device=dev)
        # V exchange for the SpMVs: halo (point-to-point) when the ranks' column
        # ranges are narrow, else the all-gather (collective: every rank builds this)
        t = shard.transitions
        cmin, cmax = _lib.C.c_int64(), _lib.C.c_int64()
        _lib.check(_lib.lib().ipi_col_range(_lib.ptr(t.col_idx), int(t.col_idx.numel()),
                                            _lib.C.byref(cmin), _lib.C.byref(cmax),
                                            _lib.stream_ptr()), "ipi_col_range")
        lo, hi = ctx.block
        need = (min(cmin.value, lo), max(cmax.value, hi - 1)) if cmax.value >= 0 else (lo, hi - 1)
        self.halo = HaloExchange(ctx.partition, ctx.rank, ctx.world, need, shard.n_global, dev)

    def exchange_async(self, local: torch.Tensor, full: torch.Tensor):
        if self.halo.enabled:
            return self.halo.exchange_async(local.contiguous(), full)
        return allgather_blocks_async(local.contiguous(), full, self.ctx.partition)

    def exchange(self, local: torch.Tensor) -> torch.Tensor:
        """V for this rank's SpMVs: every entry its rows can read is current."""
        if self.halo.enabled:
            self.halo.exchange_async(local.contiguous(), self.full).wait()
            return self.full
        return self.allgather(local)

    # -- collectives ------------------------------------------------------
    def allgather(self, local: torch.Tensor) -> torch.Tensor:
        return allgather_blocks(local.contiguous(), self.full, self.ctx.partition)

    def dot(self, a: torch.Tensor, b: torch.Tensor) -> float:
        part = torch.dot(a, b).reshape(1)
        return float(rank_ordered_sum(part, self.ctx.world)[0])

    def max(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.full.device)
        return float(rank_max(t)[0])

    def dot_partial(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        out = torch.empty(1, dtype=torch.float64, device=a.device)
        _lib.check(_lib.lib().ipi_dot_partial(_lib.ptr(a), _lib.ptr(b), a.numel(), _lib.ptr(out),
                                              _lib.stream_ptr()), "ipi_dot_partial")
        return out

    def mgs_pass(self, parts, w, v, v_next):
        h = torch.empty(1, dtype=torch.float64, device=w.device)
        nxt = torch.empty(1, dtype=torch.float64, device=w.device)
        _lib.check(_lib.lib().ipi_mgs_pass(_lib.ptr(parts), parts.numel(), _lib.ptr(h), _lib.ptr(w),
                                           _lib.ptr(v), _lib.ptr(v_next), w.numel(), _lib.ptr(nxt),
                                           _lib.stream_ptr()), "ipi_mgs_pass")
        return h, nxt

    # -- kernels ------------------------------------------------------------
    def greedy(self, v_local: torch.Tensor):
        """K1 on the shard: (policy_local int32, applied_local, global ||v - Tv||_inf)."""
        vf = self.exchange(v_local)
        pol, app, bits = self.shard.bellman(vf)
        res = float(bits.view(torch.float64)[0])
        return pol.clone(), app.clone(), self.max(res)

    def gather_policy(self, policy_local: torch.Tensor, split: bool | None = None):
        sh = self.shard
        h = sh.handle()
        nnz = _lib.C.c_int64()
        L = _lib.lib()
        _lib.check(L.ipi_policy_nnz(h, _lib.ptr(policy_local), _lib.C.byref(nnz), _lib.stream_ptr()),
                   "ipi_policy_nnz")
        dev = policy_local.device
        rp = torch.empty(sh.n_local + 1, dtype=torch.int64, device=dev)
        col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
        g = torch.empty(sh.n_local, dtype=torch.float64, device=dev)
        _lib.check(L.ipi_gather_policy(h, _lib.ptr(policy_local), _lib.ptr(rp), _lib.ptr(col),
                                       _lib.ptr(val), _lib.ptr(g), _lib.stream_ptr()),
                   "ipi_gather_policy")
        # K3 planned once per policy: with R > 1 ranks the rows are split into
        # local / remote columns so the V all-gather overlaps the local half
        # (IPI_SHARD_OVERLAP=0: one operator over the gathered vector)
        if split is None:
            split = self.ctx.world > 1 and os.environ.get("IPI_SHARD_OVERLAP", "1") != "0"
        cls = SplitShardOperator if split else DeviceOperator
        op = cls(rp, col[:nnz.value], val[:nnz.value], sh.n_local, sh.n_global, sh.state0, sh.gamma)
        return op, g

    def apply(self, P, x_local: torch.Tensor, b_local: torch.Tensor | None = None) -> torch.Tensor:
        """b - (x - gamma P x) (or x - gamma P x) on the local rows."""
        b = b_local.contiguous() if b_local is not None else None
        if isinstance(P, SplitShardOperator):
            return P.apply_overlapped(x_local.contiguous(), self.full, self.ctx.partition, b,
                                      exchange_async=self.exchange_async)
        xf = self.exchange(x_local)
        return P.apply(xf, b)

    def sweep(self, P, g_local, v_local):
        """g_pi + gamma * P_pi v (breakdown fallback, driver.py:190-193)."""
        return g_local + self.shard.gamma * (v_local - self.apply(P, v_local))


def host_richardson(ops, P, b, theta0, eff, max_it, scale):
    """inner.py:216-226 on sharded vectors."""
    theta = theta0.clone() if hasattr(theta0, "clone") else theta0.copy()
    it = 0
    while True:
        r = ops.apply(P, theta, b)
        rn = math.sqrt(ops.dot(r, r))
        if rn <= eff or it >= max_it or not math.isfinite(rn):
            break
        theta = theta + scale * r
        it += 1
    return theta, it, rn, False


def host_gmres(ops, P, b, theta0, eff, max_it, ortho: str = "mgs"):
    """Restarted GMRES(30) with Givens (inner.py:229-292) on sharded vectors.

    ``ortho="mgs"`` restates the reference's modified Gram-Schmidt: j+2
    cross-rank reductions per Arnoldi step.  ``ortho="cgs2"`` orthogonalises
    with two classical Gram-Schmidt sweeps (batched dots and one fused update
    per sweep): three reductions per step whatever j — the option SURVEY §8(e)
    names for multi-GPU runs, where each reduction is an all-gather.  Same
    stopping logic; Hessenberg entries differ from MGS at rounding level."""
    x = theta0.clone() if hasattr(theta0, "clone") else theta0.copy()
    it = 0
    r = ops.apply(P, x, b)
    rn = math.sqrt(ops.dot(r, r))
    est_target = eff
    R = GMRES_RESTART
    while rn > eff and it < max_it:
        beta = math.sqrt(ops.dot(r, r))
        if beta == 0.0 or not math.isfinite(beta):
            break
        if ortho == "cgs2":
            Vm = torch.empty((R + 1,) + tuple(r.shape), dtype=r.dtype, device=r.device)
            Vm[0] = r / beta
            V = [Vm[0]]
        else:
            V = [r / beta]
        H = [[0.0] * R for _ in range(R + 1)]
        cs = [0.0] * R
        sn = [0.0] * R
        g = [0.0] * (R + 1)
        g[0] = beta
        j = 0
        while j < R and it < max_it:
            w = ops.apply(P, V[j])
            it += 1
            if ortho == "cgs2":
                # two classical sweeps: batched shares <V_l, w>, one reduction,
                # one update w -= V^T c; then ||w||: three reductions per step
                Vj = Vm[: j + 1]
                c1 = ops.gather_sum(torch.mv(Vj, w))
                w = w - torch.mv(Vj.t(), c1)
                c2 = ops.gather_sum(torch.mv(Vj, w))
                w = w - torch.mv(Vj.t(), c2)
                vals = ops.to_host([c1 + c2, ops.gather_sum(torch.dot(w, w).reshape(1))])
            else:
                # MGS with the scalars on the device: one kernel + one all-gather of
                # the R shares per pass, one host sync per step (the H column)
                part = ops.dot_partial(V[0], w)
                hs = []
                for l in range(j + 1):
                    h, part = ops.mgs_pass(ops.gather_partials(part), w, V[l], V[l + 1] if l < j else None)
                    hs.append(h)
                vals = ops.to_host(hs + [ops.ordered_sum(ops.gather_partials(part))])
            for l in range(j + 1):
                H[l][j] = vals[l]
            hnorm = math.sqrt(vals[j + 1])
            H[j + 1][j] = hnorm
            for l in range(j):
                t = cs[l] * H[l][j] + sn[l] * H[l + 1][j]
                H[l + 1][j] = -sn[l] * H[l][j] + cs[l] * H[l + 1][j]
                H[l][j] = t
            denom = math.hypot(H[j][j], H[j + 1][j])
            if denom == 0.0:
                break
            cs[j], sn[j] = H[j][j] / denom, H[j + 1][j] / denom
            H[j][j] = denom
            H[j + 1][j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j += 1
            if abs(g[j]) <= est_target or hnorm == 0.0:
                break
            if ortho == "cgs2":
                torch.div(w, hnorm, out=Vm[j])
                V.append(Vm[j])
            else:
                V.append(w / hnorm)
        if j == 0:
            break
        y = [0.0] * j
        for i in range(j - 1, -1, -1):
            acc = g[i] - sum(H[i][k] * y[k] for k in range(i + 1, j))
            y[i] = acc / H[i][i] if H[i][i] != 0.0 else 0.0
        upd = V[0] * y[0]
        for l in range(1, j):
            upd = upd + V[l] * y[l]
        x = x + upd
        r = ops.apply(P, x, b)
        rn = math.sqrt(ops.dot(r, r))
        if rn > eff and abs(g[j]) <= est_target:
            if abs(g[j]) == 0.0:
                break
            est_target = abs(g[j]) * (eff / rn) * 0.5
    return x, it, rn, False


def solve_sharded(ops, opts, n_global: int, v0_local=None, ortho: str | None = None):
    """Algorithm 1 (driver.py:109-209) across ranks; returns a SolveResult whose
    values/policy are the gathered full vectors (on every rank).  GMRES
    orthogonalisation: ``ortho`` or IPI_SHARD_ORTHO, default MGS on one rank
    (the reference's arithmetic) and CGS2 across ranks (3 reductions per step)."""
    import time
    from .driver import STALL_WINDOW, SolveResult, SolveStatus
    from .inner import InnerSolver
    from .inner import Preconditioner
    if opts.inner not in (InnerSolver.GMRES, InnerSolver.RICHARDSON):
        raise NotImplementedError("the sharded path runs GMRES and Richardson inner solves")
    if opts.pc is not Preconditioner.NONE:
        raise NotImplementedError("the host-driven sharded driver has no preconditioner; "
                                  "use solve_sharded_native (jacobi)")
    shard = getattr(ops, "shard", None)
    if opts.mode is not None and shard is not None and opts.mode is not shard.mode:
        raise NotImplementedError("the host-driven sharded driver runs the shard's own mode; "
                                  "use solve_sharded_native for a mode override")
    if v0_local is None and opts.v0 is not None:
        lo, hi = ops.ctx.block
        v0_local = torch.as_tensor(opts.v0, dtype=torch.float64)[lo:hi].to(ops.full.device)
    if ortho is None:
        ortho = os.environ.get("IPI_SHARD_ORTHO", "cgs2" if ops.ctx.world > 1 else "mgs")
    if ortho not in ("mgs", "cgs2"):
        raise ValueError(f"unknown orthogonalisation {ortho!r}; expected 'mgs' or 'cgs2'")
    t0 = time.perf_counter()
    v = v0_local
    if v is None:
        lo, hi = ops.ctx.block
        v = torch.zeros(hi - lo, dtype=torch.float64, device=ops.full.device)
    history: list[float] = []
    inner_total = 0
    stall = 0
    k = 0
    while True:
        pol, _, res = ops.greedy(v)
        history.append(res)
        if res <= opts.tol:
            status = SolveStatus.CONVERGED
            break
        if k >= opts.max_outer:
            status = SolveStatus.OUTER_CAP
            break
        if k > 0 and res >= history[k - 1]:
            stall += 1
            if stall >= STALL_WINDOW:
                status = SolveStatus.STALLED
                break
        else:
            stall = 0
        P, g = ops.gather_policy(pol)
        if opts.ksp_max_it is not None:
            target, cap = 0.0, opts.ksp_max_it
        else:
            target, cap = opts.alpha * res, opts.max_inner
        bn = math.sqrt(ops.dot(g, g))
        eff = max(target, 1e-14 * max(1.0, bn))          # inner.py:189
        if opts.inner is InnerSolver.GMRES:
            v, its, _, _ = host_gmres(ops, P, g, v, eff, cap, ortho=ortho)
        else:
            v, its, _, _ = host_richardson(ops, P, g, v, eff, cap, opts.richardson_scale)
        inner_total += its
        k += 1
    values = ops.allgather(v).clone() if hasattr(v, "clone") else ops.allgather(v).copy()
    pol_full = ops.allgather(pol.to(values.dtype) if hasattr(pol, "to") else pol.astype(values.dtype))
    import numpy as _np
    vals_np = values.cpu().numpy() if hasattr(values, "cpu") else _np.asarray(values)
    pol_np = (pol_full.cpu().numpy() if hasattr(pol_full, "cpu") else _np.asarray(pol_full))
    return SolveResult(values=vals_np.copy(), policy=pol_np.astype(_np.int64),
                       outer_iterations=k, inner_iterations_total=inner_total,
                       residual_history=history, status=status,
                       wall_time=time.perf_counter() - t0)


# ----------------------------------------------------------------------------
# Native sharded iPI (ipi_solve_sharded): the production N > 1 path
# ----------------------------------------------------------------------------

class NativeComm:
    """The ``ipi_comm`` this rank hands to ``ipi_solve_sharded``.

    With NCCL (one process per GPU, NVLink / NVSwitch) it wraps torch's own
    communicator (``ProcessGroupNCCL._comm_ptr``): the collectives run as NCCL
    kernels on the solver's stream, nothing is staged through the host.  With
    gloo (CPU-side tests, several ranks sharing one GPU) the two callbacks copy
    the device buffers to the host, run the gloo collective and copy back — a
    functional stand-in, not a measurement.  World 1 needs no collectives."""

    def __init__(self, ctx: RankContext):
        import numpy as np
        import torch.distributed as dist
        self.ctx = ctx
        self.c = _lib.Comm()
        R = ctx.world
        starts = np.asarray(list(ctx.partition.block_starts), dtype=np.int64)
        self._starts = starts
        L = _lib.lib()
        self.kind = "local"
        import os
        force = bool(int(os.environ.get("IPI_COMM_FORCE_NCCL", "0") or 0))
        if (R > 1 or force) and dist.is_initialized() and dist.get_backend() == "nccl":
            # the communicator exists once a collective ran (eager init otherwise)
            dist.barrier()
            pg = dist.distributed_c10d._get_default_group()
            comm_ptr = pg._get_backend(torch.device("cuda"))._comm_ptr()
            _lib.check(L.ipi_comm_nccl(comm_ptr, ctx.rank, R, starts.ctypes.data,
                                       _lib.C.byref(self.c)), "ipi_comm_nccl")
            self.kind = "nccl"
        elif R > 1:
            self._cb_blocks = _lib.ALLGATHER_BLOCKS_FN(self._gloo_blocks)
            self._cb_gather = _lib.ALLGATHER_FN(self._gloo_gather)
            self.c.ctx = None
            self.c.rank, self.c.world = ctx.rank, R
            self.c.allgather_blocks = self._cb_blocks
            self.c.allgather = self._cb_gather
            self.kind = "gloo"
        else:
            _lib.check(L.ipi_comm_nccl(None, 0, 1, starts.ctypes.data, _lib.C.byref(self.c)),
                       "ipi_comm_nccl")

    # host-staged gloo collectives (callbacks from the native driver)
    def _gloo_blocks(self, _ctx, local_p, full_p, stream):
        import numpy as np
        import torch.distributed as dist
        try:
            L = _lib.lib()
            starts = self._starts
            lo, hi = int(starts[self.ctx.rank]), int(starts[self.ctx.rank + 1])
            loc = np.empty(hi - lo, dtype=np.float64)
            if hi > lo:
                _lib.check(L.ipi_memcpy_sync(loc.ctypes.data, local_p, 8 * (hi - lo), stream))
            sizes = [int(starts[q + 1] - starts[q]) for q in range(self.ctx.world)]
            mx = max(sizes)
            pad = torch.zeros(mx, dtype=torch.float64)
            pad[: hi - lo] = torch.from_numpy(loc)
            bufs = [torch.empty(mx, dtype=torch.float64) for _ in sizes]
            dist.all_gather(bufs, pad)
            full = np.concatenate([bufs[q][: sizes[q]].numpy() for q in range(len(sizes))])
            _lib.check(L.ipi_memcpy_sync(full_p, full.ctypes.data, 8 * full.size, stream))
            return 0
        except Exception:  # pragma: no cover - surfaced as the driver's error code
            import traceback
            traceback.print_exc()
            return 3

    def _gloo_gather(self, _ctx, send_p, out_p, count, stream):
        import numpy as np
        import torch.distributed as dist
        try:
            L = _lib.lib()
            snd = np.empty(count, dtype=np.float64)
            _lib.check(L.ipi_memcpy_sync(snd.ctypes.data, send_p, 8 * count, stream))
            bufs = [torch.empty(count, dtype=torch.float64) for _ in range(self.ctx.world)]
            dist.all_gather(bufs, torch.from_numpy(snd))
            out = torch.cat(bufs).numpy()
            _lib.check(L.ipi_memcpy_sync(out_p, out.ctypes.data, 8 * out.size, stream))
            return 0
        except Exception:  # pragma: no cover
            import traceback
            traceback.print_exc()
            return 3

    def __del__(self):
        if getattr(self, "kind", None) in ("nccl", "local"):
            try:
                _lib.lib().ipi_comm_nccl_destroy(_lib.C.byref(self.c))
            except Exception:
                pass


def solve_sharded_native(shard: "MdpShard", ctx: RankContext, opts, v0_local=None,
                         comm: NativeComm | None = None):
    """driver.py:109-209 across ranks through ``ipi_solve_sharded``: K1 on the
    shard with the all-gathered V, K2 on the local rows, the sharded GMRES
    (CGS2, 3 all-gathers of partial dots per Arnoldi step) or Richardson with
    every scalar on the device, one host sync per Arnoldi step and per outer
    iteration.  Honours ``opts.mode`` (overrides the shard's), ``opts.pc``
    (none / jacobi), ``opts.v0`` / ``v0_local`` (this rank's block).
    BiCGStab / TFQMR and the SOR / EXACT preconditioners raise
    NotImplementedError.  Returns a SolveResult whose values / policy are the
    gathered full vectors (identical on every rank)."""
    import numpy as np
    from .driver import SolveResult, SolveStatus
    from .inner import InnerSolver, Preconditioner
    opts.check()
    if opts.inner not in (InnerSolver.GMRES, InnerSolver.RICHARDSON):
        raise NotImplementedError(f"inner solver {opts.inner.value!r} runs on one GPU only; the "
                                  "sharded driver runs GMRES and Richardson")
    if opts.pc not in (Preconditioner.NONE, Preconditioner.JACOBI):
        raise NotImplementedError(f"preconditioner {opts.pc.value!r} is not on the device path")
    dev = shard.stage_cost.device
    lo, hi = ctx.block
    if v0_local is None and opts.v0 is not None:
        v0 = opts.v0
        v0_full = v0 if isinstance(v0, torch.Tensor) else torch.as_tensor(np.asarray(v0, np.float64))
        if tuple(v0_full.shape) != (shard.n_global,):
            from .model import ValidationError
            raise ValidationError(f"v0 length {tuple(v0_full.shape)} does not match n = {shard.n_global}")
        v0_local = v0_full[lo:hi]
    v = (torch.zeros(hi - lo, dtype=torch.float64, device=dev) if v0_local is None
         else v0_local.detach().to(dev, torch.float64).clone().contiguous())
    pol = torch.empty(hi - lo, dtype=torch.int32, device=dev)
    mode = opts.mode or shard.mode
    o = _lib.Opts(tol=opts.tol, alpha=opts.alpha, max_outer=opts.max_outer,
                  max_inner=opts.max_inner, ksp_type=_lib.KSP[opts.inner.value],
                  ksp_max_it=opts.ksp_max_it or 0, richardson_scale=opts.richardson_scale,
                  mode=_lib.MODE_MAX if mode is Mode.MAX else _lib.MODE_MIN,
                  pc_type=_lib.PC[opts.pc.value], gmres_ortho=_lib.ORTHO["cgs2"])
    comm = comm or NativeComm(ctx)
    hist = np.zeros(opts.max_outer + 2, dtype=np.float64)
    st = _lib.Stats()
    _lib.check(_lib.lib().ipi_solve_sharded(shard.handle(), _lib.C.byref(comm.c), _lib.C.byref(o),
                                            _lib.ptr(v), _lib.ptr(pol), hist.ctypes.data,
                                            hist.shape[0], _lib.C.byref(st), _lib.stream_ptr()),
               "ipi_solve_sharded")
    full = torch.empty(shard.n_global, dtype=torch.float64, device=dev)
    values = allgather_blocks(v, full, ctx.partition).clone()
    pol_full = allgather_blocks(pol.to(torch.float64), torch.empty_like(full), ctx.partition)
    nh = st.outer_iterations + 1
    return SolveResult(values=values.cpu().numpy(), policy=pol_full.cpu().numpy().astype(np.int64),
                       outer_iterations=st.outer_iterations,
                       inner_iterations_total=int(st.inner_iterations_total),
                       residual_history=[float(x) for x in hist[:nh]],
                       status=SolveStatus(_lib.STATUS[st.status]), wall_time=st.wall_time,
                       time_greedy=st.time_greedy, time_assembly=st.time_assembly,
                       time_inner=st.time_inner, values_device=values)
