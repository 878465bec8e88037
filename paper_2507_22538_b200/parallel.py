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

from dataclasses import dataclass

import torch

from . import _lib
from .model import Mode, Partition, make_partition
from .sparse import CsrMatrix

__all__ = ["MdpShard", "RankContext", "allgather_blocks", "rank_ordered_sum", "rank_max"]


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
        if full.device.type == "cuda":
            dist.all_gather_into_tensor(full, local.contiguous())
        else:
            parts = list(full.split(sizes))
            dist.all_gather(parts, local.contiguous())
        return full
    mx = max(sizes)
    pad = torch.zeros(mx, dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    buf = torch.empty(mx * R, dtype=local.dtype, device=local.device)
    if buf.device.type == "cuda":
        dist.all_gather_into_tensor(buf, pad)
    else:
        dist.all_gather(list(buf.split(mx)), pad)
    for r in range(R):
        lo, hi = partition.block(r)
        full[lo:hi] = buf[r * mx: r * mx + (hi - lo)]
    return full


def rank_ordered_sum(partial: torch.Tensor, world: int) -> torch.Tensor:
    """Deterministic all-reduce: gather the R partials, add them in rank order."""
    import torch.distributed as dist
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return partial.clone()
    parts = torch.empty((world,) + tuple(partial.shape), dtype=partial.dtype, device=partial.device)
    if partial.device.type == "cuda":
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
        if residual:
            self.res_bits.zero_()
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
