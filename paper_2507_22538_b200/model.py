"""Data model: MDP instances resident in HBM, modes, partitions, validation.

Mirrors ``mdpsolve.model`` (reference ``pkg/src/mdpsolve/model.py``): same
names, argument meaning and error messages.  Differences are in storage only:
``MdpInstance`` keeps its stage costs and transition CSR as CUDA tensors
(row_ptr int64, col int32, values fp64; layout row ``s*m + a``,
model.py:112-131) and owns the device plan handle of libipi_b200.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ValidationError

ROW_SUM_TOL = 1e-12  # model.py:21

__all__ = ["ValidationError", "Mode", "flatten_index", "Partition", "make_partition",
           "MdpInstance", "validate", "require_valid", "ROW_SUM_TOL"]


class Mode(enum.Enum):
    """Optimisation sense (model.py:28-39).  ``from_name`` also accepts the
    madupite spellings MINCOST / MAXREWARD named by the north star."""

    MIN = "min"
    MAX = "max"

    @classmethod
    def from_name(cls, name: str) -> "Mode":
        key = str(name).strip().lower()
        key = {"mincost": "min", "maxreward": "max"}.get(key, key)
        try:
            return cls(key)
        except ValueError:
            raise ValidationError(
                f"unknown mode {name!r}; expected 'min' or 'max' (or MINCOST / MAXREWARD)"
            ) from None


def flatten_index(s: int, a: int, m: int, n: int | None = None) -> int:
    """Row of (s, a) in the row-stacked matrix (model.py:42-60)."""
    if m < 1:
        raise ValidationError(f"action count must be >= 1, got {m}")
    if a < 0 or a >= m:
        raise ValidationError(f"action index {a} out of range [0, {m})")
    if s < 0 or (n is not None and s >= n):
        raise ValidationError(f"state index {s} out of range [0, {n})")
    return s * m + a


@dataclass(frozen=True)
class Partition:
    """Contiguous state blocks per rank (model.py:63-92)."""

    worker_count: int
    block_starts: tuple[int, ...]

    def __post_init__(self) -> None:
        if self.worker_count < 1:
            raise ValidationError(f"worker count must be >= 1, got {self.worker_count}")
        bs = self.block_starts
        if len(bs) != self.worker_count + 1 or bs[0] != 0:
            raise ValidationError("block_starts must have worker_count+1 entries starting at 0")
        if any(bs[i] > bs[i + 1] for i in range(self.worker_count)):
            raise ValidationError("block_starts must be non-decreasing")

    @property
    def n(self) -> int:
        return self.block_starts[-1]

    def block(self, r: int) -> tuple[int, int]:
        return self.block_starts[r], self.block_starts[r + 1]

    def block_sizes(self) -> list[int]:
        return [self.block_starts[r + 1] - self.block_starts[r] for r in range(self.worker_count)]


def make_partition(n: int, worker_count: int) -> Partition:
    """Balanced partition: rank r gets floor(n/R)+1 states if r < n mod R
    (model.py:95-109).  Used for GPU row sharding."""
    if n < 0:
        raise ValidationError(f"state count must be >= 0, got {n}")
    if worker_count < 1:
        raise ValidationError(f"worker count must be >= 1, got {worker_count}")
    base, extra = divmod(n, worker_count)
    starts = [0]
    for r in range(worker_count):
        starts.append(starts[-1] + base + (1 if r < extra else 0))
    return Partition(worker_count=worker_count, block_starts=tuple(starts))


def _device() -> torch.device:
    from . import _lib
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def as_device_f64(x, shape=None) -> torch.Tensor:
    """Contiguous fp64 CUDA copy/view of an array-like."""
    dev = _device()
    if isinstance(x, torch.Tensor):
        t = x.detach().to(device=dev, dtype=torch.float64)
    else:
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device=dev)
    t = t.contiguous()
    if shape is not None:
        t = t.reshape(shape)
    return t


class MdpInstance:
    """Complete MDP description held in HBM (model.py:112-145).

    ``stage_cost`` is an (n, m) fp64 CUDA tensor, ``transitions`` a device
    :class:`~paper_2507_22538_b200.sparse.CsrMatrix` of shape (n*m, n).
    Construction copies host inputs to the device once; the kernel plan
    (lanes per row, shared-memory V window, CTA partition) is built lazily on
    first use and cached with the instance.
    """

    def __init__(self, n: int, m: int, gamma: float, stage_cost, transitions, mode: Mode = Mode.MIN):
        from .sparse import CsrMatrix
        self.n = int(n)
        self.m = int(m)
        self.gamma = float(gamma)
        self.mode = mode
        cost = stage_cost
        if isinstance(cost, torch.Tensor) or isinstance(cost, np.ndarray):
            pass
        else:
            cost = np.asarray(cost, dtype=np.float64)
        self.stage_cost = as_device_f64(cost)
        if not isinstance(transitions, CsrMatrix):
            raise ValidationError("transitions must be a CsrMatrix")
        self.transitions = transitions
        self._handle = None
        self._handle_mode = None

    # ------------------------------------------------------------------
    def policy_is_valid(self, pi) -> bool:
        t = pi if isinstance(pi, torch.Tensor) else torch.as_tensor(np.asarray(pi))
        return tuple(t.shape) == (self.n,) and bool(((t >= 0) & (t < self.m)).all())

    def shapes_consistent(self) -> bool:
        t = self.transitions
        return (tuple(self.stage_cost.shape) == (self.n, self.m)
                and (t.rows, t.cols) == (self.n * self.m, self.n))

    def handle(self):
        """Device plan handle (ipi_mdp*); built once per instance."""
        from . import _lib
        if self._handle is not None:
            return self._handle
        if not self.shapes_consistent():
            raise ValidationError("; ".join(validate_shapes(self)) or "inconsistent instance shapes")
        L = _lib.lib()
        out = _lib.C.c_void_p()
        t = self.transitions
        rc = L.ipi_mdp_create(_lib.ptr(t.row_ptr), _lib.ptr(t.col_idx), _lib.ptr(t.values),
                              _lib.ptr(self.stage_cost), self.n, self.n, self.m, 0, self.gamma,
                              _lib.MODE_MAX if self.mode is Mode.MAX else _lib.MODE_MIN,
                              _lib.stream_ptr(), _lib.C.byref(out))
        _lib.check(rc, "ipi_mdp_create")
        self._handle = out
        return out

    def plan(self) -> dict:
        from . import _lib
        p = _lib.Plan()
        _lib.check(_lib.lib().ipi_mdp_plan(self.handle(), _lib.C.byref(p)), "ipi_mdp_plan")
        return p.as_dict()

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                from . import _lib
                torch.cuda.synchronize()
                _lib.lib().ipi_mdp_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._handle = None

    def __repr__(self) -> str:
        return (f"MdpInstance(n={self.n}, m={self.m}, gamma={self.gamma}, mode={self.mode.value}, "
                f"nnz={self.transitions.nnz})")


def validate_shapes(mdp: MdpInstance) -> list[str]:
    problems = []
    if mdp.n < 1:
        problems.append(f"state count must be >= 1, got {mdp.n}")
    if mdp.m < 1:
        problems.append(f"action count must be >= 1, got {mdp.m}")
    if not (0.0 < mdp.gamma < 1.0) or not math.isfinite(mdp.gamma):
        problems.append(f"discount factor must lie in (0, 1), got {mdp.gamma}")
    if tuple(mdp.stage_cost.shape) != (mdp.n, mdp.m):
        problems.append(f"stage cost shape {tuple(mdp.stage_cost.shape)} does not match "
                        f"(n, m) = ({mdp.n}, {mdp.m})")
    t = mdp.transitions
    if (t.rows, t.cols) != (mdp.n * mdp.m, mdp.n):
        problems.append(f"transition matrix shape ({t.rows}, {t.cols}) does not match (n*m, n) = "
                        f"({mdp.n * mdp.m}, {mdp.n})")
    return problems


def validate(mdp: MdpInstance) -> list[str]:
    """Every model invariant, checked on the device; returns the violations
    in the reference's order and wording (model.py:148-194)."""
    from . import _lib
    problems: list[str] = []
    if mdp.n < 1:
        problems.append(f"state count must be >= 1, got {mdp.n}")
    if mdp.m < 1:
        problems.append(f"action count must be >= 1, got {mdp.m}")
    if not (0.0 < mdp.gamma < 1.0) or not math.isfinite(mdp.gamma):
        problems.append(f"discount factor must lie in (0, 1), got {mdp.gamma}")
    cost_ok = tuple(mdp.stage_cost.shape) == (mdp.n, mdp.m)
    if not cost_ok:
        problems.append(f"stage cost shape {tuple(mdp.stage_cost.shape)} does not match "
                        f"(n, m) = ({mdp.n}, {mdp.m})")
    elif mdp.stage_cost.numel() and not bool(torch.isfinite(mdp.stage_cost).all()):
        flat = int(torch.nonzero(~torch.isfinite(mdp.stage_cost.reshape(-1)))[0])
        s, a = divmod(flat, mdp.m)
        problems.append(f"stage cost has non-finite entries, first at (s={s}, a={a})")
    t = mdp.transitions
    if (t.rows, t.cols) != (mdp.n * mdp.m, mdp.n):
        problems.append(f"transition matrix shape ({t.rows}, {t.cols}) does not match (n*m, n) = "
                        f"({mdp.n * mdp.m}, {mdp.n})")
        return problems
    structural = t.check()
    if structural:
        problems.extend(f"transition matrix: {msg}" for msg in structural)
        return problems
    if mdp.n < 1 or mdp.m < 1:
        return problems
    if cost_ok:
        h = mdp.handle()
        tmp = None
    else:  # validate the transitions against a placeholder cost of the right size
        tmp = MdpInstance(mdp.n, mdp.m, 0.5, torch.zeros((mdp.n, mdp.m), dtype=torch.float64,
                                                         device=t.values.device), t)
        h = tmp.handle()
    v = _lib.Validation()
    _lib.check(_lib.lib().ipi_validate(h, _lib.C.byref(v), _lib.stream_ptr()), "ipi_validate")
    if v.first_bad_prob >= 0:
        problems.append(f"transition probabilities must lie in [0, 1]; entry {v.first_bad_prob} "
                        f"is {v.first_bad_prob_value}")
    if v.n_bad_row_sums > 0:
        shown = ", ".join(f"row {v.bad_rows[i]} sums to {v.bad_row_sums[i]:.15g}"
                          for i in range(min(5, v.n_bad_row_sums)) if v.bad_rows[i] >= 0)
        more = "" if v.n_bad_row_sums <= 5 else f" (and {v.n_bad_row_sums - 5} more)"
        problems.append(f"transition rows must sum to 1 within {ROW_SUM_TOL}: {shown}{more}")
    del tmp
    return problems


def require_valid(mdp: MdpInstance) -> None:
    problems = validate(mdp)
    if problems:
        raise ValidationError("; ".join(problems))
