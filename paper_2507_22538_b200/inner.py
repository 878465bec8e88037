"""Policy-evaluation Krylov solves on the device (mirrors ``mdpsolve.inner``).

``inner_solve`` (inner.py:163-213) runs the whole solve — Richardson,
restarted GMRES(30) with Givens rotations (CGS2 or the reference's MGS), BiCGStab or TFQMR, each with the
reference's estimate-then-verify stopping and breakdown reporting — as one
persistent cooperative kernel (krylov*.cu).  Preconditioning: NONE or
JACOBI on the device path (left preconditioning exactly as the reference
applies it); SOR and EXACT (dense) are out of scope this round.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sparse import PolicyOperator

GMRES_RESTART = 30          # inner.py:40
TARGET_FLOOR_SCALE = 1e-14  # inner.py:41
DEFAULT_ASSEMBLY_CAP_NNZ = 20_000_000
DEFAULT_DENSE_CAP = 4096

__all__ = ["InnerSolver", "Preconditioner", "InnerSolveReport", "inner_solve",
           "build_preconditioner", "GMRES_RESTART", "TARGET_FLOOR_SCALE"]


class InnerSolver(enum.Enum):
    """inner.py:48-62."""

    RICHARDSON = "richardson"
    GMRES = "gmres"
    BICGSTAB = "bicgstab"
    TFQMR = "tfqmr"

    @classmethod
    def from_name(cls, name: str) -> "InnerSolver":
        try:
            return cls(name.strip().lower())
        except ValueError:
            valid = ", ".join(k.value for k in cls)
            raise ValueError(f"unknown inner solver {name!r}; supported: {valid}") from None


class Preconditioner(enum.Enum):
    """inner.py:65-84."""

    NONE = "none"
    JACOBI = "jacobi"
    SOR_FORWARD = "sor"
    EXACT = "svd"

    @classmethod
    def from_name(cls, name: str) -> "Preconditioner":
        try:
            return cls(name.strip().lower())
        except ValueError:
            valid = ", ".join(k.value for k in cls)
            raise ValueError(f"unknown preconditioner {name!r}; supported: {valid}") from None


DEVICE_KINDS = (InnerSolver.RICHARDSON, InnerSolver.GMRES, InnerSolver.BICGSTAB,
                InnerSolver.TFQMR)


@dataclass(frozen=True)
class InnerSolveReport:
    """inner.py:87-95."""

    iterations: int
    final_linear_residual_2norm: float
    converged: bool
    breakdown: bool
    target_2norm: float


class JacobiPreconditioner:
    """pc(r) = r / (1 - gamma diag(P_pi)) (inner.py:115-118), inverse diagonal in HBM."""

    def __init__(self, op: PolicyOperator):
        p = op.p_pi
        self.inv_diag = torch.empty(op.n, dtype=torch.float64, device=p.values.device)
        _lib.check(_lib.lib().ipi_jacobi_inv_diag(_lib.ptr(p.row_ptr), _lib.ptr(p.col_idx),
                                                  _lib.ptr(p.values), op.n, op.gamma,
                                                  _lib.ptr(self.inv_diag), _lib.stream_ptr()),
                   "ipi_jacobi_inv_diag")

    def __call__(self, r):
        was_np = not isinstance(r, torch.Tensor)
        t = torch.as_tensor(np.asarray(r, dtype=np.float64), device=self.inv_diag.device) \
            if was_np else r.to(self.inv_diag.device, torch.float64)
        out = t * self.inv_diag
        return out.cpu().numpy() if was_np else out


def build_preconditioner(op, kind: Preconditioner, **_):
    """NONE -> None (identity), JACOBI -> JacobiPreconditioner (inner.py:98-133).
    SOR / EXACT need explicit assembly and are not on the device path."""
    if kind is Preconditioner.NONE:
        return None
    if kind is Preconditioner.JACOBI:
        return JacobiPreconditioner(op)
    raise NotImplementedError(f"preconditioner {kind.value!r} is not on the B200 device path")


def inner_solve(op: PolicyOperator, b, theta0, target_2norm: float, max_it: int,
                kind: InnerSolver = InnerSolver.GMRES, pc=None, richardson_scale: float = 1.0,
                workers=None, halo: int = -1, ortho: str = "auto"):
    """Approximately solve (I - gamma P) theta = b from theta0 (inner.py:163-213).

    ``ortho`` (extension): GMRES orthogonalisation, "auto" (default), the
    reference's "mgs", or "cgs2"."""
    was_np = not isinstance(b, torch.Tensor)
    dev = op.p_pi.values.device
    bt = torch.as_tensor(np.asarray(b, dtype=np.float64), device=dev) if was_np else \
        b.detach().to(dev, torch.float64)
    x = torch.as_tensor(np.array(theta0, dtype=np.float64), device=dev) if not isinstance(
        theta0, torch.Tensor) else theta0.detach().to(dev, torch.float64).clone()
    if tuple(bt.shape) != (op.n,) or tuple(x.shape) != (op.n,):
        raise ValueError(f"rhs/start length must be {op.n}")
    if max_it < 1:
        raise ValueError(f"iteration cap must be >= 1, got {max_it}")
    if target_2norm < 0.0:
        raise ValueError(f"residual target must be >= 0, got {target_2norm}")
    if pc is not None and not isinstance(pc, JacobiPreconditioner):
        raise NotImplementedError("only the identity and Jacobi preconditioners run on the device")
    if kind not in DEVICE_KINDS:
        raise NotImplementedError(f"inner solver {kind.value!r} is not on the device path yet")
    if ortho not in _lib.ORTHO:
        raise ValueError(f"unknown GMRES orthogonalisation {ortho!r}; supported: "
                         f"{', '.join(_lib.ORTHO)}")
    bt = bt.contiguous()
    x = x.contiguous()
    rep = _lib.InnerReport()
    p = op.p_pi
    _lib.check(_lib.lib().ipi_inner_solve(_lib.ptr(p.row_ptr), _lib.ptr(p.col_idx),
                                          _lib.ptr(p.values), op.n, op.gamma, _lib.ptr(bt),
                                          _lib.ptr(x), float(target_2norm), int(max_it),
                                          _lib.KSP[kind.value], float(richardson_scale),
                                          _lib.ptr(pc.inv_diag) if pc is not None else None,
                                          _lib.ORTHO[ortho], _lib.C.byref(rep),
                                          _lib.stream_ptr()), "ipi_inner_solve")
    report = InnerSolveReport(iterations=rep.iterations,
                              final_linear_residual_2norm=rep.final_linear_residual_2norm,
                              converged=bool(rep.converged), breakdown=bool(rep.breakdown),
                              target_2norm=rep.target_2norm)
    return (x.cpu().numpy() if was_np else x), report
