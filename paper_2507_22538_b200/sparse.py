"""Device CSR container, SpMV, reductions, policy gather, evaluation operator.

Mirrors ``mdpsolve.sparse`` (reference ``pkg/src/mdpsolve/sparse.py``):
``CsrMatrix`` (:30-123), ``spmv`` (:189-215), ``dot``/``norm`` (:218-240),
``gather_policy_matrix``/``gather_policy_cost`` (:243-269),
``PolicyOperator`` (:272-295).  Storage is HBM: row_ptr int64, col int32
(column counts are < 2^31 for every config), values fp64.  SpMV, gather and
the evaluation operator run in libipi_b200 kernels; inputs given as numpy
come back as numpy, torch CUDA tensors stay on the device.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, ResourceLimitError

__all__ = ["CsrMatrix", "DimensionError", "ResourceLimitError", "spmv", "dot", "norm",
           "gather_policy_matrix", "gather_policy_cost", "PolicyOperator"]


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x, dtype) -> torch.Tensor:
    dev = _dev()
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x)), device=dev).to(dtype).contiguous()


class CsrMatrix:
    """Compressed sparse row matrix over float64, resident on the GPU.

    Row ``i`` stores strictly increasing column indices in
    ``col_idx[row_ptr[i]:row_ptr[i+1]]``.  The structure is verified on the
    device at construction and a violation raises ``ValueError("invalid CSR
    structure: ...")`` exactly like the reference (sparse.py:45-54).
    """

    def __init__(self, rows: int, cols: int, row_ptr, col_idx, values):
        self.rows = int(rows)
        self.cols = int(cols)
        problems = self._ingest(row_ptr, col_idx, values)
        if problems:
            raise ValueError("invalid CSR structure: " + "; ".join(problems))

    def _ingest(self, row_ptr, col_idx, values) -> list[str]:
        rows, cols = self.rows, self.cols
        if rows < 0 or cols < 0:
            self.row_ptr = self.col_idx = self.values = None
            return [f"negative shape ({rows}, {cols})"]
        rp = _to_dev(row_ptr, torch.int64).reshape(-1)
        vals = _to_dev(values, torch.float64).reshape(-1)
        narrow = isinstance(col_idx, torch.Tensor) and col_idx.dtype == torch.int32
        if narrow:  # already the device layout: no int64 round trip (2^31-nnz shards)
            ci_wide = None
            ci = _to_dev(col_idx, torch.int32).reshape(-1)
        else:
            ci_src = col_idx if isinstance(col_idx, torch.Tensor) else np.asarray(col_idx)
            ci_wide = _to_dev(ci_src, torch.int64).reshape(-1)
        problems: list[str] = []
        self.row_ptr, self.values = rp, vals
        if rp.shape[0] != rows + 1:
            self.col_idx = ci if narrow else ci_wide.to(torch.int32)
            return [f"row_ptr length {rp.shape[0]} != rows+1 = {rows + 1}"]
        if cols > np.iinfo(np.int32).max:
            raise DimensionError("column count exceeds the int32 index range of the device layout")
        if not narrow:
            # narrowing to int32 keeps order; anything beyond int32 is out of range anyway
            ci = ci_wide.clamp(-(2 ** 31), 2 ** 31 - 1).to(torch.int32)
            del ci_wide
        self.col_idx = ci
        rep = _lib.CsrReport()
        _lib.check(_lib.lib().ipi_csr_check(_lib.ptr(rp), _lib.ptr(ci), _lib.ptr(vals), rows, cols,
                                            ci.shape[0] if ci.shape[0] == vals.shape[0] else -1,
                                            _lib.C.byref(rep), _lib.stream_ptr()), "ipi_csr_check")
        if rep.bad_row_ptr:
            return ["row_ptr must be non-decreasing and start at 0"]
        if rep.nnz_mismatch:
            return [f"col_idx/values length must equal nnz = {rep.nnz}"]
        if rep.nnz:
            if rep.bad_col_range:
                problems.append(f"column indices must lie in [0, {cols})")
            if rep.bad_col_order:
                problems.append("column indices must be strictly increasing within each row")
            if rep.nonfinite_values:
                problems.append("values must all be finite")
        return problems

    def check(self) -> list[str]:
        """Structural invariants hold by construction (verified on device)."""
        return []

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def row_lengths(self) -> torch.Tensor:
        return self.row_ptr[1:] - self.row_ptr[:-1]

    def row_sums(self) -> torch.Tensor:
        return spmv(self, torch.ones(self.cols, dtype=torch.float64, device=self.values.device))

    def diagonal(self) -> torch.Tensor:
        k = min(self.rows, self.cols)
        d = torch.zeros(k, dtype=torch.float64, device=self.values.device)
        er = torch.repeat_interleave(torch.arange(self.rows, device=self.values.device),
                                     self.row_lengths())
        mask = er == self.col_idx.long()
        d[self.col_idx.long()[mask]] = self.values[mask]
        return d

    def to_dense(self) -> torch.Tensor:
        out = torch.zeros((self.rows, self.cols), dtype=torch.float64, device=self.values.device)
        er = torch.repeat_interleave(torch.arange(self.rows, device=self.values.device),
                                     self.row_lengths())
        out[er, self.col_idx.long()] = self.values
        return out

    def equals(self, other: "CsrMatrix") -> bool:
        return (self.shape == other.shape and torch.equal(self.row_ptr, other.row_ptr)
                and torch.equal(self.col_idx, other.col_idx) and torch.equal(self.values, other.values))

    def numpy(self):
        """(row_ptr int64, col_idx int32, values f64) host copies."""
        return (self.row_ptr.cpu().numpy(), self.col_idx.cpu().numpy(), self.values.cpu().numpy())

    def __repr__(self) -> str:
        return f"CsrMatrix(shape={self.shape}, nnz={self.nnz}, device={self.values.device})"


def _vec(x, n: int | None, what: str):
    """(device fp64 tensor, was_numpy) for an input vector."""
    was_np = not isinstance(x, torch.Tensor)
    t = _to_dev(x, torch.float64)
    return t, was_np


def _out(t: torch.Tensor, as_numpy: bool):
    return t.cpu().numpy() if as_numpy else t


def spmv(a: CsrMatrix, x, workers=None, block_scale: int = 1):
    """y = A x on the device (sparse.py:189-215)."""
    xt, was_np = _vec(x, a.cols, "x")
    if tuple(xt.shape) != (a.cols,):
        raise DimensionError(f"spmv: vector length {tuple(xt.shape)} incompatible with {a.shape}")
    y = torch.empty(a.rows, dtype=torch.float64, device=xt.device)
    _lib.check(_lib.lib().ipi_spmv(_lib.ptr(a.row_ptr), _lib.ptr(a.col_idx), _lib.ptr(a.values),
                                   a.rows, a.cols, _lib.ptr(xt), _lib.ptr(y), _lib.stream_ptr()),
               "ipi_spmv")
    return _out(y, was_np)


def dot(x, y, workers=None) -> float:
    xt, _ = _vec(x, None, "x")
    yt, _ = _vec(y, None, "y")
    if xt.shape != yt.shape:
        raise DimensionError(f"dot: length mismatch {tuple(xt.shape)} vs {tuple(yt.shape)}")
    return float(torch.dot(xt, yt))


def norm(x, kind: str = "two", workers=None) -> float:
    xt, _ = _vec(x, None, "x")
    if kind == "inf":
        return float(xt.abs().max()) if xt.numel() else 0.0
    if kind == "two":
        return math.sqrt(dot(xt, xt))
    raise ValueError(f"unknown norm kind {kind!r}; expected 'two' or 'inf'")


def _policy_dev(mdp, pi) -> torch.Tensor:
    t = _to_dev(pi, torch.int64)
    if tuple(t.shape) != (mdp.n,) or not bool(((t >= 0) & (t < mdp.m)).all()):
        raise ValueError("policy has wrong length or out-of-range action indices")
    return t.to(torch.int32).contiguous()


def gather_policy_matrix(mdp, pi) -> CsrMatrix:
    """n x n P_pi, row s = row s*m + pi[s] (sparse.py:243-261); K2 kernel."""
    p32 = _policy_dev(mdp, pi)
    h = mdp.handle()
    nnz = _lib.C.c_int64()
    L = _lib.lib()
    _lib.check(L.ipi_policy_nnz(h, _lib.ptr(p32), _lib.C.byref(nnz), _lib.stream_ptr()),
               "ipi_policy_nnz")
    dev = p32.device
    rp = torch.empty(mdp.n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
    _lib.check(L.ipi_gather_policy(h, _lib.ptr(p32), _lib.ptr(rp), _lib.ptr(col), _lib.ptr(val),
                                   None, _lib.stream_ptr()), "ipi_gather_policy")
    out = CsrMatrix.__new__(CsrMatrix)
    out.rows = out.cols = mdp.n
    out.row_ptr, out.col_idx, out.values = rp, col[:nnz.value], val[:nnz.value]
    return out


def gather_policy_cost(mdp, pi):
    """g_pi[s] = stage_cost[s, pi[s]] (sparse.py:264-269)."""
    was_np = not isinstance(pi, torch.Tensor)
    p = _policy_dev(mdp, pi).long()
    g = mdp.stage_cost[torch.arange(mdp.n, device=p.device), p].contiguous()
    return _out(g, was_np)


class DeviceOperator:
    """A planned K3 operator (``ipi_op_create``): J = I - gamma*P over rows
    [0, n_local) of a P_pi row block whose row r is state ``state0 + r`` of an
    ``n_global``-state system (state0 = 0, n_local = n_global unsharded).
    Planning syncs once (row statistics, locality profile); ``apply`` /
    ``spmv`` never do.  Holds references to the CSR tensors it borrows."""

    def __init__(self, row_ptr: torch.Tensor, col_idx: torch.Tensor, values: torch.Tensor,
                 n_local: int, n_global: int, state0: int, gamma: float):
        self._keep = (row_ptr, col_idx, values)
        self.n_local, self.n_global, self.state0 = int(n_local), int(n_global), int(state0)
        self.gamma = float(gamma)
        h = _lib.C.c_void_p()
        _lib.check(_lib.lib().ipi_op_create(_lib.ptr(row_ptr), _lib.ptr(col_idx), _lib.ptr(values),
                                            self.n_local, self.n_global, self.state0, self.gamma,
                                            _lib.stream_ptr(), _lib.C.byref(h)), "ipi_op_create")
        self._h = h.value

    def plan(self) -> dict:
        out = _lib.OpPlan()
        _lib.check(_lib.lib().ipi_op_get_plan(self._h, _lib.C.byref(out)), "ipi_op_get_plan")
        return out.as_dict()

    def apply(self, x_full: torch.Tensor, b: torch.Tensor | None = None,
              out: torch.Tensor | None = None) -> torch.Tensor:
        """x - gamma*(P x) on the rows (b - that when b is given)."""
        y = out if out is not None else torch.empty(self.n_local, dtype=torch.float64,
                                                    device=x_full.device)
        _lib.check(_lib.lib().ipi_op_apply(self._h, _lib.ptr(x_full), _lib.ptr(b), _lib.ptr(y),
                                           _lib.stream_ptr()), "ipi_op_apply")
        return y

    def apply_partial(self, x_full: torch.Tensor, y_partial: torch.Tensor,
                      b: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """x[s] - gamma*(y_partial + P x) on the rows (b - that when b is given):
        the remote-column half of a split apply."""
        y = out if out is not None else torch.empty(self.n_local, dtype=torch.float64,
                                                    device=x_full.device)
        _lib.check(_lib.lib().ipi_op_apply_partial(self._h, _lib.ptr(x_full), _lib.ptr(y_partial),
                                                   _lib.ptr(b), _lib.ptr(y), _lib.stream_ptr()),
                   "ipi_op_apply_partial")
        return y

    def spmv(self, x_full: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = out if out is not None else torch.empty(self.n_local, dtype=torch.float64,
                                                    device=x_full.device)
        _lib.check(_lib.lib().ipi_op_spmv(self._h, _lib.ptr(x_full), _lib.ptr(y),
                                          _lib.stream_ptr()), "ipi_op_spmv")
        return y

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().ipi_op_destroy(h)
            except Exception:
                pass
            self._h = None


class PolicyOperator:
    """Matrix-free I - gamma*P_pi; ``apply(x) = x - gamma*(P x)`` with that
    exact two-step rounding (sparse.py:272-295), one fused kernel (K3, planned
    on the first apply: ``DeviceOperator``)."""

    def __init__(self, p_pi: CsrMatrix, gamma: float):
        if p_pi.rows != p_pi.cols:
            raise DimensionError("policy transition matrix must be square")
        if not (0.0 <= gamma < 1.0):
            raise ValueError(f"discount factor must lie in [0, 1), got {gamma}")
        self.p_pi = p_pi
        self.gamma = float(gamma)
        self._op: DeviceOperator | None = None

    @property
    def n(self) -> int:
        return self.p_pi.rows

    def device_operator(self) -> DeviceOperator:
        if self._op is None:
            p = self.p_pi
            self._op = DeviceOperator(p.row_ptr, p.col_idx, p.values, self.n, self.n, 0, self.gamma)
        return self._op

    def apply(self, x, workers=None):
        xt, was_np = _vec(x, self.n, "x")
        if tuple(xt.shape) != (self.n,):
            raise DimensionError(f"apply: vector length {tuple(xt.shape)} != {self.n}")
        return _out(self.device_operator().apply(xt.contiguous()), was_np)
