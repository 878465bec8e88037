"""Bellman operators on the device (mirrors ``mdpsolve.bellman``).

``greedy_policy`` (bellman.py:44-68) is ONE launch of the fused K1 kernel:
SpMV over the (n*m) x n CSR + stage cost + gamma + per-state first-index
argmin/argmax + the residual max, never materialising the n*m product.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .model import MdpInstance, Mode, ValidationError
from .sparse import gather_policy_cost, gather_policy_matrix, norm, spmv

__all__ = ["GreedyResult", "greedy_policy", "bellman_residual", "policy_residual"]

# pinned-host-tensor path: K1 writes its outputs into the mapped host buffers
# (IPI_ZERO_COPY=0: device outputs + D2H copies after the kernel)
_ZERO_COPY = os.environ.get("IPI_ZERO_COPY", "1") != "0"


@dataclass(frozen=True)
class GreedyResult:
    """Greedy policy (int64) and ``applied = (T V)`` (bellman.py:31-41)."""

    policy: object
    applied: object


def _check_cost_vector(mdp: MdpInstance, v):
    """bellman.py:123-129; returns (device fp64 tensor, input_was_numpy)."""
    was_np = not isinstance(v, torch.Tensor)
    if was_np:
        arr = np.asarray(v, dtype=np.float64)
        if arr.shape != (mdp.n,):
            raise ValidationError(f"cost vector length {arr.shape} does not match n = {mdp.n}")
        if not np.isfinite(arr).all():
            raise ValidationError("cost vector has non-finite entries")
        _lib.require_cuda()
        t = torch.as_tensor(np.ascontiguousarray(arr), device=mdp.stage_cost.device)
    else:
        t = v.detach().to(device=mdp.stage_cost.device, dtype=torch.float64).contiguous()
        if tuple(t.shape) != (mdp.n,):
            raise ValidationError(f"cost vector length {tuple(t.shape)} does not match n = {mdp.n}")
        if not bool(torch.isfinite(t).all()):
            raise ValidationError("cost vector has non-finite entries")
    return t, was_np


def greedy_device(mdp: MdpInstance, v: torch.Tensor, mode: Mode, *, with_residual: bool = False):
    """K1 on device tensors: (policy int32, applied f64, residual-bits tensor | None)."""
    h = mdp.handle()
    dev = v.device
    pi = torch.empty(mdp.n, dtype=torch.int32, device=dev)
    applied = torch.empty(mdp.n, dtype=torch.float64, device=dev)
    res = torch.zeros(1, dtype=torch.int64, device=dev) if with_residual else None
    _lib.check(_lib.lib().ipi_bellman(h, _lib.ptr(v), _lib.MODE_MAX if mode is Mode.MAX else
                                      _lib.MODE_MIN, _lib.ptr(pi), _lib.ptr(applied), None, None,
                                      _lib.ptr(res), _lib.stream_ptr()), "ipi_bellman")
    return pi, applied, res


def greedy_policy(mdp: MdpInstance, v, mode: Mode | None = None, workers=None) -> GreedyResult:
    """Greedy policy for cost vector ``v``; ties pick the smallest action.

    Output placement follows the input: numpy in -> numpy out (int64 policy,
    like bellman.py:54); CUDA tensor in -> CUDA tensors out; CPU tensor in
    (e.g. pinned host memory) -> one H2D copy of V and one K1 launch whose
    policy / TV stores go straight to pinned host tensors (zero-copy)."""
    host_torch = isinstance(v, torch.Tensor) and v.device.type == "cpu"
    if host_torch:
        if tuple(v.shape) != (mdp.n,):
            raise ValidationError(f"cost vector length {tuple(v.shape)} does not match n = {mdp.n}")
        vt = v.to(mdp.stage_cost.device, torch.float64, non_blocking=True)
        finite = torch.isfinite(vt).all()  # read after the one sync below
        pol_h = torch.empty(mdp.n, dtype=torch.int32, pin_memory=True)
        app_h = torch.empty(mdp.n, dtype=torch.float64, pin_memory=True)
        if _ZERO_COPY:
            # K1 stores the policy / TV straight into the pinned (UVA-mapped)
            # host buffers while it streams: the D2H transfer overlaps the kernel
            md = _lib.MODE_MAX if (mode or mdp.mode) is Mode.MAX else _lib.MODE_MIN
            _lib.check(_lib.lib().ipi_bellman(mdp.handle(), _lib.ptr(vt), md, pol_h.data_ptr(),
                                              app_h.data_ptr(), None, None, None,
                                              _lib.stream_ptr()), "ipi_bellman")
        else:
            pi, applied, _ = greedy_device(mdp, vt, mode or mdp.mode)
            pol_h.copy_(pi, non_blocking=True)
            app_h.copy_(applied, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if not bool(finite):
            raise ValidationError("cost vector has non-finite entries")
        return GreedyResult(policy=pol_h, applied=app_h)
    vt, was_np = _check_cost_vector(mdp, v)
    mode = mode or mdp.mode
    pi, applied, _ = greedy_device(mdp, vt, mode)
    if was_np:
        return GreedyResult(policy=pi.cpu().numpy().astype(np.int64), applied=applied.cpu().numpy())
    return GreedyResult(policy=pi.long(), applied=applied)


def bellman_residual(mdp: MdpInstance, v, mode: Mode | None = None, workers=None):
    """``r = v - Tv`` and its infinity norm (bellman.py:71-79)."""
    vt, was_np = _check_cost_vector(mdp, v)
    _, applied, _ = greedy_device(mdp, vt, mode or mdp.mode)
    r = vt - applied
    return (r.cpu().numpy() if was_np else r), norm(r, "inf")


def policy_residual(mdp: MdpInstance, pi, v, workers=None):
    """``r = v - (g_pi + gamma P_pi v)`` and its infinity norm (bellman.py:82-93)."""
    vt, was_np = _check_cost_vector(mdp, v)
    p_pi = gather_policy_matrix(mdp, pi)
    g_pi = gather_policy_cost(mdp, torch.as_tensor(np.asarray(pi)) if not isinstance(pi, torch.Tensor) else pi)
    r = vt - (g_pi + mdp.gamma * spmv(p_pi, vt))
    return (r.cpu().numpy() if was_np else r), norm(r, "inf")
