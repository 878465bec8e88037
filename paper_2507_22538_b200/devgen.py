"""Device builders for the BASELINE configs (wrappers over ipi_gen_*).

Returns CUDA tensors in the instance layout; see generators.py for the
recipes and their host restatements.
"""

from __future__ import annotations

import torch

from . import _lib
from .generators import CONFIGS, ConfigSpec
from .model import MdpInstance, Mode
from .sparse import CsrMatrix


def _alloc(rows: int, nnz: int, dev):
    return (torch.empty(rows + 1, dtype=torch.int64, device=dev),
            torch.empty(max(nnz, 1), dtype=torch.int32, device=dev),
            torch.empty(max(nnz, 1), dtype=torch.float64, device=dev),
            torch.empty(max(rows, 1), dtype=torch.float64, device=dev))


def locality(n: int, m: int, K: int, W: int, seed: int = 0, state0: int = 0,
             n_states: int | None = None):
    """Rows of states [state0, state0+n_states) of the C2/C5 recipe."""
    _lib.require_cuda()
    ns = n - state0 if n_states is None else n_states
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = ns * m
    rp, col, val, cost = _alloc(rows, rows * K, dev)
    _lib.check(_lib.lib().ipi_gen_locality(n, m, K, W, seed, state0, ns, _lib.ptr(rp),
                                           _lib.ptr(col), _lib.ptr(val), _lib.ptr(cost),
                                           _lib.stream_ptr()), "ipi_gen_locality")
    return rp, col[:rows * K], val[:rows * K], cost[:rows].reshape(ns, m)


def pendulum(N: int, n_actions: int = 21, state0: int = 0, n_states: int | None = None):
    _lib.require_cuda()
    ns = N * N - state0 if n_states is None else n_states
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = ns * n_actions
    rp, col, val, cost = _alloc(rows, rows * 4, dev)
    _lib.check(_lib.lib().ipi_gen_pendulum(N, n_actions, state0, ns, _lib.ptr(rp), _lib.ptr(col),
                                           _lib.ptr(val), _lib.ptr(cost), _lib.stream_ptr()),
               "ipi_gen_pendulum")
    return rp, col[:rows * 4], val[:rows * 4], cost[:rows].reshape(ns, n_actions)


def sis(population: int):
    """Two passes: row lengths, host-free scan (torch.cumsum), fill."""
    _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    n, m = population + 1, 5
    rows = n * m
    rp = torch.zeros(rows + 1, dtype=torch.int64, device=dev)
    L = _lib.lib()
    _lib.check(L.ipi_gen_sis(population, 1, _lib.ptr(rp), None, None, None, _lib.stream_ptr()),
               "ipi_gen_sis")
    rp[1:] = torch.cumsum(rp[1:], 0)
    nnz = int(rp[-1])
    col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    cost = torch.empty(rows, dtype=torch.float64, device=dev)
    _lib.check(L.ipi_gen_sis(population, 2, _lib.ptr(rp), _lib.ptr(col), _lib.ptr(val),
                             _lib.ptr(cost), _lib.stream_ptr()), "ipi_gen_sis")
    return rp, col[:nnz], val[:nnz], cost.reshape(n, m)


def build_arrays(cfg: int | ConfigSpec, *, n: int | None = None, grid: int | None = None,
                 population: int | None = None, seed: int = 0, state0: int = 0,
                 n_states: int | None = None):
    """(row_ptr, col, val, cost, spec, n_total) on the device for a (scaled) config."""
    spec = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if spec.kind == "locality":
        nn = n or spec.n
        return (*locality(nn, spec.m, spec.K, spec.window, seed, state0, n_states), spec, nn)
    if spec.kind == "pendulum":
        N = grid or spec.grid
        return (*pendulum(N, spec.m, state0, n_states), spec, N * N)
    if spec.kind == "sis":
        N = population or spec.population
        return (*sis(N), spec, N + 1)
    if spec.kind == "dirichlet":
        from .generators import random_dirichlet
        nn = n or spec.n
        rp, col, val, cost = random_dirichlet(nn, spec.m, spec.K, seed)
        dev = torch.device("cuda", torch.cuda.current_device())
        return (torch.as_tensor(rp, device=dev), torch.as_tensor(col, device=dev),
                torch.as_tensor(val, device=dev), torch.as_tensor(cost, device=dev), spec, nn)
    raise ValueError(spec.kind)


def build_instance(cfg: int | ConfigSpec, **kw) -> tuple[MdpInstance, ConfigSpec]:
    rp, col, val, cost, spec, n = build_arrays(cfg, **kw)
    m = spec.m
    csr = CsrMatrix(n * m, n, rp, col, val)
    return MdpInstance(n=n, m=m, gamma=spec.gamma, stage_cost=cost, transitions=csr,
                       mode=Mode.MIN), spec
