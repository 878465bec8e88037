"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/frontend/src \
        python tests/golden/make_golden.py

The reference package ``mdpsolve`` (``/root/reference/pkg/src``) is imported
read-only; ``/root/reference`` does not exist on the GPU box, so its outputs
are frozen here as ``tests/golden/*.npz`` and committed together with this
script.  Each fixture stores the instance arrays (inputs) and what the
reference returned for them:

* ``solve`` for the listed inner solvers (values, policy, residual_history,
  status, outer/inner counts)                      driver.py:109-209
* ``greedy_policy`` at a seeded V                  bellman.py:44-68
* ``spmv`` at a seeded x                           sparse.py:189-215
* ``gather_policy_matrix/cost`` for that greedy π  sparse.py:243-269
* ``PolicyOperator.apply``                         sparse.py:294-295
* ``inner_solve`` (gmres, richardson) from V0      inner.py:163-213
* ``policy_cost_exact`` of the final policy when n <= 4096 (dense oracle)

Fixture instances: the reference's own test fixtures (FIXTURE_INSTANCE =
gen_random(20, 4, 6, 0.9, seed 123) from test_driver.py:36; 33x33 maze from
test_driver.py:133-139; rng(20240817) dense 5x3 from conftest.py:47-53,
97-99; the 1-state toy test_driver.py:40-45; SIS / pendulum small cases from
test_acceptance.py:288-290) plus scaled-down instances of the five
BASELINE configs built by ``paper_2507_22538_b200.generators``.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
for p in ("/root/reference/pkg/src", "/root/reference/pkg/frontend/src"):
    if p not in sys.path:
        sys.path.insert(0, p)

import mdpsolve as ref  # noqa: E402  (the reference itself)
from mdpsolve.problems import (  # noqa: E402
    MazeParams, PendulumParams, RandomParams, SisParams,
)

from paper_2507_22538_b200 import generators as gen  # noqa: E402


def _instance(row_ptr, col, val, cost, gamma, mode="min"):
    cost = np.asarray(cost, dtype=np.float64)
    n, m = cost.shape
    csr = ref.CsrMatrix(n * m, n, row_ptr, np.asarray(col, dtype=np.int64), val)
    return ref.MdpInstance(n=n, m=m, gamma=gamma, stage_cost=cost, transitions=csr,
                           mode=ref.Mode.MAX if mode == "max" else ref.Mode.MIN)


def _arrays(inst):
    t = inst.transitions
    return (np.asarray(t.row_ptr, dtype=np.int64), np.asarray(t.col_idx, dtype=np.int32),
            np.asarray(t.values, dtype=np.float64), np.asarray(inst.stage_cost, dtype=np.float64))


def _digest(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def record(name, inst, *, kinds=("gmres",), opts=None, seed=7, exact=True, tol=1e-8,
           jacobi_kinds=()):
    opts = dict(opts or {})
    rp, col, val, cost = _arrays(inst)
    n, m = cost.shape
    out: dict[str, np.ndarray] = dict(row_ptr=rp, col=col, val=val, cost=cost,
                                      gamma=np.float64(inst.gamma),
                                      maximize=np.bool_(inst.mode is ref.Mode.MAX))
    meta = {"name": name, "n": n, "m": m, "nnz": int(rp[-1]), "gamma": inst.gamma,
            "mode": inst.mode.value, "digest": _digest(rp, col, val, cost), "solves": {}}
    rng = np.random.default_rng(seed)
    # greedy / spmv / gather / apply / inner at a seeded V
    v = rng.random(n) * 10.0
    x = rng.standard_normal(n)
    g = ref.greedy_policy(inst, v)
    out["greedy_v"] = v
    out["greedy_policy"] = g.policy.astype(np.int64)
    out["greedy_applied"] = g.applied
    out["spmv_x"] = x
    out["spmv_y"] = ref.spmv(inst.transitions, x)
    p_pi = ref.gather_policy_matrix(inst, g.policy)
    out["gather_row_ptr"] = p_pi.row_ptr
    out["gather_col"] = p_pi.col_idx.astype(np.int32)
    out["gather_val"] = p_pi.values
    out["gather_cost"] = ref.gather_policy_cost(inst, g.policy)
    op = ref.PolicyOperator(p_pi, inst.gamma)
    out["apply_y"] = op.apply(x)
    for kind in ("gmres", "richardson", "tfqmr", "bicgstab"):
        target = 1e-3 * float(np.max(np.abs(v - g.applied)))
        theta, rep = ref.inner_solve(op, out["gather_cost"], v, target, 200,
                                     kind=ref.InnerSolver.from_name(kind))
        out[f"inner_{kind}_theta"] = theta
        out[f"inner_{kind}_target"] = np.float64(target)
        meta[f"inner_{kind}"] = {"iterations": rep.iterations,
                                 "final": rep.final_linear_residual_2norm,
                                 "converged": rep.converged, "eff": rep.target_2norm,
                                 "breakdown": rep.breakdown}
    for kind in kinds:
        so = ref.SolveOptions(inner=ref.InnerSolver.from_name(kind), tol=tol, **opts)
        res = ref.solve(inst, so)
        out[f"solve_{kind}_values"] = res.values
        out[f"solve_{kind}_policy"] = res.policy.astype(np.int64)
        out[f"solve_{kind}_history"] = np.asarray(res.residual_history)
        meta["solves"][kind] = {"status": res.status.value, "outer": res.outer_iterations,
                                "inner": res.inner_iterations_total,
                                "options": {k: (v if not hasattr(v, "value") else v.value)
                                            for k, v in opts.items()}, "tol": tol}
        if exact and n <= 4096 and res.status is ref.SolveStatus.CONVERGED:
            out[f"solve_{kind}_exact"] = ref.policy_cost_exact(inst, res.policy)
    # the same solves with the Jacobi preconditioner (inner.py:115-118)
    for kind in jacobi_kinds:
        so = ref.SolveOptions(inner=ref.InnerSolver.from_name(kind), tol=tol,
                              pc=ref.Preconditioner.JACOBI, **opts)
        res = ref.solve(inst, so)
        key = f"{kind}_jacobi"
        out[f"solve_{key}_values"] = res.values
        out[f"solve_{key}_policy"] = res.policy.astype(np.int64)
        out[f"solve_{key}_history"] = np.asarray(res.residual_history)
        meta["solves"][key] = {"status": res.status.value, "outer": res.outer_iterations,
                               "inner": res.inner_iterations_total, "options": {"pc": "jacobi"},
                               "tol": tol}
    np.savez_compressed(HERE / f"{name}.npz", **out)
    return meta


def brute_force_optimum(inst):
    """Componentwise best value over all m^n policies (conftest.py:82-94)."""
    best = None
    for pol in itertools.product(range(inst.m), repeat=inst.n):
        vv = ref.policy_cost_exact(inst, np.array(pol))
        best = vv if best is None else np.minimum(best, vv)
    return best


def main():
    metas = []
    # --- reference fixtures -------------------------------------------------
    fixture = ref.gen_random(RandomParams(n=20, m=4, nnz_per_row=6, gamma=0.9, seed=123))
    metas.append(record("ref_fixture_random", fixture,
                        kinds=("gmres", "richardson", "tfqmr", "bicgstab"),
                        jacobi_kinds=("gmres", "richardson", "tfqmr", "bicgstab")))
    rp, col, val, cost = _arrays(fixture)
    metas.append(record("ref_fixture_random_max", _instance(rp, col, val, cost, 0.9, "max"),
                        kinds=("gmres", "richardson")))
    metas.append(record("ref_maze33", ref.gen_maze(MazeParams(height=33, width=33)),
                        kinds=("gmres", "tfqmr"), jacobi_kinds=("gmres",)))
    rng = np.random.default_rng(20240817)
    p = rng.random((5, 3, 5))
    p /= p.sum(axis=2, keepdims=True)
    gcost = rng.random((5, 3))
    rows = p.reshape(15, 5)
    dense = _instance(np.arange(16, dtype=np.int64) * 5, np.tile(np.arange(5), 15),
                      rows.ravel(), gcost, 0.9)
    metas.append(record("ref_dense5x3", dense, kinds=("gmres", "richardson", "tfqmr", "bicgstab"),
                        tol=1e-9))
    np.save(HERE / "ref_dense5x3_optimum.npy", brute_force_optimum(dense))
    metas.append(record("ref_toy", _instance(np.array([0, 1]), np.array([0]), np.array([1.0]),
                                             np.array([[1.0]]), 0.5),
                        kinds=("gmres", "richardson")))
    zc = _instance(np.arange(16, dtype=np.int64) * 5, np.tile(np.arange(5), 15), rows.ravel(),
                   np.zeros((5, 3)), 0.9)
    metas.append(record("ref_zero_cost", zc, kinds=("gmres",)))
    metas.append(record("ref_sis12", ref.gen_sis(SisParams(population=12)),
                        kinds=("gmres", "tfqmr", "bicgstab")))
    metas.append(record("ref_pendulum9", ref.gen_pendulum(PendulumParams(grid_points=9,
                                                                         torque_points=5)),
                        kinds=("gmres", "tfqmr")))
    # discount sensitivity (test_acceptance.py:168-183), small n
    for gam in (0.9, 0.9999):
        inst = ref.gen_random(RandomParams(n=200, m=8, nnz_per_row=10, gamma=gam, seed=5))
        metas.append(record(f"ref_random200_g{str(gam).replace('.', 'p')}", inst,
                            kinds=("gmres", "richardson")))
    # --- scaled BASELINE-config instances (our generators, reference solve) --
    c1 = gen.random_dirichlet(100, 10, 25, seed=0)
    metas.append(record("cfg1_dirichlet_n100", _instance(*c1, 0.99),
                        kinds=("gmres", "richardson", "tfqmr", "bicgstab"),
                        jacobi_kinds=("gmres", "richardson")))
    c2 = gen.random_locality_host(256, 8, 16, 16, seed=0)
    metas.append(record("cfg2_locality_n256", _instance(*c2, 0.999), kinds=("gmres",)))
    c3 = gen.pendulum_host(12, 21)
    metas.append(record("cfg3_pendulum_g12", _instance(*c3, 0.9999),
                        kinds=("gmres", "tfqmr")))
    c4 = gen.sis_host(60)
    metas.append(record("cfg4_sis_n60", _instance(*c4, 0.9999), kinds=("gmres", "tfqmr", "bicgstab"),
                        jacobi_kinds=("gmres",)))
    c2max = _instance(*c2, 0.999, "max")
    metas.append(record("cfg2_locality_n256_max", c2max, kinds=("gmres",)))
    (HERE / "golden_index.json").write_text(json.dumps(metas, indent=1) + "\n")
    print(json.dumps([{k: m_[k] for k in ("name", "n", "m", "nnz", "solves")} for m_ in metas],
                     indent=1))


if __name__ == "__main__":
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    main()
