"""Small driver for ncu: build one BASELINE config on the device and run the
hot kernels a few times (K1 Bellman; optionally one iPI solve for the inner
persistent kernel).

    python scripts/prof_k1.py --config 2 [--reps 3] [--solve] [--scale 1]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--max-outer", type=int, default=5)
    ap.add_argument("--ksp-max-it", type=int, default=None)
    ap.add_argument("--ksp", default="gmres")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    kw = {}
    from paper_2507_22538_b200.generators import CONFIGS
    spec = CONFIGS[a.config]
    if spec.kind in ("locality", "dirichlet"):
        kw["n"] = spec.n // a.scale
    if spec.kind == "pendulum" and a.grid:
        kw["grid"] = a.grid
    t0 = time.perf_counter()
    mdp, spec = devgen.build_instance(a.config, **kw)
    torch.cuda.synchronize()
    print(f"built {spec.name} n={mdp.n} m={mdp.m} nnz={mdp.transitions.nnz} in "
          f"{time.perf_counter() - t0:.2f}s plan={mdp.plan()}", flush=True)
    v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
    from paper_2507_22538_b200.bellman import greedy_device
    for _ in range(a.reps):
        greedy_device(mdp, v, ipi.Mode.MIN, with_residual=True)
    torch.cuda.synchronize()
    if a.solve:
        kw = {"ksp_max_it": a.ksp_max_it} if a.ksp_max_it else {}
        res = ipi.solve(mdp, ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol, max_outer=a.max_outer,
                                              inner=ipi.InnerSolver(a.ksp), **kw))
        print(f"solve: {res.status.value} outer={res.outer_iterations} "
              f"inner={res.inner_iterations_total} t={res.wall_time:.3f}s "
              f"greedy={res.time_greedy:.3f} asm={res.time_assembly:.3f} inner={res.time_inner:.3f}")
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
