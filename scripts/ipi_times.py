"""iPI time-to-tolerance per config and GMRES orthogonalisation (A/B).

    python scripts/ipi_times.py [--configs 2,4] [--ortho cgs2,mgs] [--reps 2]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.generators import CONFIGS, random_dirichlet  # noqa: E402


def build(cfg):
    spec = CONFIGS[cfg]
    if spec.kind == "dirichlet":
        rp, col, val, cost = random_dirichlet(spec.n, spec.m, spec.K, seed=0)
        return ipi.MdpInstance(spec.n, spec.m, spec.gamma, cost,
                               ipi.CsrMatrix(spec.n * spec.m, spec.n, rp, col, val)), spec
    return devgen.build_instance(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,4")
    ap.add_argument("--ortho", default="cgs2,mgs")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--kind", default="gmres")
    ap.add_argument("--max-outer", type=int, default=1000)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for cfg in [int(c) for c in a.configs.split(",")]:
        mdp, spec = build(cfg)
        for ortho in a.ortho.split(","):
            opts = ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol, gmres_ortho=ortho,
                                    inner=ipi.InnerSolver.from_name(a.kind),
                                    max_outer=a.max_outer)
            ipi.solve(mdp, opts)  # warm-up
            for _ in range(a.reps):
                r = ipi.solve(mdp, opts)
                print(json.dumps({"config": spec.name, "ortho": ortho, "kind": a.kind,
                                  "status": r.status.value, "outer": r.outer_iterations,
                                  "inner": r.inner_iterations_total, "wall_s": r.wall_time,
                                  "greedy_s": r.time_greedy, "assembly_s": r.time_assembly,
                                  "inner_s": r.time_inner,
                                  "ms_per_inner_it": 1e3 * r.time_inner / max(1, r.inner_iterations_total),
                                  "final": r.residual_history[-1]}), flush=True)
        del mdp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
