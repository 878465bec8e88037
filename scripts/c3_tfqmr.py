"""C3 (pendulum 2048^2, 21 actions, gamma 0.9999) with the TFQMR inner solver —
the paper's choice for the pendulum; GMRES(30) as specified
stagnates in the reference itself.  Labelled extra, not the
BASELINE spec.

    python scripts/c3_tfqmr.py [--grid 2048] [--kind tfqmr] [--max-outer 1000]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=2048)
    ap.add_argument("--kind", default="tfqmr")
    ap.add_argument("--max-outer", type=int, default=1000)
    ap.add_argument("--max-inner", type=int, default=1000)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    mdp, spec = devgen.build_instance(3, grid=a.grid)
    opts = ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol, max_outer=a.max_outer,
                            max_inner=a.max_inner, inner=ipi.InnerSolver.from_name(a.kind))
    t0 = time.perf_counter()
    res = ipi.solve(mdp, opts)
    dt = time.perf_counter() - t0
    _, tv, _ = greedy_device(mdp, res.values_device, ipi.Mode.MIN)
    cert = float((res.values_device - tv).abs().max())
    print(json.dumps({"config": spec.name, "grid": a.grid, "kind": a.kind, "status": res.status.value,
                      "outer": res.outer_iterations, "inner": res.inner_iterations_total,
                      "wall_s": dt, "time_inner_s": res.time_inner,
                      "final_residual": res.residual_history[-1], "certificate_residual": cert,
                      "v_min": float(res.values_device.min()), "v_max": float(res.values_device.max()),
                      "history_head": res.residual_history[:5],
                      "history_tail": res.residual_history[-5:]}))


if __name__ == "__main__":
    main()
