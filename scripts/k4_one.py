"""One persistent inner solve (fixed iteration count) on the greedy policy of
V = 0: the launch an ncu capture of the inner kernel targets.

    python scripts/k4_one.py [--config 2] [--its 10] [--kind richardson] [--ortho cgs2]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import _lib, devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--its", type=int, default=10)
    ap.add_argument("--kind", default="richardson")
    ap.add_argument("--ortho", default="cgs2")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    mdp, spec = devgen.build_instance(a.config)
    pi, _, _ = greedy_device(mdp, torch.zeros(mdp.n, dtype=torch.float64, device="cuda"), ipi.Mode.MIN)
    p = ipi.gather_policy_matrix(mdp, pi.long())
    b = mdp.stage_cost[torch.arange(mdp.n, device="cuda"), pi.long()].contiguous()
    x = torch.zeros(mdp.n, dtype=torch.float64, device="cuda")
    rep = _lib.InnerReport()
    _lib.check(_lib.lib().ipi_inner_solve(
        _lib.ptr(p.row_ptr), _lib.ptr(p.col_idx), _lib.ptr(p.values), mdp.n, spec.gamma,
        _lib.ptr(b), _lib.ptr(x), 0.0, a.its, _lib.KSP[a.kind], 1.0, None, _lib.ORTHO[a.ortho],
        _lib.C.byref(rep), _lib.stream_ptr()))
    torch.cuda.synchronize()
    print("its", rep.iterations, "resid", rep.final_linear_residual_2norm)


if __name__ == "__main__":
    main()
