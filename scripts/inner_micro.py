"""Micro-benchmark of the persistent inner solver: ms per GMRES / Richardson
iteration on the greedy policy of V = 0 for the given configs (fixed
iteration counts: target 0)."""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.generators import CONFIGS, random_dirichlet  # noqa: E402
from paper_2507_22538_b200 import _lib  # noqa: E402


def build(cfg):
    spec = CONFIGS[cfg]
    if spec.kind == "dirichlet":
        rp, col, val, cost = random_dirichlet(spec.n, spec.m, spec.K, seed=0)
        return ipi.MdpInstance(spec.n, spec.m, spec.gamma, cost,
                               ipi.CsrMatrix(spec.n * spec.m, spec.n, rp, col, val)), spec
    return devgen.build_instance(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,4,2")
    ap.add_argument("--its", type=int, default=300)
    ap.add_argument("--ortho", default="cgs2,mgs")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for cfg in [int(c) for c in a.configs.split(",")]:
        mdp, spec = build(cfg)
        pi, _, _ = greedy_device(mdp, torch.zeros(mdp.n, dtype=torch.float64, device="cuda"),
                                 ipi.Mode.MIN)
        p = ipi.gather_policy_matrix(mdp, pi.long())
        b = mdp.stage_cost[torch.arange(mdp.n, device="cuda"), pi.long()].contiguous()
        plan = mdp.plan()
        kinds = [("gmres", o) for o in a.ortho.split(",")] + [("richardson", "cgs2")]
        for kind, ortho in kinds:
            res = {}
            for its in (a.its // 2, a.its):  # slope: excludes planning and launch
                for _ in range(2):
                    x = torch.zeros(mdp.n, dtype=torch.float64, device="cuda")
                    rep = _lib.InnerReport()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    rc = _lib.lib().ipi_inner_solve(_lib.ptr(p.row_ptr), _lib.ptr(p.col_idx),
                                                    _lib.ptr(p.values), mdp.n, spec.gamma, _lib.ptr(b),
                                                    _lib.ptr(x), 0.0, its, _lib.KSP[kind], 1.0, None,
                                                    _lib.ORTHO[ortho], _lib.C.byref(rep),
                                                    _lib.stream_ptr())
                    e1.record()
                    torch.cuda.synchronize()
                    _lib.check(rc)
                res[its] = (e0.elapsed_time(e1), rep.iterations)
            (t0, i0), (t1, i1) = res[a.its // 2], res[a.its]
            ms = (t1 - t0) / max(i1 - i0, 1)
            print(f"{spec.name} {kind}/{ortho}: {i1} its, {ms:.4f} ms/it (slope {i0}->{i1}), "
                  f"resid {rep.final_linear_residual_2norm:.3e} plan_halo={plan['halo']}", flush=True)
        del p, mdp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
