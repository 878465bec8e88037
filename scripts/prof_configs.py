"""Driver for ncu: one K1 (Bellman backup), one K2 (policy compaction) and one
K3 (policy-operator apply) launch per BASELINE config, to capture the kernel
choices the planner makes for C1 / C3 / C4 (C2's captures come from bench.py).

    ncu --set full -k regex:"k1_|k3_|spmv_kernel|copy_rows" \
        python scripts/prof_configs.py --configs 1,3,4

Autotuning is disabled (IPI_K1_AUTOTUNE=0, IPI_K3_AUTOTUNE=0) so each kernel
runs exactly once; C4's generic K1 uses the autotuned 8 CTAs/SM.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

os.environ.setdefault("IPI_K1_AUTOTUNE", "0")
os.environ.setdefault("IPI_K3_AUTOTUNE", "0")
os.environ.setdefault("IPI_K1_GEN_CTAS", "8")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.generators import CONFIGS, random_dirichlet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for cfg in [int(c) for c in a.configs.split(",")]:
        spec = CONFIGS[cfg]
        if spec.kind == "dirichlet":
            rp, col, val, cost = random_dirichlet(spec.n, spec.m, spec.K, seed=0)
            mdp = ipi.MdpInstance(spec.n, spec.m, spec.gamma, cost,
                                  ipi.CsrMatrix(spec.n * spec.m, spec.n, rp, col, val))
        else:
            mdp, spec = devgen.build_instance(cfg)
        v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
        pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN, with_residual=True)
        P = ipi.gather_policy_matrix(mdp, pi.long())
        op = ipi.PolicyOperator(P, spec.gamma)
        y = op.apply(v)
        torch.cuda.synchronize()
        print(spec.name, mdp.plan()["k1_variant"], op.device_operator().plan(), float(y.sum()),
              flush=True)
        del mdp, P, op
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
