"""K3 (policy operator apply) throughput on the full-size BASELINE policy
matrices: P_pi of the greedy policy of a random V for C2 / C3 / C4, timed with
CUDA events around ipi_op_apply (no host sync inside), L2 flushed (256 MB
write) before every rep.

    python scripts/k3_bench.py [--configs 2,3,4] [--reps 30]

Bytes per apply: nnz_pi*12 + 8n [x, compulsory] + 8n [y]
(+ 8n [b] for the residual form) (+ 8(n+1) row pointers for the generic
kernel only).  Prints one JSON object per (config, kernel, epilogue).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.sparse import DeviceOperator  # noqa: E402


def peak():
    p = REPO / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def time_op(op, x, b, reps):
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    y = torch.empty(op.n_local, dtype=torch.float64, device="cuda")
    for _ in range(3):
        op.apply(x, b, out=y)
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply(x, b, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--shapes", default="", help="warps:stages:waves[:l2_prefetch_steps[:halo_cap[:interleave]]] list to force, ';'-separated")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for cfg in [int(c) for c in a.configs.split(",")]:
        mdp, spec = devgen.build_instance(cfg)
        v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
        pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
        P = ipi.gather_policy_matrix(mdp, pi.long())
        n = mdp.n
        del mdp
        torch.cuda.empty_cache()
        x = torch.rand(n, dtype=torch.float64, device="cuda")
        b = torch.rand(n, dtype=torch.float64, device="cuda")
        nnz = P.values.numel()
        variants = [("planned", {})]
        for sh in [s for s in a.shapes.split(";") if s]:
            parts = sh.split(":")
            env = {"IPI_K3_WARPS": parts[0], "IPI_K3_STAGES": parts[1], "IPI_K3_WAVES": parts[2]}
            if len(parts) > 3:
                env["IPI_K3_PF"] = parts[3]
            if len(parts) > 4:
                env["IPI_K3_HALO"] = parts[4]
            if len(parts) > 5:
                env["IPI_K3_INTERLEAVE"] = parts[5]
            variants.append((f"shape{sh}", env))
        variants.append(("generic", {"IPI_K3_RING": "0"}))
        for name, env in variants:
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            op = DeviceOperator(P.row_ptr, P.col_idx, P.values, n, n, 0, spec.gamma)
            for k, val in old.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val
            plan = op.plan()
            for epi, bb in (("apply", None), ("residual", b)):
                t, tmin = time_op(op, x, bb, a.reps)
                byts = nnz * 12 + 16 * n + (8 * n if bb is not None else 0)
                if plan["variant"] == 0:
                    byts += 8 * (n + 1)
                print(json.dumps({"config": spec.name, "kernel": name, "epilogue": epi, "plan": plan,
                                  "n": n, "nnz_pi": nnz, "ms": t * 1e3, "ms_min": tmin * 1e3,
                                  "bytes": byts, "gbs": byts / t / 1e9,
                                  "frac": byts / t / 1e9 / peak(), "peak_gbs": peak()}), flush=True)
            del op
        del P
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
