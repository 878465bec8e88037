"""Per-config report: K1 Bellman throughput + roofline, inner SpMV roofline,
iPI time-to-tolerance on the GPU, and the CPU oracle beside it.

    python scripts/config_sweep.py [--configs 1,2,3,4] [--cpu] [--c3-outer 3]

Writes one JSON object per config to stdout (and gpurun_out/sweep.json).
C3 (pendulum, GMRES(30)) stalls in the reference itself: it is
run with a capped outer loop and its status is reported as-is.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.generators import CONFIGS, random_dirichlet  # noqa: E402


def peak():
    p = REPO / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def k1_bytes(n, m, nnz, uniform):
    """row pointers count only for variable-length rows."""
    rows = n * m
    return nnz * 12 + rows * 8 + n * 8 + n * 12 + (0 if uniform else (rows + 1) * 8)


def time_k1(mdp, reps=20):
    v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    for _ in range(3):
        greedy_device(mdp, v, ipi.Mode.MIN, with_residual=True)
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)  # 256 MB > L2: cold-L2 timing for the small configs
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        greedy_device(mdp, v, ipi.Mode.MIN, with_residual=True)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def time_apply(p_pi, gamma, reps=20):
    op = ipi.PolicyOperator(p_pi, gamma)
    x = torch.rand(p_pi.rows, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    for _ in range(3):
        op.apply(x)
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op.apply(x)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts)), op.device_operator().plan()


def build(cfg):
    spec = CONFIGS[cfg]
    if spec.kind == "dirichlet":
        rp, col, val, cost = random_dirichlet(spec.n, spec.m, spec.K, seed=0)
        mdp = ipi.MdpInstance(spec.n, spec.m, spec.gamma, cost,
                              ipi.CsrMatrix(spec.n * spec.m, spec.n, rp, col, val))
        return mdp, spec, (rp, col, val, cost)
    mdp, spec = devgen.build_instance(cfg)
    return mdp, spec, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--cpu", action="store_true", help="also time the numpy oracle (C1, C4)")
    ap.add_argument("--c3-outer", type=int, default=3)
    ap.add_argument("--k1-only", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    out = []
    for cfg in [int(c) for c in a.configs.split(",")]:
        t0 = time.perf_counter()
        mdp, spec, host = build(cfg)
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t0
        plan = mdp.plan()
        nnz = plan["nnz"]
        t1 = time_k1(mdp)
        b1 = k1_bytes(mdp.n, mdp.m, nnz, bool(plan["uniform_rows"]))
        rec = {"config": spec.name, "n": mdp.n, "m": mdp.m, "nnz": nnz, "build_s": t_build,
               "plan": plan, "k1_ms": t1 * 1e3, "k1_bytes": b1, "k1_gbs": b1 / t1 / 1e9,
               "k1_frac": b1 / t1 / 1e9 / peak(), "backups_per_s": mdp.n * mdp.m / t1,
               "nnz_per_s": nnz / t1}
        if a.k1_only:
            print(json.dumps(rec), flush=True)
            out.append(rec)
            del mdp
            torch.cuda.empty_cache()
            continue
        # policy evaluation SpMV (K3) on the greedy policy of V = 0
        pi, _, _ = greedy_device(mdp, torch.zeros(mdp.n, dtype=torch.float64, device="cuda"),
                                 ipi.Mode.MIN)
        p_pi = ipi.gather_policy_matrix(mdp, pi.long())
        t3, k3_plan = time_apply(p_pi, spec.gamma)
        # x once + y; the generic kernel also reads the row pointers
        b3 = p_pi.nnz * 12 + mdp.n * 16 + ((mdp.n + 1) * 8 if k3_plan["variant"] == 0 else 0)
        rec.update({"k3_ms": t3 * 1e3, "k3_bytes": b3, "k3_gbs": b3 / t3 / 1e9, "k3_plan": k3_plan,
                    "k3_frac": b3 / t3 / 1e9 / peak(), "nnz_pi": p_pi.nnz})
        del p_pi
        opts = ipi.SolveOptions(alpha=spec.alpha, tol=spec.atol)
        if cfg == 3:
            opts.max_outer = a.c3_outer
        ipi.solve(mdp, opts)          # warm-up: lazy module loading of every kernel variant
        res = ipi.solve(mdp, opts)
        rec["gpu_solve"] = {"status": res.status.value, "outer": res.outer_iterations,
                            "inner": res.inner_iterations_total, "wall_s": res.wall_time,
                            "greedy_s": res.time_greedy, "assembly_s": res.time_assembly,
                            "inner_s": res.time_inner, "final_residual": res.residual_history[-1],
                            "max_outer": opts.max_outer}
        if res.inner_iterations_total:
            rec["gpu_solve"]["ms_per_inner_iteration"] = res.time_inner / res.inner_iterations_total * 1e3
        if a.cpu and cfg in (1, 4):
            from oracle import mdp_oracle as orc
            if host is None:
                rp, col, val = mdp.transitions.numpy()
                host = (rp, col, val, mdp.stage_cost.cpu().numpy())
            rp, col, val, cost = host
            v = np.zeros(mdp.n)
            tg = time.perf_counter()
            orc.greedy(rp, col, val, cost, spec.gamma, v)
            tg = time.perf_counter() - tg
            ts = time.perf_counter()
            ref = orc.solve(rp, col, val, cost, spec.gamma, tol=spec.atol, alpha=spec.alpha)
            ts = time.perf_counter() - ts
            rec["cpu_oracle"] = {"greedy_s": tg, "backups_per_s": mdp.n * mdp.m / tg,
                                 "solve_s": ts, "status": ref.status,
                                 "outer": ref.outer_iterations, "inner": ref.inner_iterations_total,
                                 "cores": 1, "kind": "port (numpy)",
                                 "v_rel_diff": float(np.max(np.abs(ref.values - res.values)) /
                                                     max(1.0, np.abs(ref.values).max()))}
        if a.cpu:
            # C/OpenMP restatement (bitwise equal to the reference's greedy_policy) on all
            # host threads: backup throughput for every config, full solve for C1/C2/C4
            from oracle import c_oracle as co
            if host is None:
                rp, col, val = mdp.transitions.numpy()
                host = (rp, col, val, mdp.stage_cost.cpu().numpy())
            rp, col, val, cost = host
            nt = os.cpu_count() or 1
            v = np.zeros(mdp.n)
            co.greedy(rp, col, val, cost, spec.gamma, v, nthreads=nt)
            tg = time.perf_counter()
            co.greedy(rp, col, val, cost, spec.gamma, v, nthreads=nt)
            tg = time.perf_counter() - tg
            rec["cpu_c_oracle"] = {"greedy_s": tg, "backups_per_s": mdp.n * mdp.m / tg, "cores": nt,
                                   "kind": "port (C/OpenMP)"}
            if cfg in (1, 2, 4):
                ts = time.perf_counter()
                ref = co.solve(rp, col, val, cost, spec.gamma, tol=spec.atol, alpha=spec.alpha,
                               nthreads=nt)
                ts = time.perf_counter() - ts
                rec["cpu_c_oracle"].update({
                    "solve_s": ts, "status": ref.status, "outer": ref.outer_iterations,
                    "inner": ref.inner_iterations_total,
                    "v_rel_diff": float(np.max(np.abs(ref.values - res.values)) /
                                        max(1.0, np.abs(ref.values).max()))})
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del mdp
        torch.cuda.empty_cache()
    os.makedirs(REPO / "gpurun_out", exist_ok=True)
    (REPO / "gpurun_out" / "sweep.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
