"""Phase timeline of the persistent inner kernel (CTA 0's %globaltimer marks,
ipi_k4_trace): per-step durations of each phase, medians over the solve.

    python scripts/k4_trace.py [--config 2] [--its 60] [--kind gmres|richardson]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import _lib, devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--its", type=int, default=60)
    ap.add_argument("--kind", default="gmres")
    ap.add_argument("--ortho", default="auto")
    ap.add_argument("--stepped", action="store_true")
    ap.add_argument("--generic", action="store_true", help="1024-thread CGS2 kernel marks (C4)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    mdp, spec = devgen.build_instance(a.config)
    pi, _, _ = greedy_device(mdp, torch.zeros(mdp.n, dtype=torch.float64, device="cuda"), ipi.Mode.MIN)
    p = ipi.gather_policy_matrix(mdp, pi.long())
    b = mdp.stage_cost[torch.arange(mdp.n, device="cuda"), pi.long()].contiguous()
    L = _lib.lib()

    def run():
        x = torch.zeros(mdp.n, dtype=torch.float64, device="cuda")
        rep = _lib.InnerReport()
        _lib.check(L.ipi_inner_solve(_lib.ptr(p.row_ptr), _lib.ptr(p.col_idx), _lib.ptr(p.values),
                                     mdp.n, spec.gamma, _lib.ptr(b), _lib.ptr(x), 0.0, a.its,
                                     _lib.KSP[a.kind], 1.0, None, _lib.ORTHO[a.ortho],
                                     _lib.C.byref(rep),
                                     _lib.stream_ptr()))
        torch.cuda.synchronize()

    plan = mdp.plan()
    if plan["uniform_rows"] and plan["row_len_max"] == 64:
        # the standalone K3 operator on the same P_pi, for comparison
        from paper_2507_22538_b200.sparse import DeviceOperator
        op = DeviceOperator(p.row_ptr, p.col_idx, p.values, mdp.n, mdp.n, 0, spec.gamma)
        xk = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
        yk = torch.empty_like(xk)
        for _ in range(3):
            op.apply(xk, out=yk)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            op.apply(xk, out=yk)
        e1.record()
        torch.cuda.synchronize()
        print(f"K3 apply: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch, plan {op.plan()}")
        ms = _lib.C.c_float()
        yr = torch.empty_like(xk)
        _lib.check(L.ipi_k4_ring_apply_test(_lib.ptr(p.col_idx), _lib.ptr(p.values), mdp.n, spec.gamma,
                                            _lib.ptr(xk), _lib.ptr(yr), 20, _lib.C.byref(ms),
                                            _lib.stream_ptr()))
        print(f"ring_rows as a plain kernel: {ms.value / 20 * 1e3:.1f} us per launch; "
              f"bitwise equal to K3: {bool(torch.equal(yr, yk))}")
    run()
    _lib.check(L.ipi_k4_trace(1, None, 0))
    run()
    buf = np.zeros(8192, dtype=np.uint64)
    _lib.check(L.ipi_k4_trace(0, buf.ctypes.data, 8192))
    k = int(buf[0])
    t0 = buf[1:k + 1].astype(np.int64)
    if a.generic:
        # 1024-thread CGS2 kernel marks: start, spmv(+barrier), dots, update, reorth, end
        names = ["spmv+barrier", "cgs_dots+allreduce", "cgs_update+allreduce", "reorth (if any)",
                 "givens+write+barrier"]
        t = t0[3:]
        m6 = (len(t) // 6) * 6
        t6 = t[:m6].reshape(-1, 6)
        d = np.diff(t6, axis=1) / 1e3
        print(f"{spec.name} gmres/cgs2 (1024-thread kernel): {len(d)} steps; reorth in "
              f"{int((d[:, 3] > 0.5).sum())}")
        for c, nm in enumerate(names):
            print(f"  {nm:28s} median {np.median(d[:, c]):8.2f} us  p90 {np.percentile(d[:, c], 90):8.2f}")
        print(f"  step total median {np.median(d.sum(1)):.2f} us")
        return
    if a.stepped:
        # step_ortho marks: start, MGS done, end (3 per step); gaps = K3 + launches
        t3 = t0[: (len(t0) // 3) * 3].reshape(-1, 3)
        mgs = (t3[:, 1] - t3[:, 0]) / 1e3
        giv = (t3[:, 2] - t3[:, 1]) / 1e3
        gap = (t3[1:, 0] - t3[:-1, 2]) / 1e3
        print(f"stepped: {len(t3)} steps; MGS median {np.median(mgs):.1f} us (p10 {np.percentile(mgs, 10):.1f}"
              f" p90 {np.percentile(mgs, 90):.1f}); Givens+write {np.median(giv):.1f} us; "
              f"ortho end -> next ortho start (K3 + launch gaps) median {np.median(gap):.1f} us")
        per_j = {}
        for i, v in enumerate(mgs):
            per_j.setdefault(i % 30, []).append(v)
        print("  MGS us by j:", {j: round(float(np.median(v)), 1) for j, v in sorted(per_j.items())})
        return
    print(f"  initial residual pass (first SpMV of the launch): {(t0[1] - t0[0]) / 1e3:.1f} us, "
          f"its all-reduce {(t0[2] - t0[1]) / 1e3:.1f} us")
    t = t0[3:]
    if a.kind == "gmres":
        # marks: step start, spmv done, dots reduced, update reduced, V_{j+1} written + barrier
        names = ["spmv", "cgs_dots+allreduce", "cgs_update+allreduce", "givens+write+barrier",
                 "(gap)"]
    else:
        names = ["spmv", "allreduce", "x_update+barrier"]
    nph = len(names)
    dd = np.diff(t)
    m = len(dd) // nph
    d = dd[: m * nph].reshape(m, nph) / 1e3  # us
    print(f"{spec.name} {a.kind}: {len(d)} steps, marks {k}")
    for c, nm in enumerate(names[:d.shape[1]]):
        print(f"  {nm:28s} median {np.median(d[:, c]):8.2f} us   p10 {np.percentile(d[:, c], 10):8.2f}"
              f"   p90 {np.percentile(d[:, c], 90):8.2f}")
    print(f"  {'step total':28s} median {np.median(d.sum(1)):8.2f} us")


if __name__ == "__main__":
    main()
