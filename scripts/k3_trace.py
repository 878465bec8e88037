"""Per-CTA timeline of one K3 (planned policy operator) launch on C2's P_pi
(diagnostics: ipi_op_trace).  Prints the event time, the in-kernel span, CTA
start / duration / end spreads, to split K3's fixed cost into launch, ramp,
imbalance and tail.

    python scripts/k3_trace.py [--shape W:S:waves]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import _lib, devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.sparse import DeviceOperator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="11:3:1;12:3:3;12:3:6")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    mdp, spec = devgen.build_instance(2)
    v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
    pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
    P = ipi.gather_policy_matrix(mdp, pi.long())
    n = mdp.n
    del mdp
    torch.cuda.empty_cache()
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    for sh in a.shapes.split(";"):
        w, s, q = sh.split(":")
        os.environ.update(IPI_K3_WARPS=w, IPI_K3_STAGES=s, IPI_K3_WAVES=q)
        op = DeviceOperator(P.row_ptr, P.col_idx, P.values, n, n, 0, spec.gamma)
        nb = op.plan()["blocks"]
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        for _ in range(5):
            op.apply(x, out=y)
        torch.cuda.synchronize()
        recs = []
        for rep in range(5):
            _lib.check(L.ipi_op_trace(op._h, 1, None, 0))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.apply(x, out=y)
            e1.record()
            torch.cuda.synchronize()
            buf = np.zeros(3 * nb, dtype=np.uint64)
            _lib.check(L.ipi_op_trace(op._h, 0, buf.ctypes.data_as(C.c_void_p), buf.size))
            tr = buf.reshape(nb, 3).astype(np.int64)
            t0, t1 = tr[:, 1], tr[:, 2]
            base = t0.min()
            dur = (t1 - t0) / 1e3
            recs.append({"event_us": e0.elapsed_time(e1) * 1e3, "span_us": (t1.max() - base) / 1e3,
                         "start_spread_us": (t0.max() - base) / 1e3,
                         "end_spread_us": (t1.max() - t1.min()) / 1e3,
                         "cta_us_min": dur.min(), "cta_us_median": float(np.median(dur)), "cta_us_max": dur.max()})
        if os.environ.get("K3_TRACE_DETAIL"):
            # last repetition: per-CTA duration by block index and by SM id
            sm = tr[:, 0]
            order = np.argsort(dur)
            print("slowest 12 (block, sm, us):", [(int(b), int(sm[b]), round(float(dur[b]), 1)) for b in order[-12:]])
            print("fastest 12 (block, sm, us):", [(int(b), int(sm[b]), round(float(dur[b]), 1)) for b in order[:12]])
            print("by block decile (mean us):", [round(float(dur[k * nb // 10:(k + 1) * nb // 10].mean()), 1) for k in range(10)])
            prev = getattr(main, "_prev", None)
            if prev is not None and len(prev) == len(dur):
                print("corr with previous shape's per-block durations:", round(float(np.corrcoef(prev, dur)[0, 1]), 3))
            main._prev = dur.copy()
            main._runs = getattr(main, "_runs", []) + [dur.copy()]
        med = {k: float(np.median([r[k] for r in recs])) for k in recs[0]}
        print(json.dumps({"shape": sh, "blocks": nb, **{k: round(v_, 2) for k, v_ in med.items()}}), flush=True)
        del op


if __name__ == "__main__":
    main()
