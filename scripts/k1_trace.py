"""Per-CTA timeline of the K1 uniform-ring kernel on C2 (diagnostics).

    IPI_URING_WARPS=12 IPI_URING_STAGES=3 IPI_URING_WAVES=4 python scripts/k1_trace.py

Records (smid, start, end) per CTA with %globaltimer (ipi_mdp_k1_trace) for one
launch and prints the span, CTA-duration spread, per-SM busy time and the
slowest SMs — to tell a load-imbalanced tail from uniformly slow streaming.
"""

from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import _lib, devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402


def main():
    torch.cuda.set_device(0)
    mdp, spec = devgen.build_instance(2)
    plan = mdp.plan()
    v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        greedy_device(mdp, v, ipi.Mode.MIN)
    torch.cuda.synchronize()
    L = _lib.lib()
    h = mdp.handle()
    nb = plan["k1_blocks"]
    out = {"plan": plan}
    for rep in range(2):
        _lib.check(L.ipi_mdp_k1_trace(h, 1, None, 0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        greedy_device(mdp, v, ipi.Mode.MIN)
        e1.record()
        torch.cuda.synchronize()
        buf = np.zeros(3 * nb, dtype=np.uint64)
        _lib.check(L.ipi_mdp_k1_trace(h, 0, buf.ctypes.data_as(C.c_void_p), buf.size))
        tr = buf.reshape(nb, 3).astype(np.int64)
        sm, t0, t1 = tr[:, 0], tr[:, 1], tr[:, 2]
        base = t0.min()
        dur = (t1 - t0) / 1e3
        span = (t1.max() - base) / 1e3
        busy = np.zeros(sm.max() + 1)
        last = np.zeros(sm.max() + 1)
        cnt = np.zeros(sm.max() + 1, dtype=int)
        for s_, d, e in zip(sm, dur, (t1 - base) / 1e3):
            busy[s_] += d
            last[s_] = max(last[s_], e)
            cnt[s_] += 1
        used = cnt > 0
        first_start = np.sort((t0 - base) / 1e3)
        rec = {"event_ms": e0.elapsed_time(e1), "span_us": span,
               "cta_us": {"min": dur.min(), "median": float(np.median(dur)), "max": dur.max(),
                          "p10": float(np.percentile(dur, 10)), "p90": float(np.percentile(dur, 90))},
               "sm_busy_us": {"min": busy[used].min(), "median": float(np.median(busy[used])),
                              "max": busy[used].max()},
               "sm_last_end_us": {"min": last[used].min(), "median": float(np.median(last[used])),
                                  "max": last[used].max()},
               "ctas_per_sm": {"min": int(cnt[used].min()), "max": int(cnt[used].max())},
               "start_first_wave_us": {"p50": float(first_start[len(first_start) // (2 * max(1, nb // 148))]),
                                       "max_first148": float(first_start[min(147, nb - 1)])},
               "slowest_sms": [int(x) for x in np.argsort(-busy)[:8]],
               "fastest_sms": [int(x) for x in np.argsort(busy)[:8] if used[x]],
               "dur_by_block_decile": [float(np.mean(c)) for c in np.array_split(dur, 10)]}
        # per-SM mean CTA duration split by smid halves (die split hypothesis)
        half = (sm.max() + 1) // 2
        rec["mean_cta_us_smid_lo_hi"] = [float(dur[sm < half].mean()), float(dur[sm >= half].mean())]
        out[f"rep{rep}"] = rec
    print(json.dumps(out))


if __name__ == "__main__":
    main()
