"""C5 per-rank proxy on ONE GPU: build rank r's row block of the 16.7M-state C5
instance (make_partition(n, R)), run K1 with a full-length V, time it.  The
per-GPU K1 time at R ranks plus the V all-gather bound the R-GPU step; this
is a single-GPU proxy, not a multi-GPU measurement.

    python scripts/c5_shard_proxy.py --world 8 [--rank 0]
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
from paper_2507_22538_b200.generators import CONFIGS  # noqa: E402
from paper_2507_22538_b200.model import make_partition  # noqa: E402
from paper_2507_22538_b200.parallel import MdpShard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    spec = CONFIGS[5]
    lo, hi = make_partition(spec.n, a.world).block(a.rank)
    t0 = time.perf_counter()
    rp, col, val, cost = devgen.locality(spec.n, spec.m, spec.K, spec.window, 0, lo, hi - lo)
    csr = ipi.CsrMatrix((hi - lo) * spec.m, spec.n, rp, col, val)
    shard = MdpShard(spec.n, spec.m, spec.gamma, lo, cost, csr)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    v = torch.rand(spec.n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        shard.bellman(v)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        shard.bellman(v)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    nnz = csr.nnz
    rows = (hi - lo) * spec.m
    b = nnz * 12 + rows * 8 + spec.n * 8 + (hi - lo) * 12
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    print(json.dumps({"config": spec.name, "world": a.world, "rank": a.rank, "states": hi - lo,
                      "nnz": nnz, "build_s": t_build, "k1_ms": t * 1e3,
                      "backups_per_s_rank": rows / t, "k1_gbs": b / t / 1e9, "k1_frac": b / t / 1e9 / peak,
                      "plan": shard.plan()}))


if __name__ == "__main__":
    main()
