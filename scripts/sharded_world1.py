"""One native sharded iPI solve (ipi_solve_sharded) at world 1 on a C5-shaped
instance, for an ncu launch list of the sharded inner loop (run it under
``ncu --metrics gpu__time_duration.sum``; never a multi-rank command).

    python scripts/sharded_world1.py [--n 262144]
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611", RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    from paper_2507_22538_b200.parallel import MdpShard, RankContext, solve_sharded_native
    n, m, K, W, gamma = a.n, a.m, 64, 4096, 0.999
    ctx = RankContext.from_env(n)
    lo, hi = ctx.block
    rp, col, val, cost = devgen.locality(n, m, K, W, 0, lo, hi - lo)
    shard = MdpShard(n, m, gamma, lo, cost, ipi.CsrMatrix((hi - lo) * m, n, rp, col, val))
    opts = ipi.SolveOptions(alpha=1e-4, tol=1e-8, max_outer=300)
    for _ in range(a.reps):
        res = solve_sharded_native(shard, ctx, opts)
    print(f"status {res.status.value} outer {res.outer_iterations} inner {res.inner_iterations_total} "
          f"greedy {res.time_greedy * 1e3:.2f} ms assembly {res.time_assembly * 1e3:.2f} ms "
          f"inner {res.time_inner * 1e3:.2f} ms")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
