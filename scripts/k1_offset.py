"""Is K1's streaming rate address-dependent?  Re-home the C2 CSR arrays at
byte offsets from a fresh allocation and time K1 for the forced ring shape
(IPI_URING_* env) at each offset.

    IPI_URING_WARPS=12 IPI_URING_STAGES=3 IPI_URING_WAVES=4 python scripts/k1_offset.py
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402
from paper_2507_22538_b200.generators import CONFIGS  # noqa: E402


def rehome(t, off_bytes):
    es = t.element_size()
    pad = (off_bytes + es - 1) // es
    buf = torch.empty(t.numel() + pad, dtype=t.dtype, device=t.device)
    view = buf[pad:pad + t.numel()]
    view.copy_(t)
    return view


def time_k1(mdp, v, reps=10):
    for _ in range(2):
        greedy_device(mdp, v, ipi.Mode.MIN)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        greedy_device(mdp, v, ipi.Mode.MIN)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    torch.cuda.set_device(0)
    spec = CONFIGS[2]
    rp, col, val, cost = devgen.locality(spec.n, spec.m, spec.K, spec.window, 0)
    v = torch.rand(spec.n, dtype=torch.float64, device="cuda")
    for off in [0, 4096, 65536, 1 << 20, (2 << 20) + 8192, 3 << 20, 5 << 20]:
        val2, col2 = rehome(val, off), rehome(col, off // 2)
        mdp = ipi.MdpInstance(spec.n, spec.m, spec.gamma, cost,
                              ipi.CsrMatrix(spec.n * spec.m, spec.n, rp, col2, val2))
        ms = time_k1(mdp, v)
        print(f"offset {off:>9d}  val@{val2.data_ptr() % (1 << 21):>8d}  K1 {ms:.3f} ms  "
              f"blocks {mdp.plan()['k1_blocks']}", flush=True)
        del mdp, val2, col2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
