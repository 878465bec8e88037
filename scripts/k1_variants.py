"""Cross-check K1 variants (TMA ring vs register kernels) on a config:
same instance, same V -> identical policy / TV / residual expected."""

from __future__ import annotations

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.bellman import greedy_device  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(sys.argv[2]) if len(sys.argv) > 2 else None
    torch.cuda.set_device(0)
    kw = {"n": n} if n and cfg in (1, 2) else ({"grid": n} if n and cfg == 3 else {})
    rp, col, val, cost, spec, nn = devgen.build_arrays(cfg, **kw)
    out = {}
    for tma in ("1", "0"):
        os.environ["IPI_K1_TMA"] = tma
        csr = ipi.CsrMatrix(nn * spec.m, nn, rp, col, val)
        mdp = ipi.MdpInstance(nn, spec.m, spec.gamma, cost, csr)
        print("plan", tma, mdp.plan(), flush=True)
        v = torch.linspace(0, 10, nn, dtype=torch.float64, device="cuda")
        pi, ap, rb = greedy_device(mdp, v, ipi.Mode.MIN, with_residual=True)
        torch.cuda.synchronize()
        out[tma] = (pi.clone(), ap.clone(), float(rb.view(torch.float64)[0]))
        del mdp
    a, b = out["1"], out["0"]
    print("policy equal:", bool(torch.equal(a[0], b[0])), "max |dTV|:",
          float((a[1] - b[1]).abs().max()), "res", a[2], b[2])


if __name__ == "__main__":
    main()
