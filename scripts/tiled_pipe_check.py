"""Tiled K1 (variant 9) parity spot check on a C5-shaped shard: oracle vs the
loaded library (used to A/B compile-time variants of bellman_tiled.cu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IPI_K1_TILED"] = "1"
import paper_2507_22538_b200 as ipi  # noqa: E402
from oracle import mdp_oracle as orc  # noqa: E402  (checker only)
from paper_2507_22538_b200 import devgen  # noqa: E402
from paper_2507_22538_b200.generators import CONFIGS  # noqa: E402
from paper_2507_22538_b200.parallel import MdpShard  # noqa: E402

spec = CONFIGS[5]
n, m, ns, s0 = 1 << 20, 8, 7777, 123457
rp, col, val, cost = devgen.locality(n, m, spec.K, spec.window, 0, s0, ns)
sh = MdpShard(n, m, spec.gamma, s0, cost, ipi.CsrMatrix(ns * m, n, rp, col, val))
assert sh.plan()["k1_variant"] == 9, sh.plan()
v = torch.rand(n, dtype=torch.float64, device="cuda") * 10
pol, app, _ = sh.bellman(v)
rph, colh, valh, costh = (t.cpu().numpy() for t in (rp, col, val, cost))
pi_ref, ap_ref = orc.greedy(rph, colh, valh, costh, spec.gamma, v.cpu().numpy(), False)
err = float(np.max(np.abs(app.cpu().numpy() - ap_ref) / np.maximum(1.0, np.abs(ap_ref))))
print("tiled parity max rel err %.2e %s" % (err, "OK" if err < 1e-13 else "FAIL"))
