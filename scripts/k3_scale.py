import sys, json
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2507_22538_b200 as ipi
from paper_2507_22538_b200 import devgen
from paper_2507_22538_b200.bellman import greedy_device
from paper_2507_22538_b200.sparse import DeviceOperator
torch.cuda.set_device(0)
mdp, spec = devgen.build_instance(2)
v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
P = ipi.gather_policy_matrix(mdp, pi.long())
n = mdp.n
del mdp
torch.cuda.empty_cache()
x = torch.rand(n, dtype=torch.float64, device="cuda")
for frac in (1.0, 0.5, 0.25, 0.125):
    nl = int(n * frac)
    op = DeviceOperator(P.row_ptr[:nl + 1], P.col_idx[:nl * 64], P.values[:nl * 64], nl, n, 0, spec.gamma)
    y = torch.empty(nl, dtype=torch.float64, device="cuda")
    for _ in range(5): op.apply(x, out=y)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
    for a, b in evs:
        a.record(); op.apply(x, out=y); b.record()
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
    byts = nl * 64 * 12 + 16 * nl
    print(json.dumps({"rows": nl, "ms": ms, "gbs": byts / ms / 1e6, "plan": op.plan()}), flush=True)
