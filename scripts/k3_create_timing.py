"""Time planned K3 operator creation (ipi_op_create) three times on C2 P_pi:
the first includes the shape autotune, later ones hit the per-geometry cache."""
import time, torch, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_22538_b200 as ipi
from paper_2507_22538_b200 import devgen
from paper_2507_22538_b200.bellman import greedy_device
from paper_2507_22538_b200.sparse import DeviceOperator
mdp, spec = devgen.build_instance(2)
v = torch.rand(mdp.n, dtype=torch.float64, device="cuda")
pi, _, _ = greedy_device(mdp, v, ipi.Mode.MIN)
P = ipi.gather_policy_matrix(mdp, pi.long())
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    op = DeviceOperator(P.row_ptr, P.col_idx, P.values, mdp.n, mdp.n, 0, spec.gamma)
    torch.cuda.synchronize(); print("create", i, "%.1f ms" % ((time.perf_counter() - t) * 1e3), op.plan())
