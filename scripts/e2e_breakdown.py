"""Where the e2e greedy_policy step (pinned host V -> pinned host policy/TV)
spends its time beyond K1 on C2: wall-clock means over 20 calls of
(a) the public call, (b) the H2D copy alone, (c) K1 with zero-copy host
outputs, (d) K1 with device outputs, (e) isfinite(V).all() alone."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import _lib, devgen  # noqa: E402


def wall(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


mdp, spec = devgen.build_instance(2)
n = mdp.n
v_dev = torch.rand(n, dtype=torch.float64, device="cuda")
v_host = v_dev.cpu().pin_memory()
pol_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
app_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
pol_d = torch.empty(n, dtype=torch.int32, device="cuda")
app_d = torch.empty(n, dtype=torch.float64, device="cuda")
h = mdp.handle()
L = _lib.lib()
st = torch.cuda.current_stream()


def k1(p, a):
    _lib.check(L.ipi_bellman(h, _lib.ptr(v_dev), _lib.MODE_MIN, p, a, None, None, None,
                             _lib.stream_ptr()), "ipi_bellman")
    st.synchronize()


print("public greedy_policy   %.3f ms" % wall(lambda: ipi.greedy_policy(mdp, v_host)))
print("H2D 8 MB               %.3f ms" % wall(lambda: (v_dev.copy_(v_host, non_blocking=True), st.synchronize())))
print("K1 zero-copy outputs   %.3f ms" % wall(lambda: k1(pol_h.data_ptr(), app_h.data_ptr())))
print("K1 device outputs      %.3f ms" % wall(lambda: k1(_lib.ptr(pol_d), _lib.ptr(app_d))))
print("isfinite(V).all()      %.3f ms" % wall(lambda: bool(torch.isfinite(v_dev).all())))
print("pinned empty x2        %.3f ms" % wall(lambda: (torch.empty(n, dtype=torch.int32, pin_memory=True),
                                                       torch.empty(n, dtype=torch.float64, pin_memory=True))))
