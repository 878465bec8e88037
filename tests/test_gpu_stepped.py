"""The stepped GMRES(30) solver (csrc/krylov_step.cu: K3 ring operator + one
step_ortho launch per Arnoldi step) on a mid-size C2-shaped instance.

ipi_solve takes this path for uniform K = 64 rows once a CTA's slice is long
enough for MGS (n >= ~152k on 148 SMs); the full-size C2 tests cover it at
n = 2^20, this file covers ragged slices (odd n: the last CTA's slice ends on
an 8-byte tail chunk), the solver's switches and the persistent kernels as a
cross-check:

* default (pair-blocked MGS, programmatic dependent launch, r0 from K1's TV)
  against the C oracle: status and outer count equal, V to 1e-8, residual
  certificate;
* IPI_STEP_PAIR=0 (one vector per exchange, bitwise MGS), IPI_STEP_PDL=0,
  IPI_R0_FROM_TV=0 and IPI_K4_STEPPED=0 (persistent kernel) in subprocesses
  (the switches are read once per process): same status / outer count, V
  within 1e-10 relative of the default run.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = Path(__file__).resolve().parents[1]
N, M, K, W, GAMMA = 200_001, 4, 64, 2048, 0.99

_CHILD = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, {repo!r})
import paper_2507_22538_b200 as ipi
from paper_2507_22538_b200 import devgen
n, m, K, W, gamma = {n}, {m}, {k}, {w}, {gamma}
rp, col, val, cost = devgen.locality(n, m, K, W, 0, 0, n)
mdp = ipi.MdpInstance(n, m, gamma, cost, ipi.CsrMatrix(n * m, n, rp, col, val))
pc = ipi.Preconditioner.from_name(sys.argv[2] if len(sys.argv) > 2 else "none")
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 0
mode = ipi.Mode.from_name(sys.argv[4] if len(sys.argv) > 4 else "min")
res = ipi.solve(mdp, ipi.SolveOptions(alpha=1e-4, tol=1e-8, gmres_ortho="mgs", pc=pc, mode=mode,
                                      ksp_max_it=cap or None))
np.save(sys.argv[1], res.values)
print(json.dumps({{"status": res.status.value, "outer": res.outer_iterations,
                  "inner": res.inner_iterations_total, "hist": res.residual_history}}))
"""


def _child(tmp_path, tag, env, pc="none", cap=0, mode="min"):
    out = tmp_path / f"v_{tag}.npy"
    code = _CHILD.format(repo=str(REPO), n=N, m=M, k=K, w=W, gamma=GAMMA)
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", code, str(out), pc, str(cap), mode], capture_output=True,
                       text=True, env=e, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    info = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    return info, np.load(out)


def test_stepped_default_matches_c_oracle_and_switches_agree(tmp_path):
    from oracle import c_oracle as co
    import paper_2507_22538_b200 as ipi
    from paper_2507_22538_b200 import devgen

    base, v = _child(tmp_path, "default", {})
    rp, col, val, cost = (t.cpu().numpy() for t in devgen.locality(N, M, K, W, 0, 0, N))
    ref = co.solve(rp, col, val, cost, GAMMA, tol=1e-8, alpha=1e-4, kind="gmres")
    assert base["status"] == ref.status
    assert base["outer"] == ref.outer_iterations
    scale = max(1.0, np.abs(ref.values).max())
    np.testing.assert_allclose(v, ref.values, rtol=1e-8, atol=1e-8 * scale)
    _, _, r = co.greedy(rp, col, val, cost, GAMMA, v)
    assert r <= 1e-8 * 1.0001
    for tag, env in (("single", {"IPI_STEP_PAIR": "0"}), ("nopdl", {"IPI_STEP_PDL": "0"}),
                     ("r0spmv", {"IPI_R0_FROM_TV": "0"}), ("persistent", {"IPI_K4_STEPPED": "0"})):
        info, vv = _child(tmp_path, tag, env)
        assert info["status"] == base["status"], tag
        assert info["outer"] == base["outer"], tag
        np.testing.assert_allclose(vv, v, rtol=1e-10, atol=1e-10 * scale, err_msg=tag)
    # programmatic dependent launch changes no arithmetic: bitwise equal results
    _, v_nopdl = _child(tmp_path, "nopdl2", {"IPI_STEP_PDL": "0"})
    assert np.array_equal(v_nopdl, v)


def test_stepped_with_jacobi_agrees_with_the_persistent_kernel(tmp_path):
    """Left Jacobi preconditioning (inner.py:113-118) through the stepped
    solver (w = pc(A v_j) in step_ortho, z = pc(r) in step_cycle_start) against
    the persistent kernel on the same instance, and the fixed point against
    the unpreconditioned C oracle solve."""
    from oracle import c_oracle as co
    from paper_2507_22538_b200 import devgen

    a, va = _child(tmp_path, "jac_stepped", {}, pc="jacobi")
    b, vb = _child(tmp_path, "jac_persistent", {"IPI_K4_STEPPED": "0"}, pc="jacobi")
    assert a["status"] == b["status"] == "converged"
    assert a["outer"] == b["outer"]
    scale = max(1.0, np.abs(vb).max())
    np.testing.assert_allclose(va, vb, rtol=1e-10, atol=1e-10 * scale)
    rp, col, val, cost = (t.cpu().numpy() for t in devgen.locality(N, M, K, W, 0, 0, N))
    ref = co.solve(rp, col, val, cost, GAMMA, tol=1e-8, alpha=1e-4, kind="gmres")
    np.testing.assert_allclose(va, ref.values, rtol=1e-8, atol=1e-8 * scale)
    _, _, r = co.greedy(rp, col, val, cost, GAMMA, va)
    assert r <= 1e-8 * 1.0001


@pytest.mark.parametrize("cap", [7, 37])
def test_stepped_fixed_inner_iterations(tmp_path, cap):
    """Optimistic-PI style runs (driver.py:170-175: target 0, exactly ksp_max_it
    inner iterations per outer step): the cap falls inside a cycle (7) and
    across a restart (37 = 30 + 7); the stepped solver must stop on the same
    iteration as the persistent kernel."""
    a, va = _child(tmp_path, f"cap{cap}_stepped", {}, cap=cap)
    b, vb = _child(tmp_path, f"cap{cap}_persistent", {"IPI_K4_STEPPED": "0"}, cap=cap)
    assert a["status"] == b["status"]
    assert a["outer"] == b["outer"]
    assert a["inner"] == b["inner"] == cap * a["outer"]
    scale = max(1.0, np.abs(vb).max())
    np.testing.assert_allclose(va, vb, rtol=1e-9, atol=1e-9 * scale)


def test_stepped_max_mode(tmp_path):
    """MAX mode: K1's TV is the per-state maximum, and r0 = TV - V holds all the
    same; the stepped solve against the persistent kernel and the C oracle."""
    from oracle import c_oracle as co
    from paper_2507_22538_b200 import devgen

    a, va = _child(tmp_path, "max_stepped", {}, mode="max")
    b, vb = _child(tmp_path, "max_persistent", {"IPI_K4_STEPPED": "0"}, mode="max")
    assert a["status"] == b["status"] == "converged"
    assert a["outer"] == b["outer"]
    scale = max(1.0, np.abs(vb).max())
    np.testing.assert_allclose(va, vb, rtol=1e-10, atol=1e-10 * scale)
    rp, col, val, cost = (t.cpu().numpy() for t in devgen.locality(N, M, K, W, 0, 0, N))
    ref = co.solve(rp, col, val, cost, GAMMA, maximize=True, tol=1e-8, alpha=1e-4, kind="gmres")
    assert a["status"] == ref.status and a["outer"] == ref.outer_iterations
    np.testing.assert_allclose(va, ref.values, rtol=1e-8, atol=1e-8 * scale)
