"""greedy_policy's host-facing paths (the bench's e2e call): numpy in/out,
pinned CPU tensors in/out with K1 storing straight into the mapped host
buffers (zero-copy) or through D2H copies, and device tensors — all equal,
and a non-finite V raises ValidationError (bellman.py:123-129) on each path."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_22538_b200 as ipi  # noqa: E402
from paper_2507_22538_b200 import bellman, devgen  # noqa: E402


@pytest.mark.parametrize("zero_copy", [True, False])
@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_host_paths_agree(monkeypatch, zero_copy, cfg):
    monkeypatch.setattr(bellman, "_ZERO_COPY", zero_copy)
    kw = {"n": 5000} if cfg == 2 else ({"grid": 64} if cfg == 3 else {"n": 500})
    mdp, spec = devgen.build_instance(cfg, **kw)
    v = np.random.default_rng(cfg).random(mdp.n) * 10
    r_np = ipi.greedy_policy(mdp, v)
    vh = torch.as_tensor(v).pin_memory()
    r_h = ipi.greedy_policy(mdp, vh)
    r_d = ipi.greedy_policy(mdp, torch.as_tensor(v, device="cuda"))
    assert r_h.policy.device.type == "cpu" and r_h.policy.is_pinned()
    assert np.array_equal(r_h.policy.numpy(), r_np.policy)
    assert np.array_equal(r_h.applied.numpy(), r_np.applied)
    assert np.array_equal(r_d.policy.cpu().numpy(), r_np.policy)
    assert np.array_equal(r_d.applied.cpu().numpy(), r_np.applied)


@pytest.mark.parametrize("zero_copy", [True, False])
def test_non_finite_v_raises_on_host_path(monkeypatch, zero_copy):
    monkeypatch.setattr(bellman, "_ZERO_COPY", zero_copy)
    mdp, _ = devgen.build_instance(2, n=3000)
    v = torch.zeros(mdp.n, dtype=torch.float64).pin_memory()
    v[17] = float("nan")
    with pytest.raises(ipi.ValidationError, match="non-finite"):
        ipi.greedy_policy(mdp, v)
    with pytest.raises(ipi.ValidationError, match="non-finite"):
        ipi.greedy_policy(mdp, v.numpy())
