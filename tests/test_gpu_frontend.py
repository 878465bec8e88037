"""Front-end workflow on the device, mirroring the reference's frontend tests
(pkg/frontend/tests/test_frontend.py): documented workflow from MDPMAT01
files, MDP.solve == library solve, error contracts, creators."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_22538_b200 as ipi  # noqa: E402
import paper_2507_22538_b200.frontend as mf  # noqa: E402


def _maze_files(tmp_path):
    g = load_golden("ref_maze33")
    n, m = g["cost"].shape
    csr = ipi.CsrMatrix(n * m, n, g["row_ptr"], g["col"], g["val"])
    ipi.write_matrix(tmp_path / "cost.bin", g["cost"])
    ipi.write_matrix(tmp_path / "trans.bin", csr)
    return g, tmp_path / "cost.bin", tmp_path / "trans.bin"


def test_documented_workflow_from_files(tmp_path):
    g, cost, trans = _maze_files(tmp_path)
    mdp = mf.MDP()
    mdp.setStageCostMatrix(mf.Matrix.fromFile(cost))
    mdp.setTransitionProbabilityTensor(mf.Matrix.fromFile(trans))
    mdp.setOption("-discount_factor", "0.99")
    mdp.setOption("-mode", "MINCOST")
    mdp.setOption("-ksp_type", "gmres")
    res = mdp.solve()
    assert res.status is ipi.SolveStatus.CONVERGED
    np.testing.assert_allclose(res.values, g["solve_gmres_values"], rtol=1e-8, atol=1e-8)
    np.testing.assert_array_equal(res.policy, g["solve_gmres_policy"])
    # same call through the library API: bitwise identical (frontend test :43-67)
    direct = ipi.solve(mdp.instance(), ipi.SolveOptions())
    np.testing.assert_array_equal(res.values, direct.values)
    np.testing.assert_array_equal(res.policy, direct.policy)
    assert res.residual_history == direct.residual_history


def test_file_round_trip_is_exact(tmp_path):
    g, cost, trans = _maze_files(tmp_path)
    back = mf.Matrix.fromFile(trans).data
    rp, col, val = back.numpy()
    np.testing.assert_array_equal(rp, g["row_ptr"])
    np.testing.assert_array_equal(col, g["col"])
    np.testing.assert_array_equal(val, g["val"])
    np.testing.assert_array_equal(mf.Matrix.fromFile(cost).data, g["cost"])


def test_missing_discount_and_shape_mismatch(tmp_path):
    g, cost, trans = _maze_files(tmp_path)
    mdp = mf.MDP()
    mdp.setStageCostMatrix(mf.Matrix.fromFile(cost))
    mdp.setTransitionProbabilityTensor(mf.Matrix.fromFile(trans))
    with pytest.raises(ipi.ValidationError, match="discount"):
        mdp.solve()
    mdp.setStageCostMatrix(np.zeros((3, 3)))
    mdp.setOption("-discount", "0.9")
    with pytest.raises(ipi.ValidationError, match="does not match"):
        mdp.solve()
    with pytest.raises(ipi.ValidationError, match="dense"):
        mf.MDP().setStageCostMatrix(mf.Matrix.fromFile(trans))


def test_creators_constant_self_loop():
    cost = mf.createStageCostMatrix(3, 2, lambda s, a: 1.0)
    tensor = mf.createTransitionProbabilityTensor(3, 2, lambda s, a: ([s], [1.0]))
    mdp = mf.MDP()
    mdp.setStageCostMatrix(cost)
    mdp.setTransitionProbabilityTensor(tensor)
    mdp.setOption("-discount", "0.5")
    np.testing.assert_allclose(mdp.solve().values, 2.0, atol=1e-9)


def test_created_tensor_equals_file_tensor(tmp_path):
    g, _, trans = _maze_files(tmp_path)
    n, m = g["cost"].shape
    rp, col, val = g["row_ptr"], g["col"], g["val"]

    def fn(s, a):
        r = s * m + a
        return col[rp[r]:rp[r + 1]].tolist(), val[rp[r]:rp[r + 1]].tolist()

    created = mf.createTransitionProbabilityTensor(n, m, fn)
    assert created.data.equals(mf.Matrix.fromFile(trans).data)


def test_creator_errors_name_the_pair():
    with pytest.raises(ipi.ValidationError, match="pre-allocation"):
        mf.createTransitionProbabilityTensor(3, 1, lambda s, a: ([0, 1, 2], [0.2, 0.3, 0.5]),
                                             prealloc=2)
    with pytest.raises(ipi.ValidationError, match=r"s=1, a=0"):
        mf.createTransitionProbabilityTensor(2, 1, lambda s, a: ([s], [0.4 if s else 1.0]))


@pytest.mark.parametrize("mutate,pattern", [
    (lambda rp, col, val, cost: (rp, col, val * 1.5, cost), "sum to 1"),
    (lambda rp, col, val, cost: (rp, col, np.where(np.arange(val.size) == 3, -0.1, val), cost),
     "lie in \\[0, 1\\]"),
    (lambda rp, col, val, cost: (rp, col, val, np.where(np.arange(cost.size).reshape(cost.shape) == 5,
                                                        np.inf, cost)), "non-finite"),
])
def test_validate_messages(mutate, pattern):
    g = load_golden("ref_fixture_random")
    rp, col, val, cost = mutate(g["row_ptr"], g["col"], g["val"].copy(), g["cost"].copy())
    n, m = cost.shape
    mdp = ipi.MdpInstance(n, m, 0.9, cost, ipi.CsrMatrix(n * m, n, rp, col, val))
    problems = ipi.validate(mdp)
    assert any(__import__("re").search(pattern, p) for p in problems), problems
    with pytest.raises(ipi.ValidationError):
        ipi.solve(mdp)


@pytest.mark.parametrize("rp,col,val,pattern", [
    ([0, 2, 1], [0, 1], [0.5, 0.5], "non-decreasing"),
    ([0, 2, 3], [1, 0, 0], [0.5, 0.5, 1.0], "strictly increasing"),
    ([0, 2, 3], [0, 5, 0], [0.5, 0.5, 1.0], "lie in"),
    ([0, 2, 3], [0, 1, 0], [0.5, np.nan, 1.0], "finite"),
    ([0, 2, 4], [0, 1, 0], [0.5, 0.5, 1.0], "nnz"),
])
def test_csr_structure_errors(rp, col, val, pattern):
    with pytest.raises(ValueError, match=pattern):
        ipi.CsrMatrix(2, 2, np.asarray(rp), np.asarray(col), np.asarray(val))
