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


def _k64_instance(n=2000, m=4, seed=0):
    from paper_2507_22538_b200.generators import random_locality_host
    return random_locality_host(n, m, 64, 300, seed=seed)


@pytest.mark.parametrize("kind", ["prob", "sum", "order", "range", "nan", "clean"])
def test_validate_uniform_k64_streaming_kernel(kind):
    """The K = 64 streaming validation kernel reports what the reference's
    validate reports (model.py:148-194): first bad probability entry, bad row
    sums (first five rows), and the structural CSR errors."""
    n, m = 2000, 4
    rp, col, val, cost = (np.array(a, copy=True) for a in _k64_instance(n, m))
    if kind == "prob":
        val[777] = -0.25
        val[778] += 0.25
        want = "entry 777 is -0.25"
    elif kind == "sum":
        val[64 * 5 + 3] += 1e-9           # row 5
        val[64 * 901 + 10] *= 1.5         # row 901
        want = "row 5 sums to"
    elif kind == "order":
        r0 = 64 * 42
        col[r0 + 9], col[r0 + 10] = col[r0 + 10], col[r0 + 9]
        want = "strictly increasing"
    elif kind == "range":
        col[64 * 7 + 63] = n + 5
        want = "lie in \\[0"
    elif kind == "nan":
        val[4000] = np.nan
        want = "finite"
    else:
        want = None
    if kind in ("order", "range", "nan"):
        # structural errors surface from CsrMatrix construction (sparse.py:56-86)
        with pytest.raises((ipi.ValidationError, ValueError), match=want):
            ipi.CsrMatrix(n * m, n, rp, col, val)
        return
    mdp = ipi.MdpInstance(n, m, 0.9, cost, ipi.CsrMatrix(n * m, n, rp, col, val))
    probs = ipi.validate(mdp)
    if want is None:
        assert probs == []
    else:
        assert any(want in p for p in probs), probs
        if kind == "sum":
            assert "row 901" in " ".join(probs)
