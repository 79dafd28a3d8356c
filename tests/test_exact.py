"""The exact T1 = 0 path against the reference.

Fixtures: tests/golden/make_exact_golden.py (the reference's exact.py on its
own test families and two larger equality-only instances).  Bars: identical
status, iteration count, restart triggers; objectives, residual fields and
solution norms within 1e-8 * max(1, |ref|); the two no-proximal
formulations' traces within 1e-10 of each other and of the reference's; the
exact path equals the lambda path when lambda = lambda_1 (<= 1e-12).
"""

import json

import numpy as np
import pytest

import paper_2408_12179_b200 as P
from conftest import GOLDEN, one_d_problem
from paper_2408_12179_b200 import exact as E
from paper_2408_12179_b200.driver import KktResidual

EG = json.load(open(f"{GOLDEN}/exact_golden.json"))
TR = np.load(f"{GOLDEN}/exact_traces.npz")


def _close(a, b, rel=1e-8):
    return abs(a - b) <= rel * max(1.0, abs(b))


def _eq(seed, m1, n, density=0.8):
    return P.generate_known_solution_lp(seed, m1, 0, n, density)[0]


def test_row_cap():
    with pytest.raises(ValueError, match="limit"):
        E.DenseCholesky.from_matrix(P.SparseMatrix.from_dense(np.eye(3)), row_limit=2)


def test_sigma_formula_host():
    a = P.SparseMatrix.from_dense(np.eye(2))
    anchor = E.ExactIterate(np.zeros(2), np.zeros(2))
    bar = E.ExactIterate(np.array([1.5, 0.0]), np.array([3.0, 0.0]))
    res = KktResidual(1.0, 1.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    assert E.sigma_update_exact(bar, anchor, a, res) == pytest.approx(2.0)


def test_rejects_inequality_block():
    prob, _ = P.generate_known_solution_lp(2, 2, 1, 6, 0.8)
    with pytest.raises(ValueError):
        E.solve_equality_exact(prob)




@pytest.mark.gpu
def test_normal_equations():
    chol = E.DenseCholesky.from_matrix(P.SparseMatrix.from_dense(np.eye(3)))
    assert np.allclose(E.solve_normal_equations(chol, np.array([1.0, 2.0, 3.0])), [1, 2, 3])
    chol = E.DenseCholesky.from_matrix(P.SparseMatrix.from_dense([[1.0, 1.0]]))
    assert E.solve_normal_equations(chol, np.array([4.0]))[0] == pytest.approx(2.0)
    g = EG["normal"]
    dense = np.array(g["dense"])
    chol = E.DenseCholesky.from_matrix(P.SparseMatrix.from_dense(dense))
    y = E.solve_normal_equations(chol, np.array(g["rhs"]))
    assert np.max(np.abs(y - np.array(g["y"]))) <= 1e-10 * max(1.0, np.max(np.abs(g["y"])))
    aat = dense @ dense.T
    assert np.linalg.norm(aat @ y - np.array(g["rhs"])) <= 1e-10 * np.linalg.norm(g["rhs"])
    with pytest.raises(ValueError):
        E.solve_normal_equations(chol, np.zeros(4))


@pytest.mark.gpu
def test_rank_deficiency_error():
    with pytest.raises(E.RankDeficiencyError, match="lambda-proximal"):
        E.DenseCholesky.from_matrix(P.SparseMatrix.from_dense(np.array([[1.0, 0.0], [1.0, 0.0]])))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["one_d", "scaled_identity"])
def test_exact_equals_lambda_path(case):
    """lambda = lambda_1(AA*): the proximal weight vanishes and the fused
    lambda-path kernels and the exact path coincide (reference
    test_exact.py:55-81)."""
    import torch
    from paper_2408_12179_b200.device import DeviceLP
    if case == "one_d":
        prob, sigma, lam, steps = one_d_problem(), 1.0, 1.0, 30
    else:
        prob = P.LpProblem.from_dense(2.0 * np.eye(2), [2.0, 4.0], None, None, [1.0, 1.0])
        sigma, lam, steps = 0.7, 4.0, 25
    dev = DeviceLP(prob)
    dev.analyze()
    dev.scale(0, False, False)
    dev.state_reset()
    data = E._Dev(prob, 0)
    with torch.cuda.stream(data.stream):
        chol = E.DenseCholesky.from_matrix(prob.a_eq)
        z = E.ExactIterate(torch.zeros(data.m, dtype=torch.float64, device="cuda"),
                           torch.zeros(data.n, dtype=torch.float64, device="cuda"))
        st = E.ExactState(current=z, anchor=E.ExactIterate(z.y.clone(), z.x.clone()),
                          sigma=sigma, variant=P.Variant.HPR)
        for k in range(steps):
            E.hpr_exact_iterate(st, data, chol)
            dev.run_inner(1, k, k, sigma, lam * sigma, 2)
            assert np.max(np.abs(st.current.y.cpu().numpy() - dev.to_host("y"))) <= 1e-12
            assert np.max(np.abs(st.current.x.cpu().numpy() - dev.to_host("x"))) <= 1e-12
    data.close()
    dev.close()


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(EG["reports"])))
def test_reports_vs_reference(idx):
    g = EG["reports"][idx]
    seed, m1, n, dens = g["gen"]
    prob = _eq(seed, m1, n, dens)
    cfg = P.SolverConfig(tolerance=g["tol"], variant=g.get("variant", "hpr"))
    rep = E.solve_equality_exact(prob, cfg)
    d = rep.to_json_dict(include_solution=False)
    r = g["report"]
    assert d["status"] == r["status"]
    assert d["iterations"] == r["iterations"] and d["restarts"] == r["restarts"]
    assert [e["trigger"] for e in d["restart_log"]] == [e["trigger"] for e in r["restart_log"]]
    assert [e["tau"] for e in d["restart_log"]] == [e["tau"] for e in r["restart_log"]]
    for k in ("primal_objective", "dual_objective"):
        assert _close(d[k], r[k]), (k, d[k], r[k])
    for k in ("primal_infeas_rel", "dual_infeas_rel", "gap_rel"):
        assert _close(d["kkt"][k], r["kkt"][k]), (k, d["kkt"][k], r["kkt"][k])
    assert d["lambda_estimate"] == 0.0
    for f in "xyz":
        ref = r["solution_norm"][f]
        assert abs(np.linalg.norm(getattr(rep.solution, f)) - ref) <= 1e-8 * max(1.0, ref)
    if g["planted_obj"] is not None and g["tol"] <= 1e-8:
        assert rep.primal_objective == pytest.approx(g["planted_obj"], rel=1e-8, abs=1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(EG["gaps"])))
def test_trace_gap(idx):
    g = EG["gaps"][idx]
    prob = one_d_problem() if g["case"] == "one_d" else _eq(*g["case"])
    gap = E.max_trace_gap(prob, g["sigma"], g["iters"])
    assert gap <= 1e-10, gap


@pytest.mark.gpu
def test_traces_vs_reference():
    prob = _eq(7, 3, 7)
    d = E.hpr_no_prox_trace(prob, 0.9, 12)
    a = E.halpern_padmm_trace(prob, 0.9, 12)
    for f in ("y", "z", "x_half", "x_tilde"):
        assert np.max(np.abs(np.array(getattr(d, f)) - TR[f"direct_{f}"])) <= 1e-10, f
    for f in ("y", "z", "x"):
        assert np.max(np.abs(np.array(getattr(a, f)) - TR[f"avg_{f}"])) <= 1e-10, f
    assert np.array_equal(d.z[0], a.z[0])
    assert np.max(np.abs(d.x_tilde[0] - d.x_half[0])) <= 1e-12
    prob = _eq(17, 2, 6)
    d = E.hpr_no_prox_trace(prob, 0.8, 30, y0=TR["nz_y0"], x0=TR["nz_x0"])
    assert np.max(np.abs(np.array(d.y) - TR["nz_direct_y"])) <= 1e-10
    assert np.max(np.abs(np.array(d.x_half) - TR["nz_direct_x_half"])) <= 1e-10
