"""Host-side API of the drop-in (no GPU): config validation, restart / sigma
rules, report schema, problem types.  Cases mirror the reference's unit tests
(reference tests/test_driver.py:61-150, 321-331; test_sparse.py:18-39;
test_problem.py) and SPEC.md's acceptance criteria 7 and 8."""

import json
import math

import numpy as np
import pytest

import paper_2408_12179_b200 as P
from paper_2408_12179_b200.driver import (KktResidual, RestartKind, Timings, kkt_from_sums,
                                          merit_from_sums, sigma_from_norms)

CFG = P.SolverConfig()


def residual_with(primal_rel, dual_rel):
    return KktResidual(primal_rel, primal_rel, dual_rel, dual_rel, 0.0, 0.0, 0.0, 0.0, 0.0)


class TestConfig:
    def test_defaults_match_reference(self):
        c = P.SolverConfig()
        assert (c.tolerance, c.check_interval, c.alpha1, c.alpha2, c.alpha3, c.sigma0) == \
            (1e-8, 150, 0.2, 0.6, 0.2, 1.0)
        assert c.variant is P.Variant.HPR and c.ruiz_iters == 10
        assert c.pock_chambolle and c.bc_normalize and c.termination_space == "original"
        assert (c.power_tol, c.power_max_iters, c.max_iterations) == (1e-4, 5000, 1_000_000)
        assert c.time_limit_seconds == math.inf

    @pytest.mark.parametrize("kw", [dict(alpha1=0.7, alpha2=0.6), dict(alpha3=1.0),
                                    dict(tolerance=0.0), dict(check_interval=0),
                                    dict(sigma0=0.0), dict(termination_space="both")])
    def test_validation(self, kw):
        with pytest.raises(ValueError):
            P.SolverConfig(**kw)

    def test_variant_from_string(self):
        assert P.SolverConfig(variant="dr").variant is P.Variant.DR
        assert P.SolverConfig(variant="hdr-fixed").variant is P.Variant.HDR_FIXED_SIGMA

    def test_coerce_foreign_config(self):
        class Foreign:  # shaped like the reference's SolverConfig
            tolerance = 1e-6
            check_interval = 70
            variant = "hdr"
        c = P.SolverConfig.coerce(Foreign())
        assert c.tolerance == 1e-6 and c.check_interval == 70 and c.variant is P.Variant.HDR


class TestRestartRules:
    """SPEC criterion 8 / reference test_acceptance.py:178-193."""

    def test_branches_and_priority(self):
        assert P.check_restart(1.9, 10.0, 5.0, 1, 10**9, CFG) is RestartKind.SUFFICIENT
        assert P.check_restart(5.0, 10.0, 4.0, 1, 10**9, CFG) is RestartKind.STALLED
        assert P.check_restart(9.9, 10.0, 9.0, 200, 1000, CFG) is RestartKind.LONG_LOOP
        assert P.check_restart(9.9, 10.0, 9.0, 199, 1000, CFG) is None
        assert P.check_restart(1.9, 10.0, 1.0, 10**9, 10**9, CFG) is RestartKind.SUFFICIENT
        assert P.check_restart(5.0, 10.0, 4.0, 10**9, 10**9, CFG) is RestartKind.STALLED

    def test_termination_inclusive(self):
        r = residual_with(1e-6, 1e-6)
        r.gap_rel = 1e-6
        assert P.check_termination(r, 1e-6)
        r.gap_rel = 2e-6
        assert not P.check_termination(r, 1e-6)


class TestSigmaUpdate:
    """SPEC criterion 7 / reference test_acceptance.py:158-175 (lambda = 4:
    delta_y = 2 * ||y_bar - y_anchor||)."""

    @pytest.mark.parametrize("dx,dy,ep,ed,expect", [
        (2.0, 1.0, 1.0, 1.0, 1.0), (4.0, 1.0, 1.0, 1.0, 2.0), (1e-20, 1.0, 1.0, 1.0, 1.0),
        (2.0, 1e-20, 1.0, 1.0, 1.0), (4.0, 1.0, 1.0, 1e-9, 1.0), (4.0, 1.0, 1e-9, 1.0, 1.0),
        (4.0, 1.0, 0.0, 0.0, 2.0), (4.0, 1.0, 0.0, 1.0, 1.0)])
    def test_guards(self, dx, dy, ep, ed, expect):
        assert sigma_from_norms(dx, dy, 4.0, residual_with(ep, ed)) == pytest.approx(expect)


class _Sums:
    def __init__(self, **kw):
        for f in ("bar_dx2", "bar_dy2", "dy2", "dx2", "sh2", "aty2", "prim2", "dual2", "r1sq",
                  "r2sq", "cx", "by", "lz", "uz"):
            setattr(self, f, kw.get(f, 0.0))
        for f in ("n_lo", "n_up", "clamped"):
            setattr(self, f, kw.get(f, 0))


class TestScalarsFromSums:
    def test_kkt_one_d_origin(self):
        # reference test_driver.py:33-39: |Pi_D(b)| = 1, |c| = 1 -> rel 0.5
        r = kkt_from_sums(_Sums(prim2=1.0, dual2=1.0), 1.0, 1.0, 0.0)
        assert r.primal_infeas_abs == 1.0 and r.dual_infeas_abs == 1.0
        assert r.primal_infeas_rel == 0.5 and r.dual_infeas_rel == 0.5

    def test_dual_objective_terms(self):
        r = kkt_from_sums(_Sums(cx=2.0, by=5.0, lz=1.0, n_lo=1, uz=-0.5, n_up=1, clamped=2),
                          0.0, 0.0, 3.0)
        assert r.primal_objective == 5.0
        assert r.dual_objective == 5.0 + 1.0 - 0.5 + 3.0
        assert r.dual_clamped == 2

    def test_merit_one_d(self):
        # reference test_core.py:128-132: dy = -2, dx = 0, sigma = lam = 1, A = [1] -> merit 2
        # (checkpoint_merit's factor 2 applies to the half-step difference dy = -1)
        o = _Sums(dy2=1.0, dx2=0.0, aty2=1.0, sh2=1.0)
        assert merit_from_sums(o, 1.0, 1.0) == pytest.approx(2.0)

    def test_merit_negative_form_warns(self):
        o = _Sums(dy2=1.0, aty2=1.0, sh2=0.0, dx2=1.0)
        with pytest.warns(RuntimeWarning):
            merit_from_sums(o, 1.0, 0.1)


class TestReport:
    def test_schema_v1(self):
        sol = P.PrimalDualPoint(y=np.zeros(1), z=np.zeros(2), x=np.ones(2))
        rep = P.SolveReport(P.SolveStatus.OPTIMAL, 1.0, 1.0, residual_with(0.0, 0.0), 150, 1,
                            [P.RestartEvent(0, "long_loop", 150, 1.5, 0.1)], Timings(0.1, 0.2, 0.3, 0.4),
                            sol, 1.5, 2.0)
        d = rep.to_json_dict()
        assert d["schema_version"] == 1 and d["status"] == "Optimal"
        assert set(d) == {"schema_version", "status", "primal_objective", "dual_objective", "kkt",
                          "iterations", "restarts", "restart_log", "timings", "sigma_final",
                          "lambda_estimate", "solution"}
        assert d["timings"]["solve_seconds"] == pytest.approx(0.9)
        assert set(d["kkt"]) == {"primal_infeas_abs", "primal_infeas_rel", "dual_infeas_abs",
                                 "dual_infeas_rel", "gap_abs", "gap_rel", "residual_vector_norm",
                                 "primal_objective", "dual_objective", "dual_clamped"}
        json.dumps(d)
        assert "solution" not in rep.to_json_dict(include_solution=False)


class TestProblemTypes:
    def test_canonicalization(self):
        a = P.SparseMatrix.from_coo([0, 0, 1], [1, 1, 0], [2.0, 3.0, 0.0], shape=(2, 2))
        assert a.nnz == 1 and a.values.tolist() == [5.0] and a.col_indices.tolist() == [1]

    def test_invariants_rejected(self):
        with pytest.raises(ValueError):
            P.SparseMatrix(np.array([0, 2]), np.array([1, 0]), np.array([1.0, 2.0]), 1, 2)
        with pytest.raises(ValueError):
            P.SparseMatrix(np.array([0, 1]), np.array([0]), np.array([0.0]), 1, 1)

    def test_lp_validation(self):
        with pytest.raises(ValueError):
            P.LpProblem.from_dense([[1.0]], [1.0], None, None, [1.0], lower=[2.0], upper=[1.0])
        with pytest.raises(ValueError):
            P.LpProblem.from_dense([[0.0]], [1.0], None, None, [1.0])
        with pytest.raises(ValueError):
            P.LpProblem.from_dense([[1.0]], [np.inf], None, None, [1.0])

    def test_stacked(self):
        p = P.LpProblem.from_dense([[1.0, 0.0]], [1.0], [[0.0, 2.0], [3.0, 4.0]], [0.0, 1.0],
                                   [1.0, 1.0])
        assert p.m1 == 1 and p.m2 == 2 and p.m == 3
        assert np.array_equal(p.stacked_matrix.to_dense(), [[1, 0], [0, 2], [3, 4]])
        assert p.rhs.tolist() == [1.0, 0.0, 1.0]

    def test_projections_and_objectives(self):
        v = np.array([2.0, -2.0])
        assert P.project_onto_box(v, np.zeros(2), np.array([1.0, np.inf])).tolist() == [1.0, 0.0]
        assert P.project_onto_dual_cone(np.array([-3.0, -3.0]), 1).tolist() == [-3.0, 0.0]
        p = P.LpProblem.from_dense([[1.0]], [1.0], None, None, [1.0], lower=[-np.inf],
                                   upper=[np.inf])
        val, clamped = P.dual_objective(p, np.array([5.0]), np.array([1.0]))
        assert val == 5.0 and clamped == 1
        assert P.primal_objective(p, np.array([2.0])) == 2.0

    def test_reference_problem_is_accepted(self):
        """solve() accepts reference-shaped objects (duck typing of a_eq/a_ineq)."""
        from paper_2408_12179_b200.problem import stacked_arrays
        p = P.LpProblem.from_dense([[1.0, 2.0]], [1.0], [[3.0, 0.0]], [0.5], [1.0, 1.0])
        ro, ci, v, m, n, m1 = stacked_arrays(p)
        assert (m, n, m1) == (2, 2, 1) and ro.tolist() == [0, 2, 3]
        assert ci.tolist() == [0, 1, 0] and v.tolist() == [1.0, 2.0, 3.0]


@pytest.mark.parametrize("loop", ["0", "1"])
def test_packed_batch_staging_layout(loop, monkeypatch):
    """Packing into a staging buffer (solve_batch's path) gives the same arrays
    as fresh packing, at the 256-byte-aligned upload layout BatchRun uses."""
    import numpy as np
    from paper_2408_12179_b200 import generate_known_solution_lp
    from paper_2408_12179_b200.batch import PackedBatch
    monkeypatch.setenv("HPR_PACK_LOOP", loop)
    probs = [generate_known_solution_lp(s, 20 + s, 30 + 2 * s, 90 + 5 * s, 0.3)[0] for s in range(5)]
    ref = PackedBatch(probs)
    bufs = []

    def staging(nb):
        bufs.append(np.full(nb + 512, 0xAB, np.uint8))
        return bufs[-1]

    pk = PackedBatch(probs, staging=staging)
    base = bufs[0].ctypes.data
    off = 0
    for name, dt in PackedBatch.ORDER:
        a = pk.arrays[name]
        assert a.dtype == np.dtype(dt)
        assert a.ctypes.data == base + off
        assert np.array_equal(a, ref.arrays[name].astype(dt))
        off += (a.nbytes + 255) // 256 * 256
    assert list(pk.arrays) == [k for k, _ in PackedBatch.ORDER]
