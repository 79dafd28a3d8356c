"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference's golden reports.

Bars (BASELINE.json north_star):
* sparse products and the fused iteration: BIT-EXACT against the oracle on
  the same scaled problem and lambda (the kernels sum each row left to right
  with separately rounded products, like scipy's csr_matvec);
* Ruiz / Pock-Chambolle values and scale vectors: bit-exact;
* solves vs the reference's golden reports: identical status and iteration
  count, identical restart triggers, objectives and the relative residual
  fields within 1e-8 * max(1, |ref|);
* first 100 iterates normwise within 1e-10 of the reference trajectory.
"""

import json
import warnings

import numpy as np
import pytest

import paper_2408_12179_b200 as P
from conftest import GOLDEN, acceptance_suite, bounded_tiny_lp, one_d_problem, problem_from_dict
from oracle import hprlp_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-8


def _dev(prob, ruiz=10, pc=True, bc=True):
    from paper_2408_12179_b200.device import DeviceLP
    dev = DeviceLP(prob)
    dev.analyze()
    dev.scale(ruiz, pc, bc)
    return dev


def _oracle_on_device_scaling(dev, prob):
    olp = O.OracleLP.from_problem(prob)
    a = O.Csr(olp.a.rp, olp.a.ci, dev.to_host("a_val_s"), olp.n)
    return O.OracleLP(a=a, b=dev.to_host("b_s"), c=dev.to_host("c_s"),
                      lower=dev.to_host("lower_s"), upper=dev.to_host("upper_s"), m1=olp.m1)


def _close(a, b, rel=TOL):
    if not (np.isfinite(a) and np.isfinite(b)):
        return (np.isnan(a) and np.isnan(b)) or a == b
    return abs(a - b) <= rel * max(1.0, abs(b))


def _rel_close(a, b, rel, floor=0.0):
    """|a - b| <= rel * |b| + floor (both finite), or identical non-finite values."""
    if not (np.isfinite(a) and np.isfinite(b)):
        return (np.isnan(a) and np.isnan(b)) or a == b
    return abs(a - b) <= rel * abs(b) + floor + 1e-300


# sigma_next / merit / sigma_final: functions of device-reduced norms whose
# only difference from the reference is the summation order of the dot
# products (BLAS ddot vs a fixed-order tree) and the iterate rounding that
# follows from it.  Both are norms of DIFFERENCES of iterates (x_bar - x0,
# y_bar - y0: driver.py:264-278; w - w_bar: core.py:182-201), so they carry
# the iterates' absolute agreement (~1e-15 on O(1) iterates), amplified by
# |w| / |dw|.  The reference's own algorithm moves sigma_next by up to 4e-8
# relative when ONLY its norms are summed in another order
# (tests/test_oracle_golden.py::test_sigma_sensitivity_to_norm_order: exact
# fsum norms, acceptance suite at 1e-8), so 1e-9 is unattainable by any
# implementation; the bar is 5e-7 (the GPU measured <= 5e-8); the merit gets
# an absolute floor of 1e-12 on top (it shrinks to ~1e-7).
SIGMA_REL = 5e-7
MERIT_FLOOR = 1e-12


def assert_report_parity(rep, g, name="", tol=1e-8):
    """Every field of the reference's report (driver.py:154-188) except the
    timings: counts and triggers identical, objectives and all KKT fields
    within 1e-8 * max(1, |ref|), restart sigma / merit and sigma_final within
    SIGMA_REL relative (scaled up for solves deeper than 1e-8: the outer-loop
    differences those norms measure shrink with the solve tolerance ``tol``,
    the iterates' absolute agreement does not), lambda within 1e-12."""
    srel = SIGMA_REL * max(1.0, 1e-8 / tol)
    d = rep.to_json_dict(include_solution=False) if not isinstance(rep, dict) else rep
    assert d["status"] == g["status"], name
    assert d["iterations"] == g["iterations"], name
    assert d["restarts"] == g["restarts"], name
    assert len(d["restart_log"]) == len(g["restart_log"]) == d["restarts"], name
    for e, f in zip(d["restart_log"], g["restart_log"]):
        assert (e["outer_index"], e["trigger"], e["tau"]) == (
            f["outer_index"], f["trigger"], f["tau"]), (name, e, f)
        assert _rel_close(e["sigma_next"], f["sigma_next"], srel), (name, "sigma_next", e, f)
        assert _rel_close(e["merit"], f["merit"], srel, MERIT_FLOOR), (name, "merit", e, f)
    assert _rel_close(d["sigma_final"], g["sigma_final"], srel), (
        name, d["sigma_final"], g["sigma_final"])
    assert _close(d["primal_objective"], g["primal_objective"]), (name, d["primal_objective"])
    assert _close(d["dual_objective"], g["dual_objective"]), (name, d["dual_objective"])
    for k in ("primal_infeas_abs", "primal_infeas_rel", "dual_infeas_abs", "dual_infeas_rel",
              "gap_abs", "gap_rel", "residual_vector_norm", "primal_objective",
              "dual_objective"):
        assert _close(d["kkt"][k], g["kkt"][k]), (name, k, d["kkt"][k], g["kkt"][k])
    assert d["kkt"]["dual_clamped"] == g["kkt"]["dual_clamped"], name
    assert _close(d["lambda_estimate"], g["lambda_estimate"], 1e-12), name


# ---------------------------------------------------------------------------
# kernels: bit-exact against the oracle
# ---------------------------------------------------------------------------

# SELL-32-sigma / column-blocked smem-staged (HPR_CB) / SELL with A's columns
# split into blocks whose running sums are carried block to block
# (HPR_SPLIT_COLS) / staged segmented engine (HPR_STG, both phases) / SELL
# with both matrices' rows in the row-affinity order (HPR_RAO=1, 2^5-column
# blocks so small problems get a non-trivial order) / the resident small-LP
# loop (HPR_SMALL=1: one cluster launch per interval, hpr_small.cuh); every
# other engine runs on the per-iteration graph path (HPR_SMALL=0) / the
# bulk-copy-streamed SELL engine on both phases (HPR_TS=1, hpr_tsell.cuh)
ENGINES = ["sell", "cb", "split", "stg", "rao", "small", "ts"]


def _engine_env(monkeypatch, engine, n):
    monkeypatch.setenv("HPR_SMALL", "1" if engine == "small" else "0")
    monkeypatch.setenv("HPR_TS", "1" if engine == "ts" else "0")
    monkeypatch.setenv("HPR_CB", "1" if engine == "cb" else "0")
    monkeypatch.setenv("HPR_STG", "1" if engine == "stg" else "0")
    if engine == "rao":
        monkeypatch.setenv("HPR_RAO", "1")
        monkeypatch.setenv("HPR_RAO_AT", "1")
        monkeypatch.setenv("HPR_RAO_BITS", "5")
    else:
        monkeypatch.setenv("HPR_RAO", "0")
        monkeypatch.setenv("HPR_RAO_AT", "0")
    if engine == "split":
        monkeypatch.setenv("HPR_SPLIT_COLS", str(max(1, -(-n // 7))))   # 7 column blocks
    else:
        monkeypatch.delenv("HPR_SPLIT_COLS", raising=False)
        monkeypatch.setenv("HPR_SPLIT", "0")


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("variant,code", [("hpr", 2), ("hdr", 1), ("dr", 0)])
def test_iteration_bit_exact_c1(variant, code, engine, monkeypatch):
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    _engine_env(monkeypatch, engine, prob.n)
    dev = _dev(prob)
    info = dev.layout_info()
    assert (info["cb_a"] > 0 and info["cb_at"] > 0) == (engine == "cb")
    assert info["split_a"] == (7 if engine == "split" else 0)
    assert (info["stg_a"] > 0 and info["stg_at"] > 0) == (engine == "stg")
    assert (info["rao_a"], info["rao_at"]) == ((1, 1) if engine == "rao" else (0, 0))
    assert (info["ts_a"] > 0 and info["ts_at"] > 0) == (engine == "ts")
    lam = dev.power(1e-4, 5000).raw * 1.001
    slp = _oracle_on_device_scaling(dev, prob)
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 0.83, lam,
                 variant=variant)
    dev.state_reset()
    for k in range(100):
        dev.run_inner(1, k, k, 0.83, lam * 0.83, code)
        O.iterate_once(st, slp)
        if k % 9 == 0 or k == 99:
            assert np.array_equal(dev.to_host("y"), st.y), k
            assert np.array_equal(dev.to_host("x"), st.x), k
    # one graph replay of 100 iterations lands on the same bits
    dev.state_reset()
    dev.run_inner(100, 0, 0, 0.83, lam * 0.83, code)
    assert np.array_equal(dev.to_host("y"), st.y)
    assert np.array_equal(dev.to_host("x"), st.x)


@pytest.mark.parametrize("engine", ["sell", "split", "stg", "rao", "ts"])
def test_iteration_bit_exact_midsize(engine, monkeypatch):
    """140k x 140k, 7 per row: >= 131072 rows (the HPR_SORT_WIN threshold) and
    the column-split A over seven 20k-column blocks."""
    prob, _ = P.generate_planted_lp_fast(5, 70_000, 70_000, 140_000, 7)
    _engine_env(monkeypatch, engine, prob.n)
    dev = _dev(prob)
    info = dev.layout_info()
    assert info["split_a"] == (7 if engine == "split" else 0)
    assert (info["stg_a"], info["stg_at"]) == ((18, 18) if engine == "stg" else (0, 0))
    assert (info["ts_a"] > 0 and info["ts_at"] > 0) == (engine == "ts")
    lam = dev.power(1e-4, 5000).raw * 1.001
    slp = _oracle_on_device_scaling(dev, prob)
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 0.7, lam)
    dev.state_reset()
    dev.run_inner(12, 0, 0, 0.7, lam * 0.7, 2)
    for _ in range(12):
        O.iterate_once(st, slp)
    assert np.array_equal(dev.to_host("y"), st.y)
    assert np.array_equal(dev.to_host("x"), st.x)
    dev.close()


@pytest.mark.parametrize("shape", ["c1", "long_rows"])
def test_spmv_abi_bit_exact(shape):
    """hpr_spmv (the exact path's A x / A^T y) is bit-identical to the oracle's
    sequential csr_matvec on the current (unscaled) values."""
    import torch
    rng = np.random.default_rng(3)
    if shape == "c1":
        prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    else:
        a = rng.uniform(-1, 1, (30, 3000))
        a[rng.uniform(size=a.shape) < 0.5] = 0.0          # rows of ~1500 entries (long rows)
        prob = P.LpProblem.from_dense(a[:10], np.ones(10), a[10:], np.zeros(20),
                                      rng.uniform(-1, 1, 3000))
    dev = _dev(prob, 0, False, False)
    olp = O.OracleLP.from_problem(prob)
    x = rng.normal(size=olp.n)
    y = rng.normal(size=olp.m)
    with torch.cuda.stream(dev.stream):
        xd = torch.from_numpy(x).cuda()
        yd = torch.from_numpy(y).cuda()
        ax = torch.empty(olp.m, dtype=torch.float64, device="cuda")
        aty = torch.empty(olp.n, dtype=torch.float64, device="cuda")
        dev.spmv(False, xd, ax)
        dev.spmv(True, yd, aty)
    dev.stream.synchronize()
    assert np.array_equal(ax.cpu().numpy(), olp.a.matvec(x))
    assert np.array_equal(aty.cpu().numpy(), olp.transpose().matvec(y))
    dev.close()


def test_column_split_falls_back_for_very_long_block_rows(monkeypatch):
    """A row with more than 65535 entries inside one column block cannot ride
    the split layout's 16-bit slice lengths: the split is disabled and the
    unsplit SELL path (long rows summed warp-cooperatively) gives the oracle's
    bits."""
    monkeypatch.setenv("HPR_CB", "0")
    monkeypatch.setenv("HPR_STG", "0")
    monkeypatch.setenv("HPR_SPLIT_COLS", "70000")
    n = 140_000
    rng = np.random.default_rng(5)
    rows, cols, vals = [], [], []
    rows += [0] * 70_000                          # 70000 entries in block 0
    cols += list(range(0, 70_000))
    vals += rng.uniform(0.5, 1.5, 70_000).tolist()
    for i in range(1, 8):
        cc = np.sort(rng.choice(n, size=50, replace=False))
        rows += [i] * 50
        cols += cc.tolist()
        vals += rng.uniform(-1, 1, 50).tolist()
    a = P.SparseMatrix.from_coo(rows, cols, vals, (8, n))
    prob = P.LpProblem(a, P.SparseMatrix.from_coo([], [], [], (0, n)), np.ones(8), np.zeros(0),
                       rng.uniform(0, 1, n), np.zeros(n), np.full(n, 2.0))
    dev = _dev(prob)
    assert dev.layout_info()["split_a"] == 0
    lam = dev.power(1e-4, 5000).raw * 1.001
    slp = _oracle_on_device_scaling(dev, prob)
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 1.0, lam)
    dev.state_reset()
    dev.run_inner(5, 0, 0, 1.0, lam, 2)
    for _ in range(5):
        O.iterate_once(st, slp)
    assert np.array_equal(dev.to_host("y"), st.y) and np.array_equal(dev.to_host("x"), st.x)
    dev.close()


def test_scaling_and_power_vs_oracle():
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    dev = _dev(prob)
    sc_scaled, info = O.scale_lp(O.OracleLP.from_problem(prob))
    assert np.array_equal(dev.to_host("a_val_s"), sc_scaled.a.vals)
    assert np.array_equal(dev.to_host("row_scale"), info.row_scale)
    assert np.array_equal(dev.to_host("col_scale"), info.col_scale)
    for name, ref in (("b_s", sc_scaled.b), ("c_s", sc_scaled.c)):
        got = dev.to_host(name)
        assert np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))) <= 1e-15
    est = dev.power(1e-4, 5000)
    oest = O.power_lambda(sc_scaled)
    assert est.iterations == oest.iterations and bool(est.converged) == oest.converged
    assert abs(est.raw - oest.raw) <= 1e-13 * oest.raw
    # the transpose matches csr_matrix(A.T) ordering
    at = O.OracleLP.from_problem(prob).transpose()
    assert np.array_equal(dev.to_host("at_rp"), at.rp)
    assert np.array_equal(dev.to_host("at_ci"), at.ci)
    assert np.array_equal(dev.to_host("at_perm"), at.perm)


def test_c1_trajectory_vs_reference_golden():
    """Normwise 1e-10 against the reference's own first 100 iterates (its
    scaling/lambda differ from ours only through BLAS dot rounding)."""
    d = np.load(f"{GOLDEN}/c1_golden.npz")
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    dev = _dev(prob)
    lam = dev.power(1e-4, 5000).raw * 1.001
    dev.state_reset()
    done = 0
    for i, k in enumerate(d["snap_k"]):
        dev.run_inner(int(k) - done, done, done, 1.0, lam, 2)
        done = int(k)
        y, x = dev.to_host("y"), dev.to_host("x")
        ry, rx = d["snap_y"][i], d["snap_x"][i]
        rel = np.sqrt(np.sum((y - ry) ** 2) + np.sum((x - rx) ** 2)) / np.sqrt(
            np.sum(ry ** 2) + np.sum(rx ** 2))
        assert rel <= 1e-10, (k, rel)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("shape", ["ineq_only", "eq_only", "empty_rows_cols", "long_rows",
                                   "one_by_one"])
def test_edge_shapes_bit_exact(shape, engine, monkeypatch):
    rng = np.random.default_rng(7)
    if shape == "ineq_only":
        prob = P.LpProblem.from_dense(None, None, rng.uniform(-1, 1, (7, 5)), rng.uniform(-1, 0, 7),
                                      rng.uniform(0, 1, 5), upper=np.full(5, 4.0))
    elif shape == "eq_only":
        prob, _ = P.generate_known_solution_lp(11, 6, 0, 12, 0.5)
    elif shape == "empty_rows_cols":
        a = rng.uniform(-1, 1, (40, 70))
        a[rng.uniform(size=a.shape) < 0.7] = 0.0
        a[5] = 0.0
        a[:, 9] = 0.0
        a[:, 33] = 0.0
        x0 = rng.uniform(-0.5, 0.5, 70)          # feasible by construction
        prob = P.LpProblem.from_dense(a[:20], a[:20] @ x0, a[20:], a[20:] @ x0 - 0.1,
                                      rng.uniform(-1, 1, 70), lower=-np.ones(70), upper=np.ones(70))
    elif shape == "long_rows":
        # rows of 300 / 1100 / 2600 nonzeros span 2..11 chunks; one dense column
        n = 3000
        rows, cols, vals = [], [], []
        for i, ln in enumerate([300, 1100, 2600, 5, 7, 1]):
            cc = np.sort(rng.choice(n, size=ln, replace=False))
            rows += [i] * ln
            cols += cc.tolist()
            vals += rng.uniform(0.5, 2.0, ln).tolist()
        for i in range(6, 60):
            rows += [i, i]
            cols += [17, (i * 37) % n]
            vals += [1.0, -1.0]
        a = P.SparseMatrix.from_coo(rows, cols, vals, (60, n))
        dense = a.to_dense()
        x0 = rng.uniform(0.5, 1.5, n)
        prob = P.LpProblem.from_dense(dense[:30], dense[:30] @ x0, dense[30:],
                                      dense[30:] @ x0 - 0.2, rng.uniform(0, 1, n),
                                      lower=np.zeros(n), upper=np.full(n, 3.0))
    else:
        prob = one_d_problem()
    _engine_env(monkeypatch, engine, prob.n)
    dev = _dev(prob)
    if engine == "split" and prob.n >= 7:
        assert dev.layout_info()["split_a"] >= 2
    est = dev.power(1e-4, 5000)
    lam = est.raw * 1.001
    slp = _oracle_on_device_scaling(dev, prob)
    sc, _ = O.scale_lp(O.OracleLP.from_problem(prob))
    assert np.array_equal(slp.a.vals, sc.a.vals)
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 1.3, lam)
    dev.state_reset()
    dev.run_inner(60, 0, 0, 1.3, lam * 1.3, 2)
    for _ in range(60):
        O.iterate_once(st, slp)
    assert np.array_equal(dev.to_host("y"), st.y)
    assert np.array_equal(dev.to_host("x"), st.x)
    rep = P.solve(prob, P.SolverConfig(tolerance=1e-6, max_iterations=20000))
    ref = O.solve(O.OracleLP.from_problem(prob), O.OracleConfig(tolerance=1e-6, max_iterations=20000))
    assert ref["status"] == "Optimal"
    assert rep.status.value == ref["status"] and rep.iterations == ref["iterations"]
    assert _close(rep.primal_objective, ref["primal_objective"])


# ---------------------------------------------------------------------------
# solves against the reference's golden reports
# ---------------------------------------------------------------------------

def test_acceptance_suite_vs_reference(golden_reports):
    """SPEC acceptance criterion 2 instances at 1e-4 / 1e-6 / 1e-8 (60 solves)."""
    for entry in golden_reports["acceptance_suite"]:
        prob, _ = P.generate_known_solution_lp(*entry["args"])
        rep = P.solve(prob, P.SolverConfig(**entry["cfg"]))
        assert_report_parity(rep, entry["report"], str(entry["args"]) + str(entry["cfg"]["tolerance"]))
        tol = entry["cfg"]["tolerance"]
        assert max(rep.kkt.primal_infeas_rel, rep.kkt.dual_infeas_rel, rep.kkt.gap_rel) <= tol


def test_small_cases_vs_reference(golden_reports):
    """1-D, inequality-only, fixed / free variables, infeasible (iteration
    limit), MAX flip, numerical breakdown, bounded tiny LPs, degenerate LPs
    under all four variants, scaled termination space, no scaling,
    check_interval 70 with an iteration limit."""
    for case in golden_reports["small"]:
        prob = problem_from_dict(case["problem"])
        with warnings.catch_warnings(), np.errstate(all="ignore"):
            warnings.simplefilter("ignore")
            rep = P.solve(prob, P.SolverConfig(**case["cfg"]))
        assert_report_parity(rep, case["report"], case["name"], case["cfg"]["tolerance"])


def test_c1_vs_reference(golden_reports):
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    for key in ("c1", "c1_1e-8"):
        g = golden_reports[key]
        rep = P.solve(prob, P.SolverConfig(**g["cfg"]))
        assert_report_parity(rep, g["report"], key)
    d = np.load(f"{GOLDEN}/c1_golden.npz")
    rep = P.solve(prob, P.SolverConfig(tolerance=1e-4))
    assert np.allclose(rep.solution.x, d["sol_x"], rtol=1e-8, atol=1e-10)
    assert np.allclose(rep.solution.y, d["sol_y"], rtol=1e-8, atol=1e-10)
    assert np.allclose(rep.solution.z, d["sol_z"], rtol=1e-8, atol=1e-10)


def test_c2_engines_bit_identical(monkeypatch):
    """C2: the staged engine (auto-selected for the x-phase) and SELL each give
    the oracle's bits over 40 fused iterations (oracle C kernels on the
    device's scaled problem, same lambda)."""
    prob, _ = P.generate_known_solution_lp(2, 50_000, 50_000, 200_000, 2.5e-4)
    out = {}
    ref = None
    for stg in ("0", None):
        if stg is None:
            monkeypatch.delenv("HPR_STG", raising=False)
        else:
            monkeypatch.setenv("HPR_STG", stg)
        dev = _dev(prob)
        info = dev.layout_info()
        assert (info["stg_a"], info["stg_at"]) == ((0, 0) if stg == "0" else (0, 13))
        lam = dev.power(1e-4, 5000).raw * 1.001
        if ref is None:
            slp = _oracle_on_device_scaling(dev, prob)
            st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 0.9,
                         lam)
            for _ in range(40):
                O.iterate_once(st, slp)
            ref = (st.y.copy(), st.x.copy(), lam)
        assert lam == ref[2]
        dev.state_reset()
        dev.run_inner(40, 0, 0, 0.9, lam * 0.9, 2)
        out[stg] = (dev.to_host("y"), dev.to_host("x"))
        dev.close()
    for stg in ("0", None):
        assert np.array_equal(out[stg][0], ref[0]), stg
        assert np.array_equal(out[stg][1], ref[1]), stg


def test_c2_vs_reference(golden_reports):
    """C2 (m=1e5, n=2e5, nnz=5e6) at 1e-8 against the reference's report."""
    g = golden_reports["c2"]
    prob, _ = P.generate_known_solution_lp(2, 50_000, 50_000, 200_000, 2.5e-4)
    rep = P.solve(prob, P.SolverConfig(**g["cfg"]))
    assert_report_parity(rep, g["report"], "c2")
    for f in ("x", "y", "z"):
        ref = g["report"]["solution_norm"][f]
        assert abs(np.linalg.norm(getattr(rep.solution, f)) - ref) <= 1e-8 * max(1.0, ref)


def test_determinism_bit_identical():
    """SPEC acceptance criterion 10: repeated solves give identical reports."""
    for spec in acceptance_suite()[:8]:
        prob, _ = P.generate_known_solution_lp(*spec)
        a = P.solve(prob, P.SolverConfig(tolerance=1e-6))
        b = P.solve(prob, P.SolverConfig(tolerance=1e-6))
        da, db = a.to_json_dict(), b.to_json_dict()
        da.pop("timings")
        db.pop("timings")
        assert json.dumps(da, sort_keys=True) == json.dumps(db, sort_keys=True)


def test_status_paths():
    prob, _ = P.generate_known_solution_lp(12, 3, 3, 12, 0.4)
    rep = P.solve(prob, P.SolverConfig(tolerance=1e-14, time_limit_seconds=0.0,
                                       max_iterations=10**9))
    assert rep.status is P.SolveStatus.TIME_LIMIT
    rep = P.solve(one_d_problem(), P.SolverConfig(tolerance=1e-12, max_iterations=10))
    assert rep.iterations <= 10
    assert rep.status in (P.SolveStatus.ITERATION_LIMIT, P.SolveStatus.OPTIMAL)


def test_reported_point_in_box_and_cone():
    prob, pt = P.generate_known_solution_lp(2, 3, 2, 8, 0.5)
    rep = P.solve(prob, P.SolverConfig(tolerance=1e-8))
    assert rep.status is P.SolveStatus.OPTIMAL
    assert np.all(rep.solution.x >= prob.lower) and np.all(rep.solution.x <= prob.upper)
    assert np.all(rep.solution.y[prob.m1:] >= 0.0)
    assert abs(rep.primal_objective - float(prob.c @ pt.x)) <= 1e-6 * max(1.0, abs(prob.c @ pt.x))


def test_kkt_residual_vs_oracle():
    prob = bounded_tiny_lp(21, n=5, m1=2, m2=2)
    rng = np.random.default_rng(2)
    pt = P.PrimalDualPoint(y=rng.normal(size=4), z=rng.normal(size=5), x=rng.normal(size=5))
    got = P.kkt_residual(prob, pt).to_dict()
    ref = O.kkt(O.OracleLP.from_problem(prob), pt.y, pt.z, pt.x)
    for k, v in ref.items():
        assert _close(got[k], v, 1e-12), k


def test_mps_round_trip_solve_bit_for_bit():
    """reference test_mps.py:184-192 on the GPU path: a problem and its MPS
    round trip (native reader/writer) solve to identical reports and points."""
    prob, _ = P.generate_known_solution_lp(5, 4, 3, 15, 0.4)
    back = P.parse_mps(P.write_mps(prob))
    a = P.solve(prob, P.SolverConfig(tolerance=1e-8))
    b = P.solve(back, P.SolverConfig(tolerance=1e-8))
    assert a.iterations == b.iterations
    assert a.primal_objective == b.primal_objective
    assert np.array_equal(a.solution.x, b.solution.x)


def test_flow_lp_downscaled_vs_oracle():
    """C3's generator down-scaled: bit-exact iterations and a
    full solve with the reference's status / iteration count / restart
    triggers and objectives within 1e-8, against the oracle."""
    prob = P.generate_flow_lp(3, nodes=1 << 9, out_degree=4, commodities=6)
    dev = _dev(prob)
    lam = dev.power(1e-4, 5000).raw * 1.001
    slp = _oracle_on_device_scaling(dev, prob)
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 1.0, lam)
    dev.state_reset()
    dev.run_inner(80, 0, 0, 1.0, lam, 2)
    for _ in range(80):
        O.iterate_once(st, slp)
    assert np.array_equal(dev.to_host("y"), st.y)
    assert np.array_equal(dev.to_host("x"), st.x)
    cfg = dict(tolerance=1e-6, max_iterations=30000)
    rep = P.solve(prob, P.SolverConfig(**cfg))
    ref = O.solve(O.OracleLP.from_problem(prob), O.OracleConfig(**cfg))
    assert_report_parity(rep, ref, "flow_lp_downscaled")


@pytest.mark.parametrize("ts", ["0", "1", "1-slot-indices"])
def test_flow_lp_compact_many_blocks_bit_exact(ts, monkeypatch):
    """A flow LP large enough that every TS CTA walks many blocks of compact
    A^T slices (2 M columns, ~14 blocks per CTA): the cross-block look-ahead of
    the row operands and the per-block ring phases, bit-exact vs the oracle.
    Its A^T slices (one arc's 32 commodities) have lane-affine / lane-uniform
    columns, so the TS engine reads one index word per entry instead of 32
    (HPR_TS_AW=0: the slot indices, as before)."""
    monkeypatch.setenv("HPR_TS", ts[0])
    monkeypatch.setenv("HPR_TS_AW", "0" if ts.endswith("indices") else "1")
    prob = P.generate_flow_lp(5, nodes=1 << 14, out_degree=4, commodities=32)
    dev = _dev(prob)
    info = dev.layout_info()
    assert (info["ts_a"] > 0 and info["ts_at"] > 0) == (ts[0] == "1")
    if ts == "1":
        # every arc slice compressed; the K bypass columns' slice keeps its 32 words per entry
        assert 0 < info["ts_words_at"] <= info["slots_at"] // 32 + 32 * 3
        assert 0 < info["ts_words_a"] < info["slots_a"]
    else:
        assert info["ts_words_at"] == info["ts_words_a"] == 0
    lam = dev.power(1e-4, 5000).raw * 1.001
    slp = _oracle_on_device_scaling(dev, prob)
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 1.0, lam)
    dev.state_reset()
    for k in range(12):
        dev.run_inner(1, k, k, 1.0, lam, 2)
        O.iterate_once(st, slp)
        assert np.array_equal(dev.to_host("y"), st.y), k
        assert np.array_equal(dev.to_host("x"), st.x), k
    dev.close()


@pytest.mark.parametrize("smem", ["1", "0"])
def test_small_resident_loop_matches_graph_path(smem, monkeypatch):
    """The resident small-LP loop (one cluster launch per interval, default for
    C1-size LPs; slices staged in shared memory or, HPR_SMALL_SMEM=0, streamed
    from L2) and the per-iteration graph path give the same solve: same
    report, bit-identical solution."""
    monkeypatch.setenv("HPR_SMALL_SMEM", smem)
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    cfg = P.SolverConfig(tolerance=1e-8)
    reps = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("HPR_SMALL", mode)
        reps[mode] = P.solve(prob, cfg)
    a, b = reps["0"], reps["1"]
    assert a.to_json_dict(False) | {"timings": None, "device_stats": None} == \
        b.to_json_dict(False) | {"timings": None, "device_stats": None}
    for f in "xyz":
        assert np.array_equal(getattr(a.solution, f), getattr(b.solution, f))
    # one launch per interval instead of 2 x check_interval
    assert b.device_stats["launches"] < a.device_stats["launches"]


def test_time_phases_diagnostic(monkeypatch):
    """hpr_time_phases (bench.py's per-kernel roofline): both iteration kernels
    time positive; the small-LP path is reported as such."""
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    monkeypatch.setenv("HPR_SMALL", "1")
    dev = _dev(prob)
    assert dev.small_path()
    dev.close()
    monkeypatch.setenv("HPR_SMALL", "0")
    dev = _dev(prob)
    assert not dev.small_path()
    lam = dev.power(1e-4, 5000).raw * 1.001
    dev.state_reset()
    dev.run_inner(3, 0, 0, 1.0, lam, 2)
    x_us, y_us = dev.time_phases(5)
    assert x_us > 0.0 and y_us > 0.0
    dev.close()
