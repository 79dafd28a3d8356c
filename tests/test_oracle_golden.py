"""Pin the CPU oracle (oracle/hprlp_oracle.py) against fixtures produced by the
reference implementation itself (tests/golden/make_golden.py).

On the machine the fixtures were generated on the oracle reproduces the
reference bit for bit (same numpy/OpenBLAS for the dot products); elsewhere
the dot products may differ in the last bits, so floats are compared at
1e-12 relative and the discrete outputs (status, iteration counts, restart
triggers, power-method iterations) exactly.
"""

import numpy as np
import pytest

from conftest import GOLDEN, acceptance_suite, problem_from_dict
from oracle import hprlp_oracle as O
from paper_2408_12179_b200 import generate_known_solution_lp

REL = 1e-12


def close(a, b, rel=REL):
    if not (np.isfinite(a) and np.isfinite(b)):
        return (np.isnan(a) and np.isnan(b)) or a == b
    return abs(a - b) <= rel * max(1.0, abs(b))


def cfg_from(d):
    return O.OracleConfig(**d)


def assert_report_matches(r, g, rel=REL):
    assert r["status"] == g["status"]
    assert r["iterations"] == g["iterations"]
    assert r["restarts"] == g["restarts"]
    assert [e["trigger"] for e in r["restart_log"]] == [e["trigger"] for e in g["restart_log"]]
    assert [e["tau"] for e in r["restart_log"]] == [e["tau"] for e in g["restart_log"]]
    for e, f in zip(r["restart_log"], g["restart_log"]):
        assert close(e["sigma_next"], f["sigma_next"], 1e-9)
    assert close(r["primal_objective"], g["primal_objective"], rel)
    assert close(r["dual_objective"], g["dual_objective"], rel)
    for k in ("primal_infeas_rel", "dual_infeas_rel", "gap_rel"):
        assert close(r["kkt"][k], g["kkt"][k], 1e-12)
    assert r["kkt"]["dual_clamped"] == g["kkt"]["dual_clamped"]
    assert close(r["lambda_estimate"], g["lambda_estimate"], 1e-13)


def test_c1_scaling_and_lambda_pinned():
    d = np.load(f"{GOLDEN}/c1_golden.npz")
    p, _ = generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    lp = O.OracleLP.from_problem(p, use_c=False)
    scaled, info = O.scale_lp(lp)
    # max / sqrt / division are exact operations: bit-identical
    assert np.array_equal(info.row_scale, d["row_scale"])
    assert np.array_equal(info.col_scale, d["col_scale"])
    assert np.array_equal(scaled.a.vals, d["a_val_s"])
    # ||b|| + 1 goes through a BLAS dot
    assert close(info.b_factor, d["factors"][0], 1e-15)
    assert close(info.c_factor, d["factors"][1], 1e-15)
    for k in ("b_s", "c_s", "lower_s", "upper_s"):
        ref = d[k]
        got = getattr(scaled, {"b_s": "b", "c_s": "c", "lower_s": "lower", "upper_s": "upper"}[k])
        fin = np.isfinite(ref)
        assert np.array_equal(np.isfinite(got), fin)
        assert np.max(np.abs(got[fin] - ref[fin]) / np.maximum(1.0, np.abs(ref[fin]))) <= 1e-15
    est = O.power_lambda(scaled)
    assert est.iterations == int(d["lam"][2])
    assert close(est.raw, d["lam"][1], 1e-13)


def test_c1_trajectory_pinned():
    """First 100 HPR iterations on the reference's own scaled problem and lambda:
    bit-identical iterates (the SpMV order and elementwise op order match)."""
    d = np.load(f"{GOLDEN}/c1_golden.npz")
    p, _ = generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    lp = O.OracleLP.from_problem(p, use_c=False)
    a = O.Csr(lp.a.rp, lp.a.ci, d["a_val_s"], lp.n, use_c=False)
    slp = O.OracleLP(a=a, b=d["b_s"], c=d["c_s"], lower=d["lower_s"], upper=d["upper_s"], m1=lp.m1)
    st = O.State(y=np.zeros(lp.m), x=np.zeros(lp.n), ay=np.zeros(lp.m), ax=np.zeros(lp.n),
                 sigma=1.0, lam=float(d["lam"][0]))
    snaps = {int(k): i for i, k in enumerate(d["snap_k"])}
    for k in range(1, 101):
        O.iterate_once(st, slp)
        assert np.isclose(np.linalg.norm(st.y), d["traj_norms"][k - 1][0], rtol=1e-14, atol=0)
        if k in snaps:
            assert np.array_equal(st.y, d["snap_y"][snaps[k]])
            assert np.array_equal(st.x, d["snap_x"][snaps[k]])


def test_tiny_traces_pinned():
    d = np.load(f"{GOLDEN}/tiny_traces.npz")
    for name in ("t0", "t1", "t2"):
        seed, m1, m2, n, dens = d[f"{name}_args"]
        p, _ = generate_known_solution_lp(int(seed), int(m1), int(m2), int(n), float(dens))
        lp = O.OracleLP.from_problem(p, use_c=False)
        m = lp.m
        vec = d[f"{name}_vecs"]
        a = O.Csr(lp.a.rp, lp.a.ci, d[f"{name}_a_val_s"], lp.n, use_c=False)
        slp = O.OracleLP(a=a, b=vec[:m], c=vec[m:m + lp.n], lower=vec[m + lp.n:m + 2 * lp.n],
                         upper=vec[m + 2 * lp.n:], m1=lp.m1)
        st = O.State(y=np.zeros(m), x=np.zeros(lp.n), ay=np.zeros(m), ax=np.zeros(lp.n),
                     sigma=1.0, lam=float(d[f"{name}_lam"][0]))
        for k in range(100):
            O.iterate_once(st, slp)
            assert np.array_equal(st.y, d[f"{name}_y"][k]), (name, k)
            assert np.array_equal(st.x, d[f"{name}_x"][k]), (name, k)


def test_c1_full_solve_pinned(golden_reports):
    g = golden_reports["c1"]
    p, _ = generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    r = O.solve(O.OracleLP.from_problem(p, use_c=False), cfg_from(g["cfg"]))
    assert_report_matches(r, g["report"])
    assert r["power_iterations"] == g["power_iterations"]
    sol = np.load(f"{GOLDEN}/c1_golden.npz")
    assert np.allclose(r["solution"]["x"], sol["sol_x"], rtol=1e-10, atol=1e-12)
    assert np.allclose(r["solution"]["y"], sol["sol_y"], rtol=1e-10, atol=1e-12)


def test_small_cases_pinned(golden_reports):
    for case in golden_reports["small"]:
        p = problem_from_dict(case["problem"])
        with np.errstate(over="ignore", invalid="ignore"):
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                r = O.solve(O.OracleLP.from_problem(p, use_c=False), cfg_from(case["cfg"]))
        try:
            assert_report_matches(r, case["report"], rel=1e-9)
        except AssertionError as e:
            raise AssertionError(f"case {case['name']}") from e


@pytest.mark.slow
def test_acceptance_suite_pinned(golden_reports):
    suite = golden_reports["acceptance_suite"]
    for entry in suite[::3]:
        p, _ = generate_known_solution_lp(*entry["args"])
        r = O.solve(O.OracleLP.from_problem(p, use_c=False), cfg_from(entry["cfg"]))
        assert_report_matches(r, entry["report"], rel=1e-9)


def test_c_kernels_bit_identical_to_numpy_path():
    lib = O.load_clib()
    if lib is None:
        pytest.skip("oracle C kernels not built (make -C oracle)")
    p, _ = generate_known_solution_lp(1003, 8, 8, 60, 0.4)
    a = O.OracleLP.from_problem(p, use_c=False)
    b = O.OracleLP.from_problem(p, use_c=True)
    sa, _ = O.scale_lp(a)
    sb, _ = O.scale_lp(b)
    sta = O.State(np.zeros(a.m), np.zeros(a.n), np.zeros(a.m), np.zeros(a.n), 0.7, 3.0)
    stb = O.State(np.zeros(a.m), np.zeros(a.n), np.zeros(a.m), np.zeros(a.n), 0.7, 3.0)
    for _ in range(50):
        O.iterate_once(sta, sa)
        O.iterate_once(stb, sb)
    assert np.array_equal(sta.y, stb.y) and np.array_equal(sta.x, stb.x)
    x = np.random.default_rng(0).normal(size=a.n)
    assert np.array_equal(a.a.matvec(x), b.a.matvec(x))


def test_sigma_sensitivity_to_norm_order(golden_reports):
    """Why the restart sigma / merit bar is 5e-7 relative (test_gpu_parity.py
    SIGMA_REL): the reference algorithm itself, with ONLY its vector norms
    summed differently (exactly rounded fsum instead of BLAS), reproduces every
    iteration count but moves sigma_next by far more than 1e-9."""
    import math
    real = np.linalg.norm

    def fsum_norm(v, *a, **k):
        if a or k:
            return real(v, *a, **k)
        v = np.asarray(v, dtype=float).ravel()
        return math.sqrt(math.fsum(v * v))

    worst = 0.0
    entries = [e for e in golden_reports["acceptance_suite"] if e["cfg"]["tolerance"] == 1e-8]
    for entry in entries[:5]:
        prob, _ = generate_known_solution_lp(*entry["args"])
        O.np.linalg.norm = fsum_norm
        try:
            rep = O.solve(O.OracleLP.from_problem(prob), O.OracleConfig(tolerance=1e-8))
        finally:
            O.np.linalg.norm = real
        ref = entry["report"]
        assert rep["iterations"] == ref["iterations"]
        assert [e["trigger"] for e in rep["restart_log"]] == [e["trigger"] for e in ref["restart_log"]]
        for e, f in zip(rep["restart_log"], ref["restart_log"]):
            worst = max(worst, abs(e["sigma_next"] - f["sigma_next"]) / abs(f["sigma_next"]))
    assert 1e-9 < worst < 5e-7, worst
