"""Generate golden fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --c2       # + the C2 report (about a minute)

Imports the reference package from /root/reference/pkg/src and records its
outputs; nothing here is needed at test time except the files it writes:

* ``instances.json``   -- sha256 of every array of the generator outputs for
  the benchmark seeds (pins ``paper_2408_12179_b200.generate_known_solution_lp``)
* ``reports.json``      -- reference ``SolveReport.to_json_dict(False)`` plus
  lambda/power details for the acceptance-suite instances at 3 tolerances,
  the unit-test instances and C1 (and C2 with --c2)
* ``c1_golden.npz``     -- C1: ScalingInfo, scaled problem vectors, lambda,
  (y, x) after iterations 1..100 at selected k, per-iteration norms, and the
  reference solution
* ``tiny_traces.npz``   -- full 100-iteration traces for small instances
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))

import hprlp  # noqa: E402
from hprlp.core import ProblemData, SolverState, iterate_once  # noqa: E402
from hprlp.mps import generate_degenerate_lp  # noqa: E402
from hprlp.scaling import scale_problem  # noqa: E402
from hprlp.sparse import power_method_lambda_max  # noqa: E402

SNAP_K = (1, 2, 3, 5, 10, 25, 50, 100)


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode()).hexdigest()


def problem_hash(p, pt=None):
    d = {}
    for blk in ("a_eq", "a_ineq"):
        m = getattr(p, blk)
        for f in ("row_offsets", "col_indices", "values"):
            d[f"{blk}.{f}"] = sha(np.asarray(getattr(m, f)))
    for f in ("b_eq", "b_ineq", "c", "lower", "upper"):
        d[f] = sha(getattr(p, f))
    if pt is not None:
        for f in ("x", "y", "z"):
            d[f"star.{f}"] = sha(getattr(pt, f))
    return d


def acceptance_suite():
    """reference test_acceptance.py:31-41 (criterion-2 suite)."""
    specs = []
    for i in range(20):
        n = int(np.interp(i, [0, 19], [30, 200]))
        specs.append((1000 + i, max(2, n // 4), max(1, n // 4), n, min(1.0, 25.0 / n)))
    specs[-1] = (1019, 50, 50, 200, 0.25)
    return specs


def bounded_tiny_lp(seed, n=4, m1=1, m2=2):
    """reference tests/conftest.py:13-25 (fixture instance family)."""
    rng = np.random.default_rng(seed)
    lower = rng.uniform(-2.0, 0.0, size=n)
    upper = lower + rng.uniform(1.0, 3.0, size=n)
    a = rng.uniform(-2.0, 2.0, size=(m1 + m2, n))
    a[np.abs(a) < 0.3] += 0.5
    x0 = rng.uniform(lower + 0.1, upper - 0.1)
    b_eq = a[:m1] @ x0
    b_ineq = a[m1:] @ x0 - rng.uniform(0.2, 1.0, size=m2)
    c = rng.uniform(-1.5, 1.5, size=n)
    return hprlp.LpProblem.from_dense(a[:m1], b_eq, a[m1:], b_ineq, c, lower, upper)


def dense_problem_dict(p):
    """Small instances are stored explicitly (dense blocks) in the fixtures."""
    return {"a_eq": p.a_eq.to_dense().tolist() if p.m1 else [], "b_eq": p.b_eq.tolist(),
            "a_ineq": p.a_ineq.to_dense().tolist() if p.m2 else [], "b_ineq": p.b_ineq.tolist(),
            "c": p.c.tolist(), "lower": [float(v) for v in p.lower],
            "upper": [float(v) for v in p.upper], "n": p.n,
            "objective_negated": bool(p.objective_negated),
            "objective_constant": float(p.objective_constant)}


def report(p, cfg):
    rep = hprlp.solve(p, cfg)
    d = rep.to_json_dict(include_solution=False)
    d.pop("timings")
    d["solution_sha"] = {f: sha(getattr(rep.solution, f)) for f in ("x", "y", "z")}
    d["solution_norm"] = {f: float(np.linalg.norm(getattr(rep.solution, f))) for f in ("x", "y", "z")}
    return d, rep


def cfg_dict(cfg):
    return {k: (v.value if hasattr(v, "value") else v) for k, v in cfg.__dict__.items()}


def main(with_c2=False):
    out_inst, out_rep = {}, {}
    # generator pins
    for name, args in {"c1": (1, 500, 500, 2000, 0.01), "c5_0": (10000, 250, 250, 1000, 0.01),
                       "c5_1": (10001, 250, 250, 1000, 0.01), "small": (2, 3, 2, 8, 0.5)}.items():
        p, pt = hprlp.generate_known_solution_lp(*args)
        out_inst[name] = {"args": list(args), "hash": problem_hash(p, pt)}
    # acceptance-suite reports
    suite = []
    for tol in (1e-4, 1e-6, 1e-8):
        for spec in acceptance_suite():
            p, _ = hprlp.generate_known_solution_lp(*spec)
            cfg = hprlp.SolverConfig(tolerance=tol)
            d, _ = report(p, cfg)
            suite.append({"args": list(spec), "cfg": cfg_dict(cfg), "report": d})
    out_rep["acceptance_suite"] = suite
    # explicit small instances (reference unit tests), with a few config variations
    small = []
    cases = [
        ("one_d", hprlp.LpProblem.from_dense([[1.0]], [1.0], None, None, [1.0]), {}),
        ("ineq_only", hprlp.LpProblem.from_dense(None, None, [[1.0, 1.0]], [1.0], [1.0, 1.0]), {}),
        ("fixed_var", hprlp.LpProblem.from_dense([[1.0, 1.0]], [1.0], None, None, [1.0, 0.0],
                                                 lower=[0.0, 0.25], upper=[np.inf, 0.25]), {}),
        ("free_var", hprlp.LpProblem.from_dense([[1.0]], [-2.0], None, None, [1.0],
                                                lower=[-np.inf], upper=[np.inf]), {}),
        ("infeasible", hprlp.LpProblem.from_dense([[1.0], [1.0]], [1.0, 2.0], None, None, [1.0]),
         {"max_iterations": 2000}),
        ("max_flip", hprlp.LpProblem.from_dense([[1.0]], [1.0], None, None, [-3.0],
                                                objective_negated=True), {}),
        ("breakdown", hprlp.LpProblem.from_dense([[1.0]], [1.0], None, None, [1e300],
                                                 lower=[-np.inf], upper=[np.inf]),
         {"sigma0": 1e12, "ruiz_iters": 0, "pock_chambolle": False, "bc_normalize": False,
          "max_iterations": 10000}),
    ]
    for seed in range(6):
        cases.append((f"tiny_{seed}", bounded_tiny_lp(seed, n=4, m1=1, m2=2), {}))
    for seed in range(3):
        cases.append((f"degenerate_{seed}", generate_degenerate_lp(seed), {}))
        for v in ("hdr", "hdr-fixed", "dr"):
            cases.append((f"degenerate_{seed}_{v}", generate_degenerate_lp(seed),
                          {"variant": v, "max_iterations": 60000}))
    p, _ = hprlp.generate_known_solution_lp(18, 2, 2, 8, 0.5)
    cases.append(("scaled_space", p, {"termination_space": "scaled"}))
    p, _ = hprlp.generate_known_solution_lp(17, 3, 2, 9, 0.5)
    cases.append(("no_scaling", p, {"tolerance": 1e-10, "ruiz_iters": 0, "pock_chambolle": False,
                                    "bc_normalize": False}))
    cases.append(("scaling_1e-10", p, {"tolerance": 1e-10}))
    p, _ = hprlp.generate_known_solution_lp(14, 3, 3, 12, 0.4)
    cases.append(("iter_limit", p, {"tolerance": 1e-14, "max_iterations": 400,
                                    "check_interval": 70}))
    with np.errstate(over="ignore"):
        for name, p, kw in cases:
            cfg = hprlp.SolverConfig(**kw)
            d, _ = report(p, cfg)
            small.append({"name": name, "problem": dense_problem_dict(p), "cfg": cfg_dict(cfg),
                          "report": d})
    out_rep["small"] = small

    # C1 deep fixture
    p, _ = hprlp.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    scaled, info = scale_problem(p)
    data = ProblemData.from_problem(scaled)
    est = power_method_lambda_max(data.a)
    st = SolverState.origin(data, sigma=1.0, lam=est.value)
    snaps_y, snaps_x, norms = [], [], []
    for k in range(1, 101):
        iterate_once(st, data)
        norms.append((float(np.linalg.norm(st.current.y)), float(np.linalg.norm(st.current.x))))
        if k in SNAP_K:
            snaps_y.append(st.current.y.copy())
            snaps_x.append(st.current.x.copy())
    cfg = hprlp.SolverConfig(tolerance=1e-4)
    d, rep = report(p, cfg)
    out_rep["c1"] = {"cfg": cfg_dict(cfg), "report": d, "lambda_raw": est.raw,
                     "power_iterations": est.iterations, "b_factor": info.b_norm_factor,
                     "c_factor": info.c_norm_factor}
    cfg8 = hprlp.SolverConfig(tolerance=1e-8)
    d8, _ = report(p, cfg8)
    out_rep["c1_1e-8"] = {"cfg": cfg_dict(cfg8), "report": d8}
    np.savez_compressed(
        os.path.join(HERE, "c1_golden.npz"),
        row_scale=info.row_scale, col_scale=info.col_scale,
        factors=np.array([info.b_norm_factor, info.c_norm_factor]),
        a_val_s=data.a.values, b_s=data.b, c_s=data.c, lower_s=data.lower, upper_s=data.upper,
        lam=np.array([est.value, est.raw, est.iterations]), snap_k=np.array(SNAP_K),
        snap_y=np.array(snaps_y), snap_x=np.array(snaps_x), traj_norms=np.array(norms),
        sol_x=rep.solution.x, sol_y=rep.solution.y, sol_z=rep.solution.z)

    # tiny traces (100 iterations, every iterate) for three small instances
    tr = {}
    for name, (seed, m1, m2, n, dens) in {"t0": (1003, 8, 8, 60, 0.4), "t1": (2, 3, 2, 8, 0.5),
                                           "t2": (1019, 50, 50, 200, 0.25)}.items():
        p, _ = hprlp.generate_known_solution_lp(seed, m1, m2, n, dens)
        sp_, info = scale_problem(p)
        data = ProblemData.from_problem(sp_)
        est = power_method_lambda_max(data.a)
        st = SolverState.origin(data, sigma=1.0, lam=est.value)
        ys, xs = [], []
        for _ in range(100):
            iterate_once(st, data)
            ys.append(st.current.y.copy())
            xs.append(st.current.x.copy())
        tr[f"{name}_args"] = np.array([seed, m1, m2, n, dens])
        tr[f"{name}_y"] = np.array(ys)
        tr[f"{name}_x"] = np.array(xs)
        tr[f"{name}_lam"] = np.array([est.value, est.raw])
        tr[f"{name}_a_val_s"] = data.a.values
        tr[f"{name}_vecs"] = np.concatenate([data.b, data.c, data.lower, data.upper])
    np.savez_compressed(os.path.join(HERE, "tiny_traces.npz"), **tr)

    if with_c2:
        p, pt = hprlp.generate_known_solution_lp(2, 50_000, 50_000, 200_000, 2.5e-4)
        out_inst["c2"] = {"args": [2, 50_000, 50_000, 200_000, 2.5e-4], "hash": problem_hash(p, pt)}
        cfg = hprlp.SolverConfig(tolerance=1e-8)
        rep = hprlp.solve(p, cfg)
        d = rep.to_json_dict(include_solution=False)
        d["solution_norm"] = {f: float(np.linalg.norm(getattr(rep.solution, f))) for f in ("x", "y", "z")}
        out_rep["c2"] = {"cfg": cfg_dict(cfg), "report": d}
    else:
        old = os.path.join(HERE, "reports.json")
        if os.path.exists(old):
            prev = json.load(open(old))
            if "c2" in prev:
                out_rep["c2"] = prev["c2"]
            prev_i = json.load(open(os.path.join(HERE, "instances.json")))
            if "c2" in prev_i:
                out_inst["c2"] = prev_i["c2"]

    json.dump(out_inst, open(os.path.join(HERE, "instances.json"), "w"), indent=1)
    json.dump(out_rep, open(os.path.join(HERE, "reports.json"), "w"), indent=1)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main(with_c2="--c2" in sys.argv)
