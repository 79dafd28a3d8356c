"""Golden fixtures for the exact T1 = 0 path, produced by the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_exact_golden.py

Writes ``tests/golden/exact_golden.json`` (reports, normal-equation solves,
trace gaps) and ``tests/golden/exact_traces.npz`` (first iterations of both
no-proximal formulations), from the reference's exact.py
(``solve_equality_exact``, ``solve_normal_equations``, ``hpr_no_prox_trace``,
``halpern_padmm_trace``, ``max_trace_gap``) on the instance families of its
tests/test_exact.py plus two larger equality-only instances.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hprlp import (LpProblem, SolverConfig, generate_known_solution_lp,  # noqa: E402
                   halpern_padmm_trace, hpr_no_prox_trace, max_trace_gap,
                   solve_equality_exact, solve_normal_equations)
from hprlp.exact import DenseCholesky  # noqa: E402
from hprlp.sparse import SparseMatrix  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def report(rep):
    d = rep.to_json_dict(include_solution=False)
    d.pop("timings", None)
    d["solution_norm"] = {f: float(np.linalg.norm(getattr(rep.solution, f))) for f in "xyz"}
    return d


def main():
    out = {"reports": [], "normal": {}, "gaps": []}
    cases = [(50 + s, 3, 8, 0.8, 1e-10) for s in range(3)]
    cases += [(5, 300, 900, 0.02, 1e-8), (6, 1200, 3000, 0.005, 1e-6)]
    for seed, m1, n, dens, tol in cases:
        prob, pt = generate_known_solution_lp(seed, m1=m1, m2=0, n=n, density=dens)
        t = time.time()
        rep = solve_equality_exact(prob, SolverConfig(tolerance=tol))
        print(f"seed {seed} m1 {m1} n {n}: {rep.status.value} {rep.iterations} it "
              f"{time.time() - t:.1f}s", flush=True)
        out["reports"].append({"gen": [seed, m1, n, dens], "tol": tol, "report": report(rep),
                               "planted_obj": float(prob.c @ pt.x)})
    for variant in ("dr", "hdr", "hdr-fixed"):
        prob, _ = generate_known_solution_lp(51, m1=3, m2=0, n=8, density=0.8)
        rep = solve_equality_exact(prob, SolverConfig(tolerance=1e-8, variant=variant))
        out["reports"].append({"gen": [51, 3, 8, 0.8], "tol": 1e-8, "variant": variant,
                               "report": report(rep), "planted_obj": None})
    rng = np.random.default_rng(0)
    dense = rng.normal(size=(5, 9))
    chol = DenseCholesky.from_matrix(SparseMatrix.from_dense(dense))
    rhs = rng.normal(size=5)
    out["normal"] = {"dense": dense.tolist(), "rhs": rhs.tolist(),
                     "y": solve_normal_equations(chol, rhs).tolist()}
    one = LpProblem.from_dense([[1.0]], [1.0], None, None, [1.0])
    out["gaps"].append({"case": "one_d", "sigma": 1.0, "iters": 20,
                        "gap": max_trace_gap(one, 1.0, 20)})
    for seed, m1, n, sigma, iters in [(11, 3, 6, 0.37, 50), (13, 2, 5, 0.25, 40),
                                      (13, 2, 5, 1.0, 40), (13, 2, 5, 3.5, 40)]:
        prob, _ = generate_known_solution_lp(seed, m1=m1, m2=0, n=n, density=0.8)
        out["gaps"].append({"case": [seed, m1, n], "sigma": sigma, "iters": iters,
                            "gap": max_trace_gap(prob, sigma, iters)})
    arrs = {}
    prob, _ = generate_known_solution_lp(7, m1=3, m2=0, n=7, density=0.8)
    d = hpr_no_prox_trace(prob, 0.9, 12)
    a = halpern_padmm_trace(prob, 0.9, 12)
    for f in ("y", "z", "x_half", "x_tilde"):
        arrs[f"direct_{f}"] = np.array(getattr(d, f))
    for f in ("y", "z", "x"):
        arrs[f"avg_{f}"] = np.array(getattr(a, f))
    prob, _ = generate_known_solution_lp(17, m1=2, m2=0, n=6, density=0.8)
    r3 = np.random.default_rng(3)
    y0, x0 = r3.normal(size=2), r3.normal(size=6)
    d = hpr_no_prox_trace(prob, 0.8, 30, y0=y0, x0=x0)
    arrs["nz_y0"], arrs["nz_x0"] = y0, x0
    arrs["nz_direct_y"] = np.array(d.y)
    arrs["nz_direct_x_half"] = np.array(d.x_half)
    np.savez_compressed(os.path.join(HERE, "exact_traces.npz"), **arrs)
    with open(os.path.join(HERE, "exact_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote exact_golden.json, exact_traces.npz")


if __name__ == "__main__":
    main()
