"""Time the exact T1 = 0 path (GPU) on the largest reference fixture instance
(equality-only, m1 = 1200, n = 3000, tol 1e-6); the reference takes ~1.5 s on
one host core for the same solve (tests/golden/make_exact_golden.py)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.exact import solve_equality_exact
prob, _ = P.generate_known_solution_lp(6, 1200, 0, 3000, 0.005)
for rep in range(3):
    t = time.perf_counter()
    r = solve_equality_exact(prob, P.SolverConfig(tolerance=1e-6))
    dt = time.perf_counter() - t
    print(f"rep {rep}: {r.status.value} {r.iterations} it in {dt*1e3:.1f} ms wall "
          f"({r.timings.iteration_seconds*1e3:.1f} ms iterations, {r.iterations/r.timings.iteration_seconds:.0f} it/s)")
