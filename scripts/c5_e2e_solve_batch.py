"""Wall time of solve_batch (C5 e2e as bench.py measures it): pack + upload +
solve + reports per call, the BatchRun of each call freed before the next."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.batch import solve_batch
import bench
probs = bench.c5_problems(0, bench.C5_COUNT)
cfg = P.SolverConfig(tolerance=1e-8)
solve_batch(probs, cfg)
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    reps = solve_batch(probs, cfg)
    dt = time.perf_counter() - t0
    its = sum(r.iterations for r in reps)
    print(f"solve_batch {1e3*dt:.1f} ms -> {its/dt:.3e} LP-it/s", flush=True)
    del reps
