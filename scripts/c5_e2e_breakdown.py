"""Host-side breakdown of solve_batch (C5 e2e): pack / upload+setup / solve / reports."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.batch import BatchRun, PackedBatch
import bench
probs = bench.c5_problems(0, bench.C5_COUNT)
cfg = P.SolverConfig(tolerance=1e-8)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pk = PackedBatch(probs); t1 = time.perf_counter()
    run = BatchRun(pk); torch.cuda.synchronize(); t2 = time.perf_counter()
    run.launch(cfg); run.stream.synchronize(); t3 = time.perf_counter()
    reps = run.reports(cfg); t4 = time.perf_counter()
    print(f"pack {1e3*(t1-t0):.1f} ms, upload+alloc {1e3*(t2-t1):.1f} ms, solve {1e3*(t3-t2):.1f} ms, "
          f"reports {1e3*(t4-t3):.1f} ms, total {1e3*(t4-t0):.1f} ms", flush=True)
from paper_2408_12179_b200.batch import solve_batch
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    reps = solve_batch(probs, cfg)
    print(f"solve_batch (pack into pinned staging + upload + solve + reports) {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
