"""Time the C5 batch (4096 LPs m=500 n=1000 nnz=5000) on one GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.batch import BatchRun, PackedBatch
count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
t = time.time()
probs = [P.generate_known_solution_lp(10_000 + i, 250, 250, 1000, 0.01)[0] for i in range(count)]
print(f"gen {count} LPs: {time.time()-t:.1f}s", flush=True)
pk = PackedBatch(probs)
run = BatchRun(pk)
cfg = P.SolverConfig(tolerance=1e-8)
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(run.stream); run.launch(cfg); e1.record(run.stream); e1.synchronize()
    ms = e0.elapsed_time(e1)
    reps = run.reports(cfg)
    its = sum(r.iterations for r in reps)
    st = {}
    for r in reps: st[r.status.value] = st.get(r.status.value, 0) + 1
    print(f"rep {rep}: {ms:.2f} ms for {count} LPs, {its} LP-iterations -> {its/ms*1e3:.3e} LP-it/s, {count/ms*1e3:.1f} LP/s, status {st}", flush=True)
