"""C5 e2e: solve_batch wall time per 4096-LP call vs the pipeline chunk size
(PIPE_CHUNK; 4096 = one launch, no pipeline), with the device-only solve of
one launch for reference."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200 import batch as BT
from bench import c5_problems
probs = c5_problems(0, 4096)
cfg = P.SolverConfig(tolerance=1e-8)
run = BT.BatchRun(BT.PackedBatch(probs))
for _ in range(2):
    run.launch(cfg)
run.stream.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(run.stream); run.launch(cfg); e1.record(run.stream); e1.synchronize()
print(f"device one launch: {e0.elapsed_time(e1):.1f} ms")
for chunk in (4096, 2048, 1024, 512, 256):
    BT.PIPE_CHUNK = chunk
    BT.PIPE_MIN = 2048 if chunk < 4096 else 10**9
    BT.solve_batch(probs, cfg)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        reps = BT.solve_batch(probs, cfg)
        ts.append((time.perf_counter() - t) * 1e3)
    its = sum(r.iterations for r in reps)
    print(f"chunk {chunk}: " + " ".join(f"{x:.1f}" for x in ts) + f" ms  ->  {its / min(ts) * 1e3:.3e} LP-it/s")
