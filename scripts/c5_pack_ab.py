import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.batch import BatchRun, PackedBatch
from paper_2408_12179_b200.device import _Staging
import bench
probs = bench.c5_problems(0, bench.C5_COUNT)
cfg = P.SolverConfig(tolerance=1e-8)
def run(staged):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with _Staging.lock:
        pk = PackedBatch(probs, staging=(lambda nb: _Staging.get(nb).numpy()) if staged else None)
        t1 = time.perf_counter()
        r = BatchRun(pk); torch.cuda.synchronize(); t2 = time.perf_counter()
        pk.arrays = {}
    r.launch(cfg); r.stream.synchronize(); t3 = time.perf_counter()
    reps = r.reports(cfg); t4 = time.perf_counter()
    return [1e3*(t1-t0), 1e3*(t2-t1), 1e3*(t3-t2), 1e3*(t4-t3), 1e3*(t4-t0)]
for i in range(6):
    for staged in (False, True):
        v = run(staged)
        print(("staged " if staged else "fresh  ") + " ".join(f"{x:7.1f}" for x in v), flush=True)
