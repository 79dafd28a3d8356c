"""solve_batch phases in the bench's setting (a device-timed BatchRun alive,
previous reports kept), with and without the cyclic GC during the call."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.batch import BatchRun, PackedBatch
from paper_2408_12179_b200.device import _Staging
import bench
probs = bench.c5_problems(0, bench.C5_COUNT)
cfg = P.SolverConfig(tolerance=1e-8)
run0 = BatchRun(PackedBatch(probs))
for _ in range(3):
    run0.launch(cfg)
reps = run0.reports(cfg)
pk = PackedBatch(probs)


def phases():
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with _Staging.lock:
        packed = PackedBatch(probs, staging=lambda nb: _Staging.get(nb).numpy())
        t1 = time.perf_counter()
        run = BatchRun(packed)
        t2 = time.perf_counter()
        packed.arrays = {}
    run.launch(cfg); run.stream.synchronize(); t3 = time.perf_counter()
    out = run.reports(cfg); t4 = time.perf_counter()
    return out, [1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t4 - t0)]


for nogc in (False, True, False, True):
    for _ in range(3):
        if nogc:
            gc.disable()
        try:
            reps, v = phases()
        finally:
            gc.enable()
        print(("nogc " if nogc else "gc   ") + " ".join(f"{x:7.1f}" for x in v), flush=True)
