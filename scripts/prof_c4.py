"""Per-iteration timing of the C4 row-block iteration at one rank (NCCL world
size 1); with --profile, one 2-iteration graph replay is bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off`."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2408_12179_b200.driver import LAMBDA_SAFETY
from paper_2408_12179_b200.rowblock import RowBlockGroup, nccl_unique_id

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=1_250_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
t = time.time()
block, m, m1, r0 = bench.c4_block(0, 1, a.rows, 0, None)
tg = time.time() - t
grp = RowBlockGroup.distributed(block, n=bench.C4_N, m_total=m, m1_total=m1,
                                nnz_total=m * bench.C4_PER_ROW, row0=0, rank=0, world=1,
                                nccl_id=nccl_unique_id(), device=0)
grp.analyze()
grp.scale(10, True, True)
est = grp.power(1e-4, 5000)
lam = est.raw * (1.0 + LAMBDA_SAFETY)
grp.state_reset()
grp.run_inner(150, 0, 0, 1.0, lam, 2)
torch.cuda.synchronize()
times = []
for r in range(a.reps):
    grp.run_inner(150, 150 * (r + 1), 150 * (r + 1), 1.0, lam, 2)
    torch.cuda.synchronize()
    times.append(grp.last_times()[0] / 150)
bi = bench.b_iter(a.rows, bench.C4_N, a.rows * bench.C4_PER_ROW)
print(f"c4 rows={a.rows} layout={grp.layout_info()} gen={tg:.1f}s power={est.iterations} it")
print(f"per-iteration {min(times)*1e6:.1f} us  B_iter={bi/1e9:.3f} GB -> {bi/min(times)/1e9:.1f} GB/s")
if a.profile:
    grp.run_inner(2, 0, 0, 1.0, lam, 2)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    grp.run_inner(2, 2, 2, 1.0, lam, 2)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
grp.close()
