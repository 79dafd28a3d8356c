"""Where C4's e2e setup goes: group creation (H2D of the block), analyze,
scale, power, first interval (graph capture), checkpoint, close."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2408_12179_b200.driver import LAMBDA_SAFETY
from paper_2408_12179_b200.rowblock import RowBlockGroup, nccl_unique_id
block, m, m1, r0 = bench.c4_block(0, 1, 1_250_000, 0, None)
for rep in range(3):
    T = {}
    def tick(name, t0):
        torch.cuda.synchronize(); T[name] = round(1e3 * (time.perf_counter() - t0), 1); return time.perf_counter()
    t = time.perf_counter()
    nid = nccl_unique_id(); t = tick("nccl_id", t)
    g = RowBlockGroup.distributed(block, n=bench.C4_N, m_total=m, m1_total=m1, nnz_total=m * bench.C4_PER_ROW,
                                  row0=0, rank=0, world=1, nccl_id=nid, device=0); t = tick("upload", t)
    g.analyze(); t = tick("analyze+group", t)
    g.scale(10, True, True); t = tick("scale", t)
    est = g.power(1e-4, 5000); t = tick("power", t)
    lam = est.raw * (1 + LAMBDA_SAFETY)
    g.state_reset(); g.run_inner(150, 0, 0, 1.0, lam, 2); t = tick("interval1(capture)", t)
    g.run_inner(150, 150, 150, 1.0, lam, 2); t = tick("interval2", t)
    g.checkpoint(1.0, lam, 1, 0); t = tick("checkpoint", t)
    x = g.to_host("x"); t = tick("to_host_x", t)
    g.close(); t = tick("close", t)
    print(rep, T, flush=True)
