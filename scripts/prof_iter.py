"""Per-iteration timing of the fused iteration pair (for ncu and quick roofline)."""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_12179_b200.device import DeviceLP
from paper_2408_12179_b200.generators import config_instance
from bench import b_iter

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=150)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
t = time.time(); prob, tol = config_instance(a.config); tg = time.time() - t
dev = DeviceLP(prob)
t = time.time(); dev.analyze(); dev.synchronize(); ta = time.time() - t
t = time.time(); sc = dev.scale(10, True, True); ts = time.time() - t
t = time.time(); est = dev.power(1e-4, 5000); tp = time.time() - t
lam = est.raw * 1.001
dev.state_reset()
dev.run_inner(a.steps, 0, 0, 1.0, lam, 2)   # capture + warm
dev.synchronize()
times = []
for r in range(a.reps):
    dev.run_inner(a.steps, a.steps * (r + 1), a.steps * (r + 1), 1.0, lam, 2)
    dev.synchronize()
    times.append(dev.last_times()[0])
per_it = min(times) / a.steps
bi = b_iter(dev.m, dev.n, dev.nnz)
print(f"{a.config}: m={dev.m} n={dev.n} nnz={dev.nnz} layout={dev.layout_info()} gen={tg:.1f}s analyze={ta*1e3:.1f}ms scale={ts*1e3:.1f}ms power={tp*1e3:.1f}ms ({est.iterations} it)")
print(f"per-iteration {per_it*1e6:.2f} us  (median {np.median(times)/a.steps*1e6:.2f})  B_iter={bi/1e6:.1f} MB  -> {bi/per_it/1e9:.1f} GB/s")
import subprocess
print("clocks:", subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.active", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip())
