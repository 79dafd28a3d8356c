"""Where the end-to-end C2 solve() time goes (host vs device)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.device import DeviceLP
from paper_2408_12179_b200.problem import stacked_arrays
prob, tol = P.generators.config_instance("c2")
cfg = P.SolverConfig(tolerance=tol)
P.solve(prob, cfg)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sa = stacked_arrays(prob); t1 = time.perf_counter()
    dev = DeviceLP(prob); torch.cuda.synchronize(); t2 = time.perf_counter()
    dev.analyze(); torch.cuda.synchronize(); t3 = time.perf_counter()
    r = P.solve(prob, cfg, dev=dev); torch.cuda.synchronize(); t4 = time.perf_counter()
    dev.close(); t5 = time.perf_counter()
    r2 = P.solve(prob, cfg); torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"stacked {1e3*(t1-t0):.1f} ms | DeviceLP (incl. stacked+pin+H2D) {1e3*(t2-t1):.1f} | analyze {1e3*(t3-t2):.1f} | solve(dev) {1e3*(t4-t3):.1f} (timings {r.timings.to_dict()}) | close {1e3*(t5-t4):.1f} | full solve() {1e3*(t6-t5):.1f} ms")
for pinned in (True, False):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev = DeviceLP(prob, pinned_upload=pinned); torch.cuda.synchronize()
    print(f"DeviceLP pinned={pinned}: {1e3*(time.perf_counter()-t0):.1f} ms"); dev.close()
