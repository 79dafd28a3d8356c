import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200 import driver as D
from paper_2408_12179_b200.device import DeviceLP
prob, tol = P.generators.config_instance("c2")
cfg = P.SolverConfig(tolerance=tol)
P.solve(prob, cfg)
dev = D.DEVICE_POOL.free[0]
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); dev.reload(prob); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"reload {1e3*(t1-t):.2f} ms")
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); rep = P.solve(prob, cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"solve e2e {1e3*(t1-t):.2f} ms, iterations {rep.iterations}")
