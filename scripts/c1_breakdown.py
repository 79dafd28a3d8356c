"""C1 solve breakdown: the report's wall-clock phase timings and device
iteration time, over repeated solves on a resident device problem."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.device import DeviceLP
from paper_2408_12179_b200.generators import config_instance
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
prob, tol = config_instance(name)
cfg = P.SolverConfig(tolerance=tol)
dev = DeviceLP(prob)
for _ in range(3):
    P.solve(prob, cfg, dev=dev)
for _ in range(3):
    dev.analyzed = False
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = P.solve(prob, cfg, dev=dev)
    wall = time.perf_counter() - t
    tm = rep.timings
    ds = rep.device_stats
    print(f"{name}: {rep.iterations} it, wall {wall*1e3:.2f} ms | " +
          " ".join(f"{k}={getattr(tm, k)*1e3:.2f}" for k in tm.__dataclass_fields__) +
          f" | device_iteration {ds['device_iteration_seconds']*1e3:.2f} ms "
          f"({ds['device_iteration_seconds']/rep.iterations*1e6:.2f} us/it), launches {ds['launches']}")
