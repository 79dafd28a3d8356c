"""Host-side breakdown of solve(problem) end to end: where the time goes.
Usage: e2e_breakdown.py [config] (default c2)."""
import os, sys, time, collections, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200 import device as D
prob, tol = P.generators.config_instance(sys.argv[1] if len(sys.argv) > 1 else "c2")
cfg = P.SolverConfig(tolerance=tol)
T = collections.defaultdict(float)
def wrap(cls, name):
    f = getattr(cls, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[name] += time.perf_counter() - t
        return r
    setattr(cls, name, g)
for nm in ("__init__", "analyze", "scale", "power", "state_reset", "run_inner", "checkpoint", "restart", "finalize", "to_host", "close", "layout_info", "launch_count", "last_times", "reload", "solution_to_host"):
    wrap(D.DeviceLP, nm)
P.solve(prob, cfg)
for rep in range(4):
    T.clear(); gc.collect()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = P.solve(prob, cfg)
    torch.cuda.synchronize(); tot = time.perf_counter() - t0
    del r; t1 = time.perf_counter(); gc.collect(); tgc = time.perf_counter() - t1
    print(f"total {tot*1e3:.1f} ms (+gc {tgc*1e3:.1f}):", {k: round(v * 1e3, 2) for k, v in sorted(T.items(), key=lambda kv: -kv[1])}, flush=True)
