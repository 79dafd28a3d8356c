"""Wall-clock phases of one solve on a resident device problem (analysis,
scaling, power method, intervals, checkpoints, finalize, solution D2H): where
the time outside the iteration kernels goes.  Usage: solve_phases.py [config]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.device import DeviceLP
from paper_2408_12179_b200.generators import config_instance

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
prob, tol = config_instance(name)
cfg = P.SolverConfig(tolerance=tol)
dev = DeviceLP(prob)
for _ in range(2):
    P.solve(prob, cfg, dev=dev)


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep_i in range(2):
    ph = {}
    dev.analyzed = False
    t = tick(); dev.analyze(); t1 = tick(); ph["analyze"] = t1 - t
    t = t1; sc = dev.scale(cfg.ruiz_iters, cfg.pock_chambolle, cfg.bc_normalize); t1 = tick(); ph["scale"] = t1 - t
    t = t1; est = dev.power(cfg.power_tol, cfg.power_max_iters); t1 = tick(); ph["power"] = t1 - t
    t = t1; dev.state_reset(); t1 = tick(); ph["state_reset"] = t1 - t
    lam = est.raw * 1.001
    ph["run_inner"] = ph["checkpoint"] = 0.0
    for i in range(31):
        t = tick(); dev.run_inner(150, 150 * i, 150 * i, 1.0, lam, 2); t1 = tick(); ph["run_inner"] += t1 - t
        t = t1; dev.checkpoint(1.0, lam, 1, i % 2); t1 = tick(); ph["checkpoint"] += t1 - t
    t = tick(); dev.finalize(1, 0); t1 = tick(); ph["finalize"] = t1 - t
    for nm in ("cand_y", "cand_z", "cand_x"):
        t = tick(); dev.to_host(nm, 0); t1 = tick(); ph["d2h_" + nm] = t1 - t
    pf = dev.prefault_solution()
    if pf is not None:
        pf.result()
    t = tick(); dev.solution_to_host(0, pf); t1 = tick(); ph["solution_to_host(prefaulted)"] = t1 - t
    t = tick(); dev.layout_info(); t1 = tick(); ph["layout_info"] = t1 - t
    print(name, {k: round(v * 1e3, 2) for k, v in ph.items()}, "total", round(sum(ph.values()) * 1e3, 1))
    torch.cuda.synchronize()
    t = time.perf_counter(); rep = P.solve(prob, cfg, dev=dev); torch.cuda.synchronize()
    print(name, "solve() wall", round((time.perf_counter() - t) * 1e3, 1), "ms,", rep.iterations, "it")
