"""First GPU contact: parity of the fused kernels and a C1/C2 solve."""
import sys, time, os, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_12179_b200 as P
from paper_2408_12179_b200.device import DeviceLP
from oracle import hprlp_oracle as O

def compare_traj(prob, iters=100, lam=None):
    dev = DeviceLP(prob)
    dev.analyze()
    sc = dev.scale(10, True, True)
    est = dev.power(1e-4, 5000)
    lam = est.raw * (1 + 1e-3)
    # oracle on the GPU's scaled arrays
    h = {k: dev.to_host(k) for k in ("a_val_s", "b_s", "c_s", "lower_s", "upper_s")}
    olp = O.OracleLP.from_problem(prob)
    a = O.Csr(olp.a.rp, olp.a.ci, h["a_val_s"], olp.n)
    slp = O.OracleLP(a=a, b=h["b_s"], c=h["c_s"], lower=h["lower_s"], upper=h["upper_s"], m1=olp.m1)
    # oracle scaling check
    oscaled, oinfo = O.scale_lp(olp)
    print("scale: vals bit-equal", np.array_equal(oscaled.a.vals, h["a_val_s"]),
          "b rel", np.max(np.abs(oscaled.b - h["b_s"])) / max(1e-300, np.max(np.abs(oscaled.b))),
          "bf", sc.b_factor, oinfo.b_factor, "cf", sc.c_factor, oinfo.c_factor)
    oest = O.power_lambda(oscaled)
    print("power: gpu", est.raw, est.iterations, est.converged, "oracle", oest.raw, oest.iterations)
    st = O.State(y=np.zeros(slp.m), x=np.zeros(slp.n), ay=np.zeros(slp.m), ax=np.zeros(slp.n), sigma=1.0, lam=lam)
    dev.state_reset()
    worst = 0
    bitexact = True
    for k in range(iters):
        dev.run_inner(1, k, k, 1.0, lam * 1.0, 2)
        O.iterate_once(st, slp)
        gy = dev.to_host("y"); gx = dev.to_host("x")
        bitexact &= np.array_equal(gy, st.y) and np.array_equal(gx, st.x)
        rel = np.sqrt(np.sum((gy - st.y) ** 2) + np.sum((gx - st.x) ** 2)) / max(1e-300, np.sqrt(np.sum(st.y ** 2) + np.sum(st.x ** 2)))
        worst = max(worst, rel)
    print(f"trajectory {iters} it: bit-exact={bitexact} worst normwise rel={worst:.3e}")
    # graph path: 100 steps in one replay
    dev.state_reset()
    dev.run_inner(iters, 0, 0, 1.0, lam, 2)
    gy = dev.to_host("y")
    print("graph replay equals step-by-step:", np.array_equal(gy, st.y))
    dev.close()

def solve_cmp(name, prob, tol):
    t = time.time(); rep = P.solve(prob, P.SolverConfig(tolerance=tol)); t = time.time() - t
    olp = O.OracleLP.from_problem(prob)
    t2 = time.time(); orc = O.solve(olp, O.OracleConfig(tolerance=tol)); t2 = time.time() - t2
    print(f"{name}: gpu {rep.status.value} it={rep.iterations} r={rep.restarts} wall={t:.3f}s solve_s={rep.timings.solve_seconds:.4f} "
          f"| oracle {orc['status']} it={orc['iterations']} wall={t2:.2f}s")
    print("  pobj", rep.primal_objective, orc["primal_objective"], "dobj", rep.dual_objective, orc["dual_objective"])
    print("  kkt gpu", {k: f"{v:.3e}" for k, v in rep.kkt.to_dict().items()})
    print("  kkt orc", {k: f"{v:.3e}" for k, v in orc["kkt"].items()})
    print("  restarts gpu", [(e.trigger, e.tau, round(e.sigma_next, 6)) for e in rep.restart_log])
    print("  restarts orc", [(e["trigger"], e["tau"], round(e["sigma_next"], 6)) for e in orc["restart_log"]])
    print("  lam", rep.lambda_estimate, orc["lambda_estimate"], rep.device_stats)
    return rep

if __name__ == "__main__":
    print(torch.cuda.get_device_name(0))
    p1, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    compare_traj(p1)
    solve_cmp("C1", p1, 1e-4)
    solve_cmp("C1@1e-8", p1, 1e-8)
    t = time.time(); p2, _ = P.generate_known_solution_lp(2, 50_000, 50_000, 200_000, 2.5e-4); print("gen C2", time.time() - t)
    compare_traj(p2, 20)
    for i in range(2):
        t = time.time(); rep = P.solve(p2, P.SolverConfig(tolerance=1e-8)); t = time.time() - t
        print(f"C2 gpu: {rep.status.value} it={rep.iterations} wall={t:.3f}s timings={rep.timings.to_dict()} it/s={rep.iterations/rep.timings.iteration_seconds:.1f}")
    print("  restarts gpu", [(e.trigger, e.tau, round(e.sigma_next, 6)) for e in rep.restart_log])
    print("  pobj", rep.primal_objective, "kkt", rep.kkt.to_dict())
