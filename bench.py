#!/usr/bin/env python
"""Benchmark of the HPR-LP iteration loop on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c3-lite]

A step is one full solve of the configuration to its tolerance (C2: 1e-8)
starting from a problem already resident in HBM (setup = transpose/tiling,
scaling and power method are inside the step).  ``value`` = HPR iterations per
second over the K timed steps (sum over ranks; each rank solves its own replica
-- the C2 path fits one GPU, so N > 1 is weak scaling of independent solves).
``e2e`` = the same metric through the public ``solve()`` call on a host
problem, with the pinned H2D upload and the D2H of the solution inside the
timed region.  ``roofline`` is the fused x-phase + y-phase iteration pair
against the measured HBM copy bandwidth, algorithmic bytes per iteration
B_iter = 24 nnz + 4 (m + n + 2) + 8 (5 m + 8 n).

``--impl reference`` times the CPU oracle port (oracle/, the reference's
algorithm restated with sequential-order C kernels; OpenMP over all host
cores) on the same instance: each step is one 150-iteration interval.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_NAMES = {"c1": "C1: known-solution LP m=1000 n=2000 nnz=20000, tol 1e-4",
                "c2": "C2: known-solution LP m=100000 n=200000 nnz=5000000, tol 1e-8",
                "c3": "C3: multicommodity flow V=2^18 E=2^20 K=32 (nnz ~1.0e8), tol 1e-8",
                "c3-lite": "C3-lite: multicommodity flow V=2^10 K=8, tol 1e-8"}


def b_iter(m, n, nnz):
    return 24 * nnz + 4 * (m + n + 2) + 8 * (5 * m + 8 * n)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_instance(name):
    from paper_2408_12179_b200.generators import config_instance
    return config_instance(name)


def cpu_baseline_sample(prob, tol, iters=300):
    """Oracle (C kernels, all host threads) on the same instance: setup once,
    then `iters` HPR iterations timed; it/s."""
    from oracle import hprlp_oracle as O
    lib = O.load_clib()
    threads = lib.orc_set_threads(os.cpu_count() or 1) if lib is not None else 1
    lp = O.OracleLP.from_problem(prob)
    scaled, _ = O.scale_lp(lp)
    est = O.power_lambda(scaled)
    st = O.State(y=np.zeros(scaled.m), x=np.zeros(scaled.n), ay=np.zeros(scaled.m),
                 ax=np.zeros(scaled.n), sigma=1.0, lam=est.value)
    O.iterate_once(st, scaled)  # warm
    t0 = time.perf_counter()
    for _ in range(iters):
        O.iterate_once(st, scaled)
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "it/s", "cores": threads,
            "kind": "port" if lib is None else "port",
            "sample": f"{iters} HPR iterations of the same instance (oracle C kernels, "
                      f"sequential per-row sums, OpenMP {threads} threads), setup excluded"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import hprlp_oracle as O
    prob, tol = make_instance(args.config)
    lib = O.load_clib()
    threads = lib.orc_set_threads(os.cpu_count() or 1) if lib is not None else 1
    lp = O.OracleLP.from_problem(prob)
    scaled, _ = O.scale_lp(lp)
    est = O.power_lambda(scaled)
    st = O.State(y=np.zeros(scaled.m), x=np.zeros(scaled.n), ay=np.zeros(scaled.m),
                 ax=np.zeros(scaled.n), sigma=1.0, lam=est.value)
    interval = 150

    def step():
        for _ in range(interval):
            O.iterate_once(st, scaled)
        O.half_step(st, scaled)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    its = interval * args.steps
    val = its / dt
    line = {"metric": "hpr_iterations_per_sec", "value": val, "unit": "it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": CONFIG_NAMES[args.config], "tolerance": tol,
                       "step": f"{interval} HPR iterations + 1 half step (oracle port)"},
            "cpu_baseline": {"value": val, "unit": "it/s", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} x {interval} iterations"},
            "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import paper_2408_12179_b200 as P
    from paper_2408_12179_b200.device import DeviceLP

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prob, tol = make_instance(args.config)
    cfg = P.SolverConfig(tolerance=tol)
    dev = DeviceLP(prob, device=local)
    m, n, nnz = dev.m, dev.n, dev.nnz
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    # warmup (also builds the graphs)
    for _ in range(args.warmup):
        P.solve(prob, cfg, dev=dev)
    sample_clocks = ClockSampler(local)
    total_ms = 0.0
    its_total = 0
    iter_s_total = 0.0
    reps = []
    l0 = dev.launch_count()
    barrier()
    with sample_clocks:
        for _ in range(args.steps):
            flush.zero_()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            dev.stream.synchronize()
            ev0.record(dev.stream)
            rep = P.solve(prob, cfg, dev=dev)
            ev1.record(dev.stream)
            ev1.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            its_total += rep.iterations
            iter_s_total += rep.timings.iteration_seconds
            reps.append(rep)
    barrier()
    launches = dev.launch_count() - l0
    t_local = total_ms / 1e3
    t_max = t_local
    its_all = its_total
    if dist is not None:
        tt = torch.tensor([t_local, float(its_total)], dtype=torch.float64, device=f"cuda:{local}")
        tmax = tt.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        t_max, its_all = float(tmax[0]), float(tt[1])
    value = its_all / t_max

    # e2e through the public API from host arrays (upload + solve + D2H solution)
    e2e_its, e2e_t = 0, 0.0
    h2d = d2h = 0
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.solve(prob, cfg, device=local)
        torch.cuda.synchronize()
        e2e_t += time.perf_counter() - t0
        e2e_its += rep.iterations
        h2d = rep.device_stats["h2d_bytes"]
        d2h = 8 * (2 * n + m)
    e2e_val = e2e_its / e2e_t
    if dist is not None:
        tt = torch.tensor([e2e_val], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        e2e_val = float(tt[0])

    peak, peak_kind = load_peaks()
    bi = b_iter(m, n, nnz)
    achieved = bi * its_total / iter_s_total / 1e9
    line = None
    if rank == 0:
        r0 = reps[-1]
        cpu = cpu_baseline_sample(prob, tol) if ws == 1 and not args.no_cpu else None
        line = {
            "metric": "hpr_iterations_per_sec", "value": value, "unit": "it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "tolerance": tol, "m": m, "n": n,
                       "nnz": nnz, "step": "one full solve to tolerance from HBM-resident input",
                       "status": r0.status.value, "iterations_per_solve": r0.iterations,
                       "wall_time_to_tol_s": t_max / args.steps,
                       "l2": "256 MB buffer written between timed steps (flush)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "k_x_iter + k_y_iter (one HPR iteration)",
                         "bytes_per_iteration": bi, "peak_source": peak_kind},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "it/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": sample_clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIG_NAMES), default="c2")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
