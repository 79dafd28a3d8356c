#!/usr/bin/env python
"""Benchmark of the HPR-LP iteration loop on B200 (contract: DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c3-lite|c4|c5]

c1/c2/c3 (default c2 = BASELINE configs[1], the headline): a step is one full
solve to tolerance (C2: 1e-8) from a problem already resident in HBM (setup =
transpose/layout, scaling and power method are inside the step).  ``value`` =
HPR iterations per second; at N > 1 every rank solves its own replica
(independent objects, no collective: C2 fits one GPU) -- weak scaling.

c4: the row-block partitioned path: each rank owns
``--c4-rows`` rows x 100 nnz of a planted LP with n = 20M columns, generated
per rank; the A^T y partials are reduce-scattered and w all-gathered over
NCCL every iteration.  A step = one 150-iteration interval + checkpoint.
Weak scaling (rows per rank fixed; N = 8 is C4's 1e9 nnz).

c5: a batch of 4096 LPs (m=500, n=1000, nnz=5000), one whole solve per CTA,
sharded across ranks (no collective).  A step = the whole shard solved to
1e-8.  ``value`` = LP-iterations per second summed over ranks.

``e2e`` = the same metric through the public API (``solve`` /
``solve_batch`` / ``solve_distributed``) on host data, with the H2D upload and
the D2H of the solution inside the timed region.  ``roofline`` is the fused
x-phase + y-phase iteration pair against the measured HBM copy bandwidth,
B_iter = 24 nnz + 4 (m + n + 2) + 8 (5 m + 8 n) bytes per iteration.

``--impl reference`` times the CPU oracle port (oracle/: the reference
algorithm with sequential-order C kernels; OpenMP over all host cores, or a
process pool for c5) on the same instance -- the reference is pure Python, so
there is no compiled oracle/_ref.
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
                "c3-lite": "C3-lite: multicommodity flow V=2^10 K=8, tol 1e-8",
                "c4": "C4: planted LP row-block partitioned over N GPUs, n=2e7, 100 nnz/row",
                "c5": "C5: batch of 4096 LPs m=500 n=1000 nnz=5000, one per CTA, tol 1e-8"}
C4_N = 20_000_000
C4_PER_ROW = 100
C5_COUNT = 4096


def b_iter(m, n, nnz):
    return 24 * nnz + 4 * (m + n + 2) + 8 * (5 * m + 8 * n)


def load_traffic(config):
    """ncu DRAM bytes (read + write) of the x-phase + y-phase pair per iteration,
    from the committed capture summary (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        v = d.get(config)
        return None if v is None else float(v["bytes_per_iteration"])
    return None


def iteration_kernels(lay):
    """Names of the two iteration kernels the layout selected."""
    x = "k_stg<EpiXIter>" if lay.get("stg_at") else "k_sell<EpiXIter>"
    if lay.get("stg_a"):
        y = "k_stg<EpiYIter>"
    elif lay.get("split_a"):
        y = f"{lay['split_a']} x k_sell<EpiCarry..> (column-split)"
    else:
        y = "k_sell<EpiYIter>"
    return f"{x} + {y} (one HPR iteration)"


def gather_roofline(nnz, iterations, seconds, lay=None):
    """Operand gathers per second against one L1TEX wavefront per cycle per SM
    (148 SMs at the max SM clock): nnz gathers per HPR iteration for each phase
    on the SELL engine (a staged phase gathers from shared memory); None when
    both phases are staged."""
    import torch
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    mhz = float(json.load(open(p)).get("sm_max_mhz", 1965.0)) if os.path.exists(p) else 1965.0
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    peak = sms * mhz * 1e6
    lay = lay or {}
    sell_phases = int(not lay.get("stg_at")) + int(not lay.get("stg_a"))
    if sell_phases == 0:
        return None
    achieved = sell_phases * nnz * iterations / seconds
    note = (f"{sell_phases}*nnz random fp64 operand gathers from L2 per iteration, 1 L1TEX "
            "wavefront each")
    if sell_phases == 1:
        note += ("; the other phase runs on the staged engine (gathers from shared memory), "
                 "so this rate is over the whole iteration time: a lower bound")
    return {"bound": "l1tex", "achieved": achieved, "peak": peak, "unit": "gathers/s",
            "frac": achieved / peak, "note": note}


def smem_roofline(probs, lp_its_per_s):
    """C5: the batch kernel works out of each SM's shared memory (the LP is
    staged once per solve), so its bound is the shared-memory port, 128 B per
    cycle per SM.  Algorithmic shared-memory bytes per LP-iteration: A and A^T
    values + 16-bit columns (10 B per nonzero each) and one 8-byte operand
    gather per nonzero in each phase, plus the x-phase's 7 and the y-phase's 4
    n / m-vector accesses (x, anchor, c, l, u read, w, x written; y, anchor, b
    read, y written)."""
    import torch
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    mhz = float(json.load(open(p)).get("sm_max_mhz", 1965.0)) if os.path.exists(p) else 1965.0
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    m = sum(q.m for q in probs) / len(probs)
    n = sum(q.n for q in probs) / len(probs)
    nnz = sum(q.a_eq.nnz + q.a_ineq.nnz for q in probs) / len(probs)
    per_it = 2 * nnz * (10 + 8) + 8 * (7 * n + 4 * m)
    peak = sms * 128 * mhz * 1e6 / 1e9
    achieved = per_it * lp_its_per_s / 1e9
    return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None,
            "kernel": "k_batch_solve (whole solve per CTA, LP resident in shared memory)",
            "bytes_per_lp_iteration": per_it,
            "peak_source": "148 SMs x 128 B/cycle x max SM clock (architectural)"}


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


def c5_problems(lo, hi):
    from paper_2408_12179_b200.generators import generate_known_solution_lp
    return [generate_known_solution_lp(10_000 + i, 250, 250, 1000, 0.01)[0] for i in range(lo, hi)]


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU reference arm / cpu_baseline (the oracle port; test infrastructure)
# ---------------------------------------------------------------------------

def _oracle_setup(prob, power_max=5000):
    from oracle import hprlp_oracle as O
    lib = O.load_clib()
    threads = lib.orc_set_threads(cpu_threads()) if lib is not None else 1
    lp = O.OracleLP.from_problem(prob)
    scaled, _ = O.scale_lp(lp)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")        # a capped power method (C4 sample) warns
        est = O.power_lambda(scaled, max_iters=power_max)
    st = O.State(y=np.zeros(scaled.m), x=np.zeros(scaled.n), ay=np.zeros(scaled.m),
                 ax=np.zeros(scaled.n), sigma=1.0, lam=est.value)
    return O, scaled, st, threads


def cpu_baseline_sample(prob, iters=300):
    """Oracle C kernels (all host threads) on the same instance: setup once,
    then ``iters`` HPR iterations timed; it/s."""
    O, scaled, st, threads = _oracle_setup(prob)
    O.iterate_once(st, scaled)  # warm
    t0 = time.perf_counter()
    for _ in range(iters):
        O.iterate_once(st, scaled)
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"{iters} HPR iterations of the same instance (oracle C kernels, "
                      f"sequential per-row sums, OpenMP {threads} threads), setup excluded"}


def _c5_worker(i):
    from oracle import hprlp_oracle as O
    lib = O.load_clib()
    if lib is not None:
        lib.orc_set_threads(1)
    prob = c5_problems(i, i + 1)[0]
    t0 = time.perf_counter()
    rep = O.solve(O.OracleLP.from_problem(prob), O.OracleConfig(tolerance=1e-8))
    return rep["iterations"], time.perf_counter() - t0


def c5_cpu_sample(count):
    """``count`` C5 LPs solved by the oracle in a process pool over all cores;
    LP-iterations per second of wall time."""
    import multiprocessing as mp
    cores = cpu_threads()
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(min(cores, count)) as pool:
        out = pool.map(_c5_worker, range(count))
    dt = time.perf_counter() - t0
    its = sum(o[0] for o in out)
    return {"value": its / dt, "unit": "LP-it/s", "cores": min(cores, count), "kind": "port",
            "sample": f"{count} of the 4096 C5 LPs solved to 1e-8 by the oracle (one LP per "
                      f"process, {min(cores, count)} processes), wall time incl. setup"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    base = {"metric": "hpr_iterations_per_sec", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference"}
    if args.config == "c5":
        cnt = max(cpu_threads(), 16)
        vals = []
        for _ in range(args.steps):
            vals.append(c5_cpu_sample(cnt))
        val = statistics.median(v["value"] for v in vals)
        cb = dict(vals[0], value=val)
        line = dict(base, metric="hpr_lp_iterations_per_sec", value=val, unit="LP-it/s",
                    ms_per_step=None,
                    config={"workload": CONFIG_NAMES["c5"], "tolerance": 1e-8,
                            "step": cb["sample"]},
                    cpu_baseline=cb,
                    e2e={"value": val, "unit": "LP-it/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return
    if args.config == "c4":
        from paper_2408_12179_b200.generators import generate_planted_block
        rows = args.c4_rows
        m1 = rows // 2
        rp, ci, va, b, ys, m1l, (lo, up, xs, zs), cpart = generate_planted_block(
            4, m1, rows - m1, C4_N, C4_PER_ROW, 0, rows)
        prob = c4_lp((rp, ci, va, m1l, b, cpart + zs, lo, up), rows, m1)
        interval = 2
        tol = 1e-8
        power_max = 3          # per-iteration time does not depend on lambda's accuracy
    else:
        prob, tol = make_instance(args.config)
        interval = 150
        power_max = 5000
    O, scaled, st, threads = _oracle_setup(prob, power_max)

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
    val = interval * args.steps / dt
    line = dict(base, value=val, unit="it/s", ms_per_step=1e3 * dt / args.steps,
                config={"workload": CONFIG_NAMES[args.config], "tolerance": tol,
                        "step": f"{interval} HPR iterations + 1 half step (oracle port)"},
                cpu_baseline={"value": val, "unit": "it/s", "cores": threads, "kind": "port",
                              "sample": f"{args.steps} x {interval} iterations + half step"},
                e2e={"value": val, "unit": "it/s", "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": 0})
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _dist_init(ws, local):
    import torch
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist
    return None


def _max_sum(dist, local, t_local, count):
    """(max over ranks of t_local, sum over ranks of count)."""
    if dist is None:
        return t_local, count
    import torch
    tt = torch.tensor([t_local, float(count)], dtype=torch.float64, device=f"cuda:{local}")
    tmax = tt.clone()
    dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
    dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
    return float(tmax[0]), float(tt[1])


def _finish(dist, line, rank):
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = _dist_init(ws, local)
    if args.config == "c5":
        return run_c5(args, dist, ws, rank, local)
    if args.config == "c4":
        return run_c4(args, dist, ws, rank, local)
    import paper_2408_12179_b200 as P
    from paper_2408_12179_b200.device import DeviceLP

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

    for _ in range(args.warmup):             # also builds the graphs
        P.solve(prob, cfg, dev=dev)
    sample_clocks = ClockSampler(local)
    total_ms = 0.0
    its_total = 0
    iter_s_total = 0.0
    pair_ms = []
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
    t_max, its_all = _max_sum(dist, local, total_ms / 1e3, its_total)
    value = its_all / t_max

    # e2e through the public API from host arrays: every step uploads the
    # problem (pinned staging -> H2D), re-analyses it, solves and copies the
    # solution back; one untimed call first warms the device-residency pool
    e2e_its, e2e_t = 0, 0.0
    h2d = d2h = 0
    P.solve(prob, cfg, device=local)
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.solve(prob, cfg, device=local)
        torch.cuda.synchronize()
        e2e_t += time.perf_counter() - t0
        e2e_its += rep.iterations
        h2d = rep.device_stats["h2d_bytes"]
        d2h = 8 * (2 * n + m)
    t_e2e, its_e2e = _max_sum(dist, local, e2e_t, e2e_its)
    e2e_val = its_e2e / t_e2e

    peak, peak_kind = load_peaks()
    bi = b_iter(m, n, nnz)
    achieved = bi * its_total / iter_s_total / 1e9
    line = None
    if rank == 0:
        r0 = reps[-1]
        lay = r0.device_stats.get("layout", {})
        cpu = cpu_baseline_sample(prob) if ws == 1 and not args.no_cpu else None
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
                         "frac": achieved / peak,
                         "traffic": args.traffic if args.traffic is not None
                         else load_traffic(args.config),
                         "kernel": iteration_kernels(lay),
                         "bytes_per_iteration": bi, "peak_source": peak_kind,
                         "timing": "CUDA events around each 150-iteration graph replay"},
            # the bound that actually binds a small-n problem (C2): every nonzero
            # is one random 8-byte operand gather = one L1TEX wavefront per cycle per SM
            # (phases on the staged engine gather from shared memory instead)
            "roofline_gather": gather_roofline(nnz, its_total, iter_s_total, lay),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "it/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": sample_clocks.summary(),
        }
    _finish(dist, line, rank)
    return line


def run_c5(args, dist, ws, rank, local):
    import torch
    import paper_2408_12179_b200 as P
    from paper_2408_12179_b200.batch import BatchRun, PackedBatch, shard_bounds, solve_batch
    lo, hi = shard_bounds(C5_COUNT, ws, rank)
    probs = c5_problems(lo, hi)
    cfg = P.SolverConfig(tolerance=1e-8)
    run = BatchRun(PackedBatch(probs), device=local)
    for _ in range(args.warmup):
        run.launch(cfg)
    run.stream.synchronize()
    sample_clocks = ClockSampler(local)
    total_ms, its = 0.0, 0
    l0 = run.launches
    with sample_clocks:
        for _ in range(args.steps):
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(run.stream)
            run.launch(cfg)
            ev1.record(run.stream)
            ev1.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            reps = run.reports(cfg)
            its += sum(r.iterations for r in reps)
    launches = run.launches - l0
    t_max, its_all = _max_sum(dist, local, total_ms / 1e3, its)
    value = its_all / t_max
    st = {}
    for r in reps:
        st[r.status.value] = st.get(r.status.value, 0) + 1
    # e2e: solve_batch on host problems (pack + upload + solve + D2H of every
    # report); one untimed call first (device allocations, like run_ours)
    e2e_t, e2e_its = 0.0, 0
    pk = PackedBatch(probs)
    solve_batch(probs, cfg, device=local)
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = solve_batch(probs, cfg, device=local)
        e2e_t += time.perf_counter() - t0
        e2e_its += sum(r.iterations for r in reps)
    t_e2e, its_e2e = _max_sum(dist, local, e2e_t, e2e_its)
    line = None
    if rank == 0:
        cpu = c5_cpu_sample(max(cpu_threads(), 16)) if ws == 1 and not args.no_cpu else None
        line = {
            "metric": "hpr_lp_iterations_per_sec", "value": value, "unit": "LP-it/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": CONFIG_NAMES["c5"], "tolerance": 1e-8,
                       "lps_per_rank": hi - lo, "lps_total": C5_COUNT,
                       "step": "the rank's shard solved to 1e-8 in one launch (one LP per CTA)",
                       "status": st, "l2": "inputs re-read from HBM each step (490 MB > L2)",
                       "parallelism": f"batch sharded x{ws}" if ws > 1 else "single GPU"},
            "roofline": smem_roofline(probs, value),
            "cpu_baseline": cpu,
            "e2e": {"value": its_e2e / t_e2e, "unit": "LP-it/s",
                    "h2d_bytes_per_step": pk.h2d_bytes(),
                    "d2h_bytes_per_step": 8 * int(pk.row_off[-1] + 2 * pk.col_off[-1])},
            "gpu_launches": launches,
            "clocks": sample_clocks.summary(),
        }
    _finish(dist, line, rank)
    return line


def c4_block(rank, ws, rows_per_rank, local, dist):
    """This rank's rows of the weak-scaled C4 instance + the global cost vector."""
    import torch
    from paper_2408_12179_b200.generators import _planted_columns, generate_planted_block
    m = rows_per_rank * ws
    m1 = m // 2
    cols = _planted_columns(4, C4_N)
    r0, r1 = rank * rows_per_rank, (rank + 1) * rows_per_rank
    rp, ci, va, b, ys, m1l, (lo, up, xs, zs), cpart = generate_planted_block(
        4, m1, m - m1, C4_N, C4_PER_ROW, r0, r1, cols)
    if dist is not None:
        t = torch.from_numpy(cpart).to(f"cuda:{local}")
        dist.all_reduce(t)
        cpart = t.cpu().numpy()
    c = cpart + zs
    return (rp, ci, va, m1l, b, c, lo, up), m, m1, r0


def c4_lp(block, m, m1):
    """The one-rank C4 block (rows [0, m), the first m1 equalities) as an LpProblem."""
    from paper_2408_12179_b200 import LpProblem, SparseMatrix
    rp, ci, va, _m1l, b, c, lo, up = block
    return LpProblem(a_eq=SparseMatrix.from_csr_arrays(rp[:m1 + 1], ci[:rp[m1]], va[:rp[m1]], m1, C4_N),
                     a_ineq=SparseMatrix.from_csr_arrays(rp[m1:] - rp[m1], ci[rp[m1]:], va[rp[m1]:],
                                                         m - m1, C4_N),
                     b_eq=b[:m1], b_ineq=b[m1:], c=c, lower=lo, upper=up)


def c4_cpu_sample(block, m, m1, iters=6):
    """The oracle's C kernels (all host threads) on the one-rank C4 block:
    setup (scaling, 3 power steps) untimed, then ``iters`` HPR iterations."""
    O, scaled, st, threads = _oracle_setup(c4_lp(block, m, m1), 3)
    t0 = time.perf_counter()
    for _ in range(iters):
        O.iterate_once(st, scaled)
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"{iters} HPR iterations of the same rank block (oracle C kernels, "
                      f"OpenMP {threads} threads), setup excluded"}


def run_c4(args, dist, ws, rank, local):
    import torch
    import paper_2408_12179_b200 as P
    from paper_2408_12179_b200.driver import LAMBDA_SAFETY
    from paper_2408_12179_b200.rowblock import RowBlockGroup, broadcast_nccl_id, nccl_unique_id
    rows = args.c4_rows
    block, m, m1, r0 = c4_block(rank, ws, rows, local, dist)
    nid = broadcast_nccl_id(rank) if dist is not None else nccl_unique_id()
    grp = RowBlockGroup.distributed(block, n=C4_N, m_total=m, m1_total=m1,
                                    nnz_total=m * C4_PER_ROW, row0=r0, rank=rank, world=ws,
                                    nccl_id=nid, device=local)
    grp.analyze()
    grp.scale(10, True, True)
    est = grp.power(1e-4, 5000)
    lam = est.raw * (1.0 + LAMBDA_SAFETY)
    grp.state_reset()
    interval = 150
    k = 0

    def step():
        nonlocal k
        grp.run_inner(interval, k, k, 1.0, lam, 2)
        grp.checkpoint(1.0, lam, 1, 0)
        k += interval

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    sample_clocks = ClockSampler(local)
    inner_s = 0.0
    l0 = grp.launch_count()
    with sample_clocks:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(grp.stream)
        for _ in range(args.steps):
            step()
            inner_s += grp.last_times()[0]
        ev1.record(grp.stream)
        ev1.synchronize()
    t_local = ev0.elapsed_time(ev1) / 1e3
    launches = grp.launch_count() - l0
    t_max, _ = _max_sum(dist, local, t_local, 0)
    its = interval * args.steps
    value = its / t_max               # every rank advances the same iterations
    nnz_rank = rows * C4_PER_ROW
    grp.close()

    # e2e through the public API from this rank's host block: every step
    # uploads the block (pinned staging -> H2D), builds the rank group and runs
    # solve() for two 150-iteration intervals (analyse, scale, power method,
    # checkpoints, finalize, solution D2H); graphs are captured anew each time
    import types
    shell = types.SimpleNamespace(objective_constant=0.0, objective_negated=False)
    cfg = P.SolverConfig(tolerance=1e-8, max_iterations=2 * interval, check_interval=interval)
    e2e_t, e2e_its, h2d = 0.0, 0, 0
    for _ in range(max(1, min(args.steps, 2))):
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        nid = broadcast_nccl_id(rank) if dist is not None else nccl_unique_id()
        g2 = RowBlockGroup.distributed(block, n=C4_N, m_total=m, m1_total=m1,
                                       nnz_total=m * C4_PER_ROW, row0=r0, rank=rank, world=ws,
                                       nccl_id=nid, device=local)
        try:
            rep = P.solve(shell, cfg, dev=g2)
            torch.cuda.synchronize()
            e2e_t += time.perf_counter() - t0
            e2e_its += rep.iterations
            h2d = g2.h2d_bytes
        finally:
            g2.close()
    t_e2e, _ = _max_sum(dist, local, e2e_t, 0)
    e2e_val = e2e_its / t_e2e
    peak, peak_kind = load_peaks()
    bi_rank = b_iter(rows, C4_N, nnz_rank)
    achieved = bi_rank * its / inner_s / 1e9
    line = None
    if rank == 0:
        line = {
            "metric": "hpr_iterations_per_sec", "value": value, "unit": "it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": CONFIG_NAMES["c4"], "m": m, "n": C4_N,
                       "nnz": m * C4_PER_ROW, "rows_per_rank": rows,
                       "step": "150 HPR iterations + checkpoint (row-block, NCCL RS/AG per iteration)",
                       "lambda": lam, "power_iterations": est.iterations,
                       "l2": "working set > L2 (no flush needed)",
                       "parallelism": f"row-block x{ws} (NCCL)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": load_traffic("c4") if args.c4_rows == 1_250_000 else None,
                         "kernel": "per-rank iteration (A_g^T partial + slice x-phase + A_g y-phase + collectives)",
                         "bytes_per_iteration": bi_rank, "peak_source": peak_kind},
            "cpu_baseline": c4_cpu_sample(block, m, m1) if ws == 1 and not args.no_cpu else None,
            "e2e": {"value": e2e_val, "unit": "it/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * (2 * C4_N + rows),
                    "step": "upload + solve() for 300 iterations (setup included)"},
            "gpu_launches": launches,
            "clocks": sample_clocks.summary(),
        }
    _finish(dist, line, rank)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIG_NAMES), default="c2")
    ap.add_argument("--c4-rows", type=int, default=1_250_000,
                    help="rows per rank of the c4 weak-scaling instance (100 nnz each)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu DRAM bytes per iteration of the kernel pair (from profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
