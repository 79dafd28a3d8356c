#!/usr/bin/env python
"""Benchmark of the HPR-LP iteration loop on B200 (contract: DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config auto|c1|c2|c3|c3-lite|c4|c5]

Default (``auto``): N = 1 runs C3 (BASELINE configs[2], the largest
single-GPU configuration and the one the north-star target is quoted on);
N > 1 runs C4, the row-block partitioned path.  ``--gpus N`` without a
torchrun environment re-launches itself under ``torch.distributed.run`` with
N ranks (127.0.0.1 rendezvous).

c1/c2/c3: a step is one full solve to tolerance (C3: 1e-8) from a problem
already resident in HBM; the step includes transpose/layout analysis,
scaling, power method, all iterations and checkpoints.  ``value`` = HPR
iterations per second (at N > 1 every rank solves its own replica: only with
an explicit --config).

c4: the row-block partitioned path: each rank owns
``--c4-rows`` rows x 100 nnz of a planted LP with n = 20M columns, generated
per rank; the A^T y partials are reduce-scattered and w all-gathered over
NCCL every iteration.  A step = one 150-iteration interval + checkpoint.
Weak scaling: ``value`` = rank-block iterations per second (units all ranks
processed / max-over-ranks time).  At N > 1 rank 0 also times the same block
as a one-rank group (``one_rank``) so the efficiency is readable off one line.

c5: a batch of 4096 LPs (m=500, n=1000, nnz=5000), one whole solve per CTA,
sharded across ranks (no collective).  A step = the whole shard solved to
1e-8.  ``value`` = LP-iterations per second summed over ranks.

``e2e`` = the same metric through the public API (``solve`` /
``solve_batch`` / ``RowBlockGroup`` + ``solve``) on host data, with the H2D
upload and the D2H of the solution inside the timed region.  ``roofline`` is
the fused x-phase + y-phase iteration pair against the measured HBM copy
bandwidth, B_iter = 24 nnz + 4 (m + n + 2) + 8 (5 m + 8 n) bytes per
iteration, timed by CUDA events on the solver stream around every
150-iteration graph replay.

``--impl reference`` times the reference's own CPU solver (``hprlp`` installed
in baseline/_ref, through its public functions: ``scale_problem``,
``power_method_lambda_max``, ``run_inner`` / ``solve``) on the box's host cores,
on the same instance; a step is a bounded sample of the workload (C1 and C5:
whole solves; C2: 30 iterations; C3: 2 iterations; setup untimed).  Without
baseline/_ref, or for C4 (beyond the reference's memory/time), it times the
oracle port (oracle/: sequential-order C kernels, OpenMP over all host cores).
"""

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


def phase_bytes(m, n, nnz, bu=0):
    """Algorithmic bytes of the x-phase and the y-phase as hpr_time_phases
    runs them (an interval's steady-state HPR step): the matrix (12 B per
    entry) and its row pointers, the gathered vector once, the streamed row
    operands and the writes -- x re-formed from w and not stored, uniform
    bounds (bu bits) passed as scalars."""
    streams_x = 5 - (bu & 1) - ((bu >> 1) & 1)          # w (for x), c, l, u, anchor
    bx = 12 * nnz + 4 * (n + 1) + 8 * m + 8 * streams_x * n + 8 * 1 * n
    by = 12 * nnz + 4 * (m + 1) + 8 * n + 8 * 3 * m + 8 * m
    return bx, by


def phase_roofline(m, n, nnz, lay, x_us, y_us, peak):
    """Per-kernel HBM roofline of the two iteration kernels, each timed alone
    (20 back-to-back launches, CUDA events; hpr_time_phases), and the random
    operand-gather rate of each (one 8-byte gather per entry)."""
    if x_us is None:
        return None
    bx, by = phase_bytes(m, n, nnz, int(lay.get("bounds_uniform", 0)))
    kx, ky = iteration_kernels(lay).split(" (")[0].split(" + ")
    gpeak = gather_peak()
    out = {}
    for name, k, b, us in (("x_phase", kx, bx, x_us), ("y_phase", ky, by, y_us)):
        gbs = b / (us * 1e-6) / 1e9
        out[name] = {"kernel": k, "us_per_launch": us, "bytes": b, "achieved_gbs": gbs,
                     "frac": gbs / peak, "gathers_per_s": nnz / (us * 1e-6),
                     "gather_frac": nnz / (us * 1e-6) / gpeak}
    out["note"] = ("each kernel alone, 20 back-to-back launches of an interval's steady-state "
                   "step after the timed region; bytes = the phase's algorithmic bytes (x "
                   "implicit, uniform bounds as scalars); gather_frac = random operand "
                   "gathers against one L1TEX wavefront per cycle per SM (a staged phase "
                   "gathers from shared memory)")
    return out


def iteration_kernels(lay):
    """Names of the two iteration kernels the layout selected."""
    x = ("k_stg<EpiXIter>" if lay.get("stg_at") else
         "k_tsell<EpiXIter>" if lay.get("ts_at") else "k_sell<EpiXIter>")
    if lay.get("stg_a"):
        y = "k_stg<EpiYIter>"
    elif lay.get("split_a"):
        y = f"{lay['split_a']} x k_sell<EpiCarry..> (column-split)"
    elif lay.get("ts_a"):
        y = "k_tsell<EpiYIter>"
    else:
        y = "k_sell<EpiYIter>"
    return f"{x} + {y} (one HPR iteration)"


def gather_peak():
    """One L1TEX wavefront per cycle per SM at the max SM clock (gathers/s)."""
    import torch
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    mhz = float(json.load(open(p)).get("sm_max_mhz", 1965.0)) if os.path.exists(p) else 1965.0
    return torch.cuda.get_device_properties(0).multi_processor_count * mhz * 1e6


def gather_roofline(nnz, iterations, seconds, lay=None):
    """Operand gathers per second against one L1TEX wavefront per cycle per SM
    (148 SMs at the max SM clock): nnz gathers per HPR iteration for each phase
    on the SELL engine (a staged phase gathers from shared memory); None when
    both phases are staged."""
    peak = gather_peak()
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


L2_NOTE = "256 MB buffer written between timed steps (flush)"


def shared_config(config, tol, m, n, nnz):
    """The `config` object both arms print for C1-C3: the workload only (what
    each arm's step is, and its results, go in the line's `run` object), so
    the driver's same-config check compares like with like."""
    return {"workload": CONFIG_NAMES[config], "tolerance": tol, "m": int(m), "n": int(n),
            "nnz": int(nnz), "l2": L2_NOTE, "parallelism": "none (one device)"}


def c5_config(ws):
    return {"workload": CONFIG_NAMES["c5"], "tolerance": 1e-8, "lps_total": C5_COUNT,
            "l2": "inputs re-read from HBM each step (490 MB > L2)",
            "parallelism": f"batch sharded x{ws}" if ws > 1 else "none (one device)"}


def c4_config(ws, rows):
    return {"workload": CONFIG_NAMES["c4"], "tolerance": 1e-8, "n": C4_N,
            "rows_per_rank": rows, "nnz_per_rank": rows * C4_PER_ROW,
            "l2": "working set > L2 (no flush needed)",
            "parallelism": f"row-block x{ws} (NCCL)"}


def host_flush():
    """The reference arm's counterpart of the GPU arm's L2 flush: write 256 MB
    between timed steps so every step starts with cold host caches."""
    import numpy as np
    buf = np.empty(32 * 1024 * 1024, dtype=np.float64)
    buf.fill(1.0)
    return float(buf[-1])


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


def reference_cpu_sample(prob, scaled, lam, budget_s=10.0):
    """The reference's own iteration (``hprlp.core.run_inner`` from
    baseline/_ref: scipy csr_matvec + numpy, one host core) on the same
    instance in the same run: the problem as this run's GPU scaling left it
    (bit-identical to the reference's scale_problem, tests/test_gpu_parity.py)
    and this run's lambda, so the reference's 80-second setup is skipped; two
    warm-up iterations (the first builds the lazy transpose), then about
    ``budget_s`` of iterations timed.  None without baseline/_ref."""
    hprlp = import_reference()
    if hprlp is None:
        return None
    from hprlp.core import ProblemData, SolverState, Variant as RefVariant, run_inner
    from hprlp.sparse import SparseMatrix as RefSparse
    ae, ai = prob.a_eq, prob.a_ineq
    rp = np.concatenate([np.asarray(ae.row_offsets, np.int64),
                         np.asarray(ai.row_offsets, np.int64)[1:] + int(ae.row_offsets[-1])])
    ci = np.concatenate([np.asarray(ae.col_indices, np.int64), np.asarray(ai.col_indices, np.int64)])
    n = int(np.asarray(prob.c).size)
    a = RefSparse(rp, ci, np.asarray(scaled["a_val_s"], np.float64), int(rp.size - 1), n)
    data = ProblemData(a=a, b=scaled["b_s"], c=scaled["c_s"], lower=scaled["lower_s"],
                       upper=scaled["upper_s"], m1=int(ae.nrows))
    st = SolverState.origin(data, sigma=1.0, lam=float(lam), variant=RefVariant.HPR)
    run_inner(st, data, 1)                   # builds the lazy transpose
    t0 = time.perf_counter()
    run_inner(st, data, 1)
    t1 = time.perf_counter() - t0
    iters = int(max(2, min(3000, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    run_inner(st, data, iters)
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "it/s", "cores": 1, "kind": "reference",
            "sample": f"{iters} HPR iterations of hprlp's run_inner (baseline/_ref: scipy "
                      "csr_matvec + numpy, single-threaded) on the same instance in this run, "
                      "scaled by this run's GPU scaling (bit-identical to scale_problem) with "
                      "this run's lambda, after two warm-up iterations; the reference's own setup "
                      "(scaling + power method, ~80 s at C3) not repeated"}


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
    """``count`` C5 LPs solved to 1e-8 in a process pool over all cores by the
    reference itself (``hprlp.solve`` from baseline/_ref) or, without it, the
    oracle; LP-iterations per second of wall time."""
    import multiprocessing as mp
    cores = cpu_threads()
    hprlp = import_reference()
    if hprlp is not None:
        _C5_REF[:] = [to_reference_problem(hprlp, p) for p in c5_problems(0, count)]
    fn = _ref_c5_worker if hprlp is not None else _c5_worker
    who = "hprlp.solve (baseline/_ref)" if hprlp is not None else "the oracle"
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(min(cores, count)) as pool:
        out = pool.map(fn, range(count))
    dt = time.perf_counter() - t0
    _C5_REF[:] = []
    its = sum(o[0] for o in out)
    return {"value": its / dt, "unit": "LP-it/s", "cores": min(cores, count),
            "kind": "reference" if hprlp is not None else "port",
            "sample": f"{count} of the 4096 C5 LPs solved to 1e-8 by {who} (one LP per "
                      f"process, {min(cores, count)} processes), wall time incl. setup"}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The reference package (``hprlp``) installed in baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "hprlp")):
        return None
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import hprlp
        return hprlp
    except Exception:
        return None


def to_reference_problem(hprlp, prob):
    """The same instance as the reference's own ``LpProblem`` (its validation runs)."""
    from hprlp.sparse import SparseMatrix as RefSparse

    def block(a):
        return RefSparse(np.asarray(a.row_offsets, np.int64), np.asarray(a.col_indices, np.int64),
                         np.asarray(a.values, np.float64), int(a.nrows), int(a.ncols))
    return hprlp.LpProblem(a_eq=block(prob.a_eq), a_ineq=block(prob.a_ineq),
                           b_eq=np.asarray(prob.b_eq, np.float64),
                           b_ineq=np.asarray(prob.b_ineq, np.float64),
                           c=np.asarray(prob.c, np.float64),
                           lower=np.asarray(prob.lower, np.float64),
                           upper=np.asarray(prob.upper, np.float64),
                           objective_constant=float(getattr(prob, "objective_constant", 0.0)),
                           objective_negated=bool(getattr(prob, "objective_negated", False)))


def host_info():
    import platform
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": cpu_threads(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


# iterations per timed step of the reference's inner loop (a bounded sample:
# C2 ~29 ms / C3 ~0.75 s per iteration on one core)
REF_STEP_ITERS = {"c2": 30, "c3": 2, "c3-lite": 150}


_C5_REF = []     # reference-shaped C5 LPs, built before the pool forks


def _ref_c5_worker(i):
    hprlp = import_reference()
    rp = _C5_REF[i]
    t0 = time.perf_counter()
    rep = hprlp.solve(rp, hprlp.SolverConfig(tolerance=1e-8))
    return rep.iterations, time.perf_counter() - t0


def run_reference(args):
    """The CPU reference arm: rank 0 only (other torchrun ranks exit at once)."""
    ws, rank, _ = dist_env()
    ws = max(ws, args.gpus)
    if rank != 0:
        return
    config = resolve_config(args.config, ws)
    hprlp = import_reference() if config != "c4" else None
    base = {"metric": "hpr_iterations_per_sec", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference"}

    def emit(line):
        e = {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
             "d2h_bytes_per_step": 0}
        line["e2e"] = e
        line["cpu_baseline"] = dict(line["cpu_baseline"], value=line["value"])
        line.setdefault("run", {})["host"] = host_info()
        print(json.dumps(line), flush=True)

    if config == "c5":
        import multiprocessing as mp
        cores = cpu_threads()
        cnt = max(cores, 16) * 4
        pool_fn = _ref_c5_worker if hprlp is not None else _c5_worker
        if hprlp is not None:
            _C5_REF[:] = [to_reference_problem(hprlp, p) for p in c5_problems(0, cnt)]
        kind = "reference" if hprlp is not None else "port"
        ctx = mp.get_context("fork")
        vals = []
        with ctx.Pool(min(cores, cnt)) as pool:
            for i in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                out = pool.map(pool_fn, range(cnt))
                dt = time.perf_counter() - t0
                if i >= args.warmup:
                    vals.append((sum(o[0] for o in out), dt))
        val = sum(v[0] for v in vals) / sum(v[1] for v in vals)
        who = "hprlp.solve (baseline/_ref)" if hprlp is not None else "the oracle port"
        emit(dict(base, metric="hpr_lp_iterations_per_sec", value=val, unit="LP-it/s",
                  ms_per_step=1e3 * sum(v[1] for v in vals) / len(vals),
                  config=c5_config(ws),
                  run={"step": f"{cnt} of the 4096 C5 LPs solved to 1e-8 by {who}, "
                                  f"one LP per process, {min(cores, cnt)} processes"},
                  cpu_baseline={"unit": "LP-it/s", "cores": min(cores, cnt), "kind": kind,
                                "sample": f"{args.steps} x {cnt} whole LP solves"}))
        return

    if config == "c4":
        from paper_2408_12179_b200.generators import generate_planted_block
        rows = args.c4_rows
        m1 = rows // 2
        rp_, ci, va, b, ys, m1l, (lo, up, xs, zs), cpart = generate_planted_block(
            4, m1, rows - m1, C4_N, C4_PER_ROW, 0, rows)
        prob = c4_lp((rp_, ci, va, m1l, b, cpart + zs, lo, up), rows, m1)
        O, scaled, st, threads = _oracle_setup(prob, 3)
        for _ in range(args.warmup):
            O.iterate_once(st, scaled)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            O.iterate_once(st, scaled)
        dt = time.perf_counter() - t0
        block_its = args.steps / dt
        # one job iteration = ws rank blocks: the whole-job rate in the same
        # unit as our arm (rank-block iterations per second) is the block rate
        emit(dict(base, value=block_its, unit="rank-it/s", ms_per_step=1e3 * dt / args.steps,
                  config=c4_config(ws, rows),
                  run={"step": "1 HPR iteration over one rank block (oracle port; the "
                                  "reference cannot hold C4)"},
                  cpu_baseline={"unit": "rank-it/s", "cores": threads, "kind": "port",
                                "sample": f"{args.steps} iterations of one 1.25M-row block"}))
        return

    prob, tol = make_instance(config)
    wcfg = shared_config(config, tol, prob.m, prob.n, prob.a_eq.nnz + prob.a_ineq.nnz)
    if hprlp is not None:
        from hprlp.core import ProblemData, SolverState, Variant as RefVariant, run_inner
        from hprlp.scaling import scale_problem
        from hprlp.sparse import power_method_lambda_max
        rp = to_reference_problem(hprlp, prob)
        del prob
        if config == "c1":
            # the same unit as our arm: one whole solve per step
            cfg = hprlp.SolverConfig(tolerance=tol)
            for _ in range(args.warmup):
                hprlp.solve(rp, cfg)
            its, dt, wall = 0, 0.0, 0.0
            for _ in range(args.steps):
                host_flush()
                t0 = time.perf_counter()
                rep = hprlp.solve(rp, cfg)
                wall += time.perf_counter() - t0
                its += rep.iterations
            val = its / wall
            emit(dict(base, value=val, unit="it/s", ms_per_step=1e3 * wall / args.steps,
                      config=wcfg,
                      run={"step": "one full hprlp.solve to tolerance (same unit as ours)",
                           "status": rep.status.value, "iterations_per_solve": rep.iterations},
                      cpu_baseline={"unit": "it/s", "cores": 1, "kind": "reference",
                                    "sample": f"{args.steps} whole solves"}))
            return
        t0 = time.perf_counter()
        scaled, _info = scale_problem(rp, ruiz_iters=10, pock_chambolle=True, bc_normalize=True)
        data = ProblemData.from_problem(scaled)
        t_scale = time.perf_counter() - t0
        t0 = time.perf_counter()
        est = power_method_lambda_max(data.a, tol=1e-4, max_iters=5000)
        t_power = time.perf_counter() - t0
        state = SolverState.origin(data, sigma=1.0, lam=est.value, variant=RefVariant.HPR)
        s = REF_STEP_ITERS.get(config, 150)
        for _ in range(args.warmup):
            run_inner(state, data, s)
        dt = 0.0
        for _ in range(args.steps):
            host_flush()
            t0 = time.perf_counter()
            run_inner(state, data, s)
            dt += time.perf_counter() - t0
        val = s * args.steps / dt
        emit(dict(base, value=val, unit="it/s", ms_per_step=1e3 * dt / args.steps,
                  config=wcfg,
                  run={"step": f"{s} HPR iterations of the reference's run_inner "
                                  "(hprlp from baseline/_ref, its own scipy/numpy path)",
                          "setup_untimed_s": {"scale_problem": t_scale,
                                              "power_method": t_power,
                                              "power_iterations": est.iterations}},
                  cpu_baseline={"unit": "it/s", "cores": 1, "kind": "reference",
                                "sample": f"{args.steps} x {s} iterations after the "
                                          "reference's own setup (single-threaded scipy SpMV)"}))
        return

    # no baseline/_ref: the oracle port on all host threads
    O, scaled, st, threads = _oracle_setup(prob)
    interval = 150 if config != "c3" else 10

    def step():
        for _ in range(interval):
            O.iterate_once(st, scaled)

    for _ in range(args.warmup):
        step()
    dt = 0.0
    for _ in range(args.steps):
        host_flush()
        t0 = time.perf_counter()
        step()
        dt += time.perf_counter() - t0
    val = interval * args.steps / dt
    emit(dict(base, value=val, unit="it/s", ms_per_step=1e3 * dt / args.steps,
              config=wcfg,
              run={"step": f"{interval} HPR iterations (oracle port; baseline/_ref absent)"},
              cpu_baseline={"unit": "it/s", "cores": threads, "kind": "port",
                            "sample": f"{args.steps} x {interval} iterations"}))


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
    config = resolve_config(args.config, ws)
    if config == "c5":
        return run_c5(args, dist, ws, rank, local)
    if config == "c4":
        return run_c4(args, dist, ws, rank, local)
    import paper_2408_12179_b200 as P
    from paper_2408_12179_b200.device import DeviceLP

    prob, tol = make_instance(config)
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
            flush.zero_()                    # L2 flush on the default stream ...
            torch.cuda.synchronize()         # ... finished before the step starts
            dev.analyzed = False             # the step re-runs transpose + layout analysis
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(dev.stream)
            rep = P.solve(prob, cfg, dev=dev)
            ev1.record(dev.stream)
            ev1.synchronize()
            total_ms += ev0.elapsed_time(ev1)
            its_total += rep.iterations
            iter_s_total += rep.device_stats["device_iteration_seconds"]
            reps.append(rep)
    barrier()
    launches = dev.launch_count() - l0
    t_max, its_all = _max_sum(dist, local, total_ms / 1e3, its_total)
    value = its_all / t_max
    # the two iteration kernels one at a time (after the timed region: the
    # diagnostic overwrites the iterate), for the per-kernel roofline
    lay_now = dev.layout_info()
    ph_x_us, ph_y_us = (None, None) if dev.small_path() else dev.time_phases(20)
    # this run's scaled problem, for the reference's own iteration on the host
    ref_scaled = None
    if rank == 0 and ws == 1 and not args.no_cpu and import_reference() is not None:
        ref_scaled = {k: dev.to_host(k) for k in ("a_val_s", "b_s", "c_s", "lower_s", "upper_s")}

    # e2e through the public API from host arrays: every step uploads the
    # problem (pinned staging -> H2D), re-analyses it, solves and copies the
    # solution back; one untimed call first warms the device-residency pool
    e2e_its, e2e_t = 0, 0.0
    h2d = d2h = 0
    dev.close()
    del dev
    P.solve(prob, cfg, device=local)
    e2e_steps = max(3, min(args.steps, 10))
    rep = None
    for _ in range(e2e_steps):
        rep = None                      # the previous step's report is freed untimed
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
        bu = int(lay.get("bounds_uniform", 0))
        b_req = bi - 8 * n * ((bu & 1) + ((bu >> 1) & 1))
        port = cpu_baseline_sample(prob) if ws == 1 and not args.no_cpu else None
        cpu = (reference_cpu_sample(prob, ref_scaled, r0.lambda_estimate)
               if ref_scaled is not None else None)
        ref_scaled = None
        if cpu is None:
            cpu, port = port, None
        if cpu is not None:
            cpu["host"] = host_info()
        line = {
            "metric": "hpr_iterations_per_sec", "value": value, "unit": "it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": shared_config(config, tol, m, n, nnz) if ws == 1 else dict(
                shared_config(config, tol, m, n, nnz), parallelism=f"replicas x{ws}"),
            "run": {"step": "one full solve to tolerance from HBM-resident input "
                               "(transpose/layout analysis, scaling, power method, "
                               "iterations, checkpoints)",
                       "e2e_step": "solve(problem) on host arrays: pinned H2D upload, setup, "
                                   "solve, D2H of x, y, z",
                       "e2e_steps": e2e_steps,
                       "status": r0.status.value, "iterations_per_solve": r0.iterations,
                       "wall_time_to_tol_s": t_max / args.steps},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": args.traffic if args.traffic is not None
                         else load_traffic(config),
                         "kernel": iteration_kernels(lay),
                         "bytes_per_iteration": bi, "peak_source": peak_kind,
                         # l / u passed as scalars when uniform: bytes the pair must move
                         "bytes_required": b_req,
                         "frac_required": b_req * its_total / iter_s_total / 1e9 / peak,
                         "timing": "CUDA events on the solver stream around each "
                                   "150-iteration graph replay (the two iteration kernels)"},
            "roofline_phases": phase_roofline(m, n, nnz, lay_now, ph_x_us, ph_y_us, peak),
            # the bound that actually binds a small-n problem (C2): every nonzero
            # is one random 8-byte operand gather = one L1TEX wavefront per cycle per SM
            # (phases on the staged engine gather from shared memory instead)
            "roofline_gather": gather_roofline(nnz, its_total, iter_s_total, lay),
            "cpu_baseline": cpu,
            # the oracle's C kernels on every host thread (test infrastructure), for scale
            "cpu_baseline_port": port,
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
    reps = None
    for _ in range(max(1, min(args.steps, 3))):
        reps = None                     # the previous step's reports are freed untimed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = solve_batch(probs, cfg, device=local)
        e2e_t += time.perf_counter() - t0
        e2e_its += sum(r.iterations for r in reps)
    t_e2e, its_e2e = _max_sum(dist, local, e2e_t, e2e_its)
    line = None
    if rank == 0:
        cpu = c5_cpu_sample(4 * max(cpu_threads(), 16)) if ws == 1 and not args.no_cpu else None
        line = {
            "metric": "hpr_lp_iterations_per_sec", "value": value, "unit": "LP-it/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": c5_config(ws),
            "run": {"lps_per_rank": hi - lo,
                    "step": "the rank's shard solved to 1e-8 in one launch (one LP per CTA)",
                    "status": st},
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


def c4_one_rank(block, rows, local, steps, warmup):
    """Rank 0's block solved by a one-rank group (NCCL world of 1): rank-it/s."""
    import torch
    from paper_2408_12179_b200.driver import LAMBDA_SAFETY
    from paper_2408_12179_b200.rowblock import RowBlockGroup, nccl_unique_id
    rp, ci, va, m1l, b, c, lo, up = block
    grp = RowBlockGroup.distributed(block, n=C4_N, m_total=rows, m1_total=m1l,
                                    nnz_total=int(rp[-1]), row0=0, rank=0, world=1,
                                    nccl_id=nccl_unique_id(), device=local)
    try:
        grp.analyze()
        grp.scale(10, True, True)
        lam = grp.power(1e-4, 5000).raw * (1.0 + LAMBDA_SAFETY)
        grp.state_reset()
        k = 0
        for i in range(warmup + steps):
            if i == warmup:
                torch.cuda.synchronize()
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record(grp.stream)
            grp.run_inner(150, k, k, 1.0, lam, 2)
            grp.checkpoint(1.0, lam, 1, 0)
            k += 150
        ev1.record(grp.stream)
        ev1.synchronize()
        return {"value": 150 * steps / (ev0.elapsed_time(ev1) / 1e3), "unit": "rank-it/s",
                "what": "rank 0's block as a one-rank group on one GPU, same step"}
    finally:
        grp.close()


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
    # units all ranks processed / max-over-ranks time: every job iteration
    # advances each of the ws rank blocks once (weak scaling)
    value = ws * its / t_max
    nnz_rank = rows * C4_PER_ROW
    comm = grp.comm_info() if hasattr(grp, "comm_info") else None
    grp.close()

    one_rank = None
    if ws > 1:
        # the same per-rank block as a one-rank group on rank 0's GPU (the other
        # GPUs idle at the barrier): the denominator of the weak-scaling efficiency
        if dist is not None:
            dist.barrier()
        if rank == 0:
            one_rank = c4_one_rank(block, rows, local, args.steps, args.warmup)
        if dist is not None:
            dist.barrier()

    # e2e through the public API from this rank's host block: every step
    # uploads the block (pinned staging -> H2D), builds the rank group and runs
    # solve() for two 150-iteration intervals (analyse, scale, power method,
    # checkpoints, finalize, solution D2H); graphs are captured anew each time
    from paper_2408_12179_b200.rowblock import solve_row_block
    cfg = P.SolverConfig(tolerance=1e-8, max_iterations=2 * interval, check_interval=interval)
    e2e_t, e2e_its = 0.0, 0
    h2d = 0
    for _ in range(max(1, min(args.steps, 2))):
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        rep = solve_row_block(block, cfg, n=C4_N, m_total=m, m1_total=m1,
                              nnz_total=m * C4_PER_ROW, row0=r0, device=local)
        torch.cuda.synchronize()
        e2e_t += time.perf_counter() - t0
        e2e_its += rep.iterations
        h2d = rep.device_stats["h2d_bytes"]
    t_e2e, _ = _max_sum(dist, local, e2e_t, 0)
    e2e_val = ws * e2e_its / t_e2e
    peak, peak_kind = load_peaks()
    bi_rank = b_iter(rows, C4_N, nnz_rank)
    achieved = bi_rank * its / inner_s / 1e9
    line = None
    if rank == 0:
        line = {
            "metric": "hpr_iterations_per_sec", "value": value, "unit": "rank-it/s",
            "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": c4_config(ws, rows),
            "run": {"m": m, "nnz": m * C4_PER_ROW,
                       "step": "150 HPR iterations + checkpoint (row-block, NCCL RS/AG per iteration)",
                       "job_iterations_per_sec": its / t_max,
                       "unit_note": "rank-it/s = job iterations/s x ranks (each job iteration "
                                    "advances every rank's 1.25M-row block once)",
                       "one_rank": one_rank, "nccl": comm,
                       "lambda": lam, "power_iterations": est.iterations},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": load_traffic("c4") if args.c4_rows == 1_250_000 else None,
                         "kernel": "per-rank iteration (A_g^T partial + slice x-phase + A_g y-phase + collectives)",
                         "bytes_per_iteration": bi_rank, "peak_source": peak_kind},
            # what binds the rank: one random fp64 operand gather per entry and phase
            # (y_g from L2 in the A_g^T partial, w's L2-resident column blocks in the y-phase)
            "roofline_gather": gather_roofline(nnz_rank, its, inner_s),
            "cpu_baseline": c4_cpu_sample(block, m, m1) if ws == 1 and not args.no_cpu else None,
            "e2e": {"value": e2e_val, "unit": "it/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * (2 * C4_N + rows),
                    "step": "upload + solve() for 300 iterations (setup included)"},
            "gpu_launches": launches,
            "clocks": sample_clocks.summary(),
        }
    _finish(dist, line, rank)
    return line


def resolve_config(config: str, ws: int) -> str:
    """``auto``: C3 on one GPU (the headline), the row-block C4 path on N > 1."""
    if config == "auto":
        return "c3" if ws <= 1 else "c4"
    return config


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(argv, nproc: int) -> int:
    """Re-run this script under torch.distributed.run with ``nproc`` ranks
    (one per GPU, 127.0.0.1 rendezvous); rank 0 prints the JSON line."""
    env = dict(os.environ)
    env.setdefault("NCCL_ALGO", "Ring")       # fixed reduction order at a given N
    env.setdefault("NCCL_PROTO", "Simple")
    env.setdefault("NCCL_DEBUG", "INFO")      # communicator init lines show nranks
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def dry_run(args):
    """Launch check without a GPU: every rank joins a gloo group, the ranks
    are summed, rank 0 prints what it saw."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([1, rank], dtype=torch.int64)
    if ws > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "world_size": ws, "ranks_joined": int(t[0]),
                          "rank_sum": int(t[1]), "config": resolve_config(args.config, ws),
                          "NCCL_ALGO": os.environ.get("NCCL_ALGO"),
                          "NCCL_PROTO": os.environ.get("NCCL_PROTO")}), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("auto",) + tuple(CONFIG_NAMES), default="auto")
    ap.add_argument("--c4-rows", type=int, default=1_250_000,
                    help="rows per rank of the c4 weak-scaling instance (100 nnz each)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu DRAM bytes per iteration of the kernel pair (from profiles/)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch check only (gloo, no GPU work)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and (
            args.impl == "ours" or args.dry_run):
        sys.exit(self_launch(sys.argv[1:], args.gpus))
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        ws = dist_env()[0]
        if args.gpus != ws:
            ap.error(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        if ws > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        run_ours(args)


if __name__ == "__main__":
    main()
