"""Drop-in ``solve(problem, cfg) -> SolveReport`` running on the B200.

Public names, fields, defaults, validation and status semantics follow the
reference (``/root/reference/pkg/src/hprlp/driver.py``); the outer loop below is
its loop (driver.py:317-372), with every vector operation moved into
``libhprlp_b200.so``:

* setup: upload, ``hpr_analyze`` (transpose + tilings), ``hpr_scale``
  (scaling.py:72-125), ``hpr_power`` (sparse.py:165-203);
* ``run_inner`` (core.py:177-179) is one replay of a captured CUDA graph of
  ``check_interval`` fused x-phase / y-phase iterations;
* each checkpoint (driver.py:329-371) is one ``hpr_checkpoint`` call -- half
  step, unscale, KKT terms, merit and sigma-update dot products -- and the only
  device->host synchronisation of the interval.  The scalar logic (termination,
  restart criteria, sigma guards) is the reference's, evaluated on those sums.

Breakdown (non-finite iterate) is detected in-kernel; the first offending k is
reported exactly as ``NumericalBreakdownError(k)`` would be, and candidates are
double-buffered so the last good checkpoint's point is the one reported
(driver.py:323-326, 374-380).
"""

from __future__ import annotations

import enum
import math
import time
import warnings
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _native as N
from .device import DeviceLP
from .problem import PrimalDualPoint

SCHEMA_VERSION = 1
DELTA_RANGE = (1e-16, 1e12)            # driver.py:33
ERROR_RATIO_RANGE = (1e-8, 1e8)        # driver.py:34
LAMBDA_SAFETY = 1e-3                   # sparse.py:15


class Variant(enum.Enum):
    """core.py:29-43."""

    DR = "dr"
    HDR_FIXED_SIGMA = "hdr-fixed"
    HDR = "hdr"
    HPR = "hpr"

    @property
    def uses_restarts(self) -> bool:
        return self is not Variant.DR

    @property
    def updates_sigma(self) -> bool:
        return self in (Variant.HDR, Variant.HPR)


class SolveStatus(enum.Enum):
    OPTIMAL = "Optimal"
    ITERATION_LIMIT = "IterationLimit"
    TIME_LIMIT = "TimeLimit"
    NUMERICAL_ERROR = "NumericalError"


class RestartKind(enum.Enum):
    SUFFICIENT = "sufficient"
    STALLED = "stalled"
    LONG_LOOP = "long_loop"


@dataclass
class SolverConfig:
    """Same fields, defaults and validation as the reference (driver.py:50-84)."""

    tolerance: float = 1e-8
    time_limit_seconds: float = math.inf
    max_iterations: int = 1_000_000
    check_interval: int = 150
    alpha1: float = 0.2
    alpha2: float = 0.6
    alpha3: float = 0.2
    sigma0: float = 1.0
    variant: Variant = Variant.HPR
    ruiz_iters: int = 10
    pock_chambolle: bool = True
    bc_normalize: bool = True
    power_tol: float = 1e-4
    power_max_iters: int = 5000
    termination_space: str = "original"

    def __post_init__(self):
        if isinstance(self.variant, str):
            self.variant = Variant(self.variant)
        elif not isinstance(self.variant, Variant):
            # a reference hprlp.Variant (or anything with .value)
            self.variant = Variant(getattr(self.variant, "value", self.variant))
        if not 0.0 < self.alpha1 < self.alpha2 < 1.0:
            raise ValueError("need 0 < alpha1 < alpha2 < 1")
        if not 0.0 < self.alpha3 < 1.0:
            raise ValueError("need 0 < alpha3 < 1")
        if self.tolerance <= 0.0:
            raise ValueError("tolerance must be positive")
        if self.check_interval < 1:
            raise ValueError("check_interval must be >= 1")
        if self.sigma0 <= 0.0:
            raise ValueError("sigma0 must be positive")
        if self.termination_space not in ("original", "scaled"):
            raise ValueError("termination_space must be 'original' or 'scaled'")

    @classmethod
    def coerce(cls, cfg) -> "SolverConfig":
        """Accept None, our SolverConfig, or the reference's (same field names)."""
        if cfg is None:
            return cls()
        if isinstance(cfg, cls):
            return cfg
        names = [f for f in cls.__dataclass_fields__]
        return cls(**{f: getattr(cfg, f) for f in names if hasattr(cfg, f)})


@dataclass
class KktResidual:
    """driver.py:87-114."""

    primal_infeas_abs: float
    primal_infeas_rel: float
    dual_infeas_abs: float
    dual_infeas_rel: float
    gap_abs: float
    gap_rel: float
    residual_vector_norm: float
    primal_objective: float
    dual_objective: float
    dual_clamped: int = 0

    def to_dict(self) -> dict[str, Any]:
        return {k: getattr(self, k) for k in (
            "primal_infeas_abs", "primal_infeas_rel", "dual_infeas_abs", "dual_infeas_rel",
            "gap_abs", "gap_rel", "residual_vector_norm", "primal_objective",
            "dual_objective", "dual_clamped")}


@dataclass
class RestartEvent:
    """driver.py:117-127."""

    outer_index: int
    trigger: str
    tau: int
    sigma_next: float
    merit: float

    def to_dict(self) -> dict[str, Any]:
        return {"outer_index": self.outer_index, "trigger": self.trigger, "tau": self.tau,
                "sigma_next": self.sigma_next, "merit": self.merit}


@dataclass
class Timings:
    """driver.py:130-151, wall-clock like the reference's ``perf_counter``
    stage boundaries (driver.py:292-372).  The inner graph replay and the
    checkpoint share one host synchronisation, so an interval's wall time is
    split with the checkpoint's device time: checkpoint_seconds = its CUDA-event
    time + the host scalar logic, iteration_seconds = the rest of the interval.
    scaling_seconds covers upload + transpose/tiling + scaling (excluded from
    solve_seconds, as the reference excludes parsing and scaling).  The pure
    device times are in ``SolveReport.device_stats`` (``device_iteration_seconds``,
    ``device_checkpoint_seconds``)."""

    scaling_seconds: float = 0.0
    power_method_seconds: float = 0.0
    iteration_seconds: float = 0.0
    checkpoint_seconds: float = 0.0

    @property
    def solve_seconds(self) -> float:
        return self.power_method_seconds + self.iteration_seconds + self.checkpoint_seconds

    def to_dict(self) -> dict[str, Any]:
        return {"scaling_seconds": self.scaling_seconds,
                "power_method_seconds": self.power_method_seconds,
                "iteration_seconds": self.iteration_seconds,
                "checkpoint_seconds": self.checkpoint_seconds,
                "solve_seconds": self.solve_seconds}


@dataclass
class SolveReport:
    """driver.py:154-188 (schema_version 1)."""

    status: SolveStatus
    primal_objective: float
    dual_objective: float
    kkt: KktResidual
    iterations: int
    restarts: int
    restart_log: list
    timings: Timings
    solution: PrimalDualPoint
    sigma_final: float
    lambda_estimate: float
    device_stats: dict = field(default_factory=dict, repr=False)

    def to_json_dict(self, include_solution: bool = True) -> dict[str, Any]:
        out = {
            "schema_version": SCHEMA_VERSION,
            "status": self.status.value,
            "primal_objective": self.primal_objective,
            "dual_objective": self.dual_objective,
            "kkt": self.kkt.to_dict(),
            "iterations": self.iterations,
            "restarts": self.restarts,
            "restart_log": [e.to_dict() for e in self.restart_log],
            "timings": self.timings.to_dict(),
            "sigma_final": self.sigma_final,
            "lambda_estimate": self.lambda_estimate,
        }
        if include_solution:
            out["solution"] = {"x": self.solution.x.tolist(), "y": self.solution.y.tolist(),
                               "z": self.solution.z.tolist()}
        return out


# ---------------------------------------------------------------------------
# scalar rules (host): identical to the reference
# ---------------------------------------------------------------------------

def check_termination(res: KktResidual, tolerance: float) -> bool:
    """driver.py:231-235 (non-strict)."""
    return (res.gap_rel <= tolerance and res.primal_infeas_rel <= tolerance
            and res.dual_infeas_rel <= tolerance)


def check_restart(merit_now, merit_first, merit_prev, t, k, cfg) -> RestartKind | None:
    """driver.py:238-248: sufficient > stalled > long loop."""
    if merit_now <= cfg.alpha1 * merit_first:
        return RestartKind.SUFFICIENT
    if merit_now <= cfg.alpha2 * merit_first and merit_now > merit_prev:
        return RestartKind.STALLED
    if t >= cfg.alpha3 * k:
        return RestartKind.LONG_LOOP
    return None


def sigma_guards_pass(delta_x, delta_y, error_p, error_d) -> bool:
    """driver.py:251-261."""
    lo, hi = DELTA_RANGE
    if not (lo < delta_x < hi and lo < delta_y < hi):
        return False
    if error_p == 0.0:
        return error_d == 0.0
    ratio = error_d / error_p
    return ERROR_RATIO_RANGE[0] < ratio < ERROR_RATIO_RANGE[1]


def sigma_from_norms(delta_x, ynorm, lam, res: KktResidual) -> float:
    """driver.py:264-278 with the two norms already reduced on the device."""
    delta_y = math.sqrt(lam) * ynorm
    if not sigma_guards_pass(delta_x, delta_y, res.primal_infeas_rel, res.dual_infeas_rel):
        return 1.0
    return delta_x / delta_y


def kkt_from_sums(o, bnorm, cnorm, objective_constant) -> KktResidual:
    """driver.py:203-216 / problem.py:146-176 from the device-reduced sums."""
    pa = float(math.sqrt(o.prim2))
    pr = pa / (1.0 + bnorm)
    da = float(math.sqrt(o.dual2))
    dr = da / (1.0 + cnorm)
    pobj = o.cx + objective_constant
    dobj = o.by
    if o.n_lo:
        dobj += o.lz
    if o.n_up:
        dobj += o.uz
    dobj += objective_constant
    ga = abs(dobj - pobj)
    gr = ga / (1.0 + abs(dobj) + abs(pobj))
    stacked = math.sqrt(o.r1sq + o.r2sq + o.dual2)
    return KktResidual(pa, pr, da, dr, ga, gr, stacked, pobj, dobj, int(o.clamped))


def merit_from_sums(o, sigma, lam) -> float:
    """checkpoint_merit = 2 m_norm_diff(y - yb, x - xb) (core.py:182-218)."""
    q = o.sh2 / sigma
    t1 = lam * o.dy2 - o.aty2
    q += sigma * t1
    scale = sigma * lam * o.dy2 + o.dx2 / sigma
    if q < -1e-9 * max(scale, 1e-300):
        warnings.warn("negative quadratic form in the merit: lambda may "
                      "underestimate lambda_1(AA*)", RuntimeWarning)
    return 2.0 * float(np.sqrt(max(q, 0.0)))


# ---------------------------------------------------------------------------
# solve
# ---------------------------------------------------------------------------

class _DevicePool:
    """Device residencies kept between solve() calls, keyed by the problem's
    dimensions (like an FFT plan cache): a later problem of the same shape is
    uploaded into the same buffers and context, so its solve skips the device
    allocations and -- when its structure reproduces the layout -- the CUDA
    graph captures.  Inputs are always re-uploaded and re-analysed.  An entry
    is checked out for the duration of a solve, so concurrent solves never
    share one."""

    def __init__(self, capacity: int = 2, max_bytes: float | None = None):
        import threading
        self.capacity = capacity
        self.max_bytes = max_bytes   # None: a quarter of the device's memory (B200: ~45 GB)
        self.free: list[DeviceLP] = []
        self.lock = threading.Lock()

    def acquire(self, problem, device: int) -> DeviceLP:
        key = DeviceLP.problem_key(problem, device)
        with self.lock:
            for i, d in enumerate(self.free):
                if d.dims_key() == key:
                    dev = self.free.pop(i)
                    break
            else:
                dev = None
        if dev is None:
            return DeviceLP(problem, device=device)
        dev.reload(problem)
        return dev

    def release(self, dev: DeviceLP):
        limit = self.max_bytes
        if limit is None:
            import torch
            limit = 0.25 * torch.cuda.get_device_properties(dev.device).total_memory
        if 92 * dev.nnz + 160 * (dev.m + dev.n) > limit:
            dev.close()                       # large residencies are not kept
            return
        with self.lock:
            self.free.insert(0, dev)
            while len(self.free) > self.capacity:
                self.free.pop().close()

    def clear(self):
        with self.lock:
            for d in self.free:
                d.close()
            self.free.clear()


DEVICE_POOL = _DevicePool()


def solve(problem, cfg=None, *, device: int = 0, dev: DeviceLP | None = None) -> SolveReport:
    """Run the restarted HPR-LP solver on the GPU (reference driver.py:281-405).

    ``problem``: our ``LpProblem`` or the reference's (duck-typed).
    ``dev``: an already-uploaded ``DeviceLP`` of this problem (re-solves skip
    the upload; the state is reset).  Without it the problem is uploaded into
    a pooled device residency (``DEVICE_POOL``).
    """
    if dev is not None:
        return _solve(problem, cfg, dev)
    dev = DEVICE_POOL.acquire(problem, device)
    try:
        return _solve(problem, cfg, dev)
    finally:
        DEVICE_POOL.release(dev)


def _time_limit_hit(dev, wall_start: float, limit: float) -> bool:
    """driver.py:345 (wall time since the solve started).  A row-block group
    (one rank per process) must take the same branch on every rank -- one rank
    finalizing (all-gather) while another runs the next interval
    (reduce-scatter) would mismatch the collectives -- so the per-rank
    decisions are OR-reduced over the group (``any_rank``).  Every rank holds
    the same ``cfg``, so an infinite limit skips the collective everywhere."""
    if not math.isfinite(limit):
        return False
    hit = time.perf_counter() - wall_start >= limit
    agree = getattr(dev, "any_rank", None)
    return bool(agree(hit)) if agree is not None else hit


def _solve(problem, cfg, dev) -> SolveReport:
    cfg = SolverConfig.coerce(cfg)
    wall_start = time.perf_counter()
    launches0 = dev.launch_count()
    timings = Timings()
    variant = cfg.variant
    vcode = N.VARIANT_CODE[variant.value]

    prefault = getattr(dev, "prefault_solution", None)
    prefault = prefault() if prefault is not None else None   # solution arrays, off-thread
    t0 = time.perf_counter()
    if not dev.analyzed:
        dev.analyze()
    if dev.nnz == 0:
        raise ValueError("matrix must be non-zero")
    sc = dev.scale(cfg.ruiz_iters, cfg.pock_chambolle, cfg.bc_normalize)
    timings.scaling_seconds = time.perf_counter() - t0

    t0 = time.perf_counter()
    est = dev.power(cfg.power_tol, cfg.power_max_iters)
    timings.power_method_seconds = time.perf_counter() - t0
    if not est.converged:
        warnings.warn(f"power method did not converge within {est.iterations} iterations",
                      RuntimeWarning)
    lam = est.raw * (1.0 + LAMBDA_SAFETY)

    dev.state_reset()
    term_original = cfg.termination_space == "original"
    bnorm = sc.bnorm_orig if term_original else sc.bnorm_s
    cnorm = sc.cnorm_orig if term_original else sc.cnorm_s
    objective_constant = float(getattr(problem, "objective_constant", 0.0))
    objective_negated = bool(getattr(problem, "objective_negated", False))

    sigma = cfg.sigma0
    r = t = k = 0
    merit_first = None
    merit_prev = math.inf
    restart_log: list[RestartEvent] = []
    status = None
    res = None
    good_slot = None       # candidate slot of the last completed checkpoint
    slot = 0

    dev_it_s = dev_ck_s = 0.0
    while status is None:
        steps = min(cfg.check_interval, cfg.max_iterations - k)
        lamsig = lam * sigma
        tw0 = time.perf_counter()
        if steps > 0:
            dev.run_inner(steps, t, k, sigma, lamsig, vcode)
        o = dev.checkpoint(sigma, lamsig, term_original, slot)   # one sync
        tw1 = time.perf_counter()
        it_s, ck_s = dev.last_times()
        it_s = it_s if steps > 0 else 0.0
        dev_it_s += it_s
        if o.nonfinite_k >= 0:
            timings.iteration_seconds += tw1 - tw0
            # NumericalBreakdownError(k) inside run_inner: k is not advanced for
            # the failing step and no checkpoint of this interval counts.
            k = int(o.nonfinite_k)
            status = SolveStatus.NUMERICAL_ERROR
            break
        t += max(steps, 0)
        k += max(steps, 0)
        dev_ck_s += ck_s
        ck_wall = min(ck_s, tw1 - tw0)
        timings.iteration_seconds += (tw1 - tw0) - ck_wall
        timings.checkpoint_seconds += ck_wall
        res = kkt_from_sums(o, bnorm, cnorm, objective_constant)
        good_slot = slot
        slot = 1 - slot
        if check_termination(res, cfg.tolerance):
            status = SolveStatus.OPTIMAL
        elif k >= cfg.max_iterations:
            status = SolveStatus.ITERATION_LIMIT
        elif _time_limit_hit(dev, wall_start, cfg.time_limit_seconds):
            status = SolveStatus.TIME_LIMIT
        elif variant.uses_restarts:
            merit_now = merit_from_sums(o, sigma, lam)
            if merit_first is None:
                merit_first = merit_now
                merit_prev = math.inf
            kind = check_restart(merit_now, merit_first, merit_prev, t, k, cfg)
            if kind is not None:
                if variant.updates_sigma:
                    sigma_next = sigma_from_norms(math.sqrt(o.bar_dx2), math.sqrt(o.bar_dy2),
                                                  lam, res)
                else:
                    sigma_next = sigma
                restart_log.append(RestartEvent(r, kind.value, t, sigma_next, merit_now))
                dev.restart()
                sigma = sigma_next
                r += 1
                t = 0
                merit_first = None
                merit_prev = math.inf
            else:
                merit_prev = merit_now
        timings.checkpoint_seconds += time.perf_counter() - tw1      # host scalar logic

    if good_slot is None:
        # breakdown before the first checkpoint: the origin (driver.py:374-380)
        good_slot = slot
        o = dev.kkt_origin(term_original, good_slot)
        res = kkt_from_sums(o, bnorm, cnorm, objective_constant)

    fo = dev.finalize(term_original, good_slot)
    final_slot = good_slot if term_original else 1 - good_slot
    pobj = fo.cx + objective_constant
    dobj = fo.by
    if fo.n_lo:
        dobj += fo.lz
    if fo.n_up:
        dobj += fo.uz
    dobj += objective_constant
    if objective_negated:
        pobj, dobj = -pobj, -dobj
    if hasattr(dev, "solution_to_host"):
        sy, sz, sx = dev.solution_to_host(final_slot, prefault)
    else:
        sy, sz, sx = (dev.to_host(nm, final_slot) for nm in ("cand_y", "cand_z", "cand_x"))
    solution = PrimalDualPoint(y=sy, z=sz, x=sx)
    layout = dev.layout_info()
    return SolveReport(
        status=status, primal_objective=pobj, dual_objective=dobj, kkt=res, iterations=k,
        restarts=r, restart_log=restart_log, timings=timings, solution=solution,
        sigma_final=sigma, lambda_estimate=lam,
        device_stats={"lambda_raw": est.raw, "power_iterations": est.iterations,
                      "b_factor": sc.b_factor, "c_factor": sc.c_factor,
                      "launches": dev.launch_count() - launches0, "layout": layout,
                      "h2d_bytes": dev.h2d_bytes, "device_iteration_seconds": dev_it_s,
                      "device_checkpoint_seconds": dev_ck_s})


def kkt_residual(problem, point: PrimalDualPoint, *, dev: DeviceLP | None = None,
                 device: int = 0) -> KktResidual:
    """GPU kkt_residual (driver.py:191-228) of a host point on the original problem."""
    import torch
    point.check_dims(problem)
    if dev is None:
        dev = DeviceLP(problem, device=device)
    if not dev.analyzed:
        dev.analyze()
    sc = dev.scale(0, False, False)
    with torch.cuda.stream(dev.stream):
        for name, arr in (("cand_y", point.y), ("cand_x", point.x), ("cand_z", point.z)):
            dev.t[name][0].copy_(torch.from_numpy(np.ascontiguousarray(arr, np.float64)))
    o = dev.kkt(1, 0)
    return kkt_from_sums(o, sc.bnorm_orig, sc.cnorm_orig,
                         float(getattr(problem, "objective_constant", 0.0)))
