"""The exact T1 = 0 path on the GPU.

For equality-only instances whose AA* is cheap to factor (m <= 2000), the
reference (``/root/reference/pkg/src/hprlp/exact.py``) drops the proximal
weight and solves the dual subproblem exactly through a dense Cholesky factor
of AA*.  Here the iteration loop is this library's own kernels
(``csrc/hpr_exact.cuh``), ``check_interval`` iterations per CUDA-graph replay
with no host synchronisation inside the interval:

* x side (A^T y, clip, zb, u = xb + sigma (zb - c), the variant step of x) and
  the right-hand side (b - A u) / sigma: SELL kernels with fused epilogues,
  every row summed left to right from 0.0 like scipy's ``csr_matvec``;
* the two triangular solves of ``solve_normal_equations``: products with the
  explicit inverse factor L^{-1} / L^{-T}, computed once per solve (setup:
  cuSOLVER ``potrf`` via ``torch.linalg.cholesky_ex`` and one triangular solve
  against the identity) -- fully parallel per iteration instead of m
  dependent substitution steps; the y variant step and the non-finite probe
  are fused into the second product.

The checkpoint runs the same kernels in half-step mode, then ``hpr_kkt`` on
the original problem; the host makes only the scalar decisions (termination,
restart, sigma) -- the same ones as ``driver.solve``.

Names, arguments, errors and report contents follow the reference:

* ``CHOLESKY_ROW_LIMIT``, ``RankDeficiencyError``, ``DenseCholesky``  exact.py:28-59
* ``solve_normal_equations``                                        exact.py:62-67
* ``exact_half_step`` / ``hpr_exact_iterate`` (on an ``ExactState``)   exact.py:70-91
* ``sigma_update_exact``                                            exact.py:94-103
* ``solve_equality_exact``                                          exact.py:106-178
* ``hpr_no_prox_trace``, ``halpern_padmm_trace``, ``max_trace_gap``   exact.py:188-285
  (diagnostic formulations for the trace tests: device tensor ops)

Parity (tests/test_exact.py against fixtures made by the reference,
tests/golden/make_exact_golden.py): identical status, iteration count and
restart triggers, objectives and residual fields within 1e-8; traces of the
two formulations within 1e-10 of each other and of the reference's.  Bitwise
equality with LAPACK's Cholesky substitution is not attainable (blocking
order).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .device import DeviceLP
from .driver import (KktResidual, RestartEvent, SolveReport, SolverConfig, SolveStatus, Timings,
                     check_restart, check_termination, kkt_from_sums, sigma_guards_pass)
from .problem import PrimalDualPoint

CHOLESKY_ROW_LIMIT = 2000


class RankDeficiencyError(ValueError):
    """AA* is not positive definite; use the lambda-proximal path instead."""


class NumericalBreakdownError(ArithmeticError):
    """A non-finite value appeared in the iterates (core.py:46-51)."""

    def __init__(self, iteration: int):
        super().__init__(f"non-finite iterate at iteration {iteration}")
        self.iteration = iteration


def _torch():
    import torch
    return torch


def _csr_of(a):
    """(row_offsets, col_indices, values, nrows, ncols) of a SparseMatrix-like."""
    return (np.asarray(a.row_offsets), np.asarray(a.col_indices), np.asarray(a.values),
            int(a.nrows), int(a.ncols))


@dataclass(frozen=True)
class DenseCholesky:
    """Lower-triangular device factor L of AA* (L L' = AA*) for a full-row-rank
    equality block (exact.py:35-59)."""

    factor: object   # torch.float64 tensor (m, m) on the GPU
    m: int
    inverse: object = None     # L^{-1}, row-major (m, m)
    inverse_t: object = None   # L^{-T}, row-major (m, m)

    @classmethod
    def from_matrix(cls, a, row_limit: int = CHOLESKY_ROW_LIMIT, device: int = 0
                    ) -> "DenseCholesky":
        torch = _torch()
        if int(a.nrows) > row_limit:
            raise ValueError(f"m={int(a.nrows)} exceeds the dense factorization limit {row_limit}")
        ro, ci, va, m, n = _csr_of(a)
        dev = torch.device("cuda", device)
        rows = torch.from_numpy(np.repeat(np.arange(m, dtype=np.int64), np.diff(ro))).to(dev)
        cols = torch.from_numpy(ci.astype(np.int64)).to(dev)
        vals = torch.from_numpy(va.astype(np.float64)).to(dev)
        if m * n <= (1 << 27):                   # dense A (<= 1 GB): one cuBLAS DGEMM
            Ad = torch.zeros((m, n), dtype=torch.float64, device=dev)
            Ad[rows, cols] = vals                # canonical CSR: no duplicates
            aat = Ad @ Ad.T
        else:                                    # cuSPARSE SpGEMM A A'
            with torch.sparse.check_sparse_tensor_invariants(False):
                A = torch.sparse_coo_tensor(torch.stack([rows, cols]), vals, (m, n)).to_sparse_csr()
                At = torch.sparse_coo_tensor(torch.stack([cols, rows]), vals, (n, m)).to_sparse_csr()
                aat = torch.sparse.mm(A, At).to_dense()
        lower, info = torch.linalg.cholesky_ex(aat)
        if int(info.item()) != 0:
            raise RankDeficiencyError(
                "AA* is rank deficient; fall back to the lambda-proximal path")
        recon = lower @ lower.T
        scale = float(torch.linalg.norm(aat))
        if float(torch.linalg.norm(recon - aat)) > 1e-10 * max(scale, 1e-300):
            raise RankDeficiencyError("Cholesky reconstruction check failed")
        eye = torch.eye(m, dtype=torch.float64, device=dev)
        inv = torch.linalg.solve_triangular(lower, eye, upper=False).contiguous()
        return cls(factor=lower, m=m, inverse=inv, inverse_t=inv.T.contiguous())


def solve_normal_equations(chol: DenseCholesky, rhs):
    """Solve AA* y = rhs through the cached factor (exact.py:62-67): the two
    triangular solves as products with L^{-1} and L^{-T} (``hpr_trsolve``).
    ``rhs`` a device tensor (returned on the device) or a host array
    (returned on the host)."""
    import ctypes
    from . import _native as N
    torch = _torch()
    host = not isinstance(rhs, torch.Tensor)
    dev = chol.factor.device
    r = torch.as_tensor(np.asarray(rhs, np.float64)) if host else rhs
    if tuple(r.shape) != (chol.m,):
        raise ValueError("rhs length does not match the factor")
    r = r.to(device=dev, dtype=torch.float64).contiguous()
    tmp = torch.empty(chol.m, dtype=torch.float64, device=dev)
    y = torch.empty(chol.m, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    N.call("hpr_trsolve", int(chol.m), ctypes.c_void_p(chol.inverse.data_ptr()),
           ctypes.c_void_p(chol.inverse_t.data_ptr()), ctypes.c_void_p(r.data_ptr()),
           ctypes.c_void_p(tmp.data_ptr()), ctypes.c_void_p(y.data_ptr()),
           ctypes.c_void_p(stream.cuda_stream))
    if host:
        stream.synchronize()
        return y.cpu().numpy()
    return y


class _Dev:
    """Device data of an equality-only problem: the SELL layout for the sparse
    products (identity scaling: the exact path is unpreconditioned), b, c,
    bounds as device tensors, the KKT evaluation on the original problem, and
    (``bind``) the exact-path kernels' inverse factors and scratch."""

    def __init__(self, problem, device: int):
        if int(problem.m2) != 0:
            raise ValueError("the exact path requires an equality-only instance")
        self.problem = problem
        self.d = DeviceLP(problem, device=device)
        self.d.analyze()
        self.sc = self.d.scale(0, False, False)
        self.d.state_reset()
        t = self.d.t
        self.m, self.n = self.d.m, self.d.n
        self.b, self.c = t["b_s"], t["c_s"][:self.n]
        self.lower, self.upper = t["lower_s"][:self.n], t["upper_s"][:self.n]
        self.stream = self.d.stream
        torch = _torch()
        self._ybuf = torch.empty(self.m + 8, dtype=torch.float64, device=self.d.device)
        self._xbuf = torch.empty(self.n + 8, dtype=torch.float64, device=self.d.device)
        self._chol = None

    def bind(self, chol: DenseCholesky):
        """Hand the inverse factors and scratch vectors to hpr_exact_bind."""
        import ctypes
        from . import _native as N
        if self._chol is chol:
            return
        torch = _torch()
        f64 = dict(dtype=torch.float64, device=self.d.device)
        with torch.cuda.stream(self.stream):
            self._u = torch.empty(self.n + 8, **f64)
            self._rhs = torch.empty(self.m + 8, **f64)
            self._h = torch.empty(self.m + 8, **f64)
        eb = N.HprExactBufs(chol.inverse.data_ptr(), chol.inverse_t.data_ptr(),
                            self._u.data_ptr(), self._rhs.data_ptr(), self._h.data_ptr())
        N.call("hpr_exact_bind", self.d.ctx, ctypes.byref(eb))
        self._chol = chol

    def run(self, steps, t, k, sigma, variant):
        """``steps`` exact iterations on the device state (hpr_exact_run)."""
        from . import _native as N
        N.call("hpr_exact_run", self.d.ctx, int(steps), int(t), int(k), float(sigma),
               N.VARIANT_CODE[getattr(variant, "value", variant)])

    def half(self, sigma, slot=0) -> int:
        """Half step at the device state into xb/zb/yb and candidate ``slot``;
        returns the first non-finite iteration since the reset, or -1."""
        import ctypes
        from . import _native as N
        nf = ctypes.c_int64(-1)
        N.call("hpr_exact_half", self.d.ctx, float(sigma), int(slot), ctypes.byref(nf))
        return int(nf.value)

    def load(self, current, anchor=None):
        """Device state <- (y, x) [and anchor] device tensors."""
        t = self.d.t
        t["y"][:self.m].copy_(current.y)
        t["x"][:self.n].copy_(current.x)
        if anchor is not None:
            t["anc_y"][:self.m].copy_(anchor.y)
            t["anc_x"][:self.n].copy_(anchor.x)

    def apply(self, x):
        """A x (sparse.py:102-104)."""
        self._xbuf[:self.n].copy_(x)
        out = _torch().empty(self.m, dtype=_torch().float64, device=self.d.device)
        self.d.spmv(False, self._xbuf, out)
        return out

    def t_apply(self, y):
        """A' y (sparse.py:106-108)."""
        self._ybuf[:self.m].copy_(y)
        out = _torch().empty(self.n, dtype=_torch().float64, device=self.d.device)
        self.d.spmv(True, self._ybuf, out)
        return out

    def kkt(self, y=None, x=None, z=None, slot=0) -> KktResidual:
        """driver.py:191-228 on the original problem (hpr_kkt) of candidate
        ``slot`` (after storing (y, x, z) there when given)."""
        t = self.d.t
        if y is not None:
            t["cand_y"][slot][:self.m].copy_(y)
            t["cand_x"][slot][:self.n].copy_(x)
            t["cand_z"][slot][:self.n].copy_(z)
        o = self.d.kkt(1, slot)
        return kkt_from_sums(o, self.sc.bnorm_orig, self.sc.cnorm_orig,
                             float(getattr(self.problem, "objective_constant", 0.0)))

    def close(self):
        self.d.close()


@dataclass
class ExactIterate:
    y: object
    x: object


@dataclass
class ExactState:
    """SolverState of the no-proximal path (core.py:94-115, lam = 0)."""

    current: ExactIterate
    anchor: ExactIterate
    sigma: float
    variant: object
    bar: ExactIterate | None = None
    r: int = 0
    t: int = 0
    k: int = 0
    merit_first: float | None = None
    merit_prev: float = math.inf


def exact_half_step(state: ExactState, data: _Dev, chol: DenseCholesky):
    """(xb, yb, zb) for the no-proximal dual update (exact.py:70-80), by the
    exact-path kernels in half-step mode on ``state.current``."""
    data.bind(chol)
    with _torch().cuda.stream(data.stream):
        data.load(state.current)
        data.half(state.sigma)
        t = data.d.t
        return t["xb"][:data.n].clone(), t["yb"][:data.m].clone(), t["zb"][:data.n].clone()


def hpr_exact_iterate(state: ExactState, data: _Dev, chol: DenseCholesky):
    """One iteration with the exact dual solve; same variant step as the lambda
    path (exact.py:83-91): the half step, then one exact-path iteration on the
    device (the same four kernels with the variant step fused)."""
    torch = _torch()
    if data is None or int(getattr(data, "problem").m2) != 0:
        raise ValueError("the exact path requires an equality-only instance")
    xb, yb, _ = exact_half_step(state, data, chol)
    with torch.cuda.stream(data.stream):
        data.load(state.current, state.anchor)
        data.run(1, state.t, state.k, state.sigma, state.variant)
        t = data.d.t
        y_next, x_next = t["y"][:data.m].clone(), t["x"][:data.n].clone()
    if not bool(torch.isfinite(y_next).all() & torch.isfinite(x_next).all()):
        raise NumericalBreakdownError(state.k)
    state.current = ExactIterate(y_next, x_next)
    state.t += 1
    state.k += 1
    return xb, yb


def sigma_update_exact(bar, anchor, a, last_residual: KktResidual) -> float:
    """Penalty update of the no-proximal path: the dual displacement measured
    through A' (exact.py:94-103).  ``a``: the problem's ``_Dev`` (device
    iterates) or a SparseMatrix-like (host iterates)."""
    if isinstance(a, _Dev):
        torch = _torch()
        delta_x = float(torch.linalg.norm(bar.x - anchor.x))
        delta_y = float(torch.linalg.norm(a.t_apply(bar.y - anchor.y)))
    else:
        ro, ci, va, m, n = _csr_of(a)
        dy = np.asarray(bar.y, np.float64) - np.asarray(anchor.y, np.float64)
        aty = np.zeros(n)
        for i in range(m):                       # host path: tiny test instances only
            for e in range(ro[i], ro[i + 1]):
                aty[ci[e]] += va[e] * dy[i]
        delta_x = float(np.linalg.norm(np.asarray(bar.x) - np.asarray(anchor.x)))
        delta_y = float(np.linalg.norm(aty))
    if not sigma_guards_pass(delta_x, delta_y, last_residual.primal_infeas_rel,
                             last_residual.dual_infeas_rel):
        return 1.0
    return delta_x / delta_y


def _merit_no_prox(dy, dx, sigma, data: _Dev) -> float:
    """m_norm_diff(..., lam=None) (core.py:182-201): |dx + sigma A'dy|^2 / sigma."""
    torch = _torch()
    shifted = dx + sigma * data.t_apply(dy)
    q = float(torch.dot(shifted, shifted)) / sigma
    return float(np.sqrt(max(q, 0.0)))


def solve_equality_exact(problem, cfg: SolverConfig | None = None, *, device: int = 0
                         ) -> SolveReport:
    """Restarted solve of an equality-only instance with exact dual solves
    (exact.py:106-178), on the GPU.  No preconditioning is applied.  Each
    interval is one graph replay of the exact-path kernels; the checkpoint is
    the half step + KKT (one synchronisation) and the host's scalar rules."""
    torch = _torch()
    cfg = SolverConfig.coerce(cfg) if cfg is not None else SolverConfig()
    if int(problem.m2) != 0:
        raise ValueError("the exact path requires an equality-only instance")
    wall_start = time.perf_counter()
    timings = Timings()
    data = _Dev(problem, device)
    try:
        with torch.cuda.stream(data.stream):
            chol = DenseCholesky.from_matrix(problem.a_eq, device=device)
            data.bind(chol)
            t = data.d.t
            m, n = data.m, data.n
            cur_y, cur_x = t["y"][:m], t["x"][:n]          # the device state (origin)
            anc_y, anc_x = t["anc_y"][:m], t["anc_x"][:n]
            yb, xb, zb = t["yb"][:m], t["xb"][:n], t["zb"][:n]
            state = ExactState(current=ExactIterate(cur_y, cur_x),
                               anchor=ExactIterate(anc_y, anc_x), sigma=cfg.sigma0,
                               variant=cfg.variant)
            restart_log: list[RestartEvent] = []
            status = None
            res = None
            while status is None:
                steps = min(cfg.check_interval, cfg.max_iterations - state.k)
                t0 = time.perf_counter()
                data.run(steps, state.t, state.k, state.sigma, state.variant)
                data.stream.synchronize()
                state.t += steps
                state.k += steps
                timings.iteration_seconds += time.perf_counter() - t0

                t0 = time.perf_counter()
                nonfinite = data.half(state.sigma, 0)
                if nonfinite >= 0:
                    raise NumericalBreakdownError(nonfinite)
                state.bar = ExactIterate(yb, xb)
                res = data.kkt(slot=0)
                if check_termination(res, cfg.tolerance):
                    status = SolveStatus.OPTIMAL
                elif state.k >= cfg.max_iterations:
                    status = SolveStatus.ITERATION_LIMIT
                elif time.perf_counter() - wall_start >= cfg.time_limit_seconds:
                    status = SolveStatus.TIME_LIMIT
                elif cfg.variant.uses_restarts:
                    merit_now = 2.0 * _merit_no_prox(cur_y - yb, cur_x - xb, state.sigma, data)
                    if state.merit_first is None:
                        state.merit_first = merit_now
                        state.merit_prev = math.inf
                    kind = check_restart(merit_now, state.merit_first, state.merit_prev,
                                         state.t, state.k, cfg)
                    if kind is not None:
                        sigma_next = (sigma_update_exact(state.bar, state.anchor, data, res)
                                      if cfg.variant.updates_sigma else state.sigma)
                        restart_log.append(RestartEvent(
                            outer_index=state.r, trigger=kind.value, tau=state.t,
                            sigma_next=sigma_next, merit=merit_now))
                        data.d.restart()               # anchor = current = bar
                        state.sigma = sigma_next
                        state.r += 1
                        state.t = 0
                        state.merit_first = None
                        state.merit_prev = math.inf
                data.stream.synchronize()
                timings.checkpoint_seconds += time.perf_counter() - t0
            y = t["cand_y"][0][:m].cpu().numpy()
            x = t["cand_x"][0][:n].cpu().numpy()
            z = t["cand_z"][0][:n].cpu().numpy()
    finally:
        data.close()
    pobj, dobj = res.primal_objective, res.dual_objective
    if getattr(problem, "objective_negated", False):
        pobj, dobj = -pobj, -dobj
    return SolveReport(status=status, primal_objective=pobj, dual_objective=dobj, kkt=res,
                       iterations=state.k, restarts=state.r, restart_log=restart_log,
                       timings=timings, solution=PrimalDualPoint(y=y, z=z, x=x),
                       sigma_final=state.sigma, lambda_estimate=0.0)


# ---------------------------------------------------------------------------
# The two formulations of the no-proximal Halpern scheme (exact.py:181-285)
# ---------------------------------------------------------------------------

@dataclass
class DirectTrace:
    """Per-iteration tuples of the shifted-multiplier formulation (host arrays)."""

    y: list
    z: list
    x_half: list
    x_tilde: list


@dataclass
class AveragedTrace:
    """Per-iteration half-step tuples of the anchored-triple formulation."""

    y: list
    z: list
    x: list


def _clip(v, lo, up):
    """np.clip(v, l, u) == minimum(maximum(v, l), u) with numpy's NaN rules."""
    torch = _torch()
    return torch.minimum(torch.maximum(v, lo), up)


def _z_step(data: _Dev, y, x, sigma):
    v = x + sigma * (data.t_apply(y) - data.c)
    xb = _clip(v, data.lower, data.upper)
    return (xb - v) / sigma, xb


def _start(data, y0, x0):
    torch = _torch()
    f64 = dict(dtype=torch.float64, device=data.d.device)
    y = torch.zeros(data.m, **f64) if y0 is None else torch.as_tensor(
        np.asarray(y0, np.float64)).to(data.d.device)
    x = torch.zeros(data.n, **f64) if x0 is None else torch.as_tensor(
        np.asarray(x0, np.float64)).to(data.d.device)
    return y, x


def hpr_no_prox_trace(problem, sigma: float, iters: int, y0=None, x0=None, *,
                      device: int = 0) -> DirectTrace:
    """Shifted-multiplier formulation (exact.py:200-230)."""
    torch = _torch()
    if int(problem.m2) != 0:
        raise ValueError("equality-only instances required")
    data = _Dev(problem, device)
    try:
        with torch.cuda.stream(data.stream):
            chol = DenseCholesky.from_matrix(problem.a_eq, device=device)
            b, c = data.b, data.c
            y, x_tilde0 = _start(data, y0, x0)
            x_tilde = x_tilde0.clone()
            aty0 = data.t_apply(y)
            out = DirectTrace(y=[], z=[], x_half=[], x_tilde=[])
            for k in range(iters):
                z_next, x_half = _z_step(data, y, x_tilde, sigma)
                rhs = (b - data.apply(x_half + sigma * (z_next - c))) / sigma
                y_next = solve_normal_equations(chol, rhs)
                x_full = x_half + sigma * (data.t_apply(y_next) + z_next - c)
                x_tilde = (x_tilde0 + (k + 1.0) * x_full) / (k + 2.0) \
                    + (sigma / (k + 2.0)) * (aty0 - data.t_apply(y_next))
                y = y_next
                for lst, v in ((out.y, y_next), (out.z, z_next), (out.x_half, x_half),
                               (out.x_tilde, x_tilde)):
                    lst.append(v.cpu().numpy())
    finally:
        data.close()
    return out


def halpern_padmm_trace(problem, sigma: float, iters: int, y0=None, x0=None, *,
                        device: int = 0) -> AveragedTrace:
    """Anchored-triple formulation (exact.py:233-262)."""
    torch = _torch()
    if int(problem.m2) != 0:
        raise ValueError("equality-only instances required")
    data = _Dev(problem, device)
    try:
        with torch.cuda.stream(data.stream):
            chol = DenseCholesky.from_matrix(problem.a_eq, device=device)
            b, c = data.b, data.c
            y, x = _start(data, y0, x0)
            z = torch.zeros_like(x)
            anchor = (y.clone(), z.clone(), x.clone())
            out = AveragedTrace(y=[], z=[], x=[])
            for k in range(iters):
                zb, xb = _z_step(data, y, x, sigma)
                rhs = (b - data.apply(xb + sigma * (zb - c))) / sigma
                yb = solve_normal_equations(chol, rhs)
                out.y.append(yb.cpu().numpy())
                out.z.append(zb.cpu().numpy())
                out.x.append(xb.cpu().numpy())
                w_new = (k + 1.0) / (k + 2.0)
                w_anchor = 1.0 / (k + 2.0)
                y = w_anchor * anchor[0] + w_new * (2.0 * yb - y)
                z = w_anchor * anchor[1] + w_new * (2.0 * zb - z)
                x = w_anchor * anchor[2] + w_new * (2.0 * xb - x)
    finally:
        data.close()
    return out


def max_trace_gap(problem, sigma: float, iters: int, *, device: int = 0) -> float:
    """Largest componentwise gap between the two formulations' traces
    (exact.py:275-285)."""
    direct = hpr_no_prox_trace(problem, sigma, iters, device=device)
    averaged = halpern_padmm_trace(problem, sigma, iters, device=device)
    gap = 0.0
    for k in range(iters):
        gap = max(gap,
                  float(np.max(np.abs(direct.y[k] - averaged.y[k]))),
                  float(np.max(np.abs(direct.z[k] - averaged.z[k]))),
                  float(np.max(np.abs(direct.x_half[k] - averaged.x[k]))))
    return gap
