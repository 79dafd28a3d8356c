"""HPR-LP oracle: a CPU restatement of the reference solve path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module, and only as the checker / the timed CPU baseline -- never as the
product.  The product (``paper_2408_12179_b200``) runs on the GPU and fails
loudly without its CUDA library.

What it restates (reference = ``/root/reference/pkg/src/hprlp``):

* ``Csr.matvec``           -- ``sparse.py:102-108``; arithmetic of scipy's
  ``csr_matvec``: each output starts at 0.0 and adds the separately-rounded
  products ``a_ij * x_j`` left to right in stored (ascending-column) order, no
  FMA.  Vectorised across rows, sequential within a row, so it is bit-identical.
* ``Csr.transpose``        -- ``sparse.py:98-100`` (``csr_matrix(A.T)``):
  stable counting sort, rows ascending inside each column.
* ``scale_lp``             -- ``scaling.py:72-125`` with ``ruiz_scale``
  ``sparse.py:206-224``, ``pock_chambolle_scale`` 227-242,
  ``normalize_rhs_cost`` 245-250.
* ``power_lambda``         -- ``sparse.py:165-203``.
* ``iterate_once`` / ``half_step`` / ``merit`` -- ``core.py:118-218``.
* ``kkt``                  -- ``driver.py:191-228`` with ``problem.py:129-176``.
* ``solve``                -- ``driver.py:281-405`` (restart rules 238-248,
  sigma update 251-278).

Norms and dot products use ``np.linalg.norm`` / ``@`` exactly as the reference
does, so on the same machine the oracle reproduces the reference bit for bit;
``tests/test_oracle_golden.py`` pins that against fixtures generated from the
reference itself by ``tests/golden/make_golden.py``.

An optional C kernel library (``oracle/csrc/hpr_oracle.c``, built into
``oracle/_build/libhpr_oracle.so`` by ``oracle/Makefile``) runs the same
sequential per-row sums with OpenMP across rows; it is bit-identical to the
numpy path and is what the CPU baseline times.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

LAMBDA_SAFETY = 1e-3                     # sparse.py:15
DELTA_RANGE = (1e-16, 1e12)              # driver.py:33
ERROR_RATIO_RANGE = (1e-8, 1e8)          # driver.py:34

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libhpr_oracle.so")
_clib = None


def load_clib():
    """The optional OpenMP C kernels (None when not built)."""
    global _clib
    if _clib is None and os.path.exists(_LIB_PATH):
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_int64)
        lib.orc_matvec.argtypes = [ctypes.c_int64, lp, lp, dp, dp, dp]
        lib.orc_matvec.restype = None
        lib.orc_set_threads.argtypes = [ctypes.c_int]
        lib.orc_set_threads.restype = ctypes.c_int
        lib.orc_xphase.argtypes = [ctypes.c_int64, lp, lp, dp, dp, dp, dp, dp, dp, dp,
                                   dp, dp, dp, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
        lib.orc_xphase.restype = ctypes.c_int
        lib.orc_yphase.argtypes = [ctypes.c_int64, ctypes.c_int64, lp, lp, dp, dp, dp,
                                   dp, dp, dp, dp, ctypes.c_double, ctypes.c_int64,
                                   ctypes.c_int]
        lib.orc_yphase.restype = ctypes.c_int
        _clib = lib
    return _clib


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _lptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# ---------------------------------------------------------------------------
# sparse primitives
# ---------------------------------------------------------------------------

class Csr:
    """CSR matrix with a precomputed plan for sequential per-row sums."""

    def __init__(self, rp, ci, vals, ncols, use_c=True):
        self.rp = np.ascontiguousarray(rp, dtype=np.int64)
        self.ci = np.ascontiguousarray(ci, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.nrows = len(self.rp) - 1
        self.ncols = int(ncols)
        self.use_c = use_c
        lens = np.diff(self.rp)
        self._lens = lens
        self._order = np.argsort(-lens, kind="stable")
        self._starts = self.rp[:-1][self._order]
        neg_sorted = -lens[self._order]
        self._maxlen = int(lens.max()) if lens.size else 0
        self._counts = np.searchsorted(neg_sorted, -np.arange(self._maxlen), side="left")

    @property
    def nnz(self):
        return int(self.rp[-1])

    def rows_of_entries(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), self._lens)

    def with_values(self, vals):
        out = Csr.__new__(Csr)
        out.__dict__.update(self.__dict__)
        out.vals = np.ascontiguousarray(vals, dtype=np.float64)
        return out

    def matvec(self, x):
        """Sequential-order SpMV (reference sparse.py:102-108 / scipy csr_matvec)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        lib = load_clib() if self.use_c else None
        if lib is not None:
            out = np.empty(self.nrows)
            lib.orc_matvec(self.nrows, _lptr(self.rp), _lptr(self.ci), _dptr(self.vals),
                           _dptr(x), _dptr(out))
            return out
        out = np.zeros(self.nrows)
        if self._maxlen == 0:
            return out
        prod = self.vals * x[self.ci]
        for k in range(self._maxlen):
            c = int(self._counts[k])
            idx = self._order[:c]
            out[idx] += prod[self._starts[:c] + k]
        return out

    def transpose(self):
        """Stable counting-sort transpose: csr_matrix(A.T) ordering (sparse.py:98-100)."""
        perm = np.argsort(self.ci, kind="stable")
        rows = self.rows_of_entries()
        counts = np.bincount(self.ci, minlength=self.ncols)
        rpt = np.zeros(self.ncols + 1, dtype=np.int64)
        np.cumsum(counts, out=rpt[1:])
        t = Csr(rpt, rows[perm], self.vals[perm], self.nrows, use_c=self.use_c)
        t.perm = perm
        return t

    def row_max_abs(self):
        out = np.zeros(self.nrows)
        nz = self._lens > 0
        if self.nnz:
            red = np.maximum.reduceat(np.abs(self.vals), self.rp[:-1][nz])
            out[nz] = red
        return out

    def to_dense(self):
        d = np.zeros((self.nrows, self.ncols))
        d[self.rows_of_entries(), self.ci] = self.vals
        return d


def canonical_csr(rp, ci, vals, ncols):
    """SparseMatrix.from_scipy canonicalisation (sparse.py:69-81): duplicates
    summed, explicit zeros dropped, columns sorted."""
    import scipy.sparse as sp
    m = sp.csr_matrix((np.asarray(vals, np.float64), np.asarray(ci), np.asarray(rp)),
                      shape=(len(rp) - 1, ncols))
    m.sum_duplicates()
    m.eliminate_zeros()
    m.sort_indices()
    return m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.astype(np.float64)


# ---------------------------------------------------------------------------
# problem container
# ---------------------------------------------------------------------------

@dataclass
class OracleLP:
    """min <c,x> s.t. A[:m1] x = b[:m1], A[m1:] x >= b[m1:], l <= x <= u
    (reference problem.py:22-112; A is the stacked matrix of problem.py:75-82)."""

    a: Csr
    b: np.ndarray
    c: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    m1: int
    objective_constant: float = 0.0
    objective_negated: bool = False
    at: Csr | None = field(default=None, repr=False)

    @property
    def m(self):
        return self.a.nrows

    @property
    def n(self):
        return self.a.ncols

    def transpose(self):
        if self.at is None:
            self.at = self.a.transpose()
        return self.at

    @classmethod
    def from_problem(cls, p, use_c=True):
        """From a reference-shaped LpProblem (duck-typed: a_eq/a_ineq CSR blocks)."""
        n = int(p.a_eq.ncols)
        rp_e, ci_e, v_e = (np.asarray(p.a_eq.row_offsets), np.asarray(p.a_eq.col_indices),
                           np.asarray(p.a_eq.values))
        rp_i, ci_i, v_i = (np.asarray(p.a_ineq.row_offsets), np.asarray(p.a_ineq.col_indices),
                           np.asarray(p.a_ineq.values))
        rp = np.concatenate([rp_e[:-1], rp_i + rp_e[-1]]).astype(np.int64)
        ci = np.concatenate([ci_e, ci_i]).astype(np.int64)
        v = np.concatenate([v_e, v_i]).astype(np.float64)
        rp, ci, v = canonical_csr(rp, ci, v, n)
        return cls(a=Csr(rp, ci, v, n, use_c=use_c),
                   b=np.concatenate([np.asarray(p.b_eq, np.float64), np.asarray(p.b_ineq, np.float64)]),
                   c=np.asarray(p.c, np.float64).copy(),
                   lower=np.asarray(p.lower, np.float64).copy(),
                   upper=np.asarray(p.upper, np.float64).copy(),
                   m1=int(p.a_eq.nrows),
                   objective_constant=float(getattr(p, "objective_constant", 0.0)),
                   objective_negated=bool(getattr(p, "objective_negated", False)))


def proj_box(v, lower, upper):
    """problem.py:129-133."""
    return np.clip(v, lower, upper)


def proj_dual_cone(v, m1):
    """problem.py:136-143."""
    out = v.copy()
    if m1 < v.shape[0]:
        np.maximum(out[m1:], 0.0, out=out[m1:])
    return out


def primal_obj(lp, x):
    """problem.py:146-148."""
    return float(lp.c @ x) + lp.objective_constant


def dual_obj(lp, y, z):
    """problem.py:156-176: infinite active bounds contribute 0 and are counted."""
    pos = z > 0.0
    neg = z < 0.0
    lo_fin = np.isfinite(lp.lower)
    up_fin = np.isfinite(lp.upper)
    clamped = int(np.count_nonzero(pos & ~lo_fin) + np.count_nonzero(neg & ~up_fin))
    val = float(lp.b @ y)
    take_lo = pos & lo_fin
    take_up = neg & up_fin
    if np.any(take_lo):
        val += float(lp.lower[take_lo] @ z[take_lo])
    if np.any(take_up):
        val += float(lp.upper[take_up] @ z[take_up])
    return val + lp.objective_constant, clamped


# ---------------------------------------------------------------------------
# preconditioning (scaling.py:72-125)
# ---------------------------------------------------------------------------

@dataclass
class Scaling:
    row_scale: np.ndarray
    col_scale: np.ndarray
    b_factor: float
    c_factor: float

    def unscale(self, y, z, x):
        """scaling.py:45-49."""
        return (y * (self.c_factor / self.row_scale),
                z * (self.c_factor * self.col_scale),
                x * (self.b_factor / self.col_scale))


def _col_max_abs(a: Csr, at: Csr, vals):
    absv = np.abs(vals[at.perm])
    out = np.zeros(a.ncols)
    nz = at._lens > 0
    if absv.size:
        out[nz] = np.maximum.reduceat(absv, at.rp[:-1][nz])
    return out


def scale_lp(lp: OracleLP, ruiz_iters=10, pock_chambolle=True, bc_normalize=True):
    """Ruiz(iters) -> Pock-Chambolle(alpha=1) -> b/c normalisation."""
    a = lp.a
    at = lp.transpose()
    rows = a.rows_of_entries()
    vals = a.vals
    m, n = lp.m, lp.n
    row_div = np.ones(m)
    col_div = np.ones(n)
    if ruiz_iters > 0:
        rd_acc = np.ones(m)
        cd_acc = np.ones(n)
        for _ in range(ruiz_iters):
            dr = np.sqrt(a.with_values(vals).row_max_abs())
            dc = np.sqrt(_col_max_abs(a, at, vals))
            dr[dr == 0.0] = 1.0
            dc[dc == 0.0] = 1.0
            vals = vals / dr[rows] / dc[a.ci]
            rd_acc *= dr
            cd_acc *= dc
        row_div *= rd_acc
        col_div *= cd_acc
    if pock_chambolle:
        absv = np.abs(vals)
        col_sums = at.with_values(absv[at.perm]).matvec(np.ones(m))
        row_sums = a.with_values(absv).matvec(np.ones(n))
        dc = np.sqrt(col_sums)
        dr = np.sqrt(row_sums)
        dc[dc == 0.0] = 1.0
        dr[dr == 0.0] = 1.0
        vals = vals / dr[rows] / dc[a.ci]
        row_div *= dr
        col_div *= dc
    b = lp.b / row_div
    c = lp.c / col_div
    lower = lp.lower * col_div
    upper = lp.upper * col_div
    if bc_normalize:
        bf = float(np.linalg.norm(b)) + 1.0
        cf = float(np.linalg.norm(c)) + 1.0
        b = b / bf
        c = c / cf
        lower = lower / bf
        upper = upper / bf
    else:
        bf = cf = 1.0
    keep = vals != 0.0
    if np.all(keep):
        sa = a.with_values(vals)
        sat = at.with_values(vals[at.perm])
    else:  # underflow to zero is dropped by re-canonicalisation (scaling.py:107-109)
        rp, ci, v = canonical_csr(a.rp, a.ci, vals, n)
        sa = Csr(rp, ci, v, n, use_c=a.use_c)
        sat = None
    scaled = OracleLP(a=sa, b=b, c=c, lower=lower, upper=upper, m1=lp.m1,
                      objective_constant=lp.objective_constant,
                      objective_negated=lp.objective_negated, at=sat)
    return scaled, Scaling(row_div, col_div, bf, cf)


def identity_scaling(lp):
    return Scaling(np.ones(lp.m), np.ones(lp.n), 1.0, 1.0)


# ---------------------------------------------------------------------------
# power method (sparse.py:165-203)
# ---------------------------------------------------------------------------

@dataclass
class PowerEstimate:
    value: float
    raw: float
    iterations: int
    converged: bool


def power_lambda(lp: OracleLP, tol=1e-4, max_iters=5000):
    a, at = lp.a, lp.transpose()
    if a.nnz == 0:
        raise ValueError("matrix must be non-zero")
    v = np.ones(a.nrows)
    for fallback in range(a.nrows + 1):
        if np.linalg.norm(at.matvec(v)) > 0.0:
            break
        v = np.zeros(a.nrows)
        v[fallback] = 1.0
    v /= np.linalg.norm(v)
    lam_prev = 0.0
    lam = 0.0
    converged = False
    iters = 0
    for iters in range(1, max_iters + 1):
        w = a.matvec(at.matvec(v))
        lam = float(v @ w)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            break
        v = w / nw
        if iters > 1 and abs(lam - lam_prev) <= tol * max(abs(lam), 1e-300):
            converged = True
            break
        lam_prev = lam
    if not converged:
        warnings.warn(f"power method did not converge within {iters} iterations", RuntimeWarning)
    return PowerEstimate(lam * (1.0 + LAMBDA_SAFETY), lam, iters, converged)


# ---------------------------------------------------------------------------
# iteration core (core.py)
# ---------------------------------------------------------------------------

VARIANTS = ("dr", "hdr-fixed", "hdr", "hpr")


@dataclass
class State:
    y: np.ndarray
    x: np.ndarray
    ay: np.ndarray
    ax: np.ndarray
    sigma: float
    lam: float
    variant: str = "hpr"
    r: int = 0
    t: int = 0
    k: int = 0
    merit_first: float | None = None
    merit_prev: float = math.inf


class Breakdown(ArithmeticError):
    def __init__(self, k):
        super().__init__(f"non-finite iterate at iteration {k}")
        self.iteration = k


def iterate_once(st: State, lp: OracleLP):
    """core.py:163-174 + apply_variant_step 139-160."""
    at = lp.transpose()
    y, x, sigma = st.y, st.x, st.sigma
    lib = load_clib() if lp.a.use_c else None
    if lib is not None:
        return _iterate_once_c(lib, st, lp, at)
    v = x + sigma * (at.matvec(y) - lp.c)
    xb = np.clip(v, lp.lower, lp.upper)
    yb = y + (lp.b - lp.a.matvec(2.0 * xb - x)) / (st.lam * sigma)
    if lp.m1 < lp.m:
        np.maximum(yb[lp.m1:], 0.0, out=yb[lp.m1:])
    t2 = st.t + 2.0
    wn = (st.t + 1.0) / t2
    wa = 1.0 / t2
    if st.variant == "dr":
        yn, xn = yb, xb
    elif st.variant == "hpr":
        yn = wa * st.ay + wn * (2.0 * yb - y)
        xn = wa * st.ax + wn * (2.0 * xb - x)
    else:
        yn = wa * st.ay + wn * yb
        xn = wa * st.ax + wn * xb
    if not (np.all(np.isfinite(yn)) and np.all(np.isfinite(xn))):
        raise Breakdown(st.k)
    st.y, st.x = yn, xn
    st.t += 1
    st.k += 1
    return xb, yb


_VCODE = {"dr": 0, "hdr-fixed": 1, "hdr": 1, "hpr": 2}


def _iterate_once_c(lib, st, lp, at):
    """Same iteration through the fused C loops (bit-identical to the numpy path)."""
    n, m = lp.n, lp.m
    xb, w, xn = np.empty(n), np.empty(n), np.empty(n)
    yb, yn = np.empty(m), np.empty(m)
    vc = _VCODE[st.variant]
    bad = lib.orc_xphase(n, _lptr(at.rp), _lptr(at.ci), _dptr(at.vals), _dptr(st.y),
                         _dptr(st.x), _dptr(lp.c), _dptr(lp.lower), _dptr(lp.upper),
                         _dptr(st.ax), _dptr(xb), _dptr(w), _dptr(xn), st.sigma, st.t, vc)
    bad |= lib.orc_yphase(m, lp.m1, _lptr(lp.a.rp), _lptr(lp.a.ci), _dptr(lp.a.vals),
                          _dptr(w), _dptr(st.y), _dptr(lp.b), _dptr(st.ay), _dptr(yb),
                          _dptr(yn), st.lam * st.sigma, st.t, vc)
    if bad:
        raise Breakdown(st.k)
    st.y, st.x = yn, xn
    st.t += 1
    st.k += 1
    return xb, yb


def half_step(st: State, lp: OracleLP):
    """core.py:118-129."""
    at = lp.transpose()
    y, x, sigma = st.y, st.x, st.sigma
    v = x + sigma * (at.matvec(y) - lp.c)
    xb = np.clip(v, lp.lower, lp.upper)
    zb = (xb - v) / sigma
    yb = y + (lp.b - lp.a.matvec(2.0 * xb - x)) / (st.lam * sigma)
    if lp.m1 < lp.m:
        np.maximum(yb[lp.m1:], 0.0, out=yb[lp.m1:])
    return xb, yb, zb


def m_norm_diff(dy, dx, sigma, lp: OracleLP, lam):
    """core.py:182-201."""
    aty = lp.transpose().matvec(dy)
    shifted = dx + sigma * aty
    q = float(shifted @ shifted) / sigma
    if lam is not None:
        t1 = lam * float(dy @ dy) - float(aty @ aty)
        q += sigma * t1
        scale = sigma * lam * float(dy @ dy) + float(dx @ dx) / sigma
        if q < -1e-9 * max(scale, 1e-300):
            warnings.warn("negative quadratic form in the merit", RuntimeWarning)
    return float(np.sqrt(max(q, 0.0)))


def checkpoint_merit(st: State, xb, yb, lp):
    """core.py:210-218."""
    return 2.0 * m_norm_diff(st.y - yb, st.x - xb, st.sigma, lp, st.lam)


# ---------------------------------------------------------------------------
# residuals and driver (driver.py)
# ---------------------------------------------------------------------------

KKT_FIELDS = ("primal_infeas_abs", "primal_infeas_rel", "dual_infeas_abs", "dual_infeas_rel",
              "gap_abs", "gap_rel", "residual_vector_norm", "primal_objective",
              "dual_objective", "dual_clamped")


def kkt(lp: OracleLP, y, z, x):
    """driver.py:191-228."""
    ax = lp.a.matvec(x)
    prim = proj_dual_cone(lp.b - ax, lp.m1)
    pa = float(np.linalg.norm(prim))
    pr = pa / (1.0 + float(np.linalg.norm(lp.b)))
    dual_vec = lp.c - lp.transpose().matvec(y) - z
    da = float(np.linalg.norm(dual_vec))
    dr = da / (1.0 + float(np.linalg.norm(lp.c)))
    pobj = primal_obj(lp, x)
    dobj, clamped = dual_obj(lp, y, z)
    ga = abs(dobj - pobj)
    gr = ga / (1.0 + abs(dobj) + abs(pobj))
    r1 = y - proj_dual_cone(y - ax + lp.b, lp.m1)
    r2 = x - proj_box(x - z, lp.lower, lp.upper)
    stacked = math.sqrt(float(r1 @ r1) + float(r2 @ r2) + float(dual_vec @ dual_vec))
    return dict(primal_infeas_abs=pa, primal_infeas_rel=pr, dual_infeas_abs=da,
                dual_infeas_rel=dr, gap_abs=ga, gap_rel=gr, residual_vector_norm=stacked,
                primal_objective=pobj, dual_objective=dobj, dual_clamped=clamped)


def check_restart(merit_now, merit_first, merit_prev, t, k, a1, a2, a3):
    """driver.py:238-248."""
    if merit_now <= a1 * merit_first:
        return "sufficient"
    if merit_now <= a2 * merit_first and merit_now > merit_prev:
        return "stalled"
    if t >= a3 * k:
        return "long_loop"
    return None


def sigma_guards_pass(dx, dy, ep, ed):
    """driver.py:251-261."""
    lo, hi = DELTA_RANGE
    if not (lo < dx < hi and lo < dy < hi):
        return False
    if ep == 0.0:
        return ed == 0.0
    ratio = ed / ep
    return ERROR_RATIO_RANGE[0] < ratio < ERROR_RATIO_RANGE[1]


def sigma_update(bar_y, bar_x, anc_y, anc_x, lam, res):
    """driver.py:264-278."""
    dx = float(np.linalg.norm(bar_x - anc_x))
    dy = math.sqrt(lam) * float(np.linalg.norm(bar_y - anc_y))
    if not sigma_guards_pass(dx, dy, res["primal_infeas_rel"], res["dual_infeas_rel"]):
        return 1.0
    return dx / dy


@dataclass
class OracleConfig:
    """Mirror of SolverConfig defaults (driver.py:50-68)."""
    tolerance: float = 1e-8
    time_limit_seconds: float = math.inf
    max_iterations: int = 1_000_000
    check_interval: int = 150
    alpha1: float = 0.2
    alpha2: float = 0.6
    alpha3: float = 0.2
    sigma0: float = 1.0
    variant: str = "hpr"
    ruiz_iters: int = 10
    pock_chambolle: bool = True
    bc_normalize: bool = True
    power_tol: float = 1e-4
    power_max_iters: int = 5000
    termination_space: str = "original"


def solve(lp: OracleLP, cfg: OracleConfig | None = None, trace=None):
    """driver.py:281-405.  Returns a dict shaped like SolveReport.to_json_dict()
    plus 'solution' arrays, 'lambda_raw', 'power_iterations'.

    ``trace``: optional list; receives (k, y.copy(), x.copy()) after each of
    the first ``len``-bounded iterations when it is a list with attribute
    ``limit`` semantics -- used to compare trajectories.
    """
    cfg = cfg or OracleConfig()
    variant = cfg.variant
    uses_restarts = variant != "dr"
    updates_sigma = variant in ("hdr", "hpr")
    wall_start = time.perf_counter()
    timings = dict(scaling_seconds=0.0, power_method_seconds=0.0,
                   iteration_seconds=0.0, checkpoint_seconds=0.0)
    t0 = time.perf_counter()
    if cfg.ruiz_iters > 0 or cfg.pock_chambolle or cfg.bc_normalize:
        scaled, info = scale_lp(lp, cfg.ruiz_iters, cfg.pock_chambolle, cfg.bc_normalize)
    else:
        scaled, info = lp, identity_scaling(lp)
    timings["scaling_seconds"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    est = power_lambda(scaled, cfg.power_tol, cfg.power_max_iters)
    timings["power_method_seconds"] = time.perf_counter() - t0
    lam = est.value

    st = State(y=np.zeros(scaled.m), x=np.zeros(scaled.n), ay=np.zeros(scaled.m),
               ax=np.zeros(scaled.n), sigma=cfg.sigma0, lam=lam, variant=variant)
    term = lp if cfg.termination_space == "original" else scaled
    restart_log = []
    status = None
    res = None
    cand = None
    while status is None:
        steps = min(cfg.check_interval, cfg.max_iterations - st.k)
        t0 = time.perf_counter()
        try:
            for _ in range(max(steps, 0)):
                iterate_once(st, scaled)
                if trace is not None and st.k <= trace.limit:
                    trace.append((st.k, st.y.copy(), st.x.copy()))
        except Breakdown:
            timings["iteration_seconds"] += time.perf_counter() - t0
            status = "NumericalError"
            break
        timings["iteration_seconds"] += time.perf_counter() - t0

        t0 = time.perf_counter()
        xb, yb, zb = half_step(st, scaled)
        if cfg.termination_space == "original":
            cy, cz, cx = info.unscale(yb, zb, xb)
            cx = np.clip(cx, lp.lower, lp.upper)
        else:
            cy, cz, cx = yb, zb, xb
        cand = (cy, cz, cx)
        res = kkt(term, cy, cz, cx)
        if (res["gap_rel"] <= cfg.tolerance and res["primal_infeas_rel"] <= cfg.tolerance
                and res["dual_infeas_rel"] <= cfg.tolerance):
            status = "Optimal"
        elif st.k >= cfg.max_iterations:
            status = "IterationLimit"
        elif time.perf_counter() - wall_start >= cfg.time_limit_seconds:
            status = "TimeLimit"
        elif uses_restarts:
            merit_now = checkpoint_merit(st, xb, yb, scaled)
            if st.merit_first is None:
                st.merit_first = merit_now
                st.merit_prev = math.inf
            kind = check_restart(merit_now, st.merit_first, st.merit_prev, st.t, st.k,
                                 cfg.alpha1, cfg.alpha2, cfg.alpha3)
            if kind is not None:
                if updates_sigma:
                    sigma_next = sigma_update(yb, xb, st.ay, st.ax, lam, res)
                else:
                    sigma_next = st.sigma
                restart_log.append(dict(outer_index=st.r, trigger=kind, tau=st.t,
                                        sigma_next=sigma_next, merit=merit_now))
                st.ay, st.ax = yb.copy(), xb.copy()
                st.y, st.x = yb.copy(), xb.copy()
                st.sigma = sigma_next
                st.r += 1
                st.t = 0
                st.merit_first = None
                st.merit_prev = math.inf
            else:
                st.merit_prev = merit_now
        timings["checkpoint_seconds"] += time.perf_counter() - t0

    if cand is None or res is None:
        cand = (np.zeros(term.m), np.zeros(term.n), np.clip(np.zeros(term.n), term.lower, term.upper))
        res = kkt(term, *cand)
    if cfg.termination_space == "scaled":
        sy, sz, sx = info.unscale(*cand)
        sx = np.clip(sx, lp.lower, lp.upper)
    else:
        sy, sz, sx = cand
    pobj = primal_obj(lp, sx)
    dobj, _ = dual_obj(lp, sy, sz)
    if lp.objective_negated:
        pobj, dobj = -pobj, -dobj
    timings["solve_seconds"] = (timings["power_method_seconds"] + timings["iteration_seconds"]
                                + timings["checkpoint_seconds"])
    return dict(schema_version=1, status=status, primal_objective=pobj, dual_objective=dobj,
                kkt=res, iterations=st.k, restarts=st.r, restart_log=restart_log,
                timings=timings, sigma_final=st.sigma, lambda_estimate=lam,
                lambda_raw=est.raw, power_iterations=est.iterations,
                solution=dict(x=sx, y=sy, z=sz))


class Trace(list):
    """Collects (k, y, x) for k <= limit during ``solve``."""

    def __init__(self, limit):
        super().__init__()
        self.limit = limit
