"""Host-side problem types of the drop-in API.

Mirrors the reference's boundary types so code written against
``hprlp`` runs unchanged:

* ``SparseMatrix``   -- reference ``sparse.py:22-89`` (canonical CSR: sorted
  columns, duplicates summed, no explicit zeros; same field names and the same
  ``ValueError`` conditions).
* ``LpProblem``      -- reference ``problem.py:22-112`` (equality block first,
  ``>=`` inequality block, box bounds, objective constant / negation flag).
* ``PrimalDualPoint``-- reference ``problem.py:115-126``.
* ``project_onto_box`` / ``project_onto_dual_cone`` / ``primal_objective`` /
  ``dual_objective`` -- reference ``problem.py:129-176``.  These are host
  utilities for users of the API; ``solve`` never calls them -- its arithmetic
  runs in ``libhprlp_b200.so`` on the GPU.

``solve`` also accepts the reference's own ``LpProblem`` objects (duck typing:
``a_eq``/``a_ineq`` with ``row_offsets``/``col_indices``/``values``).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property
from typing import NamedTuple

import numpy as np


class DimensionMismatchError(ValueError):
    """Operand length does not match the matrix shape (reference sparse.py:18)."""


def _canonicalize(rows, cols, vals, nrows, ncols):
    """COO triplets -> canonical CSR arrays (duplicates summed, zeros dropped,
    columns ascending), the normal form of reference sparse.py:69-81."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    cols = np.asarray(cols, dtype=np.int64).reshape(-1)
    vals = np.asarray(vals, dtype=np.float64).reshape(-1)
    if rows.size and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0
                      or cols.max() >= ncols):
        raise ValueError("index out of range")
    key = rows * ncols + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    if key.size:
        first = np.ones(key.size, dtype=bool)
        first[1:] = key[1:] != key[:-1]
        seg = np.flatnonzero(first)
        summed = np.add.reduceat(vals, seg) if seg.size else vals
        ukey = key[seg]
    else:
        summed, ukey = vals, key
    keep = summed != 0.0
    summed, ukey = summed[keep], ukey[keep]
    r = ukey // ncols if ncols else ukey
    c = ukey - r * ncols
    offsets = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=nrows), out=offsets[1:])
    return offsets, c.astype(np.int64), summed.astype(np.float64)


@dataclass(frozen=True)
class SparseMatrix:
    """Immutable canonical CSR matrix (reference sparse.py:22-67)."""

    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    nrows: int
    ncols: int

    def __post_init__(self):
        ro, ci, v = self.row_offsets, self.col_indices, self.values
        if ro.shape != (self.nrows + 1,):
            raise ValueError("row_offsets must have length nrows + 1")
        if ro[0] != 0 or np.any(np.diff(ro) < 0):
            raise ValueError("row_offsets must be monotone and start at 0")
        if ro[-1] != len(v):
            raise ValueError("row_offsets[-1] must equal nnz")
        if len(ci) != len(v):
            raise ValueError("col_indices and values must have equal length")
        if v.size and np.any(v == 0.0):
            raise ValueError("explicit zeros are not allowed")
        if v.size:
            if ci.min() < 0 or ci.max() >= self.ncols:
                raise ValueError("column index out of range")
            row_start = np.zeros(len(ci), dtype=bool)
            starts = ro[:-1][np.diff(ro) > 0]
            row_start[starts] = True
            steps = np.diff(ci)
            if np.any(steps[~row_start[1:]] <= 0):
                raise ValueError("column indices must be strictly increasing within rows")

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    @classmethod
    def from_coo(cls, rows, cols, vals, shape) -> "SparseMatrix":
        ro, ci, v = _canonicalize(rows, cols, vals, int(shape[0]), int(shape[1]))
        return cls(ro, ci, v, int(shape[0]), int(shape[1]))

    @classmethod
    def from_dense(cls, arr) -> "SparseMatrix":
        a = np.atleast_2d(np.asarray(arr, dtype=np.float64))
        r, c = np.nonzero(a)
        return cls.from_coo(r, c, a[r, c], a.shape)

    @classmethod
    def from_scipy(cls, mat) -> "SparseMatrix":
        coo = mat.tocoo()
        return cls.from_coo(coo.row, coo.col, coo.data, coo.shape)

    @classmethod
    def from_csr_arrays(cls, row_offsets, col_indices, values, nrows, ncols) -> "SparseMatrix":
        """Trusting constructor for arrays already in canonical form (validated)."""
        return cls(np.asarray(row_offsets, np.int64), np.asarray(col_indices, np.int64),
                   np.asarray(values, np.float64), int(nrows), int(ncols))

    def to_dense(self) -> np.ndarray:
        d = np.zeros(self.shape)
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d


def vstack_csr(top, bottom):
    """[top; bottom] of two canonical CSR blocks with equal column counts
    (reference problem.py:75-82): concatenation keeps canonical form."""
    ro = np.concatenate([np.asarray(top.row_offsets[:-1], np.int64),
                         np.asarray(bottom.row_offsets, np.int64) + int(top.row_offsets[-1])])
    ci = np.concatenate([np.asarray(top.col_indices, np.int64),
                         np.asarray(bottom.col_indices, np.int64)])
    v = np.concatenate([np.asarray(top.values, np.float64), np.asarray(bottom.values, np.float64)])
    return ro, ci, v


@dataclass(frozen=True)
class LpProblem:
    """min <c,x> s.t. A1 x = b1, A2 x >= b2, lower <= x <= upper
    (reference problem.py:22-57, same validation)."""

    a_eq: SparseMatrix
    a_ineq: SparseMatrix
    b_eq: np.ndarray
    b_ineq: np.ndarray
    c: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    objective_constant: float = 0.0
    objective_negated: bool = False
    row_names: list | None = None
    col_names: list | None = None

    def __post_init__(self):
        n = self.a_eq.ncols
        if self.a_ineq.ncols != n:
            raise ValueError("equality and inequality blocks disagree on column count")
        if self.b_eq.shape != (self.a_eq.nrows,) or self.b_ineq.shape != (self.a_ineq.nrows,):
            raise ValueError("right-hand side lengths do not match the blocks")
        for name in ("c", "lower", "upper"):
            if getattr(self, name).shape != (n,):
                raise ValueError(f"{name} must have length {n}")
        if self.m < 1:
            raise ValueError("at least one constraint row is required")
        if self.a_eq.nnz + self.a_ineq.nnz == 0:
            raise ValueError("constraint matrix must be non-zero")
        if np.isnan(self.lower).any() or np.isnan(self.upper).any():
            raise ValueError("bounds must not contain NaN")
        if not (np.isfinite(self.c).all() and np.isfinite(self.b_eq).all()
                and np.isfinite(self.b_ineq).all()):
            raise ValueError("c and b must be finite")
        if np.any(self.lower > self.upper):
            raise ValueError("lower bound exceeds upper bound")

    @property
    def n(self) -> int:
        return self.a_eq.ncols

    @property
    def m1(self) -> int:
        return self.a_eq.nrows

    @property
    def m2(self) -> int:
        return self.a_ineq.nrows

    @property
    def m(self) -> int:
        return self.m1 + self.m2

    @cached_property
    def stacked_matrix(self) -> SparseMatrix:
        if self.m2 == 0:
            return self.a_eq
        if self.m1 == 0:
            return self.a_ineq
        ro, ci, v = vstack_csr(self.a_eq, self.a_ineq)
        return SparseMatrix(ro, ci, v, self.m, self.n)

    @cached_property
    def rhs(self) -> np.ndarray:
        return np.concatenate([self.b_eq, self.b_ineq])

    @classmethod
    def from_dense(cls, a_eq, b_eq, a_ineq, b_ineq, c, lower=None, upper=None,
                   **kwargs) -> "LpProblem":
        """Dense array-likes; empty blocks may be None (reference problem.py:89-112)."""
        c = np.asarray(c, dtype=np.float64)
        n = c.shape[0]
        if a_eq is None:
            a_eq, b_eq = np.zeros((0, n)), np.zeros(0)
        if a_ineq is None:
            a_ineq, b_ineq = np.zeros((0, n)), np.zeros(0)
        lower = np.zeros(n) if lower is None else np.asarray(lower, dtype=np.float64)
        upper = np.full(n, np.inf) if upper is None else np.asarray(upper, dtype=np.float64)
        blk = lambda a: SparseMatrix.from_dense(np.asarray(a, dtype=np.float64).reshape(-1, n))
        return cls(a_eq=blk(a_eq), a_ineq=blk(a_ineq),
                   b_eq=np.asarray(b_eq, dtype=np.float64).reshape(-1),
                   b_ineq=np.asarray(b_ineq, dtype=np.float64).reshape(-1),
                   c=c, lower=lower, upper=upper, **kwargs)


@dataclass
class PrimalDualPoint:
    """(y, z, x) candidate (reference problem.py:115-126)."""

    y: np.ndarray
    z: np.ndarray
    x: np.ndarray

    def check_dims(self, problem) -> None:
        m = problem.a_eq.nrows + problem.a_ineq.nrows
        n = problem.a_eq.ncols
        if self.y.shape != (m,) or self.z.shape != (n,) or self.x.shape != (n,):
            raise ValueError("point dimensions do not match the problem")


def project_onto_box(v, lower, upper):
    """Pi_C (reference problem.py:129-133)."""
    if v.shape != lower.shape or v.shape != upper.shape:
        raise ValueError("length mismatch in box projection")
    return np.clip(v, lower, upper)


def project_onto_dual_cone(v, m1):
    """Pi_D onto R^m1 x R^m2_+ (reference problem.py:136-143)."""
    if m1 < 0 or m1 > v.shape[0]:
        raise ValueError("m1 out of range")
    out = np.array(v, dtype=np.float64, copy=True)
    out[m1:] = np.maximum(out[m1:], 0.0)
    return out


def primal_objective(problem, x) -> float:
    """<c, x> + constant (reference problem.py:146-148)."""
    return float(problem.c @ x) + problem.objective_constant


class DualObjective(NamedTuple):
    value: float
    clamped: int


def dual_objective(problem, y, z) -> DualObjective:
    """<b,y> + sum_{z>0} l z + sum_{z<0} u z + constant; infinite active bounds
    contribute 0 and are counted (reference problem.py:156-176)."""
    rhs = np.concatenate([problem.b_eq, problem.b_ineq])
    lo_ok, up_ok = np.isfinite(problem.lower), np.isfinite(problem.upper)
    pos, neg = z > 0.0, z < 0.0
    clamped = int(np.count_nonzero(pos & ~lo_ok) + np.count_nonzero(neg & ~up_ok))
    val = float(rhs @ y)
    lo_take, up_take = pos & lo_ok, neg & up_ok
    if lo_take.any():
        val += float(problem.lower[lo_take] @ z[lo_take])
    if up_take.any():
        val += float(problem.upper[up_take] @ z[up_take])
    return DualObjective(val + problem.objective_constant, clamped)


def stacked_arrays(problem):
    """(row_offsets, col_indices, values, m, n, m1) of [A1; A2] for any
    reference-shaped problem (duck typing)."""
    top, bot = problem.a_eq, problem.a_ineq
    ro, ci, v = vstack_csr(top, bot)
    return ro, ci, v, int(top.nrows) + int(bot.nrows), int(top.ncols), int(top.nrows)
