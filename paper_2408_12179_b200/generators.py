"""Synthetic LP instances for the benchmark configurations.

* ``generate_known_solution_lp`` -- reference ``mps.py:524-610`` restated with
  the same ``numpy.random.default_rng`` call sequence, so the same seed gives a
  bit-identical instance (pinned in tests against fixtures produced by the
  reference).  Used for C1, C2 and C5.  Its row loop is inherently sequential
  (``rng.choice`` without replacement per row), exactly as in the reference.
* ``generate_flow_lp`` -- multicommodity min-cost flow (config C3; no reference
  generator exists).  Vectorised; variables arc-major / commodity-minor so the
  capacity rows and the per-node conservation blocks gather contiguous 8*K-byte
  segments of the iterate.
* ``generate_planted_lp_fast`` -- vectorised planted-solution LP with the
  distribution of ``mps.py:524-610`` but a different RNG stream (config C4
  scale, where the reference's Python row loop is infeasible).

These run on the host; they create solver input and are not part of the
solve path.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .problem import LpProblem, PrimalDualPoint, SparseMatrix


def _csr_block(csr) -> SparseMatrix:
    csr = sp.csr_matrix(csr)
    csr.sum_duplicates()
    csr.eliminate_zeros()
    csr.sort_indices()
    return SparseMatrix(csr.indptr.astype(np.int64), csr.indices.astype(np.int64),
                        csr.data.astype(np.float64), csr.shape[0], csr.shape[1])


def generate_known_solution_lp(seed: int, m1: int, m2: int, n: int, density: float = 0.3):
    """Random sparse LP with a planted optimal triple (reference mps.py:524-610).

    Returns ``(LpProblem, PrimalDualPoint)``; the point satisfies the KKT
    system to machine precision.
    """
    if n < m1:
        raise ValueError("need n >= m1")
    if not 0.0 < density <= 1.0:
        raise ValueError("density must be in (0, 1]")
    if m1 + m2 < 1:
        raise ValueError("need at least one row")
    rng = np.random.default_rng(seed)
    m = m1 + m2
    k_row = min(max(1, int(round(density * n))), n)
    row_cols, row_vals = [], []
    for _ in range(m):
        for _attempt in range(16):
            cols = rng.choice(n, size=k_row, replace=False)
            vals = rng.uniform(-2.0, 2.0, size=cols.size)
            tiny = np.abs(vals) < 0.1
            vals[tiny] += np.sign(vals[tiny] + 0.5) * 0.5
            if np.any(vals != 0.0):
                break
        else:
            raise RuntimeError("could not draw a non-zero row")
        row_cols.append(cols)
        row_vals.append(vals)
    rows = np.repeat(np.arange(m), k_row)
    a_csr = sp.csr_matrix((np.concatenate(row_vals), (rows, np.concatenate(row_cols))),
                          shape=(m, n))
    a_csr.sum_duplicates()
    a_csr.eliminate_zeros()
    a_csr.sort_indices()

    lower = np.zeros(n)
    upper = np.full(n, np.inf)
    kinds = rng.choice(4, size=n, p=[0.6, 0.2, 0.1, 0.1])
    boxed = kinds == 1
    lower[boxed] = rng.uniform(-1.0, 0.5, size=int(boxed.sum()))
    upper[boxed] = lower[boxed] + rng.uniform(0.5, 2.0, size=int(boxed.sum()))
    lower[kinds == 2] = -np.inf
    up_only = kinds == 3
    lower[up_only] = -np.inf
    upper[up_only] = rng.uniform(0.0, 2.0, size=int(up_only.sum()))

    x_star = np.empty(n)
    z_star = np.zeros(n)
    for j in range(n):
        lo, hi = lower[j], upper[j]
        roll = rng.uniform()
        if roll < 0.2 and np.isfinite(lo):
            x_star[j] = lo
            z_star[j] = rng.uniform(0.3, 1.5)
        elif roll < 0.4 and np.isfinite(hi):
            x_star[j] = hi
            z_star[j] = -rng.uniform(0.3, 1.5)
        else:
            a = lo if np.isfinite(lo) else -1.5
            bnd = hi if np.isfinite(hi) else a + 3.0
            x_star[j] = rng.uniform(a + 0.1, bnd - 0.1) if bnd - a > 0.2 else lo
            if x_star[j] == lo:
                z_star[j] = rng.uniform(0.3, 1.5)

    ax = a_csr @ x_star                      # csr_matvec order, as the reference
    b_eq = ax[:m1].copy()
    b_ineq = np.empty(m2)
    y_star = np.zeros(m)
    y_star[:m1] = rng.normal(size=m1)
    for i in range(m2):
        if rng.uniform() < 0.5:
            y_star[m1 + i] = rng.uniform(0.3, 1.5)
            b_ineq[i] = ax[m1 + i]
        else:
            b_ineq[i] = ax[m1 + i] - rng.uniform(0.5, 2.0)
    c = sp.csr_matrix(a_csr.T) @ y_star + z_star
    problem = LpProblem(a_eq=_csr_block(a_csr[:m1]), a_ineq=_csr_block(a_csr[m1:]),
                        b_eq=b_eq, b_ineq=b_ineq, c=c, lower=lower, upper=upper)
    return problem, PrimalDualPoint(y=y_star, z=z_star, x=x_star)


# ---------------------------------------------------------------------------
# C3: multicommodity flow
# ---------------------------------------------------------------------------

def generate_flow_lp(seed: int = 3, nodes: int = 1 << 18, out_degree: int = 4,
                     commodities: int = 32, bypass_cost: float = 1e3) -> LpProblem:
    """Multicommodity min-cost flow LP.

    Graph: ``nodes`` vertices, arc e = v*out_degree + j leaves v to a uniform
    random head != v.  Commodity k ships demand d_k ~ U(1,10) from s_k to t_k;
    a bypass arc s_k -> t_k (cost ``bypass_cost``, uncapacitated) keeps every
    instance feasible.  Variables x[e*K + k] >= 0 (arc-major), then the K
    bypass flows.  Rows: conservation (v, k) at v*K + k (equalities, m1 = V*K),
    then capacity -sum_k x[e,k] >= -cap_e (m2 = E), cap_e ~ U(5,50).
    Costs per arc ~ U(1,10), shared by the commodities.
    """
    rng = np.random.default_rng(seed)
    V, D, K = int(nodes), int(out_degree), int(commodities)
    E = V * D
    tail = np.repeat(np.arange(V, dtype=np.int64), D)
    head = rng.integers(0, V - 1, size=E, dtype=np.int64)
    head += head >= tail                                   # no self loops
    src = rng.integers(0, V, size=K)
    dst = rng.integers(0, V - 1, size=K)
    dst += dst >= src
    demand = rng.uniform(1.0, 10.0, size=K)
    cap = rng.uniform(5.0, 50.0, size=E)
    cost = rng.uniform(1.0, 10.0, size=E)
    n_arc = E * K
    n = n_arc + K
    m1 = V * K

    # incident arcs per node, sorted by arc id: (node, arc, sign)
    inc_node = np.concatenate([tail, head])
    inc_arc = np.concatenate([np.arange(E, dtype=np.int64), np.arange(E, dtype=np.int64)])
    inc_sgn = np.concatenate([np.ones(E), -np.ones(E)])
    order = np.lexsort((inc_arc, inc_node))
    inc_node, inc_arc, inc_sgn = inc_node[order], inc_arc[order], inc_sgn[order]
    deg = np.bincount(inc_node, minlength=V)
    node_start = np.zeros(V + 1, dtype=np.int64)
    np.cumsum(deg, out=node_start[1:])

    # conservation row (v, k) lengths: deg(v) + bypass incidences
    extra = np.zeros((V, K), dtype=np.int64)
    np.add.at(extra, (src, np.arange(K)), 1)
    np.add.at(extra, (dst, np.arange(K)), 1)
    cons_len = (deg[:, None] + extra).reshape(-1)
    cap_len = np.full(E, K, dtype=np.int64)
    rp = np.zeros(m1 + E + 1, dtype=np.int64)
    np.cumsum(np.concatenate([cons_len, cap_len]), out=rp[1:])
    nnz = int(rp[-1])
    ci = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)

    # arc entries of conservation rows: q over incident entries, k over commodities
    q = np.arange(2 * E, dtype=np.int64)
    local = q - node_start[inc_node]
    for k in range(K):
        rows = inc_node * K + k
        pos = rp[rows] + local
        ci[pos] = inc_arc * K + k
        val[pos] = inc_sgn
    # bypass entries (largest column ids -> appended at the row end)
    for k in range(K):
        for v, sgn in ((src[k], 1.0), (dst[k], -1.0)):
            row = v * K + k
            pos = rp[row + 1] - 1          # src_k != dst_k: at most one per row
            ci[pos] = n_arc + k
            val[pos] = sgn
    # capacity rows
    base = rp[m1]
    ci[base:] = (np.arange(E, dtype=np.int64)[:, None] * K + np.arange(K)).reshape(-1)
    val[base:] = -1.0

    b = np.zeros(m1 + E)
    b[src * K + np.arange(K)] += demand
    b[dst * K + np.arange(K)] -= demand
    b[m1:] = -cap
    c = np.empty(n)
    c[:n_arc] = np.repeat(cost, K)
    c[n_arc:] = bypass_cost
    a_eq = SparseMatrix.from_csr_arrays(rp[:m1 + 1], ci[:base], val[:base], m1, n)
    a_ineq = SparseMatrix.from_csr_arrays(rp[m1:] - base, ci[base:], val[base:], E, n)
    return LpProblem(a_eq=a_eq, a_ineq=a_ineq, b_eq=b[:m1], b_ineq=b[m1:], c=c,
                     lower=np.zeros(n), upper=np.full(n, np.inf))


# ---------------------------------------------------------------------------
# C4-scale planted LP (vectorised)
# ---------------------------------------------------------------------------

def generate_planted_lp_fast(seed: int, m1: int, m2: int, n: int, per_row: int):
    """Planted-solution LP with the distribution of mps.py:524-610, vectorised.

    Each row draws ``per_row`` distinct columns (rejection of duplicates by
    sorting and resampling), values U(-2,2) nudged away from 0 as in the
    reference; bounds, x*, z*, y* follow the same mixture.  Returns
    ``(LpProblem, PrimalDualPoint)``.
    """
    rng = np.random.default_rng(seed)
    m = m1 + m2
    cols = np.sort(rng.integers(0, n, size=(m, per_row), dtype=np.int64), axis=1)
    for _ in range(64):
        dup = np.zeros_like(cols, dtype=bool)
        dup[:, 1:] = cols[:, 1:] == cols[:, :-1]
        nd = int(dup.sum())
        if nd == 0:
            break
        cols[dup] = rng.integers(0, n, size=nd, dtype=np.int64)
        cols.sort(axis=1)
    vals = rng.uniform(-2.0, 2.0, size=(m, per_row))
    tiny = np.abs(vals) < 0.1
    vals[tiny] += np.sign(vals[tiny] + 0.5) * 0.5
    rp = np.arange(0, m * per_row + 1, per_row, dtype=np.int64)
    ci = cols.reshape(-1)
    va = vals.reshape(-1)
    a = sp.csr_matrix((va, ci, rp), shape=(m, n))

    lower = np.zeros(n)
    upper = np.full(n, np.inf)
    kinds = rng.choice(4, size=n, p=[0.6, 0.2, 0.1, 0.1])
    boxed = kinds == 1
    lower[boxed] = rng.uniform(-1.0, 0.5, size=int(boxed.sum()))
    upper[boxed] = lower[boxed] + rng.uniform(0.5, 2.0, size=int(boxed.sum()))
    lower[kinds == 2] = -np.inf
    lower[kinds == 3] = -np.inf
    upper[kinds == 3] = rng.uniform(0.0, 2.0, size=int((kinds == 3).sum()))
    roll = rng.uniform(size=n)
    x = np.empty(n)
    z = np.zeros(n)
    at_lo = (roll < 0.2) & np.isfinite(lower)
    at_up = ~at_lo & (roll < 0.4) & np.isfinite(upper)
    inter = ~(at_lo | at_up)
    x[at_lo] = lower[at_lo]
    z[at_lo] = rng.uniform(0.3, 1.5, size=int(at_lo.sum()))
    x[at_up] = upper[at_up]
    z[at_up] = -rng.uniform(0.3, 1.5, size=int(at_up.sum()))
    a0 = np.where(np.isfinite(lower), lower, -1.5)
    b0 = np.where(np.isfinite(upper), upper, a0 + 3.0)
    wide = inter & (b0 - a0 > 0.2)
    x[wide] = rng.uniform(a0[wide] + 0.1, b0[wide] - 0.1)
    narrow = inter & ~wide
    x[narrow] = lower[narrow]
    z[narrow] = rng.uniform(0.3, 1.5, size=int(narrow.sum()))
    ax = a @ x
    y = np.zeros(m)
    y[:m1] = rng.normal(size=m1)
    active = rng.uniform(size=m2) < 0.5
    y[m1:][active] = rng.uniform(0.3, 1.5, size=int(active.sum()))
    b = ax.copy()
    b[m1:][~active] -= rng.uniform(0.5, 2.0, size=int((~active).sum()))
    c = a.T @ y + z
    a_eq = SparseMatrix.from_csr_arrays(rp[:m1 + 1], ci[:m1 * per_row], va[:m1 * per_row], m1, n)
    a_ineq = SparseMatrix.from_csr_arrays(rp[m1:] - rp[m1], ci[m1 * per_row:],
                                          va[m1 * per_row:], m2, n)
    prob = LpProblem(a_eq=a_eq, a_ineq=a_ineq, b_eq=b[:m1], b_ineq=b[m1:], c=c,
                     lower=lower, upper=upper)
    return prob, PrimalDualPoint(y=y, z=z, x=x)


# ---------------------------------------------------------------------------
# C4: one rank's row block of a planted LP, generated independently per rank
# ---------------------------------------------------------------------------

_CHUNK = 1 << 16


def _planted_columns(seed, n):
    """Bounds, x*, z* of the planted LP (identical on every rank)."""
    rng = np.random.default_rng([seed, 0])
    lower = np.zeros(n)
    upper = np.full(n, np.inf)
    kinds = rng.choice(4, size=n, p=[0.6, 0.2, 0.1, 0.1])
    boxed = kinds == 1
    lower[boxed] = rng.uniform(-1.0, 0.5, size=int(boxed.sum()))
    upper[boxed] = lower[boxed] + rng.uniform(0.5, 2.0, size=int(boxed.sum()))
    lower[kinds >= 2] = -np.inf
    upper[kinds == 3] = rng.uniform(0.0, 2.0, size=int((kinds == 3).sum()))
    roll = rng.uniform(size=n)
    x = np.empty(n)
    z = np.zeros(n)
    at_lo = (roll < 0.2) & np.isfinite(lower)
    at_up = ~at_lo & (roll < 0.4) & np.isfinite(upper)
    inter = ~(at_lo | at_up)
    x[at_lo] = lower[at_lo]
    z[at_lo] = rng.uniform(0.3, 1.5, size=int(at_lo.sum()))
    x[at_up] = upper[at_up]
    z[at_up] = -rng.uniform(0.3, 1.5, size=int(at_up.sum()))
    a0 = np.where(np.isfinite(lower), lower, -1.5)
    b0 = np.where(np.isfinite(upper), upper, a0 + 3.0)
    wide = inter & (b0 - a0 > 0.2)
    x[wide] = rng.uniform(a0[wide] + 0.1, b0[wide] - 0.1)
    narrow = inter & ~wide
    x[narrow] = lower[narrow]
    z[narrow] = rng.uniform(0.3, 1.5, size=int(narrow.sum()))
    return lower, upper, x, z


def generate_planted_block(seed: int, m1: int, m2: int, n: int, per_row: int, r0: int, r1: int,
                           columns=None):
    """Rows [r0, r1) of the C4 planted LP (distribution of mps.py:524-610).

    Rows are drawn in chunks of 65536 from ``default_rng([seed, 1 + chunk])``,
    so a row's content does not depend on how the rows are split over ranks.
    Returns ``(row_offsets, col_indices, values, b_block, y_block, m1_local,
    (lower, upper, x*, z*), c_partial)`` where ``c_partial = A_block^T y*_block``
    -- summing it over all blocks and adding z* gives the cost vector.
    """
    lower, upper, xs, zs = columns if columns is not None else _planted_columns(seed, n)
    rows = r1 - r0
    cols = np.empty((rows, per_row), dtype=np.int64)
    vals = np.empty((rows, per_row))
    ys = np.empty(rows)
    slack = np.zeros(rows)
    for ch in range(r0 // _CHUNK, (r1 - 1) // _CHUNK + 1):
        c0, c1 = ch * _CHUNK, min((ch + 1) * _CHUNK, m1 + m2)
        rng = np.random.default_rng([seed, 1 + ch])
        cc = np.sort(rng.integers(0, n, size=(c1 - c0, per_row), dtype=np.int64), axis=1)
        for _ in range(64):
            dup = np.zeros_like(cc, dtype=bool)
            dup[:, 1:] = cc[:, 1:] == cc[:, :-1]
            nd = int(dup.sum())
            if nd == 0:
                break
            cc[dup] = rng.integers(0, n, size=nd, dtype=np.int64)
            cc.sort(axis=1)
        vv = rng.uniform(-2.0, 2.0, size=(c1 - c0, per_row))
        tiny = np.abs(vv) < 0.1
        vv[tiny] += np.sign(vv[tiny] + 0.5) * 0.5
        gi = np.arange(c0, c1)
        yy = rng.normal(size=c1 - c0)
        active = rng.uniform(size=c1 - c0) < 0.5
        ineq = gi >= m1
        yy[ineq] = np.where(active[ineq], rng.uniform(0.3, 1.5, size=int(ineq.sum())), 0.0)
        sl = np.where(ineq & ~active, rng.uniform(0.5, 2.0, size=c1 - c0), 0.0)
        lo, hi = max(c0, r0), min(c1, r1)
        cols[lo - r0:hi - r0] = cc[lo - c0:hi - c0]
        vals[lo - r0:hi - r0] = vv[lo - c0:hi - c0]
        ys[lo - r0:hi - r0] = yy[lo - c0:hi - c0]
        slack[lo - r0:hi - r0] = sl[lo - c0:hi - c0]
    rp = np.arange(0, rows * per_row + 1, per_row, dtype=np.int64)
    ci = cols.reshape(-1)
    va = vals.reshape(-1)
    a = sp.csr_matrix((va, ci, rp), shape=(rows, n))
    b = a @ xs - slack
    c_partial = a.T @ ys
    m1_local = int(min(max(m1 - r0, 0), rows))
    return rp, ci, va, b, ys, m1_local, (lower, upper, xs, zs), c_partial


# named benchmark configurations
def config_instance(name: str):
    name = name.lower()
    if name == "c1":
        return generate_known_solution_lp(1, 500, 500, 2000, 0.01)[0], 1e-4
    if name == "c2":
        return generate_known_solution_lp(2, 50_000, 50_000, 200_000, 2.5e-4)[0], 1e-8
    if name == "c3":
        return generate_flow_lp(3), 1e-8
    if name == "c3-lite":
        return generate_flow_lp(3, nodes=1 << 10, commodities=8), 1e-8
    raise ValueError(f"unknown config {name}")
