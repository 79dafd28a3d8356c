"""Instance generators: the restated reference generator reproduces the
reference's instances bit for bit (hashes recorded from the reference by
tests/golden/make_golden.py); the C3 flow generator is canonical and feasible."""

import hashlib

import numpy as np
import pytest

import paper_2408_12179_b200 as P


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode()).hexdigest()


def problem_hash(p, pt):
    d = {}
    for blk in ("a_eq", "a_ineq"):
        m = getattr(p, blk)
        for f in ("row_offsets", "col_indices", "values"):
            d[f"{blk}.{f}"] = sha(np.asarray(getattr(m, f)))
    for f in ("b_eq", "b_ineq", "c", "lower", "upper"):
        d[f] = sha(getattr(p, f))
    for f in ("x", "y", "z"):
        d[f"star.{f}"] = sha(getattr(pt, f))
    return d


@pytest.mark.parametrize("name", ["c1", "c5_0", "c5_1", "small"])
def test_known_solution_generator_matches_reference(golden_instances, name):
    g = golden_instances[name]
    p, pt = P.generate_known_solution_lp(*g["args"])
    assert problem_hash(p, pt) == g["hash"]


@pytest.mark.slow
def test_c2_generator_matches_reference(golden_instances):
    g = golden_instances["c2"]
    p, pt = P.generate_known_solution_lp(*g["args"])
    assert problem_hash(p, pt) == g["hash"]


def test_planted_point_is_kkt():
    """SPEC mps_io: the planted triple satisfies the KKT system."""
    p, pt = P.generate_known_solution_lp(3, 2, 2, 7, 0.5)
    a = p.stacked_matrix.to_dense()
    assert np.max(np.abs(a[:p.m1] @ pt.x - p.b_eq)) <= 1e-12
    assert np.all(a[p.m1:] @ pt.x - p.b_ineq >= -1e-12)
    assert np.max(np.abs(a.T @ pt.y + pt.z - p.c)) <= 1e-12


def test_flow_generator_structure():
    V, K = 64, 4
    p = P.generate_flow_lp(5, nodes=V, out_degree=4, commodities=K)
    E = V * 4
    assert p.m1 == V * K and p.m2 == E and p.n == E * K + K
    a = p.stacked_matrix
    assert a.nnz == 3 * E * K + 2 * K
    # every arc variable: +1 in its tail's row, -1 in its head's row, -1 in its capacity row
    at = a.to_dense().T
    for col in (0, 5, E * K - 1):
        nz = at[col][at[col] != 0]
        assert sorted(nz.tolist()) == [-1.0, -1.0, 1.0]
    # all-bypass flow is feasible
    x = np.zeros(p.n)
    demand = np.zeros(K)
    b = p.rhs
    for k in range(K):
        demand[k] = b[:p.m1].reshape(V, K)[:, k].max()
    x[E * K:] = demand
    d = a.to_dense()
    assert np.allclose(d[:p.m1] @ x, p.b_eq)
    assert np.all(d[p.m1:] @ x >= p.b_ineq - 1e-12)


def test_planted_fast_generator_is_kkt():
    p, pt = P.generate_planted_lp_fast(7, 20, 20, 80, 6)
    a = p.stacked_matrix.to_dense()
    assert np.max(np.abs(a[:p.m1] @ pt.x - p.b_eq)) <= 1e-12
    assert np.all(a[p.m1:] @ pt.x - p.b_ineq >= -1e-12)
    assert np.max(np.abs(a.T @ pt.y + pt.z - p.c)) <= 1e-12
    assert np.all((pt.x >= p.lower) & (pt.x <= p.upper))


def test_planted_block_generator_split_invariant_and_kkt():
    """C4 row blocks: identical rows under any split; the assembled problem has
    the planted point as an exact KKT point (oracle kkt_residual)."""
    from oracle import hprlp_oracle as O
    from paper_2408_12179_b200 import LpProblem, SparseMatrix
    from paper_2408_12179_b200.generators import _planted_columns, generate_planted_block
    m1, m2, n, per = 300, 400, 3000, 12
    cols = _planted_columns(4, n)
    whole = generate_planted_block(4, m1, m2, n, per, 0, m1 + m2, cols)
    parts = [generate_planted_block(4, m1, m2, n, per, a, b, cols)
             for a, b in ((0, 123), (123, 500), (500, 700))]
    assert np.array_equal(np.concatenate([p[1] for p in parts]), whole[1])
    assert np.array_equal(np.concatenate([p[2] for p in parts]), whole[2])
    assert np.array_equal(np.concatenate([p[3] for p in parts]), whole[3])
    assert [p[5] for p in parts] == [123, 177, 0]
    rp, ci, va, b, ys, _, (lo, up, xs, zs), cpart = whole
    c = cpart + zs
    prob = LpProblem(a_eq=SparseMatrix.from_csr_arrays(rp[:m1 + 1], ci[:rp[m1]], va[:rp[m1]], m1, n),
                     a_ineq=SparseMatrix.from_csr_arrays(rp[m1:] - rp[m1], ci[rp[m1]:], va[rp[m1]:],
                                                         m2, n),
                     b_eq=b[:m1], b_ineq=b[m1:], c=c, lower=lo, upper=up)
    res = O.kkt(O.OracleLP.from_problem(prob), ys, zs, xs)
    assert res["primal_infeas_rel"] < 1e-12 and res["dual_infeas_rel"] < 1e-12
    assert res["gap_rel"] < 1e-11
