"""The drop-in boundary exercised with the reference's OWN objects.

The reference package (``hprlp``, installed from /root/reference into
baseline/_ref by the documented pip command; skipped when absent) builds the
problems and configs -- its ``LpProblem``, ``SolverConfig`` and ``Variant`` --
and they are passed straight to this package's ``solve`` / ``kkt_residual``.
The reference's own ``solve`` runs on the same objects in the same process and
its report is the oracle (live, not a fixture).
"""

import os
import sys

import numpy as np
import pytest

import paper_2408_12179_b200 as P
from test_gpu_parity import assert_report_parity

pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "baseline", "_ref")


@pytest.fixture(scope="module")
def hprlp():
    if not os.path.isdir(os.path.join(REF_DIR, "hprlp")):
        pytest.skip("reference not installed in baseline/_ref")
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    import hprlp as mod
    return mod


def _ref_dict(rep):
    d = rep.to_json_dict(include_solution=False)
    d.pop("timings")
    return d


@pytest.mark.parametrize("variant", ["HPR", "HDR", "HDR_FIXED_SIGMA", "DR"])
def test_reference_problem_config_variant(hprlp, variant):
    prob, _ = hprlp.generate_known_solution_lp(1007, 12, 10, 80, 0.3)
    cfg = hprlp.SolverConfig(tolerance=1e-7, variant=getattr(hprlp.Variant, variant),
                             max_iterations=200_000)
    ours = P.solve(prob, cfg)
    ref = hprlp.solve(prob, cfg)
    assert_report_parity(ours, _ref_dict(ref), variant)
    assert np.allclose(ours.solution.x, ref.solution.x, rtol=1e-7, atol=1e-9)


def test_reference_c1_objects(hprlp):
    prob, _ = hprlp.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    for tol in (1e-4, 1e-8):
        cfg = hprlp.SolverConfig(tolerance=tol)
        assert_report_parity(P.solve(prob, cfg), _ref_dict(hprlp.solve(prob, cfg)), str(tol), tol)


def test_reference_mps_and_max_problem(hprlp):
    """A reference-parsed MPS problem (OBJSENSE MAX, ranges, bounds) solved
    from the reference's object."""
    text = """NAME          MAXREF
OBJSENSE
    MAX
ROWS
 N  obj
 L  c1
 G  c2
 E  c3
 L  c4
COLUMNS
    x1        obj       3.0        c1        1.0
    x1        c2        1.0        c3        1.0
    x2        obj       2.0        c1        1.0
    x2        c4        1.0
    x3        obj       -1.0       c3        1.0
    x3        c2        2.0
RHS
    rhs       c1        4.0        c2        1.0
    rhs       c3        3.0        c4        2.5
RANGES
    rng       c4        2.0
BOUNDS
 UP bnd       x1        3.0
 LO bnd       x3        -1.0
 UP bnd       x3        5.0
ENDATA
"""
    prob = hprlp.parse_mps(text)
    cfg = hprlp.SolverConfig(tolerance=1e-9)
    assert_report_parity(P.solve(prob, cfg), _ref_dict(hprlp.solve(prob, cfg)), "mps_max", 1e-9)


def test_reference_kkt_residual(hprlp):
    prob, pt = hprlp.generate_known_solution_lp(31, 20, 15, 90, 0.2)
    rng = np.random.default_rng(4)
    point = hprlp.PrimalDualPoint(y=pt.y + 0.01 * rng.normal(size=pt.y.size),
                                  z=pt.z + 0.01 * rng.normal(size=pt.z.size),
                                  x=pt.x + 0.01 * rng.normal(size=pt.x.size))
    ours = P.kkt_residual(prob, point).to_dict()
    ref = hprlp.kkt_residual(prob, point).to_dict()
    for k, v in ref.items():
        assert abs(ours[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, ours[k], v)
