import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (several seconds)")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_reports():
    return load_json("reports.json")


@pytest.fixture(scope="session")
def golden_instances():
    return load_json("instances.json")


def problem_from_dict(d):
    """Small explicit instances stored by tests/golden/make_golden.py."""
    from paper_2408_12179_b200 import LpProblem
    n = d["n"]
    a_eq = np.array(d["a_eq"], dtype=float).reshape(-1, n) if d["a_eq"] else None
    a_in = np.array(d["a_ineq"], dtype=float).reshape(-1, n) if d["a_ineq"] else None
    return LpProblem.from_dense(a_eq, d["b_eq"] if a_eq is not None else None,
                                a_in, d["b_ineq"] if a_in is not None else None, d["c"],
                                np.array(d["lower"], dtype=float), np.array(d["upper"], dtype=float),
                                objective_negated=d["objective_negated"],
                                objective_constant=d["objective_constant"])


def one_d_problem():
    """reference tests/conftest.py:7-10: min x s.t. x = 1, x >= 0."""
    from paper_2408_12179_b200 import LpProblem
    return LpProblem.from_dense([[1.0]], [1.0], None, None, [1.0])


def bounded_tiny_lp(seed, n=4, m1=1, m2=2):
    """reference tests/conftest.py:13-25 (same RNG draws)."""
    from paper_2408_12179_b200 import LpProblem
    rng = np.random.default_rng(seed)
    lower = rng.uniform(-2.0, 0.0, size=n)
    upper = lower + rng.uniform(1.0, 3.0, size=n)
    a = rng.uniform(-2.0, 2.0, size=(m1 + m2, n))
    a[np.abs(a) < 0.3] += 0.5
    x0 = rng.uniform(lower + 0.1, upper - 0.1)
    b_eq = a[:m1] @ x0
    b_ineq = a[m1:] @ x0 - rng.uniform(0.2, 1.0, size=m2)
    c = rng.uniform(-1.5, 1.5, size=n)
    return LpProblem.from_dense(a[:m1], b_eq, a[m1:], b_ineq, c, lower, upper)


def acceptance_suite():
    """reference tests/test_acceptance.py:31-41."""
    specs = []
    for i in range(20):
        n = int(np.interp(i, [0, 19], [30, 200]))
        specs.append((1000 + i, max(2, n // 4), max(1, n // 4), n, min(1.0, 25.0 / n)))
    specs[-1] = (1019, 50, 50, 200, 0.25)
    return specs
