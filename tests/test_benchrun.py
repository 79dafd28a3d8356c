"""Bench harness against the reference's bench sweep.

CPU: SGM10 known answers (reference tests/test_cli.py:19-45 and values the
reference computed, tests/golden/bench_golden.json), CSV / summary formats,
CLI error codes.  GPU: the ablation sweep over the reference-written suite
gives the reference's per-instance status / iterations / restarts for every
variant; order independence (test_cli.py:141-155).
"""

import csv
import json
import math
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2408_12179_b200 import benchrun as BR

BG = json.load(open(f"{GOLDEN}/bench_golden.json"))


def _suite(tmp_path, count=4):
    for name in sorted(BG["suite"])[:count]:
        (tmp_path / name).write_text(BG["suite"][name])
    return sorted(tmp_path.glob("*.mps"))


@pytest.mark.parametrize("case", BG["sgm10_cases"])
def test_sgm10_matches_reference(case):
    times, limit, solved, ref = case
    # same formula, own arithmetic (numpy pairwise mean): agrees to rounding
    assert BR.sgm10(times, limit, solved) == pytest.approx(ref, rel=1e-13, abs=1e-13)


def test_sgm10_known_answers():
    assert BR.sgm10([10.0, 1000.0], 3600.0, [True, True]) == pytest.approx(132.1267, abs=1e-3)
    assert BR.sgm10([0.0, 0.0], 10.0, [True, True]) == pytest.approx(0.0, abs=1e-12)
    assert BR.sgm10([5.0, 1.0], 3600.0, [True, False]) == pytest.approx(
        math.sqrt(15.0 * 3610.0) - 10.0, rel=1e-12)
    rng = np.random.default_rng(0)
    for _ in range(10):
        n = int(rng.integers(1, 21))
        t = rng.uniform(0.0, 100.0, size=n).tolist()
        direct = np.prod([x + 10.0 for x in t]) ** (1.0 / n) - 10.0
        assert BR.sgm10(t, 1e9, [True] * n) == pytest.approx(direct, rel=1e-9)
    with pytest.raises(ValueError):
        BR.sgm10([], 1.0, [])
    with pytest.raises(ValueError):
        BR.sgm10([1.0], 1.0, [True, False])


def test_csv_columns_and_error_rows(tmp_path):
    assert BR.CSV_COLUMNS == BG["csv_columns"]
    run = BR.BenchRun(instances=["a.mps"], reports=[None], errors=["OSError: boom"],
                      tolerance=1e-6, time_limit=5.0)
    BR.write_bench_csv(run, tmp_path / "o.csv")
    rows = list(csv.reader(open(tmp_path / "o.csv")))
    assert rows[0] == BR.CSV_COLUMNS
    assert rows[1] == ["a.mps", "Error(OSError: boom)"] + [""] * 8
    s = BR.bench_summary({"hpr": run})["variants"]["hpr"]
    assert s["solved"] == 0 and s["total"] == 1 and s["sgm10"] == pytest.approx(5.0)
    assert s["per_instance"][0]["status"] == "Error(OSError: boom)"


def test_directory_errors(tmp_path):
    assert BR.bench_directory(tmp_path / "missing") == 1
    assert BR.bench_directory(tmp_path) == 1
    with pytest.raises(ValueError):
        BR.bench([], None, 1.0)


@pytest.mark.gpu
def test_ablation_sweep_matches_reference(tmp_path):
    _suite(tmp_path)
    js = tmp_path / "ab.json"
    cs = tmp_path / "ab.csv"
    from paper_2408_12179_b200 import SolverConfig
    code = BR.bench_directory(tmp_path, SolverConfig(tolerance=1e-6),
                              variants=["dr", "hdr-fixed", "hdr", "hpr"], csv_out=cs, json_out=js)
    assert code == 0
    got = json.loads(js.read_text())
    assert got["schema_version"] == BG["summary"]["schema_version"]
    assert set(got["variants"]) == set(BG["summary"]["variants"])
    for label, ref in BG["summary"]["variants"].items():
        g = got["variants"][label]
        assert (g["solved"], g["total"], g["median_iterations"]) == (
            ref["solved"], ref["total"], ref["median_iterations"]), label
        for gi, ri in zip(g["per_instance"], ref["per_instance"]):
            assert Path(gi["instance"]).name == ri["instance"]
            assert (gi["status"], gi["iterations"], gi["restarts"]) == (
                ri["status"], ri["iterations"], ri["restarts"]), (label, ri["instance"])
        lines = (tmp_path / f"ab.{label}.csv").read_text().strip().splitlines()
        assert len(lines) == 1 + len(ref["per_instance"])


@pytest.mark.gpu
def test_order_independent(tmp_path):
    from paper_2408_12179_b200 import SolverConfig
    paths = _suite(tmp_path, 3)
    cfg = SolverConfig(tolerance=1e-6)
    fwd = BR.bench(paths, cfg, math.inf)
    rev = BR.bench(list(reversed(paths)), cfg, math.inf)
    f = {p: (r.iterations, r.primal_objective) for p, r in zip(fwd.instances, fwd.reports)}
    r = {p: (q.iterations, q.primal_objective) for p, q in zip(rev.instances, rev.reports)}
    assert f == r
    assert fwd.solved_count == 3 and fwd.sgm10_value >= 0.0
