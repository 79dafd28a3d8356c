"""Golden fixture for the bench harness, produced by the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_bench_golden.py

Writes ``tests/golden/bench_golden.json``: the MPS texts of a small instance
suite (reference ``write_mps`` of ``generate_known_solution_lp(40 + seed, 2, 2,
8, 0.5)``, as in the reference's tests/test_cli.py:113-118), the reference's
``bench_summary`` of the ablation sweep dr,hdr-fixed,hdr,hpr at tol 1e-6
(solve times dropped: they are host times), the CSV header and the SGM10
known answers of tests/test_cli.py:19-45.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from hprlp import generate_known_solution_lp, write_mps  # noqa: E402
from hprlp.cli import (CSV_COLUMNS, bench, bench_summary, sgm10,  # noqa: E402
                       _config_from_args)

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    suite = {}
    for seed in range(4):
        prob, _ = generate_known_solution_lp(40 + seed, m1=2, m2=2, n=8, density=0.5)
        suite[f"inst{seed}.mps"] = write_mps(prob)
    with tempfile.TemporaryDirectory() as td:
        for name, text in suite.items():
            Path(td, name).write_text(text)
        paths = sorted(Path(td).glob("*.mps"))
        runs = {}
        for label in ("dr", "hdr-fixed", "hdr", "hpr"):
            ns = argparse.Namespace(tol="1e-6", variant=label, check_interval=150, sigma0=1.0,
                                    termination_space="original", max_iterations=1_000_000,
                                    time_limit=None, no_scaling=False)
            runs[label] = bench(paths, _config_from_args(ns), math.inf)
        summ = bench_summary(runs)
    for v in summ["variants"].values():
        v.pop("sgm10")
        v.pop("time_limit")
        for inst in v["per_instance"]:
            inst["instance"] = os.path.basename(inst["instance"])
            inst.pop("solve_seconds")
    sg = [
        [[10.0, 1000.0], 3600.0, [True, True], sgm10([10.0, 1000.0], 3600.0, [True, True])],
        [[0.0, 0.0], 10.0, [True, True], sgm10([0.0, 0.0], 10.0, [True, True])],
        [[5.0, 1.0], 3600.0, [True, False], sgm10([5.0, 1.0], 3600.0, [True, False])],
        [[0.5, 2.0, 30.0], 100.0, [False, True, True], sgm10([0.5, 2.0, 30.0], 100.0,
                                                             [False, True, True])],
    ]
    out = {"suite": suite, "summary": summ, "csv_columns": CSV_COLUMNS, "sgm10_cases": sg}
    with open(os.path.join(HERE, "bench_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote bench_golden.json")


if __name__ == "__main__":
    main()
