"""Instance-suite benchmark harness on the B200 path.

The reference's ``bench`` sweep (``/root/reference/pkg/src/hprlp/cli.py``)
solves a directory of MPS instances, charges unsolved ones at the time limit,
and reports the shifted geometric mean of solve times (SGM10, the paper's
reporting convention) per solver variant, with a CSV per variant and a JSON
summary.  This module keeps those names, argument meanings, output formats and
error behaviour; every solve runs through the GPU ``solve`` (one device
context, reused across instances through the residency pool), so the times
are B200 times.

* ``sgm10``            cli.py:29-43
* ``BenchRun``         cli.py:46-77
* ``bench``            cli.py:80-97
* ``CSV_COLUMNS`` / ``write_bench_csv``   cli.py:100-121
* ``bench_summary``    cli.py:124-149
* ``bench_directory``  cli.py:213-243 (``hprlp bench DIR [--variants LIST]``)
"""

from __future__ import annotations

import csv
import json
import math
import statistics
import sys
from dataclasses import dataclass
from pathlib import Path

from .driver import SolveReport, SolverConfig, SolveStatus, solve
from .mps import load_mps

SCHEMA_VERSION = 1
VARIANTS = ("dr", "hdr-fixed", "hdr", "hpr")


def sgm10(times: list[float], limit: float, solved: list[bool], shift: float = 10.0) -> float:
    """Shifted geometric mean of solve times in log space; unsolved entries are
    charged at ``limit`` (cli.py:29-43)."""
    if not times:
        raise ValueError("need at least one time")
    if len(times) != len(solved):
        raise ValueError("times and solved flags must align")
    charged = [t if ok else limit for t, ok in zip(times, solved)]
    return math.exp(sum(math.log(t + shift) for t in charged) / len(charged)) - shift


@dataclass
class BenchRun:
    """One sweep over a list of instances (cli.py:46-77)."""

    instances: list[str]
    reports: list[SolveReport | None]
    errors: list[str | None]
    tolerance: float
    time_limit: float

    @property
    def times(self) -> list[float]:
        return [r.timings.solve_seconds if r is not None else self.time_limit
                for r in self.reports]

    @property
    def solved_flags(self) -> list[bool]:
        return [r is not None and r.status is SolveStatus.OPTIMAL for r in self.reports]

    @property
    def sgm10_value(self) -> float:
        return sgm10(self.times, self.time_limit, self.solved_flags)

    @property
    def solved_count(self) -> int:
        return sum(self.solved_flags)

    @property
    def iteration_counts(self) -> list[int]:
        return [r.iterations if r is not None else 0 for r in self.reports]


def bench(paths: list[Path], cfg: SolverConfig, time_limit: float, device: int = 0) -> BenchRun:
    """Solve every instance on the GPU; per-instance failures are recorded, not
    raised (cli.py:80-97)."""
    if not paths:
        raise ValueError("no instances to run")
    reports: list[SolveReport | None] = []
    errors: list[str | None] = []
    for path in paths:
        try:
            problem = load_mps(path)
            reports.append(solve(problem, cfg, device=device))
            errors.append(None)
        except Exception as exc:   # keep the batch going
            reports.append(None)
            errors.append(f"{type(exc).__name__}: {exc}")
    return BenchRun(instances=[str(p) for p in paths], reports=reports, errors=errors,
                    tolerance=cfg.tolerance, time_limit=time_limit)


CSV_COLUMNS = ["instance", "status", "iterations", "restarts", "solve_seconds",
               "primal_objective", "dual_objective", "primal_infeas_rel",
               "dual_infeas_rel", "gap_rel"]


def write_bench_csv(run: BenchRun, path: Path) -> None:
    """One row per instance, floats as ``repr`` (cli.py:100-121)."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(CSV_COLUMNS)
        for name, report, err in zip(run.instances, run.reports, run.errors):
            if report is None:
                writer.writerow([name, f"Error({err})"] + [""] * 8)
                continue
            writer.writerow([
                name, report.status.value, report.iterations, report.restarts,
                repr(report.timings.solve_seconds),
                repr(report.primal_objective), repr(report.dual_objective),
                repr(report.kkt.primal_infeas_rel), repr(report.kkt.dual_infeas_rel),
                repr(report.kkt.gap_rel),
            ])


def bench_summary(runs: dict[str, BenchRun]) -> dict:
    """JSON summary, schema v1 (cli.py:124-149)."""
    out = {"schema_version": SCHEMA_VERSION, "variants": {}}
    for label, run in runs.items():
        counts = run.iteration_counts
        out["variants"][label] = {
            "tolerance": run.tolerance,
            "time_limit": run.time_limit,
            "sgm10": run.sgm10_value,
            "solved": run.solved_count,
            "total": len(run.instances),
            "median_iterations": statistics.median(counts) if counts else 0,
            "per_instance": [
                {
                    "instance": name,
                    "status": r.status.value if r else f"Error({err})",
                    "iterations": r.iterations if r else None,
                    "restarts": r.restarts if r else None,
                    "solve_seconds": r.timings.solve_seconds if r else None,
                }
                for name, r, err in zip(run.instances, run.reports, run.errors)
            ],
        }
    return out


def bench_directory(directory, cfg: SolverConfig | None = None, variants=None,
                    csv_out=None, json_out=None, time_limit: float | None = None,
                    device: int = 0, out=None) -> int:
    """``hprlp bench DIR`` (cli.py:213-243): every ``*.mps`` in sorted order,
    once per variant label; a CSV per variant (``OUT.<label>.csv`` when more
    than one), the JSON summary, and the SGM10 table.  Returns the CLI exit
    code: 1 for a missing or empty directory, else 0."""
    root = Path(directory)
    if not root.is_dir():
        print(f"error: not a directory: {root}", file=sys.stderr)
        return 1
    paths = sorted(root.glob("*.mps"))
    if not paths:
        print(f"error: no .mps instances in {root}", file=sys.stderr)
        return 1
    cfg = cfg if cfg is not None else SolverConfig()
    limit = time_limit if time_limit is not None else math.inf
    labels = list(variants) if variants else [cfg.variant.value]
    runs: dict[str, BenchRun] = {}
    for label in labels:
        if label not in VARIANTS:
            raise ValueError(f"unknown variant {label!r}")
        kw = {f: getattr(cfg, f) for f in cfg.__dataclass_fields__}
        kw["variant"] = label
        if time_limit is not None:
            kw["time_limit_seconds"] = time_limit
        runs[label] = bench(paths, SolverConfig(**kw), limit, device=device)
    for label, run in runs.items():
        suffix = f".{label}" if len(runs) > 1 else ""
        if csv_out:
            base = Path(csv_out)
            write_bench_csv(run, base.with_name(base.stem + suffix + base.suffix))
    summary = bench_summary(runs)
    out = out if out is not None else sys.stdout
    if json_out:
        Path(json_out).write_text(json.dumps(summary, indent=2) + "\n")
    print("variant  sgm10  solved/total", file=out)
    for label, run in runs.items():
        print(f"{label:9s} {run.sgm10_value:10.4f}  {run.solved_count}/{len(run.instances)}",
              file=out)
    return 0
