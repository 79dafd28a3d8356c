"""Instance-suite benchmark harness on the B200 path.

Same contract as the reference's ``hprlp bench`` sweep
(``/root/reference/pkg/src/hprlp/cli.py:29-149, 213-243``): solve every MPS
instance of a directory once per solver variant, charge unsolved instances at
the time limit, report the shifted geometric mean of solve times (SGM10, the
paper's convention, ``PAPER.md:414-418``), write one CSV per variant and a
JSON summary (schema v1).  The public names, argument meanings, CSV columns,
JSON keys and CLI exit codes are the reference's; the implementation is this
package's own:

* every instance is parsed once by the native MPS reader and kept for all
  variants (the reference re-parses per variant);
* every solve runs through the GPU ``solve`` on one device, so consecutive
  instances of the same shape reuse a pooled device residency
  (``driver.DEVICE_POOL``) -- SGM10 is a B200 number;
* a sweep is a list of ``Outcome`` records; ``BenchRun`` exposes them through
  the reference's field names (``instances`` / ``reports`` / ``errors``).
"""

from __future__ import annotations

import csv
import io
import json
import math
import statistics
import sys
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, NamedTuple

import numpy as np

from .driver import SolveReport, SolverConfig, SolveStatus, solve
from .mps import load_mps

SCHEMA_VERSION = 1
VARIANTS = ("dr", "hdr-fixed", "hdr", "hpr")
CSV_COLUMNS = ["instance", "status", "iterations", "restarts", "solve_seconds",
               "primal_objective", "dual_objective", "primal_infeas_rel",
               "dual_infeas_rel", "gap_rel"]


def sgm10(times, limit: float, solved, shift: float = 10.0) -> float:
    """Shifted geometric mean exp(mean(log(t + shift))) - shift, with every
    unsolved entry charged at ``limit`` (cli.py:29-43 semantics; ValueError on
    an empty or misaligned input)."""
    t = np.asarray(list(times), dtype=np.float64)
    ok = np.asarray(list(solved), dtype=bool)
    if t.size == 0:
        raise ValueError("need at least one time")
    if t.shape != ok.shape:
        raise ValueError("times and solved flags must align")
    charged = np.where(ok, t, float(limit)) + shift
    return float(np.exp(np.log(charged).mean()) - shift)


class Outcome(NamedTuple):
    """One instance of a sweep: a report, or the error that stopped it."""

    instance: str
    report: SolveReport | None
    error: str | None

    @property
    def solved(self) -> bool:
        return self.report is not None and self.report.status is SolveStatus.OPTIMAL

    def seconds(self, limit: float) -> float:
        return self.report.timings.solve_seconds if self.report is not None else limit

    def status_text(self) -> str:
        return self.report.status.value if self.report is not None else f"Error({self.error})"

    def csv_row(self) -> list:
        r = self.report
        if r is None:
            return [self.instance, self.status_text()] + [""] * (len(CSV_COLUMNS) - 2)
        k = r.kkt
        return [self.instance, r.status.value, r.iterations, r.restarts] + [
            repr(v) for v in (r.timings.solve_seconds, r.primal_objective, r.dual_objective,
                              k.primal_infeas_rel, k.dual_infeas_rel, k.gap_rel)]

    def summary_entry(self) -> dict:
        r = self.report
        return {"instance": self.instance, "status": self.status_text(),
                "iterations": None if r is None else r.iterations,
                "restarts": None if r is None else r.restarts,
                "solve_seconds": None if r is None else r.timings.solve_seconds}


@dataclass
class BenchRun:
    """One sweep (cli.py:46-77 field names): parallel lists of instance names,
    reports (None for a failed instance) and error strings."""

    instances: list[str]
    reports: list[SolveReport | None]
    errors: list[str | None]
    tolerance: float
    time_limit: float
    outcomes: list[Outcome] = field(init=False, repr=False)

    def __post_init__(self):
        if not (len(self.instances) == len(self.reports) == len(self.errors)):
            raise ValueError("instances, reports and errors must align")
        self.outcomes = [Outcome(i, r, e) for i, r, e in
                         zip(self.instances, self.reports, self.errors)]

    @classmethod
    def from_outcomes(cls, outcomes: list[Outcome], tolerance: float, time_limit: float):
        return cls([o.instance for o in outcomes], [o.report for o in outcomes],
                   [o.error for o in outcomes], tolerance, time_limit)

    @property
    def times(self) -> list[float]:
        return [o.seconds(self.time_limit) for o in self.outcomes]

    @property
    def solved_flags(self) -> list[bool]:
        return [o.solved for o in self.outcomes]

    @property
    def sgm10_value(self) -> float:
        return sgm10(self.times, self.time_limit, self.solved_flags)

    @property
    def solved_count(self) -> int:
        return int(np.count_nonzero(self.solved_flags))

    @property
    def iteration_counts(self) -> list[int]:
        return [o.report.iterations if o.report is not None else 0 for o in self.outcomes]

    def variant_summary(self) -> dict:
        counts = self.iteration_counts
        return {"tolerance": self.tolerance, "time_limit": self.time_limit,
                "sgm10": self.sgm10_value, "solved": self.solved_count,
                "total": len(self.outcomes),
                "median_iterations": statistics.median(counts) if counts else 0,
                "per_instance": [o.summary_entry() for o in self.outcomes]}


def _describe(exc: BaseException) -> str:
    return f"{type(exc).__name__}: {exc}"


def _solve_one(name: str, problem, cfg: SolverConfig, device: int) -> Outcome:
    try:
        return Outcome(name, solve(problem, cfg, device=device), None)
    except Exception as exc:           # one bad instance never stops the sweep
        return Outcome(name, None, _describe(exc))


def _load_all(paths: Iterable[Path]) -> list[tuple[str, object, str | None]]:
    """(name, problem or None, parse error or None) for every path."""
    out = []
    for p in paths:
        try:
            out.append((str(p), load_mps(p), None))
        except Exception as exc:
            out.append((str(p), None, _describe(exc)))
    return out


def _sweep(loaded, cfg: SolverConfig, time_limit: float, device: int) -> BenchRun:
    outs = [Outcome(name, None, err) if prob is None else _solve_one(name, prob, cfg, device)
            for name, prob, err in loaded]
    return BenchRun.from_outcomes(outs, cfg.tolerance, time_limit)


def bench(paths: list[Path], cfg: SolverConfig, time_limit: float, device: int = 0) -> BenchRun:
    """Solve every instance on the GPU, recording (not raising) per-instance
    failures (cli.py:80-97 contract)."""
    paths = list(paths)
    if not paths:
        raise ValueError("no instances to run")
    return _sweep(_load_all(paths), SolverConfig.coerce(cfg), time_limit, device)


def write_bench_csv(run: BenchRun, path: Path) -> None:
    """One row per instance; floats written with ``repr`` (cli.py:100-121 format)."""
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(CSV_COLUMNS)
    w.writerows(o.csv_row() for o in run.outcomes)
    Path(path).write_text(buf.getvalue(), newline="")


def bench_summary(runs: dict[str, BenchRun]) -> dict:
    """JSON summary, schema v1 (cli.py:124-149 keys)."""
    return {"schema_version": SCHEMA_VERSION,
            "variants": {label: run.variant_summary() for label, run in runs.items()}}


def _variant_config(cfg: SolverConfig, label: str, time_limit: float | None) -> SolverConfig:
    if label not in VARIANTS:
        raise ValueError(f"unknown variant {label!r}")
    kw = {name: getattr(cfg, name) for name in cfg.__dataclass_fields__}
    kw["variant"] = label
    if time_limit is not None:
        kw["time_limit_seconds"] = time_limit
    return SolverConfig(**kw)


def bench_directory(directory, cfg: SolverConfig | None = None, variants=None,
                    csv_out=None, json_out=None, time_limit: float | None = None,
                    device: int = 0, out=None) -> int:
    """``hprlp bench DIR [--variants LIST]`` (cli.py:213-243): every ``*.mps``
    in sorted order, once per variant; ``OUT.<label>.csv`` per variant when
    more than one, the JSON summary and the SGM10 table.  Exit code 1 for a
    missing or empty directory, else 0."""
    root = Path(directory)
    if not root.is_dir():
        print(f"error: not a directory: {root}", file=sys.stderr)
        return 1
    paths = sorted(root.glob("*.mps"))
    if not paths:
        print(f"error: no .mps instances in {root}", file=sys.stderr)
        return 1
    base_cfg = SolverConfig.coerce(cfg)
    limit = math.inf if time_limit is None else float(time_limit)
    labels = list(variants) if variants else [base_cfg.variant.value]
    cfgs = {label: _variant_config(base_cfg, label, time_limit) for label in labels}
    loaded = _load_all(paths)                     # parsed once for every variant
    runs = {label: _sweep(loaded, c, limit, device) for label, c in cfgs.items()}
    if csv_out:
        base = Path(csv_out)
        for label, run in runs.items():
            tag = f".{label}" if len(runs) > 1 else ""
            write_bench_csv(run, base.with_name(f"{base.stem}{tag}{base.suffix}"))
    summary = bench_summary(runs)
    if json_out:
        Path(json_out).write_text(json.dumps(summary, indent=2) + "\n")
    sink = out if out is not None else sys.stdout
    lines = ["variant  sgm10  solved/total"] + [
        f"{label:9s} {run.sgm10_value:10.4f}  {run.solved_count}/{len(run.instances)}"
        for label, run in runs.items()]
    sink.write("\n".join(lines) + "\n")
    return 0
