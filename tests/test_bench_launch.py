"""bench.py launch contract on CPU: ``--gpus N`` without a torchrun
environment re-launches itself with N ranks (gloo dry run), and the default
workload is C3 on one GPU and the row-block C4 path on several."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_launches_n_ranks(n):
    got = _run("--gpus", str(n), "--dry-run")
    assert got["world_size"] == n and got["ranks_joined"] == n
    assert got["rank_sum"] == n * (n - 1) // 2
    assert got["config"] == "c4"                       # row-block path, not replicas
    assert got["NCCL_ALGO"] == "Ring" and got["NCCL_PROTO"] == "Simple"


def test_single_gpu_defaults_to_c3():
    got = _run("--dry-run")
    assert got["world_size"] == 1 and got["config"] == "c3"


def test_resolve_config():
    import bench
    assert bench.resolve_config("auto", 1) == "c3"
    assert bench.resolve_config("auto", 8) == "c4"
    assert bench.resolve_config("c2", 8) == "c2"


def test_reference_problem_bridge():
    """The reference arm hands the reference its own LpProblem type (skipped
    without baseline/_ref)."""
    import bench
    hprlp = bench.import_reference()
    if hprlp is None:
        pytest.skip("baseline/_ref not installed")
    from paper_2408_12179_b200 import generate_known_solution_lp
    prob, _ = generate_known_solution_lp(5, 6, 6, 30, 0.3)
    rp = bench.to_reference_problem(hprlp, prob)
    assert isinstance(rp, hprlp.LpProblem)
    assert rp.m == prob.m and rp.n == prob.n
