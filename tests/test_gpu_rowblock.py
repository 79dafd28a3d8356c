"""GPU parity of the row-block partitioned path.

The P ranks run in one process on one B200 (local transport: the collectives
are kernels) -- the same per-rank kernels, reduce-scatter / all-gather
structure and rank-order scalar sums the NCCL transport runs across GPUs.  The
NCCL transport itself is exercised at world size 1 (a real communicator; the
collectives degenerate to copies) through ``solve_distributed``.

Bars (north_star): P-rank vs reference trajectory within 1e-10 normwise over
the first 100 iterations; identical status, iteration count and restart
triggers; objectives and relative residuals within 1e-8.  P = 1 is bit-exact
with the single-context path (same per-row sums, no cross-rank sum).
"""

import os
import socket

import numpy as np
import pytest

import paper_2408_12179_b200 as P
from conftest import GOLDEN
from oracle import hprlp_oracle as O
from paper_2408_12179_b200.rowblock import RowBlockGroup, solve_partitioned
from test_gpu_parity import assert_report_parity

pytestmark = pytest.mark.gpu


def _traj_rel(y, x, ry, rx):
    return np.sqrt(np.sum((y - ry) ** 2) + np.sum((x - rx) ** 2)) / np.sqrt(
        np.sum(ry ** 2) + np.sum(rx ** 2))


@pytest.mark.parametrize("parts,chunks,ts", [(1, 1, 0), (2, 1, 0), (3, 1, 0), (5, 1, 0), (2, 3, 0),
                                             (4, 2, 0), (1, 1, 1), (3, 1, 1)])
def test_partitioned_trajectory_c1(parts, chunks, ts, monkeypatch):
    """ts = 1: every rank's A_g^T partial (and y-phase) on the TS engine."""
    monkeypatch.setenv("HPR_RB_CHUNKS", str(chunks))
    monkeypatch.setenv("HPR_TS", str(ts))
    d = np.load(f"{GOLDEN}/c1_golden.npz")
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    grp = RowBlockGroup.local(prob, parts)
    grp.analyze()
    grp.scale(10, True, True)
    est = grp.power(1e-4, 5000)
    lam = est.raw * 1.001
    grp.state_reset()
    done = 0
    for i, k in enumerate(d["snap_k"]):
        grp.run_inner(int(k) - done, done, done, 1.0, lam, 2)
        done = int(k)
        rel = _traj_rel(grp.to_host("y"), grp.to_host("x"), d["snap_y"][i], d["snap_x"][i])
        assert rel <= 1e-10, (parts, k, rel)
    grp.close()


def test_partition_one_is_bit_exact_with_single_context():
    from paper_2408_12179_b200.device import DeviceLP
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    dev = DeviceLP(prob)
    dev.analyze()
    dev.scale(10, True, True)
    lam = dev.power(1e-4, 5000).raw * 1.001
    dev.state_reset()
    dev.run_inner(60, 0, 0, 0.9, lam * 0.9, 2)
    grp = RowBlockGroup.local(prob, 1)
    grp.analyze()
    grp.scale(10, True, True)
    lam2 = grp.power(1e-4, 5000).raw * 1.001
    assert lam2 == lam
    grp.state_reset()
    grp.run_inner(60, 0, 0, 0.9, lam * 0.9, 2)
    assert np.array_equal(grp.to_host("y"), dev.to_host("y"))
    assert np.array_equal(grp.to_host("x"), dev.to_host("x"))
    grp.close()
    dev.close()


@pytest.mark.parametrize("parts,chunks", [(1, 1), (3, 1), (2, 3)])
def test_partitioned_column_split_bit_exact(parts, chunks, monkeypatch):
    """The column-split y-phase (A's columns in blocks, running sums carried
    block to block) lands on the same bits as the unsplit one."""
    monkeypatch.setenv("HPR_RB_CHUNKS", str(chunks))
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    out = []
    for split in ("0", "300"):
        if split == "0":
            monkeypatch.setenv("HPR_SPLIT", "0")
            monkeypatch.delenv("HPR_SPLIT_COLS", raising=False)
        else:
            monkeypatch.delenv("HPR_SPLIT", raising=False)
            monkeypatch.setenv("HPR_SPLIT_COLS", split)
        grp = RowBlockGroup.local(prob, parts)
        grp.analyze()
        assert all((b.layout_info()["split_a"] == 7) == (split != "0") for b in grp.blocks)
        grp.scale(10, True, True)
        lam = grp.power(1e-4, 5000).raw * 1.001
        grp.state_reset()
        grp.run_inner(60, 0, 0, 0.9, lam * 0.9, 2)
        out.append((grp.to_host("y"), grp.to_host("x")))
        grp.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("parts", [2, 4])
def test_partitioned_scaling_and_power(parts):
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    grp = RowBlockGroup.local(prob, parts)
    grp.analyze()
    sc = grp.scale(10, True, True)
    scaled, info = O.scale_lp(O.OracleLP.from_problem(prob))
    # Ruiz maxima are exact under any split; PC sums differ only in rounding
    rs = grp.to_host("row_scale")
    cs = grp.to_host("col_scale")
    assert np.max(np.abs(rs - info.row_scale) / info.row_scale) <= 1e-14
    assert np.max(np.abs(cs - info.col_scale) / info.col_scale) <= 1e-14
    assert abs(sc.b_factor - info.b_factor) <= 1e-13 * info.b_factor
    est = grp.power(1e-4, 5000)
    oest = O.power_lambda(scaled)
    assert est.iterations == oest.iterations
    assert abs(est.raw - oest.raw) <= 1e-12 * oest.raw
    grp.close()


@pytest.mark.parametrize("parts,chunks", [(2, 1), (4, 1), (3, 2)])
def test_partitioned_solve_c1_vs_reference(golden_reports, parts, chunks, monkeypatch):
    monkeypatch.setenv("HPR_RB_CHUNKS", str(chunks))
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    for key in ("c1", "c1_1e-8"):
        g = golden_reports[key]
        rep = solve_partitioned(prob, P.SolverConfig(**g["cfg"]), parts=parts)
        assert_report_parity(rep, g["report"], f"{key} P={parts}")


@pytest.mark.parametrize("parts", [2, 3])
def test_partitioned_acceptance_subset(golden_reports, parts):
    for i, entry in enumerate(golden_reports["acceptance_suite"]):
        if i % 5:
            continue
        prob, _ = P.generate_known_solution_lp(*entry["args"])
        rep = solve_partitioned(prob, P.SolverConfig(**entry["cfg"]), parts=parts)
        assert_report_parity(rep, entry["report"], f"{entry['args']} P={parts}")


def test_partitioned_solution_matches_single():
    prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
    cfg = P.SolverConfig(tolerance=1e-8)
    a = P.solve(prob, cfg)
    b = solve_partitioned(prob, cfg, parts=3)
    for u, v in ((a.solution.x, b.solution.x), (a.solution.y, b.solution.y),
                 (a.solution.z, b.solution.z)):
        assert u.shape == v.shape
        assert np.linalg.norm(u - v) <= 1e-8 * max(1.0, np.linalg.norm(u))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("chunks,ts", [(1, 0), (3, 0), (1, 1), (3, 1)])
def test_nccl_transport_world1(golden_reports, chunks, ts, monkeypatch):
    """chunks > 1 runs the overlapped pipeline (comm stream, per-chunk events,
    chunked NCCL reduce-scatter / all-gather) -- with one rank the collectives
    are copies, but the captured multi-stream graph is the P-GPU one.  ts = 1:
    the A^T partial on the TS engine, planned per column chunk when chunked."""
    monkeypatch.setenv("HPR_RB_CHUNKS", str(chunks))
    monkeypatch.setenv("HPR_TS", str(ts))
    monkeypatch.setenv("HPR_RB_NCCL_P1", "1")      # keep the NCCL collectives at one rank
    import torch
    import torch.distributed as dist
    from paper_2408_12179_b200 import _native as N
    from paper_2408_12179_b200.rowblock import solve_distributed
    assert N.load_library().hpr_nccl_available() == 1
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        prob, _ = P.generate_known_solution_lp(1, 500, 500, 2000, 0.01)
        g = golden_reports["c1"]
        rep = solve_distributed(prob, P.SolverConfig(**g["cfg"]), device=0)
        assert_report_parity(rep, g["report"], "c1 nccl world 1")
    finally:
        dist.destroy_process_group()
