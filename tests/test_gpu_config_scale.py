"""Config-scale parity (C2 and C3, BASELINE.json configs[1], configs[2]).

* C2 / C3 first 100 iterates against the REFERENCE's own trajectory
  (tests/golden/make_traj_golden.py ran hprlp's scale_problem ->
  power_method_lambda_max -> iterate_once x 100 on the same instance):
  lambda within 1e-12 with the same power-iteration count, per-snapshot norms
  and the iterate (C2: the whole vector at k = 100; C3: 4096 sampled entries
  of y and of x) normwise within 1e-10.
* C3, 100 fused iterations on the device's scaled problem bit-identical to
  the oracle's sequential C kernels (same lambda).
* C3 full solve to 1e-8 against the oracle's full solve
  (c3_oracle_report.json): status, iteration count, restart log, sigma and
  all KKT fields (assert_report_parity).

The instances are regenerated here and pinned by the sha256 the fixture
script recorded.
"""

import json
import os

import numpy as np
import pytest

import paper_2408_12179_b200 as P
from conftest import GOLDEN
from oracle import hprlp_oracle as O
from test_gpu_parity import _dev, _oracle_on_device_scaling, assert_report_parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _inst_sha(p):
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "make_traj_golden", os.path.join(GOLDEN, "make_traj_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.inst_sha(p)


def _fixture(name):
    path = os.path.join(GOLDEN, f"{name}_traj.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path}: run tests/golden/make_traj_golden.py")
    return np.load(path)


def _norm(t):
    import torch
    return float(torch.linalg.vector_norm(t).item())


def _trajectory_check(name, prob, d, full=False):
    import torch
    assert _inst_sha(prob) == str(d["inst_sha"]), "generator output changed"
    dev = _dev(prob)
    est = dev.power(1e-4, 5000)
    assert est.iterations == int(d["power_iterations"])
    assert abs(est.raw - float(d["lam"][1])) <= 1e-12 * float(d["lam"][1])
    lam = est.raw * 1.001
    dev.state_reset()
    done = 0
    iy = torch.from_numpy(d["idx_y"]).to(dev.device)
    ix = torch.from_numpy(d["idx_x"]).to(dev.device)
    probes = None
    if "dots" in d.files:
        rng = np.random.default_rng(int(d["probe_seed"]))
        probes = (torch.from_numpy(rng.uniform(-1.0, 1.0, prob.m)).to(dev.device),
                  torch.from_numpy(rng.uniform(-1.0, 1.0, prob.n)).to(dev.device))
    for i, k in enumerate(d["snap_k"]):
        dev.run_inner(int(k) - done, done, done, 1.0, lam, 2)
        done = int(k)
        dev.synchronize()
        y, x = dev.t["y"], dev.t["x"][:prob.n]
        ny, nx = d["norms"][k - 1]
        assert abs(_norm(y) - ny) <= 1e-10 * ny and abs(_norm(x) - nx) <= 1e-10 * nx, (name, k)
        if probes is not None:
            # whole-iterate checksums y.r_m, x.r_n (summation order differs from
            # numpy's: bounded by 1e-10 |v| |r|)
            for v, r, ref in ((y, probes[0], d["dots"][i][0]), (x, probes[1], d["dots"][i][1])):
                got = float(torch.dot(v, r).item())
                assert abs(got - ref) <= 1e-10 * _norm(v) * _norm(r), (name, k, got, ref)
        gy, gx = y[iy].cpu().numpy(), x[ix].cpu().numpy()
        ry, rx = d["snap_y"][i], d["snap_x"][i]
        num = np.sqrt(np.sum((gy - ry) ** 2) + np.sum((gx - rx) ** 2))
        den = np.sqrt(np.sum(ry ** 2) + np.sum(rx ** 2))
        # early iterates can be zero at every sampled entry: then exactly zero
        assert num <= 1e-10 * den if den > 0 else num == 0.0, (name, k, num, den)
    if full:
        y, x = dev.to_host("y"), dev.to_host("x")
        ry, rx = d["y100"], d["x100"]
        rel = np.sqrt(np.sum((y - ry) ** 2) + np.sum((x - rx) ** 2)) / np.sqrt(
            np.sum(ry ** 2) + np.sum(rx ** 2))
        assert rel <= 1e-10, (name, rel)
    return dev, lam


def test_c2_trajectory_vs_reference():
    prob, _ = P.generate_known_solution_lp(2, 50_000, 50_000, 200_000, 2.5e-4)
    dev, _ = _trajectory_check("c2", prob, _fixture("c2"), full=True)
    dev.close()


@pytest.fixture(scope="module")
def c3():
    return P.generate_flow_lp(3)


def test_c3_trajectory_vs_reference_and_bit_exact_vs_oracle(c3):
    dev, lam = _trajectory_check("c3", c3, _fixture("c3"))
    # the same 100 iterations on the oracle's C kernels, on the device's scaled
    # problem and lambda: bit-identical
    lib = O.load_clib()
    assert lib is not None, "oracle C kernels not built (make -C oracle)"
    lib.orc_set_threads(os.cpu_count() or 1)
    y100, x100 = dev.to_host("y"), dev.to_host("x")
    slp = _oracle_on_device_scaling(dev, c3)
    dev.close()
    st = O.State(np.zeros(slp.m), np.zeros(slp.n), np.zeros(slp.m), np.zeros(slp.n), 1.0, lam)
    for _ in range(100):
        O.iterate_once(st, slp)
    assert np.array_equal(y100, st.y) and np.array_equal(x100, st.x)


def test_c3_full_solve_vs_oracle(c3):
    path = os.path.join(GOLDEN, "c3_oracle_report.json")
    g = json.load(open(path))
    assert _inst_sha(c3) == g["inst_sha"]
    rep = P.solve(c3, P.SolverConfig(tolerance=1e-8))
    assert rep.status is P.SolveStatus.OPTIMAL
    assert_report_parity(rep, g, "c3")
    for f in ("x", "y", "z"):
        ref = g["solution_norm"][f]
        got = float(np.linalg.norm(getattr(rep.solution, f)))
        assert abs(got - ref) <= 1e-8 * max(1.0, ref), (f, got, ref)
