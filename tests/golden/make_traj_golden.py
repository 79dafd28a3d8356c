"""Config-scale golden fixtures (C2, C3) from the REFERENCE and the oracle.

Run in the build container (where /root/reference exists):

    python tests/golden/make_traj_golden.py c2        # ~1 min
    python tests/golden/make_traj_golden.py c3        # ~5 min (reference) + the oracle solve
    python tests/golden/make_traj_golden.py c3-solve  # oracle full C3 solve (~20 min, 8 cores)

Writes:

* ``c2_traj.npz`` / ``c3_traj.npz`` -- the reference's own first 100 HPR
  iterates (``hprlp``: ``scale_problem`` -> ``ProblemData.from_problem`` ->
  ``power_method_lambda_max`` -> ``iterate_once`` x 100, i.e. the preamble of
  ``driver.solve``, driver.py:293-309, and core.py:163-174): per-iteration
  norms of y and x, the entries of y and x at ~4096 sampled indices (half
  from the support of the k = 100 iterate) at the snapshot iterations, the
  checksums y.r_m and x.r_n at the snapshots (r: fixed uniform(-1, 1) probe
  vectors from ``probe_seed``), lambda and the power-iteration count; C2 also the
  full (y, x) at k = 100.  The instance is this package's generator output,
  pinned by the sha256 of every array (``inst_sha``).
* ``c3_oracle_report.json`` -- the oracle's full C3 solve to 1e-8 (the
  reference's algorithm with sequential C kernels; bit-identical to the
  reference on the same machine, tests/test_oracle_golden.py): status,
  iterations, restart log, sigma_final, objectives, KKT fields, solution norms.
  A full solve with the reference itself would take about an hour on one core.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
SNAP_K = (1, 10, 50, 100)
NSAMPLE = 4096


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode()).hexdigest()


def instance(name):
    from paper_2408_12179_b200.generators import config_instance
    return config_instance(name)[0]


def inst_sha(p) -> str:
    h = hashlib.sha256()
    for blk in (p.a_eq, p.a_ineq):
        for a in (blk.row_offsets, blk.col_indices, blk.values):
            h.update(sha(np.asarray(a)).encode())
    for a in (p.b_eq, p.b_ineq, p.c, p.lower, p.upper):
        h.update(sha(np.asarray(a)).encode())
    return h.hexdigest()


def reference_problem(hprlp, p):
    from hprlp.sparse import SparseMatrix as RS

    def blk(a):
        return RS(np.asarray(a.row_offsets, np.int64), np.asarray(a.col_indices, np.int64),
                  np.asarray(a.values, np.float64), int(a.nrows), int(a.ncols))
    return hprlp.LpProblem(a_eq=blk(p.a_eq), a_ineq=blk(p.a_ineq), b_eq=np.asarray(p.b_eq),
                           b_ineq=np.asarray(p.b_ineq), c=np.asarray(p.c),
                           lower=np.asarray(p.lower), upper=np.asarray(p.upper))


def reference_trajectory(name, full_snapshot):
    sys.path.insert(0, "/root/reference/pkg/src")
    import hprlp
    from hprlp.core import ProblemData, SolverState, iterate_once
    from hprlp.scaling import scale_problem
    from hprlp.sparse import power_method_lambda_max
    t0 = time.time()
    p = instance(name)
    print(f"{name}: generated in {time.time() - t0:.1f}s", flush=True)
    digest = inst_sha(p)
    rp = reference_problem(hprlp, p)
    del p
    scaled, info = scale_problem(rp)
    data = ProblemData.from_problem(scaled)
    print(f"{name}: scaled at {time.time() - t0:.1f}s", flush=True)
    est = power_method_lambda_max(data.a)
    print(f"{name}: lambda {est.raw!r} after {est.iterations} steps at {time.time() - t0:.1f}s",
          flush=True)
    st = SolverState.origin(data, sigma=1.0, lam=est.value)
    rng = np.random.default_rng(12345)
    # fixed probe vectors: per-snapshot checksums y.r_m, x.r_n over the whole iterate
    rm, rn = rng.uniform(-1.0, 1.0, data.m), rng.uniform(-1.0, 1.0, data.n)
    norms, snaps, dots = [], {}, []
    for k in range(1, 101):
        iterate_once(st, data)
        y, x = st.current.y, st.current.x
        norms.append((float(np.linalg.norm(y)), float(np.linalg.norm(x))))
        if k in SNAP_K:
            snaps[k] = (y.copy(), x.copy())
            dots.append((float(y @ rm), float(x @ rn)))
    print(f"{name}: 100 iterations at {time.time() - t0:.1f}s", flush=True)

    def pick(v, size):
        # half the sample from the support at k = 100 (sparse iterates), half uniform
        nz = np.flatnonzero(v)
        a = rng.choice(nz, size=min(size // 2, nz.size), replace=False) if nz.size else nz
        b = rng.choice(v.size, size=min(size - a.size, v.size), replace=False)
        return np.unique(np.concatenate([a, b]))

    iy, ix = pick(snaps[100][0], NSAMPLE), pick(snaps[100][1], NSAMPLE)
    sy = [snaps[k][0][iy] for k in SNAP_K]
    sx = [snaps[k][1][ix] for k in SNAP_K]
    out = dict(inst_sha=np.array(digest), lam=np.array([est.value, est.raw]),
               power_iterations=np.array(est.iterations), snap_k=np.array(SNAP_K),
               idx_y=iy, idx_x=ix, snap_y=np.array(sy), snap_x=np.array(sx),
               norms=np.array(norms), dots=np.array(dots), probe_seed=np.array(12345),
               b_factor=np.array(info.b_norm_factor),
               c_factor=np.array(info.c_norm_factor))
    if full_snapshot:
        out["y100"] = st.current.y.copy()
        out["x100"] = st.current.x.copy()
    np.savez_compressed(os.path.join(HERE, f"{name}_traj.npz"), **out)
    print(f"wrote {name}_traj.npz", flush=True)


def oracle_solve(name):
    from oracle import hprlp_oracle as O
    lib = O.load_clib()
    if lib is not None:
        lib.orc_set_threads(os.cpu_count() or 1)
    t0 = time.time()
    p = instance(name)
    digest = inst_sha(p)
    lp = O.OracleLP.from_problem(p)
    del p
    rep = O.solve(lp, O.OracleConfig(tolerance=1e-8))
    sol = rep.pop("solution")
    rep.pop("timings")
    rep["solution_norm"] = {f: float(np.linalg.norm(sol[f])) for f in ("x", "y", "z")}
    rep["inst_sha"] = digest
    rep["oracle_wall_s"] = time.time() - t0
    json.dump(rep, open(os.path.join(HERE, f"{name}_oracle_report.json"), "w"), indent=1)
    print(f"{name}: oracle {rep['status']} in {rep['iterations']} iterations, "
          f"{rep['oracle_wall_s']:.0f}s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["c2"]
    for w in what:
        if w == "c2":
            reference_trajectory("c2", full_snapshot=True)
        elif w == "c3":
            reference_trajectory("c3", full_snapshot=False)
        elif w == "c3-solve":
            oracle_solve("c3")
        else:
            raise SystemExit(f"unknown target {w}")
