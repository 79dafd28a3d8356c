"""Host-side logic of the row-block partitioned path, on CPU.

* ``partition_rows`` / ``block_arrays``: the nnz-balanced split and the per-rank
  arrays the multi-GPU path uploads.
* the partitioned iteration (``oracle/partitioned.py``) under a world-size-2
  ``gloo`` process group agrees with the unpartitioned oracle iteration
  (reference core.py:163-174) to 1e-12 normwise -- the math of the RS/AG split
  the CUDA group implements.
"""

import os
import socket

import numpy as np
import pytest

from paper_2408_12179_b200.generators import generate_known_solution_lp
from paper_2408_12179_b200.problem import stacked_arrays
from paper_2408_12179_b200.rowblock import block_arrays, partition_rows


def _instance():
    prob, _ = generate_known_solution_lp(1003, 30, 34, 150, 0.08)
    return prob


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 7])
def test_partition_rows_properties(parts):
    prob = _instance()
    ro, ci, v, m, n, m1 = stacked_arrays(prob)
    b = partition_rows(ro, parts)
    assert b[0] == 0 and b[-1] == m and len(b) == parts + 1
    assert np.all(np.diff(b) >= 1)
    nnz_blocks = np.diff(ro[b])
    # balanced by nonzeros to within one row of the largest row
    assert nnz_blocks.max() - nnz_blocks.min() <= 2 * int(np.diff(ro).max())


def test_partition_rows_edge_cases():
    ro = np.array([0, 0, 0, 0])                 # empty rows only
    b = partition_rows(ro, 3)
    assert list(b) == [0, 1, 2, 3]
    with pytest.raises(ValueError):
        partition_rows(np.array([0, 1]), 2)
    ro = np.array([0, 100, 101, 102, 103])      # one heavy row
    b = partition_rows(ro, 2)
    assert b[0] == 0 and b[-1] == 4 and 1 <= b[1] <= 3


def test_block_arrays_reassemble():
    prob = _instance()
    ro, ci, v, m, n, m1 = stacked_arrays(prob)
    rhs = np.concatenate([prob.b_eq, prob.b_ineq])
    b = partition_rows(ro, 3)
    got_ci, got_v, got_b, m1s = [], [], [], []
    for g in range(3):
        bro, bci, bv, bb, bm1 = block_arrays(ro, ci, v, rhs, m1, b[g], b[g + 1])
        assert bro[0] == 0 and bro[-1] == bci.size
        got_ci.append(bci)
        got_v.append(bv)
        got_b.append(bb)
        m1s.append(bm1)
    assert np.array_equal(np.concatenate(got_ci), ci)
    assert np.array_equal(np.concatenate(got_v), v)
    assert np.array_equal(np.concatenate(got_b), rhs)
    assert sum(m1s) == m1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, iters, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import hprlp_oracle as O
        from oracle.partitioned import run_rank
        prob = _instance()
        lp = O.OracleLP.from_problem(prob, use_c=False)
        scaled, _ = O.scale_lp(lp)
        lam = O.power_lambda(scaled).value
        bounds = partition_rows(scaled.a.rp, world)

        def allreduce_sum(vec):
            t = torch.from_numpy(np.ascontiguousarray(vec))
            dist.all_reduce(t)
            return t.numpy()

        def allgather(piece):
            got = [None] * world
            dist.all_gather_object(got, np.asarray(piece))
            return got

        y_blk, x = run_rank(rank, world, scaled, bounds, lam, 1.0, iters, allreduce_sum,
                            allgather)
        ys = [None] * world
        dist.all_gather_object(ys, y_blk)
        if rank == 0:
            out_q.put((np.concatenate(ys), x))
    finally:
        dist.destroy_process_group()


def test_partitioned_iteration_gloo_world2():
    import torch.multiprocessing as mp
    from oracle import hprlp_oracle as O
    iters = 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    y, x = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prob = _instance()
    lp = O.OracleLP.from_problem(prob, use_c=False)
    scaled, _ = O.scale_lp(lp)
    lam = O.power_lambda(scaled).value
    st = O.State(np.zeros(scaled.m), np.zeros(scaled.n), np.zeros(scaled.m),
                 np.zeros(scaled.n), 1.0, lam)
    for _ in range(iters):
        O.iterate_once(st, scaled)
    ref = np.concatenate([st.y, st.x])
    got = np.concatenate([y, x])
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_batch_shard_bounds_cover():
    from paper_2408_12179_b200.batch import shard_bounds
    for count in (1, 7, 4096):
        for world in (1, 2, 3, 8):
            if count < world:
                continue
            spans = [shard_bounds(count, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_batch_packing_offsets():
    from paper_2408_12179_b200.batch import PackedBatch
    probs = [generate_known_solution_lp(10_000 + i, 5, 6, 20, 0.3)[0] for i in range(3)]
    pk = PackedBatch(probs)
    a = pk.arrays
    assert pk.count == 3 and a["row_off"][-1] == 33 and a["col_off"][-1] == 60
    for i, p in enumerate(probs):
        ro, ci, v, m, n, m1 = stacked_arrays(p)
        r0 = pk.row_off[i]
        assert np.array_equal(a["rp"][r0 + i:r0 + i + m + 1], ro)
        z0, z1 = pk.nz_off[i], pk.nz_off[i + 1]
        assert np.array_equal(a["ci"][z0:z1], ci) and np.array_equal(a["val"][z0:z1], v)
        assert a["m1"][i] == m1
