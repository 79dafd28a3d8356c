"""Row-block partitioned HPR iteration on the CPU (TEST INFRASTRUCTURE ONLY).

Restates, with numpy and caller-supplied collectives, the algorithm of the
multi-GPU path (``paper_2408_12179_b200/csrc/hpr_rowblock.cuh``): rank g owns
rows [r_g, r_{g+1}) of the stacked A, computes the partial A_g^T y_g over all n
columns, the partials are summed across ranks (reduce-scatter; here an
all-reduce followed by taking the rank's column slice), the x-phase of
core.py:168-169 runs on the slice, w = 2 xb - x is all-gathered and the y-phase
(core.py:170-172) is local.  ``tests/test_rowblock_host.py`` runs it under a
world-size-2 ``gloo`` group and checks it against the unpartitioned
``hprlp_oracle.iterate_once`` (reference core.py:163-174).
"""

from __future__ import annotations

import numpy as np

from .hprlp_oracle import Csr, OracleLP


def slice_of(rank: int, world: int, n: int):
    cnt = -(-n // world)
    return min(rank * cnt, n), min((rank + 1) * cnt, n)


def run_rank(rank, world, lp: OracleLP, bounds, lam, sigma, iters, allreduce_sum, allgather):
    """``iters`` HPR iterations (t = k = 0.., anchors 0) of rank ``rank``'s block.

    allreduce_sum(vec) -> elementwise sum over ranks; allgather(piece) -> list of
    every rank's piece.  Returns (y_block, x_full)."""
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    a = lp.a
    z0, z1 = int(a.rp[r0]), int(a.rp[r1])
    blk = Csr(a.rp[r0:r1 + 1] - z0, a.ci[z0:z1], a.vals[z0:z1], lp.n, use_c=False)
    blk_t = blk.transpose()
    m1_loc = min(max(lp.m1 - r0, 0), r1 - r0)
    b = lp.b[r0:r1]
    j0, j1 = slice_of(rank, world, lp.n)
    c, lo, up = lp.c[j0:j1], lp.lower[j0:j1], lp.upper[j0:j1]
    y = np.zeros(r1 - r0)
    ay = np.zeros(r1 - r0)
    x = np.zeros(j1 - j0)
    ax = np.zeros(j1 - j0)
    lamsig = lam * sigma
    for t in range(iters):
        aty = allreduce_sum(blk_t.matvec(y))[j0:j1]          # reduce-scatter
        v = x + sigma * (aty - c)
        xb = np.clip(v, lo, up)
        w_sl = 2.0 * xb - x
        w = np.concatenate(allgather(w_sl))                   # all-gather
        yb = y + (b - blk.matvec(w)) / lamsig
        if m1_loc < yb.size:
            np.maximum(yb[m1_loc:], 0.0, out=yb[m1_loc:])
        t2 = t + 2.0
        wn, wa = (t + 1.0) / t2, 1.0 / t2
        y = wa * ay + wn * (2.0 * yb - y)
        x = wa * ax + wn * w_sl
    return y, np.concatenate(allgather(x))
