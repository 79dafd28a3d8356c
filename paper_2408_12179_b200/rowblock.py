"""Row-block partitioned HPR-LP: A split by rows over P ranks.

Rank g owns a contiguous block of the stacked rows of A, balanced by nonzeros
(``partition_rows``).  Per iteration the A_g^T y_g partials are reduce-scattered
(each rank receives ceil(n/P) summed columns), the x-phase runs on that column
slice, w is all-gathered and the y-phase is local.  See ``csrc/hpr_rowblock.cuh``.

``RowBlockGroup`` exposes the ``DeviceLP`` methods the solve loop uses, so the
reference-shaped ``driver.solve`` runs unchanged on it:

* ``RowBlockGroup.local(problem, P)`` -- all P ranks in this process on one GPU
  (collectives are kernels).  The partitioned algorithm, parity-tested on one
  device.
* ``RowBlockGroup.distributed(block, ...)`` -- one rank per process over NCCL
  (``torch.distributed`` provides the ranks and broadcasts the NCCL id).

``solve_partitioned`` / ``solve_distributed`` are the entry points.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .device import DeviceLP
from .problem import stacked_arrays

NCCL_ID_BYTES = 128


def default_chunks(nranks: int, nccl: bool) -> int:
    """Column chunks of the inner loop: with NCCL over several GPUs the chunk
    q collectives overlap the partial SpMV of chunk q+1 (HPR_RB_CHUNKS
    overrides)."""
    import os
    env = os.environ.get("HPR_RB_CHUNKS")
    if env:
        return max(1, int(env))
    return 4 if (nccl and nranks > 1) else 1


def group_dims(n: int, nranks: int, chunks: int):
    """(npad, row-block workspace bytes) of the native group."""
    npad, ws = ctypes.c_int64(0), ctypes.c_size_t(0)
    N.call("hpr_group_dims", ctypes.c_int64(n), int(nranks), int(chunks), ctypes.byref(npad),
           ctypes.byref(ws))
    return int(npad.value), int(ws.value)


def partition_rows(row_offsets, parts: int) -> np.ndarray:
    """Boundaries r_0 = 0 < ... < r_P = m of P contiguous row blocks with
    nonzeros as even as whole rows allow (block g = rows [r_g, r_{g+1})).
    Every block gets at least one row when m >= P."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    m = ro.size - 1
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if m < parts:
        raise ValueError(f"cannot split {m} rows into {parts} blocks")
    nnz = int(ro[-1])
    targets = (np.arange(1, parts, dtype=np.float64) * nnz) / parts
    # weight rows by nnz + 1 so empty rows still spread when nnz is small
    w = ro + np.arange(m + 1, dtype=np.int64)
    tw = (np.arange(1, parts, dtype=np.float64) * w[-1]) / parts
    cuts = np.searchsorted(w, tw, side="left") if nnz == 0 else np.searchsorted(ro, targets)
    b = np.concatenate([[0], cuts, [m]]).astype(np.int64)
    for g in range(1, parts):               # strictly increasing, >= 1 row each
        b[g] = min(max(b[g], b[g - 1] + 1), m - (parts - g))
    return b


def block_arrays(ro, ci, v, rhs, m1, r0, r1):
    """CSR arrays, rhs and equality count of rows [r0, r1) of the stacked A."""
    z0, z1 = int(ro[r0]), int(ro[r1])
    bro = (np.asarray(ro[r0:r1 + 1], dtype=np.int64) - z0)
    m1_local = int(min(max(m1 - r0, 0), r1 - r0))
    return bro, ci[z0:z1], v[z0:z1], np.asarray(rhs[r0:r1], np.float64), m1_local


class RowBlockGroup:
    """P row blocks + one native group (DeviceLP-compatible surface)."""

    def __init__(self, blocks, row0, n, m_total, m1_total, nnz_total, nranks, rank0, chunks,
                 nccl_id=None):
        self.blocks = blocks                   # list[DeviceLP], local ranks
        self.row0 = list(row0)
        self.P = int(nranks)
        self.rank0 = int(rank0)
        self.n = int(n)
        self.m, self.m1, self.nnz = int(m_total), int(m1_total), int(nnz_total)
        self.stream = blocks[0].stream
        self.h2d_bytes = sum(b.h2d_bytes for b in blocks)
        self.analyzed = False
        self.nccl = nccl_id is not None
        torch = _torch()
        self.chunks = int(chunks)
        self.npad, sz = group_dims(self.n, self.P, self.chunks)
        with torch.cuda.stream(self.stream):
            self.rb_ws = [torch.empty(sz, dtype=torch.uint8, device=b.device) for b in blocks]
        self._sz = sz
        self._nccl_id = nccl_id
        self.g = None

    # -- construction ---------------------------------------------------------
    @classmethod
    def local(cls, problem, parts: int, device: int = 0, stream=None):
        """All ``parts`` ranks in this process, on one device and one stream."""
        torch = _torch()
        ro, ci, v, m, n, m1 = stacked_arrays(problem)
        rhs = np.concatenate([np.asarray(problem.b_eq, np.float64),
                              np.asarray(problem.b_ineq, np.float64)])
        bounds = partition_rows(ro, parts)
        chunks = default_chunks(parts, False)
        n_pad, _ = group_dims(n, parts, chunks)
        if stream is None:
            stream = torch.cuda.Stream(device=torch.device("cuda", device))
        blocks = []
        for g in range(parts):
            bro, bci, bv, bb, bm1 = block_arrays(ro, ci, v, rhs, m1, bounds[g], bounds[g + 1])
            blocks.append(DeviceLP.from_arrays(bro, bci, bv, int(bounds[g + 1] - bounds[g]), n,
                                               bm1, bb, problem.c, problem.lower, problem.upper,
                                               device=device, stream=stream, n_alloc=n_pad))
        return cls(blocks, bounds[:-1], n, m, m1, int(ro[-1]), parts, 0, chunks)

    @classmethod
    def distributed(cls, block, *, n, m_total, m1_total, nnz_total, row0, rank, world,
                    nccl_id, device):
        """This process's rank: ``block`` = (row_offsets, col_indices, values, m1_local,
        b, c, lower, upper) of its rows; ``nccl_id`` = 128 bytes from rank 0."""
        ro, ci, v, m1_local, b, c, lo, up = block
        chunks = default_chunks(world, True)
        n_pad, _ = group_dims(n, world, chunks)
        dev = DeviceLP.from_arrays(ro, ci, v, len(ro) - 1, n, m1_local, b, c, lo, up,
                                   device=device, n_alloc=n_pad)
        return cls([dev], [row0], n, m_total, m1_total, nnz_total, world, rank, chunks,
                   nccl_id=nccl_id)

    def _create(self):
        nl = len(self.blocks)
        ctxs = (ctypes.c_void_p * nl)(*[b.ctx.value for b in self.blocks])
        wss = (ctypes.c_void_p * nl)(*[t.data_ptr() for t in self.rb_ws])
        r0 = (ctypes.c_int64 * nl)(*self.row0)
        g = ctypes.c_void_p()
        if self._nccl_id is not None:
            idb = ctypes.create_string_buffer(bytes(self._nccl_id), NCCL_ID_BYTES)
            N.call("hpr_group_create", ctypes.byref(g), nl, ctxs, wss, r0,
                   ctypes.c_size_t(self._sz), self.P, self.rank0, self.chunks, idb,
                   ctypes.c_size_t(NCCL_ID_BYTES))
        else:
            N.call("hpr_group_create", ctypes.byref(g), nl, ctxs, wss, r0,
                   ctypes.c_size_t(self._sz), self.P, self.rank0, self.chunks, None,
                   ctypes.c_size_t(0))
        self.g = g

    # -- DeviceLP surface used by driver.solve --------------------------------
    def analyze(self):
        for b in self.blocks:
            if not b.analyzed:
                b.analyze()
        if self.g is None:
            self._create()
        self.analyzed = True

    def scale(self, ruiz_iters, pock_chambolle, bc_normalize):
        out = N.HprScaleOut()
        N.call("hpr_group_scale", self.g, int(ruiz_iters), int(bool(pock_chambolle)),
               int(bool(bc_normalize)), ctypes.byref(out))
        return out

    def power(self, tol, max_iters):
        out = N.HprPowerOut()
        N.call("hpr_group_power", self.g, float(tol), int(max_iters), ctypes.byref(out))
        return out

    def state_reset(self):
        N.call("hpr_group_state_reset", self.g)

    def run_inner(self, steps, t, k, sigma, lamsig, variant_code):
        N.call("hpr_group_run_inner", self.g, int(steps), int(t), int(k), float(sigma),
               float(lamsig), int(variant_code))

    def checkpoint(self, sigma, lamsig, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_group_checkpoint", self.g, float(sigma), float(lamsig), int(term_original),
               int(slot), ctypes.byref(out))
        return out

    def restart(self):
        N.call("hpr_group_restart", self.g)

    def kkt_origin(self, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_group_kkt_origin", self.g, int(term_original), int(slot), ctypes.byref(out))
        return out

    def kkt(self, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_group_kkt", self.g, int(term_original), int(slot), ctypes.byref(out))
        return out

    def finalize(self, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_group_finalize", self.g, int(term_original), int(slot), ctypes.byref(out))
        return out

    def launch_count(self) -> int:
        if self.g is None:
            return 0
        v = ctypes.c_int64(0)
        N.call("hpr_group_launch_count", self.g, ctypes.byref(v))
        return int(v.value)

    def layout_info(self) -> dict:
        infos = [b.layout_info() for b in self.blocks]
        out = {k: sum(i[k] for i in infos) for k in infos[0]}
        for k in ("split_a", "stg_a", "stg_at", "rao_a", "rao_at"):   # block counts / flags, not sums
            out[k] = max(i[k] for i in infos)
        out["partitions"] = self.P
        return out

    def last_times(self):
        a, b = ctypes.c_double(0), ctypes.c_double(0)
        N.call("hpr_group_last_times", self.g, ctypes.byref(a), ctypes.byref(b))
        return float(a.value) / 1e3, float(b.value) / 1e3

    def synchronize(self):
        self.stream.synchronize()

    def comm_info(self) -> dict:
        """Transport and, for NCCL, the communicator's own rank count / rank /
        version (hpr_group_comm_info) plus the pinned algorithm / protocol."""
        import os
        if self.g is None:
            return {"transport": "nccl" if self.nccl else "local", "nranks": self.P}
        v = [ctypes.c_int(0) for _ in range(4)]
        N.call("hpr_group_comm_info", self.g, *[ctypes.byref(x) for x in v])
        tr, nr, rk, ver = (x.value for x in v)
        return {"transport": "nccl" if tr else "local", "nranks": nr, "rank": rk,
                "nccl_version": ver, "NCCL_ALGO": os.environ.get("NCCL_ALGO"),
                "NCCL_PROTO": os.environ.get("NCCL_PROTO")}

    def any_rank(self, flag: bool) -> bool:
        """OR of ``flag`` over all ranks of the group (a MAX all-reduce over
        torch.distributed in NCCL mode; the local transport is one process)."""
        if not (self.nccl and self.P > 1):
            return bool(flag)
        import torch.distributed as dist
        torch = _torch()
        dev = self.blocks[0].device if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return bool(int(t.item()))

    def _col_layout(self):
        """(K chunks, cw columns per rank and chunk, padded n) of hpr_group_col_layout."""
        k, cw, npad = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        N.call("hpr_group_col_layout", self.g, ctypes.byref(k), ctypes.byref(cw),
               ctypes.byref(npad))
        return int(k.value), int(cw.value), int(npad.value)

    def owned_columns(self, local: int = 0) -> np.ndarray:
        """Column indices owned by local rank ``local`` (hpr_group_col_layout)."""
        k, cw, _ = self._col_layout()
        g = self.rank0 + local
        cols = (np.arange(k)[:, None] * (self.P * cw) + g * cw + np.arange(cw)[None, :]).ravel()
        return cols[cols < self.n]

    def _gather_dev(self):
        """(torch.distributed module, tensor device) for the host-side gathers:
        the GPU over NCCL when the default group is NCCL, else host tensors
        (gloo)."""
        import torch.distributed as dist
        if dist.get_backend() == "nccl":
            return dist, self.blocks[0].device
        return dist, "cpu"

    def to_host(self, name, slot=None):
        """Row vectors: the ranks' blocks concatenated.  Column vectors:
        assembled from each rank's own slice (the only part a rank keeps
        current).  In NCCL mode the pieces move with tensor all-gathers over
        the job's torch.distributed group (device buffers over NVLink with the
        NCCL backend), not through pickled host objects."""
        torch = _torch()
        row_names = ("y", "anc_y", "yb", "dy", "b_s", "row_scale", "cand_y", "b")
        if name in row_names:
            if not (self.nccl and self.P > 1):
                return np.concatenate([b.to_host(name, slot) for b in self.blocks])
            dist, dev = self._gather_dev()
            blk = self.blocks[0]
            t = blk.t[name] if slot is None else blk.t[name][slot]
            blk.synchronize()
            mine = t[:blk.m].to(dev)
            lens = torch.zeros(self.P, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(lens, torch.tensor([blk.m], dtype=torch.int64,
                                                           device=dev))
            lens = lens.tolist()
            mx = max(lens)
            buf = torch.zeros(mx, dtype=torch.float64, device=dev)
            buf[:blk.m] = mine
            out = torch.empty(self.P * mx, dtype=torch.float64, device=dev)
            dist.all_gather_into_tensor(out, buf)
            out = out.view(self.P, mx).cpu().numpy()
            return np.concatenate([out[g, :lens[g]] for g in range(self.P)])
        # owned columns of rank g = slab g of every chunk: a (K, P, cw) view of
        # the padded vector, so the pieces move by strided copies, not fancy indexing
        k, cw, npad = self._col_layout()
        if self.P == 1:
            return self.blocks[0].to_host(name, slot)
        if self.nccl:
            dist, dev = self._gather_dev()
            blk = self.blocks[0]
            t = blk.t[name] if slot is None else blk.t[name][slot]
            blk.synchronize()
            pad = torch.zeros(k * self.P * cw, dtype=torch.float64, device=t.device)
            ln = min(t.numel(), pad.numel())
            pad[:ln] = t[:ln]
            mine = pad.view(k, self.P, cw)[:, self.rank0, :].contiguous().to(dev)
            got = torch.empty((self.P, k, cw), dtype=torch.float64, device=dev)
            dist.all_gather_into_tensor(got, mine)
            return got.permute(1, 0, 2).reshape(-1)[:self.n].cpu().numpy()
        out = np.empty(k * self.P * cw)
        slabs = out.reshape(k, self.P, cw)
        for l, b in enumerate(self.blocks):
            pad = np.zeros(k * self.P * cw)
            v = b.to_host(name, slot)
            pad[:v.size] = v
            g = self.rank0 + l
            slabs[:, g, :] = pad.reshape(k, self.P, cw)[:, g, :]
        return out[:self.n]

    def close(self):
        if self.g is not None and self.g.value:
            N.load_library().hpr_group_destroy(self.g)
            self.g = None
        for b in self.blocks:
            b.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _torch():
    import torch
    return torch


def solve_partitioned(problem, cfg=None, *, parts: int = 2, device: int = 0):
    """``solve`` with A split into ``parts`` row blocks, all on one GPU (local
    transport): the partitioned algorithm of the multi-GPU path."""
    from .driver import solve
    grp = RowBlockGroup.local(problem, parts, device=device)
    try:
        return solve(problem, cfg, dev=grp)
    finally:
        grp.close()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    N.call("hpr_nccl_unique_id", buf, ctypes.c_size_t(NCCL_ID_BYTES))
    return buf.raw


def broadcast_nccl_id(rank: int) -> bytes:
    """Rank 0 creates the NCCL id; torch.distributed broadcasts it."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class _BlockShell:
    """What ``solve`` reads from the problem when the device object is a
    row-block group: the objective constant and sense (problem.py:22-36)."""

    def __init__(self, objective_constant=0.0, objective_negated=False):
        self.objective_constant = float(objective_constant)
        self.objective_negated = bool(objective_negated)


def solve_row_block(block, cfg=None, *, n, m_total, m1_total, nnz_total, row0,
                    objective_constant: float = 0.0, objective_negated: bool = False,
                    device: int | None = None):
    """One rank per process (torch.distributed initialised by the caller), each
    rank passing ONLY its own row block -- ``block`` = (row_offsets,
    col_indices, values, m1_local, b, c, lower, upper) of rows [row0, row0 +
    m_g) of the stacked A = [A_eq; A_ineq] -- for problems no single host
    holds.  The report is the whole problem's on every rank (the row-block
    path of ``solve``)."""
    import os
    import torch.distributed as dist
    from .driver import solve
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(), dist.get_world_size()
        nid = broadcast_nccl_id(rank)
    else:                                        # a one-rank job (NCCL world of 1)
        rank, world, nid = 0, 1, nccl_unique_id()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    grp = RowBlockGroup.distributed(block, n=n, m_total=m_total, m1_total=m1_total,
                                    nnz_total=nnz_total, row0=row0, rank=rank, world=world,
                                    nccl_id=nid, device=device)
    try:
        return solve(_BlockShell(objective_constant, objective_negated), cfg, dev=grp)
    finally:
        grp.close()


def solve_distributed(problem, cfg=None, *, device: int | None = None):
    """One rank per process (torch.distributed initialised by the caller): every
    rank passes the same ``problem``; rank g uploads only its row block."""
    import torch.distributed as dist
    from .driver import solve
    rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", "0"))
    ro, ci, v, m, n, m1 = stacked_arrays(problem)
    rhs = np.concatenate([np.asarray(problem.b_eq, np.float64),
                          np.asarray(problem.b_ineq, np.float64)])
    bounds = partition_rows(ro, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    bro, bci, bv, bb, bm1 = block_arrays(ro, ci, v, rhs, m1, r0, r1)
    nid = broadcast_nccl_id(rank)
    grp = RowBlockGroup.distributed((bro, bci, bv, bm1, bb, problem.c, problem.lower,
                                     problem.upper), n=n, m_total=m, m1_total=m1,
                                    nnz_total=int(ro[-1]), row0=r0, rank=rank, world=world,
                                    nccl_id=nid, device=device)
    try:
        return solve(problem, cfg, dev=grp)
    finally:
        grp.close()
