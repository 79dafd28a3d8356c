"""Batch of small LPs, one whole restarted HPR solve per CTA (config C5).

``solve_batch(problems, cfg)`` is ``[solve(p, cfg) for p in problems]``
(reference ``driver.py:281-405`` per LP) executed as one kernel launch of
``libhprlp_b200.so`` (``csrc/hpr_batch.cuh``) -- for large batches a pipeline
of launches over chunks, overlapping host packing, upload, solve and report
assembly (``_run_pipelined``) -- where each CTA stages its LP in
shared memory and runs scaling, the power method, the inner loop, the
checkpoints, restarts and sigma updates without returning to the host.
``solve_batch_sharded`` splits the batch across the ranks of a
``torch.distributed`` job (independent units, no data-path collective).
"""

from __future__ import annotations

import ctypes
import os
import math
import threading
import warnings

import numpy as np

from . import _native as N
from .driver import (KktResidual, RestartEvent, SolveReport, SolverConfig, SolveStatus, Timings,
                     Variant)
from .problem import PrimalDualPoint

_STATUS = {0: SolveStatus.OPTIMAL, 1: SolveStatus.ITERATION_LIMIT, 2: SolveStatus.TIME_LIMIT,
           3: SolveStatus.NUMERICAL_ERROR}
_TRIGGER = {0: "sufficient", 1: "stalled", 2: "long_loop"}
_VARIANT = {Variant.DR: 0, Variant.HDR_FIXED_SIGMA: 1, Variant.HDR: 2, Variant.HPR: 3}
MAX_LOG = 64       # restart records kept per LP in the first pass (solve_batch re-runs overflows)


def _torch():
    import torch
    return torch


class PackedBatch:
    """Host-side concatenation of a list of reference-shaped LPs (sizes first,
    then every LP's arrays copied into preallocated batch arrays)."""

    # upload order of the batch arrays (BatchRun lays them out in this order,
    # each padded to 256 bytes)
    ORDER = (("row_off", np.int64), ("col_off", np.int64), ("nz_off", np.int64),
             ("m1", np.int32), ("rp", np.int32), ("ci", np.int32), ("val", np.float64),
             ("b", np.float64), ("c", np.float64), ("lower", np.float64), ("upper", np.float64),
             ("obj_const", np.float64), ("obj_neg", np.int32))

    def __init__(self, problems, staging=None):
        """``staging``: ``f(nbytes) -> uint8 numpy array`` (at least nbytes) to
        pack into at the upload layout -- a pinned buffer: packing then writes
        the bytes BatchRun copies to the device, with no second host copy and
        no page faults on fresh arrays."""
        if not problems:
            raise ValueError("empty batch")
        cnt = len(problems)
        ms = np.empty(cnt, np.int64)
        ns = np.empty(cnt, np.int64)
        nzs = np.empty(cnt, np.int64)
        m1s = np.empty(cnt, np.int32)
        oc = np.empty(cnt, np.float64)
        neg = np.empty(cnt, np.int32)
        for i, p in enumerate(problems):
            top, bot = p.a_eq, p.a_ineq
            m1s[i] = int(top.nrows)
            ms[i] = int(top.nrows) + int(bot.nrows)
            ns[i] = int(top.ncols)
            nzs[i] = (int(top.row_offsets[-1]) - int(top.row_offsets[0]) +
                      int(bot.row_offsets[-1]) - int(bot.row_offsets[0]))
            if nzs[i] == 0:
                raise ValueError("matrix must be non-zero")
            oc[i] = float(getattr(p, "objective_constant", 0.0))
            neg[i] = int(bool(getattr(p, "objective_negated", False)))
        self.count = cnt
        self.m, self.n, self.nnz = ms, ns, nzs
        self.row_off = np.concatenate([[0], np.cumsum(ms)]).astype(np.int64)
        self.col_off = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
        self.nz_off = np.concatenate([[0], np.cumsum(nzs)]).astype(np.int64)
        R, C, Z = int(self.row_off[-1]), int(self.col_off[-1]), int(self.nz_off[-1])
        lens = {"row_off": cnt + 1, "col_off": cnt + 1, "nz_off": cnt + 1, "m1": cnt,
                "rp": R + cnt, "ci": Z, "val": Z, "b": R, "c": C, "lower": C, "upper": C,
                "obj_const": cnt, "obj_neg": cnt}
        out = {}
        if staging is not None:
            nbs = [lens[k] * np.dtype(dt).itemsize for k, dt in self.ORDER]
            buf = staging(sum((nb + 255) // 256 * 256 for nb in nbs))
            o = 0
            for (k, dt), nb in zip(self.ORDER, nbs):
                out[k] = buf[o:o + nb].view(dt)
                o += (nb + 255) // 256 * 256
        host = _host_module()
        if os.environ.get("HPR_PACK_LOOP") == "1":
            rp, ci, val, b, c, lo, up = self._pack_loop(problems, ns, nzs)
        elif host is not None and os.environ.get("HPR_PACK_NATIVE", "1") == "1":
            for k, dt in self.ORDER:                 # the native packer writes these in place
                if k in ("rp", "ci", "val", "b", "c", "lower", "upper") and k not in out:
                    out[k] = np.empty(lens[k], dt)
            host.pack_batch(problems, out, self.row_off, self.col_off, self.nz_off,
                            min(8, os.cpu_count() or 1))
            rp, ci, val, b, c, lo, up = (out[k] for k in ("rp", "ci", "val", "b", "c", "lower",
                                                          "upper"))
        else:
            rp, ci, val, b, c, lo, up = self._pack_concat(problems, out)
        self.arrays = {
            "row_off": self.row_off, "col_off": self.col_off, "nz_off": self.nz_off,
            "m1": m1s, "rp": rp, "ci": ci, "val": val, "b": b, "c": c, "lower": lo, "upper": up,
            "obj_const": oc, "obj_neg": neg}
        for k, a in out.items():                 # the small arrays into the staging too
            if self.arrays[k] is not a:
                np.copyto(a, self.arrays[k], casting="unsafe")
                self.arrays[k] = a

    def _pack_concat(self, problems, out):
        """Each batch array is one np.concatenate over the LPs' pieces (the
        copies and the int64 -> int32 casts run in C), into ``out[name]`` when
        given."""
        def cat(name, parts, dt):
            if name in out:
                return np.concatenate(parts, out=out[name], casting="unsafe")
            return np.concatenate(parts, dtype=dt, casting="unsafe")

        tops = [p.a_eq for p in problems]
        bots = [p.a_ineq for p in problems]
        pieces, shift, lens = [], [], []
        for t, b in zip(tops, bots):
            tr, br = np.asarray(t.row_offsets), np.asarray(b.row_offsets)
            nt = int(tr[-1] - tr[0])
            pieces.append(tr)
            pieces.append(br[1:])
            shift.append(-int(tr[0]))
            shift.append(nt - int(br[0]))
            lens.append(len(tr))
            lens.append(len(br) - 1)
        rp = cat("rp", pieces, np.int32)
        rp += np.repeat(np.asarray(shift, np.int32), lens)
        ci = cat("ci", [x for t, b in zip(tops, bots) for x in (t.col_indices, b.col_indices)],
                 np.int32)
        val = cat("val", [x for t, b in zip(tops, bots) for x in (t.values, b.values)],
                  np.float64)
        b = cat("b", [x for p in problems for x in (p.b_eq, p.b_ineq)], np.float64)
        c = cat("c", [p.c for p in problems], np.float64)
        lo = cat("lower", [p.lower for p in problems], np.float64)
        up = cat("upper", [p.upper for p in problems], np.float64)
        return rp, ci, val, b, c, lo, up

    def _pack_loop(self, problems, ns, nzs):
        """Per-LP slice assignments into preallocated arrays (HPR_PACK_LOOP=1)."""
        cnt = self.count
        R, C, Z = int(self.row_off[-1]), int(self.col_off[-1]), int(self.nz_off[-1])
        rp = np.empty(R + cnt, np.int64)
        ci = np.empty(Z, np.int64)
        val = np.empty(Z, np.float64)
        b = np.empty(R, np.float64)
        c = np.empty(C, np.float64)
        lo = np.empty(C, np.float64)
        up = np.empty(C, np.float64)
        for i, p in enumerate(problems):
            r0, c0, z0 = int(self.row_off[i]), int(self.col_off[i]), int(self.nz_off[i])
            top, bot = p.a_eq, p.a_ineq
            mt, mb, n = int(top.nrows), int(bot.nrows), int(ns[i])
            tro, bro = np.asarray(top.row_offsets), np.asarray(bot.row_offsets)
            nt = int(tro[-1] - tro[0])
            q = r0 + i                               # LP i's m + 1 row pointers
            rp[q:q + mt + 1] = tro - tro[0]
            rp[q + mt:q + mt + mb + 1] = bro - bro[0] + nt
            ci[z0:z0 + nt] = top.col_indices
            ci[z0 + nt:z0 + int(nzs[i])] = bot.col_indices
            val[z0:z0 + nt] = top.values
            val[z0 + nt:z0 + int(nzs[i])] = bot.values
            b[r0:r0 + mt] = p.b_eq
            b[r0 + mt:r0 + mt + mb] = p.b_ineq
            c[c0:c0 + n] = p.c
            lo[c0:c0 + n] = p.lower
            up[c0:c0 + n] = p.upper
        return rp.astype(np.int32), ci.astype(np.int32), val, b, c, lo, up

    def h2d_bytes(self):
        return sum(a.nbytes for a in self.arrays.values())


_HOST = False


def _host_module():
    """The native host helpers (csrc/hpr_host.cpp, built in-tree by build.py),
    or None -- batch packing then runs in numpy."""
    global _HOST
    if _HOST is False:
        try:
            from . import _hpr_host
            _HOST = _hpr_host
        except ImportError:
            _HOST = None
    return _HOST


def _config(cfg: SolverConfig, max_log: int) -> N.HprBatchConfig:
    c = N.HprBatchConfig()
    c.tolerance = cfg.tolerance
    c.time_limit_seconds = cfg.time_limit_seconds
    c.alpha1, c.alpha2, c.alpha3 = cfg.alpha1, cfg.alpha2, cfg.alpha3
    c.sigma0 = cfg.sigma0
    c.power_tol = cfg.power_tol
    c.max_iterations = int(cfg.max_iterations)
    c.check_interval = int(cfg.check_interval)
    c.variant = _VARIANT[cfg.variant]
    c.ruiz_iters = int(cfg.ruiz_iters)
    c.pock_chambolle = int(bool(cfg.pock_chambolle))
    c.bc_normalize = int(bool(cfg.bc_normalize))
    c.power_max_iters = int(cfg.power_max_iters)
    c.term_original = int(cfg.termination_space == "original")
    c.max_log = int(max_log)
    return c


_STREAMS = {}


def _batch_stream(torch, device):
    st = _STREAMS.get(device)
    if st is None:
        st = _STREAMS[device] = torch.cuda.Stream(device=torch.device("cuda", device))
    return st


class BatchRun:
    """Device residency of one packed batch + its native solve (re-runnable)."""

    def __init__(self, packed: PackedBatch, device: int = 0, stream=None, pinned: bool = True,
                 max_log: int | None = None, staging=None):
        """``staging``: the pinned uint8 tensor ``packed`` was packed into (the
        pipelined ``solve_batch``): the upload is issued from it asynchronously
        and ``self.h2d_done`` (an event) marks when the buffer may be reused;
        otherwise the process-wide staging buffer is used and the upload is
        waited for."""
        torch = _torch()
        self.max_log = int(MAX_LOG if max_log is None else max_log)
        if not torch.cuda.is_available():
            raise N.NativeUnavailableError("CUDA device required: the batch path has no CPU fallback")
        N.load_library()
        self.packed = packed
        self.device = torch.device("cuda", device)
        self.dev_index = device
        # one stream per device for every BatchRun: the caching allocator keeps
        # freed blocks per stream, so a new stream per run would cudaMalloc anew
        self.stream = stream if stream is not None else _batch_stream(torch, device)
        # one pinned staging buffer -> one H2D copy; the inputs are views of it
        from .device import _Staging
        tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
               np.dtype(np.float64): torch.float64}
        offs, total = {}, 0
        for k, a in packed.arrays.items():
            offs[k] = total
            total += (a.nbytes + 255) // 256 * 256
        self.t = {}
        self.h2d_done = None

        def upload(stage):
            host = stage.numpy()
            base = host.ctypes.data
            for k, a in packed.arrays.items():
                if a.ctypes.data == base + offs[k]:
                    continue                      # packed in place (solve_batch)
                host[offs[k]:offs[k] + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
            with torch.cuda.stream(self.stream):
                self._inputs = torch.empty(total, dtype=torch.uint8, device=self.device)
                self._inputs.copy_(stage[:total], non_blocking=True)

        if staging is not None:
            upload(staging)
            self.h2d_done = torch.cuda.Event()
            self.h2d_done.record(self.stream)
        else:
            with _Staging.lock:
                upload(_Staging.get(total))
                self.stream.synchronize()
        for k, a in packed.arrays.items():
            self.t[k] = self._inputs[offs[k]:offs[k] + a.nbytes].view(tdt[a.dtype])
        self.h2d_bytes = total
        pb = N.HprBatchProblem()
        pb.count = packed.count
        pb.total_rows = int(packed.row_off[-1])
        pb.total_cols = int(packed.col_off[-1])
        pb.total_nnz = int(packed.nz_off[-1])
        pb.max_m = int(packed.m.max())
        pb.max_n = int(packed.n.max())
        pb.max_nnz = int(packed.nnz.max())
        for k in ("row_off", "col_off", "nz_off", "m1", "rp", "ci", "val", "b", "c", "lower",
                  "upper", "obj_const", "obj_neg"):
            setattr(pb, k, self.t[k].data_ptr())
        self.pb = pb
        wsb = ctypes.c_size_t(0)
        N.call("hpr_batch_workspace_bytes", ctypes.byref(pb), ctypes.byref(wsb))
        f64 = dict(dtype=torch.float64, device=self.device)
        with torch.cuda.stream(self.stream):
            self.ws = torch.empty(int(wsb.value), dtype=torch.uint8, device=self.device)
            self.x = torch.empty(max(pb.total_cols, 1), **f64)
            self.z = torch.empty(max(pb.total_cols, 1), **f64)
            self.y = torch.empty(max(pb.total_rows, 1), **f64)
            self.res = torch.empty(packed.count * ctypes.sizeof(N.HprBatchResult),
                                   dtype=torch.uint8, device=self.device)
            self.log = torch.empty(packed.count * self.max_log * ctypes.sizeof(N.HprRestartRec),
                                   dtype=torch.uint8, device=self.device)
        self.launches = 0

    def launch(self, cfg: SolverConfig):
        c = _config(cfg, self.max_log)
        N.call("hpr_batch_solve", ctypes.byref(self.pb), ctypes.byref(c),
               ctypes.c_void_p(self.ws.data_ptr()), ctypes.c_size_t(self.ws.numel()),
               ctypes.c_void_p(self.res.data_ptr()), ctypes.c_void_p(self.log.data_ptr()),
               ctypes.c_void_p(self.x.data_ptr()), ctypes.c_void_p(self.y.data_ptr()),
               ctypes.c_void_p(self.z.data_ptr()), self.dev_index,
               ctypes.c_void_p(self.stream.cuda_stream))
        # transpose keys + iota + cub sort (3) + col count + gather + rpt + solve
        self.launches += 9

    def reports(self, cfg: SolverConfig) -> list[SolveReport]:
        self.stream.synchronize()
        # thousands of small report objects: no cyclic-GC passes while they are built
        import gc
        was = gc.isenabled()
        gc.disable()
        try:
            return _build_reports(self.packed, self.res.cpu().numpy(), self.log.cpu().numpy(),
                                  self.x.cpu().numpy(), self.y.cpu().numpy(), self.z.cpu().numpy(),
                                  self.max_log)
        finally:
            if was:
                gc.enable()


class RestartLogOverflow(RuntimeWarning):
    """A batch LP restarted more often than its restart-log capacity: its
    report's ``restart_log`` is truncated (``solve_batch`` re-runs such LPs
    with a log large enough, so its reports are always complete)."""


def _build_reports(pk: PackedBatch, raw, lraw, x, y, z, max_log: int = MAX_LOG) -> list[SolveReport]:
    """SolveReports of a batch from the device result records (column-wise
    numpy views of the C structs; the solution arrays are views of fresh host
    copies of the batch vectors)."""
    rs = np.frombuffer(np.ascontiguousarray(raw).tobytes(), dtype=np.dtype(N.HprBatchResult),
                       count=pk.count)
    recs = np.frombuffer(np.ascontiguousarray(lraw).tobytes(), dtype=np.dtype(N.HprRestartRec),
                         count=pk.count * max_log).reshape(pk.count, max_log)
    col = {f: rs[f].tolist() for f in rs.dtype.names if f != "kkt"}
    kkts = rs["kkt"].tolist()
    if any(p and not c for p, c in zip(col["power_iterations"], col["power_converged"])):
        for p, c in zip(col["power_iterations"], col["power_converged"]):
            if p and not c:
                warnings.warn(f"power method did not converge within {p} iterations",
                              RuntimeWarning)
    for neg in col["merit_negative"]:
        if neg:
            warnings.warn("negative quadratic form in the merit: lambda may underestimate "
                          "lambda_1(AA*)", RuntimeWarning)
    ro, co = pk.row_off.tolist(), pk.col_off.tolist()
    over = sum(1 for v in col["n_log"] if v > max_log)
    if over:
        warnings.warn(f"{over} LP(s) restarted more than {max_log} times: restart_log truncated",
                      RestartLogOverflow)
    nlog = [min(v, max_log) for v in col["n_log"]]
    lmax = max(nlog) if nlog else 0
    rec_cols = {f: recs[f][:, :lmax].tolist() for f in recs.dtype.names}
    out = []
    for i in range(pk.count):
        k = kkts[i]
        kkt = KktResidual(k[0], k[1], k[2], k[3], k[4], k[5], k[6], k[7], k[8],
                          col["dual_clamped"][i])
        log = [RestartEvent(rec_cols["outer_index"][i][q], _TRIGGER[rec_cols["trigger"][i][q]],
                            rec_cols["tau"][i][q], rec_cols["sigma_next"][i][q],
                            rec_cols["merit"][i][q]) for q in range(nlog[i])]
        sol = PrimalDualPoint(y=y[ro[i]:ro[i + 1]], z=z[co[i]:co[i + 1]], x=x[co[i]:co[i + 1]])
        out.append(SolveReport(
            status=_STATUS[col["status"][i]], primal_objective=col["primal_objective"][i],
            dual_objective=col["dual_objective"][i], kkt=kkt, iterations=col["iterations"][i],
            restarts=col["restarts"][i], restart_log=log,
            timings=Timings(iteration_seconds=col["device_seconds"][i]), solution=sol,
            sigma_final=col["sigma_final"][i], lambda_estimate=col["lambda_estimate"][i],
            device_stats={"lambda_raw": col["lambda_raw"][i],
                          "power_iterations": col["power_iterations"][i],
                          "b_factor": col["b_factor"][i], "c_factor": col["c_factor"][i],
                          "batch_index": i}))
    return out


PIPE_CHUNK = 1024      # LPs per pipelined launch (C5, native packing: 4096 / 2048 / 1024 / 512 / 256 -> 161-196 / 124-131 / 122-128 / 122-181 / 129-132 ms per call)
PIPE_MIN = 2048        # batches smaller than this run as one launch


class _PipeStaging:
    """Two process-wide pinned staging buffers per device (chunk j packs into
    slot j % 2 while chunk j - 1's upload is in flight from the other);
    ``lock`` serialises pipelined calls (they share the slots)."""

    bufs: dict = {}
    lock = threading.Lock()

    @classmethod
    def get(cls, device, slot, nbytes):
        torch = _torch()
        key = (device, slot)
        b = cls.bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = cls.bufs[key] = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8,
                                            pin_memory=True)
        return b


_PIPE_STREAMS = {}


def _pipe_streams(torch, device):
    st = _PIPE_STREAMS.get(device)
    if st is None:
        st = _PIPE_STREAMS[device] = [_batch_stream(torch, device),
                                      torch.cuda.Stream(device=torch.device("cuda", device))]
    return st


def _launch_chunks(problems, cfg, device, streams, bounds):
    """Pack, upload and launch every chunk; returns the BatchRuns."""
    runs, pending = [], [None, None]
    for j in range(len(bounds) - 1):
        slot = j % 2
        if pending[slot] is not None:
            pending[slot].synchronize()           # that slot's previous upload is done
        holder = {}

        def stage(nb, slot=slot, holder=holder):
            holder["t"] = _PipeStaging.get(device, slot, nb)
            return holder["t"].numpy()

        packed = PackedBatch(problems[bounds[j]:bounds[j + 1]], staging=stage)
        run = BatchRun(packed, device=device, stream=streams[slot], staging=holder["t"])
        packed.arrays = {}                        # views of the staging buffer: released
        pending[slot] = run.h2d_done
        run.launch(cfg)
        runs.append(run)
    for ev in pending:                            # the slots are free for the next call
        if ev is not None:
            ev.synchronize()
    return runs


def _run_pipelined(problems, cfg, device):
    """Chunks of PIPE_CHUNK LPs: the host packs chunk j + 1 (into the other
    pinned slot) while chunk j uploads and solves; consecutive chunks launch on
    two streams so one launch's tail CTAs overlap the next launch's first
    wave; chunk j's reports are built while the later chunks solve.  Every LP
    is solved by its own CTA independently of the rest of the batch, so the
    reports are identical to one launch over the whole batch."""
    torch = _torch()
    streams = _pipe_streams(torch, device)
    bounds = list(range(0, len(problems), PIPE_CHUNK)) + [len(problems)]
    with _PipeStaging.lock:
        runs = _launch_chunks(problems, cfg, device, streams, bounds)
    reps = []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RestartLogOverflow)
        for j, run in enumerate(runs):
            for r in run.reports(cfg):
                r.device_stats["batch_index"] += bounds[j]
                reps.append(r)
    return reps


def solve_batch(problems, cfg=None, *, device: int = 0) -> list[SolveReport]:
    """``[solve(p, cfg) for p in problems]`` as device launches of one CTA per
    LP (one launch, or pipelined chunks of PIPE_CHUNK LPs for batches of at
    least PIPE_MIN)."""
    cfg = SolverConfig.coerce(cfg)
    if math.isfinite(cfg.time_limit_seconds):
        warnings.warn("batch time limits are measured per CTA on the device clock",
                      RuntimeWarning)
    from .device import _Staging
    if not _torch().cuda.is_available():
        raise N.NativeUnavailableError("CUDA device required: the batch path has no CPU fallback")
    problems = list(problems)
    if len(problems) >= PIPE_MIN and os.environ.get("HPR_BATCH_PIPE", "1") != "0":
        reps = _run_pipelined(problems, cfg, device)
    else:
        with _Staging.lock:
            # pack straight into the pinned staging buffer, then one H2D copy
            packed = PackedBatch(problems, staging=lambda nb: _Staging.get(nb).numpy())
            run = BatchRun(packed, device=device)
            packed.arrays = {}                    # views of the staging buffer: released
        run.launch(cfg)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RestartLogOverflow)
            reps = run.reports(cfg)
    over = [i for i, r in enumerate(reps) if r.restarts > len(r.restart_log)]
    if over:
        # the reference logs every restart: re-solve the LPs whose log overflowed
        # with room for all of them (each CTA's solve is deterministic and
        # independent of the rest of the batch, so the results are identical)
        need = max(reps[i].restarts for i in over)
        with _Staging.lock:
            sub = PackedBatch([problems[i] for i in over])
        rerun = BatchRun(sub, device=device, max_log=need)
        rerun.launch(cfg)
        for i, r in zip(over, rerun.reports(cfg)):
            r.device_stats["batch_index"] = i
            reps[i] = r
    return reps


def shard_bounds(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced shard [lo, hi) of ``count`` LPs for ``rank``."""
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def solve_batch_sharded(problems, cfg=None, *, device: int | None = None):
    """Each rank of a torch.distributed job solves its shard; returns this
    rank's reports and its [lo, hi) range (no data-path collective)."""
    import os
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    lo, hi = shard_bounds(len(problems), world, rank)
    return solve_batch(problems[lo:hi], cfg, device=device), (lo, hi)
