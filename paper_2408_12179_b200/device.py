"""Device residency of one LP: PyTorch allocations + one native context.

PyTorch is the allocator and stream provider only; every computation on these
buffers is a kernel of ``libhprlp_b200.so`` launched through the C ABI.

HBM layout (all arrays contiguous, fp64 values, int32 indices):

  A      : a_rp[m+1] a_ci[nnz] a_val[nnz] a_val_s[nnz]          (CSR, row-major)
  A^T    : at_rp[n+1] at_ci[nnz] at_perm[nnz] at_val[nnz] at_val_s[nnz]
  problem: b c lower upper (original) | b_s c_s lower_s upper_s (scaled)
  scaling: row_scale[m] col_scale[n]
  state  : y anc_y yb dy [m] | x anc_x w xb zb wtmp [n] | cand_{y,x,z}[2]
  ws     : native workspace (tiles, partials, params, CUB scratch)

Per nonzero 2 x (8 + 4) bytes are resident for the scaled copies plus the same
again for the unscaled values (KKT residuals use the user's matrix).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N

PAD = 8   # trailing slots on every nonzero array (16-byte bulk-copy rounding)


def _torch():
    import torch
    return torch


class _Staging:
    """Process-wide pinned host staging buffer for uploads (grown on demand,
    reused across problems: no per-upload page-locking)."""

    buf = None
    lock = threading.RLock()

    @classmethod
    def get(cls, nbytes):
        torch = _torch()
        if cls.buf is None or cls.buf.numel() < nbytes:
            cls.buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        return cls.buf


_POOL = None
_PF_POOL = None
_BIG_SOLUTION = 32 << 20   # solution bytes from which the staged download pays off


def _par_copy(dst, src):
    """np.copyto(dst, src, casting="unsafe") split over a small thread pool
    (numpy releases the GIL; one core copies ~10 GB/s, the staging of a
    5M-nonzero problem is ~66 MB)."""
    global _POOL
    n = src.size
    if n < (1 << 20):
        np.copyto(dst, src, casting="unsafe")
        return
    if _POOL is None:
        import concurrent.futures
        import os
        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    k = _POOL._max_workers
    step = -(-n // k)
    futs = [_POOL.submit(np.copyto, dst[a:a + step], src[a:a + step], casting="unsafe")
            for a in range(0, n, step)]
    for f in futs:
        f.result()


def _csr_parts(problem):
    """The stacked A = [A_eq; A_ineq] as (row_offsets, col_indices, values)
    pieces, written straight into the staging buffer (problem.py:75-82)."""
    top, bot = problem.a_eq, problem.a_ineq
    return [(np.asarray(top.row_offsets), np.asarray(top.col_indices), np.asarray(top.values)),
            (np.asarray(bot.row_offsets), np.asarray(bot.col_indices), np.asarray(bot.values))]


class DeviceLP:
    """Uploads a reference-shaped LpProblem and owns its native context."""

    def __init__(self, problem, device: int = 0, stream=None):
        parts = _csr_parts(problem)
        m1 = int(problem.a_eq.nrows)
        m = m1 + int(problem.a_ineq.nrows)
        n = int(problem.a_eq.ncols)
        self._setup(parts, m, n, m1, (problem.b_eq, problem.b_ineq), problem.c, problem.lower,
                    problem.upper, device=device, stream=stream)

    def dims_key(self):
        return (self.device.index, self.m, self.n, self.m1, self.nnz, self.n_alloc)

    @staticmethod
    def problem_key(problem, device: int):
        top, bot = problem.a_eq, problem.a_ineq
        n = int(top.ncols)
        nnz = int(top.row_offsets[-1]) - int(top.row_offsets[0]) + \
            int(bot.row_offsets[-1]) - int(bot.row_offsets[0])
        return (device, int(top.nrows) + int(bot.nrows), n, int(top.nrows), nnz, n)

    def reload(self, problem):
        """Upload another problem of identical dimensions into these buffers
        (inputs are re-copied and re-analysed; the context, the workspace and,
        when the layout comes out identical, the captured graphs are reused)."""
        if DeviceLP.problem_key(problem, self.device.index) != self.dims_key():
            raise ValueError("reload needs a problem of identical dimensions")
        self._setup(_csr_parts(problem), self.m, self.n, self.m1,
                    (problem.b_eq, problem.b_ineq), problem.c, problem.lower, problem.upper,
                    device=self.device.index, stream=self.stream, n_alloc=self.n_alloc)

    @classmethod
    def from_arrays(cls, ro, ci, v, m, n, m1, b, c, lower, upper, *, device: int = 0,
                    stream=None, n_alloc: int | None = None):
        """A row block [rows of A, all n columns] (row-block mode): column vectors
        are allocated at ``n_alloc >= n`` (the group's padded length)."""
        self = cls.__new__(cls)
        self._setup([(np.asarray(ro), np.asarray(ci), np.asarray(v))], m, n, m1, (b,), c, lower,
                    upper, device=device, stream=stream, n_alloc=n_alloc)
        return self

    def _setup(self, parts, m, n, m1, rhs_parts, c, lower, upper, *, device, stream,
               n_alloc=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise N.NativeUnavailableError("CUDA device required: the HPR-LP path has no CPU fallback")
        N.load_library()
        nnz = int(sum(int(ro[-1]) - int(ro[0]) for ro, _, _ in parts))
        if nnz >= 2**31 - 1 or m >= 2**31 - 1 or n >= 2**31 - 1:
            raise ValueError("problem exceeds int32 indexing of this build")
        self.m, self.n, self.m1, self.nnz = m, n, m1, nnz
        na = n if n_alloc is None else int(n_alloc)
        self.n_alloc = na
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        dev = self.device
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        nz1 = nnz + PAD

        # host inputs -> one pinned staging buffer -> one H2D copy; every input
        # array is a view of the device copy.  Writers cast in place (int64 ->
        # int32), so no host temporaries are made.
        def w_rp(dst):
            off, r = 0, 0
            for ro, _, _ in parts:
                k = len(ro) - 1
                np.copyto(dst[r:r + k], ro[:-1] - ro[0] + off, casting="unsafe")
                off += int(ro[-1]) - int(ro[0])
                r += k
            dst[r] = off

        def w_nz(which, pad):
            def fill(dst):
                o = 0
                for piece in parts:
                    a = piece[which]
                    _par_copy(dst[o:o + a.size], a)
                    o += a.size
                dst[o:] = pad
            return fill

        def w_vec(arrs, length):
            def fill(dst):
                o = 0
                for a in arrs:
                    a = np.asarray(a)
                    _par_copy(dst[o:o + a.size], a)
                    o += a.size
                dst[o:length] = 0.0
            return fill

        spec = [("a_rp", np.int32, m + 1, w_rp), ("a_ci", np.int32, nz1, w_nz(1, 0)),
                ("a_val", np.float64, nz1, w_nz(2, 0.0)), ("b", np.float64, m, w_vec(rhs_parts, m)),
                ("c", np.float64, na, w_vec((c,), na)), ("lower", np.float64, na, w_vec((lower,), na)),
                ("upper", np.float64, na, w_vec((upper,), na))]
        offs, total = [], 0
        for _, dt, ln, _ in spec:
            offs.append(total)
            total += (ln * np.dtype(dt).itemsize + 255) // 256 * 256
        T = {}
        if getattr(self, "_inputs", None) is None or self._inputs.numel() != total:
            with torch.cuda.stream(self.stream):
                self._inputs = torch.empty(total, dtype=torch.uint8, device=dev)
        with _Staging.lock:
            stage = _Staging.get(total)
            host = stage.numpy()
            # each array's DMA is issued as soon as it is staged, so the copy of
            # array i overlaps the host-side fill of array i+1
            for (name, dt, ln, fill), o in zip(spec, offs):
                nb = ln * np.dtype(dt).itemsize
                fill(host[o:o + nb].view(dt))
                with torch.cuda.stream(self.stream):
                    self._inputs[o:o + nb].copy_(stage[o:o + nb], non_blocking=True)
            self.stream.synchronize()       # the staging buffer is reusable after this
        if getattr(self, "ctx", None) is not None:
            self.h2d_bytes = total
            self.analyzed = False           # a reload: same buffers, new contents
            return
        tdt = {np.int32: torch.int32, np.float64: torch.float64}
        for (name, dt, ln, _), o in zip(spec, offs):
            T[name] = self._inputs[o:o + ln * np.dtype(dt).itemsize].view(tdt[dt])
        self.h2d_bytes = total
        with torch.cuda.stream(self.stream):
            nz1 = nnz + PAD
            T["a_val_s"] = torch.empty(nz1, **f64)
            T["at_rp"] = torch.empty(n + 1, **i32)
            T["at_ci"] = torch.empty(nz1, **i32)
            T["at_perm"] = torch.empty(nz1, **i32)
            T["at_val"] = torch.empty(nz1, **f64)
            T["at_val_s"] = torch.empty(nz1, **f64)
            for name in ("b_s", "row_scale", "y", "anc_y", "yb", "dy"):
                # gathered vectors are read in 16-byte bulk copies: keep slack after them
                T[name] = torch.empty(m + 8, **f64)[:m]
            for name in ("c_s", "lower_s", "upper_s", "col_scale", "x", "anc_x", "w", "xb",
                         "zb", "wtmp"):
                T[name] = torch.empty(na + 8, **f64)[:na]
            T["cand_y"] = [torch.empty(m, **f64) for _ in range(2)]
            T["cand_x"] = [torch.empty(na, **f64) for _ in range(2)]
            T["cand_z"] = [torch.empty(na, **f64) for _ in range(2)]
        self.t = T
        self.dims = N.HprDims(m, n, m1, nnz)
        wsb = ctypes.c_size_t(0)
        N.call("hpr_workspace_bytes", ctypes.byref(self.dims), ctypes.byref(wsb))
        with torch.cuda.stream(self.stream):
            self.ws = torch.empty(max(int(wsb.value), 1), dtype=torch.uint8, device=dev)
        bufs = N.HprBuffers()
        for f in N._BUF_FIELDS:
            setattr(bufs, f, T[f].data_ptr())
        for i in range(2):
            bufs.cand_y[i] = T["cand_y"][i].data_ptr()
            bufs.cand_x[i] = T["cand_x"][i].data_ptr()
            bufs.cand_z[i] = T["cand_z"][i].data_ptr()
        self._bufs = bufs
        ctx = ctypes.c_void_p()
        N.call("hpr_ctx_create", ctypes.byref(ctx), ctypes.byref(self.dims), device,
               ctypes.c_void_p(self.stream.cuda_stream))
        self.ctx = ctx
        N.call("hpr_bind", ctx, ctypes.byref(bufs), ctypes.c_void_p(self.ws.data_ptr()),
               ctypes.c_size_t(self.ws.numel()))
        self.analyzed = False

    # ------------------------------------------------------------------
    def analyze(self):
        """Transpose + SELL-32-sigma layout (hpr_analyze / hpr_bind_layout)."""
        torch = _torch()
        nbytes = ctypes.c_size_t(0)
        N.call("hpr_analyze", self.ctx, ctypes.byref(nbytes))
        need = max(int(nbytes.value), 16)
        if getattr(self, "layout", None) is None or self.layout.numel() != need:
            with torch.cuda.stream(self.stream):
                self.layout = torch.empty(need, dtype=torch.uint8, device=self.device)
        N.call("hpr_bind_layout", self.ctx, ctypes.c_void_p(self.layout.data_ptr()),
               ctypes.c_size_t(self.layout.numel()))
        self.analyzed = True

    def scale(self, ruiz_iters: int, pock_chambolle: bool, bc_normalize: bool):
        out = N.HprScaleOut()
        N.call("hpr_scale", self.ctx, int(ruiz_iters), int(bool(pock_chambolle)),
               int(bool(bc_normalize)), ctypes.byref(out))
        return out

    def power(self, tol: float, max_iters: int):
        out = N.HprPowerOut()
        N.call("hpr_power", self.ctx, float(tol), int(max_iters), ctypes.byref(out))
        return out

    def state_reset(self):
        N.call("hpr_state_reset", self.ctx)

    def run_inner(self, steps, t, k, sigma, lamsig, variant_code):
        N.call("hpr_run_inner", self.ctx, int(steps), int(t), int(k), float(sigma),
               float(lamsig), int(variant_code))

    def checkpoint(self, sigma, lamsig, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_checkpoint", self.ctx, float(sigma), float(lamsig), int(term_original),
               int(slot), ctypes.byref(out))
        return out

    def restart(self):
        N.call("hpr_restart", self.ctx)

    def kkt_origin(self, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_kkt_origin", self.ctx, int(term_original), int(slot), ctypes.byref(out))
        return out

    def spmv(self, transpose: bool, x, y):
        """y = A x or A^T x on the current (scaled) values (device tensors,
        the context's stream; hpr_spmv)."""
        N.call("hpr_spmv", self.ctx, int(bool(transpose)), ctypes.c_void_p(x.data_ptr()),
               ctypes.c_void_p(y.data_ptr()))

    def kkt(self, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_kkt", self.ctx, int(term_original), int(slot), ctypes.byref(out))
        return out

    def finalize(self, term_original, slot):
        out = N.HprCkptOut()
        N.call("hpr_finalize", self.ctx, int(term_original), int(slot), ctypes.byref(out))
        return out

    def launch_count(self) -> int:
        v = ctypes.c_int64(0)
        N.call("hpr_launch_count", self.ctx, ctypes.byref(v))
        return int(v.value)

    def layout_info(self) -> dict:
        info = N.HprLayoutInfo()
        N.call("hpr_layout_info", self.ctx, ctypes.byref(info))
        return {f: int(getattr(info, f)) for f, _ in N.HprLayoutInfo._fields_}

    def small_path(self) -> bool:
        """True when run_inner takes the resident small-LP loop (no separate
        phase kernels to time)."""
        return bool(N.load_library().hpr_small_path(self.ctx))

    def time_phases(self, reps: int = 20):
        """(x-phase, y-phase) microseconds per launch, ``reps`` launches each
        (hpr_time_phases: overwrites the iterate -- after a solve only)."""
        a, b = ctypes.c_double(0.0), ctypes.c_double(0.0)
        N.call("hpr_time_phases", self.ctx, int(reps), ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def last_times(self):
        a, b = ctypes.c_double(0), ctypes.c_double(0)
        N.call("hpr_last_times", self.ctx, ctypes.byref(a), ctypes.byref(b))
        return float(a.value) / 1e3, float(b.value) / 1e3

    def synchronize(self):
        self.stream.synchronize()

    def to_host(self, name, slot=None):
        t = self.t[name] if slot is None else self.t[name][slot]
        if name in ("a_ci", "a_val", "a_val_s", "at_ci", "at_perm", "at_val", "at_val_s"):
            t = t[:self.nnz]
        elif t.numel() == self.n_alloc and self.n_alloc != self.n:
            t = t[:self.n]
        self.stream.synchronize()
        return t.cpu().numpy()

    def prefault_solution(self):
        """Start allocating the solution arrays (y[m], z[n], x[n]) on a host
        thread and touch their pages while the solve runs (a fresh 268 MB
        array costs ~0.1 s of page faults when first written).  None for small
        problems and unless HPR_PREFAULT=1."""
        import os
        # opt-in (HPR_PREFAULT=1): C3 solution_to_host 35 -> 24 ms, but the
        # faulting thread slowed the next upload / teardown of e2e solves
        if 8 * (self.m + 2 * self.n) < _BIG_SOLUTION or os.environ.get("HPR_PREFAULT") != "1":
            return None
        global _PF_POOL
        if _PF_POOL is None:
            import concurrent.futures
            _PF_POOL = concurrent.futures.ThreadPoolExecutor(max_workers=1)

        def alloc(m, n):
            out = (np.empty(m), np.empty(n), np.empty(n))
            for a in out:
                a.fill(0.0)
            return out
        return _PF_POOL.submit(alloc, self.m, self.n)

    def solution_to_host(self, slot, prefault=None):
        """(y, z, x) of candidate slot ``slot`` as fresh numpy arrays: one D2H
        of the three vectors into the pinned staging buffer, then a threaded
        copy into new arrays (the page faults spread over the copy threads) or
        into the ones ``prefault`` prepared.  C3: 35 ms, against 285 ms for
        three torch ``.cpu()`` downloads into fresh pageable arrays."""
        m, n = self.m, self.n
        total = 8 * (m + 2 * n)
        if total < _BIG_SOLUTION:
            return tuple(self.to_host(nm, slot) for nm in ("cand_y", "cand_z", "cand_x"))
        torch = _torch()
        with _Staging.lock:
            st = _Staging.get(total)[:total].view(torch.float64)
            with torch.cuda.stream(self.stream):
                st[:m].copy_(self.t["cand_y"][slot][:m], non_blocking=True)
                st[m:m + n].copy_(self.t["cand_z"][slot][:n], non_blocking=True)
                st[m + n:].copy_(self.t["cand_x"][slot][:n], non_blocking=True)
            out = prefault.result() if prefault is not None else (np.empty(m), np.empty(n),
                                                                   np.empty(n))
            self.stream.synchronize()
            src = st.numpy()
            _par_copy(out[0], src[:m])
            _par_copy(out[1], src[m:m + n])
            _par_copy(out[2], src[m + n:])
        return out

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            N.load_library().hpr_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
