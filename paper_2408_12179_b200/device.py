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

import numpy as np

from . import _native as N
from .problem import stacked_arrays

PAD = 8   # trailing slots on every nonzero array (16-byte bulk-copy rounding)


def _torch():
    import torch
    return torch


class DeviceLP:
    """Uploads a reference-shaped LpProblem and owns its native context."""

    def __init__(self, problem, device: int = 0, stream=None, pinned_upload: bool = True):
        ro, ci, v, m, n, m1 = stacked_arrays(problem)
        rhs = np.concatenate([np.asarray(problem.b_eq, np.float64),
                              np.asarray(problem.b_ineq, np.float64)])
        self._setup(ro, ci, v, m, n, m1, rhs, problem.c, problem.lower, problem.upper,
                    device=device, stream=stream, pinned_upload=pinned_upload)

    @classmethod
    def from_arrays(cls, ro, ci, v, m, n, m1, b, c, lower, upper, *, device: int = 0,
                    stream=None, n_alloc: int | None = None, pinned_upload: bool = True):
        """A row block [rows of A, all n columns] (row-block mode): column vectors
        are allocated at ``n_alloc >= n`` (the group's padded length)."""
        self = cls.__new__(cls)
        self._setup(ro, ci, v, m, n, m1, b, c, lower, upper, device=device, stream=stream,
                    pinned_upload=pinned_upload, n_alloc=n_alloc)
        return self

    def _setup(self, ro, ci, v, m, n, m1, rhs, c, lower, upper, *, device, stream,
               pinned_upload, n_alloc=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise N.NativeUnavailableError("CUDA device required: the HPR-LP path has no CPU fallback")
        N.load_library()
        nnz = int(ro[-1])
        if nnz >= 2**31 - 1 or m >= 2**31 - 1 or n >= 2**31 - 1:
            raise ValueError("problem exceeds int32 indexing of this build")
        self.m, self.n, self.m1, self.nnz = m, n, m1, nnz
        na = n if n_alloc is None else int(n_alloc)
        self.n_alloc = na
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        self.h2d_bytes = 0
        dev = self.device
        f64 = dict(dtype=torch.float64, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        with torch.cuda.stream(self.stream):
            def up(arr, dtype, length=None):
                a = np.ascontiguousarray(arr, dtype=dtype)
                if length is not None and length > a.size:
                    a = np.concatenate([a, np.zeros(length - a.size, dtype=dtype)])
                t = torch.from_numpy(a)
                if pinned_upload:
                    t = t.pin_memory()
                self.h2d_bytes += t.numel() * t.element_size()
                return t.to(dev, non_blocking=True)

            T = {}
            # nonzero arrays carry PAD trailing slots: the tile engine's bulk copies
            # round every tile up to 16-byte boundaries
            T["a_rp"] = up(ro, np.int32)
            T["a_ci"] = up(np.concatenate([ci, np.zeros(PAD)]), np.int32)
            T["a_val"] = up(np.concatenate([v, np.zeros(PAD)]), np.float64)
            T["b"] = up(rhs, np.float64)
            T["c"] = up(c, np.float64, na)
            T["lower"] = up(lower, np.float64, na)
            T["upper"] = up(upper, np.float64, na)
            nz1 = nnz + PAD
            T["a_val_s"] = torch.empty(nz1, **f64)
            T["at_rp"] = torch.empty(n + 1, **i32)
            T["at_ci"] = torch.empty(nz1, **i32)
            T["at_perm"] = torch.empty(nz1, **i32)
            T["at_val"] = torch.empty(nz1, **f64)
            T["at_val_s"] = torch.empty(nz1, **f64)
            for name in ("b_s", "row_scale", "y", "anc_y", "yb", "dy"):
                T[name] = torch.empty(m, **f64)
            for name in ("c_s", "lower_s", "upper_s", "col_scale", "x", "anc_x", "w", "xb",
                         "zb", "wtmp"):
                T[name] = torch.empty(na, **f64)
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
        with torch.cuda.stream(self.stream):
            self.layout = torch.empty(max(int(nbytes.value), 16), dtype=torch.uint8,
                                      device=self.device)
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

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            N.load_library().hpr_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
