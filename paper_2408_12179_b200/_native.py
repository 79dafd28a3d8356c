"""ctypes binding of ``libhprlp_b200.so`` (the C ABI in ``include/hprlp_b200.h``).

The library is built in-tree by ``paper_2408_12179_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or CUDA is unavailable every entry point raises ``NativeUnavailableError``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPR_LIB_PATH") or os.path.join(_HERE, "libhprlp_b200.so")

HPR_OK = 0
_ERRNAMES = {-1: "HPR_EINVAL", -2: "HPR_ECUDA", -3: "HPR_ENCCL", -4: "HPR_ENOMEM",
             -5: "HPR_ESTATE"}
VARIANT_CODE = {"dr": 0, "hdr-fixed": 1, "hdr": 1, "hpr": 2}


class NativeUnavailableError(RuntimeError):
    """The CUDA library is not built or no GPU is present (no CPU fallback exists)."""


class NativeError(RuntimeError):
    def __init__(self, code, fn, msg):
        super().__init__(f"{fn} failed with {_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


c_double_p = ctypes.POINTER(ctypes.c_double)


class HprDims(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("m1", ctypes.c_int64),
                ("nnz", ctypes.c_int64)]


_BUF_FIELDS = [
    "a_rp", "a_ci", "a_val", "a_val_s", "at_rp", "at_ci", "at_perm", "at_val", "at_val_s",
    "b", "c", "lower", "upper", "b_s", "c_s", "lower_s", "upper_s", "row_scale", "col_scale",
    "y", "x", "anc_y", "anc_x", "w", "yb", "xb", "zb", "dy", "wtmp",
]


class HprBuffers(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in _BUF_FIELDS] + [
        ("cand_y", ctypes.c_void_p * 2), ("cand_x", ctypes.c_void_p * 2),
        ("cand_z", ctypes.c_void_p * 2)]


class HprScaleOut(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in
                ("b_factor", "c_factor", "bnorm_orig", "cnorm_orig", "bnorm_s", "cnorm_s")]


class HprPowerOut(ctypes.Structure):
    _fields_ = [("value", ctypes.c_double), ("raw", ctypes.c_double),
                ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32)]


CKPT_DOUBLE_FIELDS = ("bar_dx2", "bar_dy2", "dy2", "dx2", "sh2", "aty2", "prim2", "dual2",
                      "r1sq", "r2sq", "cx", "by", "lz", "uz")


class HprCkptOut(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in CKPT_DOUBLE_FIELDS] + [
        ("n_lo", ctypes.c_int64), ("n_up", ctypes.c_int64), ("clamped", ctypes.c_int64),
        ("nonfinite_k", ctypes.c_int64)]


class HprLayoutInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("slices_a", "slices_at", "slots_a", "slots_at",
                                               "long_rows_a", "long_rows_at", "cb_a", "cb_at",
                                               "split_a", "stg_a", "stg_at", "rao_a", "rao_at",
                                               "bounds_uniform", "ts_a", "ts_at", "ts_words_a",
                                               "ts_words_at")]


class HprBatchProblem(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("total_rows", ctypes.c_int64),
                ("total_cols", ctypes.c_int64), ("total_nnz", ctypes.c_int64),
                ("max_m", ctypes.c_int32), ("max_n", ctypes.c_int32), ("max_nnz", ctypes.c_int64),
                ("row_off", ctypes.c_void_p), ("col_off", ctypes.c_void_p),
                ("nz_off", ctypes.c_void_p), ("m1", ctypes.c_void_p), ("rp", ctypes.c_void_p),
                ("ci", ctypes.c_void_p), ("val", ctypes.c_void_p), ("b", ctypes.c_void_p),
                ("c", ctypes.c_void_p), ("lower", ctypes.c_void_p), ("upper", ctypes.c_void_p),
                ("obj_const", ctypes.c_void_p), ("obj_neg", ctypes.c_void_p)]


class HprBatchConfig(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in ("tolerance", "time_limit_seconds", "alpha1",
                                                "alpha2", "alpha3", "sigma0", "power_tol")] + [
        ("max_iterations", ctypes.c_int64)] + [
        (f, ctypes.c_int32) for f in ("check_interval", "variant", "ruiz_iters", "pock_chambolle",
                                      "bc_normalize", "power_max_iters", "term_original",
                                      "max_log")]


class HprRestartRec(ctypes.Structure):
    _fields_ = [("outer_index", ctypes.c_int32), ("trigger", ctypes.c_int32),
                ("tau", ctypes.c_int64), ("sigma_next", ctypes.c_double),
                ("merit", ctypes.c_double)]


class HprBatchResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("restarts", ctypes.c_int32),
                ("iterations", ctypes.c_int64)] + [
        (f, ctypes.c_int32) for f in ("power_iterations", "power_converged", "dual_clamped",
                                      "n_log", "merit_negative", "power_failed")] + [
        ("primal_objective", ctypes.c_double), ("dual_objective", ctypes.c_double),
        ("kkt", ctypes.c_double * 9)] + [
        (f, ctypes.c_double) for f in ("sigma_final", "lambda_estimate", "lambda_raw",
                                       "b_factor", "c_factor", "device_seconds")]


class HprExactBufs(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("linv", "linv_t", "u", "rhs", "h")]


# name -> (restype, argtypes); every int-returning function is error-checked
_SIGS = {
    "hpr_abi_version": (ctypes.c_int, []),
    "hpr_last_error": (ctypes.c_char_p, []),
    "hpr_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(HprDims), ctypes.POINTER(ctypes.c_size_t)]),
    "hpr_ctx_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(HprDims),
                                      ctypes.c_int, ctypes.c_void_p]),
    "hpr_ctx_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_bind": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HprBuffers), ctypes.c_void_p,
                                ctypes.c_size_t]),
    "hpr_analyze": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]),
    "hpr_bind_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "hpr_scale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(HprScaleOut)]),
    "hpr_power": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                 ctypes.POINTER(HprPowerOut)]),
    "hpr_state_reset": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_run_inner": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_int]),
    "hpr_checkpoint": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_int, ctypes.POINTER(HprCkptOut)]),
    "hpr_restart": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_kkt_origin": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(HprCkptOut)]),
    "hpr_kkt": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(HprCkptOut)]),
    "hpr_finalize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(HprCkptOut)]),
    "hpr_launch_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "hpr_layout_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HprLayoutInfo)]),
    "hpr_spmv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "hpr_small_path": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_time_phases": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double)]),
    "hpr_last_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double)]),
    # exact T1 = 0 path (hpr_exact.cuh)
    "hpr_exact_bind": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(HprExactBufs)]),
    "hpr_exact_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_double, ctypes.c_int]),
    "hpr_exact_half": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int64)]),
    "hpr_trsolve": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]),
    # row-block partitioned mode (hpr_rowblock.cuh)
    "hpr_nccl_available": (ctypes.c_int, []),
    "hpr_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t]),
    "hpr_group_dims": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_size_t)]),
    "hpr_group_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_int64), ctypes.c_size_t,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_size_t]),
    "hpr_group_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_group_col_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(ctypes.c_int64)]),
    "hpr_group_scale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(HprScaleOut)]),
    "hpr_group_power": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                       ctypes.POINTER(HprPowerOut)]),
    "hpr_group_state_reset": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_group_run_inner": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int]),
    "hpr_group_checkpoint": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(HprCkptOut)]),
    "hpr_group_restart": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_group_kkt_origin": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(HprCkptOut)]),
    "hpr_group_kkt": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(HprCkptOut)]),
    "hpr_group_finalize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(HprCkptOut)]),
    "hpr_group_last_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_double)]),
    "hpr_group_launch_count": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "hpr_group_comm_info": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 4),
    # batch of small LPs (hpr_batch.cuh)
    "hpr_batch_smem_bytes": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                            ctypes.POINTER(ctypes.c_size_t)]),
    "hpr_batch_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(HprBatchProblem),
                                                 ctypes.POINTER(ctypes.c_size_t)]),
    "hpr_batch_solve": (ctypes.c_int, [ctypes.POINTER(HprBatchProblem),
                                       ctypes.POINTER(HprBatchConfig), ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int, ctypes.c_void_p]),
    # MPS reader / writer (hpr_mps.cpp; typed precisely by paper_2408_12179_b200.mps)
    "hpr_mps_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_void_p]),
    "hpr_mps_last_error": (ctypes.c_char_p, []),
    "hpr_mps_free": (ctypes.c_int, [ctypes.c_void_p]),
    "hpr_mps_write": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p,
                                     ctypes.c_void_p]),
    "hpr_mps_free_text": (ctypes.c_int, [ctypes.c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load_library(path: str = LIB_PATH):
    """Load and type the library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hpr_abi_version() != 1:
        raise NativeUnavailableError("ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, fn: str):
    if rc != HPR_OK:
        msg = load_library().hpr_last_error()
        raise NativeError(rc, fn, msg.decode() if msg else "")


def call(name: str, *args):
    lib = load_library()
    rc = getattr(lib, name)(*args)
    check(rc, name)
    return rc
