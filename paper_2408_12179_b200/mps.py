"""MPS reading and writing through the native reader (``csrc/hpr_mps.cpp``).

Same public names and semantics as the reference (``hprlp/mps.py``):
``parse_mps(text) -> LpProblem``, ``load_mps(path)``, ``write_mps(problem,
name) -> str`` and ``MpsParseError`` (a ``ValueError`` carrying ``line_no``).
The text is tokenised and assembled in C++ (one pass, canonical CSR blocks
built directly), so a large instance goes from disk to ``solve`` without a
Python-level loop over its entries.
"""

from __future__ import annotations

import ctypes
import re
import warnings

import numpy as np

from . import _native as N
from .problem import LpProblem, SparseMatrix


class MpsParseError(ValueError):
    """mps.py:22-25: raised with the 1-based line number of the offending record."""

    def __init__(self, message: str, line_no: int):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class _Result(ctypes.Structure):
    _fields_ = [("m1", ctypes.c_int64), ("m2", ctypes.c_int64), ("n", ctypes.c_int64),
                ("eq_rp", ctypes.POINTER(ctypes.c_int64)), ("eq_ci", ctypes.POINTER(ctypes.c_int64)),
                ("eq_val", ctypes.POINTER(ctypes.c_double)),
                ("in_rp", ctypes.POINTER(ctypes.c_int64)), ("in_ci", ctypes.POINTER(ctypes.c_int64)),
                ("in_val", ctypes.POINTER(ctypes.c_double)),
                ("b_eq", ctypes.POINTER(ctypes.c_double)), ("b_ineq", ctypes.POINTER(ctypes.c_double)),
                ("c", ctypes.POINTER(ctypes.c_double)), ("lower", ctypes.POINTER(ctypes.c_double)),
                ("upper", ctypes.POINTER(ctypes.c_double)),
                ("objective_constant", ctypes.c_double), ("objective_negated", ctypes.c_int32),
                ("extra_objective_rows", ctypes.c_int32),
                ("row_names", ctypes.c_void_p), ("col_names", ctypes.c_void_p),
                ("name", ctypes.c_char_p)]


class _Problem(ctypes.Structure):
    _fields_ = [("m1", ctypes.c_int64), ("m2", ctypes.c_int64), ("n", ctypes.c_int64),
                ("eq_rp", ctypes.c_void_p), ("eq_ci", ctypes.c_void_p), ("eq_val", ctypes.c_void_p),
                ("in_rp", ctypes.c_void_p), ("in_ci", ctypes.c_void_p), ("in_val", ctypes.c_void_p),
                ("b_eq", ctypes.c_void_p), ("b_ineq", ctypes.c_void_p), ("c", ctypes.c_void_p),
                ("lower", ctypes.c_void_p), ("upper", ctypes.c_void_p),
                ("objective_constant", ctypes.c_double), ("objective_negated", ctypes.c_int32),
                ("row_names", ctypes.c_char_p), ("col_names", ctypes.c_char_p)]


def _lib():
    lib = N.load_library()
    if not getattr(lib, "_mps_typed", False):
        lib.hpr_mps_parse.argtypes = [ctypes.c_char_p, ctypes.c_size_t,
                                      ctypes.POINTER(ctypes.POINTER(_Result))]
        lib.hpr_mps_parse.restype = ctypes.c_int
        lib.hpr_mps_last_error.restype = ctypes.c_char_p
        lib.hpr_mps_free.argtypes = [ctypes.POINTER(_Result)]
        lib.hpr_mps_write.argtypes = [ctypes.POINTER(_Problem), ctypes.c_char_p,
                                      ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(ctypes.c_size_t)]
        lib.hpr_mps_write.restype = ctypes.c_int
        lib.hpr_mps_free_text.argtypes = [ctypes.c_void_p]
        lib._mps_typed = True
    return lib


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _names(ptr, count):
    if count == 0:
        return []
    out, off = [], 0
    for _ in range(count):
        s = ctypes.string_at(ptr + off)
        out.append(s.decode("utf-8"))
        off += len(s) + 1
    return out


def parse_mps(text: str | bytes) -> LpProblem:
    """Parse MPS text into the standard minimisation form (mps.py:281)."""
    if isinstance(text, str):
        text = text.encode("utf-8")
    lib = _lib()
    res = ctypes.POINTER(_Result)()
    rc = lib.hpr_mps_parse(text, len(text), ctypes.byref(res))
    if rc != 0:
        msg = lib.hpr_mps_last_error().decode()
        m = re.match(r"line (-?\d+): (.*)", msg, re.S)
        if m:
            raise MpsParseError(m.group(2), int(m.group(1)))
        raise RuntimeError(msg)
    try:
        r = res.contents
        m1, m2, n = int(r.m1), int(r.m2), int(r.n)
        if r.extra_objective_rows:
            warnings.warn(f"dropped {r.extra_objective_rows} extra objective row(s)", UserWarning)
        erp = _arr(r.eq_rp, m1 + 1, np.int64)
        irp = _arr(r.in_rp, m2 + 1, np.int64)
        a_eq = SparseMatrix.from_csr_arrays(erp, _arr(r.eq_ci, int(erp[-1]), np.int64),
                                            _arr(r.eq_val, int(erp[-1]), np.float64), m1, n)
        a_in = SparseMatrix.from_csr_arrays(irp, _arr(r.in_ci, int(irp[-1]), np.int64),
                                            _arr(r.in_val, int(irp[-1]), np.float64), m2, n)
        return LpProblem(a_eq=a_eq, a_ineq=a_in, b_eq=_arr(r.b_eq, m1, np.float64),
                         b_ineq=_arr(r.b_ineq, m2, np.float64), c=_arr(r.c, n, np.float64),
                         lower=_arr(r.lower, n, np.float64), upper=_arr(r.upper, n, np.float64),
                         objective_constant=float(r.objective_constant),
                         objective_negated=bool(r.objective_negated),
                         row_names=_names(r.row_names, m1 + m2),
                         col_names=_names(r.col_names, n))
    finally:
        lib.hpr_mps_free(res)


def load_mps(path) -> LpProblem:
    with open(path, "rb") as fh:
        return parse_mps(fh.read())


def write_mps(problem, name: str = "LP") -> str:
    """Standard form back to MPS text; parse_mps(write_mps(p)) reproduces p
    (mps.py:295-364)."""
    p = problem
    m1, m2, n = int(p.a_eq.nrows), int(p.a_ineq.nrows), int(p.a_eq.ncols)
    keep = []

    def arr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a.ctypes.data

    rows = getattr(p, "row_names", None)
    cols = getattr(p, "col_names", None)
    pr = _Problem(m1, m2, n, arr(p.a_eq.row_offsets, np.int64), arr(p.a_eq.col_indices, np.int64),
                  arr(p.a_eq.values, np.float64), arr(p.a_ineq.row_offsets, np.int64),
                  arr(p.a_ineq.col_indices, np.int64), arr(p.a_ineq.values, np.float64),
                  arr(p.b_eq, np.float64), arr(p.b_ineq, np.float64), arr(p.c, np.float64),
                  arr(p.lower, np.float64), arr(p.upper, np.float64),
                  float(getattr(p, "objective_constant", 0.0)),
                  int(bool(getattr(p, "objective_negated", False))),
                  ("\0".join(rows) + "\0").encode() if rows and len(rows) == m1 + m2 else None,
                  ("\0".join(cols) + "\0").encode() if cols and len(cols) == n else None)
    lib = _lib()
    text = ctypes.c_void_p()
    ln = ctypes.c_size_t(0)
    rc = lib.hpr_mps_write(ctypes.byref(pr), name.encode(), ctypes.byref(text), ctypes.byref(ln))
    if rc != 0:
        raise RuntimeError(lib.hpr_mps_last_error().decode())
    try:
        return ctypes.string_at(text.value, ln.value).decode("utf-8")
    finally:
        lib.hpr_mps_free_text(text)
