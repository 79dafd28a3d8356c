"""The native batch packer (csrc/hpr_host.cpp) writes exactly the arrays the
numpy concatenation path writes (CPU only: no device needed)."""
import numpy as np
import pytest

import paper_2408_12179_b200 as P
from paper_2408_12179_b200 import batch as BT


def _probs():
    rng = np.random.default_rng(4)
    out = [P.generate_known_solution_lp(300 + i, 7 + i % 3, 5 + i % 4, 30 + i, 0.3)[0]
           for i in range(40)]
    # an equality-only and an inequality-only LP, int32 index arrays
    out.append(P.LpProblem.from_dense(rng.uniform(-1, 1, (4, 6)), np.ones(4), None, None,
                                      rng.uniform(0, 1, 6)))
    out.append(P.LpProblem.from_dense(None, None, rng.uniform(-1, 1, (3, 5)), -np.ones(3),
                                      rng.uniform(0, 1, 5)))
    return out


def test_native_pack_matches_numpy(monkeypatch):
    if BT._host_module() is None:
        pytest.skip("native host module not built")
    probs = _probs()
    monkeypatch.setenv("HPR_PACK_NATIVE", "0")
    ref = BT.PackedBatch(probs)
    monkeypatch.setenv("HPR_PACK_NATIVE", "1")
    got = BT.PackedBatch(probs)
    for k, a in ref.arrays.items():
        assert got.arrays[k].dtype == a.dtype, k
        assert np.array_equal(got.arrays[k], a), k
    # into a staging buffer (the upload layout), as solve_batch does
    buf = np.zeros(1 << 22, np.uint8)
    st = BT.PackedBatch(probs, staging=lambda nb: buf)
    for k, a in ref.arrays.items():
        assert np.array_equal(st.arrays[k], a), k


def test_native_pack_rejects_bad_dtype(monkeypatch):
    host = BT._host_module()
    if host is None:
        pytest.skip("native host module not built")
    probs = _probs()[:2]
    pk = BT.PackedBatch(probs)
    import types
    q = probs[1]
    probs[1] = types.SimpleNamespace(a_eq=q.a_eq, a_ineq=q.a_ineq, b_eq=q.b_eq, b_ineq=q.b_ineq,
                                     c=q.c.astype(np.float32), lower=q.lower, upper=q.upper)
    out = {k: np.empty_like(v) for k, v in pk.arrays.items()}
    with pytest.raises(ValueError):
        host.pack_batch(probs, out, pk.row_off, pk.col_off, pk.nz_off, 2)
