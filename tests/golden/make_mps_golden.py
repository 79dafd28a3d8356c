"""Golden fixtures for the MPS reader / writer, produced by the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_mps_golden.py

Writes ``tests/golden/mps_golden.json``: for every case, the MPS text and what
the reference's ``parse_mps`` returns (dense blocks, vectors, names, flags,
warnings) or the ``MpsParseError`` message; for generated problems also the
reference's ``write_mps`` text.  Test-time code only reads the JSON.
"""

from __future__ import annotations

import json
import math
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import hprlp  # noqa: E402
from hprlp.mps import generate_degenerate_lp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _f(v):
    v = float(v)
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if math.isnan(v):
        return "nan"
    return v


def describe(p):
    return {"m1": p.m1, "m2": p.m2, "n": p.n,
            "a_eq": {"rp": p.a_eq.row_offsets.tolist(), "ci": p.a_eq.col_indices.tolist(),
                     "v": [_f(x) for x in p.a_eq.values]},
            "a_ineq": {"rp": p.a_ineq.row_offsets.tolist(), "ci": p.a_ineq.col_indices.tolist(),
                       "v": [_f(x) for x in p.a_ineq.values]},
            "b_eq": [_f(x) for x in p.b_eq], "b_ineq": [_f(x) for x in p.b_ineq],
            "c": [_f(x) for x in p.c], "lower": [_f(x) for x in p.lower],
            "upper": [_f(x) for x in p.upper],
            "objective_constant": _f(p.objective_constant),
            "objective_negated": bool(p.objective_negated),
            "row_names": list(p.row_names or []), "col_names": list(p.col_names or [])}


TEXT_CASES = {
    "l_row": "NAME T\nROWS\n N OBJ\n L C1\nCOLUMNS\n X1 OBJ 1.0 C1 1.0\n X2 C1 1.0\nRHS\n R C1 2.0\nENDATA\n",
    "max_objective_rhs": "NAME T\nOBJSENSE\n    MAX\nROWS\n N OBJ\n G C1\nCOLUMNS\n X1 OBJ 3.0 C1 1.0\nRHS\n R C1 1.0 OBJ 2.0\nENDATA\n",
    "objsense_inline": "NAME T\nOBJSENSE MAXIMIZE\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 OBJ 3.0 C1 1.0\n X2 OBJ -1 C1 1\nRHS\n C1 1.0\nENDATA\n",
    "ranges_all_kinds": ("NAME R\nROWS\n N OBJ\n G G1\n L L1\n E E1\n E E2\nCOLUMNS\n"
                         " X1 OBJ 1.0 G1 2.0\n X1 L1 1.0 E1 1.0\n X2 E2 1.0 L1 -1.0\n X2 G1 1.0\n"
                         "RHS\n RHS G1 1.0 L1 4.0\n RHS E1 2.0 E2 -1.0\nRANGES\n RNG G1 4.0 L1 -3.0\n"
                         " RNG E1 -3.0 E2 2.5\nENDATA\n"),
    "bounds_all_kinds": ("NAME B\nROWS\n N COST\n E R1\nCOLUMNS\n A COST 1 R1 1\n B COST 2 R1 1\n"
                         " C COST 3 R1 1\n D COST 4 R1 1\n E COST 5 R1 1\n F R1 1\n G R1 2\n"
                         "RHS\n RHS R1 10\nBOUNDS\n LO BND A -2.5\n UP BND A 7\n FX BND B 1.25\n"
                         " FR BND C\n MI BND D\n UP BND D 3\n PL BND E\n BV BND F\n up BND G 1e3\n"
                         "ENDATA\n"),
    "markers_comments_tabs": ("* a comment\nNAME\tTABS\nROWS\n N\tOBJ\n G\tC1\n\n* another\n"
                              "COLUMNS\n    MARKER                 'MARKER'                 'INTORG'\n"
                              "\tX1\tOBJ\t1.5\tC1\t2\n    MARKER                 'MARKER'                 'INTEND'\n"
                              " X2 C1 3\nRHS\n RHS C1 1\nENDATA\n"),
    "duplicates_and_zeros": ("NAME D\nROWS\n N OBJ\n E C1\n G C2\nCOLUMNS\n X1 C1 1.0 C1 2.0\n"
                             " X1 C2 0.0 OBJ 1\n X2 C2 5.0 C2 -5.0\n X3 OBJ 2 OBJ 3 C1 1e-300\n"
                             "RHS\n RHS C1 1\nENDATA\n"),
    "numeric_forms": ("NAME N\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 OBJ 1_000.5 C1 +.5\n"
                      " X2 OBJ 5. C1 -2E-3\n X3 OBJ 1e1_0 C1 3\nRHS\n C1 7\nBOUNDS\n UP B X1 Infinity\n"
                      " LO B X2 -INF\nENDATA\n"),
    "crlf": "NAME T\r\nROWS\r\n N OBJ\r\n E C1\r\nCOLUMNS\r\n X1 OBJ 1.0 C1 1.0\r\nRHS\r\n R C1 3\r\nENDATA\r\n",
    "extra_objective": "NAME T\nROWS\n N OBJ\n N OBJ2\n E C1\nCOLUMNS\n X1 OBJ 1.0 C1 1.0 OBJ2 5\nRHS\n R C1 1.0\nENDATA\n",
    "extra_objective_warn": "NAME T\nROWS\n N OBJ\n N OBJ2\n N OBJ3\n E C1\nCOLUMNS\n X1 OBJ 1.0 C1 1.0\nRHS\n R C1 1.0\nENDATA\n",
    "no_endata_free_rhs": "NAME T\nROWS\n N OBJ\n G C1\nCOLUMNS\n X1 OBJ 1 C1 1\nRHS\n C1 4\n",
    # errors
    "err_unknown_row": "NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 OBJ 1.0 NOPE 1.0\nRHS\nENDATA\n",
    "err_section_order": "NAME T\nCOLUMNS\n X1 OBJ 1.0\nROWS\n N OBJ\nENDATA\n",
    "err_rhs_before_columns": "NAME T\nROWS\n N OBJ\nRHS\n R C1 1\nENDATA\n",
    "err_conflicting_bounds": ("NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 OBJ 1.0 C1 1.0\n"
                               "BOUNDS\n LO BND X1 5.0\n UP BND X1 1.0\nENDATA\n"),
    "err_bad_numeric": "NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 OBJ 0x10 C1 1.0\nENDATA\n",
    "err_bad_row_kind": "NAME T\nROWS\n Q C1\nENDATA\n",
    "err_duplicate_row": "NAME T\nROWS\n N OBJ\n E C1\n G C1\nENDATA\n",
    "err_unknown_section": "NAME T\nROWS\n N OBJ\n E C1\nFOO\nENDATA\n",
    "err_bound_kind": "NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 C1 1\nBOUNDS\n ZZ B X1 1\nENDATA\n",
    "err_bound_unknown_col": "NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 C1 1\nBOUNDS\n UP B X9 1\nENDATA\n",
    "err_ranges_objective": "NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 C1 1\nRANGES\n R OBJ 1\nENDATA\n",
    "err_columns_arity": "NAME T\nROWS\n N OBJ\n E C1\nCOLUMNS\n X1 C1\nENDATA\n",
    "err_missing_columns": "NAME T\nROWS\n N OBJ\n E C1\nENDATA\n",
    "err_data_before_section": " X1 C1 1\nNAME T\n",
}


def parse_case(text):
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        try:
            p = hprlp.parse_mps(text)
        except hprlp.MpsParseError as e:
            return {"error": str(e), "line_no": e.line_no}
    return {"problem": describe(p), "warnings": [str(x.message) for x in w]}


def main():
    out = {"text_cases": {}, "generated": []}
    for name, text in TEXT_CASES.items():
        out["text_cases"][name] = {"text": text, **parse_case(text)}
    gens = []
    for seed in range(3):
        prob, _ = hprlp.generate_known_solution_lp(seed, m1=4, m2=3, n=9, density=0.5)
        gens.append((f"known_{seed}", prob))
    gens.append(("degenerate_7", generate_degenerate_lp(7)))
    rng = np.random.default_rng(5)
    q = hprlp.QapInstance(3, rng.integers(0, 5, (3, 3)).astype(float),
                          rng.integers(1, 6, (3, 3)).astype(float))
    gens.append(("qap3", hprlp.generate_qap_lp(q)))
    prob, _ = hprlp.generate_known_solution_lp(11, m1=2, m2=2, n=6, density=0.6)
    flipped = type(prob)(a_eq=prob.a_eq, a_ineq=prob.a_ineq, b_eq=prob.b_eq, b_ineq=prob.b_ineq,
                         c=prob.c, lower=prob.lower, upper=prob.upper, objective_constant=1.5,
                         objective_negated=True)
    gens.append(("negated_11", flipped))
    for name, p in gens:
        text = hprlp.write_mps(p, name="G")
        out["generated"].append({"name": name, "problem": describe(p), "text": text,
                                 "reparsed": describe(hprlp.parse_mps(text))})
    with open(os.path.join(HERE, "mps_golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("cases:", len(out["text_cases"]), "generated:", len(out["generated"]))


if __name__ == "__main__":
    main()
