"""B200-native HPR-LP: the restarted Halpern Peaceman-Rachford LP iteration
loop (arXiv 2408.12179) on hand-written sm_100a CUDA.

Drop-in for the reference's solve path: ``solve(problem, cfg) -> SolveReport``
with the reference's ``SolverConfig`` option names and ``SolveReport`` result
object (reference ``hprlp/driver.py``).  The arithmetic runs in
``libhprlp_b200.so`` (C ABI: ``include/hprlp_b200.h``); there is no CPU path.
"""

from .driver import (KktResidual, RestartEvent, RestartKind, SolveReport, SolverConfig,
                     SolveStatus, Timings, Variant, check_restart, check_termination,
                     kkt_residual, sigma_guards_pass, solve)
from .batch import solve_batch, solve_batch_sharded
from .rowblock import solve_distributed, solve_row_block
from .generators import generate_flow_lp, generate_known_solution_lp, generate_planted_lp_fast
from .exact import (halpern_padmm_trace, hpr_no_prox_trace, max_trace_gap, solve_equality_exact,
                    solve_normal_equations)
from .mps import MpsParseError, load_mps, parse_mps, write_mps
from .problem import (DimensionMismatchError, LpProblem, PrimalDualPoint, SparseMatrix,
                      dual_objective, primal_objective, project_onto_box,
                      project_onto_dual_cone)

__version__ = "0.1.0"

__all__ = [
    "DimensionMismatchError", "KktResidual", "LpProblem", "MpsParseError", "load_mps",
    "parse_mps", "write_mps", "PrimalDualPoint", "RestartEvent",
    "RestartKind", "SolveReport", "SolveStatus", "SolverConfig", "SparseMatrix", "Timings",
    "Variant", "check_restart", "check_termination", "dual_objective",
    "generate_flow_lp", "halpern_padmm_trace", "hpr_no_prox_trace", "max_trace_gap",
    "solve_equality_exact", "solve_normal_equations", "generate_known_solution_lp", "generate_planted_lp_fast",
    "kkt_residual", "primal_objective", "project_onto_box", "project_onto_dual_cone",
    "sigma_guards_pass", "solve", "solve_batch", "solve_batch_sharded", "solve_distributed", "solve_row_block",
]
