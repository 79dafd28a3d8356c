/* hprlp_b200.h -- C ABI of the B200-native HPR-LP iteration loop.
 *
 * The reference (/root/reference/pkg/src/hprlp) is pure Python; its only seam on
 * this path is `solve(problem, cfg) -> SolveReport` (driver.py:281).  The
 * functions below replace, one for one, the internal steps that `solve` runs
 * between building ProblemData and writing the report (driver.py:293-372):
 *
 *   hpr_analyze      <- SparseMatrix._csr_t (sparse.py:98-100): the explicit
 *                       transpose, built lazily by the reference on first use;
 *                       also plans the SELL-32-sigma iteration layout
 *   hpr_bind_layout  <- (no reference counterpart) binds + fills that layout
 *   hpr_scale        <- scale_problem (scaling.py:72-125)
 *   hpr_power        <- power_method_lambda_max (sparse.py:165-203)
 *   hpr_run_inner    <- run_inner / iterate_once (core.py:163-179)
 *   hpr_checkpoint   <- half_step (core.py:118-129) + ScalingInfo.unscale_point
 *                       (scaling.py:45-49) + clip (driver.py:336) + kkt_residual
 *                       (driver.py:191-228) + the dot products of m_norm_diff
 *                       (core.py:182-201) and sigma_update (driver.py:273-274)
 *   hpr_restart      <- anchor = current = bar (driver.py:363-364)
 *   hpr_kkt_origin   <- the origin fallback of driver.py:374-380
 *   hpr_kkt          <- kkt_residual (driver.py:191-228) of a caller-supplied point
 *   hpr_finalize     <- the final unscale + objectives (driver.py:382-391)
 *
 * Conventions
 *   - Every function returns HPR_OK (0) or a negative HPR_E* code and never
 *     aborts; hpr_last_error() gives the message of the calling thread's last
 *     failure.
 *   - All array pointers are DEVICE pointers owned by the caller (the Python
 *     host allocates them with PyTorch).  The context owns only its CUDA graphs,
 *     events, pinned scalar buffers and the carve-up of the caller's workspace.
 *   - Index arrays are int32 (nnz < 2^31); values are IEEE fp64.
 *   - Work is asynchronous on the context's stream except where a function
 *     returns host scalars (hpr_analyze, hpr_scale, hpr_power, hpr_checkpoint,
 *     hpr_kkt, hpr_kkt_origin, hpr_finalize), which synchronise once.
 *   - One context per (device, stream); calls on one context must be serialised
 *     by the caller; distinct contexts may run concurrently.
 *   - Non-finite iterates are data (hpr_ckpt_out.nonfinite_k), not errors,
 *     preserving the reference's status semantics (driver.py:323-326).
 */
#ifndef HPRLP_B200_H
#define HPRLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPR_OK 0
#define HPR_EINVAL (-1)
#define HPR_ECUDA (-2)
#define HPR_ENCCL (-3)
#define HPR_ENOMEM (-4)
#define HPR_ESTATE (-5)

#define HPR_VARIANT_DR 0        /* core.py:146-147 */
#define HPR_VARIANT_HDR 1       /* core.py:151-153 (HDR and HDR-fixed-sigma) */
#define HPR_VARIANT_HPR 2       /* core.py:148-150 */

#define HPR_ABI_VERSION 1

typedef struct hpr_ctx hpr_ctx;

typedef struct hpr_dims {
  int64_t m;    /* rows of the stacked A = [A1; A2] (problem.py:75-82) */
  int64_t n;    /* columns */
  int64_t m1;   /* equality rows (first m1 rows) */
  int64_t nnz;  /* structural nonzeros of the canonical CSR (sparse.py:22-35) */
} hpr_dims;

/* Device buffers supplied by the caller.  Sizes in element counts. */
typedef struct hpr_buffers {
  /* A (m x n), canonical CSR: inputs */
  const int32_t *a_rp;   /* m+1 */
  const int32_t *a_ci;   /* nnz, strictly increasing within rows */
  const double *a_val;   /* nnz, the user's (unscaled) values */
  double *a_val_s;       /* nnz, scaled values (written by hpr_scale) */
  /* A^T (n x m), CSR (written by hpr_analyze / hpr_scale) */
  int32_t *at_rp;        /* n+1 */
  int32_t *at_ci;        /* nnz */
  int32_t *at_perm;      /* nnz: A^T entry k is A entry at_perm[k] */
  double *at_val;        /* nnz, unscaled */
  double *at_val_s;      /* nnz, scaled */
  /* original problem vectors: inputs */
  const double *b, *c, *lower, *upper;      /* m, n, n, n */
  /* scaled problem and scaling factors (written by hpr_scale) */
  double *b_s, *c_s, *lower_s, *upper_s;    /* m, n, n, n */
  double *row_scale, *col_scale;            /* m, n */
  /* iterate state w = (y, x), anchor, reflection w = 2 xb - x */
  double *y, *x, *anc_y, *anc_x, *w;        /* m, n, m, n, n */
  /* checkpoint half-step (scaled space) and scratch */
  double *yb, *xb, *zb, *dy, *wtmp;         /* m, n, n, m, n */
  /* candidate (termination-space) points, two slots */
  double *cand_y[2], *cand_x[2], *cand_z[2];
} hpr_buffers;

typedef struct hpr_scale_out {
  double b_factor, c_factor;   /* ScalingInfo.b_norm_factor / c_norm_factor */
  double bnorm_orig, cnorm_orig, bnorm_s, cnorm_s;  /* ||b||, ||c|| of both problems */
} hpr_scale_out;

typedef struct hpr_power_out {
  double value;      /* raw * (1 + 1e-3) (sparse.py:202) */
  double raw;
  int32_t iterations;
  int32_t converged;
} hpr_power_out;

/* Scalars of one checkpoint.  Sums of squares / dot products are reduced in a
 * fixed order (deterministic, bit-reproducible run to run). */
typedef struct hpr_ckpt_out {
  /* half step, scaled space */
  double bar_dx2;   /* ||xb - anchor_x||^2          (driver.py:273) */
  double bar_dy2;   /* ||yb - anchor_y||^2          (driver.py:274) */
  double dy2;       /* ||y - yb||^2                 (core.py:195,197) */
  double dx2;       /* ||x - xb||^2                 (core.py:197) */
  double sh2;       /* ||dx + sigma A^T dy||^2      (core.py:192-193) */
  double aty2;      /* ||A^T dy||^2                 (core.py:195) */
  /* KKT on the termination-space problem (driver.py:203-216) */
  double prim2;     /* ||Pi_D(b - A x)||^2 */
  double dual2;     /* ||c - A^T y - z||^2 */
  double r1sq, r2sq;
  double cx;        /* <c, x> */
  double by;        /* <b, y> */
  double lz, uz;    /* sum l_i z_i (z_i > 0, l_i finite), sum u_i z_i (z_i < 0, u_i finite) */
  int64_t n_lo, n_up, clamped;
  int64_t nonfinite_k;  /* first iteration k with a non-finite iterate, or -1 */
} hpr_ckpt_out;

int hpr_abi_version(void);
const char *hpr_last_error(void);

/* Bytes of the workspace the caller must allocate for these dims. */
int hpr_workspace_bytes(const hpr_dims *dims, size_t *bytes);

/* stream: a cudaStream_t (non-default) the context works on. */
int hpr_ctx_create(hpr_ctx **out, const hpr_dims *dims, int device, void *stream);
int hpr_ctx_destroy(hpr_ctx *ctx);

int hpr_bind(hpr_ctx *ctx, const hpr_buffers *bufs, void *workspace, size_t workspace_bytes);

/* Builds A^T (stable: rows ascending within each column, matching
 * csr_matrix(A.T)) and its permutation, and plans the SELL-32-sigma layout of A
 * and A^T used by every sparse product: slices of 32 rows (one per lane),
 * rows sorted by length inside windows of 256, entries column-major inside a
 * slice, rows longer than 1024 kept in CSR.  *layout_bytes receives the size
 * of the layout buffer the caller must allocate and pass to hpr_bind_layout. */
int hpr_analyze(hpr_ctx *ctx, size_t *layout_bytes);

/* Binds the layout buffer and fills it (column indices, CSR->slot map,
 * unscaled values).  Must follow hpr_analyze. */
int hpr_bind_layout(hpr_ctx *ctx, void *layout, size_t layout_bytes);

/* Ruiz(ruiz_iters) -> Pock-Chambolle(alpha=1) -> b/c normalisation on the
 * device.  With all three off the scaled problem is a copy (identity_scaling). */
int hpr_scale(hpr_ctx *ctx, int ruiz_iters, int pock_chambolle, int bc_normalize,
              hpr_scale_out *out);

/* Power method for lambda_1(A A^T) of the scaled A; HPR_EINVAL if the all-ones
 * and every basis start vector have A^T v = 0. */
int hpr_power(hpr_ctx *ctx, double tol, int max_iters, hpr_power_out *out);

/* y = x = anchors = 0; clears the non-finite marker. */
int hpr_state_reset(hpr_ctx *ctx);

/* `steps` iterations from inner counter t and total counter k with penalty
 * sigma and lam*sigma (the reference's single rounded product, core.py:170).
 * Replays a cached CUDA graph of `steps` iterations.  Asynchronous. */
int hpr_run_inner(hpr_ctx *ctx, int steps, int64_t t, int64_t k, double sigma,
                  double lamsig, int variant);

/* Half step + candidate (slot) + KKT + merit/sigma dot products.  One sync. */
int hpr_checkpoint(hpr_ctx *ctx, double sigma, double lamsig, int term_original, int slot,
                   hpr_ckpt_out *out);

/* anchor = current = (yb, xb) of the last checkpoint.  Asynchronous. */
int hpr_restart(hpr_ctx *ctx);

/* Candidate (slot) = (0, 0, clip(0, l, u)) on the termination problem and its KKT. */
int hpr_kkt_origin(hpr_ctx *ctx, int term_original, int slot, hpr_ckpt_out *out);

/* KKT residual terms of whatever the caller stored in candidate `slot`
 * (kkt_residual, driver.py:191-228, on the original or the scaled problem). */
int hpr_kkt(hpr_ctx *ctx, int term_original, int slot, hpr_ckpt_out *out);

/* Final solution: for the scaled termination space, unscale candidate `slot`
 * into slot `1 - slot` and clip; objectives of the solution on the original
 * problem are returned in out->cx / by / lz / uz / n_lo / n_up. */
int hpr_finalize(hpr_ctx *ctx, int term_original, int slot, hpr_ckpt_out *out);

/* Kernel launches issued by this context so far (graph nodes counted per replay). */
int hpr_launch_count(hpr_ctx *ctx, int64_t *count);

/* Statistics of the SELL layout (slices, slots incl. padding, long rows). */
typedef struct hpr_layout_info_t {
  int64_t slices_a, slices_at, slots_a, slots_at, long_rows_a, long_rows_at;
  int64_t cb_a, cb_at;   /* padded entries of the column-blocked layout (0: SELL engine) */
  int64_t split_a;       /* column blocks of A's split y-phase layout (0: not split) */
  int64_t stg_a, stg_at; /* staged-engine vector chunks of A / A^T (0: engine off) */
  int64_t rao_a, rao_at; /* 1: SELL rows in the row-affinity order (gathered vector > L2) */
  int64_t bounds_uniform; /* after hpr_scale: bit 0 every scaled lower bound equal, bit 1
                             every upper bound equal (passed as scalars, not streamed) */
  int64_t ts_a, ts_at;   /* blocks of the bulk-copy-streamed (TS) iteration engine (0: off) */
  int64_t ts_words_a, ts_words_at; /* the TS engine's column-index words (one per entry in
                             lane-affine / lane-uniform slices; 0: it reads the slot indices) */
} hpr_layout_info_t;
int hpr_layout_info(hpr_ctx *ctx, hpr_layout_info_t *info);

/* Plain sparse product on the bound problem's current (scaled) values:
 * y = A x (transpose = 0, x: n, y: m) or y = A^T x (transpose = 1, x: m,
 * y: n); each row summed left to right from 0.0 like scipy's csr_matvec.
 * Replaces SparseMatrix.apply / t_apply (sparse.py:102-108) for the exact
 * T1 = 0 path (exact.py:70-75, 94-103, 200-272); asynchronous on the
 * context's stream.  Requires hpr_analyze + hpr_bind_layout + hpr_scale. */
int hpr_spmv(hpr_ctx *ctx, int transpose, const double *x, double *y);

/* ------------------------------------------------------------------------
 * Exact T1 = 0 path (csrc/hpr_exact.cuh).  Replaces
 * the inner loop of solve_equality_exact (exact.py:125-129 ->
 * hpr_exact_iterate, exact.py:83-91) and its checkpoint half step
 * (exact_half_step, exact.py:70-80) for an equality-only problem (m1 == m)
 * bound with identity scaling (hpr_scale(ctx, 0, 0, 0)).  The dense solve
 * through the Cholesky factor L of AA* (solve_normal_equations,
 * exact.py:62-67) is two triangular products with the explicit inverse
 * factor: linv = L^{-1} (lower) and linv_t = L^{-T} (upper), both m x m
 * row-major device arrays the caller computes once per solve.
 * ------------------------------------------------------------------------ */
typedef struct hpr_exact_bufs {
  const double *linv;    /* m x m row-major, L^{-1} */
  const double *linv_t;  /* m x m row-major, L^{-T} */
  double *u;             /* n scratch: xb + sigma (zb - c) */
  double *rhs;           /* m scratch: (b - A u) / sigma */
  double *h;             /* m scratch: L^{-1} rhs */
} hpr_exact_bufs;
int hpr_exact_bind(hpr_ctx *ctx, const hpr_exact_bufs *bufs);
/* `steps` exact iterations from counters (t, k) at penalty sigma (one CUDA
 * graph replay per distinct `steps`); y, x advance in place; asynchronous. */
int hpr_exact_run(hpr_ctx *ctx, int steps, int64_t t, int64_t k, double sigma, int variant);
/* The half step at the current point: xb, zb -> xb/zb buffers and
 * cand_x/cand_z[slot], yb -> yb and cand_y[slot]; then hpr_kkt(ctx, 1, slot)
 * gives the residuals.  *nonfinite_k = first iteration with a non-finite
 * iterate since hpr_state_reset, or -1.  Synchronises once. */
int hpr_exact_half(hpr_ctx *ctx, double sigma, int slot, int64_t *nonfinite_k);
/* y = L^{-T} (L^{-1} rhs) (solve_normal_equations, exact.py:62-67) with the
 * inverse factors above; tmp: m scratch; asynchronous on `stream`. */
int hpr_trsolve(int m, const double *linv, const double *linv_t, const double *rhs, double *tmp,
                double *y, void *stream);

/* Device time (ms) of the last hpr_run_inner and of the last checkpoint,
 * measured with CUDA events on the context stream. */
int hpr_last_times(hpr_ctx *ctx, double *inner_ms, double *ckpt_ms);
/* Diagnostic (bench.py): `reps` back-to-back launches of the x-phase kernel
   (an interval's steady-state step: for HPR, x re-formed from w and not
   stored), then of the y-phase kernel, on the engines the layout selected; average
   microseconds per launch from CUDA events on the context's stream.  Runs
   iterations on the current state (the iterate is overwritten): call it after
   a solve, never inside one. */
int hpr_time_phases(hpr_ctx *ctx, int reps, double *x_us, double *y_us);
/* 1 when hpr_run_inner runs the resident small-LP loop (one cluster launch
   per interval, hpr_small.cuh) for this context's layout, else 0. */
int hpr_small_path(hpr_ctx *ctx);

/* ------------------------------------------------------------------------
 * Row-block partitioned mode (paper_2408_12179_b200/csrc/
 * hpr_rowblock.cuh).  Replaces the same reference steps as the single-context
 * calls above (driver.py:293-391) for an A split by rows across P ranks.
 *
 * Each rank is an ordinary hpr_ctx created for its row block: dims
 * (m_g, n, m1_g, nnz_g) with A_g = the block's rows (all n columns), bound
 * with buffers whose column-indexed arrays (c, lower, upper, *_s, col_scale,
 * x, anc_x, w, xb, zb, wtmp, cand_x, cand_z) hold npad doubles
 * (hpr_group_dims), then hpr_analyze + hpr_bind_layout as usual.  The group
 * then takes over: scale / power / run_inner / checkpoint / restart / finalize.
 * Columns are split into `chunks` chunks of nranks slices of cw columns; rank
 * g owns slice g of every chunk.  With NCCL and chunks > 1 the inner loop
 * overlaps chunk q's collectives with the partial SpMV of chunk q+1.
 *
 * Transports:
 *   nccl_id != NULL: NCCL, one local rank per process (nlocal = 1), rank0 =
 *     this process's rank; the id comes from hpr_nccl_unique_id on rank 0 and
 *     is broadcast by the caller (torch.distributed).  libnccl.so.2 is
 *     resolved with dlopen (the copy already loaded by PyTorch).
 *   nccl_id == NULL: local, all nranks ranks in this process on one device
 *     and one stream (nlocal = nranks, rank0 = 0); collectives are kernels.
 * ------------------------------------------------------------------------ */
typedef struct hpr_group hpr_group;

int hpr_nccl_available(void);
int hpr_nccl_unique_id(void *id, size_t bytes);          /* bytes >= 128 */

/* padded column length and per-rank row-block workspace (partials, reduced
 * owned entries, gathered scalars) for n columns over nranks ranks */
int hpr_group_dims(int64_t n, int nranks, int chunks, int64_t *npad, size_t *ws_bytes);

int hpr_group_create(hpr_group **out, int nlocal, hpr_ctx *const *ctxs, void *const *rb_ws,
                     const int64_t *row0, size_t rb_ws_bytes, int nranks, int rank0, int chunks,
                     const void *nccl_id, size_t id_bytes);
int hpr_group_destroy(hpr_group *g);
/* rank g owns columns q*nranks*cw + g*cw + [0, cw) for q < chunks */
int hpr_group_col_layout(hpr_group *g, int64_t *chunks, int64_t *cw, int64_t *npad);

/* scale_problem (scaling.py:72-125): Ruiz column maxima all-reduced (MAX),
 * Pock-Chambolle column sums all-reduced (SUM), norms summed over ranks. */
int hpr_group_scale(hpr_group *g, int ruiz_iters, int pock_chambolle, int bc_normalize,
                    hpr_scale_out *out);
/* power_method_lambda_max (sparse.py:165-203): A^T v reduce-scatter + all-gather. */
int hpr_group_power(hpr_group *g, double tol, int max_iters, hpr_power_out *out);
int hpr_group_state_reset(hpr_group *g);
/* run_inner (core.py:177-179): per iteration A_g^T y_g partial -> reduce-scatter
 * -> x-phase on the slice -> all-gather w -> local y-phase; one CUDA graph. */
int hpr_group_run_inner(hpr_group *g, int steps, int64_t t, int64_t k, double sigma,
                        double lamsig, int variant);
/* checkpoint: as hpr_checkpoint; sums are reduced per rank then across ranks in
 * rank order, so every rank receives identical scalars. */
int hpr_group_checkpoint(hpr_group *g, double sigma, double lamsig, int term_original,
                         int slot, hpr_ckpt_out *out);
int hpr_group_restart(hpr_group *g);
int hpr_group_kkt_origin(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out);
int hpr_group_kkt(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out);
/* final unscale + all-gather of x and z (every rank then holds full x, z and
 * its own rows of y) + objectives on the original problem */
int hpr_group_finalize(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out);
int hpr_group_last_times(hpr_group *g, double *inner_ms, double *ckpt_ms);
int hpr_group_launch_count(hpr_group *g, int64_t *count);
/* transport (1 = NCCL, 0 = local kernels), and -- from the NCCL communicator
 * itself when NCCL is used -- its rank count, this rank and the NCCL version */
int hpr_group_comm_info(hpr_group *g, int *transport, int *nranks, int *rank, int *version);

/* ------------------------------------------------------------------------
 * Batch of small LPs (BASELINE config C5; csrc/hpr_batch.cuh): one whole
 * restarted HPR solve per CTA -- scaling, power method, inner loop,
 * checkpoints, restarts, sigma updates and the report all on the device.
 * Replaces `solve` (driver.py:281-405) applied to each LP of the batch.
 * Every LP must fit one CTA's shared memory (hpr_batch_smem_bytes <= the
 * device's opt-in maximum, 227 KB on B200: e.g. m=500, n=1000, nnz=5000).
 * ------------------------------------------------------------------------ */
typedef struct hpr_batch_problem {
  int64_t count;
  int64_t total_rows, total_cols, total_nnz;
  int32_t max_m, max_n;
  int64_t max_nnz;
  const int64_t *row_off, *col_off, *nz_off;   /* count + 1, device */
  const int32_t *m1;                           /* count: equality rows of each LP */
  const int32_t *rp;      /* total_rows + count: LP i's m_i + 1 local row pointers at row_off[i] + i */
  const int32_t *ci;      /* total_nnz: local column ids, strictly increasing within a row */
  const double *val;      /* total_nnz */
  const double *b;        /* total_rows */
  const double *c, *lower, *upper;             /* total_cols */
  const double *obj_const;                     /* count */
  const int32_t *obj_neg;                      /* count: 1 = MAX problem (report negated) */
} hpr_batch_problem;

#define HPR_BATCH_DR 0
#define HPR_BATCH_HDR_FIXED 1
#define HPR_BATCH_HDR 2
#define HPR_BATCH_HPR 3

typedef struct hpr_batch_config {   /* SolverConfig (driver.py:50-68) */
  double tolerance, time_limit_seconds, alpha1, alpha2, alpha3, sigma0, power_tol;
  int64_t max_iterations;
  int32_t check_interval, variant, ruiz_iters, pock_chambolle, bc_normalize, power_max_iters;
  int32_t term_original;   /* termination_space == "original" */
  int32_t max_log;         /* restart records kept per LP */
} hpr_batch_config;

typedef struct hpr_restart_rec {    /* RestartEvent (driver.py:117-127) */
  int32_t outer_index, trigger;     /* 0 sufficient, 1 stalled, 2 long_loop */
  int64_t tau;
  double sigma_next, merit;
} hpr_restart_rec;

typedef struct hpr_batch_result {   /* SolveReport fields (driver.py:154-188) */
  int32_t status;                   /* 0 Optimal, 1 IterationLimit, 2 TimeLimit, 3 NumericalError */
  int32_t restarts;
  int64_t iterations;
  int32_t power_iterations, power_converged, dual_clamped, n_log, merit_negative, power_failed;
  double primal_objective, dual_objective;
  double kkt[9];   /* primal abs/rel, dual abs/rel, gap abs/rel, residual norm, pobj, dobj */
  double sigma_final, lambda_estimate, lambda_raw, b_factor, c_factor, device_seconds;
} hpr_batch_result;

int hpr_batch_smem_bytes(int32_t max_m, int32_t max_n, int64_t max_nnz, size_t *bytes);
int hpr_batch_workspace_bytes(const hpr_batch_problem *p, size_t *bytes);
/* Asynchronous on `stream`.  results[count]; log[count * max_log]; x, z
 * (total_cols) and y (total_rows) receive each LP's solution. */
int hpr_batch_solve(const hpr_batch_problem *p, const hpr_batch_config *cfg, void *workspace,
                    size_t ws_bytes, hpr_batch_result *results, hpr_restart_rec *log,
                    double *x, double *y, double *z, int device, void *stream);

/* ------------------------------------------------------------------------
 * MPS reader / writer (host code) with the semantics of
 * the reference's mps.py (read_document 60-154, document_to_problem 157-278,
 * write_mps 295-364): standard minimisation form, equality rows first, then
 * >= rows (L rows negated, RANGES split), OBJSENSE MAX negates c.
 * ------------------------------------------------------------------------ */
typedef struct hpr_mps_result {
  int64_t m1, m2, n;
  int64_t *eq_rp, *eq_ci;       /* m1 + 1, nnz: canonical CSR of the equality block */
  double *eq_val;
  int64_t *in_rp, *in_ci;       /* m2 + 1, nnz: the >= block */
  double *in_val;
  double *b_eq, *b_ineq, *c, *lower, *upper;
  double objective_constant;
  int32_t objective_negated;
  int32_t extra_objective_rows; /* N rows after the first (dropped; the caller warns) */
  char *row_names;              /* m1 + m2 NUL-terminated names, back to back */
  char *col_names;              /* n names */
  char *name;                   /* NAME section */
} hpr_mps_result;

/* HPR_EINVAL on a malformed file: hpr_mps_last_error() = "line N: message". */
int hpr_mps_parse(const char *text, size_t len, hpr_mps_result **out);
const char *hpr_mps_last_error(void);
int hpr_mps_free(hpr_mps_result *r);

typedef struct hpr_mps_problem {
  int64_t m1, m2, n;
  const int64_t *eq_rp, *eq_ci;
  const double *eq_val;
  const int64_t *in_rp, *in_ci;
  const double *in_val;
  const double *b_eq, *b_ineq, *c, *lower, *upper;
  double objective_constant;
  int32_t objective_negated;
  const char *row_names;        /* NULL: EQ<i> / GE<i> */
  const char *col_names;        /* NULL: X<j> */
} hpr_mps_problem;

/* *text is malloc'ed (release with hpr_mps_free_text). */
int hpr_mps_write(const hpr_mps_problem *p, const char *name, char **text, size_t *len);
int hpr_mps_free_text(char *text);

#ifdef __cplusplus
}
#endif
#endif /* HPRLP_B200_H */
