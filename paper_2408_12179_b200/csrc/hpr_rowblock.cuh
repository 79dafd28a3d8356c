// hpr_rowblock.cuh -- row-block partitioned HPR-LP across ranks.
//
// Included at the end of hpr_capi.cu (same translation unit: it reuses the
// context internals).  A group is P ranks; rank g owns a contiguous block R_g
// of the stacked rows of A (balanced by nonzeros), i.e. an ordinary hpr_ctx
// whose dims are (m_g, n, m1_g, nnz_g): A_g is m_g x n and its transpose A_g^T
// is n x m_g.  Everything row-indexed (y, b, anchors, row scale) is local.
// Column-indexed vectors are allocated at length npad on every rank; the
// columns are split into K chunks of P slices of cw columns and rank g owns
// slice g of every chunk (hpr_group_dims / hpr_group_col_layout).
//
// One inner iteration (core.py:168-172):
//   p_g   = A_g^T y_g                        SELL kernel, n partial outputs
//   aty   = reduce-scatter(sum_g p_g)        rank g receives its owned columns
//   x, w  = x-phase epilogue on owned cols   (EpiXIter)
//   w     = all-gather(w)                    every rank needs all of w
//   y_g   = y-phase on A_g w                 local SELL kernel (EpiYIter)
// i.e. the north star's all-reduce of the A^T y partials, split as RS + AG so
// the n-length elementwise work is done once, not P times.  With NCCL and K > 1
// the four steps run chunk by chunk: chunk q's reduce-scatter, epilogue and
// all-gather (on a second stream) overlap the partial SpMV of chunk q+1.
// Checkpoint sums (KKT, merit, sigma) are per-rank fixed-order partials, then
// all-gathered and summed in rank order, so every rank makes the same host
// decisions.
//
// Two transports behind one interface:
//   * NCCL (one rank per process, one GPU each; ncclReduceScatter /
//     ncclAllGather / ncclAllReduce captured in the inner-loop CUDA graph);
//     libnccl is resolved with dlopen at group creation (the copy PyTorch
//     already loaded), so the library itself has no link-time NCCL dependency.
//   * local (all P ranks in this process on ONE device and ONE stream): the
//     collectives are small kernels over the P ranks' buffers.  This runs the
//     partitioned algorithm bit-for-bit as P GPUs would except for the order of
//     the cross-rank sums (rank order here; NCCL's ring order there), and is how
//     the partitioned path is parity-tested on a single GPU.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace hpr {

constexpr int kMaxLocal = 8;

struct PtrSet {
  double *p[kMaxLocal];
};

// x-phase partial of A_g^T v (row-block mode): out[j] = s
#ifndef HPR_STORE_MINB
#define HPR_STORE_MINB 8   // the A_g^T partial: 64 registers, spill-free (C4 rank -0.7 %)
#endif
struct EpiStore {
  static constexpr int NQ = 0;
  static constexpr int kMinBlocks = HPR_STORE_MINB;
  double *out;
  const PowState *S;   // optional gate (power method)
  __device__ bool enter() { return S == nullptr || !S->done; }
  __device__ void prefetch(int) {}
  __device__ void finish(int j, double s, double *) { out[j] = s; }
};

// Column ownership: the padded column range is K chunks of CW = P*cw columns;
// rank g owns columns i*CW + g*cw + [0, cw) of every chunk i.  Owned entries
// are enumerated idx = i*cw + t; the reduce-scattered partials of rank g are
// stored in that order (xslice[idx]).  K = 1 is one contiguous slice per rank.
__device__ __forceinline__ long long owned_col(int idx, int gr, int cw, int CW) {
  const int i = idx / cw;
  return (long long)i * CW + (long long)gr * cw + (idx - i * cw);
}

// column epilogue over the owned columns of chunks [i0, i1): epi.finish(j, s[idx])
template <class Epi>
__global__ void __launch_bounds__(kThreads)
k_cols(int gr, int cw, int CW, int i0, int i1, int n, const double *__restrict__ s, Epi epi,
       double *part) {
  double acc[Epi::NQ > 0 ? Epi::NQ : 1];
#pragma unroll
  for (int q = 0; q < (Epi::NQ > 0 ? Epi::NQ : 1); ++q) acc[q] = 0.0;
  if (!epi.enter()) return;
  for (int idx = i0 * cw + blockIdx.x * kThreads + threadIdx.x; idx < i1 * cw;
       idx += gridDim.x * kThreads) {
    const long long j = owned_col(idx, gr, cw, CW);
    if (j < n) {
      epi.prefetch((int)j);
      epi.finish((int)j, s[idx], acc);
    }
  }
  if constexpr (Epi::NQ > 0) block_reduce_store<Epi::NQ>(acc, part, gridDim.x);
}

// sum of squares over the owned entries (owned columns of a, or a compact slice)
__global__ void __launch_bounds__(kThreads)
k_owned_sumsq(const double *a, int compact, int gr, int cw, int CW, int cnt, int n, double *part) {
  double acc[1] = {0.0};
  for (int idx = blockIdx.x * kThreads + threadIdx.x; idx < cnt; idx += gridDim.x * kThreads) {
    const long long j = owned_col(idx, gr, cw, CW);
    if (j < n) acc[0] = __dadd_rn(acc[0], sq(compact ? a[idx] : a[j]));
  }
  block_reduce_store<1>(acc, part, gridDim.x);
}

// owned entries of a compact slice into their positions of a full vector
__global__ void k_owned_scatter(const double *slice, double *vec, int gr, int cw, int CW, int cnt) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < cnt; idx += gridDim.x * blockDim.x)
    vec[owned_col(idx, gr, cw, CW)] = slice[idx];
}

// ---- local transport: all ranks' buffers on one device ----------------------
// out_g[i*cw + t] = sum_{r = 0..P-1} part_r[i*CW + g*cw + t]   (rank order)
__global__ void k_rs_local(PtrSet part, PtrSet out, int P, int K, int cw, int CW) {
  const long long per = (long long)K * cw, total = (long long)P * per;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(e / per), idx = (int)(e % per);
    const long long pos = owned_col(idx, g, cw, CW);
    double s = 0.0;
    for (int r = 0; r < P; ++r) s = __dadd_rn(s, part.p[r][pos]);
    out.p[g][idx] = s;
  }
}
// in-place all-gather: every rank's owned entries copied to the other ranks
__global__ void k_ag_local(PtrSet vec, int P, int K, int cw, int CW) {
  const long long per = (long long)K * cw, total = (long long)P * per;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(e / per), idx = (int)(e % per);
    const long long pos = owned_col(idx, g, cw, CW);
    const double v = vec.p[g][pos];
    for (int r = 0; r < P; ++r)
      if (r != g) vec.p[r][pos] = v;
  }
}
// all-reduce in place over n entries (op 0 = sum in rank order, 2 = max)
__global__ void k_ar_local(PtrSet v, int P, int n, int op) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double s = v.p[0][j];
    for (int r = 1; r < P; ++r) s = op == 2 ? fmax(s, v.p[r][j]) : __dadd_rn(s, v.p[r][j]);
    for (int r = 0; r < P; ++r) v.p[r][j] = s;
  }
}
// checkpoint scalars: res_r[q] = sum over ranks in rank order; slot nonfin = min
__global__ void k_scal_local(PtrSet res, int P, int nq, int nonfin) {
  const int q = threadIdx.x;
  if (q >= nq) return;
  double s = res.p[0][q];
  for (int r = 1; r < P; ++r) s = q == nonfin ? fmin(s, res.p[r][q]) : __dadd_rn(s, res.p[r][q]);
  for (int r = 0; r < P; ++r) res.p[r][q] = s;
}
// NCCL transport: gath = P x 64 all-gathered results -> res (rank order)
__global__ void k_scal_gathered(const double *gath, int P, int nq, int nonfin, double *res) {
  const int q = threadIdx.x;
  if (q >= nq) return;
  double s = gath[q];
  for (int r = 1; r < P; ++r) s = q == nonfin ? fmin(s, gath[r * 64 + q]) : __dadd_rn(s, gath[r * 64 + q]);
  res[q] = s;
}
// first non-finite k as a double (1e300 = none) so it rides the scalar reduction
__global__ void k_nonfin_to_result(const IterParams *P, double *slot) {
  *slot = P->nonfinite_k == ~0ULL ? 1e300 : (double)P->nonfinite_k;
}
// power-method start vector: basis vector e_fb (global row fb) or ones
__global__ void k_basis(double *v, int m, int local_row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    v[i] = i == local_row ? 1.0 : 0.0;
}

}  // namespace hpr

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  void *h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclReduceScatter) reduceScatter = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommCount) commCount = nullptr;          // optional (diagnostics)
  decltype(&ncclCommUserRank) commUserRank = nullptr;
  decltype(&ncclGetVersion) getVersion = nullptr;
  bool ok = false;
};

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // Fixed reduction order run to run at a given P: ring reduce-scatter with
    // the Simple protocol unless the caller pinned something else (NCCL reads
    // these when a communicator is created).
    setenv("NCCL_ALGO", "Ring", 0);
    setenv("NCCL_PROTO", "Simple", 0);
    // prefer the copy already in the process (PyTorch's), else the loader's
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.h = h;
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
      api.reduceScatter = (decltype(api.reduceScatter))dlsym(h, "ncclReduceScatter");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
      api.commCount = (decltype(api.commCount))dlsym(h, "ncclCommCount");
      api.commUserRank = (decltype(api.commUserRank))dlsym(h, "ncclCommUserRank");
      api.getVersion = (decltype(api.getVersion))dlsym(h, "ncclGetVersion");
      api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce &&
               api.reduceScatter && api.allGather && api.errStr;
    }
  });
  return api;
}

#define NK(call)                                                                           \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(HPR_ENCCL, std::string(#call) + ": " + nccl().errStr(r_));               \
  } while (0)

// per-rank buffers of the row-block mode (carved from the caller's rb workspace)
struct RbRank {
  hpr_ctx *c = nullptr;
  double *xpart = nullptr;   // npad: partial A_g^T v (entries >= n stay 0)
  double *xslice = nullptr;  // K * cw: reduce-scattered owned entries
  double *gath = nullptr;    // P * 64: all-gathered scalars (NCCL transport)
  int64_t row0 = 0;          // first global row
};

// chunk geometry: K chunks of P slices of cw columns (cw a multiple of A^T's
// SELL sorting window when K > 1, so a chunk is a whole number of windows)
void rb_dims(int64_t n, int P, int K, int64_t *cw, int64_t *npad) {
  int64_t w = (n + (int64_t)K * P - 1) / ((int64_t)K * P);
  const int win = sort_win(n);
  if (K > 1) w = (w + win - 1) / win * win;
  *cw = std::max<int64_t>(w, 1);
  *npad = *cw * P * K;
}

size_t rb_layout(int64_t n, int P, int K, size_t *o_xpart, size_t *o_xslice, size_t *o_gath) {
  int64_t cw, npad;
  rb_dims(n, P, K, &cw, &npad);
  size_t off = 0;
  *o_xpart = off;
  off = align_up(off + sizeof(double) * npad, 256);
  *o_xslice = off;
  off = align_up(off + sizeof(double) * cw * K, 256);
  *o_gath = off;
  off = align_up(off + sizeof(double) * 64 * P, 256);
  return off;
}

}  // namespace

struct hpr_group {
  int P = 1;          // ranks in the group
  int rank0 = 0;      // global rank of local rank 0
  int nlocal = 1;
  int64_t n = 0;
  int K = 1;                       // column chunks (overlap granularity)
  int64_t cw = 0, CW = 0, npad = 0;
  std::vector<RbRank> r;
  ncclComm_t comm = nullptr;
  bool use_nccl = false;
  cudaStream_t stream = nullptr;   // ctx[0]'s stream (local transport: shared)
  cudaStream_t comm_stream = nullptr;          // NCCL + chunk epilogues, K > 1
  std::vector<cudaEvent_t> ev_chunk;           // per chunk: partial SpMV done
  cudaEvent_t ev_comm = nullptr;               // comm stream joined back
  std::map<int, cudaGraphExec_t> inner_graphs;
  cudaGraphExec_t pow_graph = nullptr;
  bool inner_timed = false, ckpt_timed = false;

  bool single = false;             // one rank, no collectives on the column vectors
  int gr(int l) const { return rank0 + l; }    // global rank of local rank l
  int owned() const { return (int)(K * cw); }
};

namespace {

PtrSet ptrs(hpr_group *g, double *RbRank::*f) {
  PtrSet s{};
  for (int l = 0; l < g->nlocal; ++l) s.p[l] = g->r[l].*f;
  return s;
}

// sum of xpart over ranks -> xslice (owned entries) of each rank, chunks [i0, i1)
int g_reduce_scatter(hpr_group *g, cudaStream_t st = nullptr, int i0 = 0, int i1 = -1) {
  if (!st) st = g->stream;
  if (i1 < 0) i1 = g->K;
  if (g->single) return HPR_OK;            // one rank: xslice aliases xpart
  if (g->use_nccl) {
    for (int i = i0; i < i1; ++i)
      NK(nccl().reduceScatter(g->r[0].xpart + (size_t)i * g->CW, g->r[0].xslice + (size_t)i * g->cw,
                              (size_t)g->cw, ncclFloat64, ncclSum, g->comm, st));
    return HPR_OK;
  }
  if (g->P == 1) {
    CK(cudaMemcpyAsync(g->r[0].xslice, g->r[0].xpart, sizeof(double) * g->cw * g->K,
                       cudaMemcpyDeviceToDevice, st));
    return HPR_OK;
  }
  const long long total = (long long)g->P * g->owned();
  k_rs_local<<<grid_for(total), 256, 0, st>>>(ptrs(g, &RbRank::xpart), ptrs(g, &RbRank::xslice),
                                              g->P, g->K, (int)g->cw, (int)g->CW);
  CKL();
  g->r[0].c->launches += 1;
  return HPR_OK;
}

// in-place all-gather: every rank's full vector vec(l) receives the other
// ranks' owned entries (chunks [i0, i1))
template <class VecOf>
int g_all_gather(hpr_group *g, VecOf vec, cudaStream_t st = nullptr, int i0 = 0, int i1 = -1) {
  if (!st) st = g->stream;
  if (i1 < 0) i1 = g->K;
  if (g->single) return HPR_OK;            // one rank owns every column
  if (g->use_nccl) {
    double *v = vec(0);
    for (int i = i0; i < i1; ++i)
      NK(nccl().allGather(v + (size_t)i * g->CW + (size_t)g->gr(0) * g->cw, v + (size_t)i * g->CW,
                          (size_t)g->cw, ncclFloat64, g->comm, st));
    return HPR_OK;
  }
  if (g->P == 1) return HPR_OK;
  PtrSet pv{};
  for (int l = 0; l < g->nlocal; ++l) pv.p[l] = vec(l);
  const long long total = (long long)g->P * g->owned();
  k_ag_local<<<grid_for(total), 256, 0, st>>>(pv, g->P, g->K, (int)g->cw, (int)g->CW);
  CKL();
  g->r[0].c->launches += 1;
  return HPR_OK;
}

// in-place all-reduce of an n-vector (Ruiz column max / PC column sums)
template <class VecOf>
int g_all_reduce(hpr_group *g, VecOf vec, int64_t count, bool is_max) {
  if (g->P == 1 && !g->use_nccl) return HPR_OK;
  if (g->use_nccl) {
    NK(nccl().allReduce(vec(0), vec(0), (size_t)count, ncclFloat64, is_max ? ncclMax : ncclSum,
                        g->comm, g->r[0].c->stream));
    return HPR_OK;
  }
  PtrSet pv{};
  for (int l = 0; l < g->nlocal; ++l) pv.p[l] = vec(l);
  k_ar_local<<<grid_for(count), 256, 0, g->stream>>>(pv, g->P, (int)count, is_max ? 2 : 0);
  CKL();
  g->r[0].c->launches += 1;
  return HPR_OK;
}

// group sum of every rank's results[0..R_COUNT) (rank order), min for R_NONFIN
int g_scalars(hpr_group *g) {
  if (g->P == 1 && !g->use_nccl) return HPR_OK;
  if (g->use_nccl) {
    hpr_ctx *c = g->r[0].c;
    NK(nccl().allGather(c->results, g->r[0].gath, 64, ncclFloat64, g->comm, c->stream));
    k_scal_gathered<<<1, 64, 0, c->stream>>>(g->r[0].gath, g->P, R_COUNT, R_NONFIN, c->results);
    CKL();
    c->launches += 1;
    return HPR_OK;
  }
  PtrSet pr{};
  for (int l = 0; l < g->nlocal; ++l) pr.p[l] = g->r[l].c->results;
  k_scal_local<<<1, 64, 0, g->stream>>>(pr, g->P, R_COUNT, R_NONFIN);
  CKL();
  g->r[0].c->launches += 1;
  return HPR_OK;
}

int g_fetch(hpr_group *g) {
  // every rank holds the same reduced scalars; read local rank 0's
  return fetch_results(g->r[0].c);
}

// SELL launch of A_l^T with the store epilogue into xpart (over all n rows)
int g_at_partial(hpr_group *g, int l, bool scaled, const double *v, const PowState *gate) {
  hpr_ctx *c = g->r[l].c;
  EpiStore es{};
  es.out = g->r[l].xpart;
  es.S = gate;
  if (scaled && c->ts_at && c->ts_chunk_sl == 0)   // TS engine (iteration x-phase)
    return launch_ts(c, c->mat_at(true), c->ts_blk + c->ts_nb_a + 1, c->ts_nb_at, v, es);
  return launch_sell(c, c->mat_at(scaled), v, es, nullptr, nullptr);
}

// the partial of one column chunk: rows [q*CW, (q+1)*CW) of A_l^T (whole SELL
// windows); the long rows ride with chunk 0 so they precede every reduction
int g_at_partial_chunk(hpr_group *g, int l, const double *v, int q) {
  hpr_ctx *c = g->r[l].c;
  if (c->ts_at && c->ts_chunk_sl == g->CW / kSlice && q + 1 < (int)c->ts_at_off.size()) {
    // TS engine over chunk q's own blocks (global slice ids; long rows with chunk 0)
    SellMat M = c->mat_at(true);
    if (q > 0) M.nlong = 0;
    EpiStore es{};
    es.out = g->r[l].xpart;
    es.S = nullptr;
    const int o = c->ts_at_off[q], nq = c->ts_at_off[q + 1] - o - 1;
    return launch_ts(c, M, c->ts_blk + c->ts_nb_a + 1 + o, nq, v, es);
  }
  SellMat M = c->mat_at(true);
  const long long s0 = (long long)q * g->CW / kSlice;
  M.slice_ptr += s0;
  M.slice_row += s0 * kSlice;
  M.slice_len += s0 * kSlice;
  M.compact = 0;   // a compact slice's row is 32 s + lane in the unshifted numbering
  M.nslices = (int)std::max<long long>(0, std::min<long long>(g->CW / kSlice, M.nslices - s0));
  if (q > 0) M.nlong = 0;
  EpiStore es{};
  es.out = g->r[l].xpart;
  es.S = nullptr;
  return launch_sell(c, M, v, es, nullptr, nullptr);
}

template <class Epi>
int g_cols(hpr_group *g, int l, const Epi &epi, double *part, int *grid_out,
           cudaStream_t st = nullptr, int i0 = 0, int i1 = -1) {
  hpr_ctx *c = g->r[l].c;
  if (!st) st = c->stream;
  if (i1 < 0) i1 = g->K;
  const int cnt = (i1 - i0) * (int)g->cw;
  const int grid = std::max(1, std::min(grid_for(std::max(cnt, 1), kThreads), c->num_sms * 16));
  k_cols<Epi><<<grid, kThreads, 0, st>>>(g->gr(l), (int)g->cw, (int)g->CW, i0, i1, (int)g->n,
                                         g->r[l].xslice, epi, part);
  CKL();
  c->launches += 1;
  if (grid_out) *grid_out = grid;
  return HPR_OK;
}

int g_check(hpr_group *g) {
  if (!g) return fail(HPR_EINVAL, "null group");
  for (auto &rr : g->r) {
    int rc = check_ctx(rr.c, true, false);
    if (rc) return rc;
  }
  return HPR_OK;
}

int g_check_scaled(hpr_group *g) {
  int rc = g_check(g);
  if (rc) return rc;
  for (auto &rr : g->r)
    if (!rr.c->scaled) return fail(HPR_ESTATE, "hpr_group_scale has not been called");
  return HPR_OK;
}

// KKT terms of candidate `slot` on every rank: rows local, columns on the slice
int g_kkt(hpr_group *g, int term_original, int slot, std::vector<std::vector<RedSeg>> &segs) {
  for (int l = 0; l < g->nlocal; ++l) {
    hpr_ctx *c = g->r[l].c;
    int rc = g_at_partial(g, l, !term_original, c->B.cand_y[slot], nullptr);
    if (rc) return rc;
  }
  int rc = g_reduce_scatter(g);
  if (rc) return rc;
  for (int l = 0; l < g->nlocal; ++l) {
    hpr_ctx *c = g->r[l].c;
    const hpr_buffers &B = c->B;
    Parts P = parts_of(c);
    EpiKktRow er{};
    er.b = term_original ? B.b : B.b_s;
    er.cy = B.cand_y[slot];
    er.m1 = (int)c->d.m1;
    int ga = 0, gat = 0;
    rc = launch_sell(c, c->mat_a(!term_original), B.cand_x[slot], er, P.krow, &ga);
    if (rc) return rc;
    EpiKktCol ec{};
    ec.c = term_original ? B.c : B.c_s;
    ec.lo = term_original ? B.lower : B.lower_s;
    ec.up = term_original ? B.upper : B.upper_s;
    ec.cx = B.cand_x[slot];
    ec.cz = B.cand_z[slot];
    rc = g_cols(g, l, ec, P.kcol, &gat);
    if (rc) return rc;
    auto &sg = segs[l];
    sg.push_back({P.krow + 0 * ga, ga, R_PRIM2});
    sg.push_back({P.krow + 1 * ga, ga, R_BY});
    sg.push_back({P.krow + 2 * ga, ga, R_R1});
    const int outs[8] = {R_DUAL2, R_CX, R_LZ, R_UZ, R_NLO, R_NUP, R_CLAMP, R_R2};
    for (int q = 0; q < 8; ++q) sg.push_back({P.kcol + q * gat, gat, outs[q]});
  }
  return HPR_OK;
}

int g_reduce_all(hpr_group *g, std::vector<std::vector<RedSeg>> &segs, bool with_nonfin) {
  for (int l = 0; l < g->nlocal; ++l) {
    hpr_ctx *c = g->r[l].c;
    CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, c->stream));
    if (!segs[l].empty()) {
      int rc = reduce_final(c, segs[l]);
      if (rc) return rc;
    }
    if (with_nonfin) {
      k_nonfin_to_result<<<1, 1, 0, c->stream>>>(c->params, c->results + R_NONFIN);
      CKL();
      c->launches += 1;
    } else {
      k_fill<<<1, 32, 0, c->stream>>>(c->results + R_NONFIN, 1e300, 1);
      CKL();
      c->launches += 1;
    }
  }
  return g_scalars(g);
}

void g_fill_out(hpr_group *g, hpr_ckpt_out *o) {
  fill_out(g->r[0].c, o);
  const double nf = g->r[0].c->h_results[R_NONFIN];
  o->nonfinite_k = nf >= 1e299 ? -1 : (int64_t)nf;
}

int g_kkt_common(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out) {
  std::vector<std::vector<RedSeg>> segs(g->nlocal);
  int rc = g_kkt(g, term_original, slot, segs);
  if (rc) return rc;
  rc = g_reduce_all(g, segs, false);
  if (rc) return rc;
  rc = g_fetch(g);
  if (rc) return rc;
  g_fill_out(g, out);
  return HPR_OK;
}

}  // namespace

extern "C" {

int hpr_nccl_available(void) { return nccl().ok ? 1 : 0; }

int hpr_nccl_unique_id(void *id, size_t bytes) {
  if (!id || bytes < sizeof(ncclUniqueId)) return fail(HPR_EINVAL, "id buffer too small");
  if (!nccl().ok) return fail(HPR_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId u;
  NK(nccl().getUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return HPR_OK;
}

int hpr_group_dims(int64_t n, int nranks, int chunks, int64_t *npad, size_t *ws_bytes) {
  if (!npad || !ws_bytes || n < 1 || nranks < 1 || chunks < 1) return fail(HPR_EINVAL, "bad argument");
  int64_t cw;
  rb_dims(n, nranks, chunks, &cw, npad);
  size_t a, b, c;
  *ws_bytes = rb_layout(n, nranks, chunks, &a, &b, &c);
  return HPR_OK;
}

int hpr_group_create(hpr_group **out, int nlocal, hpr_ctx *const *ctxs, void *const *rb_ws,
                     const int64_t *row0, size_t rb_ws_bytes, int nranks, int rank0, int chunks,
                     const void *nccl_id, size_t id_bytes) {
  if (!out || !ctxs || !rb_ws || !row0 || nlocal < 1 || nranks < 1 || chunks < 1)
    return fail(HPR_EINVAL, "bad argument");
  if (nlocal > kMaxLocal) return fail(HPR_EINVAL, "too many local ranks");
  const bool use_nccl = nccl_id != nullptr;
  if (use_nccl && nlocal != 1) return fail(HPR_EINVAL, "NCCL transport: one local rank per process");
  if (!use_nccl && (nlocal != nranks || rank0 != 0))
    return fail(HPR_EINVAL, "local transport: all ranks must be local");
  const int64_t n = ctxs[0]->d.n;
  size_t o_xpart, o_xslice, o_gath;
  const size_t need = rb_layout(n, nranks, chunks, &o_xpart, &o_xslice, &o_gath);
  if (rb_ws_bytes < need) return fail(HPR_EINVAL, "row-block workspace too small");
  for (int l = 0; l < nlocal; ++l) {
    if (!ctxs[l] || !rb_ws[l]) return fail(HPR_EINVAL, "null context or workspace");
    if (ctxs[l]->d.n != n) return fail(HPR_EINVAL, "ranks disagree on n");
    if (!use_nccl && (ctxs[l]->stream != ctxs[0]->stream || ctxs[l]->device != ctxs[0]->device))
      return fail(HPR_EINVAL, "local transport: ranks must share one device and stream");
  }
  hpr_group *g = new hpr_group();
  g->P = nranks;
  g->rank0 = rank0;
  g->nlocal = nlocal;
  g->n = n;
  g->K = chunks;
  rb_dims(n, nranks, chunks, &g->cw, &g->npad);
  g->CW = g->cw * nranks;
  g->stream = ctxs[0]->stream;
  if (use_nccl && chunks > 1)   // the overlapped x-phase launches A^T chunk by chunk: TS plan per chunk
    for (int l = 0; l < nlocal; ++l) {
      ctxs[l]->ts_chunk_sl = (int)(g->CW / kSlice);
      cudaSetDevice(ctxs[l]->device);
      if (int rc = ts_plan(ctxs[l])) {
        delete g;
        return rc;
      }
    }
  g->use_nccl = use_nccl;
  {
    const char *force = getenv("HPR_RB_NCCL_P1");
    g->single = nranks == 1 && !(use_nccl && force && force[0] == '1');
  }
  for (int l = 0; l < nlocal; ++l) {
    RbRank rr;
    rr.c = ctxs[l];
    char *w = (char *)rb_ws[l];
    rr.xpart = (double *)(w + o_xpart);
    rr.xslice = (double *)(w + o_xslice);
    rr.gath = (double *)(w + o_gath);
    rr.row0 = row0[l];
    // one rank owns every column in order: the reduced slice IS the partial
    // (HPR_RB_NCCL_P1=1 keeps the NCCL calls at world size 1, for tests)
    const char *force = getenv("HPR_RB_NCCL_P1");
    if (nranks == 1 && !(use_nccl && force && force[0] == '1')) rr.xslice = rr.xpart;
    g->r.push_back(rr);
    // the partial's padding rows (n .. npad) are never written: keep them 0
    cudaMemsetAsync(rr.xpart, 0, sizeof(double) * g->npad, g->stream);
  }
  if (use_nccl && chunks > 1) {
    cudaSetDevice(ctxs[0]->device);
    cudaStreamCreateWithFlags(&g->comm_stream, cudaStreamNonBlocking);
    g->ev_chunk.resize(chunks);
    for (auto &e : g->ev_chunk) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_comm, cudaEventDisableTiming);
  }
  if (g->use_nccl) {
    if (!nccl().ok) {
      delete g;
      return fail(HPR_ENCCL, "libnccl.so.2 not loadable");
    }
    if (id_bytes < sizeof(ncclUniqueId)) {
      delete g;
      return fail(HPR_EINVAL, "bad NCCL id");
    }
    ncclUniqueId u;
    std::memcpy(&u, nccl_id, sizeof(u));
    cudaSetDevice(ctxs[0]->device);
    ncclResult_t r = nccl().commInitRank(&g->comm, nranks, u, rank0);
    if (r != ncclSuccess) {
      delete g;
      return fail(HPR_ENCCL, std::string("ncclCommInitRank: ") + nccl().errStr(r));
    }
  }
  *out = g;
  return HPR_OK;
}

int hpr_group_destroy(hpr_group *g) {
  if (!g) return HPR_OK;
  for (auto &kv : g->inner_graphs) cudaGraphExecDestroy(kv.second);
  if (g->pow_graph) cudaGraphExecDestroy(g->pow_graph);
  if (g->comm) nccl().commDestroy(g->comm);
  for (auto &e : g->ev_chunk) cudaEventDestroy(e);
  if (g->ev_comm) cudaEventDestroy(g->ev_comm);
  if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
  delete g;
  return HPR_OK;
}

int hpr_group_col_layout(hpr_group *g, int64_t *chunks, int64_t *cw, int64_t *npad) {
  if (!g || !chunks || !cw || !npad) return fail(HPR_EINVAL, "bad argument");
  *chunks = g->K;
  *cw = g->cw;
  *npad = g->npad;
  return HPR_OK;
}

// scale_problem (scaling.py:72-125) across the row blocks: row factors are
// local, column factors are reduced (max for Ruiz -- exact; sum for PC).
int hpr_group_scale(hpr_group *g, int ruiz_iters, int pock_chambolle, int bc_normalize,
                    hpr_scale_out *out) {
  int rc = g_check(g);
  if (rc) return rc;
  CK(cudaSetDevice(g->r[0].c->device));
  const int n = (int)g->n;
  auto dcv = [&](int l) { return g->r[l].c->dvec_n; };
  for (auto &rr : g->r) {
    hpr_ctx *c = rr.c;
    const hpr_buffers &B = c->B;
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(B.a_val_s, B.a_val, sizeof(double) * c->d.nnz, cudaMemcpyDeviceToDevice, s));
    k_fill<<<grid_for(c->d.m), 256, 0, s>>>(B.row_scale, 1.0, c->d.m);
    k_fill<<<grid_for(n), 256, 0, s>>>(B.col_scale, 1.0, n);
    CKL();
    c->launches += 2;
  }
  auto pass = [&](bool ruiz) -> int {
    for (auto &rr : g->r) {
      hpr_ctx *c = rr.c;
      const hpr_buffers &B = c->B;
      const int m = (int)c->d.m;
      if (ruiz) {
        k_row_maxabs<<<grid_for(m), 256, 0, c->stream>>>(B.a_rp, B.a_val_s, m, c->dvec_m);
        k_col_maxabs<<<grid_for(n), 256, 0, c->stream>>>(B.at_rp, B.at_perm, B.a_val_s, n, c->dvec_n);
      } else {
        k_row_abssum<<<grid_for(m), 256, 0, c->stream>>>(B.a_rp, B.a_val_s, m, c->dvec_m);
        k_col_abssum<<<grid_for(n), 256, 0, c->stream>>>(B.at_rp, B.at_perm, B.a_val_s, n, c->dvec_n);
      }
      CKL();
      c->launches += 2;
    }
    int rc2 = g_all_reduce(g, dcv, n, ruiz);
    if (rc2) return rc2;
    for (auto &rr : g->r) {
      hpr_ctx *c = rr.c;
      const hpr_buffers &B = c->B;
      const int m = (int)c->d.m;
      k_sqrt_div<<<grid_for(m), 256, 0, c->stream>>>(c->dvec_m, B.row_scale, m);
      k_sqrt_div<<<grid_for(n), 256, 0, c->stream>>>(c->dvec_n, B.col_scale, n);
      k_scale_vals<<<grid_for((int64_t)m * 32), 256, 0, c->stream>>>(B.a_rp, B.a_ci, B.a_val_s,
                                                                     c->dvec_m, c->dvec_n, m);
      CKL();
      c->launches += 3;
    }
    return HPR_OK;
  };
  for (int it = 0; it < ruiz_iters; ++it) {
    rc = pass(true);
    if (rc) return rc;
  }
  if (pock_chambolle) {
    rc = pass(false);
    if (rc) return rc;
  }
  for (auto &rr : g->r) {
    hpr_ctx *c = rr.c;
    const hpr_buffers &B = c->B;
    const int m = (int)c->d.m;
    k_scale_vecs<<<grid_for(std::max(m, n)), 256, 0, c->stream>>>(
        B.b, B.row_scale, B.b_s, m, B.c, B.lower, B.upper, B.col_scale, B.c_s, B.lower_s,
        B.upper_s, n);
    CKL();
    c->launches += 1;
  }
  // sum of squares of a row vector (local rows) and of a column vector (own slice)
  auto sumsq_pair = [&](bool orig, int slot_b, int slot_c, std::vector<std::vector<RedSeg>> &segs,
                        int bank) -> int {
    for (int l = 0; l < g->nlocal; ++l) {
      hpr_ctx *c = g->r[l].c;
      const hpr_buffers &B = c->B;
      Parts P = parts_of(c);
      const int m = (int)c->d.m;
      const int nb0 = sumsq_blocks(m), nb1 = sumsq_blocks(g->owned());
      double *pb = P.misc + (2 * bank) * kSumsqBlocks, *pc = P.misc + (2 * bank + 1) * kSumsqBlocks;
      k_sumsq<<<nb0, kThreads, 0, c->stream>>>(orig ? B.b : B.b_s, m, pb);
      k_owned_sumsq<<<nb1, kThreads, 0, c->stream>>>(orig ? B.c : B.c_s, 0, g->gr(l), (int)g->cw,
                                                     (int)g->CW, g->owned(), n, pc);
      CKL();
      c->launches += 2;
      segs[l].push_back({pb, nb0, slot_b});
      segs[l].push_back({pc, nb1, slot_c});
    }
    return HPR_OK;
  };
  if (bc_normalize) {
    std::vector<std::vector<RedSeg>> segs(g->nlocal);
    rc = sumsq_pair(false, R_SUMSQ0, R_SUMSQ1, segs, 0);
    if (rc) return rc;
    rc = g_reduce_all(g, segs, false);
    if (rc) return rc;
    for (auto &rr : g->r) {
      hpr_ctx *c = rr.c;
      const hpr_buffers &B = c->B;
      k_factors<<<1, 32, 0, c->stream>>>(c->results + R_SUMSQ0, c->fac);
      k_bc_normalize<<<grid_for(std::max((int)c->d.m, n)), 256, 0, c->stream>>>(
          B.b_s, (int)c->d.m, B.c_s, B.lower_s, B.upper_s, n, c->fac);
      CKL();
      c->launches += 2;
    }
  } else {
    for (auto &rr : g->r) {
      k_fill<<<1, 32, 0, rr.c->stream>>>(rr.c->fac, 1.0, 2);
      CKL();
    }
  }
  for (auto &rr : g->r) {
    hpr_ctx *c = rr.c;
    const hpr_buffers &B = c->B;
    const long long nnz = c->d.nnz;
    if (nnz > 0) {
      k_gather_vals<<<grid_for(nnz), 256, 0, c->stream>>>(B.at_perm, B.a_val_s, B.at_val_s, nnz);
      k_sell_scatter<<<grid_for(nnz), 256, 0, c->stream>>>(c->sa.pos, B.a_val_s, c->sa.val_s, nnz);
      k_sell_scatter<<<grid_for(nnz), 256, 0, c->stream>>>(c->sat.pos, B.at_val_s, c->sat.val_s, nnz);
      if (c->sp.on)
        k_sell_scatter<<<grid_for(nnz), 256, 0, c->stream>>>(c->sp.S.pos, B.a_val_s, c->sp.S.val_s, nnz);
      CKL();
      c->launches += 3;
    }
  }
  std::vector<std::vector<RedSeg>> segs(g->nlocal);
  rc = sumsq_pair(true, R_SUMSQ0, R_SUMSQ1, segs, 0);
  if (rc) return rc;
  rc = sumsq_pair(false, R_SUMSQ2, R_SUMSQ3, segs, 1);
  if (rc) return rc;
  rc = g_reduce_all(g, segs, false);
  if (rc) return rc;
  double fac[2];
  CK(cudaMemcpyAsync(fac, g->r[0].c->fac, sizeof(fac), cudaMemcpyDeviceToHost, g->r[0].c->stream));
  rc = g_fetch(g);
  if (rc) return rc;
  const double *h = g->r[0].c->h_results;
  if (out) {
    out->b_factor = fac[0];
    out->c_factor = fac[1];
    out->bnorm_orig = std::sqrt(h[R_SUMSQ0]);
    out->cnorm_orig = std::sqrt(h[R_SUMSQ1]);
    out->bnorm_s = std::sqrt(h[R_SUMSQ2]);
    out->cnorm_s = std::sqrt(h[R_SUMSQ3]);
  }
  for (auto &rr : g->r) rr.c->scaled = true;
  for (auto &kv : g->inner_graphs) cudaGraphExecDestroy(kv.second);
  g->inner_graphs.clear();
  return HPR_OK;
}

// power_method_lambda_max (sparse.py:165-203) over the row blocks.
int hpr_group_power(hpr_group *g, double tol, int max_iters, hpr_power_out *out) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  if (!out) return fail(HPR_EINVAL, "null out");
  CK(cudaSetDevice(g->r[0].c->device));
  int64_t m_total = 0, nnz_total = 0;
  for (auto &rr : g->r) {
    m_total += rr.c->d.m;
    nnz_total += rr.c->d.nnz;
  }
  if (g->use_nccl) {
    // global row count / nnz: one tiny all-reduce through the scalar path
    hpr_ctx *c = g->r[0].c;
    double h[2] = {(double)m_total, (double)nnz_total};
    CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, c->stream));
    CK(cudaMemcpyAsync(c->results, h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
    k_fill<<<1, 32, 0, c->stream>>>(c->results + R_NONFIN, 1e300, 1);
    rc = g_scalars(g);
    if (rc) return rc;
    rc = g_fetch(g);
    if (rc) return rc;
    m_total = (int64_t)c->h_results[0];
    nnz_total = (int64_t)c->h_results[1];
  }
  if (nnz_total == 0) return fail(HPR_EINVAL, "matrix must be non-zero");
  PowState st{};
  st.tol = tol;
  st.max_iters = max_iters;
  auto vbuf = [&](int l) { return g->r[l].c->B.yb; };
  auto ubuf = [&](int l) { return g->r[l].c->B.wtmp; };
  auto wbuf = [&](int l) { return g->r[l].c->B.dy; };
  // start vector: all ones, then basis vectors e_0, e_1, ... while A^T v == 0
  bool found = false;
  int64_t fb_found = -2;
  for (int64_t fb = -1; fb < m_total && !found; ++fb) {
    std::vector<std::vector<RedSeg>> segs(g->nlocal);
    for (int l = 0; l < g->nlocal; ++l) {
      hpr_ctx *c = g->r[l].c;
      const int m = (int)c->d.m;
      if (fb < 0) {
        k_fill<<<grid_for(m), 256, 0, c->stream>>>(vbuf(l), 1.0, m);
      } else {
        const int64_t lr = fb - g->r[l].row0;
        k_basis<<<grid_for(m), 256, 0, c->stream>>>(vbuf(l), m, (lr >= 0 && lr < m) ? (int)lr : -1);
      }
      CKL();
      c->launches += 1;
      rc = g_at_partial(g, l, true, vbuf(l), nullptr);
      if (rc) return rc;
    }
    rc = g_reduce_scatter(g);
    if (rc) return rc;
    for (int l = 0; l < g->nlocal; ++l) {
      hpr_ctx *c = g->r[l].c;
      Parts P = parts_of(c);
      const int nb = sumsq_blocks(g->owned());
      k_owned_sumsq<<<nb, kThreads, 0, c->stream>>>(g->r[l].xslice, 1, g->gr(l), (int)g->cw,
                                                    (int)g->CW, g->owned(), (int)g->n, P.powt);
      CKL();
      c->launches += 1;
      segs[l].push_back({P.powt, nb, R_POW_U2});
    }
    rc = g_reduce_all(g, segs, false);
    if (rc) return rc;
    rc = g_fetch(g);
    if (rc) return rc;
    if (std::sqrt(g->r[0].c->h_results[R_POW_U2]) > 0.0) {
      found = true;
      fb_found = fb;
    }
  }
  if (!found) return fail(HPR_EINVAL, "A^T v = 0 for every start vector");
  if (fb_found == -1) {
    const double inv = 1.0 / std::sqrt((double)m_total);
    for (int l = 0; l < g->nlocal; ++l) {
      hpr_ctx *c = g->r[l].c;
      k_fill<<<grid_for(c->d.m), 256, 0, c->stream>>>(vbuf(l), inv, c->d.m);
      CKL();
      c->launches += 1;
    }
  }
  for (auto &rr : g->r)
    CK(cudaMemcpyAsync(rr.c->pow, &st, sizeof(st), cudaMemcpyHostToDevice, rr.c->stream));
  if (max_iters <= 0) {
    out->value = out->raw = 0.0;
    out->iterations = out->converged = 0;
    return HPR_OK;
  }
  if (!g->pow_graph) {
    cudaGraph_t gr;
    std::vector<long long> before;
    for (auto &rr : g->r) before.push_back(rr.c->launches);
    CK(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kPowBatch && !rc; ++i) {
      std::vector<std::vector<RedSeg>> segs(g->nlocal);
      // u = A^T v: partial -> reduce-scatter -> all-gather
      for (int l = 0; l < g->nlocal && !rc; ++l) rc = g_at_partial(g, l, true, vbuf(l), g->r[l].c->pow);
      if (!rc) rc = g_reduce_scatter(g);
      for (int l = 0; l < g->nlocal && !rc; ++l) {
        hpr_ctx *c = g->r[l].c;
        k_owned_scatter<<<grid_for(g->owned()), 256, 0, c->stream>>>(
            g->r[l].xslice, ubuf(l), g->gr(l), (int)g->cw, (int)g->CW, g->owned());
        c->launches += 1;
      }
      if (!rc) rc = g_all_gather(g, ubuf);
      // w = A_g u, local sums v.w and w.w
      for (int l = 0; l < g->nlocal && !rc; ++l) {
        hpr_ctx *c = g->r[l].c;
        Parts P = parts_of(c);
        EpiPowA ea{};
        ea.v = vbuf(l);
        ea.wv = wbuf(l);
        ea.S = c->pow;
        int ga = 0;
        rc = launch_sell(c, c->mat_a(true), ubuf(l), ea, P.powa, &ga);
        segs[l].push_back({P.powa, ga, R_POW_VW});
        segs[l].push_back({P.powa + ga, ga, R_POW_WW});
      }
      if (!rc) rc = g_reduce_all(g, segs, false);
      for (int l = 0; l < g->nlocal && !rc; ++l) {
        hpr_ctx *c = g->r[l].c;
        k_pow_step<<<1, kThreads, 0, c->stream>>>(c->results + R_POW_VW, 1, c->pow);
        k_pow_norm<<<grid_for(c->d.m), 256, 0, c->stream>>>(wbuf(l), vbuf(l), (int)c->d.m, c->pow);
        k_pow_norm_done<<<1, 1, 0, c->stream>>>(c->pow);
        c->launches += 3;
      }
    }
    cudaError_t e = cudaStreamEndCapture(g->stream, &gr);
    if (rc) {
      if (e == cudaSuccess) cudaGraphDestroy(gr);
      return rc;
    }
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("pow capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&g->pow_graph, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("pow instantiate: ") + cudaGetErrorString(e));
    for (int l = 0; l < g->nlocal; ++l) g->r[l].c->launches = before[l];
  }
  hpr_ctx *c0 = g->r[0].c;
  for (;;) {
    CK(cudaGraphLaunch(g->pow_graph, g->stream));
    c0->launches += (long long)kPowBatch * (6 * g->nlocal + 1);
    CK(cudaMemcpyAsync(c0->h_pow, c0->pow, sizeof(PowState), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    if (c0->h_pow->done) break;
  }
  out->raw = c0->h_pow->lam;
  out->value = c0->h_pow->lam * (1.0 + 1e-3);
  out->iterations = c0->h_pow->iters;
  out->converged = c0->h_pow->converged;
  return HPR_OK;
}

int hpr_group_state_reset(hpr_group *g) {
  int rc = g_check(g);
  if (rc) return rc;
  for (auto &rr : g->r) {
    rc = hpr_state_reset(rr.c);
    if (rc) return rc;
  }
  return HPR_OK;
}

// run_inner (core.py:177-179) over the row blocks, one CUDA graph per `steps`.
int hpr_group_run_inner(hpr_group *g, int steps, int64_t t, int64_t k, double sigma,
                        double lamsig, int variant) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  if (steps <= 0) return HPR_OK;
  if (variant < 0 || variant > 2) return fail(HPR_EINVAL, "bad variant");
  CK(cudaSetDevice(g->r[0].c->device));
  auto it = g->inner_graphs.find(steps);
  if (it == g->inner_graphs.end()) {
    std::vector<long long> before;
    for (auto &rr : g->r) before.push_back(rr.c->launches);
    cudaGraph_t gr;
    CK(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
    auto wvec = [&](int l) { return g->r[l].c->B.w; };
    auto xepi = [&](int l, int i) {
      const hpr_buffers &B = g->r[l].c->B;
      EpiXIter ex{};
      ex.c = B.c_s;
      ex.lo = B.lower_s;
      ex.up = B.upper_s;
      ex.anc = B.anc_x;
      ex.x = B.x;
      ex.w = B.w;
      ex.P = g->r[l].c->params;
      ex.step = i;
      return ex;
    };
    const bool overlap = g->use_nccl && g->K > 1 && g->comm_stream;
    for (int i = 0; i < steps && !rc; ++i) {
      if (overlap) {
        // chunk by chunk: the partial A_g^T y of chunk q is reduce-scattered,
        // finished (x-phase epilogue) and all-gathered on the comm stream while
        // the partial of chunk q+1 is computed on the main stream
        hpr_ctx *c = g->r[0].c;
        for (int q = 0; q < g->K && !rc; ++q) {
          rc = g_at_partial_chunk(g, 0, c->B.y, q);
          if (rc) break;
          CK(cudaEventRecord(g->ev_chunk[q], c->stream));
          CK(cudaStreamWaitEvent(g->comm_stream, g->ev_chunk[q], 0));
          rc = g_reduce_scatter(g, g->comm_stream, q, q + 1);
          if (!rc) rc = g_cols(g, 0, xepi(0, i), nullptr, nullptr, g->comm_stream, q, q + 1);
          if (!rc) rc = g_all_gather(g, wvec, g->comm_stream, q, q + 1);
        }
        if (rc) break;
        CK(cudaEventRecord(g->ev_comm, g->comm_stream));
        CK(cudaStreamWaitEvent(c->stream, g->ev_comm, 0));
      } else {
        for (int l = 0; l < g->nlocal && !rc; ++l) rc = g_at_partial(g, l, true, g->r[l].c->B.y, nullptr);
        if (!rc) rc = g_reduce_scatter(g);
        for (int l = 0; l < g->nlocal && !rc; ++l) rc = g_cols(g, l, xepi(l, i), nullptr, nullptr);
        if (!rc) rc = g_all_gather(g, wvec);
      }
      for (int l = 0; l < g->nlocal && !rc; ++l) {
        hpr_ctx *c = g->r[l].c;
        const hpr_buffers &B = c->B;
        EpiYIter ey{};
        ey.b = B.b_s;
        ey.anc = B.anc_y;
        ey.y = B.y;
        ey.P = c->params;
        ey.m1 = (int)c->d.m1;
        ey.step = i;
        rc = launch_a_iter(c, B.w, ey, false);
      }
    }
    cudaError_t e = cudaStreamEndCapture(g->stream, &gr);
    if (rc) {
      if (e == cudaSuccess) cudaGraphDestroy(gr);
      return rc;
    }
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exe;
    e = cudaGraphInstantiate(&exe, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    for (int l = 0; l < g->nlocal; ++l) g->r[l].c->launches = before[l];
    it = g->inner_graphs.emplace(steps, exe).first;
  }
  for (auto &rr : g->r) {
    k_set_params<<<1, 1, 0, rr.c->stream>>>(rr.c->params, sigma, lamsig, (long long)t, (long long)k,
                                            variant);
    CKL();
  }
  hpr_ctx *c0 = g->r[0].c;
  CK(cudaEventRecord(c0->ev0, g->stream));
  CK(cudaGraphLaunch(it->second, g->stream));
  CK(cudaEventRecord(c0->ev1, g->stream));
  g->inner_timed = true;
  c0->inner_timed = true;
  // per step: nlocal x (A^T partial + slice epilogue + y phase) + the collectives
  const int coll = (g->P == 1 || g->use_nccl) ? 0 : 2;
  long long split_extra = 0;   // column-split y-phase: NB launches instead of one
  for (int l = 0; l < g->nlocal; ++l) split_extra += g->r[l].c->sp.on ? g->r[l].c->sp.NB - 1 : 0;
  c0->launches += g->nlocal + (long long)steps * (3 * g->nlocal + coll + split_extra);
  return HPR_OK;
}

// checkpoint (driver.py:329-339 + core.py:118-129, 182-218) over the row blocks
int hpr_group_checkpoint(hpr_group *g, double sigma, double lamsig, int term_original, int slot,
                         hpr_ckpt_out *out) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(g->r[0].c->device));
  hpr_ctx *c0 = g->r[0].c;
  CK(cudaEventRecord(c0->ev2, g->stream));
  std::vector<std::vector<RedSeg>> segs(g->nlocal);
  // half step, x part: A^T y partial -> RS -> slice epilogue
  for (int l = 0; l < g->nlocal && !rc; ++l) rc = g_at_partial(g, l, true, g->r[l].c->B.y, nullptr);
  if (!rc) rc = g_reduce_scatter(g);
  for (int l = 0; l < g->nlocal && !rc; ++l) {
    hpr_ctx *c = g->r[l].c;
    const hpr_buffers &B = c->B;
    Parts P = parts_of(c);
    CandCtx cc{term_original, c->fac, B.row_scale, B.col_scale, B.lower, B.upper};
    EpiXHalf ex{};
    ex.x = B.x;
    ex.c = B.c_s;
    ex.lo = B.lower_s;
    ex.up = B.upper_s;
    ex.anc = B.anc_x;
    ex.xb_out = B.xb;
    ex.zb_out = B.zb;
    ex.wtmp = B.wtmp;
    ex.cx_out = B.cand_x[slot];
    ex.cz_out = B.cand_z[slot];
    ex.cc = cc;
    ex.sigma = sigma;
    int gx = 0;
    rc = g_cols(g, l, ex, P.xhalf, &gx);
    segs[l].push_back({P.xhalf, gx, R_BAR_DX2});
    segs[l].push_back({P.xhalf + gx, gx, R_DX2});
  }
  if (rc) return rc;
  // the y phase and the row KKT terms gather wtmp and cand_x over all columns
  rc = g_all_gather(g, [&](int l) { return g->r[l].c->B.wtmp; });
  if (!rc) rc = g_all_gather(g, [&](int l) { return g->r[l].c->B.cand_x[slot]; });
  for (int l = 0; l < g->nlocal && !rc; ++l) {
    hpr_ctx *c = g->r[l].c;
    const hpr_buffers &B = c->B;
    Parts P = parts_of(c);
    CandCtx cc{term_original, c->fac, B.row_scale, B.col_scale, B.lower, B.upper};
    EpiYHalf ey{};
    ey.y = B.y;
    ey.b = B.b_s;
    ey.anc = B.anc_y;
    ey.yb_out = B.yb;
    ey.dy_out = B.dy;
    ey.cy_out = B.cand_y[slot];
    ey.cc = cc;
    ey.lamsig = lamsig;
    ey.m1 = (int)c->d.m1;
    int gy = 0;
    rc = launch_sell(c, c->mat_a(true), B.wtmp, ey, P.yhalf, &gy);
    segs[l].push_back({P.yhalf, gy, R_DY2});
    segs[l].push_back({P.yhalf + gy, gy, R_BAR_DY2});
  }
  // merit: A^T dy partial -> RS -> slice epilogue
  for (int l = 0; l < g->nlocal && !rc; ++l) rc = g_at_partial(g, l, true, g->r[l].c->B.dy, nullptr);
  if (!rc) rc = g_reduce_scatter(g);
  for (int l = 0; l < g->nlocal && !rc; ++l) {
    hpr_ctx *c = g->r[l].c;
    Parts P = parts_of(c);
    EpiMeritCol em{};
    em.x = c->B.x;
    em.xb = c->B.xb;
    em.sigma = sigma;
    int gm = 0;
    rc = g_cols(g, l, em, P.merit, &gm);
    segs[l].push_back({P.merit, gm, R_SH2});
    segs[l].push_back({P.merit + gm, gm, R_ATY2});
  }
  if (!rc) rc = g_kkt(g, term_original, slot, segs);
  if (!rc) rc = g_reduce_all(g, segs, true);
  if (rc) return rc;
  CK(cudaEventRecord(c0->ev3, g->stream));
  rc = g_fetch(g);
  if (rc) return rc;
  c0->ckpt_timed = true;
  g->ckpt_timed = true;
  g_fill_out(g, out);
  return HPR_OK;
}

int hpr_group_restart(hpr_group *g) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  for (auto &rr : g->r) {
    rc = hpr_restart(rr.c);
    if (rc) return rc;
  }
  return HPR_OK;
}

int hpr_group_kkt_origin(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  for (auto &rr : g->r) {
    hpr_ctx *c = rr.c;
    const hpr_buffers &B = c->B;
    const int m = (int)c->d.m, n = (int)c->d.n;
    k_origin_cand<<<grid_for(std::max(m, n)), 256, 0, c->stream>>>(
        B.cand_y[slot], m, B.cand_z[slot], B.cand_x[slot], term_original ? B.lower : B.lower_s,
        term_original ? B.upper : B.upper_s, n);
    CKL();
    c->launches += 1;
  }
  return g_kkt_common(g, term_original, slot, out);
}

int hpr_group_kkt(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  return g_kkt_common(g, term_original, slot, out);
}

// final unscale (driver.py:382-386) + all-gather of x and z + objectives
int hpr_group_finalize(hpr_group *g, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = g_check_scaled(g);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  int fs = slot;
  if (!term_original) {
    fs = 1 - slot;
    for (auto &rr : g->r) {
      hpr_ctx *c = rr.c;
      const hpr_buffers &B = c->B;
      const int m = (int)c->d.m, n = (int)c->d.n;
      k_unscale<<<grid_for(std::max(m, n)), 256, 0, c->stream>>>(
          B.cand_y[slot], B.cand_z[slot], B.cand_x[slot], B.cand_y[fs], B.cand_z[fs],
          B.cand_x[fs], B.row_scale, B.col_scale, c->fac, B.lower, B.upper, m, n);
      CKL();
      c->launches += 1;
    }
  }
  // x and z are valid on each rank's slice only: gather them
  rc = g_all_gather(g, [&](int l) { return g->r[l].c->B.cand_x[fs]; });
  if (!rc) rc = g_all_gather(g, [&](int l) { return g->r[l].c->B.cand_z[fs]; });
  if (rc) return rc;
  return g_kkt_common(g, 1, fs, out);
}

int hpr_group_last_times(hpr_group *g, double *inner_ms, double *ckpt_ms) {
  if (!g) return fail(HPR_EINVAL, "null group");
  return hpr_last_times(g->r[0].c, inner_ms, ckpt_ms);
}

int hpr_group_comm_info(hpr_group *g, int *transport, int *nranks, int *rank, int *version) {
  if (!g || !transport || !nranks || !rank || !version) return fail(HPR_EINVAL, "null argument");
  *transport = g->use_nccl ? 1 : 0;
  *nranks = g->P;
  *rank = g->rank0;
  *version = 0;
  if (g->use_nccl && g->comm) {
    NcclApi &api = nccl();
    if (api.commCount) NK(api.commCount(g->comm, nranks));
    if (api.commUserRank) NK(api.commUserRank(g->comm, rank));
    if (api.getVersion) NK(api.getVersion(version));
  }
  return HPR_OK;
}

int hpr_group_launch_count(hpr_group *g, int64_t *count) {
  if (!g || !count) return fail(HPR_EINVAL, "null argument");
  int64_t s = 0;
  for (auto &rr : g->r) s += rr.c->launches;
  *count = s;
  return HPR_OK;
}

}  // extern "C"
