// hpr_capi.cu -- C ABI (include/hprlp_b200.h) over the sm_100a kernels.
//
// Host-side orchestration only: workspace carve-up, the transpose/tiling
// analysis, the scaling and power-method passes, CUDA-graph capture of the
// inner loop, the checkpoint sequence and its single device->host readback.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/hprlp_b200.h"
#include "hpr_kernels.cuh"

using namespace hpr;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(HPR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

#define CKL()                                                                              \
  do {                                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      return fail(HPR_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_));     \
  } while (0)

constexpr int kBucket = 2048;   // tile nonzero bucket
constexpr int kLongLen = 1024;  // rows longer than this get their own tile
constexpr int kCap = kBucket + kLongLen;
constexpr int kPowBatch = 8;    // power steps per graph replay

// result slots of the final reduction (see hpr_ckpt_out)
enum {
  R_BAR_DX2, R_DX2, R_DY2, R_BAR_DY2, R_PRIM2, R_BY, R_R1, R_DUAL2, R_CX, R_LZ, R_UZ, R_NLO,
  R_NUP, R_CLAMP, R_R2, R_SH2, R_ATY2, R_SUMSQ0, R_SUMSQ1, R_SUMSQ2, R_SUMSQ3, R_POW_U2, R_COUNT
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int64_t tile_bound(int64_t nrows, int64_t nnz) {
  int64_t b = nnz / kBucket + nrows / kThreads + 2 * (nnz / kLongLen) + 4;
  return std::min<int64_t>(b, nrows + 1);
}

struct Layout {
  size_t tiles_a, tiles_at, flags, pos, keys_out, iota, row_of, cub_tmp, cub_bytes, dvec_m,
      dvec_n, part, part_count, params, pow, results, fac, total;
};

int cub_temp_bytes(const hpr_dims &d, size_t *bytes) {
  size_t s1 = 0, s2 = 0;
  int nnz = (int)d.nnz;
  int nmax = (int)std::max(d.m, d.n);
  CK(cub::DeviceRadixSort::SortPairs(nullptr, s1, (const int *)nullptr, (int *)nullptr,
                                     (const int *)nullptr, (int *)nullptr, nnz, 0, 32));
  CK(cub::DeviceScan::ExclusiveSum(nullptr, s2, (const int *)nullptr, (int *)nullptr, nmax));
  *bytes = std::max(s1, s2);
  return HPR_OK;
}

Layout make_layout(const hpr_dims &d, size_t cub_bytes) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const int64_t nmax = std::max(d.m, d.n);
  const int64_t tb_a = tile_bound(d.m, d.nnz), tb_at = tile_bound(d.n, d.nnz);
  L.tiles_a = take(sizeof(int) * (tb_a + 1));
  L.tiles_at = take(sizeof(int) * (tb_at + 1));
  L.flags = take(sizeof(int) * (nmax + 1));
  L.pos = take(sizeof(int) * (nmax + 1));
  L.keys_out = take(sizeof(int) * std::max<int64_t>(d.nnz, 1));
  L.iota = take(sizeof(int) * std::max<int64_t>(d.nnz, 1));
  L.row_of = take(sizeof(int) * std::max<int64_t>(d.nnz, 1));
  L.cub_bytes = cub_bytes;
  L.cub_tmp = take(std::max<size_t>(cub_bytes, 16));
  L.dvec_m = take(sizeof(double) * std::max<int64_t>(d.m, 1));
  L.dvec_n = take(sizeof(double) * std::max<int64_t>(d.n, 1));
  // partials: x_half 2, merit 2, kkt_col 8 per A^T tile; y_half 2, kkt_row 3 per A tile;
  // plus sum-of-squares passes over max(m, n) with up to 4 * 1024 CTAs
  L.part_count = (size_t)12 * tb_at + (size_t)5 * tb_a + 4 * 1024 + 3 * std::max(tb_a, tb_at);
  L.part = take(sizeof(double) * L.part_count);
  L.params = take(sizeof(IterParams));
  L.pow = take(sizeof(PowState));
  L.results = take(sizeof(double) * 64);
  L.fac = take(sizeof(double) * 2);
  L.total = off;
  (void)nmax;
  return L;
}

int grid_for(int64_t n, int threads = 256, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

}  // namespace

struct hpr_ctx {
  hpr_dims d{};
  int device = 0;
  cudaStream_t stream = nullptr;
  hpr_buffers B{};
  bool bound = false, analyzed = false, scaled = false;
  char *ws = nullptr;
  Layout L{};
  int *tiles_a = nullptr, *tiles_at = nullptr;
  int ntiles_a = 0, ntiles_at = 0;
  double *part = nullptr, *results = nullptr, *fac = nullptr, *dvec_m = nullptr, *dvec_n = nullptr;
  IterParams *params = nullptr;
  PowState *pow = nullptr;
  double *h_results = nullptr;       // pinned
  IterParams *h_params = nullptr;    // pinned
  PowState *h_pow = nullptr;         // pinned
  std::map<int, cudaGraphExec_t> inner_graphs;
  cudaGraphExec_t pow_graph = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  bool inner_timed = false, ckpt_timed = false;
  long long launches = 0;

  TileMat mat_a(const double *val) const {
    return TileMat{B.a_rp, B.a_ci, val, tiles_a, ntiles_a, kCap};
  }
  TileMat mat_at(const double *val) const {
    return TileMat{B.at_rp, B.at_ci, val, tiles_at, ntiles_at, kCap};
  }
  static size_t smem() { return sizeof(double) * (size_t)(kCap + (kCap >> 4) + 16); }
};

namespace {

int set_smem_attrs() {
  static bool done = false;
  if (done) return HPR_OK;
  const int bytes = (int)hpr_ctx::smem();
  CK(cudaFuncSetAttribute(k_x_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_y_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_x_half, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_y_half, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_kkt_row, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_kkt_col, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_merit_col, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_pow_t, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(k_pow_a, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done = true;
  return HPR_OK;
}

// parts layout inside ctx->part (in doubles)
struct Parts {
  double *xhalf, *yhalf, *krow, *kcol, *merit, *misc;
};
Parts parts_of(const hpr_ctx *c) {
  Parts p;
  const size_t ta = std::max(c->ntiles_a, 1), tat = std::max(c->ntiles_at, 1);
  p.xhalf = c->part;
  p.merit = p.xhalf + 2 * tat;
  p.kcol = p.merit + 2 * tat;
  p.yhalf = p.kcol + 8 * tat;
  p.krow = p.yhalf + 2 * ta;
  p.misc = p.krow + 3 * ta;
  return p;
}

// partial buffer for a k_sumsq pass over n elements (<= 1024 CTAs)
int sumsq_blocks(int64_t n) { return grid_for(n, kThreads, 1024); }

int build_tiles(hpr_ctx *c, const int *rp, int nrows, int *tile_row, int *ntiles_out) {
  int *flags = (int *)(c->ws + c->L.flags);
  int *pos = (int *)(c->ws + c->L.pos);
  const int g = grid_for(nrows);
  k_tile_flags<<<g, 256, 0, c->stream>>>(rp, nrows, kBucket, kLongLen, flags);
  CKL();
  size_t tb = c->L.cub_bytes;
  CK(cub::DeviceScan::ExclusiveSum(c->ws + c->L.cub_tmp, tb, flags, pos, nrows, c->stream));
  k_tile_scatter<<<g, 256, 0, c->stream>>>(flags, pos, nrows, tile_row);
  CKL();
  c->launches += 3;
  int hp = 0, hf = 0;
  CK(cudaMemcpyAsync(&hp, pos + nrows - 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&hf, flags + nrows - 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *ntiles_out = hp + hf;
  return HPR_OK;
}

// fixed-order final reduction of a list of partial segments into ctx->results
int reduce_final(hpr_ctx *c, const std::vector<RedSeg> &segs) {
  RedList L{};
  L.nseg = (int)segs.size();
  for (size_t i = 0; i < segs.size(); ++i) L.seg[i] = segs[i];
  k_reduce_final<<<L.nseg, kThreads, 0, c->stream>>>(L, c->results);
  CKL();
  c->launches += 1;
  return HPR_OK;
}

int fetch_results(hpr_ctx *c) {
  CK(cudaMemcpyAsync(c->h_results, c->results, sizeof(double) * R_COUNT, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaMemcpyAsync(c->h_params, c->params, sizeof(IterParams), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return HPR_OK;
}

// sum of squares of a device vector into results[slot] (deterministic)
int sumsq_into(hpr_ctx *c, const double *a, int64_t n, double *partbuf, int slot) {
  const int nb = sumsq_blocks(n);
  k_sumsq<<<nb, kThreads, 0, c->stream>>>(a, n, partbuf);
  CKL();
  c->launches += 1;
  return reduce_final(c, {RedSeg{partbuf, nb, slot}});
}

void fill_out(const hpr_ctx *c, hpr_ckpt_out *o) {
  const double *r = c->h_results;
  o->bar_dx2 = r[R_BAR_DX2];
  o->dx2 = r[R_DX2];
  o->dy2 = r[R_DY2];
  o->bar_dy2 = r[R_BAR_DY2];
  o->prim2 = r[R_PRIM2];
  o->by = r[R_BY];
  o->r1sq = r[R_R1];
  o->dual2 = r[R_DUAL2];
  o->cx = r[R_CX];
  o->lz = r[R_LZ];
  o->uz = r[R_UZ];
  o->n_lo = (int64_t)r[R_NLO];
  o->n_up = (int64_t)r[R_NUP];
  o->clamped = (int64_t)r[R_CLAMP];
  o->r2sq = r[R_R2];
  o->sh2 = r[R_SH2];
  o->aty2 = r[R_ATY2];
  o->nonfinite_k = c->h_params->nonfinite_k == ULLONG_MAX ? -1 : (int64_t)c->h_params->nonfinite_k;
}

// KKT kernels on the termination problem for candidate `slot` (+ reduction segments)
int launch_kkt(hpr_ctx *c, int term_original, const double *cy, const double *cx,
               const double *cz, std::vector<RedSeg> &segs) {
  const hpr_buffers &B = c->B;
  Parts P = parts_of(c);
  const size_t sm = hpr_ctx::smem();
  const double *aval = term_original ? B.a_val : B.a_val_s;
  const double *atval = term_original ? B.at_val : B.at_val_s;
  k_kkt_row<<<c->ntiles_a, kThreads, sm, c->stream>>>(c->mat_a(aval), cx, cy,
                                                       term_original ? B.b : B.b_s,
                                                       (int)c->d.m1, P.krow);
  CKL();
  k_kkt_col<<<c->ntiles_at, kThreads, sm, c->stream>>>(
      c->mat_at(atval), cy, cx, cz, term_original ? B.c : B.c_s,
      term_original ? B.lower : B.lower_s, term_original ? B.upper : B.upper_s, P.kcol);
  CKL();
  c->launches += 2;
  const int ta = c->ntiles_a, tat = c->ntiles_at;
  segs.push_back({P.krow + 0 * ta, ta, R_PRIM2});
  segs.push_back({P.krow + 1 * ta, ta, R_BY});
  segs.push_back({P.krow + 2 * ta, ta, R_R1});
  const int outs[8] = {R_DUAL2, R_CX, R_LZ, R_UZ, R_NLO, R_NUP, R_CLAMP, R_R2};
  for (int q = 0; q < 8; ++q) segs.push_back({P.kcol + q * tat, tat, outs[q]});
  return HPR_OK;
}

int check_ctx(hpr_ctx *c, bool need_analyzed = true, bool need_scaled = false) {
  if (!c) return fail(HPR_EINVAL, "null context");
  if (!c->bound) return fail(HPR_ESTATE, "hpr_bind has not been called");
  if (need_analyzed && !c->analyzed) return fail(HPR_ESTATE, "hpr_analyze has not been called");
  if (need_scaled && !c->scaled) return fail(HPR_ESTATE, "hpr_scale has not been called");
  return HPR_OK;
}

}  // namespace

extern "C" {

int hpr_abi_version(void) { return HPR_ABI_VERSION; }

const char *hpr_last_error(void) { return g_err.c_str(); }

int hpr_workspace_bytes(const hpr_dims *dims, size_t *bytes) {
  if (!dims || !bytes) return fail(HPR_EINVAL, "null argument");
  if (dims->m < 1 || dims->n < 1 || dims->nnz < 0 || dims->m1 < 0 || dims->m1 > dims->m)
    return fail(HPR_EINVAL, "invalid dims");
  if (dims->nnz >= INT_MAX || dims->m >= INT_MAX || dims->n >= INT_MAX)
    return fail(HPR_EINVAL, "dims exceed int32 indexing");
  size_t cb = 0;
  int rc = cub_temp_bytes(*dims, &cb);
  if (rc) return rc;
  *bytes = make_layout(*dims, cb).total;
  return HPR_OK;
}

int hpr_ctx_create(hpr_ctx **out, const hpr_dims *dims, int device, void *stream) {
  if (!out || !dims) return fail(HPR_EINVAL, "null argument");
  if (!stream) return fail(HPR_EINVAL, "a non-default stream is required (graph capture)");
  hpr_ctx *c = new hpr_ctx();
  c->d = *dims;
  c->device = device;
  c->stream = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_results, sizeof(double) * 64);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_params, sizeof(IterParams));
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_pow, sizeof(PowState));
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev2);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev3);
  if (e != cudaSuccess) {
    hpr_ctx_destroy(c);
    return fail(HPR_ECUDA, std::string("ctx_create: ") + cudaGetErrorString(e));
  }
  int rc = set_smem_attrs();
  if (rc) {
    hpr_ctx_destroy(c);
    return rc;
  }
  *out = c;
  return HPR_OK;
}

int hpr_ctx_destroy(hpr_ctx *c) {
  if (!c) return HPR_OK;
  for (auto &kv : c->inner_graphs) cudaGraphExecDestroy(kv.second);
  if (c->pow_graph) cudaGraphExecDestroy(c->pow_graph);
  if (c->h_results) cudaFreeHost(c->h_results);
  if (c->h_params) cudaFreeHost(c->h_params);
  if (c->h_pow) cudaFreeHost(c->h_pow);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->ev2) cudaEventDestroy(c->ev2);
  if (c->ev3) cudaEventDestroy(c->ev3);
  delete c;
  return HPR_OK;
}

int hpr_bind(hpr_ctx *c, const hpr_buffers *bufs, void *workspace, size_t ws_bytes) {
  if (!c || !bufs || !workspace) return fail(HPR_EINVAL, "null argument");
  size_t cb = 0;
  int rc = cub_temp_bytes(c->d, &cb);
  if (rc) return rc;
  Layout L = make_layout(c->d, cb);
  if (ws_bytes < L.total) return fail(HPR_EINVAL, "workspace too small");
  const void *req[] = {bufs->a_rp, bufs->a_ci, bufs->a_val, bufs->a_val_s, bufs->at_rp,
                       bufs->at_ci, bufs->at_perm, bufs->at_val, bufs->at_val_s, bufs->b,
                       bufs->c, bufs->lower, bufs->upper, bufs->b_s, bufs->c_s, bufs->lower_s,
                       bufs->upper_s, bufs->row_scale, bufs->col_scale, bufs->y, bufs->x,
                       bufs->anc_y, bufs->anc_x, bufs->w, bufs->yb, bufs->xb, bufs->zb, bufs->dy,
                       bufs->wtmp, bufs->cand_y[0], bufs->cand_y[1], bufs->cand_x[0],
                       bufs->cand_x[1], bufs->cand_z[0], bufs->cand_z[1]};
  for (const void *p : req)
    if (!p && c->d.nnz > 0) return fail(HPR_EINVAL, "a required buffer pointer is null");
  c->B = *bufs;
  c->ws = (char *)workspace;
  c->L = L;
  c->tiles_a = (int *)(c->ws + L.tiles_a);
  c->tiles_at = (int *)(c->ws + L.tiles_at);
  c->part = (double *)(c->ws + L.part);
  c->results = (double *)(c->ws + L.results);
  c->fac = (double *)(c->ws + L.fac);
  c->dvec_m = (double *)(c->ws + L.dvec_m);
  c->dvec_n = (double *)(c->ws + L.dvec_n);
  c->params = (IterParams *)(c->ws + L.params);
  c->pow = (PowState *)(c->ws + L.pow);
  for (auto &kv : c->inner_graphs) cudaGraphExecDestroy(kv.second);
  c->inner_graphs.clear();
  if (c->pow_graph) {
    cudaGraphExecDestroy(c->pow_graph);
    c->pow_graph = nullptr;
  }
  c->bound = true;
  c->analyzed = c->scaled = false;
  return HPR_OK;
}

int hpr_analyze(hpr_ctx *c) {
  int rc = check_ctx(c, false);
  if (rc) return rc;
  CK(cudaSetDevice(c->device));
  const hpr_dims &d = c->d;
  const hpr_buffers &B = c->B;
  const int nnz = (int)d.nnz, m = (int)d.m, n = (int)d.n;
  int *keys_out = (int *)(c->ws + c->L.keys_out);
  int *iota = (int *)(c->ws + c->L.iota);
  int *row_of = (int *)(c->ws + c->L.row_of);
  if (nnz > 0) {
    k_iota<<<grid_for(nnz), 256, 0, c->stream>>>(iota, nnz);
    CKL();
    int end_bit = 1;
    while ((1LL << end_bit) < n) ++end_bit;
    size_t tb = c->L.cub_bytes;
    // stable LSD radix sort by column: rows stay ascending inside each column,
    // the ordering csr_matrix(A.T) produces (sparse.py:98-100)
    CK(cub::DeviceRadixSort::SortPairs(c->ws + c->L.cub_tmp, tb, B.a_ci, keys_out, iota,
                                       B.at_perm, nnz, 0, end_bit, c->stream));
    k_col_count<<<grid_for(nnz), 256, 0, c->stream>>>(keys_out, nnz, n, B.at_rp);
    CKL();
    k_row_of<<<grid_for(m), 256, 0, c->stream>>>(B.a_rp, m, row_of);
    CKL();
    k_gather_t<<<grid_for(nnz), 256, 0, c->stream>>>(B.at_perm, row_of, B.a_val, B.at_ci,
                                                      B.at_val, nnz);
    CKL();
    c->launches += 5;
  } else {
    k_fill_empty_rpt<<<grid_for(n + 1), 256, 0, c->stream>>>(B.at_rp, n);
    CKL();
    c->launches += 1;
  }
  rc = build_tiles(c, B.a_rp, m, c->tiles_a, &c->ntiles_a);
  if (rc) return rc;
  rc = build_tiles(c, B.at_rp, n, c->tiles_at, &c->ntiles_at);
  if (rc) return rc;
  if (c->ntiles_a > tile_bound(m, nnz) || c->ntiles_at > tile_bound(n, nnz))
    return fail(HPR_ESTATE, "tile count exceeds its bound");
  c->analyzed = true;
  return HPR_OK;
}

int hpr_scale(hpr_ctx *c, int ruiz_iters, int pock_chambolle, int bc_normalize,
              hpr_scale_out *out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  CK(cudaSetDevice(c->device));
  const hpr_dims &d = c->d;
  const hpr_buffers &B = c->B;
  const int m = (int)d.m, n = (int)d.n;
  const long long nnz = d.nnz;
  cudaStream_t s = c->stream;
  double *dr = c->dvec_m, *dc = c->dvec_n;
  CK(cudaMemcpyAsync(B.a_val_s, B.a_val, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
  k_fill<<<grid_for(m), 256, 0, s>>>(B.row_scale, 1.0, m);
  k_fill<<<grid_for(n), 256, 0, s>>>(B.col_scale, 1.0, n);
  CKL();
  c->launches += 2;
  const int wg = grid_for((int64_t)m * 32);
  for (int it = 0; it < ruiz_iters; ++it) {  // sparse.py:216-223
    k_row_maxabs<<<grid_for(m), 256, 0, s>>>(B.a_rp, B.a_val_s, m, dr);
    k_col_maxabs<<<grid_for(n), 256, 0, s>>>(B.at_rp, B.at_perm, B.a_val_s, n, dc);
    k_sqrt_div<<<grid_for(m), 256, 0, s>>>(dr, B.row_scale, m);
    k_sqrt_div<<<grid_for(n), 256, 0, s>>>(dc, B.col_scale, n);
    k_scale_vals<<<wg, 256, 0, s>>>(B.a_rp, B.a_ci, B.a_val_s, dr, dc, m);
    CKL();
    c->launches += 5;
  }
  if (pock_chambolle) {  // sparse.py:232-242
    k_row_abssum<<<grid_for(m), 256, 0, s>>>(B.a_rp, B.a_val_s, m, dr);
    k_col_abssum<<<grid_for(n), 256, 0, s>>>(B.at_rp, B.at_perm, B.a_val_s, n, dc);
    k_sqrt_div<<<grid_for(m), 256, 0, s>>>(dr, B.row_scale, m);
    k_sqrt_div<<<grid_for(n), 256, 0, s>>>(dc, B.col_scale, n);
    k_scale_vals<<<wg, 256, 0, s>>>(B.a_rp, B.a_ci, B.a_val_s, dr, dc, m);
    CKL();
    c->launches += 5;
  }
  const int g = grid_for(std::max(m, n));
  k_scale_vecs<<<g, 256, 0, s>>>(B.b, B.row_scale, B.b_s, m, B.c, B.lower, B.upper,
                                 B.col_scale, B.c_s, B.lower_s, B.upper_s, n);
  CKL();
  c->launches += 1;
  Parts P = parts_of(c);
  if (bc_normalize) {  // sparse.py:245-250, scaling.py:98-101
    const int nb0 = sumsq_blocks(m), nb1 = sumsq_blocks(n);
    k_sumsq<<<nb0, kThreads, 0, s>>>(B.b_s, m, P.misc);
    k_sumsq<<<nb1, kThreads, 0, s>>>(B.c_s, n, P.misc + 1024);
    CKL();
    c->launches += 2;
    rc = reduce_final(c, {RedSeg{P.misc, nb0, R_SUMSQ0}, RedSeg{P.misc + 1024, nb1, R_SUMSQ1}});
    if (rc) return rc;
    k_factors<<<1, 32, 0, s>>>(c->results + R_SUMSQ0, c->fac);
    k_bc_normalize<<<g, 256, 0, s>>>(B.b_s, m, B.c_s, B.lower_s, B.upper_s, n, c->fac);
    CKL();
    c->launches += 2;
  } else {
    const double ones[2] = {1.0, 1.0};
    CK(cudaMemcpyAsync(c->fac, ones, sizeof(ones), cudaMemcpyHostToDevice, s));
  }
  if (nnz > 0) {
    k_gather_vals<<<grid_for(nnz), 256, 0, s>>>(B.at_perm, B.a_val_s, B.at_val_s, nnz);
    CKL();
    c->launches += 1;
  }
  // ||b||, ||c|| of the original and the scaled problem (relative residual denominators)
  const int nbm = sumsq_blocks(m), nbn = sumsq_blocks(n);
  k_sumsq<<<nbm, kThreads, 0, s>>>(B.b, m, P.misc);
  k_sumsq<<<nbn, kThreads, 0, s>>>(B.c, n, P.misc + 1024);
  k_sumsq<<<nbm, kThreads, 0, s>>>(B.b_s, m, P.misc + 2048);
  k_sumsq<<<nbn, kThreads, 0, s>>>(B.c_s, n, P.misc + 3072);
  CKL();
  c->launches += 4;
  rc = reduce_final(c, {RedSeg{P.misc, nbm, R_SUMSQ0}, RedSeg{P.misc + 1024, nbn, R_SUMSQ1},
                        RedSeg{P.misc + 2048, nbm, R_SUMSQ2}, RedSeg{P.misc + 3072, nbn, R_SUMSQ3}});
  if (rc) return rc;
  double fac[2];
  CK(cudaMemcpyAsync(fac, c->fac, sizeof(fac), cudaMemcpyDeviceToHost, s));
  rc = fetch_results(c);
  if (rc) return rc;
  if (out) {
    out->b_factor = fac[0];
    out->c_factor = fac[1];
    out->bnorm_orig = std::sqrt(c->h_results[R_SUMSQ0]);
    out->cnorm_orig = std::sqrt(c->h_results[R_SUMSQ1]);
    out->bnorm_s = std::sqrt(c->h_results[R_SUMSQ2]);
    out->cnorm_s = std::sqrt(c->h_results[R_SUMSQ3]);
  }
  c->scaled = true;
  return HPR_OK;
}

int hpr_power(hpr_ctx *c, double tol, int max_iters, hpr_power_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out) return fail(HPR_EINVAL, "null out");
  if (c->d.nnz == 0) return fail(HPR_EINVAL, "matrix must be non-zero");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  const int m = (int)c->d.m, n = (int)c->d.n;
  cudaStream_t s = c->stream;
  double *v = B.yb, *u = B.wtmp, *wv = B.dy;   // scratch reuse (before the iterations)
  Parts P = parts_of(c);
  const size_t sm = hpr_ctx::smem();
  PowState st{};
  st.tol = tol;
  st.max_iters = max_iters;
  // all-ones start; fall back to basis vectors while A^T v == 0 (sparse.py:176-182)
  int start = -2;
  for (int fb = -1; fb < m; ++fb) {
    if (fb < 0) {
      k_fill<<<grid_for(m), 256, 0, s>>>(v, 1.0, m);
    } else {
      k_fill<<<grid_for(m), 256, 0, s>>>(v, 0.0, m);
      const double one = 1.0;
      CK(cudaMemcpyAsync(v + fb, &one, sizeof(double), cudaMemcpyHostToDevice, s));
      CK(cudaStreamSynchronize(s));   // `one` lives on this stack frame
    }
    CK(cudaMemcpyAsync(c->pow, &st, sizeof(st), cudaMemcpyHostToDevice, s));
    k_pow_t<<<c->ntiles_at, kThreads, sm, s>>>(c->mat_at(B.at_val_s), v, u, c->pow, P.misc);
    CKL();
    c->launches += 2;
    rc = reduce_final(c, {RedSeg{P.misc, c->ntiles_at, R_POW_U2}});
    if (rc) return rc;
    rc = fetch_results(c);
    if (rc) return rc;
    if (std::sqrt(c->h_results[R_POW_U2]) > 0.0) {
      start = fb;
      break;
    }
  }
  if (start == -2) return fail(HPR_EINVAL, "A^T v = 0 for every start vector");
  // v /= ||v||: ||ones(m)|| = sqrt(m) exactly; a basis vector has norm 1
  if (start == -1) {
    const double inv = 1.0 / std::sqrt((double)m);
    k_fill<<<grid_for(m), 256, 0, s>>>(v, inv, m);
    CKL();
    c->launches += 1;
  }
  CK(cudaMemcpyAsync(c->pow, &st, sizeof(st), cudaMemcpyHostToDevice, s));
  if (max_iters <= 0) {
    out->value = 0.0;
    out->raw = 0.0;
    out->iterations = 0;
    out->converged = 0;
    return HPR_OK;
  }
  if (!c->pow_graph) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kPowBatch; ++i) {
      k_pow_t<<<c->ntiles_at, kThreads, sm, s>>>(c->mat_at(B.at_val_s), v, u, c->pow, P.misc);
      k_pow_a<<<c->ntiles_a, kThreads, sm, s>>>(c->mat_a(B.a_val_s), u, v, wv, c->pow,
                                                P.misc + c->ntiles_at);
      k_pow_step<<<1, kThreads, 0, s>>>(P.misc + c->ntiles_at, c->ntiles_a, c->pow);
      k_pow_norm<<<grid_for(m), 256, 0, s>>>(wv, v, m, c->pow);
      k_pow_norm_done<<<1, 1, 0, s>>>(c->pow);
    }
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("pow capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->pow_graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("pow instantiate: ") + cudaGetErrorString(e));
  }
  for (;;) {
    CK(cudaGraphLaunch(c->pow_graph, s));
    c->launches += 5 * kPowBatch;
    CK(cudaMemcpyAsync(c->h_pow, c->pow, sizeof(PowState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (c->h_pow->done) break;
  }
  out->raw = c->h_pow->lam;
  out->value = c->h_pow->lam * (1.0 + 1e-3);
  out->iterations = c->h_pow->iters;
  out->converged = c->h_pow->converged;
  (void)n;
  return HPR_OK;
}

int hpr_state_reset(hpr_ctx *c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  const size_t mb = sizeof(double) * c->d.m, nb = sizeof(double) * c->d.n;
  CK(cudaMemsetAsync(B.y, 0, mb, s));
  CK(cudaMemsetAsync(B.anc_y, 0, mb, s));
  CK(cudaMemsetAsync(B.x, 0, nb, s));
  CK(cudaMemsetAsync(B.anc_x, 0, nb, s));
  CK(cudaMemsetAsync(B.w, 0, nb, s));
  IterParams p{};
  p.nonfinite_k = ULLONG_MAX;
  CK(cudaMemcpyAsync(c->params, &p, sizeof(p), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return HPR_OK;
}

int hpr_run_inner(hpr_ctx *c, int steps, int64_t t, int64_t k, double sigma, double lamsig,
                  int variant) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (steps <= 0) return HPR_OK;
  if (variant < 0 || variant > 2) return fail(HPR_EINVAL, "bad variant");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  auto it = c->inner_graphs.find(steps);
  if (it == c->inner_graphs.end()) {
    const size_t sm = hpr_ctx::smem();
    const TileMat A = c->mat_a(B.a_val_s), AT = c->mat_at(B.at_val_s);
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < steps; ++i) {
      k_x_iter<<<c->ntiles_at, kThreads, sm, s>>>(AT, B.y, B.x, B.w, B.c_s, B.lower_s,
                                                  B.upper_s, B.anc_x, c->params, i);
      k_y_iter<<<c->ntiles_a, kThreads, sm, s>>>(A, B.w, B.y, B.b_s, B.anc_y, (int)c->d.m1,
                                                 c->params, i);
    }
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t ex;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    it = c->inner_graphs.emplace(steps, ex).first;
  }
  k_set_params<<<1, 1, 0, s>>>(c->params, sigma, lamsig, (long long)t, (long long)k, variant);
  CKL();
  CK(cudaEventRecord(c->ev0, s));
  CK(cudaGraphLaunch(it->second, s));
  CK(cudaEventRecord(c->ev1, s));
  c->inner_timed = true;
  c->launches += 1 + 2LL * steps;
  return HPR_OK;
}

int hpr_checkpoint(hpr_ctx *c, double sigma, double lamsig, int term_original, int slot,
                   hpr_ckpt_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  const size_t sm = hpr_ctx::smem();
  Parts P = parts_of(c);
  CandCtx cc{term_original, c->fac, B.row_scale, B.col_scale, B.lower, B.upper};
  CK(cudaEventRecord(c->ev2, s));
  k_x_half<<<c->ntiles_at, kThreads, sm, s>>>(c->mat_at(B.at_val_s), B.y, B.x, B.c_s, B.lower_s,
                                              B.upper_s, B.anc_x, B.xb, B.zb, B.wtmp,
                                              B.cand_x[slot], B.cand_z[slot], cc, sigma, P.xhalf);
  CKL();
  k_y_half<<<c->ntiles_a, kThreads, sm, s>>>(c->mat_a(B.a_val_s), B.wtmp, B.y, B.b_s, B.anc_y,
                                             (int)c->d.m1, lamsig, B.yb, B.dy, B.cand_y[slot], cc,
                                             P.yhalf);
  CKL();
  k_merit_col<<<c->ntiles_at, kThreads, sm, s>>>(c->mat_at(B.at_val_s), B.dy, B.x, B.xb, sigma,
                                                 P.merit);
  CKL();
  c->launches += 3;
  std::vector<RedSeg> segs;
  const int ta = c->ntiles_a, tat = c->ntiles_at;
  segs.push_back({P.xhalf, tat, R_BAR_DX2});
  segs.push_back({P.xhalf + tat, tat, R_DX2});
  segs.push_back({P.yhalf, ta, R_DY2});
  segs.push_back({P.yhalf + ta, ta, R_BAR_DY2});
  segs.push_back({P.merit, tat, R_SH2});
  segs.push_back({P.merit + tat, tat, R_ATY2});
  rc = launch_kkt(c, term_original, B.cand_y[slot], B.cand_x[slot], B.cand_z[slot], segs);
  if (rc) return rc;
  rc = reduce_final(c, segs);
  if (rc) return rc;
  CK(cudaEventRecord(c->ev3, s));
  rc = fetch_results(c);
  if (rc) return rc;
  c->ckpt_timed = true;
  fill_out(c, out);
  return HPR_OK;
}

int hpr_restart(hpr_ctx *c) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  const size_t mb = sizeof(double) * c->d.m, nb = sizeof(double) * c->d.n;
  CK(cudaMemcpyAsync(B.y, B.yb, mb, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(B.anc_y, B.yb, mb, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(B.x, B.xb, nb, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(B.anc_x, B.xb, nb, cudaMemcpyDeviceToDevice, s));
  return HPR_OK;
}

int hpr_kkt_origin(hpr_ctx *c, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  const int m = (int)c->d.m, n = (int)c->d.n;
  k_origin_cand<<<grid_for(std::max(m, n)), 256, 0, s>>>(
      B.cand_y[slot], m, B.cand_z[slot], B.cand_x[slot], term_original ? B.lower : B.lower_s,
      term_original ? B.upper : B.upper_s, n);
  CKL();
  c->launches += 1;
  std::vector<RedSeg> segs;
  rc = launch_kkt(c, term_original, B.cand_y[slot], B.cand_x[slot], B.cand_z[slot], segs);
  if (rc) return rc;
  CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, s));
  rc = reduce_final(c, segs);
  if (rc) return rc;
  rc = fetch_results(c);
  if (rc) return rc;
  fill_out(c, out);
  return HPR_OK;
}

int hpr_kkt(hpr_ctx *c, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  std::vector<RedSeg> segs;
  rc = launch_kkt(c, term_original, B.cand_y[slot], B.cand_x[slot], B.cand_z[slot], segs);
  if (rc) return rc;
  CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, c->stream));
  rc = reduce_final(c, segs);
  if (rc) return rc;
  rc = fetch_results(c);
  if (rc) return rc;
  fill_out(c, out);
  return HPR_OK;
}

int hpr_finalize(hpr_ctx *c, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  const int m = (int)c->d.m, n = (int)c->d.n;
  int fs = slot;
  if (!term_original) {
    fs = 1 - slot;
    k_unscale<<<grid_for(std::max(m, n)), 256, 0, s>>>(
        B.cand_y[slot], B.cand_z[slot], B.cand_x[slot], B.cand_y[fs], B.cand_z[fs],
        B.cand_x[fs], B.row_scale, B.col_scale, c->fac, B.lower, B.upper, m, n);
    CKL();
    c->launches += 1;
  }
  std::vector<RedSeg> segs;
  rc = launch_kkt(c, 1, B.cand_y[fs], B.cand_x[fs], B.cand_z[fs], segs);
  if (rc) return rc;
  CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, s));
  rc = reduce_final(c, segs);
  if (rc) return rc;
  rc = fetch_results(c);
  if (rc) return rc;
  fill_out(c, out);
  return HPR_OK;
}

int hpr_launch_count(hpr_ctx *c, int64_t *count) {
  if (!c || !count) return fail(HPR_EINVAL, "null argument");
  *count = c->launches;
  return HPR_OK;
}

int hpr_tile_info(hpr_ctx *c, int64_t *ntiles_a, int64_t *ntiles_at) {
  if (!c || !ntiles_a || !ntiles_at) return fail(HPR_EINVAL, "null argument");
  *ntiles_a = c->ntiles_a;
  *ntiles_at = c->ntiles_at;
  return HPR_OK;
}

int hpr_last_times(hpr_ctx *c, double *inner_ms, double *ckpt_ms) {
  if (!c || !inner_ms || !ckpt_ms) return fail(HPR_EINVAL, "null argument");
  float a = 0.f, b = 0.f;
  if (c->inner_timed) CK(cudaEventElapsedTime(&a, c->ev0, c->ev1));
  if (c->ckpt_timed) CK(cudaEventElapsedTime(&b, c->ev2, c->ev3));
  *inner_ms = a;
  *ckpt_ms = b;
  return HPR_OK;
}

}  // extern "C"
