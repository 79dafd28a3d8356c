// hpr_capi.cu -- C ABI (include/hprlp_b200.h) over the sm_100a kernels.
//
// Host-side orchestration only: workspace carve-up, the transpose and
// SELL-32-sigma layout analysis, the scaling and power-method passes, CUDA-graph
// capture of the inner loop, the checkpoint sequence and its single
// device->host readback.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hprlp_b200.h"
#include "hpr_kernels.cuh"
#include "hpr_cb.cuh"
#include "hpr_stg.cuh"
#include "hpr_tsell.cuh"
#include "hpr_exact.cuh"

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

#ifndef HPR_PDL
#define HPR_PDL 0       // programmatic dependent launch between inner-loop phases (measured: no gain in graphs)
#endif
#ifndef HPR_CARVEOUT
#define HPR_CARVEOUT -1   // SELL kernels' preferred shared-memory carve-out (-1: driver default)
#endif
#ifndef HPR_TS_DEFAULT
#define HPR_TS_DEFAULT 2    // TS engine selection without HPR_TS: 0 never, 1 always, 2 auto
#endif
#ifndef HPR_L2KEEP
#define HPR_L2KEEP 4    // matrix L2 policy: 0 evict_first, 1 keep A, 2 keep A^T, 3 normal, 4 auto
#endif
#ifndef HPR_SELL_U
#define HPR_SELL_U 4    // entries per lane per batch without gather-ahead (2 / 8: C3 +20 % / +100 %)
#endif
#ifndef HPR_GA_U
#define HPR_GA_U 3      // entries per lane per batch on the gather-ahead path (4: 80 registers + spills; 3: C2 48.2 -> 46.3 us, C4 rank 1625 -> 1590 us per iteration)
#endif
#ifndef HPR_GA_MIN
#define HPR_GA_MIN 12   // avg row length from which the SELL lanes gather one batch ahead
#endif                  // (measured: C2 (25/50 per row) -5 %, C3 (3/8-32 per row) +18 % -> long rows only
#ifndef HPR_X_IMPLICIT
#define HPR_X_IMPLICIT 1    // HPR inner loop: x re-formed from w inside an interval (EpiXIter)
#endif
#ifndef HPR_TS_U_AW
#define HPR_TS_U_AW 3   // entries per lane per batch of the index-word TS kernel (4: spills)
#endif
#ifndef HPR_TS_AW
#define HPR_TS_AW 0   // 1: TS engine reads per-slice index words (lane-affine / uniform slices: one per entry); C3 x-phase 833 -> 877 us/iteration (slower, profiles/r02_ts_index_words.txt)
#endif
#ifndef HPR_COMPACT_HDR
#define HPR_COMPACT_HDR 1   // compact SELL slices (32 consecutive equal-length rows) skip the per-lane header
#endif
#ifndef HPR_POW_BATCH
#define HPR_POW_BATCH 16   // 8 / 16 / 32 measured 17.55-17.73 / 17.78-17.79 / 17.76-17.78 k it/s on C2
#endif
constexpr int kPowBatch = HPR_POW_BATCH;   // power steps per graph replay
constexpr int kMaxGridPerSm = 8;  // CTAs per SM cap of the SELL kernels (partials sizing)
constexpr int kSumsqBlocks = 1024;

// result slots of the final reduction (see hpr_ckpt_out)
enum {
  R_BAR_DX2, R_DX2, R_DY2, R_BAR_DY2, R_PRIM2, R_BY, R_R1, R_DUAL2, R_CX, R_LZ, R_UZ, R_NLO,
  R_NUP, R_CLAMP, R_R2, R_SH2, R_ATY2, R_SUMSQ0, R_SUMSQ1, R_SUMSQ2, R_SUMSQ3, R_POW_U2, R_NONFIN, R_POW_VW,
  R_POW_WW, R_COUNT
};

// Function attributes are per device, and concurrent solves may launch from
// several host threads: the configured dynamic shared memory (and the SELL
// kernels' occupancy) is remembered per (kernel, device) under a mutex.
std::mutex g_attr_mu;
std::map<std::pair<const void *, int>, int> g_attr;

template <class K>
int ensure_dyn_smem(K kern, int bytes) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int &have = g_attr[{(const void *)kern, dev}];
  if (bytes > have) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
  }
  return 0;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int64_t windows_of(int64_t nrows) { return (nrows + kWindow - 1) / kWindow; }

// per-matrix plan arrays in the main workspace
struct PlanOff {
  size_t slice_row, slice_len, slice_slots, slice_ptr, long_flag, long_rows, nsel;
};

// column-blocked (CB) engine plan arrays of one matrix (persistent, workspace)
struct CbOff {
  bool on = false;
  int G = 0, NB = 0;
  size_t row_start = 0, gstart = 0, gseg = 0, rpb_base = 0;
};

constexpr int kCbW = 8192;           // doubles per CB column block (64 KB)
constexpr int kCbMaxSmem = 227 * 1024 - 1024;

// The CB engine replaces L1TEX-bound random gathers by staging the operand
// vector through shared memory; it pays a full pass over the vector per SM.
// Model (B200): staging ~95 GB/s per SM, gathers ~0.55 x one L1TEX wavefront
// per cycle.  Override with HPR_CB=0 (never) / HPR_CB=1 (whenever it fits).
bool cb_wanted(int64_t rows, int64_t cols, int64_t nnz) {
  if (rows < 1 || cols < 1 || nnz < 1) return false;
  const int64_t NB = (cols + kCbW - 1) / kCbW;
  if (NB > 4096) return false;
  const char *env = getenv("HPR_CB");
  if (env && env[0] == '0') return false;
  if (env && env[0] == '1') return true;
  if (!(env && env[0] == 'a')) return false;   // measured slower than SELL on C2 so far: opt-in
  const double G = 148.0;
  const double t_cb = cols * 8.0 / 95e9 + (10.0 * nnz + 4.0 * rows * NB) / (G * 95e9);
  const double t_sell = nnz / (G * 1.92e9 * 0.55);
  return t_cb < 0.8 * t_sell;
}

// Column-split layout of A for the y-phase (hpr_kernels.cuh: EpiCarry): when
// the gathered n-vector is larger than L2 and the rows are long enough that
// the carried running sums (16 B per row per extra block) cost far less than
// the HBM sectors the random gathers would miss on, the columns are cut into
// NB blocks of W columns (W * 8 B = 32 MB stays L2-resident while every row
// walks that block).  HPR_SPLIT=0 disables it, HPR_SPLIT_COLS=<W> forces it.
constexpr int64_t kSplitCols = 4 << 20;
constexpr int kSplitMaxBlocks = 64;
struct SplitOff {
  bool on = false;
  int NB = 1, W = 0, m_pad = 0;
  int64_t V = 0;                 // virtual rows NB * m_pad
  PlanOff po;
  size_t vrp = 0, psum = 0;
};
SplitOff split_plan_of(const hpr_dims &d) {
  SplitOff o;
  if (d.m < 1 || d.n < 1 || d.nnz < 1) return o;
  const char *env = getenv("HPR_SPLIT");
  if (env && env[0] == '0') return o;
  int64_t W = kSplitCols;
  const char *wc = getenv("HPR_SPLIT_COLS");
  const bool forced = wc && atoll(wc) > 0;
  if (forced) W = atoll(wc);
  const int64_t NB = (d.n + W - 1) / W;
  if (NB < 2 || NB > kSplitMaxBlocks) return o;
  if (!forced && (double)d.nnz < 16.0 * (double)(NB - 1) * (double)d.m) return o;
  o.on = true;
  o.NB = (int)NB;
  o.W = (int)W;
  const int win = sort_win(d.m);     // windows never straddle two column blocks
  o.m_pad = (int)((d.m + win - 1) / win * win);
  o.V = (int64_t)o.NB * o.m_pad;
  if (o.V >= INT_MAX - kWindow) o.on = false;
  return o;
}

// STG engine (hpr_stg.cuh) for one matrix: rows x cols (cols = the staged
// vector).  Auto when the vector is reused enough for streaming it through
// every SM to beat gathering it (nnz >= 40 cols), the matrix is large enough
// to fill the GPU, and it fits the engine's limits; HPR_STG=0 never, =1
// whenever it fits.  The column-split and CB layouts take precedence.
constexpr int kStgMaxG = 160;
struct StgOff {
  bool on = false;
  int NB = 0;
  int64_t items = 0;          // rows * NB
  size_t row_start = 0, goff = 0;
};
// transpose: the matrix is A^T (x-phase).  HPR_STG=x / =y: force it for the
// x-phase (A^T) / y-phase (A) only.
StgOff stg_plan_of(int64_t rows, int64_t cols, int64_t nnz, bool transpose) {
  StgOff o;
  if (rows < 1 || cols < 1 || nnz < 1) return o;
  const int64_t NB = (cols + kStgW - 1) / kStgW;
  if (NB > 64 || rows * NB >= INT_MAX) return o;
  const char *env = getenv("HPR_STG");
  if (env && env[0] == '0') return o;
  if (env && ((env[0] == 'x' && !transpose) || (env[0] == 'y' && transpose))) return o;
  const bool forced = env && (env[0] == '1' || env[0] == 'x' || env[0] == 'y');
  if (!forced && (nnz < 40 * cols || rows < 148 * 64)) return o;
  o.on = true;
  o.NB = (int)NB;
  o.items = rows * NB;
  return o;
}

struct Layout {
  StgOff sa, sat;
  size_t stg_key = 0, stg_lrow = 0, stg_skey = 0, stg_slrow = 0, stg_gstart = 0, stg_rbytes = 0,
         stg_flag = 0;
  SplitOff sp;
  PlanOff pa, pat;
  CbOff ca, cat;
  size_t cb_key = 0, cb_lrow = 0;
  size_t keys_out, iota, row_of, cub_tmp, cub_bytes, dvec_m, dvec_n, part, part_count, params,
      pow, results, fac, flags, total;
};

int cub_temp_bytes(const hpr_dims &d, size_t *bytes) {
  size_t s1 = 0, s2 = 0, s3 = 0;
  const int nnz = (int)d.nnz;
  const int nmax = (int)std::max(d.m, d.n);
  const SplitOff sp = split_plan_of(d);
  const int smax = (int)std::max<int64_t>(windows_of(nmax) * (kWindow / kSlice) + 1,
                                          sp.on ? sp.V + 1 : 0);
  CK(cub::DeviceRadixSort::SortPairs(nullptr, s1, (const int *)nullptr, (int *)nullptr,
                                     (const int *)nullptr, (int *)nullptr, nnz, 0, 32));
  CK(cub::DeviceScan::ExclusiveSum(nullptr, s2, (const int *)nullptr, (int *)nullptr, smax));
  CK(cub::DeviceSelect::Flagged(nullptr, s3, cub::CountingInputIterator<int>(0),
                                (const int *)nullptr, (int *)nullptr, (int *)nullptr,
                                std::max<int64_t>(nmax, sp.V)));
  size_t s4 = 0, s5 = 0;
  for (const StgOff &o : {stg_plan_of(d.m, d.n, d.nnz, false), stg_plan_of(d.n, d.m, d.nnz, true)}) {
    if (!o.on) continue;
    size_t a = 0, b = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, a, (const unsigned *)nullptr, (unsigned *)nullptr,
                                       (const int *)nullptr, (int *)nullptr, (int)o.items, 0, 32));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, b, (const long long *)nullptr, (long long *)nullptr,
                                     (int)(kStgMaxG * o.NB + 1)));
    s4 = std::max(s4, a);
    s5 = std::max(s5, b);
  }
  *bytes = std::max(std::max(s1, std::max(s2, s3)), std::max(s4, s5));
  return HPR_OK;
}

Layout make_layout(const hpr_dims &d, size_t cub_bytes) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 16), 256);
    return o;
  };
  auto plan = [&](int64_t nrows) {
    PlanOff p;
    const int64_t nw = windows_of(nrows);
    const int64_t ns = nw * (kWindow / kSlice);
    p.slice_row = take(sizeof(int) * nw * kWindow);
    p.slice_len = take(sizeof(unsigned short) * nw * kWindow);
    p.slice_slots = take(sizeof(int) * (ns + 1));
    p.slice_ptr = take(sizeof(int) * (ns + 1));
    p.long_flag = take(sizeof(int) * nrows);
    p.long_rows = take(sizeof(int) * nrows);
    p.nsel = take(2 * sizeof(int));   // [selected long rows, compact slice prefix]
    return p;
  };
  L.pa = plan(d.m);
  L.pat = plan(d.n);
  L.sp = split_plan_of(d);
  if (L.sp.on) {
    L.sp.po = plan(L.sp.V);
    L.sp.vrp = take(sizeof(int) * (L.sp.V + 1));
    L.sp.psum = take(sizeof(double) * d.m);
  }
  auto cbplan = [&](int64_t rows, int64_t cols) {
    CbOff o;
    o.on = cb_wanted(rows, cols, d.nnz);
    if (!o.on) return o;
    o.G = (int)std::min<int64_t>(148 * 8, rows);     // placeholder upper bound, fixed at analyze
    o.NB = (int)((cols + kCbW - 1) / kCbW);
    const int64_t ng = (int64_t)o.G * o.NB;
    o.row_start = take(sizeof(int) * (o.G + 1));
    o.gstart = take(sizeof(int) * (ng + 1));
    o.gseg = take(sizeof(long long) * (ng + 1));
    o.rpb_base = take(sizeof(long long) * (ng + 1));
    return o;
  };
  L.ca = cbplan(d.m, d.n);
  L.cat = cbplan(d.n, d.m);
  auto stgplan = [&](int64_t rows, int64_t cols, bool transpose) {
    StgOff o = stg_plan_of(rows, cols, d.nnz, transpose);
    if (!o.on) return o;
    o.row_start = take(sizeof(int) * (kStgMaxG + 1));
    o.goff = take(sizeof(long long) * ((size_t)kStgMaxG * o.NB + 1));
    return o;
  };
  L.sa = L.ca.on ? StgOff{} : stgplan(d.m, d.n, false);
  L.sat = L.cat.on ? StgOff{} : stgplan(d.n, d.m, true);
  if (L.sa.on || L.sat.on) {
    const int64_t it = std::max(L.sa.items, L.sat.items);
    const int64_t ng = (int64_t)kStgMaxG * std::max(L.sa.NB, L.sat.NB) + 1;
    L.stg_key = take(sizeof(unsigned) * it);
    L.stg_lrow = take(sizeof(int) * it);
    L.stg_skey = take(sizeof(unsigned) * it);
    L.stg_slrow = take(sizeof(int) * it);
    L.stg_gstart = take(sizeof(long long) * (ng + 1));
    L.stg_rbytes = take(sizeof(long long) * (ng + 1));
    L.stg_flag = take(sizeof(int));
  }
  if (L.ca.on || L.cat.on) {
    L.cb_key = take(sizeof(int) * d.nnz);
    L.cb_lrow = take(sizeof(int) * d.nnz);
  }
  L.keys_out = take(sizeof(int) * d.nnz);
  L.iota = take(sizeof(int) * d.nnz);
  L.row_of = take(sizeof(int) * d.nnz);
  L.cub_bytes = cub_bytes;
  L.cub_tmp = take(cub_bytes);
  L.dvec_m = take(sizeof(double) * d.m);
  L.dvec_n = take(sizeof(double) * d.n);
  // per-CTA partials of the SELL kernels (<= kMaxGridPerSm CTAs per SM, <= 1024 SMs):
  // x_half 2, y_half 2, merit 2, kkt_row 3, kkt_col 8, pow_t 1, pow_a 2 (= 20),
  // plus 4 sum-of-squares passes of up to kSumsqBlocks CTAs
  L.part_count = (size_t)20 * kMaxGridPerSm * 1024 + 4 * kSumsqBlocks;
  L.part = take(sizeof(double) * L.part_count);
  L.params = take(sizeof(IterParams));
  L.pow = take(sizeof(PowState));
  L.results = take(sizeof(double) * 64);
  L.fac = take(sizeof(double) * 2);
  L.flags = take(sizeof(unsigned int) * 4);
  L.total = off;
  return L;
}

int grid_for(int64_t n, int threads = 256, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// one matrix in SELL form
struct Sell {
  int nrows = 0, nslices = 0, nlong = 0;
  long long slots = 0;
  unsigned short *slice_len = nullptr;
  int *slice_row = nullptr, *slice_slots = nullptr, *slice_ptr = nullptr, *long_flag = nullptr,
      *long_rows = nullptr, *nsel = nullptr;
  int *ci = nullptr, *pos = nullptr;
  double *val_s = nullptr, *val0 = nullptr;
  bool affinity = false;   // rows in the row-affinity order (row_affinity_order)
  int compact = 0;         // leading compact slices (SellMat::compact)
};

}  // namespace

struct hpr_ctx {
  hpr_dims d{};
  int device = 0;
  cudaStream_t stream = nullptr;
  hpr_buffers B{};
  bool bound = false, analyzed = false, laid_out = false, scaled = false;
  char *ws = nullptr;
  Layout L{};
  Sell sa, sat;
  struct Split {
    bool on = false;
    int NB = 1, W = 0, m_pad = 0, S_m = 0;   // S_m: slices per block
    int *vrp = nullptr;
    double *psum = nullptr;
    Sell S;
  } sp;
  struct Cb {
    bool on = false;
    int G = 0, NB = 0, rows_cap = 0, seg_cap = 0, smem = 0, stages = 2;
    long long npad = 0, nrpb = 0;
    int *row_start = nullptr, *gstart = nullptr, *rpb = nullptr;
    long long *gseg = nullptr, *rpb_base = nullptr, *pos = nullptr;
    unsigned short *ci = nullptr;
    double *val = nullptr;
  } cba, cbat;
  struct Stg {
    bool on = false;
    int G = 0, NB = 0, rows_cap = 0, rec_cap = 0, stages = 2, smem = 0;
    long long rec_total = 0;
    int *row_start = nullptr, *pos = nullptr;
    long long *goff = nullptr;
    unsigned char *rec = nullptr;
  } sta, stat;
  const Stg *stg_sorted = nullptr;   // whose sorted items the STG temporaries hold
  // TS engine (hpr_tsell.cuh) for the iteration phases: block cuts of A
  // (ts_blk[0 .. ts_nb_a]) and A^T (ts_blk + ts_nb_a + 1), ctx-owned
  int *ts_blk = nullptr;               // in the caller's layout buffer (ts_bytes)
  long long ts_T[2] = {0, 0};          // block weight targets (0: TS off for A / A^T)
  long long ts_cap_n[2] = {0, 0};      // reserved list entries
  int ts_nb_a = 0, ts_nb_at = 0;
  // TS index words (SellMat::aw / aptr) of A / A^T, in the layout buffer after
  // the block lists: reserved at hpr_analyze (ts_aw_cap words, 0: off), filled
  // at hpr_bind_layout (ts_aw_words used)
  long long ts_aw_cap[2] = {0, 0}, ts_aw_words[2] = {0, 0};
  int *ts_aw[2] = {nullptr, nullptr}, *ts_aptr[2] = {nullptr, nullptr};
  // small-LP loop staging (small_smem_plan): cluster size it was planned for,
  // per-CTA slot capacity of A^T / A, dynamic shared-memory bytes
  int small_G = -1, small_cap[2] = {0, 0}, small_smem = 0;
  bool ts_a = false, ts_at = false;
  // row-block column chunks of A^T (slices per chunk, 0: one range): the A^T
  // plan is then cut per chunk, chunk q = blocks [ts_at_off[q], ts_at_off[q+1])
  int ts_chunk_sl = 0;
  std::vector<int> ts_at_off;
  int num_sms = 148;
  double *part = nullptr, *results = nullptr, *fac = nullptr, *dvec_m = nullptr, *dvec_n = nullptr;
  IterParams *params = nullptr;
  PowState *pow = nullptr;
  unsigned int *flags = nullptr;
  int bounds_uniform = 0;          // see EpiXIter
  int keep_a = 0, keep_at = 0;     // L2 policy of the A / A^T streams (SellMat::keep)
  // persisting-L2 window on the dual iterate y (HPR_L2WIN): attached to the
  // inner-loop SELL launches while they are captured (l2win_active)
  bool l2win_active = false;
  cudaAccessPolicyWindow l2win{};
  double lo_u = 0.0, up_u = 0.0;
  double *h_results = nullptr;       // pinned
  IterParams *h_params = nullptr;    // pinned
  PowState *h_pow = nullptr;         // pinned
  std::map<int, cudaGraphExec_t> inner_graphs;
  // exact T1 = 0 path (hpr_exact.cuh): the inverse factor and scratch vectors,
  // and its own per-interval graphs
  struct Exact {
    bool on = false;
    const double *linv = nullptr, *linv_t = nullptr;
    double *u = nullptr, *rhs = nullptr, *h = nullptr;
    std::map<int, cudaGraphExec_t> graphs;
  } exa;
  void drop_inner_graphs() {
    for (auto &kv : inner_graphs) cudaGraphExecDestroy(kv.second);
    inner_graphs.clear();
    for (auto &kv : exa.graphs) cudaGraphExecDestroy(kv.second);
    exa.graphs.clear();
  }
  cudaGraphExec_t pow_graph = nullptr;
  std::vector<long long> graph_sig;   // layout identity the graphs were captured against
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  bool inner_timed = false, ckpt_timed = false;
  long long launches = 0;

  SellMat mat(const Sell &S, const int *rp, const int *ci, const double *csr_val, bool scaled) const {
    const int ga = S.nslices > 0 && S.slots >= (long long)HPR_GA_MIN * 32 * S.nslices;
    return SellMat{S.slice_ptr, S.slice_row, S.slice_len, S.ci, scaled ? S.val_s : S.val0, rp, ci, csr_val,
                   S.long_rows, S.nslices, S.nlong, ga, 0, HPR_COMPACT_HDR ? S.compact : 0};
  }
  CbMat cbmat(const Cb &C, int ncols) const {
    return CbMat{C.row_start, C.gseg, C.rpb, C.rpb_base, C.ci, C.val, C.G, C.NB, kCbW, ncols,
                 C.rows_cap, C.seg_cap, C.stages};
  }
  StgMat stgmat(const Stg &T, int ncols) const {
    return StgMat{T.row_start, T.goff, T.rec, T.G, T.NB, ncols, T.rows_cap, T.rec_cap, T.stages};
  }
  SellMat mat_a(bool scaled) const {
    SellMat M = mat(sa, B.a_rp, B.a_ci, scaled ? B.a_val_s : B.a_val, scaled);
    M.keep = keep_a;
    return M;
  }
  // block b of the column-split A (scaled values; iteration y-phase only)
  SellMat mat_split(int b) const {
    const Sell &S = sp.S;
    const size_t so = (size_t)b * sp.S_m;
    SellMat M{S.slice_ptr + so, S.slice_row + so * kSlice, S.slice_len + so * kSlice, S.ci, S.val_s,
              nullptr, nullptr, nullptr, nullptr, sp.S_m, 0, 0, keep_a};
    M.ga = (long long)(S.slots) >= (long long)HPR_GA_MIN * 32 * S.nslices;
    return M;
  }
  SellMat mat_at(bool scaled) const {
    SellMat M = mat(sat, B.at_rp, B.at_ci, scaled ? B.at_val_s : B.at_val, scaled);
    M.keep = keep_at;
    return M;
  }
};

namespace {

// Launch the SELL kernel for epilogue Epi: grid = min(windows, occupancy x SMs);
// returns the grid (= partials per quantity).
template <int U, bool GA, class Epi>
int launch_sell_u(hpr_ctx *c, const SellMat &M, const double *xg, const Epi &epi, double *part,
                  int *grid_out, bool pdl) {
  int occ = 0;
  {
    const void *kf = (const void *)k_sell<U, GA, Epi>;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int &o = g_attr[{kf, c->device}];
    if (o == 0) {
      if (HPR_CARVEOUT >= 0)   // shared-memory carve-out: 0 = the whole unified array as L1
        CK(cudaFuncSetAttribute(k_sell<U, GA, Epi>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                HPR_CARVEOUT));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sell<U, GA, Epi>, kThreads, 0));
      if (o < 1) return fail(HPR_ECUDA, "SELL kernel does not fit on an SM");
      o = std::min(o, kMaxGridPerSm);
    }
    occ = o;
  }
  const int nwin = (M.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  const int grid = std::max(1, std::min(nwin, occ * c->num_sms));
  if ((pdl && HPR_PDL) || c->l2win_active) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl && HPR_PDL) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (c->l2win_active) {
      at[na].id = cudaLaunchAttributeAccessPolicyWindow;
      at[na++].val.accessPolicyWindow = c->l2win;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, k_sell<U, GA, Epi>, M, xg, epi, part));
  } else {
    k_sell<U, GA, Epi><<<grid, kThreads, 0, c->stream>>>(M, xg, epi, part);
  }
  CKL();
  c->launches += 1;
  if (grid_out) *grid_out = grid;
  return HPR_OK;
}

// entries in flight per lane follow the matrix's average row length
template <class Epi>
int launch_sell(hpr_ctx *c, const SellMat &M, const double *xg, const Epi &epi, double *part,
                int *grid_out, bool pdl = false) {
  return M.ga ? launch_sell_u<HPR_GA_U, true>(c, M, xg, epi, part, grid_out, pdl)
              : launch_sell_u<HPR_SELL_U, false>(c, M, xg, epi, part, grid_out, pdl);
}

// The y-phase product A w with the phase epilogue: one SELL launch, or NB
// launches over the column-split layout carrying the running sums.
template <class Epi>
int launch_a_iter(hpr_ctx *c, const double *wg, const Epi &epi, bool pdl) {
  if (!c->sp.on) return launch_sell(c, c->mat_a(true), wg, epi, nullptr, nullptr, pdl);
  for (int b = 0; b + 1 < c->sp.NB; ++b) {
    EpiCarry ec{};
    ec.psum = c->sp.psum;
    ec.first = b == 0;
    int rc = launch_sell(c, c->mat_split(b), wg, ec, nullptr, nullptr, pdl && b == 0);
    if (rc) return rc;
  }
  EpiCarryIn<Epi> el{};
  static_cast<Epi &>(el) = epi;
  el.psum = c->sp.psum;
  return launch_sell(c, c->mat_split(c->sp.NB - 1), wg, el, nullptr, nullptr, false);
}

// parts layout inside ctx->part (in doubles)
struct Parts {
  double *xhalf, *yhalf, *merit, *krow, *kcol, *powt, *powa, *misc;
};
Parts parts_of(const hpr_ctx *c) {
  const size_t g = (size_t)kMaxGridPerSm * 1024;
  Parts p;
  p.xhalf = c->part;
  p.yhalf = p.xhalf + 2 * g;
  p.merit = p.yhalf + 2 * g;
  p.krow = p.merit + 2 * g;
  p.kcol = p.krow + 3 * g;
  p.powt = p.kcol + 8 * g;
  p.powa = p.powt + 1 * g;
  p.misc = p.powa + 2 * g;
  return p;
}

int sumsq_blocks(int64_t n) { return grid_for(n, kThreads, kSumsqBlocks); }

// Row affinity order of a matrix whose gathered vector (ncols doubles) does
// not fit in L2 (k_row_mode_block): rows stably radix-sorted by the column block
// holding most of their entries.  Scratch: keys_out / row_of (nnz ints each,
// free once the transpose is built); needs nnz >= 2 nrows.  Returns the order
// (row_of + nrows) or nullptr when not used.  HPR_RAO (A) / HPR_RAO_AT (A^T)
// = 0 / 1 force it off / on; HPR_RAO_BITS sets the block width (default 2^20
// columns = 8 MB of the vector).
const int *row_affinity_order(hpr_ctx *c, const int *rp, const int *ci, int nrows, int64_t ncols,
                              bool transpose, int *rc) {
  *rc = HPR_OK;
  const char *env = getenv(transpose ? "HPR_RAO_AT" : "HPR_RAO");
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
  bool want = 8.0 * (double)ncols > (double)l2;
  if (env && env[0] == '0') want = false;
  if (env && env[0] == '1') want = true;
  if (!want || nrows < 2 || c->d.nnz < 2 * (int64_t)nrows) return nullptr;
  int bits = 20;   // C3 sweep (us/iteration): 12: 976, 14: 981, 16: 942, 18: 919, 20: 916, 22: 921, off: 946
  if (const char *eb = getenv("HPR_RAO_BITS")) bits = std::max(0, std::min(30, atoi(eb)));
  int *key = (int *)(c->ws + c->L.keys_out), *skey = key + nrows;
  int *iota = (int *)(c->ws + c->L.row_of), *order = iota + nrows;
  cudaStream_t s = c->stream;
  k_row_mode_block<<<grid_for(nrows), 256, 0, s>>>(rp, ci, nrows, bits, key);
  k_iota<<<grid_for(nrows), 256, 0, s>>>(iota, nrows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *rc = fail(HPR_ECUDA, std::string("row affinity: ") + cudaGetErrorString(e));
    return nullptr;
  }
  int end_bit = 1;
  while (end_bit < 31 && (1LL << end_bit) <= ((ncols - 1) >> bits)) ++end_bit;
  size_t tb = c->L.cub_bytes;
  e = cub::DeviceRadixSort::SortPairs(c->ws + c->L.cub_tmp, tb, key, skey, iota, order, nrows, 0,
                                      end_bit, s);
  if (e != cudaSuccess) {
    *rc = fail(HPR_ECUDA, std::string("row affinity sort: ") + cudaGetErrorString(e));
    return nullptr;
  }
  c->launches += 3;
  return order;
}

// SELL plan of one matrix: slice order, slot offsets, long-row list
int plan_sell(hpr_ctx *c, const PlanOff &po, const int *rp, int nrows, Sell &S,
              int long_thresh = kLongRow, int m_pad = 0, int m_real = 0,
              const int *order = nullptr) {
  S.nrows = nrows;
  const int nw = (int)windows_of(nrows);
  S.nslices = nw * (kWindow / kSlice);
  const int win = sort_win(m_pad ? m_pad : nrows);   // split plans: the real row count
  S.slice_row = (int *)(c->ws + po.slice_row);
  S.slice_len = (unsigned short *)(c->ws + po.slice_len);
  S.slice_slots = (int *)(c->ws + po.slice_slots);
  S.slice_ptr = (int *)(c->ws + po.slice_ptr);
  S.long_flag = (int *)(c->ws + po.long_flag);
  S.long_rows = (int *)(c->ws + po.long_rows);
  S.nsel = (int *)(c->ws + po.nsel);
  cudaStream_t s = c->stream;
  CK(cudaMemsetAsync(S.slice_slots + S.nslices, 0, sizeof(int), s));
  k_fill_int<<<1, 1, 0, s>>>(S.nsel + 1, 1, S.nslices);   // compact prefix: min over slices
  CKL();
  if (win == kSortWinBig)
    k_sell_plan<kSortWinBig><<<(nrows + win - 1) / win, win, 0, s>>>(
        rp, nrows, 1, S.slice_row, S.slice_len, S.slice_slots, S.long_flag, long_thresh, m_pad,
        m_real, order, S.nsel + 1);
  else
    k_sell_plan<kWindow><<<nw, kWindow, 0, s>>>(rp, nrows, 1, S.slice_row, S.slice_len,
                                                S.slice_slots, S.long_flag, long_thresh, m_pad,
                                                m_real, order, S.nsel + 1);
  S.affinity = order != nullptr;
  CKL();
  size_t tb = c->L.cub_bytes;
  CK(cub::DeviceScan::ExclusiveSum(c->ws + c->L.cub_tmp, tb, S.slice_slots, S.slice_ptr,
                                   S.nslices + 1, s));
  tb = c->L.cub_bytes;
  CK(cub::DeviceSelect::Flagged(c->ws + c->L.cub_tmp, tb, cub::CountingInputIterator<int>(0),
                                S.long_flag, S.long_rows, S.nsel, nrows, s));
  c->launches += 3;
  int total = 0, nl[2] = {0, 0};
  CK(cudaMemcpyAsync(&total, S.slice_ptr + S.nslices, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(nl, S.nsel, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (total < 0) return fail(HPR_EINVAL, "SELL slot count overflows int32");
  S.slots = total;
  S.nlong = nl[0];
  S.compact = (m_pad == 0 && !order) ? nl[1] : 0;
  return HPR_OK;
}

// ---- STG engine: items, plan (hpr_analyze), layout (hpr_bind_layout) ----
// (CTA, chunk, row) items of the rows, stably sorted by (CTA, chunk, count
// desc); group starts into L.stg_gstart
int stg_sort(hpr_ctx *c, const hpr_ctx::Stg &T, const int *rp, const int *ci, int rows) {
  cudaStream_t s = c->stream;
  const Layout &L = c->L;
  unsigned *key = (unsigned *)(c->ws + L.stg_key), *skey = (unsigned *)(c->ws + L.stg_skey);
  int *lrow = (int *)(c->ws + L.stg_lrow), *slrow = (int *)(c->ws + L.stg_slrow);
  long long *gstart = (long long *)(c->ws + L.stg_gstart);
  const long long items = (long long)rows * T.NB;
  const int ng = T.G * T.NB;
  k_stg_items<<<grid_for(rows), 256, 0, s>>>(rp, ci, rows, T.row_start, T.G, T.NB, key, lrow,
                                             (int *)(c->ws + L.stg_flag));
  CKL();
  int end_bit = 17;
  while ((1LL << (end_bit - 16)) < ng) ++end_bit;
  size_t tb = L.cub_bytes;
  CK(cub::DeviceRadixSort::SortPairs(c->ws + L.cub_tmp, tb, key, skey, lrow, slrow, (int)items, 0,
                                     end_bit, s));
  k_stg_gstart<<<grid_for(items), 256, 0, s>>>(skey, items, ng, gstart);
  CKL();
  c->launches += 3;
  c->stg_sorted = &T;
  return HPR_OK;
}

int stg_plan(hpr_ctx *c, const StgOff &o, const int *rp, const int *ci, int rows,
             hpr_ctx::Stg &T) {
  T = hpr_ctx::Stg{};
  if (!o.on || c->d.nnz == 0 || c->num_sms > kStgMaxG) return HPR_OK;
  cudaStream_t s = c->stream;
  const Layout &L = c->L;
  T.G = std::min(c->num_sms, rows);
  T.NB = o.NB;
  T.row_start = (int *)(c->ws + o.row_start);
  T.goff = (long long *)(c->ws + o.goff);
  k_cb_rowstart<<<1, 256, 0, s>>>(rp, rows, T.G, T.row_start);
  CKL();
  CK(cudaMemsetAsync(c->ws + L.stg_flag, 0, sizeof(int), s));
  c->launches += 1;
  int rc = stg_sort(c, T, rp, ci, rows);
  if (rc) return rc;
  const int ng = T.G * T.NB;
  long long *rbytes = (long long *)(c->ws + L.stg_rbytes);
  k_stg_recsize<<<(ng + 127) / 128, 128, 0, s>>>((unsigned *)(c->ws + L.stg_skey),
                                                 (long long *)(c->ws + L.stg_gstart), ng, rbytes);
  CKL();
  CK(cudaMemsetAsync(rbytes + ng, 0, sizeof(long long), s));
  size_t tb = L.cub_bytes;
  CK(cub::DeviceScan::ExclusiveSum(c->ws + L.cub_tmp, tb, rbytes, T.goff, ng + 1, s));
  c->launches += 2;
  std::vector<int> hrs(T.G + 1);
  std::vector<long long> hgo(ng + 1);
  int flag = 0;
  CK(cudaMemcpyAsync(hrs.data(), T.row_start, sizeof(int) * (T.G + 1), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hgo.data(), T.goff, sizeof(long long) * (ng + 1), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&flag, c->ws + L.stg_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int g = 0; g < T.G; ++g) T.rows_cap = std::max(T.rows_cap, hrs[g + 1] - hrs[g]);
  long long rc_max = 0;
  for (int q = 0; q < ng; ++q) rc_max = std::max(rc_max, hgo[q + 1] - hgo[q]);
  T.rec_total = hgo[ng];
  T.rec_cap = (int)std::min<long long>(rc_max, INT_MAX / 2);
  T.stages = kStgMaxStages;
  while (T.stages > 2 && stg_smem_bytes(T.stages, T.rows_cap, T.rec_cap) > kCbMaxSmem) --T.stages;
  T.smem = stg_smem_bytes(T.stages, T.rows_cap, T.rec_cap);
  T.on = !flag && rc_max <= kCbMaxSmem && T.smem <= kCbMaxSmem && T.rows_cap < (int)kStgPad &&
         T.rec_total / 8 < INT_MAX;
  return HPR_OK;
}

size_t stg_bytes(const hpr_ctx::Stg &T, int64_t nnz) {
  if (!T.on) return 0;
  return align_up((size_t)T.rec_total + 256, 256) + align_up((size_t)nnz * 4 + 256, 256);
}

int stg_layout(hpr_ctx *c, char *&p, hpr_ctx::Stg &T, const int *rp, const int *ci, int rows) {
  if (!T.on) return HPR_OK;
  cudaStream_t s = c->stream;
  const long long nnz = c->d.nnz;
  T.rec = (unsigned char *)p;
  p += align_up((size_t)T.rec_total + 256, 256);
  T.pos = (int *)p;
  p += align_up((size_t)nnz * 4 + 256, 256);
  CK(cudaMemsetAsync(T.rec, 0, (size_t)T.rec_total, s));
  if (c->stg_sorted != &T) {          // hpr_analyze's sort of this matrix was overwritten
    int rc = stg_sort(c, T, rp, ci, rows);
    if (rc) return rc;
  }
  const int ng = T.G * T.NB;
  const size_t sh = sizeof(int) * ((size_t)T.rows_cap / 32 + 3);
  k_stg_fill<<<ng, 256, sh, s>>>(rp, ci, T.row_start, T.NB, (unsigned *)(c->ws + c->L.stg_skey),
                                 (int *)(c->ws + c->L.stg_slrow),
                                 (long long *)(c->ws + c->L.stg_gstart), T.goff, T.rec, T.pos);
  CKL();
  c->launches += 1;
  return HPR_OK;
}

// TS engine for the iteration phases (hpr_tsell.cuh): HPR_TS=0 never, 1
// whenever the SELL kernel would run, 2 (auto) when the matrix stream does not
// fit in L2.  A matrix qualifies when its largest slice leaves a block target
// T of at least a quarter of a stage.  ts_select (hpr_analyze) decides and
// sizes the block lists -- they live in the caller's layout buffer -- and
// ts_plan (hpr_bind_layout, and again when a row-block group cuts A^T into
// column chunks) fills them.
constexpr int kTsMaxChunks = 64;   // A^T column chunks the reserved block list covers
int ts_select(hpr_ctx *c) {
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
  const char *env = getenv("HPR_TS");
  const int mode_all = env ? atoi(env) : HPR_TS_DEFAULT;
  cudaStream_t s = c->stream;
  const Sell *SS[2] = {&c->sa, &c->sat};
  const bool other[2] = {c->sp.on || c->sta.on || c->cba.on, c->stat.on || c->cbat.on};
  for (int q = 0; q < 2; ++q) {
    c->ts_T[q] = 0;
    c->ts_cap_n[q] = 0;
    const Sell &S = *SS[q];
    const char *em = getenv(q ? "HPR_TS_AT" : "HPR_TS_A");   // per-matrix override
    const int mode = em ? atoi(em) : mode_all;
    if (mode == 0 || S.nslices == 0 || other[q]) continue;
    // auto: a matrix stream larger than L2 with short rows (<= 8 slots per lane
    // on average), mostly in compact slices.  C3 (us/iteration): A^T (3 per
    // row, compact) on TS 997 -> 849; A (10.7 per row, HBM gathers of w) on TS
    // is slower (+52); C4's A_g^T (6.25 per row, sigma-sorted, 28 % padding)
    // too (1668 -> 1896 us per rank iteration): both stay on k_sell
    if (mode != 1 && (12.0 * (double)S.slots <= (double)l2 || S.slots > 8LL * kSlice * S.nslices ||
                      2LL * S.compact < S.nslices))
      continue;
    int *dmax = (int *)c->part;   // scratch: no partials are live during analysis
    size_t tb = c->L.cub_bytes;
    CK(cub::DeviceReduce::Max(c->ws + c->L.cub_tmp, tb, S.slice_slots, dmax, S.nslices, s));
    int mx = 0;
    CK(cudaMemcpyAsync(&mx, dmax, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->launches += 1;
    const long long t = (long long)kTsCap - mx - kTsSw;
    if (t < kTsCap / 4) continue;
    c->ts_T[q] = t;
    const long long nb = (S.slots + (long long)kTsSw * S.nslices + t - 1) / t;
    // entries: nb + 1 for one range; per column chunk at most one more block
    // and one end entry each (A^T in the row-block overlap path)
    c->ts_cap_n[q] = nb + 1 + (q ? 2LL * kTsMaxChunks : 0);
    // index words (hpr_tsell.cuh): worst case one word per slot
    const char *ea = getenv("HPR_TS_AW");
    c->ts_aw_cap[q] = (ea ? atoi(ea) : HPR_TS_AW) ? S.slots + 16 : 0;
  }
  return HPR_OK;
}

size_t ts_aw_bytes(const hpr_ctx *c, int q) {
  const Sell &S = q ? c->sat : c->sa;
  if (c->ts_T[q] <= 0 || c->ts_aw_cap[q] <= 0) return 0;
  return align_up(sizeof(int) * (size_t)(S.nslices + 16), 256) +
         align_up(sizeof(int) * (size_t)c->ts_aw_cap[q], 256);
}

size_t ts_bytes(const hpr_ctx *c) {
  return align_up(sizeof(int) * (size_t)(c->ts_cap_n[0] + c->ts_cap_n[1]) + 16, 256) +
         ts_aw_bytes(c, 0) + ts_aw_bytes(c, 1);
}

// Fill the TS index words of A (q = 0) / A^T (q = 1) from the laid-out SELL
// column indices: per slice, one word per entry when every entry's 32 lane
// columns are lane-affine or lane-uniform, else the slot words unchanged.
int ts_aw_layout(hpr_ctx *c, char *base) {
  cudaStream_t s = c->stream;
  char *p = base + align_up(sizeof(int) * (size_t)(c->ts_cap_n[0] + c->ts_cap_n[1]) + 16, 256);
  for (int q = 0; q < 2; ++q) {
    c->ts_aw[q] = c->ts_aptr[q] = nullptr;
    c->ts_aw_words[q] = 0;
    if (ts_aw_bytes(c, q) == 0) continue;
    const Sell &S = q ? c->sat : c->sa;
    int *aptr = (int *)p;
    p += align_up(sizeof(int) * (size_t)(S.nslices + 16), 256);
    int *aw = (int *)p;
    p += align_up(sizeof(int) * (size_t)c->ts_aw_cap[q], 256);
    CK(cudaMemsetAsync(aptr, 0, sizeof(int) * (size_t)(S.nslices + 16), s));
    const long long thr = 32LL * (S.nslices + 1);
    k_aw_count<<<(unsigned)((thr + 255) / 256), 256, 0, s>>>(S.slice_ptr, S.ci, S.nslices, aptr);
    CKL();
    size_t tb = c->L.cub_bytes;
    CK(cub::DeviceScan::ExclusiveSum(c->ws + c->L.cub_tmp, tb, aptr, aptr, S.nslices + 1, s));
    int total = 0;
    CK(cudaMemcpyAsync(&total, aptr + S.nslices, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (total + 16 > c->ts_aw_cap[q]) return fail(HPR_EINVAL, "TS index words exceed their reservation");
    CK(cudaMemsetAsync(aw, 0, sizeof(int) * (size_t)(total + 16), s));
    k_aw_fill<<<(unsigned)((thr + 255) / 256), 256, 0, s>>>(S.slice_ptr, S.ci, S.nslices, aptr, aw);
    CKL();
    c->launches += 3;
    c->ts_aw[q] = aw;
    c->ts_aptr[q] = aptr;
    c->ts_aw_words[q] = total;
  }
  return HPR_OK;
}

int ts_plan(hpr_ctx *c) {
  cudaStream_t s = c->stream;
  const long long *T = c->ts_T;
  int nb[2] = {0, 0};
  if (T[0] > 0) nb[0] = (int)((c->sa.slots + (long long)kTsSw * c->sa.nslices + T[0] - 1) / T[0]);
  // A^T in chunks (row-block overlap path): block counts per chunk from the
  // chunk boundaries' slot offsets
  std::vector<int> off_at(2, 0), lo_at(1, 0), hi_at(1, c->sat.nslices);
  if (T[1] > 0) {
    const Sell &S = c->sat;
    int cs = c->ts_chunk_sl > 0 ? c->ts_chunk_sl : S.nslices;
    if ((S.nslices + cs - 1) / cs > kTsMaxChunks) {   // not reserved: whole-matrix plan only
      c->ts_chunk_sl = 0;
      cs = S.nslices;
    }
    const int kc = (S.nslices + cs - 1) / cs;
    std::vector<int> bnd(kc + 1);
    for (int q = 0; q <= kc; ++q) bnd[q] = std::min(S.nslices, q * cs);
    std::vector<int> sp(kc + 1);
    for (int q = 0; q <= kc; ++q)
      CK(cudaMemcpyAsync(&sp[q], S.slice_ptr + bnd[q], sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    off_at.assign(kc + 1, 0);
    lo_at.assign(kc, 0);
    hi_at.assign(kc, 0);
    for (int q = 0; q < kc; ++q) {
      const long long wq = (long long)(sp[q + 1] - sp[q]) + (long long)kTsSw * (bnd[q + 1] - bnd[q]);
      const int nq = bnd[q + 1] > bnd[q] ? (int)((wq + T[1] - 1) / T[1]) : 0;
      off_at[q + 1] = off_at[q] + nq + 1;   // + 1: the range's end entry
      lo_at[q] = bnd[q];
      hi_at[q] = bnd[q + 1];
    }
    nb[1] = off_at[kc] - 1;   // whole-matrix launches: one list (the end entries are empty blocks)
    if (off_at[kc] > c->ts_cap_n[1]) return fail(HPR_EINVAL, "TS block list exceeds its reservation");
  }
  const bool changed = (T[0] > 0) != c->ts_a || (T[1] > 0) != c->ts_at || nb[0] != c->ts_nb_a ||
                       nb[1] != c->ts_nb_at || off_at != c->ts_at_off;
  if (T[0] > 0)
    k_ts_plan<<<(nb[0] + 256) / 256, 256, 0, s>>>(c->sa.slice_ptr, 0, c->sa.nslices, T[0], nb[0],
                                                   c->ts_blk);
  if (T[1] > 0)
    for (size_t q = 0; q + 1 < off_at.size(); ++q) {
      const int nq = off_at[q + 1] - off_at[q] - 1;
      k_ts_plan<<<(nq + 256) / 256, 256, 0, s>>>(c->sat.slice_ptr, lo_at[q], hi_at[q], T[1], nq,
                                                  c->ts_blk + nb[0] + 1 + off_at[q]);
      c->launches += 1;
    }
  CKL();
  c->launches += (int)(T[0] > 0);
  if (changed) {   // the captured inner-loop and power graphs hold the plan
    c->drop_inner_graphs();
    if (c->pow_graph) {
      cudaGraphExecDestroy(c->pow_graph);
      c->pow_graph = nullptr;
    }
  }
  c->ts_a = T[0] > 0;
  c->ts_at = T[1] > 0;
  c->ts_nb_a = nb[0];
  c->ts_nb_at = nb[1];
  c->ts_at_off = off_at;
  return HPR_OK;
}

// the TS x-phase streams its row operands and results evict-first (compact
// slices: whole warp segments), so the gathered y keeps the L2 (HPR_TS_EF)
#ifndef HPR_TS_EF
#define HPR_TS_EF 1
#endif
#ifndef HPR_Y_EF
#define HPR_Y_EF 1
#endif
EpiXIter ts_ef(EpiXIter e) {
  // walking the blocks last to first (HPR_TS_REV), the w written last is the
  // start of the y-phase's gather order: kept (normal stores), not evict-first
  e.ef = HPR_TS_EF ? (HPR_TS_REV ? 1 : 3) : 0;
  return e;
}

template <class Epi>
int launch_ts(hpr_ctx *c, const SellMat &M0, const int *blk, int nblk, const double *xg,
              const Epi &epi) {
  SellMat M = M0;   // the matrix's index words, when laid out
  for (int q = 0; q < 2; ++q)
    if (c->ts_aw[q] && M.slice_ptr == (q ? c->sat : c->sa).slice_ptr) {
      M.aw = c->ts_aw[q];
      M.aptr = c->ts_aptr[q];
    }
  if (M.aw) {
    if (int e = ensure_dyn_smem(k_tsell<HPR_TS_U_AW, Epi, true>, kTsSmem)) return e;
    k_tsell<HPR_TS_U_AW, Epi, true><<<c->num_sms * kTsCps, kTsThreads, kTsSmem, c->stream>>>(
        M, xg, epi, blk, nblk);
  } else {
    if (int e = ensure_dyn_smem(k_tsell<HPR_TS_U, Epi, false>, kTsSmem)) return e;
    k_tsell<HPR_TS_U, Epi, false><<<c->num_sms * kTsCps, kTsThreads, kTsSmem, c->stream>>>(
        M, xg, epi, blk, nblk);
  }
  CKL();
  c->launches += 1;
  return HPR_OK;
}

template <class Epi>
int launch_stg(hpr_ctx *c, const hpr_ctx::Stg &T, int ncols, const double *xg, const Epi &epi) {
  if (int e = ensure_dyn_smem(k_stg<Epi>, T.smem)) return e;
  k_stg<Epi><<<T.G, kStgThreads, T.smem, c->stream>>>(c->stgmat(T, ncols), xg, epi);
  CKL();
  c->launches += 1;
  return HPR_OK;
}

// ---- column-split layout of A (SplitOff): plan at hpr_analyze ----
int split_plan(hpr_ctx *c) {
  hpr_ctx::Split &P = c->sp;
  P = hpr_ctx::Split{};
  const SplitOff &o = c->L.sp;
  if (!o.on) return HPR_OK;
  cudaStream_t s = c->stream;
  P.NB = o.NB;
  P.W = o.W;
  P.m_pad = o.m_pad;
  P.S_m = o.m_pad / kSlice;
  P.vrp = (int *)(c->ws + o.vrp);
  P.psum = (double *)(c->ws + o.psum);
  k_split_count<<<grid_for(o.m_pad), 256, 0, s>>>(c->B.a_rp, c->B.a_ci, (int)c->d.m, o.m_pad, o.W,
                                                  o.NB, P.vrp);
  CKL();
  CK(cudaMemsetAsync(P.vrp + o.V, 0, sizeof(int), s));
  size_t tb = c->L.cub_bytes;
  CK(cub::DeviceScan::ExclusiveSum(c->ws + c->L.cub_tmp, tb, P.vrp, P.vrp, (int)o.V + 1, s));
  c->launches += 2;
  // every virtual row stays in the slices (lengths <= 65535); otherwise no split
  int rc = plan_sell(c, o.po, P.vrp, (int)o.V, P.S, 65535, o.m_pad, (int)c->d.m);
  if (rc) return rc;
  if (P.S.nlong > 0) {
    P = hpr_ctx::Split{};
    return HPR_OK;
  }
  P.on = true;
  return HPR_OK;
}

size_t split_bytes(const hpr_ctx::Split &P, int64_t nnz) {
  if (!P.on) return 0;
  return align_up((size_t)P.S.slots * 4 + 256, 256) + align_up((size_t)P.S.slots * 8 + 256, 256) +
         align_up((size_t)nnz * 4 + 256, 256);
}

// ---- column-split layout: fill at hpr_bind_layout (scaled values at hpr_scale) ----
int split_layout(hpr_ctx *c, char *&p) {
  hpr_ctx::Split &P = c->sp;
  if (!P.on) return HPR_OK;
  Sell &S = P.S;
  const long long nnz = c->d.nnz;
  cudaStream_t s = c->stream;
  S.ci = (int *)p;
  p += align_up((size_t)S.slots * 4 + 256, 256);
  S.val_s = (double *)p;
  p += align_up((size_t)S.slots * 8 + 256, 256);
  S.pos = (int *)p;
  p += align_up((size_t)nnz * 4 + 256, 256);
  S.val0 = nullptr;
  CK(cudaMemsetAsync(S.ci, 0, (size_t)S.slots * 4, s));
  CK(cudaMemsetAsync(S.val_s, 0, (size_t)S.slots * 8, s));
  CK(cudaMemsetAsync(S.pos, 0xff, (size_t)nnz * 4, s));
  k_split_fill<<<grid_for((int64_t)S.nslices * 32), 256, 0, s>>>(
      c->B.a_rp, c->B.a_ci, P.vrp, S.slice_ptr, S.slice_row, S.nslices, P.m_pad, P.W, S.ci, S.pos);
  CKL();
  c->launches += 1;
  return HPR_OK;
}

size_t sell_bytes(const Sell &S, int64_t nnz) {
  return align_up((size_t)S.slots * 4 + 256, 256) + 2 * align_up((size_t)S.slots * 8 + 256, 256) +
         align_up((size_t)nnz * 4 + 256, 256);
}

int layout_sell(hpr_ctx *c, char *&p, Sell &S, const int *rp, const int *ci, const double *val0) {
  const long long nnz = c->d.nnz;
  cudaStream_t s = c->stream;
  S.ci = (int *)p;
  p += align_up((size_t)S.slots * 4 + 256, 256);
  S.val_s = (double *)p;
  p += align_up((size_t)S.slots * 8 + 256, 256);
  S.val0 = (double *)p;
  p += align_up((size_t)S.slots * 8 + 256, 256);
  S.pos = (int *)p;
  p += align_up((size_t)nnz * 4 + 256, 256);
  CK(cudaMemsetAsync(S.ci, 0, (size_t)S.slots * 4, s));
  CK(cudaMemsetAsync(S.val_s, 0, (size_t)S.slots * 8, s));
  CK(cudaMemsetAsync(S.val0, 0, (size_t)S.slots * 8, s));
  CK(cudaMemsetAsync(S.pos, 0xff, (size_t)nnz * 4, s));   // -1: long-row entries
  k_sell_fill<<<grid_for((int64_t)S.nslices * 32), 256, 0, s>>>(rp, ci, S.slice_ptr, S.slice_row,
                                                                S.nslices, S.ci, S.pos);
  CKL();
  if (nnz > 0) {
    k_sell_scatter<<<grid_for(nnz), 256, 0, s>>>(S.pos, val0, S.val0, nnz);
    CKL();
  }
  c->launches += 2;
  return HPR_OK;
}

// ---- CB engine: plan (hpr_analyze) and layout (hpr_bind_layout) ----
// keys + stable sort of the entries by (CTA, column block); leaves the sorted
// keys in L.keys_out, the permutation in L.row_of, local rows in L.cb_lrow
int cb_sort(hpr_ctx *c, const hpr_ctx::Cb &C, const int *rp, const int *ci) {
  cudaStream_t s = c->stream;
  const long long nnz = c->d.nnz;
  int *key = (int *)(c->ws + c->L.cb_key), *lrow = (int *)(c->ws + c->L.cb_lrow);
  int *skey = (int *)(c->ws + c->L.keys_out), *iota = (int *)(c->ws + c->L.iota);
  int *perm = (int *)(c->ws + c->L.row_of);
  k_cb_keys<<<C.G, 256, 0, s>>>(rp, ci, C.row_start, C.G, C.NB, kCbW, key, lrow);
  k_iota<<<grid_for(nnz), 256, 0, s>>>(iota, nnz);
  CKL();
  int end_bit = 1;
  while ((1LL << end_bit) < (long long)C.G * C.NB) ++end_bit;
  size_t tb = c->L.cub_bytes;
  CK(cub::DeviceRadixSort::SortPairs(c->ws + c->L.cub_tmp, tb, key, skey, iota, perm, (int)nnz, 0,
                                     end_bit, s));
  c->launches += 4;
  return HPR_OK;
}

int cb_plan(hpr_ctx *c, const CbOff &o, const int *rp, const int *ci, int rows, hpr_ctx::Cb &C) {
  C = hpr_ctx::Cb{};
  if (!o.on || c->d.nnz == 0) return HPR_OK;
  cudaStream_t s = c->stream;
  C.G = std::min(c->num_sms, rows);
  if (C.G > std::min<int64_t>(148 * 8, rows)) return HPR_OK;     // workspace sized for fewer
  C.NB = o.NB;
  C.row_start = (int *)(c->ws + o.row_start);
  C.gstart = (int *)(c->ws + o.gstart);
  C.gseg = (long long *)(c->ws + o.gseg);
  C.rpb_base = (long long *)(c->ws + o.rpb_base);
  k_cb_rowstart<<<1, 256, 0, s>>>(rp, rows, C.G, C.row_start);
  CKL();
  int rc = cb_sort(c, C, rp, ci);
  if (rc) return rc;
  const long long ng = (long long)C.G * C.NB;
  k_cb_count<<<grid_for(c->d.nnz), 256, 0, s>>>((int *)(c->ws + c->L.keys_out), c->d.nnz, (int)ng,
                                                C.gstart);
  k_cb_pad<<<1, 1, 0, s>>>(C.gstart, C.row_start, C.G, C.NB, C.gseg, C.rpb_base);
  CKL();
  c->launches += 3;
  std::vector<int> hrs(C.G + 1);
  std::vector<long long> hseg(ng + 1);
  CK(cudaMemcpyAsync(hrs.data(), C.row_start, sizeof(int) * (C.G + 1), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hseg.data(), C.gseg, sizeof(long long) * (ng + 1), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int g = 0; g < C.G; ++g) {
    const int rg = hrs[g + 1] - hrs[g];
    C.rows_cap = std::max(C.rows_cap, rg);
    C.nrpb += (long long)C.NB * ((rg + 1 + 3) / 4 * 4);
  }
  for (long long q = 0; q < ng; ++q) C.seg_cap = (int)std::max<long long>(C.seg_cap, hseg[q + 1] - hseg[q]);
  C.npad = hseg[ng];
  C.stages = kCbMaxStages;
  while (C.stages > 2 && cb_smem(kCbW, C.seg_cap, C.rows_cap, C.stages).total > kCbMaxSmem) --C.stages;
  C.smem = cb_smem(kCbW, C.seg_cap, C.rows_cap, C.stages).total;
  C.on = C.smem <= kCbMaxSmem && C.npad < INT_MAX && C.rows_cap <= kCbMaxRpt * kCbThreads;
  return HPR_OK;
}

size_t cb_bytes(const hpr_ctx::Cb &C, int64_t nnz) {
  if (!C.on) return 0;
  return align_up((size_t)C.npad * 8 + 256, 256) + align_up((size_t)C.npad * 2 + 256, 256) +
         align_up((size_t)C.nrpb * 4 + 256, 256) + align_up((size_t)nnz * 8 + 256, 256);
}

int cb_layout(hpr_ctx *c, char *&p, hpr_ctx::Cb &C, const int *rp, const int *ci) {
  if (!C.on) return HPR_OK;
  cudaStream_t s = c->stream;
  const long long nnz = c->d.nnz;
  C.val = (double *)p;
  p += align_up((size_t)C.npad * 8 + 256, 256);
  C.ci = (unsigned short *)p;
  p += align_up((size_t)C.npad * 2 + 256, 256);
  C.rpb = (int *)p;
  p += align_up((size_t)C.nrpb * 4 + 256, 256);
  C.pos = (long long *)p;
  p += align_up((size_t)nnz * 8 + 256, 256);
  CK(cudaMemsetAsync(C.val, 0, (size_t)C.npad * 8, s));
  CK(cudaMemsetAsync(C.ci, 0, (size_t)C.npad * 2, s));
  CK(cudaMemsetAsync(C.rpb, 0, (size_t)C.nrpb * 4, s));
  int rc = cb_sort(c, C, rp, ci);
  if (rc) return rc;
  const long long ng = (long long)C.G * C.NB;
  k_cb_empty<<<(int)ng, 128, 0, s>>>(C.gstart, C.rpb_base, C.row_start, C.G, C.NB, C.rpb);
  k_cb_fill<<<grid_for(nnz), 256, 0, s>>>((int *)(c->ws + c->L.keys_out), (int *)(c->ws + c->L.row_of),
                                          (int *)(c->ws + c->L.cb_lrow), ci, C.gstart, C.gseg,
                                          C.rpb_base, C.row_start, C.NB, kCbW, nnz, C.ci, C.rpb,
                                          C.pos);
  CKL();
  c->launches += 2;
  return HPR_OK;
}

template <int RPT, class Epi>
int launch_cb_r(hpr_ctx *c, const hpr_ctx::Cb &C, int ncols, const double *xg, const Epi &epi) {
  if (int e = ensure_dyn_smem(k_cb<RPT, Epi>, kCbMaxSmem)) return e;
  k_cb<RPT, Epi><<<C.G, kCbThreads + 32, C.smem, c->stream>>>(c->cbmat(C, ncols), xg, epi, nullptr);
  CKL();
  c->launches += 1;
  return HPR_OK;
}

template <class Epi>
int launch_cb(hpr_ctx *c, const hpr_ctx::Cb &C, int ncols, const double *xg, const Epi &epi) {
  const int rpt = (C.rows_cap + kCbThreads - 1) / kCbThreads;
  if (rpt <= 1) return launch_cb_r<1>(c, C, ncols, xg, epi);
  if (rpt == 2) return launch_cb_r<2>(c, C, ncols, xg, epi);
  if (rpt == 3) return launch_cb_r<3>(c, C, ncols, xg, epi);
  return launch_cb_r<4>(c, C, ncols, xg, epi);
}

// fixed-order final reduction of a list of partial segments into ctx->results
int reduce_final(hpr_ctx *c, const std::vector<RedSeg> &segs) {
  RedList L{};
  if (segs.size() > 24) return fail(HPR_EINVAL, "too many reduction segments");
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

// KKT kernels on the termination problem for a candidate (+ reduction segments)
int launch_kkt(hpr_ctx *c, int term_original, const double *cy, const double *cx,
               const double *cz, std::vector<RedSeg> &segs) {
  const hpr_buffers &B = c->B;
  Parts P = parts_of(c);
  EpiKktRow er{};
  er.b = term_original ? B.b : B.b_s;
  er.cy = cy;
  er.m1 = (int)c->d.m1;
  int ga = 0, gat = 0;
  int rc = launch_sell(c, c->mat_a(!term_original), cx, er, P.krow, &ga);
  if (rc) return rc;
  EpiKktCol ec{};
  ec.c = term_original ? B.c : B.c_s;
  ec.lo = term_original ? B.lower : B.lower_s;
  ec.up = term_original ? B.upper : B.upper_s;
  ec.cx = cx;
  ec.cz = cz;
  rc = launch_sell(c, c->mat_at(!term_original), cy, ec, P.kcol, &gat);
  if (rc) return rc;
  segs.push_back({P.krow + 0 * ga, ga, R_PRIM2});
  segs.push_back({P.krow + 1 * ga, ga, R_BY});
  segs.push_back({P.krow + 2 * ga, ga, R_R1});
  const int outs[8] = {R_DUAL2, R_CX, R_LZ, R_UZ, R_NLO, R_NUP, R_CLAMP, R_R2};
  for (int q = 0; q < 8; ++q) segs.push_back({P.kcol + q * gat, gat, outs[q]});
  return HPR_OK;
}

int check_ctx(hpr_ctx *c, bool need_layout = true, bool need_scaled = false) {
  if (!c) return fail(HPR_EINVAL, "null context");
  if (!c->bound) return fail(HPR_ESTATE, "hpr_bind has not been called");
  if (need_layout && !c->laid_out)
    return fail(HPR_ESTATE, "hpr_analyze + hpr_bind_layout have not been called");
  if (need_scaled && !c->scaled) return fail(HPR_ESTATE, "hpr_scale has not been called");
  return HPR_OK;
}

int kkt_common(hpr_ctx *c, int term_original, int slot, hpr_ckpt_out *out) {
  const hpr_buffers &B = c->B;
  std::vector<RedSeg> segs;
  int rc = launch_kkt(c, term_original, B.cand_y[slot], B.cand_x[slot], B.cand_z[slot], segs);
  if (rc) return rc;
  CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, c->stream));
  rc = reduce_final(c, segs);
  if (rc) return rc;
  rc = fetch_results(c);
  if (rc) return rc;
  fill_out(c, out);
  return HPR_OK;
}

}  // namespace

#include "hpr_small.cuh"

namespace {

// ---- resident small-LP inner loop (hpr_small.cuh) ----
// Cluster size for the resident loop, or 0 for the graph path: used when both
// SELL layouts have <= kSmallMaxWin windows (HPR_SMALL=0 disables it,
// HPR_SMALL=1 forces it whenever a cluster can be launched).
int small_cluster(hpr_ctx *c) {
  const char *env = getenv("HPR_SMALL");
  if (env && env[0] == '0') return 0;
  // the staged / column-blocked / column-split engines are large-problem
  // layouts: when one is on (forced), the graph path runs it
  if (!(env && env[0] == '1') && (c->sta.on || c->stat.on || c->cba.on || c->cbat.on || c->sp.on))
    return 0;
  const int wa = (c->sa.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  const int wat = (c->sat.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  const int wmax = std::max(wa, wat);
  if (!(env && env[0] == '1') && wmax > kSmallMaxWin) return 0;
  int G = std::max(1, std::min(kSmallMaxCluster, wmax));
  return G;
}

// Shared-memory staging of the small loop (k_small_inner): per CTA the largest
// owned slot count of A^T / A and the bytes of both stages; 0 when the stages
// exceed the budget or HPR_SMALL_SMEM=0 (the loop then streams from L2).
size_t small_stage_bytes(int nsl, int cap) {
  return 4 * (size_t)((nsl + 4) & ~3) + 4 * (size_t)nsl * kSlice +
         2 * (size_t)((nsl * kSlice + 7) & ~7) + 16 + 12 * (size_t)cap + 16;
}
int small_smem_plan(hpr_ctx *c, int G) {
  if (c->small_G == G) return HPR_OK;
  c->small_G = G;
  c->small_cap[0] = c->small_cap[1] = 0;
  c->small_smem = 0;
  const char *env = getenv("HPR_SMALL_SMEM");
  if (env && env[0] == '0') return HPR_OK;
  int caps[2] = {0, 0};
  size_t bytes[2] = {0, 0};
  const Sell *SS[2] = {&c->sat, &c->sa};
  for (int q = 0; q < 2; ++q) {
    const Sell &S = *SS[q];
    std::vector<int> sp(S.nslices + 1);
    CK(cudaMemcpyAsync(sp.data(), S.slice_ptr, sizeof(int) * (S.nslices + 1),
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const int nwin = (S.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
    const int nown = (nwin + G - 1) / G;
    for (int g = 0; g < G; ++g) {
      long long slots = 0;
      for (int win = g; win < nwin; win += G)
        for (int w = 0; w < kWarpsPerCta; ++w) {
          const int sl = win * kWarpsPerCta + w;
          if (sl < S.nslices) slots += sp[sl + 1] - sp[sl];
        }
      caps[q] = (int)std::max<long long>(caps[q], slots);
    }
    bytes[q] = small_stage_bytes(nown * kWarpsPerCta, std::max(caps[q], 1)) + 16;
  }
  // within the default 48 KB (more dynamic shared memory cut B200's maximum
  // cluster size for this kernel from 16 to 8): A first (longer rows, more
  // dependent batches per slice), then A^T if it fits too
  constexpr size_t kBudget = 48 * 1024;
  size_t total = 0;
  if (bytes[1] <= kBudget) {
    c->small_cap[1] = std::max(caps[1], 1);
    total += bytes[1];
  }
  if (total + bytes[0] <= kBudget) {
    c->small_cap[0] = std::max(caps[0], 1);
    total += bytes[0];
  }
  c->small_smem = (int)total;
  return HPR_OK;
}

template <bool GAX, bool GAY>
int launch_small(hpr_ctx *c, int G, const SellMat &AT, const SellMat &A, const EpiXIter &ex,
                 const EpiYIter &ey, int steps) {
  auto kern = k_small_inner<GAX, GAY>;
  if (int e = small_smem_plan(c, G)) return e;

  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int &o = g_attr[{(const void *)kern, c->device}];
    if (o == 0) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      o = 1;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.dynamicSmemBytes = c->small_smem;
  CK(cudaLaunchKernelEx(&cfg, kern, AT, A, (const double *)c->B.y, (const double *)c->B.w, ex, ey,
                        steps, (int)HPR_X_IMPLICIT, c->small_cap[0], c->small_cap[1]));
  CKL();
  return HPR_OK;
}

template <bool GAX, bool GAY>
int launch_small_power(hpr_ctx *c, int G, const SellMat &AT, const SellMat &A, double *v,
                       double *u, double *wv, double *part) {
  auto kern = k_small_power<GAX, GAY>;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int &o = g_attr[{(const void *)kern, c->device}];
    if (o == 0) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      o = 1;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, AT, A, v, u, wv, part, c->pow, (int)c->d.m));
  CKL();
  c->launches += 1;
  return HPR_OK;
}

int run_small(hpr_ctx *c, int steps, int64_t t, int64_t k, double sigma, double lamsig,
              int variant) {
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  const SellMat A = c->mat_a(true), AT = c->mat_at(true);
  EpiXIter ex{};
  ex.c = B.c_s;
  ex.lo = B.lower_s;
  ex.up = B.upper_s;
  ex.bounds_uniform = c->bounds_uniform;
  ex.lo_u = c->lo_u;
  ex.up_u = c->up_u;
  ex.anc = B.anc_x;
  ex.x = B.x;
  ex.w = B.w;
  ex.P = c->params;
  EpiYIter ey{};
  ey.b = B.b_s;
  ey.anc = B.anc_y;
  ey.y = B.y;
  ey.P = c->params;
  ey.m1 = (int)c->d.m1;
  const int G = small_cluster(c);
  k_set_params<<<1, 1, 0, s>>>(c->params, sigma, lamsig, (long long)t, (long long)k, variant);
  CKL();
  CK(cudaEventRecord(c->ev0, s));
  int rc = AT.ga ? (A.ga ? launch_small<true, true>(c, G, AT, A, ex, ey, steps)
                         : launch_small<true, false>(c, G, AT, A, ex, ey, steps))
                 : (A.ga ? launch_small<false, true>(c, G, AT, A, ex, ey, steps)
                         : launch_small<false, false>(c, G, AT, A, ex, ey, steps));
  if (rc) return rc;
  CK(cudaEventRecord(c->ev1, s));
  c->inner_timed = true;
  c->launches += 2;
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
  if (dims->nnz >= INT_MAX || dims->m >= INT_MAX - kWindow || dims->n >= INT_MAX - kWindow)
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
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    hpr_ctx_destroy(c);
    return fail(HPR_ECUDA, std::string("ctx_create: ") + cudaGetErrorString(e));
  }
  *out = c;
  return HPR_OK;
}

int hpr_ctx_destroy(hpr_ctx *c) {
  if (!c) return HPR_OK;
  c->drop_inner_graphs();
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
    if (!p) return fail(HPR_EINVAL, "a required buffer pointer is null");
  c->B = *bufs;
  c->ws = (char *)workspace;
  c->L = L;
  c->part = (double *)(c->ws + L.part);
  c->results = (double *)(c->ws + L.results);
  c->fac = (double *)(c->ws + L.fac);
  c->dvec_m = (double *)(c->ws + L.dvec_m);
  c->dvec_n = (double *)(c->ws + L.dvec_n);
  c->params = (IterParams *)(c->ws + L.params);
  c->pow = (PowState *)(c->ws + L.pow);
  c->flags = (unsigned int *)(c->ws + L.flags);
  // the whole result / parameter blocks are read back at every checkpoint:
  // defined contents even in the slots a given call does not write
  CK(cudaSetDevice(c->device));
  CK(cudaMemsetAsync(c->results, 0, sizeof(double) * R_COUNT, c->stream));
  CK(cudaMemsetAsync(c->params, 0, sizeof(IterParams), c->stream));
  c->drop_inner_graphs();
  c->exa = hpr_ctx::Exact{};
  if (c->pow_graph) {
    cudaGraphExecDestroy(c->pow_graph);
    c->pow_graph = nullptr;
  }
  c->graph_sig.clear();
  c->bound = true;
  c->analyzed = c->laid_out = c->scaled = false;
  return HPR_OK;
}

int hpr_analyze(hpr_ctx *c, size_t *layout_bytes) {
  int rc = check_ctx(c, false);
  if (rc) return rc;
  if (!layout_bytes) return fail(HPR_EINVAL, "null layout_bytes");
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
  {
    const int *order = row_affinity_order(c, B.a_rp, B.a_ci, m, n, false, &rc);
    if (rc) return rc;
    rc = plan_sell(c, c->L.pa, B.a_rp, m, c->sa, kLongRow, 0, 0, order);
  }
  if (rc) return rc;
  {
    const int *order = row_affinity_order(c, B.at_rp, B.at_ci, n, m, true, &rc);
    if (rc) return rc;
    rc = plan_sell(c, c->L.pat, B.at_rp, n, c->sat, kLongRow, 0, 0, order);
  }
  if (rc) return rc;
  rc = cb_plan(c, c->L.ca, B.a_rp, B.a_ci, m, c->cba);
  if (rc) return rc;
  rc = cb_plan(c, c->L.cat, B.at_rp, B.at_ci, n, c->cbat);
  if (rc) return rc;
  rc = split_plan(c);
  if (rc) return rc;
  c->stg_sorted = nullptr;
  rc = stg_plan(c, c->L.sa, B.a_rp, B.a_ci, m, c->sta);
  if (rc) return rc;
  rc = stg_plan(c, c->L.sat, B.at_rp, B.at_ci, n, c->stat);
  if (rc) return rc;
  rc = ts_select(c);
  if (rc) return rc;
  *layout_bytes = ts_bytes(c) + sell_bytes(c->sa, d.nnz) + sell_bytes(c->sat, d.nnz) +
                  cb_bytes(c->cba, d.nnz) + cb_bytes(c->cbat, d.nnz) + split_bytes(c->sp, d.nnz) +
                  stg_bytes(c->sta, d.nnz) + stg_bytes(c->stat, d.nnz);
  c->analyzed = true;
  c->laid_out = false;
  return HPR_OK;
}

int hpr_bind_layout(hpr_ctx *c, void *layout, size_t bytes) {
  int rc = check_ctx(c, false);
  if (rc) return rc;
  if (!c->analyzed) return fail(HPR_ESTATE, "hpr_analyze has not been called");
  if (!layout) return fail(HPR_EINVAL, "null layout");
  if (bytes < ts_bytes(c) + sell_bytes(c->sa, c->d.nnz) + sell_bytes(c->sat, c->d.nnz) +
                  cb_bytes(c->cba, c->d.nnz) + cb_bytes(c->cbat, c->d.nnz) +
                  split_bytes(c->sp, c->d.nnz) + stg_bytes(c->sta, c->d.nnz) +
                  stg_bytes(c->stat, c->d.nnz))
    return fail(HPR_EINVAL, "layout buffer too small");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  char *p = (char *)layout;
  c->ts_blk = (int *)p;   // TS block lists (filled by ts_plan below)
  p += ts_bytes(c);
  rc = layout_sell(c, p, c->sa, B.a_rp, B.a_ci, B.a_val);
  if (rc) return rc;
  rc = layout_sell(c, p, c->sat, B.at_rp, B.at_ci, B.at_val);
  if (rc) return rc;
  rc = cb_layout(c, p, c->cba, B.a_rp, B.a_ci);
  if (rc) return rc;
  rc = cb_layout(c, p, c->cbat, B.at_rp, B.at_ci);
  if (rc) return rc;
  rc = split_layout(c, p);
  if (rc) return rc;
  rc = stg_layout(c, p, c->sta, B.a_rp, B.a_ci, (int)c->d.m);
  if (rc) return rc;
  rc = stg_layout(c, p, c->stat, B.at_rp, B.at_ci, (int)c->d.n);
  if (rc) return rc;
  rc = ts_aw_layout(c, (char *)c->ts_blk);
  if (rc) return rc;
  CK(cudaStreamSynchronize(c->stream));
  // the captured graphs hold the layout's pointers and the plans' counts: keep
  // them when a re-analysed problem reproduces both (a re-solve of the same
  // structure), drop them otherwise
  std::vector<long long> sig = {(long long)(uintptr_t)layout, (long long)bytes};
  for (const Sell *S : {&c->sa, &c->sat, &c->sp.S})
    for (long long v : {(long long)S->nslices, S->slots, (long long)S->nlong, (long long)S->affinity})
      sig.push_back(v);
  for (long long v : {(long long)c->sp.on, (long long)c->sp.NB, (long long)c->sp.W}) sig.push_back(v);
  for (const hpr_ctx::Stg *T : {&c->sta, &c->stat})
    for (long long v : {(long long)T->on, (long long)T->G, (long long)T->NB, (long long)T->rows_cap,
                        (long long)T->rec_cap, T->rec_total, (long long)T->stages})
      sig.push_back(v);
  for (const hpr_ctx::Cb *C : {&c->cba, &c->cbat})
    for (long long v : {(long long)C->on, (long long)C->G, (long long)C->NB, (long long)C->rows_cap,
                        (long long)C->seg_cap, (long long)C->stages, C->npad, C->nrpb})
      sig.push_back(v);
  if (sig != c->graph_sig) {
    c->drop_inner_graphs();
    if (c->pow_graph) {
      cudaGraphExecDestroy(c->pow_graph);
      c->pow_graph = nullptr;
    }
    c->graph_sig = sig;
  }
  c->keep_a = c->keep_at = 0;
  {
    // L2 policy of the matrix streams (SellMat::keep)
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
    const double a_bytes = 12.0 * (double)c->sa.slots, at_bytes = 12.0 * (double)c->sat.slots;
    switch (HPR_L2KEEP) {
      case 1: c->keep_a = 1; break;
      case 2: c->keep_at = 1; break;
      case 3: c->keep_a = c->keep_at = 2; break;
      case 4:
        if (at_bytes <= 0.6 * l2) c->keep_at = 1;
        else if (a_bytes <= 0.6 * l2) c->keep_a = 1;
        break;
      default: break;
    }
  }
  rc = ts_plan(c);
  if (rc) return rc;
  c->small_G = -1;   // the small loop's staging plan follows the layout
  c->laid_out = true;
  c->scaled = false;
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
    k_sumsq<<<nb1, kThreads, 0, s>>>(B.c_s, n, P.misc + kSumsqBlocks);
    CKL();
    c->launches += 2;
    rc = reduce_final(c, {RedSeg{P.misc, nb0, R_SUMSQ0},
                          RedSeg{P.misc + kSumsqBlocks, nb1, R_SUMSQ1}});
    if (rc) return rc;
    k_factors<<<1, 32, 0, s>>>(c->results + R_SUMSQ0, c->fac);
    k_bc_normalize<<<g, 256, 0, s>>>(B.b_s, m, B.c_s, B.lower_s, B.upper_s, n, c->fac);
    CKL();
    c->launches += 2;
  } else {
    k_fill<<<1, 32, 0, s>>>(c->fac, 1.0, 2);
    CKL();
  }
  if (nnz > 0) {
    k_gather_vals<<<grid_for(nnz), 256, 0, s>>>(B.at_perm, B.a_val_s, B.at_val_s, nnz);
    k_sell_scatter<<<grid_for(nnz), 256, 0, s>>>(c->sa.pos, B.a_val_s, c->sa.val_s, nnz);
    k_sell_scatter<<<grid_for(nnz), 256, 0, s>>>(c->sat.pos, B.at_val_s, c->sat.val_s, nnz);
    if (c->sp.on) k_sell_scatter<<<grid_for(nnz), 256, 0, s>>>(c->sp.S.pos, B.a_val_s, c->sp.S.val_s, nnz);
    CKL();
    c->launches += 3 + (int)c->sp.on;
    if (c->sta.on)
      k_sell_scatter<<<grid_for(nnz), 256, 0, s>>>(c->sta.pos, B.a_val_s, (double *)c->sta.rec, nnz);
    if (c->stat.on)
      k_sell_scatter<<<grid_for(nnz), 256, 0, s>>>(c->stat.pos, B.at_val_s, (double *)c->stat.rec, nnz);
    c->launches += (int)c->sta.on + (int)c->stat.on;
    if (c->cba.on) k_cb_scatter<<<grid_for(nnz), 256, 0, s>>>(c->cba.pos, B.a_val_s, c->cba.val, nnz);
    if (c->cbat.on) k_cb_scatter<<<grid_for(nnz), 256, 0, s>>>(c->cbat.pos, B.at_val_s, c->cbat.val, nnz);
    CKL();
    c->launches += (int)c->cba.on + (int)c->cbat.on;
  }
  // ||b||, ||c|| of the original and the scaled problem (relative residual denominators)
  const int nbm = sumsq_blocks(m), nbn = sumsq_blocks(n);
  k_sumsq<<<nbm, kThreads, 0, s>>>(B.b, m, P.misc);
  k_sumsq<<<nbn, kThreads, 0, s>>>(B.c, n, P.misc + kSumsqBlocks);
  k_sumsq<<<nbm, kThreads, 0, s>>>(B.b_s, m, P.misc + 2 * kSumsqBlocks);
  k_sumsq<<<nbn, kThreads, 0, s>>>(B.c_s, n, P.misc + 3 * kSumsqBlocks);
  CKL();
  c->launches += 4;
  rc = reduce_final(c, {RedSeg{P.misc, nbm, R_SUMSQ0},
                        RedSeg{P.misc + kSumsqBlocks, nbn, R_SUMSQ1},
                        RedSeg{P.misc + 2 * kSumsqBlocks, nbm, R_SUMSQ2},
                        RedSeg{P.misc + 3 * kSumsqBlocks, nbn, R_SUMSQ3}});
  if (rc) return rc;
  // uniform scaled bounds (x-phase reads a scalar instead of the vector)
  const unsigned int ones[2] = {1u, 1u};
  CK(cudaMemcpyAsync(c->flags, ones, sizeof(ones), cudaMemcpyHostToDevice, s));
  k_uniform<<<grid_for(n), 256, 0, s>>>(B.lower_s, n, c->flags);
  k_uniform<<<grid_for(n), 256, 0, s>>>(B.upper_s, n, c->flags + 1);
  CKL();
  c->launches += 2;
  unsigned int hfl[2];
  double hb[2];
  CK(cudaMemcpyAsync(hfl, c->flags, sizeof(hfl), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hb, B.lower_s, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hb + 1, B.upper_s, sizeof(double), cudaMemcpyDeviceToHost, s));
  double fac[2];
  CK(cudaMemcpyAsync(fac, c->fac, sizeof(fac), cudaMemcpyDeviceToHost, s));
  rc = fetch_results(c);
  if (rc) return rc;
  const int bu = (hfl[0] ? 1 : 0) | (hfl[1] ? 2 : 0);
  if (bu != c->bounds_uniform || (bu && (std::memcmp(&hb[0], &c->lo_u, 8) || std::memcmp(&hb[1], &c->up_u, 8)))) {
    c->drop_inner_graphs();
  }
  c->bounds_uniform = bu;
  c->lo_u = hb[0];
  c->up_u = hb[1];
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
  const int m = (int)c->d.m;
  cudaStream_t s = c->stream;
  double *v = B.yb, *u = B.wtmp, *wv = B.dy;   // scratch reuse (before the iterations)
  Parts P = parts_of(c);
  PowState st{};
  st.tol = tol;
  st.max_iters = max_iters;
  EpiPowT et{};
  et.u = u;
  et.S = c->pow;
  EpiPowA ea{};
  ea.v = v;
  ea.wv = wv;
  ea.S = c->pow;
  // all-ones start; fall back to basis vectors while A^T v == 0 (sparse.py:176-182)
  int start = -2;
  for (int fb = -1; fb < m; ++fb) {
    if (fb < 0) {
      k_fill<<<grid_for(m), 256, 0, s>>>(v, 1.0, m);
    } else {
      k_fill<<<grid_for(m), 256, 0, s>>>(v, 0.0, m);
      k_fill<<<1, 32, 0, s>>>(v + fb, 1.0, 1);
    }
    CK(cudaMemcpyAsync(c->pow, &st, sizeof(st), cudaMemcpyHostToDevice, s));
    int gt = 0;
    rc = launch_sell(c, c->mat_at(true), v, et, P.powt, &gt);
    if (rc) return rc;
    rc = reduce_final(c, {RedSeg{P.powt, gt, R_POW_U2}});
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
  if (const int G = small_cluster(c)) {
    // small LP: every step in one resident cluster launch (hpr_small.cuh)
    const SellMat A = c->mat_a(true), AT = c->mat_at(true);
    rc = AT.ga ? (A.ga ? launch_small_power<true, true>(c, G, AT, A, v, u, wv, P.powa)
                       : launch_small_power<true, false>(c, G, AT, A, v, u, wv, P.powa))
               : (A.ga ? launch_small_power<false, true>(c, G, AT, A, v, u, wv, P.powa)
                       : launch_small_power<false, false>(c, G, AT, A, v, u, wv, P.powa));
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->h_pow, c->pow, sizeof(PowState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out->raw = c->h_pow->lam;
    out->value = c->h_pow->lam * (1.0 + 1e-3);
    out->iterations = c->h_pow->iters;
    out->converged = c->h_pow->converged;
    return HPR_OK;
  }
  if (!c->pow_graph) {
    cudaGraph_t g;
    const long long before = c->launches;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kPowBatch; ++i) {
      int ga = 0;
      if (c->stat.on || c->ts_at) {   // u = A^T v without the (unused) norm partials
        EpiPowTu eu{};
        eu.u = u;
        eu.S = c->pow;
        rc = c->stat.on ? launch_stg(c, c->stat, (int)c->d.m, v, eu)
                        : launch_ts(c, c->mat_at(true), c->ts_blk + c->ts_nb_a + 1, c->ts_nb_at, v, eu);
      } else {
        rc = launch_sell(c, c->mat_at(true), v, et, P.powt, nullptr);
      }
      // A u with the power step in its last CTA, then v = w / ||w||
      EpiPowAStep eas{};
      static_cast<EpiPowA &>(eas) = ea;
      if (!rc) rc = launch_sell(c, c->mat_a(true), u, eas, P.powa, &ga);
      if (rc) {
        cudaStreamEndCapture(s, &g);
        return rc;
      }
      k_pow_norm<<<grid_for(m), 256, 0, s>>>(wv, v, m, c->pow);
    }
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("pow capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->pow_graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess)
      return fail(HPR_ECUDA, std::string("pow instantiate: ") + cudaGetErrorString(e));
    c->launches = before;   // captured, not executed
  }
  for (;;) {
    CK(cudaGraphLaunch(c->pow_graph, s));
    c->launches += 3 * kPowBatch;
    CK(cudaMemcpyAsync(c->h_pow, c->pow, sizeof(PowState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (c->h_pow->done) break;
  }
  out->raw = c->h_pow->lam;
  out->value = c->h_pow->lam * (1.0 + 1e-3);
  out->iterations = c->h_pow->iters;
  out->converged = c->h_pow->converged;
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
  k_reset_params<<<1, 1, 0, s>>>(c->params);
  CKL();
  CK(cudaStreamSynchronize(s));
  return HPR_OK;
}

// Persisting-L2 window over y for the inner loop (HPR_L2WIN=1, opt-in): the
// dual iterate is gathered by the x-phase (random segments) and streamed by
// the y-phase; with a window it stays L2-resident while the matrix and the
// n-vectors stream past it.  The device's persisting carve-out is raised to
// the window (capped at the device maximum); hitRatio covers the remainder.
int l2_window_setup(hpr_ctx *c) {
  c->l2win_active = false;
  const char *env = getenv("HPR_L2WIN");
  if (!(env && env[0] == '1')) return HPR_OK;
  int maxp = 0, maxw = 0;
  CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, c->device));
  CK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, c->device));
  if (maxp <= 0 || maxw <= 0) return HPR_OK;
  const size_t ybytes = sizeof(double) * (size_t)c->d.m;
  size_t limit = 0;
  CK(cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize));
  const size_t want = std::min(ybytes, (size_t)maxp);
  if (limit < want) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
  CK(cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize));
  cudaAccessPolicyWindow w{};
  w.base_ptr = (void *)c->B.y;
  w.num_bytes = std::min(ybytes, (size_t)maxw);
  w.hitRatio = (float)std::min(1.0, (double)limit / (double)w.num_bytes);
  w.hitProp = cudaAccessPropertyPersisting;
  w.missProp = cudaAccessPropertyStreaming;
  c->l2win = w;
  c->l2win_active = true;
  return HPR_OK;
}

// the inner-loop epilogues of the graph path (step fields set per launch)
static void iter_epilogues(const hpr_ctx *c, EpiXIter &ex, EpiYIter &ey) {
  const hpr_buffers &B = c->B;
  ex = EpiXIter{};
  ex.c = B.c_s;
  ex.lo = B.lower_s;
  ex.up = B.upper_s;
  ex.bounds_uniform = c->bounds_uniform;
  ex.lo_u = c->lo_u;
  ex.up_u = c->up_u;
  ex.anc = B.anc_x;
  ex.x = B.x;
  ex.w = B.w;
  ex.P = c->params;
  ey = EpiYIter{};
  ey.b = B.b_s;
  ey.anc = B.anc_y;
  ey.y = B.y;
  ey.P = c->params;
  ey.m1 = (int)c->d.m1;
  ey.ef = HPR_Y_EF && c->ts_at;   // with the TS x-phase (HBM-bound problems)
}

// one x-phase / y-phase launch on the engine the layout selected
static int launch_x_phase(hpr_ctx *c, const EpiXIter &ex, bool pdl) {
  const hpr_buffers &B = c->B;
  return c->stat.on ? launch_stg(c, c->stat, (int)c->d.m, B.y, ex)
         : c->cbat.on ? launch_cb(c, c->cbat, (int)c->d.m, B.y, ex)
         : c->ts_at ? launch_ts(c, c->mat_at(true), c->ts_blk + c->ts_nb_a + 1, c->ts_nb_at, B.y,
                                ts_ef(ex))
                    : launch_sell(c, c->mat_at(true), B.y, ex, nullptr, nullptr, pdl);
}
static int launch_y_phase(hpr_ctx *c, const EpiYIter &ey) {
  const hpr_buffers &B = c->B;
  return c->sta.on ? launch_stg(c, c->sta, (int)c->d.n, B.w, ey)
         : c->cba.on ? launch_cb(c, c->cba, (int)c->d.n, B.w, ey)
         : c->ts_a ? launch_ts(c, c->mat_a(true), c->ts_blk, c->ts_nb_a, B.w, ey)
                   : launch_a_iter(c, B.w, ey, true);
}

int hpr_run_inner(hpr_ctx *c, int steps, int64_t t, int64_t k, double sigma, double lamsig,
                  int variant) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (steps <= 0) return HPR_OK;
  if (variant < 0 || variant > 2) return fail(HPR_EINVAL, "bad variant");
  CK(cudaSetDevice(c->device));
  if (small_cluster(c) > 0) return run_small(c, steps, t, k, sigma, lamsig, variant);
  const hpr_buffers &B = c->B;
  cudaStream_t s = c->stream;
  auto it = c->inner_graphs.find(steps);
  if (it == c->inner_graphs.end()) {
    const SellMat A = c->mat_a(true), AT = c->mat_at(true);
    EpiXIter ex{};
    EpiYIter ey{};
    iter_epilogues(c, ex, ey);
    cudaGraph_t g;
    const long long before = c->launches;
    if (int e2 = l2_window_setup(c)) return e2;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < steps; ++i) {
      ex.step = i;
      ey.step = i;
      // HPR: x implicit between the interval's first read and last write
      ex.x_from_w = HPR_X_IMPLICIT && i > 0;
      ex.x_store = !HPR_X_IMPLICIT || i == steps - 1;
      // the first kernel of the graph follows the k_set_params launch: plain edge
      int rc2 = launch_x_phase(c, ex, i > 0);
      if (!rc2) rc2 = launch_y_phase(c, ey);
      if (rc2) {
        c->l2win_active = false;
        cudaStreamEndCapture(s, &g);
        return rc2;
      }
    }
    c->l2win_active = false;
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exe;
    e = cudaGraphInstantiate(&exe, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    c->launches = before;   // captured, not executed
    it = c->inner_graphs.emplace(steps, exe).first;
  }
  k_set_params<<<1, 1, 0, s>>>(c->params, sigma, lamsig, (long long)t, (long long)k, variant);
  CKL();
  CK(cudaEventRecord(c->ev0, s));
  CK(cudaGraphLaunch(it->second, s));
  CK(cudaEventRecord(c->ev1, s));
  c->inner_timed = true;
  c->launches += 1 + (1LL + (c->sp.on ? c->sp.NB : 1)) * steps;
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
  Parts P = parts_of(c);
  CandCtx cc{term_original, c->fac, B.row_scale, B.col_scale, B.lower, B.upper};
  CK(cudaEventRecord(c->ev2, s));
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
  int gx = 0, gy = 0, gm = 0;
  rc = launch_sell(c, c->mat_at(true), B.y, ex, P.xhalf, &gx);
  if (rc) return rc;
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
  rc = launch_sell(c, c->mat_a(true), B.wtmp, ey, P.yhalf, &gy);
  if (rc) return rc;
  EpiMeritCol em{};
  em.x = B.x;
  em.xb = B.xb;
  em.sigma = sigma;
  rc = launch_sell(c, c->mat_at(true), B.dy, em, P.merit, &gm);
  if (rc) return rc;
  std::vector<RedSeg> segs;
  segs.push_back({P.xhalf, gx, R_BAR_DX2});
  segs.push_back({P.xhalf + gx, gx, R_DX2});
  segs.push_back({P.yhalf, gy, R_DY2});
  segs.push_back({P.yhalf + gy, gy, R_BAR_DY2});
  segs.push_back({P.merit, gm, R_SH2});
  segs.push_back({P.merit + gm, gm, R_ATY2});
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
  const int m = (int)c->d.m, n = (int)c->d.n;
  k_origin_cand<<<grid_for(std::max(m, n)), 256, 0, c->stream>>>(
      B.cand_y[slot], m, B.cand_z[slot], B.cand_x[slot], term_original ? B.lower : B.lower_s,
      term_original ? B.upper : B.upper_s, n);
  CKL();
  c->launches += 1;
  return kkt_common(c, term_original, slot, out);
}

int hpr_kkt(hpr_ctx *c, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  return kkt_common(c, term_original, slot, out);
}

int hpr_finalize(hpr_ctx *c, int term_original, int slot, hpr_ckpt_out *out) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!out || slot < 0 || slot > 1) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  const hpr_buffers &B = c->B;
  const int m = (int)c->d.m, n = (int)c->d.n;
  int fs = slot;
  if (!term_original) {
    fs = 1 - slot;
    k_unscale<<<grid_for(std::max(m, n)), 256, 0, c->stream>>>(
        B.cand_y[slot], B.cand_z[slot], B.cand_x[slot], B.cand_y[fs], B.cand_z[fs],
        B.cand_x[fs], B.row_scale, B.col_scale, c->fac, B.lower, B.upper, m, n);
    CKL();
    c->launches += 1;
  }
  return kkt_common(c, 1, fs, out);
}

int hpr_launch_count(hpr_ctx *c, int64_t *count) {
  if (!c || !count) return fail(HPR_EINVAL, "null argument");
  *count = c->launches;
  return HPR_OK;
}

int hpr_layout_info(hpr_ctx *c, hpr_layout_info_t *info) {
  if (!c || !info) return fail(HPR_EINVAL, "null argument");
  info->slices_a = c->sa.nslices;
  info->slices_at = c->sat.nslices;
  info->slots_a = c->sa.slots;
  info->slots_at = c->sat.slots;
  info->long_rows_a = c->sa.nlong;
  info->long_rows_at = c->sat.nlong;
  info->cb_a = c->cba.on ? c->cba.npad : 0;
  info->cb_at = c->cbat.on ? c->cbat.npad : 0;
  info->split_a = c->sp.on ? c->sp.NB : 0;
  info->stg_a = c->sta.on ? c->sta.NB : 0;
  info->stg_at = c->stat.on ? c->stat.NB : 0;
  info->rao_a = c->sa.affinity;
  info->rao_at = c->sat.affinity;
  info->bounds_uniform = c->bounds_uniform;
  info->ts_a = c->ts_a ? c->ts_nb_a : 0;
  info->ts_at = c->ts_at ? c->ts_nb_at : 0;
  info->ts_words_a = c->ts_aw[0] ? c->ts_aw_words[0] : 0;
  info->ts_words_at = c->ts_aw[1] ? c->ts_aw_words[1] : 0;
  return HPR_OK;
}

int hpr_small_path(hpr_ctx *c) { return c && c->analyzed && small_cluster(c) > 0 ? 1 : 0; }

int hpr_time_phases(hpr_ctx *c, int reps, double *x_us, double *y_us) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (reps < 1 || !x_us || !y_us) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  EpiXIter ex{};
  EpiYIter ey{};
  iter_epilogues(c, ex, ey);
  ex.step = ey.step = 1;
  ex.x_from_w = HPR_X_IMPLICIT;   // an interval's steady-state step (x implicit for HPR)
  ex.x_store = !HPR_X_IMPLICIT;
  CK(cudaEventRecord(c->ev0, s));
  for (int r = 0; r < reps && !rc; ++r) rc = launch_x_phase(c, ex, false);
  CK(cudaEventRecord(c->ev1, s));
  for (int r = 0; r < reps && !rc; ++r) rc = launch_y_phase(c, ey);
  CK(cudaEventRecord(c->ev2, s));
  if (rc) return rc;
  CK(cudaEventSynchronize(c->ev2));
  float a = 0.f, b = 0.f;
  CK(cudaEventElapsedTime(&a, c->ev0, c->ev1));
  CK(cudaEventElapsedTime(&b, c->ev1, c->ev2));
  *x_us = 1e3 * a / reps;
  *y_us = 1e3 * b / reps;
  c->inner_timed = c->ckpt_timed = false;   // the events now hold this measurement
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

#include "hpr_rowblock.cuh"
#include "hpr_batch.cuh"

extern "C" int hpr_spmv(hpr_ctx *c, int transpose, const double *x, double *y) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!x || !y) return fail(HPR_EINVAL, "null vector");
  CK(cudaSetDevice(c->device));
  EpiStore e{};
  e.out = y;
  e.S = nullptr;
  return launch_sell(c, transpose ? c->mat_at(true) : c->mat_a(true), x, e, nullptr, nullptr);
}

// ---------------------------------------------------------------------------
// exact T1 = 0 path (hpr_exact.cuh; exact.py:62-91)
// ---------------------------------------------------------------------------
namespace {

int launch_trmv_store(cudaStream_t s, const double *T, int m, int lower, const double *v,
                      double *out) {
  EpiTrStore e{out};
  const int grid = (m + kTrThreads / 32 - 1) / (kTrThreads / 32);
  k_trmv<EpiTrStore><<<grid, kTrThreads, 0, s>>>(T, m, lower, v, e);
  CKL();
  return HPR_OK;
}

// one exact iteration (half = 0) or the checkpoint's half step (half = 1)
int exact_step(hpr_ctx *c, int step, int half, double sigma, int slot) {
  const hpr_buffers &B = c->B;
  const hpr_ctx::Exact &E = c->exa;
  const int m = (int)c->d.m;
  EpiExactX ex{};
  ex.c = B.c_s;
  ex.lo = B.lower_s;
  ex.up = B.upper_s;
  ex.anc = B.anc_x;
  ex.x = B.x;
  ex.u = E.u;
  ex.xb_out = B.xb;
  ex.zb_out = B.zb;
  ex.cx_out = B.cand_x[slot];
  ex.cz_out = B.cand_z[slot];
  ex.P = c->params;
  ex.step = step;
  ex.half = half;
  ex.sigma_half = sigma;
  int rc = launch_sell(c, c->mat_at(true), B.y, ex, nullptr, nullptr);
  if (rc) return rc;
  EpiExactRhs er{};
  er.b = B.b_s;
  er.rhs = E.rhs;
  er.P = c->params;
  er.half = half;
  er.sigma_half = sigma;
  rc = launch_sell(c, c->mat_a(true), E.u, er, nullptr, nullptr);
  if (rc) return rc;
  rc = launch_trmv_store(c->stream, E.linv, m, 1, E.rhs, E.h);
  if (rc) return rc;
  EpiTrY ey{};
  ey.anc = B.anc_y;
  ey.y = B.y;
  ey.yb_out = B.yb;
  ey.cy_out = B.cand_y[slot];
  ey.P = c->params;
  ey.step = step;
  ey.half = half;
  const int grid = (m + kTrThreads / 32 - 1) / (kTrThreads / 32);
  k_trmv<EpiTrY><<<grid, kTrThreads, 0, c->stream>>>(E.linv_t, m, 0, E.h, ey);
  CKL();
  c->launches += 2;
  return HPR_OK;
}

}  // namespace

extern "C" int hpr_exact_bind(hpr_ctx *c, const hpr_exact_bufs *eb) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!eb || !eb->linv || !eb->linv_t || !eb->u || !eb->rhs || !eb->h)
    return fail(HPR_EINVAL, "null exact-path buffer");
  if (c->d.m1 != c->d.m) return fail(HPR_EINVAL, "the exact path requires an equality-only instance");
  for (auto &kv : c->exa.graphs) cudaGraphExecDestroy(kv.second);
  c->exa.graphs.clear();
  c->exa.linv = eb->linv;
  c->exa.linv_t = eb->linv_t;
  c->exa.u = eb->u;
  c->exa.rhs = eb->rhs;
  c->exa.h = eb->h;
  c->exa.on = true;
  return HPR_OK;
}

extern "C" int hpr_exact_run(hpr_ctx *c, int steps, int64_t t, int64_t k, double sigma,
                             int variant) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!c->exa.on) return fail(HPR_ESTATE, "hpr_exact_bind first");
  if (steps <= 0) return HPR_OK;
  if (variant < 0 || variant > 2) return fail(HPR_EINVAL, "bad variant");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  auto it = c->exa.graphs.find(steps);
  if (it == c->exa.graphs.end()) {
    cudaGraph_t g;
    const long long before = c->launches;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < steps; ++i) {
      int rc2 = exact_step(c, i, 0, 0.0, 0);
      if (rc2) {
        cudaStreamEndCapture(s, &g);
        return rc2;
      }
    }
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exe;
    e = cudaGraphInstantiate(&exe, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HPR_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    c->launches = before;   // captured, not executed
    it = c->exa.graphs.emplace(steps, exe).first;
  }
  k_set_params<<<1, 1, 0, s>>>(c->params, sigma, 0.0, (long long)t, (long long)k, variant);
  CKL();
  CK(cudaEventRecord(c->ev0, s));
  CK(cudaGraphLaunch(it->second, s));
  CK(cudaEventRecord(c->ev1, s));
  c->inner_timed = true;
  c->launches += 1 + 4LL * steps;
  return HPR_OK;
}

extern "C" int hpr_exact_half(hpr_ctx *c, double sigma, int slot, int64_t *nonfinite_k) {
  int rc = check_ctx(c, true, true);
  if (rc) return rc;
  if (!c->exa.on) return fail(HPR_ESTATE, "hpr_exact_bind first");
  if (slot < 0 || slot > 1 || !nonfinite_k) return fail(HPR_EINVAL, "bad argument");
  CK(cudaSetDevice(c->device));
  rc = exact_step(c, 0, 1, sigma, slot);
  if (rc) return rc;
  unsigned long long nf = 0;
  CK(cudaMemcpyAsync(&nf, &c->params->nonfinite_k, sizeof(nf), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *nonfinite_k = nf == ULLONG_MAX ? -1 : (int64_t)nf;
  return HPR_OK;
}

extern "C" int hpr_trsolve(int m, const double *linv, const double *linv_t, const double *rhs,
                           double *tmp, double *y, void *stream) {
  if (m <= 0 || !linv || !linv_t || !rhs || !tmp || !y) return fail(HPR_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = launch_trmv_store(s, linv, m, 1, rhs, tmp);
  if (rc) return rc;
  return launch_trmv_store(s, linv_t, m, 0, tmp, y);
}
