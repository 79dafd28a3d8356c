// hpr_kernels.cuh -- sm_100a device code of the HPR-LP iteration loop.
//
// Every sparse product here is a "row tile" kernel: a CTA owns a contiguous
// range of CSR rows (<= kThreads rows, <= tile_cap nonzeros), streams that
// range's values and column indices with coalesced loads, gathers the operand
// vector, stores the rounded products a_ij * x_j in shared memory, and then
// thread r adds its row's products left to right starting from 0.0.  That is
// exactly the arithmetic of scipy's csr_matvec, which the reference's
// SparseMatrix.apply / t_apply use (sparse.py:102-108) -- GPU and CPU sparse
// products are bit-identical -- and the sum is deterministic with no atomics.
// The row's owner thread then runs the fused elementwise epilogue (projection,
// Halpern averaging, residual terms) so the vector never makes an extra HBM
// round trip.  Reductions go warp-shuffle -> shared memory -> per-tile partial
// -> one fixed-order final pass.
//
// The whole library is compiled with -fmad=false: as in numpy, every product
// and sum is rounded separately.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace hpr {

constexpr int kThreads = 256;           // CTA size of all tile kernels
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ int pad_idx(int p) { return p + (p >> 4); }  // smem bank spread

// numpy maximum/minimum: NaN in the first operand propagates, ties return the
// second operand (np.clip == minimum(maximum(v, l), u)).
__device__ __forceinline__ double np_max(double a, double b) { return (isnan(a) || a > b) ? a : b; }
__device__ __forceinline__ double np_min(double a, double b) { return (isnan(a) || a < b) ? a : b; }
__device__ __forceinline__ double np_clip(double v, double l, double u) { return np_min(np_max(v, l), u); }

// Streaming loads for the matrix (read once per product): L1 no-allocate and an
// L2 evict-first policy so the gathered vectors keep the L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_stream(const double *ptr, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int *ptr, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}

struct TileMat {
  const int *rp;        // nrows + 1
  const int *ci;        // nnz
  const double *val;    // nnz
  const int *tile_row;  // ntiles + 1
  int ntiles;
  int cap;              // max nonzeros per (short-row) tile = smem products
};

// Parameters of the inner iterations, resident in device memory so a captured
// graph replays with new sigma / counters without re-instantiation.
struct IterParams {
  double sigma;
  double lamsig;
  long long t0;
  long long k0;
  int variant;
  int pad_;
  unsigned long long nonfinite_k;   // ULLONG_MAX = none
};

// Power-method state (sparse.py:184-198), advanced entirely on the device.
struct PowState {
  double lam, lam_prev, nw, tol;
  int iters, max_iters, converged, done, norm_pending, pad_;
};

// ---------------------------------------------------------------------------
// products of one tile (or one chunk of a long row) into shared memory
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tile_products(const TileMat &M, const double *__restrict__ xg,
                                              int z0, int nz, double *sprod, uint64_t pol) {
  int p = threadIdx.x;
  // 4 independent gathers in flight per thread
  for (; p + 3 * kThreads < nz; p += 4 * kThreads) {
    int j0 = ld_stream(M.ci + z0 + p, pol);
    int j1 = ld_stream(M.ci + z0 + p + kThreads, pol);
    int j2 = ld_stream(M.ci + z0 + p + 2 * kThreads, pol);
    int j3 = ld_stream(M.ci + z0 + p + 3 * kThreads, pol);
    double a0 = ld_stream(M.val + z0 + p, pol);
    double a1 = ld_stream(M.val + z0 + p + kThreads, pol);
    double a2 = ld_stream(M.val + z0 + p + 2 * kThreads, pol);
    double a3 = ld_stream(M.val + z0 + p + 3 * kThreads, pol);
    double x0 = __ldg(xg + j0), x1 = __ldg(xg + j1), x2 = __ldg(xg + j2), x3 = __ldg(xg + j3);
    sprod[pad_idx(p)] = __dmul_rn(a0, x0);
    sprod[pad_idx(p + kThreads)] = __dmul_rn(a1, x1);
    sprod[pad_idx(p + 2 * kThreads)] = __dmul_rn(a2, x2);
    sprod[pad_idx(p + 3 * kThreads)] = __dmul_rn(a3, x3);
  }
  for (; p < nz; p += kThreads) {
    int j = ld_stream(M.ci + z0 + p, pol);
    double a = ld_stream(M.val + z0 + p, pol);
    sprod[pad_idx(p)] = __dmul_rn(a, __ldg(xg + j));
  }
}

// Row sums of one tile.  Returns the sum for row `r` (owner thread) and whether
// this thread owns a row.  Long single-row tiles are chunked; thread 0 keeps the
// running left-to-right sum, so the order is still the sequential one.
__device__ __forceinline__ double tile_row_sum(const TileMat &M, const double *__restrict__ xg,
                                               double *sprod, int &r, bool &active) {
  const uint64_t pol = policy_evict_first();
  const int tile = blockIdx.x;
  const int r0 = M.tile_row[tile], r1 = M.tile_row[tile + 1];
  const int z0 = M.rp[r0];
  const int nz = M.rp[r1] - z0;
  double s = 0.0;
  if (nz <= M.cap) {
    tile_products(M, xg, z0, nz, sprod, pol);
    __syncthreads();
    r = r0 + threadIdx.x;
    active = r < r1;
    if (active) {
      const int a = M.rp[r] - z0, e = M.rp[r + 1] - z0;
      for (int k = a; k < e; ++k) s = __dadd_rn(s, sprod[pad_idx(k)]);
    }
  } else {
    r = r0;
    active = threadIdx.x == 0;
    for (int c0 = 0; c0 < nz; c0 += M.cap) {
      const int cn = min(M.cap, nz - c0);
      tile_products(M, xg, z0 + c0, cn, sprod, pol);
      __syncthreads();
      if (threadIdx.x == 0)
        for (int k = 0; k < cn; ++k) s = __dadd_rn(s, sprod[pad_idx(k)]);
      __syncthreads();
    }
  }
  return s;
}

// Fixed-order block reduction of NQ values: the block totals end up in v[] of
// thread 0 (other threads' v[] are clobbered).  Warp shuffle tree, then warp 0
// combines the per-warp sums -- same tree every launch, so bit-reproducible.
template <int NQ>
__device__ __forceinline__ void block_reduce(double (&v)[NQ]) {
  __shared__ double red[NQ][kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double a = v[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, off));
    if (lane == 0) red[q][warp] = a;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double a = lane < kWarps ? red[q][lane] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, off));
      v[q] = a;
    }
  }
}

// Block reduction; thread 0 stores part[q*stride + blockIdx.x].
template <int NQ>
__device__ __forceinline__ void block_reduce_store(double (&v)[NQ], double *part, int stride) {
  block_reduce<NQ>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) part[q * stride + blockIdx.x] = v[q];
  }
}

__device__ __forceinline__ double sq(double a) { return __dmul_rn(a, a); }

__device__ __forceinline__ void halpern_weights(long long t, double &wa, double &wn) {
  // core.py:142-144
  const double t2 = __dadd_rn((double)t, 2.0);
  wn = __ddiv_rn(__dadd_rn((double)t, 1.0), t2);
  wa = __ddiv_rn(1.0, t2);
}

__device__ __forceinline__ void mark_nonfinite(IterParams *P, long long k) {
  atomicMin(&P->nonfinite_k, (unsigned long long)k);
}

// ---------------------------------------------------------------------------
// inner iteration: x phase over A^T rows (core.py:168-169 + 149-153)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_x_iter(TileMat AT, const double *__restrict__ y, double *__restrict__ x, double *__restrict__ w,
         const double *__restrict__ c, const double *__restrict__ lo, const double *__restrict__ up,
         const double *__restrict__ anc_x, IterParams *P, int step) {
  extern __shared__ double sprod[];
  int j;
  bool active;
  const double aty = tile_row_sum(AT, y, sprod, j, active);
  if (!active) return;
  const double sigma = P->sigma;
  const int variant = P->variant;
  const long long t = P->t0 + step;
  const double xj = x[j];
  const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, c[j])));
  const double xb = np_clip(v, lo[j], up[j]);
  const double wj = __dsub_rn(__dmul_rn(2.0, xb), xj);
  double xn;
  if (variant == 0) {
    xn = xb;
  } else {
    double wa, wn;
    halpern_weights(t, wa, wn);
    xn = __dadd_rn(__dmul_rn(wa, anc_x[j]), __dmul_rn(wn, variant == 2 ? wj : xb));
  }
  w[j] = wj;
  x[j] = xn;
  if (!isfinite(xn)) mark_nonfinite(P, P->k0 + step);
}

// y phase over A rows (core.py:170-172 + 149-153); y updated in place.
__global__ void __launch_bounds__(kThreads)
k_y_iter(TileMat A, const double *__restrict__ w, double *__restrict__ y,
         const double *__restrict__ b, const double *__restrict__ anc_y, int m1, IterParams *P,
         int step) {
  extern __shared__ double sprod[];
  int i;
  bool active;
  const double s = tile_row_sum(A, w, sprod, i, active);
  if (!active) return;
  const int variant = P->variant;
  const long long t = P->t0 + step;
  const double yi = y[i];
  double yb = __dadd_rn(yi, __ddiv_rn(__dsub_rn(b[i], s), P->lamsig));
  if (i >= m1) yb = np_max(yb, 0.0);
  double yn;
  if (variant == 0) {
    yn = yb;
  } else {
    double wa, wn;
    halpern_weights(t, wa, wn);
    const double tgt = variant == 2 ? __dsub_rn(__dmul_rn(2.0, yb), yi) : yb;
    yn = __dadd_rn(__dmul_rn(wa, anc_y[i]), __dmul_rn(wn, tgt));
  }
  y[i] = yn;
  if (!isfinite(yn)) mark_nonfinite(P, P->k0 + step);
}

// ---------------------------------------------------------------------------
// checkpoint kernels
// ---------------------------------------------------------------------------
struct CandCtx {
  int term_original;
  const double *b_factor_c_factor;   // device [bf, cf]
  const double *row_scale, *col_scale;
  const double *lo0, *up0;           // original bounds (clip target)
};

// half step x part (core.py:123-125) + candidate unscale/clip (scaling.py:46,48;
// driver.py:334-336) + ||xb - anchor_x||^2 and ||x - xb||^2.
__global__ void __launch_bounds__(kThreads)
k_x_half(TileMat AT, const double *__restrict__ y, const double *__restrict__ x,
         const double *__restrict__ c, const double *__restrict__ lo, const double *__restrict__ up,
         const double *__restrict__ anc_x, double *__restrict__ xb_out, double *__restrict__ zb_out,
         double *__restrict__ wtmp, double *__restrict__ cx_out, double *__restrict__ cz_out,
         CandCtx cc, double sigma, double *part) {
  extern __shared__ double sprod[];
  int j;
  bool active;
  const double aty = tile_row_sum(AT, y, sprod, j, active);
  double acc[2] = {0.0, 0.0};
  if (active) {
    const double xj = x[j];
    const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, c[j])));
    const double xb = np_clip(v, lo[j], up[j]);
    const double zb = __ddiv_rn(__dsub_rn(xb, v), sigma);
    xb_out[j] = xb;
    zb_out[j] = zb;
    wtmp[j] = __dsub_rn(__dmul_rn(2.0, xb), xj);
    acc[0] = sq(__dsub_rn(xb, anc_x[j]));
    acc[1] = sq(__dsub_rn(xj, xb));
    if (cc.term_original) {
      const double bf = cc.b_factor_c_factor[0], cf = cc.b_factor_c_factor[1];
      const double cs = cc.col_scale[j];
      cx_out[j] = np_clip(__dmul_rn(xb, __ddiv_rn(bf, cs)), cc.lo0[j], cc.up0[j]);
      cz_out[j] = __dmul_rn(zb, __dmul_rn(cf, cs));
    } else {
      cx_out[j] = xb;
      cz_out[j] = zb;
    }
  }
  block_reduce_store<2>(acc, part, gridDim.x);
}

// half step y part (core.py:126-128) + candidate y + ||y - yb||^2, ||yb - anchor_y||^2.
__global__ void __launch_bounds__(kThreads)
k_y_half(TileMat A, const double *__restrict__ wtmp, const double *__restrict__ y,
         const double *__restrict__ b, const double *__restrict__ anc_y, int m1, double lamsig,
         double *__restrict__ yb_out, double *__restrict__ dy_out, double *__restrict__ cy_out,
         CandCtx cc, double *part) {
  extern __shared__ double sprod[];
  int i;
  bool active;
  const double s = tile_row_sum(A, wtmp, sprod, i, active);
  double acc[2] = {0.0, 0.0};
  if (active) {
    const double yi = y[i];
    double yb = __dadd_rn(yi, __ddiv_rn(__dsub_rn(b[i], s), lamsig));
    if (i >= m1) yb = np_max(yb, 0.0);
    const double dy = __dsub_rn(yi, yb);
    yb_out[i] = yb;
    dy_out[i] = dy;
    acc[0] = sq(dy);
    acc[1] = sq(__dsub_rn(yb, anc_y[i]));
    cy_out[i] = cc.term_original
                    ? __dmul_rn(yb, __ddiv_rn(cc.b_factor_c_factor[1], cc.row_scale[i]))
                    : yb;
  }
  block_reduce_store<2>(acc, part, gridDim.x);
}

// KKT row terms over the termination problem's A (driver.py:203-206, 211, 214).
__global__ void __launch_bounds__(kThreads)
k_kkt_row(TileMat A, const double *__restrict__ cx, const double *__restrict__ cy,
          const double *__restrict__ b, int m1, double *part) {
  extern __shared__ double sprod[];
  int i;
  bool active;
  const double ax = tile_row_sum(A, cx, sprod, i, active);
  double acc[3] = {0.0, 0.0, 0.0};
  if (active) {
    const double bi = b[i], yi = cy[i];
    double prim = __dsub_rn(bi, ax);
    double tproj = __dadd_rn(__dsub_rn(yi, ax), bi);
    if (i >= m1) {
      prim = np_max(prim, 0.0);
      tproj = np_max(tproj, 0.0);
    }
    acc[0] = sq(prim);
    acc[1] = __dmul_rn(bi, yi);
    acc[2] = sq(__dsub_rn(yi, tproj));
  }
  block_reduce_store<3>(acc, part, gridDim.x);
}

// KKT column terms over the termination problem's A^T (driver.py:207-215,
// problem.py:146-176).
__global__ void __launch_bounds__(kThreads)
k_kkt_col(TileMat AT, const double *__restrict__ cy, const double *__restrict__ cx,
          const double *__restrict__ cz, const double *__restrict__ c, const double *__restrict__ lo,
          const double *__restrict__ up, double *part) {
  extern __shared__ double sprod[];
  int j;
  bool active;
  const double aty = tile_row_sum(AT, cy, sprod, j, active);
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (active) {
    const double cj = c[j], zj = cz[j], xj = cx[j], l = lo[j], u = up[j];
    acc[0] = sq(__dsub_rn(__dsub_rn(cj, aty), zj));
    acc[1] = __dmul_rn(cj, xj);
    if (zj > 0.0) {
      if (isfinite(l)) { acc[2] = __dmul_rn(l, zj); acc[4] = 1.0; } else { acc[6] = 1.0; }
    } else if (zj < 0.0) {
      if (isfinite(u)) { acc[3] = __dmul_rn(u, zj); acc[5] = 1.0; } else { acc[6] = 1.0; }
    }
    acc[7] = sq(__dsub_rn(xj, np_clip(__dsub_rn(xj, zj), l, u)));
  }
  block_reduce_store<8>(acc, part, gridDim.x);
}

// merit terms over the scaled A^T (core.py:191-197): aty = A^T dy.
__global__ void __launch_bounds__(kThreads)
k_merit_col(TileMat AT, const double *__restrict__ dy, const double *__restrict__ x,
            const double *__restrict__ xb, double sigma, double *part) {
  extern __shared__ double sprod[];
  int j;
  bool active;
  const double aty = tile_row_sum(AT, dy, sprod, j, active);
  double acc[2] = {0.0, 0.0};
  if (active) {
    const double dx = __dsub_rn(x[j], xb[j]);
    acc[0] = sq(__dadd_rn(dx, __dmul_rn(sigma, aty)));
    acc[1] = sq(aty);
  }
  block_reduce_store<2>(acc, part, gridDim.x);
}

// ---------------------------------------------------------------------------
// fixed-order final reduction: one CTA per segment
// ---------------------------------------------------------------------------
struct RedSeg {
  const double *src;
  int count;
  int out;
};
struct RedList {
  RedSeg seg[24];
  int nseg;
};

__global__ void __launch_bounds__(kThreads) k_reduce_final(RedList L, double *out) {
  const RedSeg sg = L.seg[blockIdx.x];
  double a[1] = {0.0};
  for (int i = threadIdx.x; i < sg.count; i += kThreads) a[0] = __dadd_rn(a[0], sg.src[i]);
  block_reduce<1>(a);
  if (threadIdx.x == 0) out[sg.out] = a[0];
}

// ---------------------------------------------------------------------------
// power method (sparse.py:176-198) -- all decisions on the device
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_pow_t(TileMat AT, const double *__restrict__ v, double *__restrict__ u, const PowState *S,
        double *part) {
  if (S->done) return;
  extern __shared__ double sprod[];
  int j;
  bool active;
  const double s = tile_row_sum(AT, v, sprod, j, active);
  double acc[1] = {0.0};
  if (active) {
    u[j] = s;
    acc[0] = sq(s);
  }
  block_reduce_store<1>(acc, part, gridDim.x);
}

__global__ void __launch_bounds__(kThreads)
k_pow_a(TileMat A, const double *__restrict__ u, const double *__restrict__ v,
        double *__restrict__ wv, const PowState *S, double *part) {
  if (S->done) return;
  extern __shared__ double sprod[];
  int i;
  bool active;
  const double s = tile_row_sum(A, u, sprod, i, active);
  double acc[2] = {0.0, 0.0};
  if (active) {
    wv[i] = s;
    acc[0] = __dmul_rn(v[i], s);
    acc[1] = sq(s);
  }
  block_reduce_store<2>(acc, part, gridDim.x);
}

// one CTA: reduce the v.w and w.w partials in fixed order, then the scalar
// logic of one power step (sparse.py:188-198).
__global__ void __launch_bounds__(kThreads) k_pow_step(const double *part, int ntiles, PowState *S) {
  if (S->done) return;
  double a[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < ntiles; i += kThreads) {
    a[0] = __dadd_rn(a[0], part[i]);
    a[1] = __dadd_rn(a[1], part[ntiles + i]);
  }
  block_reduce<2>(a);
  if (threadIdx.x == 0) {
    const double lam = a[0];
    const double nw = sqrt(a[1]);
    S->iters += 1;
    S->lam = lam;
    S->nw = nw;
    if (nw == 0.0) {
      S->done = 1;                       // break before v = w / nw
      return;
    }
    S->norm_pending = 1;                 // v = w / nw
    if (S->iters > 1 && fabs(__dsub_rn(lam, S->lam_prev)) <=
                            __dmul_rn(S->tol, fmax(fabs(lam), 1e-300))) {
      S->converged = 1;
      S->done = 1;
    } else {
      S->lam_prev = lam;
      if (S->iters >= S->max_iters) S->done = 1;
    }
  }
}

__global__ void k_pow_norm(const double *__restrict__ wv, double *__restrict__ v, int m,
                           PowState *S) {
  if (!S->norm_pending) return;
  const double nw = S->nw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    v[i] = __ddiv_rn(wv[i], nw);
}

__global__ void k_pow_norm_done(PowState *S) { S->norm_pending = 0; }

// ---------------------------------------------------------------------------
// setup kernels: transpose helpers, tiling, scaling
// ---------------------------------------------------------------------------
__global__ void k_iota(int *a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

__global__ void k_row_of(const int *rp, int nrows, int *row_of) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x)
    for (int k = rp[i]; k < rp[i + 1]; ++k) row_of[k] = i;
}

__global__ void k_col_count(const int *sorted_cols, long long nnz, int ncols, int *rpt) {
  // rpt[j] = first position of column j in the sorted key array (lower bound);
  // written by the entry that starts each run, gaps filled for empty columns.
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int cur = sorted_cols[k];
    const int prev = k == 0 ? -1 : sorted_cols[k - 1];
    for (int j = prev + 1; j <= cur; ++j) rpt[j] = (int)k;
    if (k == nnz - 1)
      for (int j = cur + 1; j <= ncols; ++j) rpt[j] = (int)nnz;
  }
}

__global__ void k_fill_empty_rpt(int *rpt, int ncols) {
  // nnz == 0 corner: all offsets zero
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= ncols; j += gridDim.x * blockDim.x)
    rpt[j] = 0;
}

__global__ void k_gather_t(const int *perm, const int *row_of, const double *val, int *at_ci,
                          double *at_val, long long nnz) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int p = perm[k];
    at_ci[k] = row_of[p];
    at_val[k] = val[p];
  }
}

// tile boundaries: a new tile starts at row i if i is a multiple of kThreads
// rows into ... (see analyze()): bucket change, row-group change, or a long row.
__global__ void k_tile_flags(const int *rp, int nrows, int bucket, int long_len, int *flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x) {
    int f;
    if (i == 0) {
      f = 1;
    } else {
      const int len_i = rp[i + 1] - rp[i], len_p = rp[i] - rp[i - 1];
      f = (i % kThreads == 0) || (rp[i] / bucket != rp[i - 1] / bucket) || (len_i > long_len) ||
          (len_p > long_len);
    }
    flags[i] = f;
  }
}

__global__ void k_tile_scatter(const int *flags, const int *pos, int nrows, int *tile_row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x) {
    if (flags[i]) tile_row[pos[i]] = i;
    if (i == nrows - 1) {
      const int nt = pos[i] + flags[i];
      tile_row[nt] = nrows;
    }
  }
}

// Ruiz: per-row max |a| (exact; any order), per-column via the transpose perm.
__global__ void k_row_maxabs(const int *rp, const double *val, int nrows, double *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x) {
    double mx = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) mx = fmax(mx, fabs(val[k]));
    out[i] = mx;
  }
}
__global__ void k_col_maxabs(const int *rpt, const int *perm, const double *val, int ncols,
                             double *out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += gridDim.x * blockDim.x) {
    double mx = 0.0;
    for (int k = rpt[j]; k < rpt[j + 1]; ++k) mx = fmax(mx, fabs(val[perm[k]]));
    out[j] = mx;
  }
}
// Pock-Chambolle alpha = 1: sequential abs sums (np.add.at order, sparse.py:235,237).
__global__ void k_row_abssum(const int *rp, const double *val, int nrows, double *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) s = __dadd_rn(s, fabs(val[k]));
    out[i] = s;
  }
}
__global__ void k_col_abssum(const int *rpt, const int *perm, const double *val, int ncols,
                             double *out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = rpt[j]; k < rpt[j + 1]; ++k) s = __dadd_rn(s, fabs(val[perm[k]]));
    out[j] = s;
  }
}
// d = sqrt(s); d==0 -> 1; acc *= d  (sparse.py:217-223, 238-241)
__global__ void k_sqrt_div(double *d, double *acc, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = sqrt(d[i]);
    if (v == 0.0) v = 1.0;
    d[i] = v;
    acc[i] = __dmul_rn(acc[i], v);
  }
}
// vals / dr[row] / dc[col] (sparse.py:127): two divisions, left to right.
__global__ void k_scale_vals(const int *rp, const int *ci, double *val, const double *dr,
                             const double *dc, int nrows) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nrows; i += nwarps) {
    const double d = dr[i];
    for (int k = rp[i] + lane; k < rp[i + 1]; k += 32) val[k] = __ddiv_rn(__ddiv_rn(val[k], d), dc[ci[k]]);
  }
}
__global__ void k_gather_vals(const int *perm, const double *src, double *dst, long long nnz) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x)
    dst[k] = src[perm[k]];
}
__global__ void k_fill(double *a, double v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}
// scaling.py:93-96: b / row_div, c / col_div, l * col_div, u * col_div
__global__ void k_scale_vecs(const double *b, const double *rd, double *bs, int m, const double *c,
                             const double *lo, const double *up, const double *cd, double *cs,
                             double *los, double *ups, int n) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < m; i += nt) bs[i] = __ddiv_rn(b[i], rd[i]);
  for (int j = tid; j < n; j += nt) {
    const double d = cd[j];
    cs[j] = __ddiv_rn(c[j], d);
    los[j] = __dmul_rn(lo[j], d);
    ups[j] = __dmul_rn(up[j], d);
  }
}
// per-CTA partial of sum a_i^2 (for ||b||, ||c||); part[blockIdx.x]
__global__ void __launch_bounds__(kThreads) k_sumsq(const double *a, long long n, double *part) {
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    acc[0] = __dadd_rn(acc[0], sq(a[i]));
  block_reduce_store<1>(acc, part, gridDim.x);
}
// scaling.py:98-101 with bf = sqrt(sum b^2) + 1 computed here from reduced sums
__global__ void k_bc_normalize(double *bs, int m, double *cs, double *los, double *ups, int n,
                               const double *fac) {
  const double bf = fac[0], cf = fac[1];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < m; i += nt) bs[i] = __ddiv_rn(bs[i], bf);
  for (int j = tid; j < n; j += nt) {
    cs[j] = __ddiv_rn(cs[j], cf);
    los[j] = __ddiv_rn(los[j], bf);
    ups[j] = __ddiv_rn(ups[j], bf);
  }
}
__global__ void k_factors(const double *sums, double *fac) {
  // sums = [sum b_s^2, sum c_s^2]; fac = [bf, cf]
  if (threadIdx.x == 0) {
    fac[0] = __dadd_rn(sqrt(sums[0]), 1.0);
    fac[1] = __dadd_rn(sqrt(sums[1]), 1.0);
  }
}

// candidate at the origin (driver.py:376-379) and final unscale (driver.py:382-384)
__global__ void k_origin_cand(double *cy, int m, double *cz, double *cx, const double *lo,
                              const double *up, int n) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < m; i += nt) cy[i] = 0.0;
  for (int j = tid; j < n; j += nt) {
    cz[j] = 0.0;
    cx[j] = np_clip(0.0, lo[j], up[j]);
  }
}
__global__ void k_unscale(const double *sy, const double *sz, const double *sx, double *oy,
                          double *oz, double *ox, const double *rs, const double *cs,
                          const double *fac, const double *lo0, const double *up0, int m, int n) {
  const double bf = fac[0], cf = fac[1];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < m; i += nt) oy[i] = __dmul_rn(sy[i], __ddiv_rn(cf, rs[i]));
  for (int j = tid; j < n; j += nt) {
    const double c = cs[j];
    ox[j] = np_clip(__dmul_rn(sx[j], __ddiv_rn(bf, c)), lo0[j], up0[j]);
    oz[j] = __dmul_rn(sz[j], __dmul_rn(cf, c));
  }
}

__global__ void k_set_params(IterParams *P, double sigma, double lamsig, long long t0,
                             long long k0, int variant) {
  P->sigma = sigma;
  P->lamsig = lamsig;
  P->t0 = t0;
  P->k0 = k0;
  P->variant = variant;
}

}  // namespace hpr
