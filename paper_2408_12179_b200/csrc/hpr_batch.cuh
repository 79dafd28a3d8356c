// hpr_batch.cuh -- K11: a batch of small LPs, one whole restarted HPR solve per CTA
// (BASELINE config C5: 4096 x (m=500, n=1000, nnz=5000)).
//
// Included at the end of hpr_capi.cu.  Each CTA owns one LP for the whole
// solve: it stages the LP's CSR A and CSR A^T (scaled values), the iterate, the
// anchors and the scaled problem vectors in shared memory (~210 KB at C5) and
// runs the reference's complete pipeline on the SM with no host round trip:
//
//   scale_problem            scaling.py:72-125 (Ruiz x10, Pock-Chambolle, b/c norm)
//   power_method_lambda_max  sparse.py:165-203
//   the restarted loop       driver.py:317-372 (iterate_once core.py:163-174,
//                            half_step 118-129, kkt_residual driver.py:191-228,
//                            merit core.py:182-218, restart rules 238-248,
//                            sigma update 251-278, status priority 341-346)
//   the report               driver.py:374-391
//
// Arithmetic order is the single-LP path's: every sparse product is a
// sequential left-to-right sum of separately rounded products (scipy
// csr_matvec), one thread per row (x-phase: per column over A^T).  Norms and
// dots are fixed-order block reductions (warp shuffle tree, then the 16 warp
// partials summed in warp order), evaluated identically by every thread so the
// scalar decisions need no broadcast.  Original-value KKT terms read A and A^T
// from global memory (L2) at checkpoints only.
#pragma once

namespace hpr {
namespace batch {

#ifndef HPR_BATCH_THREADS
#define HPR_BATCH_THREADS 512
#endif
constexpr int kBT = HPR_BATCH_THREADS;   // threads per CTA (one LP)
constexpr int kWTab = 256;          // Halpern weights tabulated per refill
constexpr int kBW = kBT / 32;

struct Prob {
  const int64_t *row_off, *col_off, *nz_off;
  const int *m1;
  const int *rp;                    // LP i's local row pointers at row_off[i] + i
  const int *ci;
  const double *val;
  const int *grpt;                  // transpose row pointers (global positions), col_off[i] + i
  const int *cit;                   // transpose column indices (local rows)
  const double *valt;               // transpose original values
  const double *b, *c, *lo, *up;
  const double *obj_const;
  const int *obj_neg;
};

struct Cfg {
  double tol, time_limit, a1, a2, a3, sigma0, power_tol;
  long long max_iter;
  int check_interval, variant, uses_restarts, updates_sigma;
  int ruiz, pc, bc, power_max, term_original, max_log;
};

struct Out {
  hpr_batch_result *res;
  hpr_restart_rec *log;
  double *x, *y, *z;                // solution (also the checkpoint candidate)
  double *dy;                       // scratch, row-indexed
};

// fixed-order block sum of NQ values; every thread receives the totals
template <int NQ>
__device__ __forceinline__ void bsum(double (&v)[NQ], double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double a = v[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, off));
    if (lane == 0) red[q * kBW + warp] = a;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double s = 0.0;
    for (int w = 0; w < kBW; ++w) s = __dadd_rn(s, red[q * kBW + w]);
    v[q] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef HPR_BATCH_PROF
#define HPR_BATCH_PROF 0
#endif
#ifndef HPR_BATCH_SROW
#define HPR_BATCH_SROW 1   // 1: batches of 4 entries (loads in flight together, then the ordered adds)
#endif

// Shared-memory matrices are stored POSITION-MAJOR: rows sorted by length
// (longest first, perm[p] = row at position p), row p's entries contiguous
// from st[p] in ascending column order, every row padded to an odd length so
// the 32 lanes of a warp (consecutive positions, equal lengths) hit distinct
// shared-memory banks (the CSR layout put 4-way conflicts on every load).
// Column indices are 16-bit (LPs of a batch have < 65536 rows and columns).
typedef unsigned short u16;

// sequential sum of the row at position p against vector v
__device__ __forceinline__ double srow(const int *st, const u16 *ln, const u16 *ci,
                                       const double *val, const double *v, int p) {
  double s = 0.0;
  int e = st[p];
  const int e1 = e + ln[p];
#if HPR_BATCH_SROW
  for (; e + 4 <= e1; e += 4) {
    int c[4];
    double a[4], x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = ci[e + u];
      a[u] = val[e + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = v[c[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) s = __dadd_rn(s, __dmul_rn(a[u], x[u]));
  }
#endif
  for (; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(val[e], v[ci[e]]));
  return s;
}

// two rows at once (independent chains interleaved: twice the shared-memory
// loads in flight per thread); each row still summed left to right.  p1 < 0: none
__device__ __forceinline__ void srow2(const int *st, const u16 *ln, const u16 *ci,
                                      const double *val, const double *v, int p0, int p1,
                                      double &s0, double &s1) {
  s0 = 0.0;
  s1 = 0.0;
  int e0 = st[p0], e1 = p1 >= 0 ? st[p1] : 0;
  const int z0 = e0 + ln[p0], z1 = p1 >= 0 ? e1 + ln[p1] : 0;
#if HPR_BATCH_SROW
  while (e0 + 2 <= z0 && e1 + 2 <= z1) {
    const int c0 = ci[e0], c1 = ci[e0 + 1], d0 = ci[e1], d1 = ci[e1 + 1];
    const double a0 = val[e0], a1 = val[e0 + 1], b0 = val[e1], b1 = val[e1 + 1];
    const double x0 = v[c0], x1 = v[c1], y0 = v[d0], y1 = v[d1];
    s0 = __dadd_rn(s0, __dmul_rn(a0, x0));
    s1 = __dadd_rn(s1, __dmul_rn(b0, y0));
    s0 = __dadd_rn(s0, __dmul_rn(a1, x1));
    s1 = __dadd_rn(s1, __dmul_rn(b1, y1));
    e0 += 2;
    e1 += 2;
  }
#endif
  while (e0 < z0 && e1 < z1) {
    const double q0 = __dmul_rn(val[e0], v[ci[e0]]);
    const double q1 = __dmul_rn(val[e1], v[ci[e1]]);
    s0 = __dadd_rn(s0, q0);
    s1 = __dadd_rn(s1, q1);
    ++e0;
    ++e1;
  }
  for (; e0 < z0; ++e0) s0 = __dadd_rn(s0, __dmul_rn(val[e0], v[ci[e0]]));
  for (; e1 < z1; ++e1) s1 = __dadd_rn(s1, __dmul_rn(val[e1], v[ci[e1]]));
}

// same for a global-memory CSR (original values at checkpoints); v in global
// memory written earlier by this CTA (plain coherent loads, no __ldg)
__device__ __forceinline__ double grow(const int *rp, int base, const int *ci, const double *val,
                                       const double *v, int r) {
  double s = 0.0;
  const int e1 = rp[r + 1] - base;
  for (int e = rp[r] - base; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(val[e], v[ci[e]]));
  return s;
}

size_t smem_bytes(int m, int n, long long nnz) {
  const size_t slots = 2 * (size_t)nnz + m + n;  // A and A^T, rows padded to odd lengths
  size_t b = 0;
  b += slots * 8;                              // av, atv
  b += 8 * (size_t)(5 * m + 8 * n);            // y ay bs yb rs | x ax w cs ls us csc xb
  b += 4 * (size_t)(m + n);                    // ast, atst (row starts by position)
  b += slots * 2;                              // aci, atci (16-bit)
  b += 2 * (size_t)(m + n) * 2;                // alen, atlen, aperm, atperm
  b = (b + 15) / 16 * 16;
  b += 8 * (size_t)24 * kBW;                   // reduction scratch
  b += 16 * (size_t)kWTab;                     // Halpern weight table
  return b;
}

__global__ void __launch_bounds__(kBT, 1) k_batch_solve(Prob P, Cfg C, Out O) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lp = blockIdx.x, tid = threadIdx.x;
  const unsigned long long t_start = gtimer();
#if HPR_BATCH_PROF
  const long long tk0 = clock64();
#endif
  const long long r0 = P.row_off[lp], c0 = P.col_off[lp], z0 = P.nz_off[lp];
  const int m = (int)(P.row_off[lp + 1] - r0), n = (int)(P.col_off[lp + 1] - c0);
  const int nnz = (int)(P.nz_off[lp + 1] - z0);
  const int m1 = P.m1[lp];
  // ---- carve shared memory ----
  double *p = (double *)smraw;
  double *av = p; p += nnz + m;
  double *atv = p; p += nnz + n;
  double *y = p; p += m;
  double *ay = p; p += m;
  double *bs = p; p += m;
  double *yb = p; p += m;
  double *rs = p; p += m;
  double *x = p; p += n;
  double *ax = p; p += n;
  double *w = p; p += n;
  double *cs = p; p += n;
  double *ls = p; p += n;
  double *us = p; p += n;
  double *csc = p; p += n;
  double *xb = p; p += n;
  int *ast = (int *)p;
  int *atst = ast + m;
  u16 *aci = (u16 *)(atst + n);
  u16 *atci = aci + nnz + m;
  u16 *alen = atci + nnz + n;
  u16 *atlen = alen + m;
  u16 *aperm = atlen + n;
  u16 *atperm = aperm + m;
  double *red = (double *)(((uintptr_t)(atperm + n) + 15) & ~(uintptr_t)15);
  double *wtab = red + 24 * kBW;
  // global views of this LP
  const int *grp = P.rp + r0 + lp;             // local row pointers (m + 1)
  const int *gci = P.ci + z0;
  const double *gval = P.val + z0;
  const int *gtrp = P.grpt + c0 + lp;          // global positions (n + 1)
  const int *gtci = P.cit + z0;
  const double *gtval = P.valt + z0;
  const double *b0 = P.b + r0, *c0v = P.c + c0, *l0 = P.lo + c0, *u0 = P.up + c0;
  double *ox = O.x + c0, *oy = O.y + r0, *oz = O.z + c0, *gdy = O.dy + r0;
  const int tz = (int)z0;

  // ---- position-major shared-memory copies of A and A^T ----
  // ranks by (length desc, index asc); the lengths are staged in shared
  // memory first (yb / xb as scratch: written again before their first use),
  // so the all-pairs rank loop reads broadcast shared-memory words
  int *lenA = (int *)yb, *lenT = (int *)xb;
  u16 *rankA = (u16 *)ay, *rankT = (u16 *)ax;   // row / column -> position (scratch too)
  for (int i = tid; i < m; i += kBT) lenA[i] = grp[i + 1] - grp[i];
  for (int j = tid; j < n; j += kBT) lenT[j] = gtrp[j + 1] - gtrp[j];
  __syncthreads();
  for (int i = tid; i < m; i += kBT) {
    const int li = lenA[i];
    int rank = 0;
    for (int q = 0; q < m; ++q) {
      const int lq = lenA[q];
      rank += (lq > li) || (lq == li && q < i);
    }
    aperm[rank] = (u16)i;
    alen[rank] = (u16)li;
    rankA[i] = (u16)rank;
  }
  for (int j = tid; j < n; j += kBT) {
    const int lj = lenT[j];
    int rank = 0;
    for (int q = 0; q < n; ++q) {
      const int lq = lenT[q];
      rank += (lq > lj) || (lq == lj && q < j);
    }
    atperm[rank] = (u16)j;
    atlen[rank] = (u16)lj;
    rankT[j] = (u16)rank;
  }
  __syncthreads();
  if (tid == 0) {                                // row starts, every row padded to odd length
    int o = 0;
    for (int q = 0; q < m; ++q) {
      ast[q] = o;
      o += alen[q] | 1;
    }
  } else if (tid == 32) {
    int o = 0;
    for (int q = 0; q < n; ++q) {
      atst[q] = o;
      o += atlen[q] | 1;
    }
  }
  __syncthreads();
  for (int q = tid; q < m; q += kBT) {
    const int i = aperm[q], g0 = grp[i], L = alen[q], o = ast[q];
    for (int k2 = 0; k2 < L; ++k2) {
      av[o + k2] = gval[g0 + k2];
      aci[o + k2] = rankT[gci[g0 + k2]];     // column ids -> A^T positions
    }
    if (!(L & 1)) {
      av[o + L] = 0.0;
      aci[o + L] = 0;
    }
  }
  for (int q = tid; q < n; q += kBT) {
    const int j = atperm[q], g0 = gtrp[j] - tz, L = atlen[q], o = atst[q];
    for (int k2 = 0; k2 < L; ++k2) {
      atv[o + k2] = gtval[g0 + k2];
      atci[o + k2] = rankA[gtci[g0 + k2]];   // row ids -> A positions
    }
    if (!(L & 1)) {
      atv[o + L] = 0.0;
      atci[o + L] = 0;
    }
  }
  for (int i = tid; i < m; i += kBT) rs[i] = 1.0;
  for (int j = tid; j < n; j += kBT) csc[j] = 1.0;
  __syncthreads();

  // ---- scale_problem (scaling.py:81-103) ----
  // one pass: row divisors in yb, column divisors in xb, then both value copies
  // become (v / dr[row]) / dc[col]
  // (POSITION SPACE: every m-vector is indexed by the A position q of row
  // aperm[q], every n-vector by the A^T position of column atperm[q]; the
  // stored column ids are positions too, so all loops below are coalesced)
  auto apply_pass = [&]() {
    for (int q = tid; q < m; q += kBT) {
      const double d = yb[q];
      rs[q] = __dmul_rn(rs[q], d);
      for (int e = ast[q]; e < ast[q] + alen[q]; ++e) av[e] = __ddiv_rn(__ddiv_rn(av[e], d), xb[aci[e]]);
    }
    for (int q = tid; q < n; q += kBT) {
      const double d = xb[q];
      csc[q] = __dmul_rn(csc[q], d);
      for (int e = atst[q]; e < atst[q] + atlen[q]; ++e)
        atv[e] = __ddiv_rn(__ddiv_rn(atv[e], yb[atci[e]]), d);
    }
    __syncthreads();
  };
  for (int it = 0; it < C.ruiz; ++it) {
    for (int q = tid; q < m; q += kBT) {
      double mx = 0.0;
      for (int e = ast[q]; e < ast[q] + alen[q]; ++e) mx = fmax(mx, fabs(av[e]));
      double d = sqrt(mx);
      yb[q] = d == 0.0 ? 1.0 : d;
    }
    for (int q = tid; q < n; q += kBT) {
      double mx = 0.0;
      for (int e = atst[q]; e < atst[q] + atlen[q]; ++e) mx = fmax(mx, fabs(atv[e]));
      double d = sqrt(mx);
      xb[q] = d == 0.0 ? 1.0 : d;
    }
    __syncthreads();
    apply_pass();
  }
  if (C.pc) {
    for (int q = tid; q < m; q += kBT) {
      double s = 0.0;
      for (int e = ast[q]; e < ast[q] + alen[q]; ++e) s = __dadd_rn(s, fabs(av[e]));
      double d = sqrt(s);
      yb[q] = d == 0.0 ? 1.0 : d;
    }
    for (int q = tid; q < n; q += kBT) {
      double s = 0.0;
      for (int e = atst[q]; e < atst[q] + atlen[q]; ++e) s = __dadd_rn(s, fabs(atv[e]));
      double d = sqrt(s);
      xb[q] = d == 0.0 ? 1.0 : d;
    }
    __syncthreads();
    apply_pass();
  }
  for (int q = tid; q < m; q += kBT) bs[q] = __ddiv_rn(b0[aperm[q]], rs[q]);
  for (int q = tid; q < n; q += kBT) {
    const int j = atperm[q];
    cs[q] = __ddiv_rn(c0v[j], csc[q]);
    ls[q] = __dmul_rn(l0[j], csc[q]);
    us[q] = __dmul_rn(u0[j], csc[q]);
  }
  __syncthreads();
  double bf = 1.0, cf = 1.0;
  if (C.bc) {
    double v2[2] = {0.0, 0.0};
    for (int i = tid; i < m; i += kBT) v2[0] = __dadd_rn(v2[0], sq(bs[i]));
    for (int j = tid; j < n; j += kBT) v2[1] = __dadd_rn(v2[1], sq(cs[j]));
    bsum<2>(v2, red);
    bf = __dadd_rn(sqrt(v2[0]), 1.0);
    cf = __dadd_rn(sqrt(v2[1]), 1.0);
    for (int i = tid; i < m; i += kBT) bs[i] = __ddiv_rn(bs[i], bf);
    for (int j = tid; j < n; j += kBT) {
      cs[j] = __ddiv_rn(cs[j], cf);
      ls[j] = __ddiv_rn(ls[j], bf);
      us[j] = __ddiv_rn(us[j], bf);
    }
    __syncthreads();
  }
  // ||b||, ||c|| of the termination problem (relative residual denominators)
  double bnorm, cnorm;
  {
    double v2[2] = {0.0, 0.0};
    for (int q = tid; q < m; q += kBT) v2[0] = __dadd_rn(v2[0], sq(C.term_original ? b0[aperm[q]] : bs[q]));
    for (int q = tid; q < n; q += kBT) v2[1] = __dadd_rn(v2[1], sq(C.term_original ? c0v[atperm[q]] : cs[q]));
    bsum<2>(v2, red);
    bnorm = sqrt(v2[0]);
    cnorm = sqrt(v2[1]);
  }

#if HPR_BATCH_PROF
  long long tp_setup = clock64(), tp_pow = 0, tp_it = 0, tp_ck = 0;
#endif
  // ---- power method (sparse.py:165-203): v in yb, u in w, A u in ay ----
  int start = -2;
  for (int fb = -1; fb < m; ++fb) {
    for (int q = tid; q < m; q += kBT) yb[q] = fb < 0 ? 1.0 : ((int)aperm[q] == fb ? 1.0 : 0.0);
    __syncthreads();
    double u2[1] = {0.0};
    for (int q = tid; q < n; q += kBT) u2[0] = __dadd_rn(u2[0], sq(srow(atst, atlen, atci, atv, yb, q)));
    bsum<1>(u2, red);
    if (sqrt(u2[0]) > 0.0) {
      start = fb;
      break;
    }
  }
  double lam = 0.0, lam_prev = 0.0;
  int piters = 0, pconv = 0;
  if (start == -1) {
    const double inv = 1.0 / sqrt((double)m);
    for (int i = tid; i < m; i += kBT) yb[i] = inv;
  }
  __syncthreads();
  if (start != -2) {
    for (int it = 1; it <= C.power_max; ++it) {
      piters = it;
      for (int q = tid; q < n; q += kBT) w[q] = srow(atst, atlen, atci, atv, yb, q);
      __syncthreads();
      double d2[2] = {0.0, 0.0};
      for (int q = tid; q < m; q += kBT) {
        const double s = srow(ast, alen, aci, av, w, q);
        ay[q] = s;
        d2[0] = __dadd_rn(d2[0], __dmul_rn(yb[q], s));
        d2[1] = __dadd_rn(d2[1], sq(s));
      }
      bsum<2>(d2, red);
      lam = d2[0];
      const double nw = sqrt(d2[1]);
      if (nw == 0.0) break;
      for (int i = tid; i < m; i += kBT) yb[i] = __ddiv_rn(ay[i], nw);
      __syncthreads();
      if (it > 1 && fabs(__dsub_rn(lam, lam_prev)) <= __dmul_rn(C.power_tol, fmax(fabs(lam), 1e-300))) {
        pconv = 1;
        break;
      }
      lam_prev = lam;
    }
  }
  const double lam_raw = lam;
  const double lamv = lam * (1.0 + 1e-3);

  // ---- state (SolverState.origin, core.py:110-115) ----
  for (int i = tid; i < m; i += kBT) y[i] = ay[i] = 0.0;
  for (int j = tid; j < n; j += kBT) x[j] = ax[j] = 0.0;
  __syncthreads();
  double sigma = C.sigma0;
  long long k = 0, t = 0;
  int r = 0, status = -1, nlog = 0, have_ckpt = 0, merit_neg = 0;
  bool have_first = false;
  double merit_first = 0.0, merit_prev = INFINITY;
  double kk[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double lz = 0.0, uz = 0.0;
  long long clamped = 0;
  const double oc = P.obj_const[lp];
  const bool term_orig = C.term_original != 0;

  // KKT terms of the candidate in (oy, oz, ox) on the termination problem;
  // results into kk[] (driver.py:203-216)
  auto kkt = [&](double (&s)[11]) {
    for (int q = tid; q < m; q += kBT) {
      const int i = aperm[q];
      // scaled termination space: the candidate is (yb, xb) in shared memory
      const double axi = term_orig ? grow(grp, 0, gci, gval, ox, i) : srow(ast, alen, aci, av, xb, q);
      const double bi = term_orig ? b0[i] : bs[q];
      const double yi = oy[i];
      double prim = __dsub_rn(bi, axi);
      double tproj = __dadd_rn(__dsub_rn(yi, axi), bi);
      if (i >= m1) {
        prim = np_max(prim, 0.0);
        tproj = np_max(tproj, 0.0);
      }
      s[0] = __dadd_rn(s[0], sq(prim));
      s[1] = __dadd_rn(s[1], __dmul_rn(bi, yi));
      s[2] = __dadd_rn(s[2], sq(__dsub_rn(yi, tproj)));
    }
    for (int q = tid; q < n; q += kBT) {
      const int j = atperm[q];
      const double aty = term_orig ? grow(gtrp, tz, gtci, gtval, oy, j) : srow(atst, atlen, atci, atv, yb, q);
      const double cj = term_orig ? c0v[j] : cs[q];
      const double l = term_orig ? l0[j] : ls[q];
      const double u = term_orig ? u0[j] : us[q];
      const double zj = oz[j], xj = ox[j];
      s[3] = __dadd_rn(s[3], sq(__dsub_rn(__dsub_rn(cj, aty), zj)));
      s[4] = __dadd_rn(s[4], __dmul_rn(cj, xj));
      if (zj > 0.0) {
        if (isfinite(l)) {
          s[5] = __dadd_rn(s[5], __dmul_rn(l, zj));
          s[7] += 1.0;
        } else {
          s[9] += 1.0;
        }
      } else if (zj < 0.0) {
        if (isfinite(u)) {
          s[6] = __dadd_rn(s[6], __dmul_rn(u, zj));
          s[8] += 1.0;
        } else {
          s[9] += 1.0;
        }
      }
      s[10] = __dadd_rn(s[10], sq(__dsub_rn(xj, np_clip(__dsub_rn(xj, zj), l, u))));
    }
  };
  auto kkt_finish = [&](const double (&s)[11]) {
    // s: prim2 by r1 dual2 cx lz uz nlo nup clamped r2   (kkt_from_sums)
    const double pa = sqrt(s[0]);
    const double pr = pa / (1.0 + bnorm);
    const double da = sqrt(s[3]);
    const double dr = da / (1.0 + cnorm);
    const double pobj = s[4] + oc;
    double dobj = s[1];
    if (s[7] != 0.0) dobj += s[5];
    if (s[8] != 0.0) dobj += s[6];
    dobj += oc;
    const double ga = fabs(dobj - pobj);
    const double gr = ga / (1.0 + fabs(dobj) + fabs(pobj));
    kk[0] = pa; kk[1] = pr; kk[2] = da; kk[3] = dr; kk[4] = ga; kk[5] = gr;
    kk[6] = sqrt(s[2] + s[10] + s[3]);
    kk[7] = pobj; kk[8] = dobj;
    lz = s[5]; uz = s[6];
    clamped = (long long)s[9];
  };

#if HPR_BATCH_PROF
  tp_pow = clock64();
#endif
#ifndef HPR_BATCH_REG
#define HPR_BATCH_REG 1
#endif
  const bool reg = HPR_BATCH_REG && n <= 2 * kBT && m <= kBT;
  while (status < 0) {
#if HPR_BATCH_PROF
    const long long tq0 = clock64();
#endif
    const long long steps = C.max_iter - k < C.check_interval ? C.max_iter - k : C.check_interval;
    const double lamsig = lamv * sigma;
    bool broke = false;
    const long long t_seg = t;
    if (reg) {
      // register-resident interval (HPR_BATCH_REG): thread tid owns columns
      // tid, tid + kBT and row tid for the whole interval, so x and the
      // column / row constants (c, l, u, anchors, b) stay in registers; only
      // the gathered vectors (w, y) go through shared memory.  Same operations
      // in the same order as the loop below: bit-identical.
      const int j0 = tid < n ? tid : -1, j1 = tid + kBT < n ? tid + kBT : -1;
      const int qr = tid < m ? tid : -1;
      double xr0 = 0.0, xr1 = 0.0, cr0 = 0.0, cr1 = 0.0, lr0 = 0.0, lr1 = 0.0, ur0 = 0.0,
             ur1 = 0.0, ar0 = 0.0, ar1 = 0.0, yr = 0.0, br = 0.0, ayr = 0.0;
      bool ineq = false;
      if (j0 >= 0) { xr0 = x[j0]; cr0 = cs[j0]; lr0 = ls[j0]; ur0 = us[j0]; ar0 = ax[j0]; }
      if (j1 >= 0) { xr1 = x[j1]; cr1 = cs[j1]; lr1 = ls[j1]; ur1 = us[j1]; ar1 = ax[j1]; }
      if (qr >= 0) { yr = y[qr]; br = bs[qr]; ayr = ay[qr]; ineq = aperm[qr] >= m1; }
      for (long long st = 0; st < steps; ++st) {
        if (st % kWTab == 0) {
          for (int q = tid; q < kWTab; q += kBT) {
            const double tq = (double)(t_seg + st + q);
            const double t2 = tq + 2.0;          // core.py:142-144
            wtab[2 * q] = (tq + 1.0) / t2;
            wtab[2 * q + 1] = 1.0 / t2;
          }
          __syncthreads();
        }
        const double wn = wtab[2 * (st % kWTab)], wa = wtab[2 * (st % kWTab) + 1];
        int bad = 0;
        if (j0 >= 0) {                           // x phase (core.py:168-169)
          double aty0, aty1;
          srow2(atst, atlen, atci, atv, y, j0, j1, aty0, aty1);
          {
            const double v = __dadd_rn(xr0, __dmul_rn(sigma, __dsub_rn(aty0, cr0)));
            const double xbj = np_clip(v, lr0, ur0);
            const double wj = __dsub_rn(__dmul_rn(2.0, xbj), xr0);
            const double xn = C.variant == 0 ? xbj
                              : __dadd_rn(__dmul_rn(wa, ar0), __dmul_rn(wn, C.variant == 2 ? wj : xbj));
            w[j0] = wj;
            xr0 = xn;
            bad |= !isfinite(xn);
          }
          if (j1 >= 0) {
            const double v = __dadd_rn(xr1, __dmul_rn(sigma, __dsub_rn(aty1, cr1)));
            const double xbj = np_clip(v, lr1, ur1);
            const double wj = __dsub_rn(__dmul_rn(2.0, xbj), xr1);
            const double xn = C.variant == 0 ? xbj
                              : __dadd_rn(__dmul_rn(wa, ar1), __dmul_rn(wn, C.variant == 2 ? wj : xbj));
            w[j1] = wj;
            xr1 = xn;
            bad |= !isfinite(xn);
          }
        }
        __syncthreads();
        if (qr >= 0) {                           // y phase (core.py:170-172)
          const double s2 = srow(ast, alen, aci, av, w, qr);
          double ybi = __dadd_rn(yr, __ddiv_rn(__dsub_rn(br, s2), lamsig));
          if (ineq) ybi = np_max(ybi, 0.0);
          double yn = ybi;
          if (C.variant != 0) {
            const double tg = C.variant == 2 ? __dsub_rn(__dmul_rn(2.0, ybi), yr) : ybi;
            yn = __dadd_rn(__dmul_rn(wa, ayr), __dmul_rn(wn, tg));
          }
          y[qr] = yn;
          yr = yn;
          bad |= !isfinite(yn);
        }
        if (__syncthreads_or(bad)) {
          broke = true;
          break;
        }
        ++t;
        ++k;
      }
      if (j0 >= 0) x[j0] = xr0;
      if (j1 >= 0) x[j1] = xr1;
      __syncthreads();
    } else
    for (long long st = 0; st < steps; ++st) {
      if (st % kWTab == 0) {                     // Halpern weights of the next kWTab steps
        for (int q = tid; q < kWTab; q += kBT) {
          const double tq = (double)(t_seg + st + q);
          const double t2 = tq + 2.0;            // core.py:142-144
          wtab[2 * q] = (tq + 1.0) / t2;
          wtab[2 * q + 1] = 1.0 / t2;
        }
        __syncthreads();
      }
      const double wn = wtab[2 * (st % kWTab)], wa = wtab[2 * (st % kWTab) + 1];
      int bad = 0;
      for (int q = tid; q < n; q += 2 * kBT) {   // x phase (core.py:168-169), 2 columns
        const int q2 = q + kBT < n ? q + kBT : -1;
        double aty0, aty1;
        srow2(atst, atlen, atci, atv, y, q, q2, aty0, aty1);
        for (int h = 0; h < 2; ++h) {
        const int jj = h ? q2 : q;
        if (jj < 0) break;
        const double aty = h ? aty1 : aty0;
        const int j = jj;                        // position
        const double xj = x[j];
        const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, cs[j])));
        const double xbj = np_clip(v, ls[j], us[j]);
        const double wj = __dsub_rn(__dmul_rn(2.0, xbj), xj);
        const double xn = C.variant == 0 ? xbj
                                         : __dadd_rn(__dmul_rn(wa, ax[j]), __dmul_rn(wn, C.variant == 2 ? wj : xbj));
        w[j] = wj;
        x[j] = xn;
        bad |= !isfinite(xn);
        }
      }
      __syncthreads();
      for (int q = tid; q < m; q += kBT) {       // y phase (core.py:170-172)
        const double s = srow(ast, alen, aci, av, w, q);
        const double yi = y[q];
        double ybi = __dadd_rn(yi, __ddiv_rn(__dsub_rn(bs[q], s), lamsig));
        if (aperm[q] >= m1) ybi = np_max(ybi, 0.0);
        double yn = ybi;
        if (C.variant != 0) {
          const double tg = C.variant == 2 ? __dsub_rn(__dmul_rn(2.0, ybi), yi) : ybi;
          yn = __dadd_rn(__dmul_rn(wa, ay[q]), __dmul_rn(wn, tg));
        }
        y[q] = yn;
        bad |= !isfinite(yn);
      }
      if (__syncthreads_or(bad)) {              // NumericalBreakdownError(k)
        broke = true;
        break;
      }
      ++t;
      ++k;
    }
#if HPR_BATCH_PROF
    const long long tq1 = clock64();
    tp_it += tq1 - tq0;
#endif
    if (broke) {
      status = 3;
      break;
    }
    // ---- checkpoint: half step (core.py:118-129) + candidate (driver.py:333-336) ----
    double s17[17];
#pragma unroll
    for (int q = 0; q < 17; ++q) s17[q] = 0.0;
    for (int q = tid; q < n; q += kBT) {
      const int j = atperm[q];                   // column (global arrays), q: position
      const double aty = srow(atst, atlen, atci, atv, y, q);
      const double xj = x[q];
      const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, cs[q])));
      const double xbj = np_clip(v, ls[q], us[q]);
      const double zbj = __ddiv_rn(__dsub_rn(xbj, v), sigma);
      xb[q] = xbj;
      w[q] = __dsub_rn(__dmul_rn(2.0, xbj), xj);
      s17[0] = __dadd_rn(s17[0], sq(__dsub_rn(xbj, ax[q])));     // bar_dx2
      s17[1] = __dadd_rn(s17[1], sq(__dsub_rn(xj, xbj)));        // dx2
      if (term_orig) {
        const double cj = csc[q];
        ox[j] = np_clip(__dmul_rn(xbj, __ddiv_rn(bf, cj)), l0[j], u0[j]);
        oz[j] = __dmul_rn(zbj, __dmul_rn(cf, cj));
      } else {
        ox[j] = xbj;
        oz[j] = zbj;
      }
    }
    __syncthreads();
    for (int q = tid; q < m; q += kBT) {
      const int i = aperm[q];                    // row (global arrays), q: position
      const double s = srow(ast, alen, aci, av, w, q);
      const double yi = y[q];
      double ybi = __dadd_rn(yi, __ddiv_rn(__dsub_rn(bs[q], s), lamsig));
      if (i >= m1) ybi = np_max(ybi, 0.0);
      const double dyi = __dsub_rn(yi, ybi);
      yb[q] = ybi;
      gdy[q] = dyi;                              // by position (gathered through atci)
      s17[2] = __dadd_rn(s17[2], sq(dyi));                       // dy2
      s17[3] = __dadd_rn(s17[3], sq(__dsub_rn(ybi, ay[q])));     // bar_dy2
      oy[i] = term_orig ? __dmul_rn(ybi, __ddiv_rn(cf, rs[q])) : ybi;
    }
    __syncthreads();
    // merit terms (core.py:191-197): A^T dy
    for (int q = tid; q < n; q += kBT) {
      double a = 0.0;
      for (int e = atst[q]; e < atst[q] + atlen[q]; ++e) a = __dadd_rn(a, __dmul_rn(atv[e], gdy[atci[e]]));
      const double dx = __dsub_rn(x[q], xb[q]);
      s17[4] = __dadd_rn(s17[4], sq(__dadd_rn(dx, __dmul_rn(sigma, a))));   // sh2
      s17[5] = __dadd_rn(s17[5], sq(a));                                    // aty2
    }
    double s11[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    kkt(s11);
#pragma unroll
    for (int q = 0; q < 11; ++q) s17[6 + q] = s11[q];
    bsum<17>(s17, red);
#pragma unroll
    for (int q = 0; q < 11; ++q) s11[q] = s17[6 + q];
    kkt_finish(s11);
    have_ckpt = 1;
    if (kk[5] <= C.tol && kk[1] <= C.tol && kk[3] <= C.tol) {
      status = 0;
    } else if (k >= C.max_iter) {
      status = 1;
    } else if (C.time_limit < INFINITY && (double)(gtimer() - t_start) * 1e-9 >= C.time_limit) {
      status = 2;
    } else if (C.uses_restarts) {
      double q = s17[4] / sigma;
      const double t1 = __dsub_rn(__dmul_rn(lamv, s17[2]), s17[5]);
      q = __dadd_rn(q, __dmul_rn(sigma, t1));
      const double scale = sigma * lamv * s17[2] + s17[1] / sigma;
      if (q < -1e-9 * fmax(scale, 1e-300)) merit_neg = 1;
      const double merit = 2.0 * sqrt(fmax(q, 0.0));
      if (!have_first) {
        have_first = true;
        merit_first = merit;
        merit_prev = INFINITY;
      }
      int kind = -1;                              // check_restart (driver.py:238-248)
      if (merit <= C.a1 * merit_first) kind = 0;
      else if (merit <= C.a2 * merit_first && merit > merit_prev) kind = 1;
      else if ((double)t >= C.a3 * (double)k) kind = 2;
      if (kind >= 0) {
        double sigma_next = sigma;
        if (C.updates_sigma) {                    // sigma_update (driver.py:251-278)
          const double dxn = sqrt(s17[0]);
          const double dyn = sqrt(lamv) * sqrt(s17[3]);
          bool ok = 1e-16 < dxn && dxn < 1e12 && 1e-16 < dyn && dyn < 1e12;
          if (ok) {
            const double ep = kk[1], ed = kk[3];
            if (ep == 0.0) {
              ok = ed == 0.0;
            } else {
              const double ratio = ed / ep;
              ok = 1e-8 < ratio && ratio < 1e8;
            }
          }
          sigma_next = ok ? dxn / dyn : 1.0;
        }
        if (tid == 0 && nlog < C.max_log) {
          hpr_restart_rec &rec = O.log[(long long)lp * C.max_log + nlog];
          rec.outer_index = r;
          rec.trigger = kind;
          rec.tau = t;
          rec.sigma_next = sigma_next;
          rec.merit = merit;
        }
        ++nlog;
        for (int i = tid; i < m; i += kBT) y[i] = ay[i] = yb[i];   // driver.py:363-364
        for (int j = tid; j < n; j += kBT) x[j] = ax[j] = xb[j];
        __syncthreads();
        sigma = sigma_next;
        ++r;
        t = 0;
        have_first = false;
        merit_prev = INFINITY;
      } else {
        merit_prev = merit;
      }
    }
  }

  // ---- finish (driver.py:374-391) ----
  if (!have_ckpt) {     // breakdown before the first checkpoint: the origin
    for (int q = tid; q < m; q += kBT) {
      oy[aperm[q]] = 0.0;
      yb[q] = 0.0;                               // the scaled candidate kkt() reads
    }
    for (int q = tid; q < n; q += kBT) {
      const int j = atperm[q];
      oz[j] = 0.0;
      ox[j] = np_clip(0.0, term_orig ? l0[j] : ls[q], term_orig ? u0[j] : us[q]);
      xb[q] = ox[j];
    }
    __syncthreads();
    double s11[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    kkt(s11);
    bsum<11>(s11, red);
    kkt_finish(s11);
  }
  if (!term_orig) {     // unscale + clip (driver.py:382-386)
    for (int q = tid; q < m; q += kBT) {
      const int i = aperm[q];
      oy[i] = __dmul_rn(oy[i], __ddiv_rn(cf, rs[q]));
    }
    for (int q = tid; q < n; q += kBT) {
      const int j = atperm[q];
      const double cj = csc[q];
      ox[j] = np_clip(__dmul_rn(ox[j], __ddiv_rn(bf, cj)), l0[j], u0[j]);
      oz[j] = __dmul_rn(oz[j], __dmul_rn(cf, cj));
    }
    __syncthreads();
  }
  // objectives of the solution on the original problem (driver.py:388-391)
  double f[6] = {0, 0, 0, 0, 0, 0};     // cx by lz uz nlo nup
  for (int i = tid; i < m; i += kBT) f[1] = __dadd_rn(f[1], __dmul_rn(b0[i], oy[i]));
  for (int j = tid; j < n; j += kBT) {
    const double zj = oz[j];
    f[0] = __dadd_rn(f[0], __dmul_rn(c0v[j], ox[j]));
    if (zj > 0.0 && isfinite(l0[j])) {
      f[2] = __dadd_rn(f[2], __dmul_rn(l0[j], zj));
      f[4] += 1.0;
    } else if (zj < 0.0 && isfinite(u0[j])) {
      f[3] = __dadd_rn(f[3], __dmul_rn(u0[j], zj));
      f[5] += 1.0;
    }
  }
  bsum<6>(f, red);
  if (tid == 0) {
    double pobj = f[0] + oc;
    double dobj = f[1];
    if (f[4] != 0.0) dobj += f[2];
    if (f[5] != 0.0) dobj += f[3];
    dobj += oc;
    if (P.obj_neg[lp]) {
      pobj = -pobj;
      dobj = -dobj;
    }
    hpr_batch_result &R = O.res[lp];
    R.status = status;
    R.restarts = r;
    R.iterations = k;
    R.power_iterations = piters;
    R.power_converged = pconv;
    R.dual_clamped = (int)clamped;
    R.n_log = nlog;
    R.merit_negative = merit_neg;
    R.power_failed = start == -2;
    R.primal_objective = pobj;
    R.dual_objective = dobj;
    for (int q = 0; q < 9; ++q) R.kkt[q] = kk[q];
    R.sigma_final = sigma;
    R.lambda_estimate = lamv;
    R.lambda_raw = lam_raw;
    R.b_factor = bf;
    R.c_factor = cf;
    R.device_seconds = (double)(gtimer() - t_start) * 1e-9;
#if HPR_BATCH_PROF
    if (lp < 3)
      printf("batch prof lp=%d setup+scale=%lld power=%lld iterations=%lld (%lld its) rest=%lld cycles\n", lp,
             tp_setup - tk0, tp_pow - tp_setup, tp_it, (long long)k, clock64() - tp_pow - tp_it);
#endif
  }
}

// ---- transpose of the whole batch (block-diagonal matrix) ----
__global__ void k_batch_keys(const int64_t *row_off, const int64_t *col_off, const int64_t *nz_off,
                             const int *rp, const int *ci, int *key, int *rowl, int count) {
  const int lp = blockIdx.x;
  if (lp >= count) return;
  const long long r0 = row_off[lp], c0 = col_off[lp], z0 = nz_off[lp];
  const int m = (int)(row_off[lp + 1] - r0);
  const int *lrp = rp + r0 + lp;
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    for (int e = lrp[i]; e < lrp[i + 1]; ++e) {
      key[z0 + e] = (int)(c0 + ci[z0 + e]);
      rowl[z0 + e] = i;
    }
}
__global__ void k_batch_gather(const int *perm, const int *rowl, const double *val, int *cit,
                               double *valt, long long nnz) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int p = perm[k];
    cit[k] = rowl[p];
    valt[k] = val[p];
  }
}
// grpt[c0 + lp + j] = global position of column j of LP lp (n + 1 entries per LP)
__global__ void k_batch_rpt(const int64_t *col_off, const int *gcount_rpt, int *grpt, int count) {
  const int lp = blockIdx.x;
  if (lp >= count) return;
  const long long c0 = col_off[lp];
  const int n = (int)(col_off[lp + 1] - c0);
  for (int j = threadIdx.x; j <= n; j += blockDim.x) grpt[c0 + lp + j] = gcount_rpt[c0 + j];
}

}  // namespace batch
}  // namespace hpr

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

struct BatchWs {
  size_t key, rowl, iota, perm, skey, gcrpt, grpt, cit, valt, dy, cub, cub_bytes, total;
};

int batch_layout(const hpr_batch_problem *p, BatchWs *L) {
  const long long nnz = p->total_nnz, nr = p->total_rows, nc = p->total_cols;
  size_t cb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, cb, (const int *)nullptr, (int *)nullptr,
                                     (const int *)nullptr, (int *)nullptr, (int)std::max(nnz, 1LL),
                                     0, 32));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 16), 256);
    return o;
  };
  L->key = take(4 * nnz);
  L->rowl = take(4 * nnz);
  L->iota = take(4 * nnz);
  L->perm = take(4 * nnz);
  L->skey = take(4 * nnz);
  L->gcrpt = take(4 * (nc + 1));
  L->grpt = take(4 * (nc + p->count));
  L->cit = take(4 * nnz);
  L->valt = take(8 * nnz);
  L->dy = take(8 * nr);
  L->cub_bytes = cb;
  L->cub = take(cb);
  L->total = off;
  return HPR_OK;
}

}  // namespace

extern "C" {

int hpr_batch_smem_bytes(int32_t max_m, int32_t max_n, int64_t max_nnz, size_t *bytes) {
  if (!bytes || max_m < 1 || max_n < 1 || max_nnz < 0) return fail(HPR_EINVAL, "bad argument");
  *bytes = hpr::batch::smem_bytes(max_m, max_n, max_nnz);
  return HPR_OK;
}

int hpr_batch_workspace_bytes(const hpr_batch_problem *p, size_t *bytes) {
  if (!p || !bytes) return fail(HPR_EINVAL, "null argument");
  if (p->count < 1 || p->total_nnz < 0 || p->total_nnz >= INT_MAX || p->total_cols >= INT_MAX)
    return fail(HPR_EINVAL, "invalid batch dims");
  BatchWs L;
  int rc = batch_layout(p, &L);
  if (rc) return rc;
  *bytes = L.total;
  return HPR_OK;
}

int hpr_batch_solve(const hpr_batch_problem *p, const hpr_batch_config *cfg, void *workspace,
                    size_t ws_bytes, hpr_batch_result *results, hpr_restart_rec *log,
                    double *x, double *y, double *z, int device, void *stream) {
  using namespace hpr::batch;
  if (!p || !cfg || !workspace || !results || !x || !y || !z) return fail(HPR_EINVAL, "null argument");
  if (cfg->max_log > 0 && !log) return fail(HPR_EINVAL, "null restart log");
  if (cfg->variant < 0 || cfg->variant > 3) return fail(HPR_EINVAL, "bad variant");
  if (cfg->check_interval < 1 || !(cfg->tolerance > 0.0)) return fail(HPR_EINVAL, "bad config");
  BatchWs L;
  int rc = batch_layout(p, &L);
  if (rc) return rc;
  if (ws_bytes < L.total) return fail(HPR_EINVAL, "batch workspace too small");
  if (p->max_m > 65535 || p->max_n > 65535)
    return fail(HPR_EINVAL, "an LP of the batch exceeds 65535 rows or columns");
  const size_t smem = smem_bytes(p->max_m, p->max_n, p->max_nnz);
  int dev_smem = 0;
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  if (smem > (size_t)dev_smem)
    return fail(HPR_EINVAL, "an LP of the batch does not fit in one CTA's shared memory (" +
                                std::to_string(smem) + " > " + std::to_string(dev_smem) + " bytes)");
  cudaStream_t s = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  int *key = (int *)(ws + L.key), *rowl = (int *)(ws + L.rowl), *iota = (int *)(ws + L.iota);
  int *perm = (int *)(ws + L.perm), *skey = (int *)(ws + L.skey);
  int *gcrpt = (int *)(ws + L.gcrpt), *grpt = (int *)(ws + L.grpt), *cit = (int *)(ws + L.cit);
  double *valt = (double *)(ws + L.valt), *dy = (double *)(ws + L.dy);
  const long long nnz = p->total_nnz;
  const int nc = (int)p->total_cols;
  const int count = (int)p->count;
  // stable transpose of the block-diagonal batch matrix: sort by global column,
  // rows stay ascending inside a column (csr_matrix(A.T) order, sparse.py:98-100)
  if (nnz > 0) {
    k_batch_keys<<<count, 128, 0, s>>>(p->row_off, p->col_off, p->nz_off, p->rp, p->ci, key, rowl,
                                       count);
    k_iota<<<grid_for(nnz), 256, 0, s>>>(iota, nnz);
    CKL();
    int end_bit = 1;
    while ((1LL << end_bit) < nc) ++end_bit;
    size_t tb = L.cub_bytes;
    CK(cub::DeviceRadixSort::SortPairs(ws + L.cub, tb, key, skey, iota, perm, (int)nnz, 0, end_bit, s));
    k_col_count<<<grid_for(nnz), 256, 0, s>>>(skey, nnz, nc, gcrpt);
    k_batch_gather<<<grid_for(nnz), 256, 0, s>>>(perm, rowl, p->val, cit, valt, nnz);
    CKL();
  } else {
    k_fill_empty_rpt<<<grid_for(nc + 1), 256, 0, s>>>(gcrpt, nc);
    CKL();
  }
  k_batch_rpt<<<count, 128, 0, s>>>(p->col_off, gcrpt, grpt, count);
  CKL();
  Prob P{p->row_off, p->col_off, p->nz_off, p->m1, p->rp, p->ci, p->val, grpt, cit, valt,
         p->b, p->c, p->lower, p->upper, p->obj_const, p->obj_neg};
  Cfg C{};
  C.tol = cfg->tolerance;
  C.time_limit = cfg->time_limit_seconds;
  C.a1 = cfg->alpha1;
  C.a2 = cfg->alpha2;
  C.a3 = cfg->alpha3;
  C.sigma0 = cfg->sigma0;
  C.power_tol = cfg->power_tol;
  C.max_iter = cfg->max_iterations;
  C.check_interval = cfg->check_interval;
  // variant codes of the batch config: 0 DR, 1 HDR-fixed, 2 HDR, 3 HPR
  C.variant = cfg->variant == 0 ? 0 : (cfg->variant == 3 ? 2 : 1);
  C.uses_restarts = cfg->variant != 0;
  C.updates_sigma = cfg->variant >= 2;
  C.ruiz = cfg->ruiz_iters;
  C.pc = cfg->pock_chambolle;
  C.bc = cfg->bc_normalize;
  C.power_max = cfg->power_max_iters;
  C.term_original = cfg->term_original;
  C.max_log = cfg->max_log;
  Out O{results, log, x, y, z, dy};
  CK(cudaFuncSetAttribute(k_batch_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_batch_solve<<<count, kBT, smem, s>>>(P, C, O);
  CKL();
  return HPR_OK;
}

}  // extern "C"
