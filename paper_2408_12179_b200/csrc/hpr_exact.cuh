// hpr_exact.cuh -- the exact T1 = 0 path on device.
//
// Reference: /root/reference/pkg/src/hprlp/exact.py.  For an equality-only LP
// with m <= 2000 the dual subproblem is solved exactly through the Cholesky
// factor L of AA* (exact.py:35-67) instead of the lambda-proximal step.  One
// iteration (exact.py:70-91 + core.py:139-160) is four kernels, captured
// check_interval times into one CUDA graph like the lambda path:
//
//   1. k_sell<EpiExactX>   over A^T rows: aty = A^T y; v = x + sigma (aty - c);
//                          xb = clip(v, l, u); zb = (xb - v) / sigma;
//                          u = xb + sigma (zb - c); x <- variant step (in place)
//   2. k_sell<EpiExactRhs> over A rows: rhs = (b - A u) / sigma
//   3. k_trmv<EpiTrStore>  h = L^{-1} rhs          (forward solve)
//   4. k_trmv<EpiTrY>      yb = L^{-T} h            (backward solve);
//                          y <- variant step (in place), non-finite probe
//
// The two triangular solves are products with the explicit inverse factor
// L^{-1} (and its transpose, both stored row-major so every row is one
// coalesced stream): the factor is fixed for the whole solve, so its O(m^3)
// inversion is paid once at setup (DenseCholesky.from_matrix) and each
// iteration's solve becomes two fully parallel triangular matrix-vector
// products (<= 2 x 16 MB at m = 2000, L2-resident) instead of two
// latency-bound substitutions of m dependent steps.  Each row's dot product is
// a fixed-order sum (lane-strided partial sums, fixed shuffle tree), so runs
// are bit-reproducible; against the reference's LAPACK substitution the
// solves agree to rounding (bitwise equality with LAPACK is not attainable
// either way: its blocking order differs).
#pragma once

namespace hpr {

// x side of the exact half step + the variant step of x (exact.py:73-78,
// core.py:139-153).  half = 1: the checkpoint's half step -- xb, zb go to
// xb_out / zb_out and the candidate slot, x is left alone.
struct EpiExactX {
  static constexpr int NQ = 0;
  static constexpr int kMinBlocks = HPR_SELL_MINB_RED;   // 72 registers spill here
  const double *c, *lo, *up, *anc;
  double *x, *u;
  double *xb_out, *zb_out, *cx_out, *cz_out;
  IterParams *P;
  int step, half;
  double sigma_half;
  double sigma, wa, wn, xj, cj, lj, uj, aj;
  int variant;
  __device__ bool enter() {
    if (half) {
      sigma = sigma_half;
      variant = 0;
    } else {
      sigma = P->sigma;
      variant = P->variant;
      halpern_weights(P->t0 + step, wa, wn);
    }
    return true;
  }
  __device__ void prefetch(int j) {
    xj = ld_epi(x + j);
    cj = ld_epi(c + j);
    lj = ld_epi(lo + j);
    uj = ld_epi(up + j);
    aj = variant ? ld_epi(anc + j) : 0.0;
  }
  __device__ void finish(int j, double aty, double *) {
    const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, cj)));
    const double xb = np_clip(v, lj, uj);
    const double zb = __ddiv_rn(__dsub_rn(xb, v), sigma);
    u[j] = __dadd_rn(xb, __dmul_rn(sigma, __dsub_rn(zb, cj)));
    if (half) {
      xb_out[j] = xb;
      zb_out[j] = zb;
      cx_out[j] = xb;
      cz_out[j] = zb;
      return;
    }
    double xn = xb;
    if (variant != 0) {
      const double tgt = variant == 2 ? __dsub_rn(__dmul_rn(2.0, xb), xj) : xb;
      xn = __dadd_rn(__dmul_rn(wa, aj), __dmul_rn(wn, tgt));
    }
    x[j] = xn;
    if (!isfinite(xn)) atomicMin(&P->nonfinite_k, (unsigned long long)(P->k0 + step));
  }
};

// rhs = (b - A u) / sigma (exact.py:79)
struct EpiExactRhs {
  static constexpr int NQ = 0;
  const double *b;
  double *rhs;
  IterParams *P;
  int half;
  double sigma_half;
  double sigma, bi;
  __device__ bool enter() {
    sigma = half ? sigma_half : P->sigma;
    return true;
  }
  __device__ void prefetch(int i) { bi = ld_epi(b + i); }
  __device__ void finish(int i, double s, double *) {
    rhs[i] = __ddiv_rn(__dsub_rn(bi, s), sigma);
  }
};

// forward solve output: h = L^{-1} rhs
struct EpiTrStore {
  double *out;
  __device__ void enter() {}
  __device__ void finish(int i, double s) { out[i] = s; }
};

// backward solve output yb = L^{-T} h + the variant step of y (core.py:139-153
// + the non-finite probe of core.py:155-157); half = 1: yb to yb_out and the
// candidate slot, y left alone.
struct EpiTrY {
  const double *anc;
  double *y, *yb_out, *cy_out;
  IterParams *P;
  int step, half;
  double wa, wn;
  int variant;
  __device__ void enter() {
    if (half) {
      variant = 0;
    } else {
      variant = P->variant;
      halpern_weights(P->t0 + step, wa, wn);
    }
  }
  __device__ void finish(int i, double yb) {
    if (half) {
      yb_out[i] = yb;
      cy_out[i] = yb;
      return;
    }
    double yn = yb;
    if (variant != 0) {
      const double yi = y[i];
      const double tgt = variant == 2 ? __dsub_rn(__dmul_rn(2.0, yb), yi) : yb;
      yn = __dadd_rn(__dmul_rn(wa, anc[i]), __dmul_rn(wn, tgt));
    }
    y[i] = yn;
    if (!isfinite(yn)) atomicMin(&P->nonfinite_k, (unsigned long long)(P->k0 + step));
  }
};

constexpr int kTrThreads = 256;
constexpr int kTrUnroll = 8;   // row elements in flight per lane

// Triangular matrix-vector product with a row-major m x m matrix T whose
// nonzeros in row i are columns [0, i] (lower) or [i, m) (upper): one warp per
// row.  Lane l sums elements j = j0 + l, j0 + l + 32, ... in ascending order
// (each product rounded, then added), then a fixed xor-free shuffle-down tree
// combines the 32 lane sums: the same order every launch.
template <class Epi>
__global__ void __launch_bounds__(kTrThreads)
k_trmv(const double *__restrict__ T, int m, int lower, const double *__restrict__ v, Epi epi) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (kTrThreads / 32) + (threadIdx.x >> 5);
  if (row >= m) return;
  epi.enter();
  const int j0 = lower ? 0 : row, j1 = lower ? row + 1 : m;
  const double *t = T + (size_t)row * m;
  double s = 0.0;
  int j = j0 + lane;
  for (; j + 32 * (kTrUnroll - 1) < j1; j += 32 * kTrUnroll) {
    double a[kTrUnroll], b[kTrUnroll];
#pragma unroll
    for (int u = 0; u < kTrUnroll; ++u) {
      a[u] = __ldg(t + j + 32 * u);
      b[u] = __ldg(v + j + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < kTrUnroll; ++u) s = __dadd_rn(s, __dmul_rn(a[u], b[u]));
  }
  for (; j < j1; j += 32) s = __dadd_rn(s, __dmul_rn(__ldg(t + j), __ldg(v + j)));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
  if (lane == 0) epi.finish(row, s);
}

}  // namespace hpr
