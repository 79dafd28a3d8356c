// hpr_small.cuh -- the resident inner loop for small LPs (launch-latency path).
//
// Reference: run_inner / iterate_once (core.py:163-179).  For an LP whose
// SELL layouts have at most kSmallMaxWin windows per matrix (C1: A^T 16, A 8
// windows of 128 rows), the 2 x check_interval kernels of an interval's graph
// are launch-latency bound (a few microseconds each, for a microsecond of
// work).  Here ONE launch of one thread-block cluster (<= 16 CTAs, one per
// SM) runs the whole interval: each CTA owns a fixed set of windows of A^T and
// of A (the same static assignment as k_sell), and the two phases of every
// iteration are separated by hardware cluster barriers
// (barrier.cluster.arrive.release / wait.acquire) instead of kernel
// boundaries.  The iterates y and w that other CTAs of the launch write are
// gathered with weak coherent loads (ld_coherent), ordered by the barrier's
// acquire; the matrix streams stay on the non-coherent path (read-only).
//
// The per-row arithmetic is the same sell_slice / long_row code and the same
// EpiXIter / EpiYIter epilogues as the graph path, so the iterates are
// bit-identical to it (tests/test_gpu_parity.py forces both).
#pragma once

namespace hpr {

constexpr int kSmallMaxCluster = 16;   // non-portable cluster size limit on B200
constexpr int kSmallMaxWin = 64;       // windows per matrix up to which the path is used

__device__ __forceinline__ void cluster_barrier() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool GA, class Epi>
__device__ __forceinline__ void small_phase(const SellMat &M, const double *xg, Epi &epi,
                                            uint64_t pol) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int nwin = (M.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  double acc[1] = {0.0};
  for (int win = blockIdx.x; win < nwin; win += G) {
    const SliceHdr h = load_hdr(M, win * kWarpsPerCta + wib, lane);
    sell_slice<GA ? HPR_GA_U : HPR_SELL_U, GA, Epi, true>(M, h, lane, xg, epi, acc, pol);
  }
  for (int li = blockIdx.x * kWarpsPerCta + wib; li < M.nlong; li += G * kWarpsPerCta)
    long_row<Epi, true>(M, M.long_rows[li], lane, xg, epi, acc, pol);
}

// Shared-memory residency of a CTA's slices (HPR_SMALL_SMEM): the CTA's
// windows of one matrix (win = blockIdx.x + q G), slice by slice, each slice's
// slots in their SELL order; per owned slice (q, warp) its shared-memory slot
// base and, for a non-compact slice, the lanes' rows / lengths.  Loaded once
// per interval launch, read every iteration (the matrix streams no longer go
// to L2).
struct SmallStage {
  int *base;            // [kSmallMaxOwn * kWarpsPerCta]
  int *row;             // [kSmallMaxOwn * kWarpsPerCta * 32]
  unsigned short *len;  // same
  int *ci;
  double *val;
};
constexpr int kSmallMaxOwn = kSmallMaxWin / 1;   // windows per CTA (G >= 1)

__device__ __forceinline__ int small_stage(const SellMat &M, SmallStage &S, unsigned char *p,
                                           int cap_slots) {
  const int G = gridDim.x, tid = threadIdx.x;
  const int nwin = (M.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  const int nown = blockIdx.x < nwin ? (nwin - blockIdx.x + G - 1) / G : 0;
  const int nsl = nown * kWarpsPerCta;
  S.base = (int *)p;
  S.row = S.base + ((nsl + 4) & ~3);
  S.len = (unsigned short *)(S.row + nsl * kSlice);
  unsigned char *q = (unsigned char *)(S.len + ((nsl * kSlice + 7) & ~7));
  S.val = (double *)(((uintptr_t)q + 15) & ~(uintptr_t)15);
  S.ci = (int *)(S.val + cap_slots);
  // slot bases (thread 0 scans the owned slices' sizes in order)
  if (tid == 0) {
    int o = 0;
    for (int k = 0; k < nsl; ++k) {
      const int s = (blockIdx.x + (k / kWarpsPerCta) * G) * kWarpsPerCta + k % kWarpsPerCta;
      S.base[k] = o;
      if (s < M.nslices) o += M.slice_ptr[s + 1] - M.slice_ptr[s];
    }
    S.base[nsl] = o;
  }
  __syncthreads();
  for (int k = 0; k < nsl; ++k) {
    const int s = (blockIdx.x + (k / kWarpsPerCta) * G) * kWarpsPerCta + k % kWarpsPerCta;
    if (s >= M.nslices) break;
    const int a = M.slice_ptr[s], n = M.slice_ptr[s + 1] - a, b = S.base[k];
    for (int t = tid; t < n; t += kThreads) {
      S.val[b + t] = M.val[a + t];
      S.ci[b + t] = M.ci[a + t];
    }
    if (tid < kSlice) {
      const SliceHdr h = load_hdr(M, s, tid);
      S.row[k * kSlice + tid] = h.row;
      S.len[k * kSlice + tid] = (unsigned short)h.len;
    }
  }
  __syncthreads();
  return nsl;
}

template <bool GA, class Epi>
__device__ __forceinline__ void small_phase_sm(const SellMat &M, const SmallStage &S,
                                               const double *xg, Epi &epi, uint64_t pol) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int nwin = (M.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  double acc[1] = {0.0};
  SellMat Ms = M;
  Ms.ci = S.ci;
  Ms.val = S.val;
  for (int win = blockIdx.x, q = 0; win < nwin; win += G, ++q) {
    const int k = q * kWarpsPerCta + wib, s = win * kWarpsPerCta + wib;
    SliceHdr h{-1, 0, 0, 0};
    if (s < M.nslices) {
      h.row = S.row[k * kSlice + lane];
      h.len = S.len[k * kSlice + lane];
      h.base = S.base[k];
      h.slen = (S.base[k + 1] - S.base[k]) / kSlice;
    }
    sell_slice<GA ? HPR_GA_U : HPR_SELL_U, GA, Epi, true, true>(Ms, h, lane, xg, epi, acc, pol);
  }
  for (int li = blockIdx.x * kWarpsPerCta + wib; li < M.nlong; li += G * kWarpsPerCta)
    long_row<Epi, true>(M, M.long_rows[li], lane, xg, epi, acc, pol);
}

// `steps` HPR iterations: x-phase over A^T (gathers y), barrier, y-phase over
// A (gathers w), barrier.  x_implicit: HPR keeps x implicit between the first
// and last step (EpiXIter).  cap_a / cap_at > 0: the CTA's slices of A / A^T
// are staged in shared memory (capacity in slots; A first, then A^T).
template <bool GAX, bool GAY>
__global__ void __launch_bounds__(kThreads)
k_small_inner(SellMat AT, SellMat A, const double *y, const double *w, EpiXIter ex, EpiYIter ey,
              int steps, int x_implicit, int cap_at, int cap_a) {
  extern __shared__ __align__(16) unsigned char small_sm[];
  const uint64_t pol = policy_evict_last();      // the whole LP stays in L2
  SmallStage SAT{}, SA{};
  const bool sm_at = cap_at > 0, sm_a = cap_a > 0;
  unsigned char *p = small_sm;
  if (sm_a) {
    small_stage(A, SA, p, cap_a);
    p = (unsigned char *)(((uintptr_t)(SA.ci + cap_a) + 15) & ~(uintptr_t)15);
  }
  if (sm_at) small_stage(AT, SAT, p, cap_at);
  for (int i = 0; i < steps; ++i) {
    ex.step = i;
    ex.x_from_w = x_implicit && i > 0;
    ex.x_store = !x_implicit || i == steps - 1;
    ex.enter();
    if (sm_at) small_phase_sm<GAX>(AT, SAT, y, ex, pol);
    else small_phase<GAX>(AT, y, ex, pol);
    cluster_barrier();
    ey.step = i;
    ey.enter();
    if (sm_a) small_phase_sm<GAY>(A, SA, w, ey, pol);
    else small_phase<GAY>(A, w, ey, pol);
    cluster_barrier();
  }
}

// The power method (sparse.py:184-198) for the same small LPs: one cluster
// launch runs every step -- u = A^T v, w = A u with the per-CTA partials of
// v.w and ||w||^2, the fixed-order step on CTA 0 (pow_step_block, as the graph
// path's last CTA), v = w / ||w|| -- with cluster barriers between the
// phases, until PowState.done.  The state and the vectors other CTAs write
// are read with coherent loads after the barriers' acquire.
__device__ __forceinline__ int pow_done(const PowState *S) {
  return *(volatile const int *)&S->done;
}

template <bool GAX, bool GAY>
__global__ void __launch_bounds__(kThreads)
k_small_power(SellMat AT, SellMat A, double *v, double *u, double *wv, double *part, PowState *S,
              int m) {
  const uint64_t pol = policy_evict_last();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = gridDim.x;
  EpiPowTu eu{};
  eu.u = u;
  eu.S = S;
  EpiPowA ea{};
  ea.v = v;
  ea.wv = wv;
  ea.S = S;
  while (!pow_done(S)) {
    small_phase<GAX>(AT, v, eu, pol);                 // u = A^T v
    cluster_barrier();
    double acc[2] = {0.0, 0.0};                       // w = A u, partials of v.w, ||w||^2
    {
      const int nwin = (A.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
      for (int win = blockIdx.x; win < nwin; win += G) {
        const SliceHdr h = load_hdr(A, win * kWarpsPerCta + wib, lane);
        sell_slice<GAY ? HPR_GA_U : HPR_SELL_U, GAY, EpiPowA, true>(A, h, lane, u, ea, acc, pol);
      }
      for (int li = blockIdx.x * kWarpsPerCta + wib; li < A.nlong; li += G * kWarpsPerCta)
        long_row<EpiPowA, true>(A, A.long_rows[li], lane, u, ea, acc, pol);
    }
    block_reduce_store<2>(acc, part, G);
    cluster_barrier();
    if (blockIdx.x == 0) pow_step_block(part, G, S);  // lambda, ||w||, convergence
    cluster_barrier();
    if (*(volatile const int *)&S->norm_pending) {    // v = w / ||w||
      const double nw = *(volatile const double *)&S->nw;
      for (int i = blockIdx.x * kThreads + threadIdx.x; i < m; i += G * kThreads)
        v[i] = __ddiv_rn(ld_coherent(wv + i), nw);
    }
    cluster_barrier();
  }
}

}  // namespace hpr
