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

#include <type_traits>
#include <utility>

namespace hpr {

constexpr int kThreads = 128;           // CTA size of the SELL / reduction kernels
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
// a matrix small enough to stay in L2 between iterations (SellMat::keep)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
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

// Operand-vector gathers of the SELL kernels.  HPR_GATHER_LD selects the
// load: 0 = ld.global.nc (L1-allocating), 1 = ld.global.nc without L1
// allocation, 2 = ld.global.cg (L2 only).
#ifndef HPR_GATHER_LD
#define HPR_GATHER_LD 0
#endif
__device__ __forceinline__ double ld_gather(const double *ptr) {
#if HPR_GATHER_LD == 1
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(ptr));
  return v;
#elif HPR_GATHER_LD == 2
  return __ldcg(ptr);
#else
  return __ldg(ptr);
#endif
}

// Gathers of a vector other CTAs of the same launch write (the resident
// small-LP loop, hpr_small.cuh): a weak coherent load -- ordered after the
// cluster barrier's acquire -- never the non-coherent path.
__device__ __forceinline__ double ld_coherent(const double *ptr) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(ptr) : "memory");
  return v;
}
template <bool COH>
__device__ __forceinline__ double gather(const double *ptr) {
  if constexpr (COH) return ld_coherent(ptr);
  else return ld_gather(ptr);
}

// Row operands of the iteration epilogues (read once per iteration): with
// HPR_EPI_NA they bypass L1 allocation so the gathered vector keeps the L1.
#ifndef HPR_EPI_NA
#define HPR_EPI_NA 0
#endif
// evict-first streaming access of a row operand (TS x-phase: whole 256-byte
// warp segments, nothing shared between warps) -- the gathered vector keeps L2
__device__ __forceinline__ double ld_ef(const double *ptr, uint64_t pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_ef(double *ptr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_epi(const double *ptr) {
#if HPR_EPI_NA
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(ptr));
  return v;
#else
  return *ptr;
#endif
}

// Device layout of one matrix for the iteration kernels: SELL-32-sigma.
// Rows are grouped in slices of 32 (lane i of a warp owns one row); inside a
// window of kWindow rows they are ordered by decreasing length so a slice's
// rows have similar lengths.  A slice stores its entries column-major
// (entry k of all 32 rows is contiguous), so the warp's loads of values and
// column indices are fully coalesced while each lane still adds its own row's
// products in the CSR (ascending-column) order -- the reference's order.
// Rows longer than kLongRow are kept out of the slices and summed by a whole
// warp from the CSR arrays (same order).
struct SellMat {
  const int *slice_ptr;    // nslices + 1 (slot offsets)
  const int *slice_row;    // nslices * 32: row of (slice, lane) or -1
  const unsigned short *slice_len;  // nslices * 32: that row's length (0 for padding)
  const int *ci;           // slots
  const double *val;       // slots
  const int *rp;           // CSR row pointers
  const int *csr_ci;       // CSR (for long rows)
  const double *csr_val;
  const int *long_rows;
  int nslices;
  int nlong;
  int ga;                  // long rows: gather one batch ahead (HPR_GA_MIN)
  int keep;                // L2 policy of the matrix streams: 0 evict_first, 1 evict_last, 2 normal
  // slices [0, compact) are compact: slice s holds rows 32 s .. 32 s + 31 (no
  // reordering) all of the slice's length, so their per-lane header
  // (slice_row / slice_len, 6 bytes a row) is never read -- the row follows
  // from s and the lane, the length from slice_ptr
  int compact;
  // TS engine only (hpr_tsell.cuh): the slot column indices re-encoded per
  // slice -- one word per entry where the 32 lanes' columns are lane-affine
  // (ci = base + lane) or lane-uniform (ci = base, bit 31 set), else the
  // slice's 32 words per entry unchanged; slice s's words start at aptr[s].
  // nullptr: the TS engine reads ci
  const int *aw = nullptr;
  const int *aptr = nullptr;
};

constexpr int kSlice = 32;
constexpr int kWindow = kThreads;       // one CTA's 4 slices (the SELL kernels' work unit)
// sigma: rows are sorted by length inside windows of sort_win(nrows) rows.
// HPR_SORT_WIN=1024 for large matrices cuts slice padding (C4's A^T 28 % -> 4 %)
// but measured slower (C2 57.1 vs 53.6 us, C4 1837 vs 1618 us per iteration):
// a slice's 32 rows then spread over 1024 rows, so the epilogue's vector loads
// and stores stop coalescing, and CTA windows get unequal work.  Default 128.
#ifndef HPR_SORT_WIN
#define HPR_SORT_WIN 128   // 1024 measured slower (C2 +6 %, C4 +13 %): uncoalesced epilogue rows
#endif
constexpr int kSortWinBig = HPR_SORT_WIN;
constexpr long long kSortBigRows = 131072;
__host__ __device__ inline int sort_win(long long nrows) {
  return nrows >= kSortBigRows ? kSortWinBig : kWindow;
}
constexpr int kLongRow = 1024;
constexpr int kWarpsPerCta = kThreads / 32;
#ifndef HPR_UNROLL
#define HPR_UNROLL 4
#endif

#ifndef HPR_LATE_PREFETCH
#define HPR_LATE_PREFETCH 0   // load the epilogue's row operands after the row's sum (fewer live registers)
#endif
constexpr int kUnroll = HPR_UNROLL;     // entries per lane in flight (x2: software pipelined)

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
  int iters, max_iters, converged, done, norm_pending;
  unsigned arrive;                  // CTAs of the fused A u + power-step launch (EpiPowA)
};

// ---------------------------------------------------------------------------
// TMA bulk copies + mbarrier (sm_90+ async proxy)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}

#ifndef HPR_GA_LEAN
#define HPR_GA_LEAN 1   // gather-ahead pipeline loads values one batch ahead: 8 fewer live registers (C2 -1.1 %)
#endif

// ---------------------------------------------------------------------------
// the SELL engine
// ---------------------------------------------------------------------------
// Epi (per-thread functor copy) provides
//   static constexpr int NQ;                      reduction quantities (may be 0)
//   bool enter();                                 uniform early-out (power method)
//   void prefetch(int r);                         load the row's operand vectors
//   void finish(int r, double s, double *acc);    fused elementwise + reduction terms
// per-lane slice header: the lane's row and length, the slice's slot range
struct SliceHdr {
  int row, len, base, slen;
};
__device__ __forceinline__ SliceHdr load_hdr(const SellMat &M, int s, int lane) {
  SliceHdr h{-1, 0, 0, 0};
  if (s < M.nslices) {
    h.base = M.slice_ptr[s];
    h.slen = (M.slice_ptr[s + 1] - h.base) / kSlice;
    if (s < M.compact) {
      h.row = s * kSlice + lane;
      h.len = h.slen;
    } else {
      h.row = M.slice_row[s * kSlice + lane];
      h.len = M.slice_len[s * kSlice + lane];
    }
  }
  return h;
}

// An epilogue with init(r) starts row r's running sum there instead of at 0.0
// (column-split layout: the sum carried over from the previous column block).
template <class E, class = void>
struct has_init : std::false_type {};
template <class E>
struct has_init<E, std::void_t<decltype(std::declval<E &>().init(0))>> : std::true_type {};

// An epilogue with final(part, nparts) runs it in the LAST CTA of the launch to
// finish (ticket counter), after every CTA's partials are stored: the
// fixed-order reduction and the scalar step fused into the product kernel.
template <class E, class = void>
struct has_final : std::false_type {};
template <class E>
struct has_final<E, std::void_t<decltype(std::declval<E &>().final(nullptr, 0))>>
    : std::true_type {};

// matrix-stream load: global (streaming, L2 hint) or, SM = true, a copy of the
// slices in shared memory (the resident small-LP loop)
template <bool SM, class T>
__device__ __forceinline__ T ld_mat(const T *ptr, uint64_t pol) {
  if constexpr (SM) return *ptr;
  else return ld_stream(ptr, pol);
}

template <int U, bool GA, class Epi, bool COH = false, bool SM = false>
__device__ __forceinline__ void sell_slice(const SellMat &M, const SliceHdr &h, int lane,
                                           const double *__restrict__ xg, Epi &epi, double *acc,
                                           uint64_t pol) {
  const int row = h.row, len = h.len, slen = h.slen;
#if !HPR_LATE_PREFETCH
  if (row >= 0) epi.prefetch(row);
#endif
  const int *cp = M.ci + h.base + lane;
  const double *vp = M.val + h.base + lane;
  double sum = 0.0;
  if constexpr (has_init<Epi>::value)
    if (row >= 0) sum = epi.init(row);
  // software pipeline: the streaming loads of batch i+1 are in flight while
  // batch i's operand gathers complete and its products are added in order
  int c[U];
  double v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < len) {
      c[u] = ld_mat<SM>(cp + u * kSlice, pol);
      v[u] = ld_mat<SM>(vp + u * kSlice, pol);
    }
  if constexpr (GA && HPR_GA_LEAN) {
  // lean depth-2 pipeline: batch k+1's gathers and batch k+2's column
  // indices are in flight while batch k's products are added; batch k+1's
  // values are loaded one batch (not two) ahead -- 8 fewer live registers
  double x0[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < len) x0[u] = gather<COH>(xg + c[u]);
  int c1[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (U + u < len) c1[u] = ld_mat<SM>(cp + (U + u) * kSlice, pol);
  for (int k = 0; k < slen; k += U) {
    double x1[U], v1[U];
    int c2[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + U + u < len) {
        x1[u] = gather<COH>(xg + c1[u]);
        v1[u] = ld_mat<SM>(vp + (k + U + u) * kSlice, pol);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + 2 * U + u < len) c2[u] = ld_mat<SM>(cp + (k + 2 * U + u) * kSlice, pol);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < len) sum = __dadd_rn(sum, __dmul_rn(v[u], x0[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = v1[u];
      x0[u] = x1[u];
      c1[u] = c2[u];
    }
  }
  } else if constexpr (GA) {
  // depth-2 pipeline: batch k+1's operand gathers and batch k+2's matrix loads
  // are in flight while batch k's products are added (long rows: the gather
  // latency is exposed once per two batches instead of once per batch)
  double x0[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < len) x0[u] = gather<COH>(xg + c[u]);
  int c1[U];
  double v1[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (U + u < len) {
      c1[u] = ld_mat<SM>(cp + (U + u) * kSlice, pol);
      v1[u] = ld_mat<SM>(vp + (U + u) * kSlice, pol);
    }
  for (int k = 0; k < slen; k += U) {
    double x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + U + u < len) x1[u] = gather<COH>(xg + c1[u]);
    int c2[U];
    double v2[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + 2 * U + u < len) {
        c2[u] = ld_mat<SM>(cp + (k + 2 * U + u) * kSlice, pol);
        v2[u] = ld_mat<SM>(vp + (k + 2 * U + u) * kSlice, pol);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < len) sum = __dadd_rn(sum, __dmul_rn(v[u], x0[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = v1[u];
      x0[u] = x1[u];
      c1[u] = c2[u];
      v1[u] = v2[u];
    }
  }
  } else {
  for (int k = 0; k < slen; k += U) {
    int cn[U];
    double vn[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + U + u < len) {
        cn[u] = ld_mat<SM>(cp + (k + U + u) * kSlice, pol);
        vn[u] = ld_mat<SM>(vp + (k + U + u) * kSlice, pol);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < len) xv[u] = gather<COH>(xg + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < len) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = cn[u];
      v[u] = vn[u];
    }
  }
  }
#if HPR_LATE_PREFETCH
  if (row >= 0) epi.prefetch(row);
#endif
  if (row >= 0) epi.finish(row, sum, acc);
}

// a long row: the warp forms 32 products at a time, lane 0 adds them in order
template <class Epi, bool COH = false>
__device__ __forceinline__ void long_row(const SellMat &M, int row, int lane,
                                         const double *__restrict__ xg, Epi &epi, double *acc,
                                         uint64_t pol) {
  if (lane == 0) epi.prefetch(row);
  const int z0 = M.rp[row], z1 = M.rp[row + 1];
  double sum = 0.0;
  for (int c0 = z0; c0 < z1; c0 += 32) {
    const int kk = c0 + lane;
    double p = 0.0;
    if (kk < z1)
      p = __dmul_rn(ld_stream(M.csr_val + kk, pol), gather<COH>(xg + ld_stream(M.csr_ci + kk, pol)));
    const int cnt = min(32, z1 - c0);
    for (int i = 0; i < cnt; ++i) {
      const double q = __shfl_sync(0xffffffffu, p, i);
      if (lane == 0) sum = __dadd_rn(sum, q);
    }
  }
  if (lane == 0) epi.finish(row, sum, acc);
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

// One CTA = 8 warps; CTA c handles sorting windows c, c + G, ... (warp w takes
// slice 8*window + w), then the long rows are strided over all warps.  Static
// assignment keeps the per-CTA partial sums deterministic.
#ifndef HPR_SELL_MINB
#define HPR_SELL_MINB 7      // min resident CTAs per SM of the reduction-free instances (register cap 72; 6 / cap 80: C3 1033 -> 946 us/iteration, 7: 832 -> 824, profiles/r02_sell_minb.txt)
#endif
#ifndef HPR_SELL_MINB_RED
#define HPR_SELL_MINB_RED 6  // instances with per-CTA partial sums (checkpoint epilogues: more live values; spill at 72)
#endif
// resident-CTA floor of a reduction-free / reduction epilogue; an epilogue
// with more live values can ask for the lower floor (static kMinBlocks)
template <class E, class = void>
struct sell_min_blocks
    : std::integral_constant<int, (E::NQ > 0 ? HPR_SELL_MINB_RED : HPR_SELL_MINB)> {};
template <class E>
struct sell_min_blocks<E, std::void_t<decltype(E::kMinBlocks)>>
    : std::integral_constant<int, E::kMinBlocks> {};
#ifndef HPR_SELL_MINB_GA
#define HPR_SELL_MINB_GA 6   // the gather-ahead (long-row) instances (C2's y-phase: 7 is 1 % slower)
#endif
template <class E, class = void>
struct sell_min_blocks_ga : std::integral_constant<int, HPR_SELL_MINB_GA> {};
template <class E>
struct sell_min_blocks_ga<E, std::void_t<decltype(E::kMinBlocksGA)>>
    : std::integral_constant<int, E::kMinBlocksGA> {};
template <int U, bool GA, class Epi>
__global__ void __launch_bounds__(kThreads, GA ? sell_min_blocks_ga<Epi>::value
                                                : sell_min_blocks<Epi>::value)
k_sell(SellMat M, const double *__restrict__ xg, Epi epi, double *part) {
  double acc[Epi::NQ > 0 ? Epi::NQ : 1];
#pragma unroll
  for (int q = 0; q < (Epi::NQ > 0 ? Epi::NQ : 1); ++q) acc[q] = 0.0;
  if (!epi.enter()) return;
  const uint64_t pol = M.keep == 1 ? policy_evict_last()
                       : M.keep == 2 ? policy_evict_normal() : policy_evict_first();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwin = (M.nslices + kWarpsPerCta - 1) / kWarpsPerCta;
  const int G = gridDim.x;
  // the next window's slice header is loaded while this one is processed, so
  // a slice costs two dependent memory round trips (matrix, gather), not three
  // programmatic dependent launch (inner-loop graph): let the next phase's CTAs
  // be scheduled as this grid drains; only the static slice header is read
  // before the previous phase's results (gathered vector, iterates) are waited for
  asm volatile("griddepcontrol.launch_dependents;");
  {
    SliceHdr h = load_hdr(M, blockIdx.x * kWarpsPerCta + wib, lane);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int win = blockIdx.x; win < nwin; win += G) {
      const SliceHdr hn = load_hdr(M, (win + G) * kWarpsPerCta + wib, lane);
      sell_slice<U, GA>(M, h, lane, xg, epi, acc, pol);
      h = hn;
    }
  }
  for (int li = blockIdx.x * kWarpsPerCta + wib; li < M.nlong; li += gridDim.x * kWarpsPerCta)
    long_row(M, M.long_rows[li], lane, xg, epi, acc, pol);
  if constexpr (Epi::NQ > 0) block_reduce_store<Epi::NQ>(acc, part, gridDim.x);
  if constexpr (has_final<Epi>::value) {
    __shared__ unsigned ticket;
    __threadfence();                     // this CTA's partials before its ticket
    __syncthreads();
    if (threadIdx.x == 0) ticket = atomicAdd(epi.arrive_counter(), 1u);
    __syncthreads();
    if (ticket == gridDim.x - 1) {
      __threadfence();                   // every CTA's partials visible
      epi.final(part, gridDim.x);
    }
  }
}

// ---------------------------------------------------------------------------
// inner iteration epilogues
// ---------------------------------------------------------------------------
// x phase over A^T rows (core.py:168-169 + 149-153): x updated in place,
// w = 2 xb - x for the y phase.
//
// HPR (variant 2) keeps x implicit inside an interval: x_{k+1} = wa_k anc +
// wn_k w_k exactly (core.py:149-150), so a step with x_from_w set re-forms
// x_k from the previous step's w (same operands, same rounding: the same
// bits) instead of reading x, and a step without x_store skips the x write
// -- one n-vector of HBM traffic less per iteration.  The inner-loop graph
// sets x_from_w on steps 1.. and x_store on the last step only, so x is
// materialised at every interval end (checkpoint, restart, the host); other
// variants always read and write x.
struct EpiXIter {
  static constexpr int NQ = 0;
  const double *c, *lo, *up, *anc;
  double *x, *w;
  IterParams *P;
  int step;
  int bounds_uniform;        // bit 0: every lower bound equals lo_u, bit 1: upper / up_u
  int x_from_w = 0, x_store = 1;
  int ef = 0;                // bit 0: row operands, bit 1: results streamed evict-first (TS engine)
  double lo_u, up_u;
  double sigma, wa, wn, wa0, wn0, xj, cj, lj, uj, aj;
  int variant, implicit;
  uint64_t pol;
  __device__ bool enter() {
    if (ef) pol = policy_evict_first();
    sigma = P->sigma;
    variant = P->variant;
    halpern_weights(P->t0 + step, wa, wn);
    implicit = variant == 2 && x_from_w;
    if (implicit) halpern_weights(P->t0 + step - 1, wa0, wn0);
    return true;
  }
  __device__ double ld(const double *p) const { return ef ? ld_ef(p, pol) : ld_epi(p); }
  __device__ void prefetch(int j) {
    xj = ld(implicit ? w + j : x + j);
    cj = ld(c + j);
    lj = (bounds_uniform & 1) ? lo_u : ld(lo + j);
    uj = (bounds_uniform & 2) ? up_u : ld(up + j);
    aj = variant ? ld(anc + j) : 0.0;
  }
  __device__ void finish(int j, double aty, double *) {
    if (implicit) xj = __dadd_rn(__dmul_rn(wa0, aj), __dmul_rn(wn0, xj));   // x_k from w_{k-1}
    const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, cj)));
    const double xb = np_clip(v, lj, uj);
    const double wj = __dsub_rn(__dmul_rn(2.0, xb), xj);
    const double xn =
        variant == 0 ? xb : __dadd_rn(__dmul_rn(wa, aj), __dmul_rn(wn, variant == 2 ? wj : xb));
    if (ef & 2) {
      st_ef(w + j, wj, pol);
      if (x_store || variant != 2) st_ef(x + j, xn, pol);
    } else {
      w[j] = wj;
      if (x_store || variant != 2) x[j] = xn;
    }
    if (!isfinite(xn)) atomicMin(&P->nonfinite_k, (unsigned long long)(P->k0 + step));
  }
};

// y phase over A rows (core.py:170-172 + 149-153): y updated in place.
struct EpiYIter {
  static constexpr int NQ = 0;
  const double *b, *anc;
  double *y;
  IterParams *P;
  int step, m1;
  int ef = 0;                // row operands / results streamed evict-first
  double lamsig, wa, wn, yi, bi, ai;
  int variant;
  uint64_t pol;
  __device__ bool enter() {
    if (ef) pol = policy_evict_first();
    lamsig = P->lamsig;
    variant = P->variant;
    halpern_weights(P->t0 + step, wa, wn);
    return true;
  }
  __device__ double ld(const double *p) const { return ef ? ld_ef(p, pol) : ld_epi(p); }
  __device__ void prefetch(int i) {
    yi = ld(y + i);
    bi = ld(b + i);
    ai = variant ? ld(anc + i) : 0.0;
  }
  __device__ void finish(int i, double s, double *) {
    double yb = __dadd_rn(yi, __ddiv_rn(__dsub_rn(bi, s), lamsig));
    if (i >= m1) yb = np_max(yb, 0.0);
    double yn = yb;
    if (variant != 0) {
      const double tgt = variant == 2 ? __dsub_rn(__dmul_rn(2.0, yb), yi) : yb;
      yn = __dadd_rn(__dmul_rn(wa, ai), __dmul_rn(wn, tgt));
    }
    if (ef) st_ef(y + i, yn, pol);
    else y[i] = yn;
    if (!isfinite(yn)) atomicMin(&P->nonfinite_k, (unsigned long long)(P->k0 + step));
  }
};

// Column-split layout (hpr_capi.cu: Split): A's columns are cut into NB blocks
// small enough for the gathered vector's block to stay in L2; block b's
// kernel continues every row's running sum from block b-1 (psum), so each row
// is still summed in ascending column order from 0.0 -- bit-identical to the
// unsplit product.  Blocks 0..NB-2 store the running sums, the last block
// hands them to the phase's real epilogue (EpiCarryIn).
struct EpiCarry {
  static constexpr int NQ = 0;
  static constexpr int kMinBlocksGA = 7;   // C4's column-split blocks: 72 registers, -1 %
  double *psum;
  int first;
  __device__ bool enter() { return true; }
  __device__ double init(int r) { return first ? 0.0 : psum[r]; }
  __device__ void prefetch(int) {}
  __device__ void finish(int r, double s, double *) { psum[r] = s; }
};
template <class Epi>
struct EpiCarryIn : Epi {
  static constexpr int kMinBlocksGA = 7;
  const double *psum;
  __device__ double init(int r) { return psum[r]; }
};

// ---------------------------------------------------------------------------
// checkpoint epilogues
// ---------------------------------------------------------------------------
struct CandCtx {
  int term_original;
  const double *fac;                 // device [b_factor, c_factor]
  const double *row_scale, *col_scale;
  const double *lo0, *up0;           // original bounds (clip target)
};

// half step x part (core.py:123-125) + candidate unscale/clip (scaling.py:46,48;
// driver.py:334-336); sums ||xb - anchor_x||^2, ||x - xb||^2.
struct EpiXHalf {
  static constexpr int NQ = 2;
  const double *x, *c, *lo, *up, *anc;
  double *xb_out, *zb_out, *wtmp, *cx_out, *cz_out;
  CandCtx cc;
  double sigma, bf, cf;
  double xj, cj, lj, uj, aj, csj, l0, u0;
  __device__ bool enter() {
    bf = cc.fac[0];
    cf = cc.fac[1];
    return true;
  }
  __device__ void prefetch(int j) {
    xj = x[j];
    cj = c[j];
    lj = lo[j];
    uj = up[j];
    aj = anc[j];
    if (cc.term_original) {
      csj = cc.col_scale[j];
      l0 = cc.lo0[j];
      u0 = cc.up0[j];
    }
  }
  __device__ void finish(int j, double aty, double *acc) {
    const double v = __dadd_rn(xj, __dmul_rn(sigma, __dsub_rn(aty, cj)));
    const double xb = np_clip(v, lj, uj);
    const double zb = __ddiv_rn(__dsub_rn(xb, v), sigma);
    xb_out[j] = xb;
    zb_out[j] = zb;
    wtmp[j] = __dsub_rn(__dmul_rn(2.0, xb), xj);
    acc[0] = __dadd_rn(acc[0], sq(__dsub_rn(xb, aj)));
    acc[1] = __dadd_rn(acc[1], sq(__dsub_rn(xj, xb)));
    if (cc.term_original) {
      cx_out[j] = np_clip(__dmul_rn(xb, __ddiv_rn(bf, csj)), l0, u0);
      cz_out[j] = __dmul_rn(zb, __dmul_rn(cf, csj));
    } else {
      cx_out[j] = xb;
      cz_out[j] = zb;
    }
  }
};

// half step y part (core.py:126-128) + candidate y; sums ||y - yb||^2, ||yb - anchor_y||^2.
struct EpiYHalf {
  static constexpr int NQ = 2;
  const double *y, *b, *anc;
  double *yb_out, *dy_out, *cy_out;
  CandCtx cc;
  double lamsig, cf;
  int m1;
  double yi, bi, ai, rsi;
  __device__ bool enter() {
    cf = cc.fac[1];
    return true;
  }
  __device__ void prefetch(int i) {
    yi = y[i];
    bi = b[i];
    ai = anc[i];
    if (cc.term_original) rsi = cc.row_scale[i];
  }
  __device__ void finish(int i, double s, double *acc) {
    double yb = __dadd_rn(yi, __ddiv_rn(__dsub_rn(bi, s), lamsig));
    if (i >= m1) yb = np_max(yb, 0.0);
    const double dy = __dsub_rn(yi, yb);
    yb_out[i] = yb;
    dy_out[i] = dy;
    acc[0] = __dadd_rn(acc[0], sq(dy));
    acc[1] = __dadd_rn(acc[1], sq(__dsub_rn(yb, ai)));
    cy_out[i] = cc.term_original ? __dmul_rn(yb, __ddiv_rn(cf, rsi)) : yb;
  }
};

// KKT row terms over the termination problem's A (driver.py:203-206, 211, 214).
struct EpiKktRow {
  static constexpr int NQ = 3;
  const double *b, *cy;
  int m1;
  double bi, yi;
  __device__ bool enter() { return true; }
  __device__ void prefetch(int i) {
    bi = b[i];
    yi = cy[i];
  }
  __device__ void finish(int i, double ax, double *acc) {
    double prim = __dsub_rn(bi, ax);
    double tproj = __dadd_rn(__dsub_rn(yi, ax), bi);
    if (i >= m1) {
      prim = np_max(prim, 0.0);
      tproj = np_max(tproj, 0.0);
    }
    acc[0] = __dadd_rn(acc[0], sq(prim));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(bi, yi));
    acc[2] = __dadd_rn(acc[2], sq(__dsub_rn(yi, tproj)));
  }
};

// KKT column terms over the termination problem's A^T (driver.py:207-215,
// problem.py:146-176).
struct EpiKktCol {
  static constexpr int NQ = 8;
  const double *c, *lo, *up, *cx, *cz;
  double cj, zj, xj, l, u;
  __device__ bool enter() { return true; }
  __device__ void prefetch(int j) {
    cj = c[j];
    zj = cz[j];
    xj = cx[j];
    l = lo[j];
    u = up[j];
  }
  __device__ void finish(int j, double aty, double *acc) {
    acc[0] = __dadd_rn(acc[0], sq(__dsub_rn(__dsub_rn(cj, aty), zj)));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(cj, xj));
    if (zj > 0.0) {
      if (isfinite(l)) {
        acc[2] = __dadd_rn(acc[2], __dmul_rn(l, zj));
        acc[4] += 1.0;
      } else {
        acc[6] += 1.0;
      }
    } else if (zj < 0.0) {
      if (isfinite(u)) {
        acc[3] = __dadd_rn(acc[3], __dmul_rn(u, zj));
        acc[5] += 1.0;
      } else {
        acc[6] += 1.0;
      }
    }
    acc[7] = __dadd_rn(acc[7], sq(__dsub_rn(xj, np_clip(__dsub_rn(xj, zj), l, u))));
  }
};

// merit terms over the scaled A^T (core.py:191-197): aty = A^T dy.
struct EpiMeritCol {
  static constexpr int NQ = 2;
  const double *x, *xb;
  double sigma, xj, xbj;
  __device__ bool enter() { return true; }
  __device__ void prefetch(int j) {
    xj = x[j];
    xbj = xb[j];
  }
  __device__ void finish(int j, double aty, double *acc) {
    const double dx = __dsub_rn(xj, xbj);
    acc[0] = __dadd_rn(acc[0], sq(__dadd_rn(dx, __dmul_rn(sigma, aty))));
    acc[1] = __dadd_rn(acc[1], sq(aty));
  }
};

// power method (sparse.py:189-191): u = A^T v (sum u^2 for the start check),
// w = A u with v.w and w.w.
struct EpiPowT {
  static constexpr int NQ = 1;
  double *u;
  const PowState *S;
  __device__ bool enter() { return !S->done; }
  __device__ void prefetch(int) {}
  __device__ void finish(int j, double s, double *acc) {
    u[j] = s;
    acc[0] = __dadd_rn(acc[0], sq(s));
  }
};
// u = A^T v without the norm (the in-loop power step only uses EpiPowA's sums;
// staged-engine eligible)
struct EpiPowTu {
  static constexpr int NQ = 0;
  double *u;
  const PowState *S;
  __device__ bool enter() { return !S->done; }
  __device__ void prefetch(int) {}
  __device__ void finish(int j, double s, double *) { u[j] = s; }
};
struct EpiPowA {
  static constexpr int NQ = 2;
  const double *v;
  double *wv;
  PowState *S;
  double vi;
  __device__ bool enter() { return !S->done; }
  __device__ void prefetch(int i) { vi = v[i]; }
  __device__ void finish(int i, double s, double *acc) {
    wv[i] = s;
    acc[0] = __dadd_rn(acc[0], __dmul_rn(vi, s));
    acc[1] = __dadd_rn(acc[1], sq(s));
  }
};

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

// one CTA: reduce the v.w and w.w partials in fixed order, then the scalar
// logic of one power step (sparse.py:188-198).
__device__ __forceinline__ void pow_step_block(const double *part, int nparts, PowState *S) {
  double a[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < nparts; i += kThreads) {
    a[0] = __dadd_rn(a[0], part[i]);
    a[1] = __dadd_rn(a[1], part[nparts + i]);
  }
  block_reduce<2>(a);
  if (threadIdx.x == 0) {
    const double lam = a[0];
    const double nw = sqrt(a[1]);
    S->iters += 1;
    S->lam = lam;
    S->nw = nw;
    S->arrive = 0;
    if (nw == 0.0) {
      S->done = 1;                       // break before v = w / nw
      S->norm_pending = 0;
      return;
    }
    S->norm_pending = 1;                 // v = w / nw (k_pow_norm; recomputing it is idempotent)
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

__global__ void __launch_bounds__(kThreads) k_pow_step(const double *part, int nparts, PowState *S) {
  if (S->done) return;
  pow_step_block(part, nparts, S);
}

// EpiPowA whose last CTA also runs the power step (k_pow_step fused in)
struct EpiPowAStep : EpiPowA {
  __device__ unsigned *arrive_counter() { return &S->arrive; }
  __device__ void final(const double *part, int nparts) { pow_step_block(part, nparts, S); }
};

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




// SELL plan: CTA per sorting window of WIN rows.  Rows are ranked by (length
// desc, index asc); long rows and padding go last with row = -1.  Writes
// slice_row and the slot count of each slice (32 * longest row in it); the
// arrays cover nrows rounded up to kWindow (a last partial window stops there).
// ``order`` (optional, non-split plans only): the rows in processing order --
// window w takes rows order[w*WIN ...] instead of rows w*WIN ... (the row
// affinity order below).  A row's own sum is unaffected: only which rows share
// a window / slice, and when they are processed, changes.
template <int WIN>
__global__ void __launch_bounds__(WIN) k_sell_plan(const int *rp, int nrows, int sort_rows,
                                                   int *slice_row, unsigned short *slice_len,
                                                   int *slice_slots, int *long_flag,
                                                   int long_thresh, int m_pad, int m_real,
                                                   const int *order, int *compact_prefix) {
  __shared__ int key[WIN];
  __shared__ int skey[WIN];
  __shared__ int srow[WIN];
  const int t = threadIdx.x;
  const int r_in = blockIdx.x * WIN + t;
  const int r = (order && r_in < nrows) ? order[r_in] : r_in;
  const int rows_pad = (nrows + kWindow - 1) / kWindow * kWindow;
  int k = -2;
  // column-split plans (m_pad > 0): virtual rows b * m_pad + i with i >= m_real are padding
  if (r_in < nrows && (m_pad == 0 || r % m_pad < m_real)) {
    const int len = rp[r + 1] - rp[r];
    k = len > long_thresh ? -1 : len;
    long_flag[r] = len > long_thresh;
  } else if (r_in < nrows) {
    long_flag[r] = 0;
  }
  key[t] = k;
  __syncthreads();
  int rank = t;
  if (sort_rows) {
    rank = 0;
    for (int j = 0; j < WIN; ++j) {
      const int kj = key[j];
      rank += (kj > k) || (kj == k && j < t);
    }
  }
  skey[rank] = k;
  srow[rank] = k >= 0 && m_pad == 0 ? r : -1;
  const int p = blockIdx.x * WIN + rank;
  if (p < rows_pad) {
    // column-split plans store the real row i of virtual row b * m_pad + i
    slice_row[p] = k >= 0 ? (m_pad ? r % m_pad : r) : -1;
    slice_len[p] = (unsigned short)(k >= 0 ? k : 0);
  }
  __syncthreads();
  if (t < WIN / kSlice && blockIdx.x * WIN + t * kSlice < rows_pad) {
    int mx = 0;
    for (int i = 0; i < kSlice; ++i) mx = max(mx, skey[t * kSlice + i]);
    slice_slots[blockIdx.x * (WIN / kSlice) + t] = mx * kSlice;
    // compact slice: rows 32 s .. 32 s + 31 in place, all of equal length
    const int sl = blockIdx.x * (WIN / kSlice) + t;
    bool compact = true;
    for (int i = 0; i < kSlice && compact; ++i)
      compact = srow[t * kSlice + i] == sl * kSlice + i && skey[t * kSlice + i] == mx;
    if (!compact) atomicMin(compact_prefix, sl);
  }
}

// Row affinity key (the SELL plan's processing order when the gathered
// vector exceeds L2): the column block (2^bits columns) holding most of the
// row's entries -- the longest run of equal ci >> bits, the row's columns being
// ascending; ties go to the lowest block; empty rows key 0.  Rows sorted
// stably by it are processed together with the other rows that gather the same
// vector block, so a block fetched from HBM by one row is an L2 hit for the
// next (C3: a capacity row re-reads exactly the flow segment its tail node's
// conservation rows just read).
__global__ void k_row_mode_block(const int *rp, const int *ci, int nrows, int bits, int *key) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int z0 = rp[r], z1 = rp[r + 1];
    int best = 0, best_len = 0, cur = -1, cur_len = 0;
    for (int z = z0; z < z1; ++z) {
      const int b = ci[z] >> bits;
      cur_len = b == cur ? cur_len + 1 : 1;
      cur = b;
      if (cur_len > best_len) {
        best_len = cur_len;
        best = cur;
      }
    }
    key[r] = best;
  }
}

// fill slot column indices and the CSR -> slot map (warp per slice)
__global__ void k_sell_fill(const int *rp, const int *ci, const int *slice_ptr,
                            const int *slice_row, int nslices, int *sell_ci, int *sell_pos) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += nw) {
    const int row = slice_row[s * kSlice + lane];
    if (row < 0) continue;
    const int z0 = rp[row], len = rp[row + 1] - z0, base = slice_ptr[s];
    for (int k = 0; k < len; ++k) {
      const int pos = base + k * kSlice + lane;
      sell_ci[pos] = ci[z0 + k];
      sell_pos[z0 + k] = pos;
    }
  }
}

// Column-split layout: entry counts of the virtual rows (b, i) = b * m_pad + i
// (row i's entries with column in [b W, (b+1) W)); thread per row, columns ascend.
__global__ void k_split_count(const int *rp, const int *ci, int nrows, int m_pad, int W, int NB,
                              int *cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m_pad; i += gridDim.x * blockDim.x) {
    int k = i < nrows ? rp[i] : 0;
    const int z1 = i < nrows ? rp[i + 1] : 0;
    for (int b = 0; b < NB; ++b) {
      const long long hi = (long long)(b + 1) * W;
      int c0 = 0;
      while (k < z1 && ci[k] < hi) {
        ++k;
        ++c0;
      }
      cnt[(long long)b * m_pad + i] = c0;
    }
  }
}

// Column-split layout: slot column indices and the CSR -> slot map (warp per
// slice; a virtual row's entries are a contiguous run of its CSR row)
__global__ void k_split_fill(const int *rp, const int *ci, const int *vrp, const int *slice_ptr,
                             const int *slice_row, int nslices, int m_pad, int W, int *sell_ci,
                             int *sell_pos) {
  const int slices_per_block = m_pad / kSlice;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += nw) {
    const int i = slice_row[s * kSlice + lane];
    if (i < 0) continue;
    const int b = s / slices_per_block, v = b * m_pad + i;
    const int len = vrp[v + 1] - vrp[v], base = slice_ptr[s];
    if (len == 0) continue;
    const long long lo = (long long)b * W;
    int a = rp[i], e = rp[i + 1];
    while (a < e) {                        // first entry with column >= b W
      const int mid = (a + e) >> 1;
      if (ci[mid] < lo) a = mid + 1; else e = mid;
    }
    for (int k = 0; k < len; ++k) {
      const int pos = base + k * kSlice + lane;
      sell_ci[pos] = ci[a + k];
      sell_pos[a + k] = pos;
    }
  }
}

// CSR values -> slots (entries of long rows have sell_pos = -1)
__global__ void k_sell_scatter(const int *sell_pos, const double *src, double *dst, long long nnz) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int p = sell_pos[k];
    if (p >= 0) dst[p] = src[k];
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
__global__ void k_fill_int(int *a, int n, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
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

// flag[0] &= (a[j] is bitwise a[0] for every j): uniform bound vectors (e.g.
// x >= 0) are then passed to the x-phase as a scalar instead of streamed
__global__ void k_uniform(const double *a, long long n, unsigned int *flag) {
  const unsigned long long a0 = __double_as_longlong(a[0]);
  bool same = true;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    same &= (unsigned long long)__double_as_longlong(a[i]) == a0;
  if (!__all_sync(0xffffffffu, same) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0u);
}

__global__ void k_reset_params(IterParams *P) {
  P->sigma = 0.0;
  P->lamsig = 0.0;
  P->t0 = 0;
  P->k0 = 0;
  P->variant = 0;
  P->pad_ = 0;
  P->nonfinite_k = ~0ULL;
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
