// hpr_stg.cuh -- staged SpMV engine ("STG") for the iteration phases.
//
// Why: a random 8-byte gather from an L2-resident vector costs the SM one
// outstanding L1 miss; measured, B200 sustains ~0.5-0.6 such gathers per cycle
// per SM whatever the kernel does (scripts/microbench/dsmem_gather.cu: 0.48
// loads/clk/SM from global, 0.2-0.6 from cluster DSMEM, 4.9 from the SM's own
// shared memory).  The SELL kernels sit at that ceiling on C2.  When the
// operand vector is reused enough (nnz >= 40 * its length), streaming it
// through every SM's shared memory in 64 KB chunks (bulk copies, ~100 GB/s per
// SM) and gathering from there is cheaper: C2's x-phase (A^T against y, 50
// uses per element) 53.3 -> 46.4 us per iteration; its y-phase (25 uses) is
// faster with SELL (+13 us with STG), so auto selects the x-phase only.
//
// Layout (hpr_capi.cu: Stg, built at hpr_analyze / hpr_bind_layout): one
// persistent CTA per SM owns a contiguous, nnz-balanced range of rows.  For
// each column chunk b (kStgW columns) the CTA's entries in that chunk form one
// RECORD, loaded with one bulk copy next to the vector chunk:
//     int nsl | int soff[nsl + 1] | u16 lrow[32 nsl] | u16 lci[slots] | f64 val[slots]
// The rows with entries in the chunk are sorted by their entry count there
// (descending, then row) and cut into slices of 32 (lane i of a warp owns one
// row); a slice stores its entries column-major (entry k of the 32 rows
// contiguous), padded to the slice's longest row with lci = 0xFFFF.  A lane
// adds its row's products left to right onto the row's running sum, which
// lives in shared memory across chunks.  Chunks ascend and entries ascend
// inside a chunk, so every row is still summed in ascending column order from
// 0.0 with separately rounded products -- bit-identical to scipy's csr_matvec
// and to the SELL engine.  After the last chunk the phase epilogue (EpiXIter /
// EpiYIter) runs on every row.  A producer warp keeps S stages in flight
// (full / empty mbarriers); the consumer warps meet at a named barrier per
// chunk, since consecutive chunks may give a row to different warps.
#pragma once

namespace hpr {

#ifndef HPR_STG_WARPS
#define HPR_STG_WARPS 24   // measured on C2's x-phase: 16 -> 47.5, 24 -> 46.4, 28 -> 48.5 us/iteration
#endif
#ifndef HPR_STG_COLBITS
#define HPR_STG_COLBITS 13 // 4096-column chunks (4 stages) measured slower: per-chunk cost dominates
#endif
#ifndef HPR_STG_SPW
#define HPR_STG_SPW 1   // 2 / 3 slices per warp at once measured slower (51.5 / 61.5 vs 46.9 us)
#endif
constexpr int kStgWarps = HPR_STG_WARPS;
constexpr int kStgSpw = HPR_STG_SPW;                // slices in flight per consumer warp            // consumer warps (+ 1 producer warp)
constexpr int kStgThreads = (kStgWarps + 1) * 32;
constexpr int kStgColBits = HPR_STG_COLBITS;
constexpr int kStgW = 1 << kStgColBits;             // doubles per staged vector chunk (64 KB)
constexpr int kStgMaxStages = 4;
constexpr unsigned short kStgPad = 0xFFFF;

struct StgMat {
  const int *row_start;        // G + 1
  const long long *goff;       // G * NB + 1: byte offset of record (g, b) (16-byte aligned)
  const unsigned char *rec;
  int G, NB, ncols, rows_cap, rec_cap, stages;
};

__host__ __device__ inline int stg_align16(long long b) { return (int)((b + 15) & ~15LL); }
__host__ __device__ inline int stg_stage_bytes(int rec_cap) { return kStgW * 8 + stg_align16(rec_cap); }
__host__ __device__ inline int stg_smem_bytes(int stages, int rows_cap, int rec_cap) {
  return stages * stg_stage_bytes(rec_cap) + stg_align16((long long)rows_cap * 8);
}
// byte offsets inside a record with nsl slices and `slots` slots
__host__ __device__ inline int stg_lrow_off(int nsl) { return stg_align16(4LL * (nsl + 2)); }
__host__ __device__ inline int stg_lci_off(int nsl) { return stg_lrow_off(nsl) + 64 * nsl; }
__host__ __device__ inline long long stg_val_off(int nsl, long long slots) {
  return stg_lci_off(nsl) + 2 * slots;
}
__host__ __device__ inline long long stg_rec_bytes(int nsl, long long slots) {
  return stg_val_off(nsl, slots) + 8 * slots;
}

template <class Epi>
__global__ void __launch_bounds__(kStgThreads, 1)
k_stg(StgMat M, const double *__restrict__ xg, Epi epi) {
  static_assert(Epi::NQ == 0, "STG engine: iteration epilogues only");
  extern __shared__ __align__(128) unsigned char stg_sm[];
  __shared__ uint64_t full[kStgMaxStages], empty[kStgMaxStages];
  if (!epi.enter()) return;
  const int g = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = M.stages, SB = stg_stage_bytes(M.rec_cap);
  double *psum = (double *)(stg_sm + (size_t)S * SB);
  const int r0 = M.row_start[g], rows = M.row_start[g + 1] - r0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kStgWarps);
    }
    fence_mbar_init();
  }
  for (int i = tid; i < rows; i += kStgThreads) psum[i] = 0.0;
  __syncthreads();

  if (warp == kStgWarps) {                       // producer: vector chunk + record, per chunk
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();
      for (int b = 0; b < M.NB; ++b) {
        const int st = b % S;
        if (b >= S) mbar_wait(&empty[st], (uint32_t)(((b / S) - 1) & 1));
        unsigned char *base = stg_sm + (size_t)st * SB;
        double *dst = (double *)base;
        const int ncol = min(kStgW, M.ncols - b * kStgW);
        const uint32_t vbytes = (uint32_t)(ncol * 8) & ~15u;
        if (ncol & 1) dst[ncol - 1] = xg[(size_t)b * kStgW + ncol - 1];   // before the arrive (release)
        const long long q = (long long)g * M.NB + b;
        const uint32_t rbytes = (uint32_t)(M.goff[q + 1] - M.goff[q]);
        mbar_expect_tx(&full[st], vbytes + rbytes);
#ifndef HPR_STG_VPIECES
#define HPR_STG_VPIECES 1   // bulk copies per vector chunk
#endif
        for (int pc = 0; pc < HPR_STG_VPIECES; ++pc) {
          const uint32_t pb = (vbytes / HPR_STG_VPIECES) & ~15u;
          const uint32_t o = pc * pb, nb = pc + 1 == HPR_STG_VPIECES ? vbytes - o : pb;
          if (nb)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                ::"r"(smem_u32((unsigned char *)dst + o)), "l"((const unsigned char *)(xg + (size_t)b * kStgW) + o),
                  "r"(nb), "r"(smem_u32(&full[st]))
                : "memory");
        }
        if (rbytes) bulk_g2s(base + kStgW * 8, M.rec + M.goff[q], rbytes, &full[st], keep);
      }
    }
    return;
  }

  for (int b = 0; b < M.NB; ++b) {
    const int st = b % S;
    const unsigned char *base = stg_sm + (size_t)st * SB;
    const double *wv = (const double *)base;
    const unsigned char *R = base + kStgW * 8;
    mbar_wait(&full[st], (uint32_t)((b / S) & 1));
    const long long q = (long long)g * M.NB + b;
    const int nsl = M.goff[q + 1] > M.goff[q] ? *(const int *)R : 0;
    const int *soff = (const int *)R + 1;
    const unsigned short *lrow = (const unsigned short *)(R + stg_lrow_off(nsl));
    const unsigned short *lci = (const unsigned short *)(R + stg_lci_off(nsl));
    const double *val = (const double *)(R + stg_val_off(nsl, nsl ? soff[nsl] : 0));
    // each warp runs kStgSpw slices at once (independent chains)
    for (int j0 = warp; j0 < nsl; j0 += kStgSpw * kStgWarps) {
      int lr[kStgSpw], s0[kStgSpw], L[kStgSpw];
      double sm_[kStgSpw];
      int Lmax = 0;
#pragma unroll
      for (int q = 0; q < kStgSpw; ++q) {
        const int j = j0 + q * kStgWarps;
        lr[q] = kStgPad;
        s0[q] = 0;
        L[q] = 0;
        if (j < nsl) {
          lr[q] = lrow[j * 32 + lane];
          s0[q] = soff[j] + lane;
          L[q] = (soff[j + 1] - soff[j]) >> 5;
        }
        Lmax = max(Lmax, L[q]);
      }
#pragma unroll
      for (int q = 0; q < kStgSpw; ++q) sm_[q] = lr[q] != kStgPad ? psum[lr[q]] : 0.0;
      // batches of 4 slots per slice, predicated
      for (int k = 0; k < Lmax; k += 4) {
        unsigned c[kStgSpw][4];
        double v[kStgSpw][4], x[kStgSpw][4];
#pragma unroll
        for (int q = 0; q < kStgSpw; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool on = lr[q] != kStgPad && k + u < L[q];
            c[q][u] = on ? lci[s0[q] + (k + u) * 32] : kStgPad;
            v[q][u] = on ? val[s0[q] + (k + u) * 32] : 0.0;
          }
#pragma unroll
        for (int q = 0; q < kStgSpw; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) x[q][u] = c[q][u] != kStgPad ? wv[c[q][u]] : 0.0;
#pragma unroll
        for (int q = 0; q < kStgSpw; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c[q][u] != kStgPad) sm_[q] = __dadd_rn(sm_[q], __dmul_rn(v[q][u], x[q][u]));
      }
#pragma unroll
      for (int q = 0; q < kStgSpw; ++q)
        if (lr[q] != kStgPad) psum[lr[q]] = sm_[q];
    }
    // every consumer is done with chunk b (its stage and its running sums)
    asm volatile("bar.sync 1, %0;" ::"n"(kStgWarps * 32) : "memory");
    if (lane == 0) {
      fence_proxy_async();                       // generic reads before the async refill
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
  }
  for (int i = tid; i < rows; i += kStgWarps * 32) {
    epi.prefetch(r0 + i);
    epi.finish(r0 + i, psum[i], nullptr);
  }
}

// ---- layout construction ----
// items (CTA g, chunk b, local row): key = (g * NB + b) << 16 | (65535 - count),
// value = local row.  Thread per row; a count above 65534 raises *overflow.
__global__ void k_stg_items(const int *rp, const int *ci, int nrows, const int *row_start, int G,
                            int NB, unsigned *key, int *lrow, int *overflow) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    int a = 0, z = G;                           // CTA of row r: last g with row_start[g] <= r
    while (z - a > 1) {
      const int mid = (a + z) >> 1;
      if (row_start[mid] <= r) a = mid; else z = mid;
    }
    const int g = a, lr = r - row_start[g];
    int e = rp[r];
    const int e1 = rp[r + 1];
    for (int b = 0; b < NB; ++b) {
      const long long hi = (long long)(b + 1) * kStgW;
      int cnt = 0;
      while (e < e1 && ci[e] < hi) {
        ++e;
        ++cnt;
      }
      if (cnt > 65534) {
        *overflow = 1;
        cnt = 65534;
      }
      const size_t it = (size_t)r * NB + b;
      key[it] = ((unsigned)(g * NB + b) << 16) | (unsigned)(65535 - cnt);
      lrow[it] = lr;
    }
  }
}

// record geometry of group q from its sorted items [gs, ge): slices, slots, bytes
__device__ __forceinline__ void stg_group_geom(const unsigned *skey, long long gs, long long ge,
                                               int *nsl_out, long long *slots_out) {
  long long a = gs, z = ge;                     // first item with count 0
  while (a < z) {
    const long long mid = (a + z) >> 1;
    if ((skey[mid] & 0xFFFFu) == 0xFFFFu) z = mid; else a = mid + 1;
  }
  const long long ne = a - gs;
  const int nsl = (int)((ne + 31) / 32);
  long long slots = 0;
  for (int j = 0; j < nsl; ++j) slots += 32LL * (65535 - (int)(skey[gs + 32LL * j] & 0xFFFFu));
  *nsl_out = nsl;
  *slots_out = slots;
}

// group starts from the sorted keys (group id = key >> 16)
__global__ void k_stg_gstart(const unsigned *skey, long long nitems, int ngroups, long long *gstart) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nitems;
       k += (long long)gridDim.x * blockDim.x) {
    const int cur = (int)(skey[k] >> 16);
    const int prev = k == 0 ? -1 : (int)(skey[k - 1] >> 16);
    for (int q = prev + 1; q <= cur; ++q) gstart[q] = k;
    if (k == nitems - 1)
      for (int q = cur + 1; q <= ngroups; ++q) gstart[q] = nitems;
  }
}

__global__ void k_stg_recsize(const unsigned *skey, const long long *gstart, int ngroups,
                              long long *rbytes) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ngroups) return;
  int nsl;
  long long slots;
  stg_group_geom(skey, gstart[q], gstart[q + 1], &nsl, &slots);
  rbytes[q] = nsl ? stg_align16(stg_rec_bytes(nsl, slots)) : 0;
}

// fill record q (one CTA per record); pos[csr entry] = index of its value
// among the doubles of the record array (rec viewed as double*)
__global__ void k_stg_fill(const int *rp, const int *ci, const int *row_start, int NB,
                           const unsigned *skey, const int *slrow, const long long *gstart,
                           const long long *goff, unsigned char *rec, int *pos) {
  extern __shared__ int sh_soff[];
  const int q = blockIdx.x;
  const int g = q / NB, b = q % NB;
  const long long gs = gstart[q], ge = gstart[q + 1];
  __shared__ int s_nsl;
  __shared__ long long s_slots;
  if (threadIdx.x == 0) {
    int nsl;
    long long slots;
    stg_group_geom(skey, gs, ge, &nsl, &slots);
    s_nsl = nsl;
    s_slots = slots;
    int acc = 0;
    for (int j = 0; j < nsl; ++j) {
      sh_soff[j] = acc;
      acc += 32 * (65535 - (int)(skey[gs + 32LL * j] & 0xFFFFu));
    }
    sh_soff[nsl] = acc;
  }
  __syncthreads();
  const int nsl = s_nsl;
  if (nsl == 0) return;
  const long long slots = s_slots;
  unsigned char *R = rec + goff[q];
  int *hdr = (int *)R;
  unsigned short *lrow = (unsigned short *)(R + stg_lrow_off(nsl));
  unsigned short *lci = (unsigned short *)(R + stg_lci_off(nsl));
  const long long vbase = (goff[q] + stg_val_off(nsl, slots)) / 8;
  if (threadIdx.x == 0) hdr[0] = nsl;
  for (int j = threadIdx.x; j <= nsl; j += blockDim.x) hdr[1 + j] = sh_soff[j];
  const long long ne_cap = 32LL * nsl;
  for (long long t = threadIdx.x; t < ne_cap; t += blockDim.x) {
    const int j = (int)(t >> 5), lane = (int)(t & 31);
    const long long it = gs + t;
    const int L = (sh_soff[j + 1] - sh_soff[j]) >> 5;
    int len = 0;
    if (it < ge) len = 65535 - (int)(skey[it] & 0xFFFFu);
    if (len == 0) {
      lrow[t] = kStgPad;
      for (int k = 0; k < L; ++k) lci[sh_soff[j] + k * 32 + lane] = kStgPad;
      continue;
    }
    const int lr = slrow[it];
    lrow[t] = (unsigned short)lr;
    const int r = row_start[g] + lr;
    int a = rp[r], z = rp[r + 1];
    const long long lo = (long long)b * kStgW;
    while (a < z) {                              // first entry with column >= b W
      const int mid = (a + z) >> 1;
      if (ci[mid] < lo) a = mid + 1; else z = mid;
    }
    for (int k = 0; k < L; ++k) {
      const int slot = sh_soff[j] + k * 32 + lane;
      if (k < len) {
        lci[slot] = (unsigned short)(ci[a + k] & (kStgW - 1));
        pos[a + k] = (int)(vbase + slot);
      } else {
        lci[slot] = kStgPad;
      }
    }
  }
}

}  // namespace hpr
