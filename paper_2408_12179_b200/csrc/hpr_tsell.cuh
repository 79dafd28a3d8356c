// hpr_tsell.cuh -- bulk-copy-streamed SELL engine ("TS") for the iteration
// phases of HBM-bound problems.
//
// Why: on the SELL engine (k_sell) every lane keeps its matrix batch (column
// indices + values) in registers while the operand gathers are outstanding, so
// the bytes an SM has in flight are capped by its register file (80 registers
// per thread, 24 warps per SM, long-scoreboard stalls).  Here a producer warp
// streams the matrix into a shared-memory ring with cp.async.bulk (the copy
// engine: no registers, no L1 miss slots) and the consumer warps only gather
// the operand vector and add.
//
// Layout: the SellMat of k_sell, unchanged, cut into BLOCKS of consecutive
// slices (hpr_capi.cu: ts_plan): a block's slots, slice offsets and -- for
// non-compact slices -- per-lane row / length headers are each one contiguous
// range, copied by one bulk copy apiece into a ring stage.  Blocks go to the
// persistent CTAs round-robin (CTA g: blocks g, g + G, ...) so, as with k_sell's
// windows, all SMs work on neighbouring rows at any time (the row-affinity
// order's L2 locality of the gathered vector survives).  The CTA's slices,
// in block order, go to its consumer warps round-robin (the rotation carries
// across blocks, so short blocks still spread over every warp); lane i adds its row's products
// in slot order -- ascending column, from 0.0, each product rounded: the
// arithmetic of k_sell and scipy's csr_matvec, so results are bit-identical.
// Each consumer warp waits on every block's full barrier and arrives once on
// its empty barrier, so the ring's phases stay in step.
#pragma once

namespace hpr {

#ifndef HPR_TS_WARPS
#define HPR_TS_WARPS 24      // consumer warps per CTA (+1 producer)
#endif
#ifndef HPR_TS_CAP
#define HPR_TS_CAP 4096      // slots per ring stage (48 KB of matrix; C3 x-phase: 2048 x 6 stages 898, 4096 x 3 870 us/iteration)
#endif
#ifndef HPR_TS_STAGES
#define HPR_TS_STAGES 3      // ring stages
#endif
#ifndef HPR_TS_U
#define HPR_TS_U 4           // entries per lane per batch
#endif
#ifndef HPR_TS_SW
#define HPR_TS_SW 32         // plan weight of a slice (bounds the slices per block; C3: 32 849, 64 863, 128 (4 stages) 878 us/iteration)
#endif
#ifndef HPR_TS_CPS
#define HPR_TS_CPS 1         // persistent CTAs per SM
#endif
constexpr int kTsCps = HPR_TS_CPS;
constexpr int kTsWarps = HPR_TS_WARPS;
constexpr int kTsThreads = (kTsWarps + 1) * 32;
constexpr int kTsCap = HPR_TS_CAP;
constexpr int kTsStages = HPR_TS_STAGES;
constexpr int kTsSw = HPR_TS_SW;
constexpr int kTsMaxSl = kTsCap / kTsSw + 1;          // slices per block (plan: weight cut)
constexpr int kTsPtrInts = (kTsMaxSl + 1 + 8 + 3) & ~3;   // slice offsets, 16-byte aligned superset
// stage layout: val[cap] f64 | ci[cap + 8] i32 (slot indices, or the block's
// index words, 16-byte aligned superset) | sptr[kTsPtrInts] i32 | aptr[kTsPtrInts] i32
// | srow[32 maxsl] i32 | slen[32 maxsl] u16
constexpr int kTsOffCi = kTsCap * 8;
constexpr int kTsOffPtr = kTsOffCi + (kTsCap + 8) * 4;
constexpr int kTsOffAp = kTsOffPtr + kTsPtrInts * 4;
constexpr int kTsOffRow = kTsOffAp + kTsPtrInts * 4;
constexpr int kTsOffLen = kTsOffRow + kTsMaxSl * kSlice * 4;
constexpr int kTsStageBytes = (kTsOffLen + kTsMaxSl * kSlice * 2 + 127) & ~127;
constexpr int kTsSmem = kTsStages * kTsStageBytes;

// Block b = slices [blk[b], blk[b+1]) of the slice range [s_lo, s_hi): cut
// where the weight slice_ptr[s] + kTsSw s crosses base + b T (T + the largest
// slice + kTsSw <= kTsCap, checked by the host), so a block holds <= kTsCap
// slots and <= T / kTsSw + 1 slices; empty slices cost weight too.  Ranges let
// the row-block path plan each column chunk on its own (no block straddles one).
__global__ void k_ts_plan(const int *slice_ptr, int s_lo, int s_hi, long long T, int nblk,
                          int *blk) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nblk) return;
  if (b == nblk) {
    blk[b] = s_hi;
    return;
  }
  const long long target = (long long)slice_ptr[s_lo] + (long long)kTsSw * s_lo + T * b;
  int a = s_lo, z = s_hi;
  while (a < z) {
    const int mid = (a + z) >> 1;
    if ((long long)slice_ptr[mid] + (long long)kTsSw * mid < target) a = mid + 1; else z = mid;
  }
  blk[b] = a;
}

// Index words of the TS engine (SellMat::aw / aptr).  k_aw_count: one warp per
// slice; cnt[s] = entries per lane when every entry's 32 lane columns are
// lane-affine (c = c0 + lane) or lane-uniform (c = c0), else 32 x entries
// (cnt[nslices] = 0; the exclusive scan of cnt is aptr).
__global__ void k_aw_count(const int *__restrict__ slice_ptr, const int *__restrict__ ci,
                           int nslices, int *cnt) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw > nslices) return;
  if (gw == nslices) {
    if (lane == 0) cnt[nslices] = 0;
    return;
  }
  const int p = slice_ptr[gw], len = (slice_ptr[gw + 1] - p) / kSlice;
  bool ok = true;
  for (int k = 0; k < len && ok; ++k) {
    const int col = ci[p + k * kSlice + lane];
    const int c0 = __shfl_sync(0xffffffffu, col, 0);
    const bool aff = __all_sync(0xffffffffu, col == c0 + lane);
    const bool uni = __all_sync(0xffffffffu, col == c0);
    ok = aff || uni;
  }
  if (lane == 0) cnt[gw] = ok ? len : kSlice * len;
}

// k_aw_fill: the words -- per entry c0 (lane-affine) or c0 | 2^31 (uniform) for
// a compressed slice, the slot indices unchanged otherwise
__global__ void k_aw_fill(const int *__restrict__ slice_ptr, const int *__restrict__ ci,
                          int nslices, const int *__restrict__ aptr, int *aw) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= nslices) return;
  const int p = slice_ptr[gw], len = (slice_ptr[gw + 1] - p) / kSlice;
  const int o = aptr[gw];
  const bool per_lane = aptr[gw + 1] - o != len;
  for (int k = 0; k < len; ++k) {
    const int col = ci[p + k * kSlice + lane];
    if (per_lane) {
      aw[o + k * kSlice + lane] = col;
    } else {
      const int c0 = __shfl_sync(0xffffffffu, col, 0);
      const bool uni = __all_sync(0xffffffffu, col == c0);
      if (lane == 0) aw[o + k] = uni ? (int)((unsigned)c0 | 0x80000000u) : c0;
    }
  }
}

#ifndef HPR_TS_REV
#define HPR_TS_REV 0         // 1: each CTA walks its blocks last to first (C3: 836.3 vs 833.1 us, off)
#endif
// the i-th block a CTA processes, as an index into its round-robin share
__device__ __forceinline__ int ts_bi(int i, int nmine) { return HPR_TS_REV ? nmine - 1 - i : i; }

template <int U, class Epi, bool AW>
__global__ void __launch_bounds__(kTsThreads, kTsCps)
k_tsell(SellMat M, const double *__restrict__ xg, Epi epi, const int *__restrict__ blk, int nblk) {
  static_assert(Epi::NQ == 0, "TS engine: iteration epilogues only");
  extern __shared__ __align__(128) unsigned char ts_sm[];
  __shared__ uint64_t full[kTsStages], empty[kTsStages];
  if (!epi.enter()) return;
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nmine = g < nblk ? (nblk - g + G - 1) / G : 0;
  if (tid == 0) {
    for (int s = 0; s < kTsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTsWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");

  if (warp == kTsWarps) {   // producer warp: the matrix does not depend on the previous phase
    const uint64_t pol = M.keep == 1 ? policy_evict_last()
                         : M.keep == 2 ? policy_evict_normal() : policy_evict_first();
    const uint64_t hpol = policy_evict_normal();
    for (int i0 = 0; i0 < nmine; i0 += 32) {
      // 32 blocks' slice ranges at once (one lane each), handed to lane 0
      int sb = 0, se = 0, pa = 0, pz = 0, wa = 0, wz = 0;
      if (i0 + lane < nmine) {
        const int b = g + ts_bi(i0 + lane, nmine) * G;
        sb = blk[b];
        se = blk[b + 1];
        pa = M.slice_ptr[sb];
        pz = M.slice_ptr[se];
        if (AW) {
          wa = M.aptr[sb];
          wz = M.aptr[se];
        }
      }
      const int cnt = min(32, nmine - i0);
      for (int j = 0; j < cnt; ++j) {
        const int s_b = __shfl_sync(0xffffffffu, sb, j), s_e = __shfl_sync(0xffffffffu, se, j);
        const int p_a = __shfl_sync(0xffffffffu, pa, j), p_z = __shfl_sync(0xffffffffu, pz, j);
        const int w_a = __shfl_sync(0xffffffffu, wa, j), w_z = __shfl_sync(0xffffffffu, wz, j);
        if (lane == 0) {
          const int i = i0 + j, st = i % kTsStages;
          if (i >= kTsStages) mbar_wait(&empty[st], (uint32_t)(((i / kTsStages) - 1) & 1));
          unsigned char *S = ts_sm + (size_t)st * kTsStageBytes;
          const uint32_t ns = (uint32_t)(p_z - p_a);
          const int q0 = s_b & ~3, q1 = (s_e + 1 + 3) & ~3;      // aligned slice-offset range
          const int nh = s_e > M.compact ? s_e - max(s_b, M.compact) : 0;   // non-compact slices
          const int h0 = max(s_b, M.compact);
          // index words: the aligned superset [w_a & ~3, (w_z + 3) & ~3)
          const int a0 = w_a & ~3, a1 = (w_z + 3) & ~3;
          const uint32_t nwb = AW ? (uint32_t)(a1 - a0) * 4u : ns * 4u;
          uint32_t bytes = ns * 8u + nwb + (uint32_t)(q1 - q0) * 4u * (AW ? 2u : 1u);
          if (nh > 0) bytes += (uint32_t)nh * (kSlice * 6);
          mbar_expect_tx(&full[st], bytes);
          if (ns) bulk_g2s(S, M.val + p_a, ns * 8u, &full[st], pol);
          if (nwb) bulk_g2s(S + kTsOffCi, AW ? M.aw + a0 : M.ci + p_a, nwb, &full[st], pol);
          bulk_g2s(S + kTsOffPtr, M.slice_ptr + q0, (uint32_t)(q1 - q0) * 4u, &full[st], hpol);
          if (AW)
            bulk_g2s(S + kTsOffAp, M.aptr + q0, (uint32_t)(q1 - q0) * 4u, &full[st], hpol);
          if (nh > 0) {
            bulk_g2s(S + kTsOffRow + (h0 - s_b) * kSlice * 4, M.slice_row + (size_t)h0 * kSlice,
                     (uint32_t)nh * kSlice * 4u, &full[st], hpol);
            bulk_g2s(S + kTsOffLen + (h0 - s_b) * kSlice * 2, M.slice_len + (size_t)h0 * kSlice,
                     (uint32_t)nh * kSlice * 2u, &full[st], hpol);
          }
        }
      }
    }
    return;
  }

  asm volatile("griddepcontrol.wait;" ::: "memory");
  int nb_s = 0, nb_e = 0;
  if (nmine > 0) {
    nb_s = blk[g + ts_bi(0, nmine) * G];
    nb_e = blk[g + ts_bi(0, nmine) * G + 1];
  }
  int rot = 0;   // slices of the CTA's earlier blocks: the warp rotation continues across blocks
  for (int i = 0; i < nmine; ++i) {
    const int st = i % kTsStages;
    const int s_b = nb_s, s_e = nb_e;
    if (i + 1 < nmine) {   // next block's slice range, loaded one block ahead
      nb_s = blk[g + ts_bi(i + 1, nmine) * G];
      nb_e = blk[g + ts_bi(i + 1, nmine) * G + 1];
    }
    const unsigned char *S = ts_sm + (size_t)st * kTsStageBytes;
    const double *rv = (const double *)S;
    const int *rc = (const int *)(S + kTsOffCi);
    const int *sptr = (const int *)(S + kTsOffPtr) - (s_b & ~3);   // indexed by slice id
    const int *aptr = (const int *)(S + kTsOffAp) - (s_b & ~3);
    const int *srow = (const int *)(S + kTsOffRow);
    const unsigned short *slen_l = (const unsigned short *)(S + kTsOffLen);
    mbar_wait(&full[st], (uint32_t)((i / kTsStages) & 1));
    const int p0 = sptr[s_b];
    const int w0 = AW ? aptr[s_b] & ~3 : 0;
    for (int s = s_b + (warp - rot % kTsWarps + kTsWarps) % kTsWarps; s < s_e; s += kTsWarps) {
      const int a = sptr[s] - p0;   // slot offset inside the stage
      const int slen = (sptr[s + 1] - sptr[s]) / kSlice;
      // column of entry k: per-lane words (slot order) or one word per entry
      int wo = a;
      bool per_lane = true;
      if (AW) {
        wo = aptr[s] - w0;
        per_lane = aptr[s + 1] - aptr[s] != slen;
      }
      auto col = [&](int k) -> int {
        if (per_lane) return rc[wo + k * kSlice + lane];
        const int wd = rc[wo + k];
        return (wd & 0x7fffffff) + (wd < 0 ? 0 : lane);
      };
      int row, len;
      if (s < M.compact) {
        row = s * kSlice + lane;
        len = slen;
      } else {
        row = srow[(s - s_b) * kSlice + lane];
        len = slen_l[(s - s_b) * kSlice + lane];
      }
      if (row >= 0) epi.prefetch(row);
      double sum = 0.0;
      if constexpr (has_init<Epi>::value)
        if (row >= 0) sum = epi.init(row);
      // depth-2: batch k+1's gathers are in flight while batch k is added
      double v0[U], x0[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < len) {
          const int p = a + u * kSlice + lane;
          v0[u] = rv[p];
          x0[u] = gather<false>(xg + col(u));
        }
      for (int k = 0; k < slen; k += U) {
        double v1[U], x1[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (k + U + u < len) {
            const int p = a + (k + U + u) * kSlice + lane;
            v1[u] = rv[p];
            x1[u] = gather<false>(xg + col(k + U + u));
          }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (k + u < len) sum = __dadd_rn(sum, __dmul_rn(v0[u], x0[u]));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          v0[u] = v1[u];
          x0[u] = x1[u];
        }
      }
      if (row >= 0) epi.finish(row, sum, nullptr);
    }
    rot += s_e - s_b;
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async();   // generic-proxy reads before the bulk refill
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
  }
  const uint64_t pol = policy_evict_first();
  for (int li = g * kTsWarps + warp; li < M.nlong; li += G * kTsWarps)
    long_row(M, M.long_rows[li], lane, xg, epi, nullptr, pol);
}

}  // namespace hpr
