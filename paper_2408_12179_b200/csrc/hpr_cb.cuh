// hpr_cb.cuh -- column-blocked, shared-memory-staged SpMV engine ("CB").
//
// For matrices whose operand vector is small next to the work (C2: n = 2e5,
// nnz = 5e6), the SELL engine's cost is the operand gather: every nonzero is a
// random 8-byte load that occupies one L1TEX wavefront (measured: the C2
// iteration kernels sit at 50-60 % L1TEX / LTS throughput with ~30 % warps
// active).  The CB engine instead stages the operand vector through shared
// memory, one column block of kCbW doubles at a time, and gathers from there:
//
//   * one persistent CTA per SM owns a contiguous, nnz-balanced range of rows;
//   * the matrix is regrouped by (CTA, column block): group (g, b) holds the
//     entries of CTA g's rows whose columns fall in block b, row-major with
//     ascending columns inside a row, 16-byte aligned, with per-row offsets;
//   * per block, ONE thread issues 1D bulk copies (cp.async.bulk, mbarrier
//     completion) of the vector block, the group's values, its 16-bit local
//     column indices and its row offsets into a pipeline stage; the other
//     stage is being consumed meanwhile;
//   * each thread owns rows and carries their running sums across blocks in
//     shared memory: blocks ascend, entries ascend inside a block, so every
//     row is still summed left to right from 0.0 with separately rounded
//     products -- bit-identical to scipy's csr_matvec and to the SELL engine;
//   * after the last block the same epilogue functors (EpiXIter / EpiYIter)
//     run per row.
#pragma once

namespace hpr {

constexpr int kCbThreads = 512;      // consumer threads (+ one producer warp)
constexpr int kCbWarps = kCbThreads / 32;
constexpr int kCbMaxStages = 4;
constexpr int kCbMaxRpt = 4;         // rows per consumer thread (register running sums)

struct CbMat {
  const int *row_start;        // G + 1
  const long long *gseg;       // G * NB + 1: padded start of group (g, b) in the entry arrays
  const int *rpb;              // per group: rows_g + 1 offsets relative to the group start
  const long long *rpb_base;   // G * NB: start of group (g, b) in rpb (16-byte aligned)
  const unsigned short *ci;    // column - b * W
  const double *val;
  int G, NB, W, ncols;
  int rows_cap;                // >= max rows_g (shared-memory sizing)
  int seg_cap;                 // >= max padded group entries
  int stages;                  // pipeline depth (2..kCbMaxStages)
};

struct CbSmem {                // byte offsets inside the dynamic shared memory
  int wbuf, sval, sci, srpb, rs, stage_bytes, total;
};

__host__ __device__ inline int cb_align16(int b) { return (b + 15) & ~15; }

__host__ __device__ inline CbSmem cb_smem(int W, int seg_cap, int rows_cap, int stages) {
  CbSmem s;
  const int w = W * 8, v = seg_cap * 8, c = cb_align16(seg_cap * 2), r = cb_align16((rows_cap + 1) * 4);
  s.stage_bytes = w + v + c + r;
  s.wbuf = 0;
  s.sval = w;
  s.sci = w + v;
  s.srpb = w + v + c;
  s.rs = stages * s.stage_bytes;
  s.total = s.rs;
  return s;
}

__device__ __forceinline__ void bulk_g2s_nohint(void *dst, const void *src, uint32_t bytes,
                                                uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Warp-specialised pipeline: warp kCbWarps (the producer) issues the bulk copies
// of block b into stage b % S as soon as every consumer warp has released that
// stage (per-stage "empty" mbarriers); the consumer warps wait on the stage's
// "full" mbarrier, add their rows' products into REGISTER running sums (RPT
// rows per thread) and release it -- no CTA-wide barrier in the loop.
template <int RPT, class Epi>
__global__ void __launch_bounds__(kCbThreads + 32, 1)
k_cb(CbMat M, const double *__restrict__ xg, Epi epi, double *part) {
  extern __shared__ __align__(128) unsigned char cbsm[];
  __shared__ uint64_t full[kCbMaxStages], empty[kCbMaxStages];
  double acc[Epi::NQ > 0 ? Epi::NQ : 1];
#pragma unroll
  for (int q = 0; q < (Epi::NQ > 0 ? Epi::NQ : 1); ++q) acc[q] = 0.0;
  if (!epi.enter()) return;
  const int g = blockIdx.x, tid = threadIdx.x;
  const int r0 = M.row_start[g], rows = M.row_start[g + 1] - r0;
  const int S = M.stages;
  const CbSmem L = cb_smem(M.W, M.seg_cap, M.rows_cap, S);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCbWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= kCbThreads) {                       // producer warp
    if (tid == kCbThreads) {
      for (int b = 0; b < M.NB; ++b) {
        const int st = b % S;
        if (b >= S) mbar_wait(&empty[st], (uint32_t)(((b / S) - 1) & 1));
        unsigned char *base = cbsm + st * L.stage_bytes;
        const long long q = (long long)g * M.NB + b;
        const long long e0 = M.gseg[q], e1 = M.gseg[q + 1];
        const int wcols = min(M.W, M.ncols - b * M.W);
        const uint32_t wb = (uint32_t)cb_align16(wcols * 8);
        const uint32_t vb = (uint32_t)((e1 - e0) * 8);            // e1 - e0: multiple of 8
        const uint32_t cb = (uint32_t)((e1 - e0) * 2);
        const uint32_t rb = (uint32_t)cb_align16((rows + 1) * 4);
        mbar_expect_tx(&full[st], wb + vb + cb + rb);
        bulk_g2s_nohint(base + L.wbuf, xg + (long long)b * M.W, wb, &full[st]);
        if (vb) {
          bulk_g2s_nohint(base + L.sval, M.val + e0, vb, &full[st]);
          bulk_g2s_nohint(base + L.sci, M.ci + e0, cb, &full[st]);
        }
        bulk_g2s_nohint(base + L.srpb, M.rpb + M.rpb_base[q], rb, &full[st]);
      }
    }
    return;
  }
  double rs[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) rs[j] = 0.0;
  for (int b = 0; b < M.NB; ++b) {
    const int st = b % S;
    mbar_wait(&full[st], (uint32_t)((b / S) & 1));
    const unsigned char *base = cbsm + st * L.stage_bytes;
    const double *wv = (const double *)(base + L.wbuf);
    const double *sv = (const double *)(base + L.sval);
    const unsigned short *sc = (const unsigned short *)(base + L.sci);
    const int *sr = (const int *)(base + L.srpb);
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int i = tid + j * kCbThreads;
      if (i < rows) {
        double s = rs[j];
        const int k1 = sr[i + 1];
        for (int k = sr[i]; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(sv[k], wv[sc[k]]));
        rs[j] = s;
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) {
      fence_proxy_async();                       // generic reads before the async refill
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int i = tid + j * kCbThreads;
    if (i < rows) {
      epi.prefetch(r0 + i);
      epi.finish(r0 + i, rs[j], acc);
    }
  }
  if constexpr (Epi::NQ > 0) static_assert(Epi::NQ == 0, "CB engine: iteration epilogues only");
}

// ---- layout construction (hpr_analyze) ----
// row_start[g] = first row whose prefix nnz reaches g * nnz / G (then forced
// strictly increasing so every CTA owns at least one row).  One block: thread
// g binary-searches its boundary, thread 0 applies the monotone fix-up.
__global__ void k_cb_rowstart(const int *rp, int nrows, int G, int *row_start) {
  const long long nnz = rp[nrows];
  for (int g = 1 + threadIdx.x; g < G; g += blockDim.x) {
    const long long target = (nnz * g) / G;
    int a = 0, z = nrows;
    while (a < z) {                                // first row r with rp[r] >= target
      const int mid = (a + z) >> 1;
      if ((long long)rp[mid] >= target) z = mid; else a = mid + 1;
    }
    row_start[g] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    row_start[0] = 0;
    int prev = 0;
    for (int g = 1; g < G; ++g) {
      int a = row_start[g];
      a = max(a, prev + 1);                        // >= 1 row for this CTA
      a = min(a, nrows - (G - g));                 // >= 1 row for each later CTA
      row_start[g] = a;
      prev = a;
    }
    row_start[G] = nrows;
  }
}

// key of every entry = g * NB + column block; local row of the entry
__global__ void k_cb_keys(const int *rp, const int *ci, const int *row_start, int G, int NB, int W,
                          int *key, int *lrow) {
  const int g = blockIdx.x;
  const int r0 = row_start[g], r1 = row_start[g + 1];
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x)
    for (int e = rp[r]; e < rp[r + 1]; ++e) {
      key[e] = g * NB + ci[e] / W;
      lrow[e] = r - r0;
    }
}

// group sizes from the sorted keys: cnt[q] for q < G * NB
__global__ void k_cb_count(const int *skey, long long nnz, int ngroups, int *gstart) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int cur = skey[k];
    const int prev = k == 0 ? -1 : skey[k - 1];
    for (int q = prev + 1; q <= cur; ++q) gstart[q] = (int)k;
    if (k == nnz - 1)
      for (int q = cur + 1; q <= ngroups; ++q) gstart[q] = (int)nnz;
  }
}

// padded group starts (8-entry alignment) and rpb bases (4-int alignment)
__global__ void k_cb_pad(const int *gstart, const int *row_start, int G, int NB, long long *gseg,
                         long long *rpb_base) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long e = 0, r = 0;
  for (int g = 0; g < G; ++g) {
    const int rows = row_start[g + 1] - row_start[g];
    for (int b = 0; b < NB; ++b) {
      const int q = g * NB + b;
      gseg[q] = e;
      rpb_base[q] = r;
      e += ((long long)(gstart[q + 1] - gstart[q]) + 7) / 8 * 8;
      r += ((long long)rows + 1 + 3) / 4 * 4;
    }
  }
  gseg[(long long)G * NB] = e;
}

// entries to their padded positions; per-group row offsets; CSR -> CB map
__global__ void k_cb_fill(const int *skey, const int *perm, const int *lrow, const int *ci,
                          const int *gstart, const long long *gseg, const long long *rpb_base,
                          const int *row_start, int NB, int W, long long nnz, unsigned short *cci,
                          int *rpb, long long *pos) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x) {
    const int q = skey[k];
    const int p = perm[k];
    const int rel = (int)(k - gstart[q]);
    const long long dst = gseg[q] + rel;
    const int b = q % NB;
    cci[dst] = (unsigned short)(ci[p] - b * W);
    pos[p] = dst;
    // row offsets: this entry starts its row inside the group -> rows (prev, row] begin here
    const int row = lrow[p];
    const int prow = (k > gstart[q]) ? lrow[perm[k - 1]] : -1;
    int *rr = rpb + rpb_base[q];
    for (int j = prow + 1; j <= row; ++j) rr[j] = rel;
    if (k + 1 == gstart[q + 1]) {               // last entry of the group
      const int g = q / NB;
      const int rows = row_start[g + 1] - row_start[g];
      for (int j = row + 1; j <= rows; ++j) rr[j] = rel + 1;
    }
  }
}

// empty groups: all row offsets 0
__global__ void k_cb_empty(const int *gstart, const long long *rpb_base, const int *row_start,
                           int G, int NB, int *rpb) {
  const int q = blockIdx.x;
  if (q >= G * NB) return;
  if (gstart[q + 1] != gstart[q]) return;
  const int g = q / NB;
  const int rows = row_start[g + 1] - row_start[g];
  for (int j = threadIdx.x; j <= rows; j += blockDim.x) rpb[rpb_base[q] + j] = 0;
}

// CSR values -> CB slots
__global__ void k_cb_scatter(const long long *pos, const double *src, double *dst, long long nnz) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
       k += (long long)gridDim.x * blockDim.x)
    dst[pos[k]] = src[k];
}

}  // namespace hpr
