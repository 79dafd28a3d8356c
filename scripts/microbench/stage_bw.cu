// Microbenchmark: how fast can every SM receive a whole vector into shared
// memory, block by block, with 1D bulk copies (unicast) or cluster multicast?
// (Design probe for a column-blocked, smem-staged SpMV; not product code.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

template <int Q>
__global__ void __launch_bounds__(128) k_stage(const double *v, int nblocks, int blk_elems, double *out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  const uint32_t rank = Q > 1 ? cta_rank() : 0;
  const int slice = blk_elems / Q;
  const uint32_t bytes = blk_elems * 8;
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (Q > 1) cluster_sync(); else __syncthreads();
  auto issue = [&](int b) {
    const int buf = b & 1;
    mbar_expect_tx(&bar[buf], bytes);
    const double *src = v + (size_t)b * blk_elems + rank * slice;
    double *dst = sm + buf * blk_elems + rank * slice;
    if (Q > 1) {
      const uint16_t mask = (uint16_t)((1u << Q) - 1);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                   ::"r"(smem_u32(dst)), "l"(src), "r"((uint32_t)(slice * 8)), "r"(smem_u32(&bar[buf])), "h"(mask) : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(&bar[buf])) : "memory");
    }
  };
  double acc = 0.0;
  if (tid == 0) issue(0);
  for (int b = 0; b < nblocks; ++b) {
    if (tid == 0 && b + 1 < nblocks) issue(b + 1);
    mbar_wait(&bar[b & 1], (b >> 1) & 1);
    for (int i = tid; i < blk_elems; i += 128) acc += sm[(b & 1) * blk_elems + i];
    if (Q > 1) cluster_sync(); else __syncthreads();   // buffer b&1 free again in every CTA
  }
  if (acc == 12345.678) out[blockIdx.x] = acc;
}

template <int Q>
void run(const double *v, double *out, int n_elems, int blk_elems, int nsm) {
  const int nblocks = n_elems / blk_elems;
  const int grid = (nsm / Q) * Q;
  size_t smem = 2 * (size_t)blk_elems * 8;
  cudaFuncSetAttribute(k_stage<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (Q > 8) cudaFuncSetAttribute(k_stage<Q>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = Q; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, k_stage<Q>, v, nblocks, blk_elems, out);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k_stage<Q>, v, nblocks, blk_elems, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  const double us = 1e3 * ms / reps;
  printf("Q=%2d grid=%3d vec=%.2f MB blk=%3d KB: %.2f us per pass -> per-SM receive %.1f GB/s, aggregate delivered %.2f TB/s, L2 reads (ideal) %.1f MB  %s\n",
         Q, grid, n_elems * 8 / 1e6, blk_elems * 8 / 1024, us, n_elems * 8 / us / 1e3, (double)grid * n_elems * 8 / us / 1e6,
         (double)grid / Q * n_elems * 8 / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int n = 200000 / 1024 * 1024;   // ~1.6 MB (C2's w)
  double *v, *out; cudaMalloc(&v, n * 8); cudaMalloc(&out, 4096 * 8); cudaMemset(v, 0, n * 8);
  for (int blk : {4096, 8192, 12288}) {
    const int nn = n / blk * blk;
    run<1>(v, out, nn, blk, nsm);
    run<2>(v, out, nn, blk, nsm);
    run<4>(v, out, nn, blk, nsm);
    run<8>(v, out, nn, blk, nsm);
    run<16>(v, out, nn, blk, nsm);
  }
  return 0;
}
