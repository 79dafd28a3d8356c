// Microbenchmark: random 8-byte gathers from a vector held in the distributed
// shared memory of a thread-block cluster (each CTA holds 1/C of it) vs the
// same gathers from global memory (L2-resident vector) vs the CTA's own smem.
// Design probe for a DSMEM-resident operand vector in the SELL SpMV (not
// product code).  One CTA per SM, 768 threads, 8 independent loads per thread
// in flight per step.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kT = 768;
constexpr int kILP = 8;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// mode 0: DSMEM (cluster of C, each CTA holds nloc doubles); 1: global gather
// over C * nloc doubles; 2: own-smem gather over nloc doubles
template <int MODE>
__global__ void __launch_bounds__(kT, 1) k_gather(const double *g, int nloc, int C, int steps,
                                                  double *out) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  for (int i = tid; i < nloc; i += kT) sm[i] = (double)(i & 1023);
  if (MODE == 0) cluster_sync(); else __syncthreads();
  const uint32_t base = smem_u32(sm);
  const uint32_t total = (uint32_t)nloc * (MODE == 2 ? 1u : (uint32_t)C);
  double acc = 0.0;
  uint32_t seed = (blockIdx.x * kT + tid) * 0x9e3779b9u;
  for (int s = 0; s < steps; ++s) {
    double v[kILP];
#pragma unroll
    for (int u = 0; u < kILP; ++u) {
      const uint32_t idx = hash32(seed + (uint32_t)(s * kILP + u)) % total;
      if (MODE == 0) {
        const uint32_t rank = idx / (uint32_t)nloc, off = idx - rank * (uint32_t)nloc;
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + off * 8), "r"(rank));
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v[u]) : "r"(ra));
      } else if (MODE == 1) {
        v[u] = __ldg(g + idx);
      } else {
        v[u] = sm[idx];
      }
    }
#pragma unroll
    for (int u = 0; u < kILP; ++u) acc += v[u];
  }
  if (MODE == 0) cluster_sync();
  if (acc == -1.0) out[blockIdx.x] = acc;
}

template <int MODE>
int run(int C, int nloc, int steps, const double *g, double *out, int nsm) {
  const size_t smem = (size_t)nloc * 8;
  CK(cudaFuncSetAttribute(k_gather<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (MODE == 0 && C > 8) CK(cudaFuncSetAttribute(k_gather<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  const int grid = MODE == 0 ? (nsm / C) * C : nsm;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MODE == 0 ? C : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (MODE == 0) {
    CK(cudaOccupancyMaxActiveClusters(&ncl, k_gather<MODE>, &cfg));
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, k_gather<MODE>, g, nloc, C, steps, out));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
  }
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const double loads = (double)grid * kT * steps * kILP;
  const double per_sm_clk = loads / grid / (ms * 1e-3 * clk * 1e3);
  printf("mode=%s C=%2d grid=%3d active_clusters=%3d vec=%7.1f KB: %.3f ms, %.3f loads/clk/SM, %.1f G loads/s total\n",
         MODE == 0 ? "dsmem " : MODE == 1 ? "global" : "smem  ", C, grid, ncl,
         (MODE == 2 ? nloc : (double)nloc * C) * 8 / 1024.0, ms, per_sm_clk, loads / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *g, *out;
  const int nmax = 1 << 21;
  CK(cudaMalloc(&g, sizeof(double) * nmax));
  CK(cudaMemset(g, 0, sizeof(double) * nmax));
  CK(cudaMalloc(&out, sizeof(double) * 1024));
  const int steps = 400;
  for (int C : {2, 4, 8, 16}) {
    const int nloc = 25600;   // 200 KB per CTA
    if (run<0>(C, nloc, steps, g, out, nsm)) return 1;
    if (run<1>(C, nloc, steps, g, out, nsm)) return 1;
  }
  run<2>(1, 25600, steps, g, out, nsm);
  return 0;
}
