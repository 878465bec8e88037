// Micro-benchmark: random 8-byte gather throughput from distributed shared
// memory (a V window spread over a thread-block cluster) vs local shared
// memory vs L2 (__ldg from an L2-resident buffer).  Decides whether a
// cluster-wide V window can beat the L2 gathers that bound K1 on C5 rank
// blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_gather dsmem_gather.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int kLogSlice = 14;  // 16384 doubles = 128 KB per CTA
constexpr int kSlice = 1 << kLogSlice;
constexpr int kU = 8;

__device__ __forceinline__ unsigned xs(unsigned& s) {
  s ^= s << 13;
  s ^= s >> 17;
  s ^= s << 5;
  return s;
}

// mode 0: DSMEM across the cluster, 1: local shared memory, 2: L2 (__ldg)
template <int MODE>
__global__ void __launch_bounds__(512, 1) gather(const double* __restrict__ g, int iters, int cl,
                                                 double* out) {
  extern __shared__ double slice[];
  cg::cluster_group cluster = cg::this_cluster();
  for (int i = threadIdx.x; i < kSlice; i += blockDim.x) slice[i] = (double)(i + blockIdx.x);
  cluster.sync();
  unsigned s = 0x9E3779B9u ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
  const unsigned mask = (unsigned)(cl << kLogSlice) - 1u;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned idx = xs(s) & mask;
      if (MODE == 0) {
        const double* p = cluster.map_shared_rank(slice + (idx & (kSlice - 1)), idx >> kLogSlice);
        v[u] = *p;
      } else if (MODE == 1) {
        v[u] = slice[idx & (kSlice - 1)];
      } else {
        v[u] = __ldg(g + idx);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += v[u];
  }
  cluster.sync();
  if (acc == 1.2345) out[0] = acc;
}

template <int MODE>
static float run(int cl, int blocks, int threads, int iters, const double* g, double* out) {
  auto fn = gather<MODE>;
  const int smem = kSlice * 8;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cl > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cudaOccupancyMaxActiveClusters(&nclusters, (void*)fn, &cfg);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, fn, g, iters, cl, out);  // warm
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, fn, g, iters, cl, out);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double gathers = (double)blocks * threads * iters * kU;
  const int active = blocks < nclusters * cl ? blocks : nclusters * cl;
  printf("mode %d cluster %2d blocks %3d (max active clusters %d) threads %d: %.3f ms, %.2f Ggathers/s, "
         "%.2f gathers/clk/SM (1.965 GHz, %d SMs) %s\n",
         MODE, cl, blocks, nclusters, threads, ms, gathers / ms * 1e-6,
         gathers / (ms * 1e-3) / 1.965e9 / active, active, e == cudaSuccess ? "" : cudaGetErrorString(e));
  return ms;
}

int main() {
  double *g, *out;
  cudaMalloc(&g, sizeof(double) * (16 << kLogSlice));
  cudaMemset(g, 0, sizeof(double) * (16 << kLogSlice));
  cudaMalloc(&out, 8);
  const int iters = 2000;
  for (int threads : {256, 512}) {
    for (int cl : {2, 4, 8, 16}) {
      const int blocks = (148 / cl) * cl;
      run<0>(cl, blocks, threads, iters, g, out);
    }
    run<1>(8, 144, threads, iters, g, out);
    run<2>(8, 144, threads, iters, g, out);
    run<2>(1, 148, threads, iters, g, out);
  }
  return 0;
}
