// Micro-benchmark: achievable HBM read bandwidth on this B200 for a pure
// streaming read (the ceiling K1/K3 read against), vs the copy peak in
// MEASURED_PEAKS.json.  Variants: 16-byte ld.global.nc loads (U in flight per
// thread), and per-warp cp.async rings into shared memory (K1's scheme).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(512) rd_ld(const double2* __restrict__ p, size_t n2, double* out) {
  double acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) acc += __ldcs(p + i).x;
  if (acc == 1.2345) out[0] = acc;
}

__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// each warp streams a contiguous range through an S-stage ring of CH-byte chunks
template <int S, int CH>
__global__ void __launch_bounds__(1024, 1) rd_ring(const char* __restrict__ p, size_t bytes, double* out) {
  extern __shared__ __align__(16) char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t gw = (size_t)blockIdx.x * nw + warp, tw = (size_t)gridDim.x * nw;
  const size_t per = bytes / tw / CH * CH;
  const char* base = p + gw * per;
  const size_t nb = per / CH;
  char* ring = sm + warp * S * CH;
  const unsigned rs = (unsigned)__cvta_generic_to_shared(ring);
  double acc = 0;
  auto issue = [&](size_t i, int st) {
    if (i < nb)
      for (int c = lane; c < CH / 16; c += 32) cp16(rs + st * CH + 16 * c, base + i * CH + 16 * c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < S; ++s) issue(s, s);
  int st = 0;
  for (size_t i = 0; i < nb; ++i) {
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    __syncwarp();
    const double* d = reinterpret_cast<const double*>(ring + st * CH);
    for (int c = lane; c < CH / 8; c += 32) acc += d[c];
    __syncwarp();
    issue(i + S, st);
    st = st + 1 == S ? 0 : st + 1;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? (size_t)(atof(argv[1]) * (1ull << 30)) / 65536 * 65536 : (16ull << 30);
  char* p;
  double* out;
  if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 8);
  cudaMemset(p, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-28s %8.3f ms  %7.0f GB/s  (%s)\n", name, best, bytes / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  const size_t n2 = bytes / 16;
  for (int bps : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ld.nc v2 U=4 %dx512/SM", bps);
    timeit(nm, [&] { rd_ld<4><<<sms * bps, 512>>>((const double2*)p, n2, out); });
    snprintf(nm, 64, "ld.nc v2 U=8 %dx512/SM", bps);
    timeit(nm, [&] { rd_ld<8><<<sms * bps, 512>>>((const double2*)p, n2, out); });
  }
  {
    auto f = rd_ring<4, 1024>;
    int smem = 32 * 4 * 1024;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("cp.async ring 32w x 4 x 1KB", [&] { f<<<sms, 1024, smem>>>(p, bytes, out); });
    auto g = rd_ring<3, 2048>;
    int smem2 = 32 * 3 * 2048;
    cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    timeit("cp.async ring 32w x 3 x 2KB", [&] { g<<<sms, 1024, smem2>>>(p, bytes, out); });
    auto h = rd_ring<3, 3072>;
    int smem3 = 12 * 3 * 3072;
    cudaFuncSetAttribute(h, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    timeit("cp.async ring 12w x 3 x 3KB", [&] { h<<<sms, 384, smem3>>>(p, bytes, out); });
  }
  return 0;
}
