// Do GPU-scope (strong) loads/stores issued by several lanes of one warp to
// different 128-byte lines serialise?  Warp ping-pong between CTA 0 and CTA 1:
// L lanes each store a word to their own line, the peer's L lanes poll theirs,
// and reply the same way; cycles per round trip for L = 1..32 and per access kind.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strong_warp strong_warp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int LK>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p) {
  unsigned long long v;
  if (LK == 0) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (LK == 1) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (LK == 2) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <int SK>
__device__ __forceinline__ void st(unsigned long long* p, unsigned long long v) {
  if (SK == 0) asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  if (SK == 1) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  if (SK == 2) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  if (SK == 3) asm volatile("st.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int LK, int SK>
__global__ void ping(unsigned long long* a, unsigned long long* b, int L, int stride, int n, long long* out) {
  if (threadIdx.x >= 32 || blockIdx.x > 1) return;
  const int lane = threadIdx.x;
  const long long t0 = clock64();
  for (unsigned long long i = 1; i <= (unsigned long long)n; ++i) {
    if (blockIdx.x == 0) {
      if (lane < L) st<SK>(a + lane * stride, i);
      if (lane < L) while (ld<LK>(b + lane * stride) != i) {}
      __syncwarp();
    } else {
      if (lane < L) while (ld<LK>(a + lane * stride) != i) {}
      __syncwarp();
      if (lane < L) st<SK>(b + lane * stride, i);
    }
  }
  if (lane == 0) out[blockIdx.x] = (clock64() - t0) / n;
}

int main() {
  unsigned long long* buf;
  long long* out;
  cudaMalloc(&buf, 1 << 20);
  cudaMalloc(&out, 64);
  long long h[2];
  const char* ln[] = {"ld.cg", "ld.relaxed.gpu", "ld.volatile"};
  const char* sn[] = {"st.cg", "st.relaxed.gpu", "st.volatile", "st"};
#define RUN(LK, SK)                                                                       \
  for (int stride : {16, 1})                                                              \
    for (int L : {1, 2, 4, 8, 16, 32}) {                                                  \
      cudaMemset(buf, 0, 1 << 20);                                                        \
      ping<LK, SK><<<2, 32>>>(buf, buf + 32768, L, stride, 2000, out);                    \
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);                                     \
      printf("%-15s %-15s stride %2d words, %2d lanes: %5lld cycles per round trip (%s)\n", ln[LK], sn[SK], stride, L, h[0], \
             cudaGetErrorString(cudaGetLastError()));                                     \
    }
  RUN(1, 1) RUN(0, 0) RUN(2, 2) RUN(0, 3) RUN(1, 3)
  return 0;
}
