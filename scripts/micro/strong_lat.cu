// Latency of L2-coherent accesses from one thread (idle GPU) and under polling load:
// dependent chains of ld.global.cg / ld.relaxed.gpu / ld.acquire.gpu / ld.volatile /
// atom.add / st.relaxed.gpu+ld (ping) over addresses spread across L2 slices.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strong_lat strong_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p) {
  unsigned long long v;
  if (KIND == 0) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (KIND == 1) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (KIND == 2) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (KIND == 3) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (KIND == 4) asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], 0;" : "=l"(v) : "l"(p) : "memory");
  if (KIND == 5) asm volatile("ld.relaxed.cta.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (KIND == 6) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int KIND>
__global__ void chain(const unsigned long long* buf, int stride_words, int n, long long* out) {
  if (threadIdx.x != 0) return;
  const unsigned long long* p = buf + (size_t)blockIdx.x * 4096;
  unsigned long long off = 0;
  for (int i = 0; i < 16; ++i) off += ld<KIND>(p + off + (i % 8) * stride_words);  // warm (zeros)
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) off += ld<KIND>(p + off + (i % 8) * stride_words);
  const long long t1 = clock64();
  out[blockIdx.x] = (t1 - t0) / n + (long long)off;
}

// ping-pong between CTA 0 and CTA 1 through two words: round trip time of
// st.relaxed.gpu -> polled by the peer with ld<KIND> -> st back -> polled here
template <int KIND>
__global__ void ping(unsigned long long* a, unsigned long long* b, int n, long long* out) {
  if (threadIdx.x != 0 || blockIdx.x > 1) return;
  const long long t0 = clock64();
  for (unsigned long long i = 1; i <= (unsigned long long)n; ++i) {
    if (blockIdx.x == 0) {
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(i) : "memory");
      while (ld<KIND>(b) != i) {}
    } else {
      while (ld<KIND>(a) != i) {}
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(b), "l"(i) : "memory");
    }
  }
  out[blockIdx.x] = (clock64() - t0) / n;
}

int main() {
  unsigned long long* buf;
  long long* out;
  cudaMalloc(&buf, 148 * 4096 * 8 + (1 << 20));
  cudaMemset(buf, 0, 148 * 4096 * 8 + (1 << 20));
  cudaMalloc(&out, 148 * 8);
  const char* names[] = {"ld.cg", "ld.relaxed.gpu", "ld.acquire.gpu", "ld.volatile", "atom.add 0", "ld.relaxed.cta", "ld.cv"};
  long long h[148];
#define RUN(K)                                                                      \
  for (int blocks : {1, 148}) {                                                     \
    chain<K><<<blocks, 32>>>(buf, 64, 2000, out);                                   \
    cudaMemcpy(h, out, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);          \
    long long mn = h[0], mx = h[0];                                                 \
    for (int i = 0; i < blocks; ++i) { mn = h[i] < mn ? h[i] : mn; mx = h[i] > mx ? h[i] : mx; } \
    printf("%-16s chain, %3d CTAs: %lld..%lld cycles per load (%s)\n", names[K], blocks, mn, mx, cudaGetErrorString(cudaGetLastError())); \
  }
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6)
#define PING(K)                                                                     \
  {                                                                                 \
    cudaMemset(buf, 0, 1 << 16);                                                    \
    ping<K><<<148, 32>>>(buf, buf + 512, 2000, out);                                \
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);                                 \
    printf("%-16s ping-pong CTA0<->CTA1: %lld cycles per round trip (%s)\n", names[K], h[0], cudaGetErrorString(cudaGetLastError())); \
  }
  PING(0) PING(1) PING(2) PING(3) PING(6)
  return 0;
}
