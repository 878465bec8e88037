// Micro-benchmark: deterministic grid all-reduce of one double with a central
// reducer and LL-style self-validating words (no counter, no fences):
//   each CTA posts its partial as two 8-byte words (32 data bits | 32-bit call
//   number); warp 0 of CTA 0 polls the 148 mailboxes (lane i takes CTAs i,
//   i+32, ... and adds them in that order, then the xor tree: the same order as
//   the counter-barrier all-reduce), and publishes the sum in NCOPY replicated
//   slots (128 bytes apart, so the pollers spread over L2 slices); every other
//   CTA polls its copy.
// Modes: 0 = counter barrier (red.release + ld.acquire spin) + ordered read
//            (K4's grid_allreduce), 1 = central reducer, NCOPY copies.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o allreduce_ll allreduce_ll.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(~0u, v, o));
  return v;
}
__device__ __forceinline__ void ll_store(unsigned long long* dst, double v, unsigned call) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = (bits & 0xffffffffull) | ((unsigned long long)call << 32);
  const unsigned long long w1 = (bits >> 32) | ((unsigned long long)call << 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ bool ll_try(const unsigned long long* src, unsigned call, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(src) : "memory");
  if ((unsigned)(w0 >> 32) != call || (unsigned)(w1 >> 32) != call) return false;
  v = __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
  return true;
}

template <int MODE, int NCOPY>
__global__ void __launch_bounds__(512, 1) k(double* partials, unsigned* ctr, unsigned long long* mb,
                                            unsigned long long* pub, int iters, double* out, long long* prof) {
  __shared__ double red[32];
  long long c_red = 0, c_comm = 0, c_bc = 0;
  __shared__ double bc;
  const int nb = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc = threadIdx.x * 1e-3 + blockIdx.x;
  unsigned call = 0;
  for (int it = 0; it < iters; ++it) {
    ++call;
    const long long t0 = clock64();
    double t = warp_sum(acc);
    if (lane == 0) red[warp] = t;
    __syncthreads();
    if (warp == 0) {
      t = warp_sum(lane < nw ? red[lane] : 0.0);
      const long long t1 = clock64();
      if (MODE == 0) {
        if (lane == 0) {
          partials[(it & 1) * nb + blockIdx.x] = t;
          asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
          unsigned seen;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
          } while (seen < call * nb);
        }
        __syncwarp();
        double s = 0;
        for (int i = lane; i < nb; i += 32) s = __dadd_rn(s, __ldcg(partials + (it & 1) * nb + i));
        s = warp_sum(s);
        if (lane == 0) bc = s;
      } else {
        if (blockIdx.x != 0) {
          if (lane == 0) {
            ll_store(mb + 2 * blockIdx.x, t, call);
            const unsigned long long* src = pub + (blockIdx.x % NCOPY) * 16;
            double s;
            while (!ll_try(src, call, s)) {}
            bc = s;
          }
        } else {
          // reducer: lane i owns CTAs i, i+32, ...; all its polls in flight together
          double v[8];
          unsigned need = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            v[q] = 0.0;
            const int c = lane + 32 * q;
            if (c < nb && c != 0) need |= 1u << q;
          }
          if (lane == 0) v[0] = t;
          while (need) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (need & (1u << q)) {
                double x;
                if (ll_try(mb + 2 * (lane + 32 * q), call, x)) {
                  v[q] = x;
                  need &= ~(1u << q);
                }
              }
          }
          double s = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (lane + 32 * q < nb) s = __dadd_rn(s, v[q]);
          s = warp_sum(s);
          if (lane < NCOPY) ll_store(pub + lane * 16, s, call);
          if (lane == 0) bc = s;
        }
      }
      const long long t2 = clock64();
      c_red += t1 - t0; c_comm += t2 - t1;
    }
    __syncthreads();
    acc = __dadd_rn(acc, bc * 1e-30);
  }
  if (threadIdx.x == 0 && blockIdx.x == 1) out[MODE] = acc;
  if (threadIdx.x == 0 && blockIdx.x < 2) { prof[blockIdx.x * 2] = c_red; prof[blockIdx.x * 2 + 1] = c_comm; }
}

template <int MODE, int NCOPY>
void run(int sms, int threads, double* partials, unsigned* ctr, unsigned long long* mb,
         unsigned long long* pub, double* out, long long* prof) {
  const int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(ctr, 0, 4096);
    cudaMemset(mb, 0, 16 * 1024);
    cudaMemset(pub, 0, 16 * 1024);
    void* args[] = {&partials, &ctr, &mb, &pub, (void*)&iters, &out, &prof};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k<MODE, NCOPY>, sms, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double h[4] = {};
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    long long hp[4]; cudaMemcpy(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost);
    if (rep) printf("   cycles/call: cta0 reduce %lld comm %lld | cta1 reduce %lld comm %lld\n", hp[0]/iters, hp[1]/iters, hp[2]/iters, hp[3]/iters);
    if (rep)
      printf("mode %d ncopy %2d threads %4d: %.3f us per all-reduce (%s) check %.17g\n", MODE, NCOPY, threads,
             ms * 1e3 / iters, cudaGetErrorString(e), h[MODE]);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *partials, *out;
  unsigned long long *mb, *pub;
  unsigned* ctr;
  cudaMalloc(&partials, 16 * sms * sizeof(double));
  cudaMalloc(&mb, 16 * 1024);
  cudaMalloc(&pub, 16 * 1024);
  cudaMalloc(&out, 64);
  cudaMalloc(&ctr, 4096);
  long long* prof; cudaMalloc(&prof, 64);
  for (int nb : {2, 8, 32, 74, 148}) {
    printf("--- %d CTAs\n", nb);
    run<0, 1>(nb, 512, partials, ctr, mb, pub, out, prof);
    run<1, 1>(nb, 512, partials, ctr, mb, pub, out, prof);
    run<1, 16>(nb, 512, partials, ctr, mb, pub, out, prof);
  }
  return 0;
}
