// Central-reducer LL all-reduce variants (see allreduce_ll.cu): where does the
// fan-in cost come from?  PAD = mailbox stride in 16-byte units (1: packed, 2: one
// 32-byte sector each, 8: one 128-byte line each); RW = reducer warps (1: lane owns
// ceil(nb/32) slots; 5: one slot per lane, combined through shared memory in the
// same order).  WIDE = 1: every lane of the posting warp posts (no effect on data).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o allreduce_ll2 allreduce_ll2.cu
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

template <int PAD, int RW>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* mb, unsigned long long* pub, int iters,
                                            double* out, long long* prof) {
  __shared__ double red[32];
  __shared__ double xs[8][32];
  __shared__ double bc;
  const int nb = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc = threadIdx.x * 1e-3 + blockIdx.x;
  unsigned call = 0;
  long long c_comm = 0;
  for (int it = 0; it < iters; ++it) {
    ++call;
    double t = warp_sum(acc);
    if (lane == 0) red[warp] = t;
    __syncthreads();
    const long long t1 = clock64();
    if (blockIdx.x != 0) {
      if (warp == 0) {
        t = warp_sum(lane < nw ? red[lane] : 0.0);
        if (lane == 0) {
          ll_store(mb + 2 * PAD * blockIdx.x, t, call);
          double s;
          while (!ll_try(pub, call, s)) {}
          bc = s;
        }
      }
    } else if (RW == 1) {
      if (warp == 0) {
        t = warp_sum(lane < nw ? red[lane] : 0.0);
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
              if (ll_try(mb + 2 * PAD * (lane + 32 * q), call, x)) {
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
        if (lane == 0) {
          ll_store(pub, s, call);
          bc = s;
        }
      }
    } else {
      // RW warps: warp q polls CTA lane + 32 q; warp 0 first reduces the block's own partial
      if (warp < RW) {
        const int c = lane + 32 * warp;
        double x = 0.0;
        if (warp == 0) {
          const double own = warp_sum(lane < nw ? red[lane] : 0.0);
          if (lane == 0) x = own;
        }
        if (c != 0 && c < nb) while (!ll_try(mb + 2 * PAD * c, call, x)) {}
        xs[warp][lane] = x;
        asm volatile("bar.sync 1, %0;" ::"r"(RW * 32) : "memory");
        if (warp == 0) {
          double s = 0;
#pragma unroll
          for (int q = 0; q < RW; ++q)
            if (lane + 32 * q < nb) s = __dadd_rn(s, xs[q][lane]);
          s = warp_sum(s);
          if (lane == 0) {
            ll_store(pub, s, call);
            bc = s;
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) c_comm += clock64() - t1;
    acc = __dadd_rn(acc, bc * 1e-30);
  }
  if (threadIdx.x == 0 && blockIdx.x == 1) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x < 2) prof[blockIdx.x] = c_comm;
}

template <int PAD, int RW>
void run(int nb, unsigned long long* mb, unsigned long long* pub, double* out, long long* prof) {
  const int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(mb, 0, 64 * 1024);
    cudaMemset(pub, 0, 4096);
    void* args[] = {&mb, &pub, (void*)&iters, &out, &prof};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k<PAD, RW>, nb, 512, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double h = 0;
    long long hp[2];
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hp, prof, 16, cudaMemcpyDeviceToHost);
    if (rep)
      printf("nb %3d pad %d reducer warps %d: %.3f us per all-reduce, comm cycles cta0 %lld cta1 %lld (%s) check %.17g\n",
             nb, PAD, RW, ms * 1e3 / iters, hp[0] / iters, hp[1] / iters, cudaGetErrorString(e), h);
  }
}

int main() {
  double* out;
  unsigned long long *mb, *pub;
  long long* prof;
  cudaMalloc(&mb, 64 * 1024);
  cudaMalloc(&pub, 4096);
  cudaMalloc(&out, 64);
  cudaMalloc(&prof, 64);
  for (int nb : {32, 74, 148}) {
    run<1, 1>(nb, mb, pub, out, prof);
    run<2, 1>(nb, mb, pub, out, prof);
    run<8, 1>(nb, mb, pub, out, prof);
    run<1, 5>(nb, mb, pub, out, prof);
    run<2, 5>(nb, mb, pub, out, prof);
    run<8, 5>(nb, mb, pub, out, prof);
  }
  return 0;
}
