// The stepped solver's LL all-reduce (krylov_step.cu: ll_post / ll_wait_result) in isolation,
// 148 CTAs x 512 threads, for NV = 1 and 3 values, and a packed variant:
//   MODE 0: as in the solver: value k of CTA c in mailbox [k][c]; reducer warp 5k+q polls value k of
//           CTAs 32q+lane (15 polling warps for NV = 3); results in NV slots polled by NV lanes.
//   MODE 1: packed: the NV values of CTA c sit in one 64-byte mailbox; reducer warp q polls all NV
//           messages of CTAs 32q+lane (5 polling warps, NV loads in flight per lane), sums them
//           lane-wise and runs the NV xor trees interleaved; one lane publishes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o allreduce_ll3 allreduce_ll3.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr unsigned kFull = 0xffffffffu;
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <int NV>
__device__ __forceinline__ void warp_sum_n(double (&t)[NV]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double o[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) o[k] = __shfl_xor_sync(kFull, t[k], off);
#pragma unroll
    for (int k = 0; k < NV; ++k) t[k] = add_rn(t[k], o[k]);
  }
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
__device__ __forceinline__ double ll_wait(const unsigned long long* src, unsigned call) {
  double v;
  while (!ll_try(src, call, v)) {}
  return v;
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

struct Sh {
  double red[3 * 32];
  double xs[3][5][32];
  double bc[4];
};

template <int NV, int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* board, int iters, double* out) {
  __shared__ Sh sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nb = gridDim.x, nthr = blockDim.x;
  unsigned long long* pub = board + 2 * 4 * (long long)nb;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = threadIdx.x * 1e-3 + blockIdx.x + k;
  unsigned call = 0;
  for (int it = 0; it < iters; ++it) {
    ++call;
    if (blockIdx.x != 0) {
      if (warp != 0) {
        double t[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) t[k] = acc[k];
        warp_sum_n<NV>(t);
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < NV; ++k) sh.red[k * 32 + warp] = t[k];
        }
        bar_arrive(1, nthr);
        bar_sync(3, nthr);
        bar_sync(2, nthr);
      } else {
        bar_sync(1, nthr);
        const int nw = nthr >> 5;
        double t[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) t[k] = lane >= 1 && lane < nw ? sh.red[k * 32 + lane] : 0.0;
        warp_sum_n<NV>(t);
#pragma unroll
        for (int k = 0; k < NV; ++k)
          if (lane == k) {
            if (MODE == 0) ll_store(board + 2 * ((long long)k * nb + blockIdx.x), t[k], call);
            else ll_store(board + 2 * (4 * (long long)blockIdx.x + k), t[k], call);
          }
        bar_arrive(3, nthr);
        if (lane < NV) sh.bc[lane] = ll_wait(pub + 2 * lane, call);
        bar_arrive(2, nthr);
      }
    } else {
      if (MODE == 0) {
        if (warp < 5 * NV) {
          const int kk = warp / 5, q = warp % 5, c = lane + 32 * q;
          sh.xs[kk][q][lane] = c >= 1 && c < nb ? ll_wait(board + 2 * ((long long)kk * nb + c), call) : 0.0;
        }
        __syncthreads();
        if (warp < NV) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < 5; ++q)
            if (lane + 32 * q < nb) s = add_rn(s, sh.xs[warp][q][lane]);
          double t[1] = {s};
          warp_sum_n<1>(t);
          if (lane == 0) {
            ll_store(pub + 2 * warp, t[0], call);
            sh.bc[warp] = t[0];
          }
        }
      } else {
        if (warp < 5) {
          const int c = lane + 32 * warp;
          double x[NV];
#pragma unroll
          for (int kk = 0; kk < NV; ++kk) x[kk] = 0.0;
          if (c >= 1 && c < nb) {
            unsigned need = (1u << NV) - 1;
            while (need) {
#pragma unroll
              for (int kk = 0; kk < NV; ++kk)
                if (need & (1u << kk)) {
                  double v;
                  if (ll_try(board + 2 * (4 * (long long)c + kk), call, v)) {
                    x[kk] = v;
                    need &= ~(1u << kk);
                  }
                }
            }
          }
#pragma unroll
          for (int kk = 0; kk < NV; ++kk) sh.xs[kk][warp][lane] = x[kk];
          asm volatile("bar.sync 4, 160;" ::: "memory");
        }
        if (warp == 0) {
          double t[NV];
#pragma unroll
          for (int kk = 0; kk < NV; ++kk) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < 5; ++q)
              if (lane + 32 * q < nb) s = add_rn(s, sh.xs[kk][q][lane]);
            t[kk] = s;
          }
          warp_sum_n<NV>(t);
#pragma unroll
          for (int kk = 0; kk < NV; ++kk)
            if (lane == kk) {
              ll_store(pub + 2 * kk, t[kk], call);
              sh.bc[kk] = t[kk];
            }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = add_rn(acc[k], sh.bc[k] * 1e-30);
  }
  if (threadIdx.x == 40 && blockIdx.x == 1) out[0] = acc[0] + acc[NV - 1];
}

template <int NV, int MODE>
void run(int nb, unsigned long long* board, double* out) {
  const int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(board, 0, 64 * 1024);
    void* args[] = {&board, (void*)&iters, &out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k<NV, MODE>, nb, 512, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double h = 0;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    if (rep)
      printf("nb %3d NV %d mode %d: %.3f us per all-reduce (%s) check %.17g\n", nb, NV, MODE, ms * 1e3 / iters,
             cudaGetErrorString(e), h);
    fflush(stdout);
  }
}

int main() {
  double* out;
  unsigned long long* board;
  cudaMalloc(&board, 64 * 1024);
  cudaMalloc(&out, 64);
  run<1, 0>(148, board, out);
  run<3, 0>(148, board, out);
  run<1, 1>(148, board, out);
  run<3, 1>(148, board, out);
  run<2, 1>(148, board, out);
  return 0;
}
