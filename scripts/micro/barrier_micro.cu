// Micro-benchmark: cost of one deterministic grid all-reduce in a persistent
// cooperative kernel (148 CTAs x 1024 threads), three implementations:
//   0: cooperative-groups grid.sync() between partial write and ordered read (K4 today)
//   1: hand-rolled barrier: one release atomic per CTA + acquire spin, ordered read
//   3: LL-style flagged partials: each CTA stores (partial halves | epoch) as
//      8-byte words; readers poll the words of all CTAs (no atomics, no counter).
//   2: last-arriver reduce: the last CTA to arrive sums the partials in order and
//      publishes (value, epoch); the others spin on the epoch word.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_micro barrier_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(~0u, v, o));
  return v;
}
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

template <int MODE>
__global__ void __launch_bounds__(1024) k(double* partials, unsigned* ctr, double* pub, int iters, double* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  __shared__ double bc;
  const int nb = gridDim.x;
  double acc = threadIdx.x * 1e-3 + blockIdx.x;
  unsigned epoch = 0;
  for (int it = 0; it < iters; ++it) {
    double t = block_sum(acc, red);
    if (MODE == 0) {
      if (threadIdx.x == 0) partials[(it & 1) * nb + blockIdx.x] = t;
      grid.sync();
      if (threadIdx.x < 32) {
        double s = 0;
        for (int i = threadIdx.x; i < nb; i += 32) s = __dadd_rn(s, partials[(it & 1) * nb + i]);
        s = warp_sum(s);
        if (threadIdx.x == 0) bc = s;
      }
    } else if (MODE == 1) {
      ++epoch;
      if (threadIdx.x == 0) {
        partials[(it & 1) * nb + blockIdx.x] = t;
        red_release(ctr, 1u);
        while (ld_acquire(ctr) < epoch * nb) {}
      }
      __syncwarp();
      if (threadIdx.x < 32) {
        double s = 0;
        for (int i = threadIdx.x; i < nb; i += 32) s = __dadd_rn(s, __ldcg(partials + (it & 1) * nb + i));
        s = warp_sum(s);
        if (threadIdx.x == 0) bc = s;
      }
    } else if (MODE == 3) {
      ++epoch;
      unsigned long long* slots = reinterpret_cast<unsigned long long*>(partials + 4 * nb);
      if (threadIdx.x == 0) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(t);
        const unsigned long long w0 = (bits & 0xffffffffull) | ((unsigned long long)epoch << 32);
        const unsigned long long w1 = (bits >> 32) | ((unsigned long long)epoch << 32);
        unsigned long long* dst = slots + ((epoch & 1) * nb + blockIdx.x) * 2;
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(w0), "l"(w1) : "memory");
      }
      if (threadIdx.x < 32) {
        double s = 0;
        for (int i = threadIdx.x; i < nb; i += 32) {
          const unsigned long long* src = slots + ((epoch & 1) * nb + i) * 2;
          unsigned long long w0, w1;
          do {
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(src) : "memory");
          } while ((unsigned)(w0 >> 32) != epoch || (unsigned)(w1 >> 32) != epoch);
          s = __dadd_rn(s, __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32))));
        }
        s = warp_sum(s);
        if (threadIdx.x == 0) bc = s;
      }
    } else if (MODE == 4) {
      // arrivals spread over 8 counters (one 128-byte line each) so the 148
      // release adds do not serialise on one L2 address; the leader polls all
      // 8 with relaxed loads (one round trip per poll) and then fences.
      ++epoch;
      if (threadIdx.x == 0) {
        partials[(it & 1) * nb + blockIdx.x] = t;
        red_release(ctr + 64 + (blockIdx.x & 7) * 32, 1u);
      }
      if (threadIdx.x < 8) {
        const unsigned per = (unsigned)((nb - threadIdx.x + 7) / 8);
        unsigned v;
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + 64 + threadIdx.x * 32) : "memory");
        } while (v < epoch * per);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncwarp();
      if (threadIdx.x < 32) {
        double s = 0;
        for (int i = threadIdx.x; i < nb; i += 32) s = __dadd_rn(s, __ldcg(partials + (it & 1) * nb + i));
        s = warp_sum(s);
        if (threadIdx.x == 0) bc = s;
      }
    } else {
      ++epoch;
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) partials[(it & 1) * nb + blockIdx.x] = t;
        unsigned old = 0;
        if (threadIdx.x == 0) old = atom_add_acqrel(ctr, 1u);
        old = __shfl_sync(~0u, old, 0);
        if (old == epoch * nb - 1) {  // last arriver: ordered sum, publish
          double s = 0;
          for (int i = threadIdx.x; i < nb; i += 32) s = __dadd_rn(s, __ldcg(partials + (it & 1) * nb + i));
          s = warp_sum(s);
          if (threadIdx.x == 0) {
            pub[(it & 1) * 2] = s;
            __threadfence();
            red_release(ctr + 32, 1u);
          }
          if (threadIdx.x == 0) bc = s;
        } else if (threadIdx.x == 0) {
          while (ld_acquire(ctr + 32) < epoch) {}
          bc = __ldcg(pub + (it & 1) * 2);
        }
      }
    }
    __syncthreads();
    acc = __dadd_rn(acc, bc * 1e-30);
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[MODE] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *partials, *pub, *out;
  unsigned* ctr;
  cudaMalloc(&partials, 16 * sms * sizeof(double));
  cudaMalloc(&pub, 64);
  cudaMalloc(&out, 64);
  cudaMalloc(&ctr, 4096);
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode)
  for (int threads = 1024; threads >= 128; threads /= 2) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 4096);
      cudaMemset(partials, 0, 16 * sms * sizeof(double));
      void* args[] = {&partials, &ctr, &pub, (void*)&iters, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      const void* fn = mode == 0 ? (const void*)k<0> : mode == 1 ? (const void*)k<1> : mode == 2 ? (const void*)k<2> : mode == 3 ? (const void*)k<3> : (const void*)k<4>;
      cudaError_t e = cudaLaunchCooperativeKernel(fn, sms, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("mode %d threads %4d: %.3f us per all-reduce (%s)\n", mode, threads, ms * 1e3 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
