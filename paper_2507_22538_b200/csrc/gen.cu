// gen.cu — device builders for the BASELINE configs (C2/C5 locality random,
// C3 pendulum, C4 SIS).  Recipes are documented in generators.py and
// DESIGN.md (Appendix-B decisions); generated arrays feed both the GPU path and
// (after a D2H copy) the CPU oracle, so parity never depends on two
// generators agreeing.  Compiled with --fmad=false so the float formulas match
// the host restatement operation-for-operation.
#include <algorithm>

#include "handle.cuh"

namespace ipi {

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11)
// ---------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double u53_open0(uint32_t x0, uint32_t x1) {
  const uint64_t bits = ((uint64_t)x1 << 21) | (x0 >> 11);
  return ((double)bits + 1.0) * 0x1.0p-53;
}
__device__ __forceinline__ double u53_closed0(uint32_t x0, uint32_t x1) {
  const uint64_t bits = ((uint64_t)x1 << 21) | (x0 >> 11);
  return (double)bits * 0x1.0p-53;
}

constexpr uint32_t kTagCand = 0xC2C5u, kTagWeight = 0xD1D1u, kTagCost = 0xC057u;
constexpr uint32_t kLocalProb = 3865470566u;  // floor(0.9 * 2^32)
constexpr int kMaxK = 128;
constexpr int kGenWarps = 8;

// warp per (s, a) row
__global__ void __launch_bounds__(kGenWarps * 32) gen_locality_kernel(
    int64_t n, int m, int K, int64_t W, uint64_t seed, int64_t state0, int64_t n_states,
    int64_t* row_ptr, int32_t* col, double* val, double* cost) {
  __shared__ int32_t chosen[kGenWarps][kMaxK];
  __shared__ int32_t sorted_[kGenWarps][kMaxK];
  __shared__ double ew[kGenWarps][kMaxK];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t rows = n_states * (int64_t)m;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t lr = (int64_t)blockIdx.x * kGenWarps + wid; lr < rows;
       lr += (int64_t)gridDim.x * kGenWarps) {
    const int64_t s = state0 + lr / m;
    const int64_t r = s * m + lr % m;  // global row
    const uint32_t r_lo = (uint32_t)r, r_hi = (uint32_t)(r >> 32);
    const int64_t lo = s - W < 0 ? 0 : s - W;
    const int64_t hi = s + W > n - 1 ? n - 1 : s + W;
    const uint64_t span = (uint64_t)(hi - lo + 1);
    int count = 0;
    for (uint32_t t0 = 0; count < K; t0 += 32) {
      const U4 o = philox(U4{t0 + lane, r_lo, r_hi, kTagCand}, k0, k1);
      const uint64_t pos = ((uint64_t)o.z << 32) | o.y;
      const int c = o.x < kLocalProb ? (int)(lo + (int64_t)__umul64hi(pos, span))
                                     : (int)__umul64hi(pos, (uint64_t)n);
      bool fresh = true;
      for (int j = 0; j < count; ++j) fresh &= chosen[wid][j] != c;
      for (int j = 0; j < 32; ++j) {
        const int cj = __shfl_sync(kFull, c, j);
        fresh &= !(j < lane && cj == c);
      }
      const unsigned bal = __ballot_sync(kFull, fresh);
      const int pos_in = count + __popc(bal & ((1u << lane) - 1u));
      if (fresh && pos_in < K) chosen[wid][pos_in] = c;
      count += __popc(bal);
      if (count > K) count = K;
      __syncwarp();
    }
    // rank sort of K distinct values
    for (int i = lane; i < K; i += 32) {
      const int v = chosen[wid][i];
      int rank = 0;
      for (int j = 0; j < K; ++j) rank += chosen[wid][j] < v;
      sorted_[wid][rank] = v;
    }
    for (int i = lane; i < K; i += 32) {
      const U4 o = philox(U4{(uint32_t)i, r_lo, r_hi, kTagWeight}, k0, k1);
      ew[wid][i] = -log(u53_open0(o.x, o.y));
    }
    __syncwarp();
    double total = 0.0;
    for (int i = 0; i < K; ++i) total += ew[wid][i];  // sequential, like the host recipe
    const int64_t base = lr * (int64_t)K;
    for (int i = lane; i < K; i += 32) {
      col[base + i] = sorted_[wid][i];
      val[base + i] = ew[wid][i] / total;
    }
    if (lane == 0) {
      const U4 o = philox(U4{0u, r_lo, r_hi, kTagCost}, k0, k1);
      cost[lr] = u53_closed0(o.x, o.y);
      row_ptr[lr] = base;
      if (lr == rows - 1) row_ptr[rows] = rows * (int64_t)K;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// C3 pendulum: thread per (s, a) row
// ---------------------------------------------------------------------------
__global__ void gen_pendulum_kernel(int N, int na, int64_t state0, int64_t n_states,
                                    int64_t* row_ptr, int32_t* col, double* val, double* cost) {
  const double PI = 3.141592653589793;
  const double h_t = 2.0 * PI / N;
  const double h_o = 2.0 * 10.0 / (N - 1);
  const int64_t rows = n_states * (int64_t)na;
  for (int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lr < rows;
       lr += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = state0 + lr / na;
    const int a = (int)(lr % na);
    const int64_t it = s / N, jo = s % N;
    const double theta = -PI + (double)it * h_t;
    const double omega = -10.0 + (double)jo * h_o;
    const double u = na == 1 ? 0.0 : -3.0 + (double)a * (2.0 * 3.0 / (na - 1));
    cost[lr] = (theta * theta + 0.1 * (omega * omega)) + 0.01 * (u * u);
    const double om_next = omega + 0.01 * (9.81 * sin(theta) + u);
    const double th_next = theta + 0.01 * om_next;
    const double fa_ = (th_next + PI) / h_t;
    const double fa = floor(fa_);
    const double ft = fa_ - fa;
    const long long fi = (long long)fa;
    const int64_t i0 = ((fi % N) + N) % N;
    const int64_t i1 = (i0 + 1) % N;
    double oc = om_next < -10.0 ? -10.0 : (om_next > 10.0 ? 10.0 : om_next);
    const double t = (oc + 10.0) / h_o;
    long long j0 = (long long)floor(t);
    j0 = j0 < 0 ? 0 : (j0 > N - 2 ? N - 2 : j0);
    const double fo = t - (double)j0;
    const int64_t j1 = j0 + 1;
    int64_t c[4] = {i0 * N + j0, i0 * N + j1, i1 * N + j0, i1 * N + j1};
    double w[4] = {(1.0 - ft) * (1.0 - fo), (1.0 - ft) * fo, ft * (1.0 - fo), ft * fo};
    if (i1 < i0) {  // wrap: the i1 block sorts first
      int64_t tc0 = c[0], tc1 = c[1];
      double tw0 = w[0], tw1 = w[1];
      c[0] = c[2]; c[1] = c[3]; c[2] = tc0; c[3] = tc1;
      w[0] = w[2]; w[1] = w[3]; w[2] = tw0; w[3] = tw1;
    }
    const int64_t base = lr * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      col[base + k] = (int32_t)c[k];
      val[base + k] = w[k];
    }
    row_ptr[lr] = base;
    if (lr == rows - 1) row_ptr[rows] = rows * 4;
  }
}

// ---------------------------------------------------------------------------
// C4 SIS: block per (s, a) row; exact convolution of two binomial pmfs.
// ---------------------------------------------------------------------------
__constant__ double c_betas[5] = {0.5, 0.35, 0.25, 0.15, 0.05};
__constant__ double c_weights[5] = {0.0, 0.2, 0.5, 1.0, 2.0};
constexpr int kSisThreads = 256;
constexpr int kSisMaxSupport = 2048;  // per pmf (support with pmf >= 1e-32)
constexpr int kSisSmem = 4 * kSisMaxSupport * 8;  // px, py, conv (2x)
constexpr double kSisRecovery = 0.1;
constexpr double kSisTrunc = 1e-14;
constexpr double kLogFloor = -73.68;  // log(1e-32)

__global__ void lfact_kernel(int N, double* lf) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= N; k += gridDim.x * blockDim.x)
    lf[k] = lgamma((double)k + 1.0);
}

__device__ __forceinline__ double binom_logpmf(const double* lf, int nn, int k, double lp, double l1p) {
  return lf[nn] - lf[k] - lf[nn - k] + (double)k * lp + (double)(nn - k) * l1p;
}

// Support [lo, hi] of Bin(nn, p) restricted to pmf >= 1e-32 (unimodal).
__device__ void binom_support(const double* lf, int nn, double p, int* lo_out, int* hi_out,
                              int* red_lo, int* red_hi) {
  if (p <= 0.0 || nn == 0) {
    *lo_out = 0;
    *hi_out = 0;
    return;
  }
  if (p >= 1.0) {
    *lo_out = nn;
    *hi_out = nn;
    return;
  }
  const double lp = log(p), l1p = log1p(-p);
  int lo = nn + 1, hi = -1;
  for (int k = threadIdx.x; k <= nn; k += blockDim.x) {
    if (binom_logpmf(lf, nn, k, lp, l1p) >= kLogFloor) {
      lo = min(lo, k);
      hi = max(hi, k);
    }
  }
  if (threadIdx.x == 0) {
    *red_lo = nn + 1;
    *red_hi = -1;
  }
  __syncthreads();
  atomicMin(red_lo, lo);
  atomicMax(red_hi, hi);
  __syncthreads();
  *lo_out = *red_lo;
  *hi_out = *red_hi;
  __syncthreads();
}

__global__ void __launch_bounds__(kSisThreads) gen_sis_kernel(int N, const double* lf, int pass,
                                                               int64_t* row_ptr, int32_t* col,
                                                               double* val, double* cost,
                                                               int* overflow) {
  extern __shared__ double sis_smem[];
  double* px = sis_smem;
  double* py = px + kSisMaxSupport;
  double* conv = py + kSisMaxSupport;
  __shared__ int red[2];
  __shared__ int cnt_sh;
  __shared__ double tot_sh;
  const int m = 5;
  const int64_t rows = (int64_t)(N + 1) * m;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int s = (int)(r / m), a = (int)(r % m);
    const double q = -expm1(-(c_betas[a] * (double)s) / (double)N);
    int xlo, xhi, ylo, yhi;
    binom_support(lf, s, kSisRecovery, &xlo, &xhi, &red[0], &red[1]);
    binom_support(lf, N - s, q, &ylo, &yhi, &red[0], &red[1]);
    const int nx = xhi - xlo + 1, ny = yhi - ylo + 1;
    if (nx > kSisMaxSupport || ny > kSisMaxSupport) {
      if (threadIdx.x == 0) atomicAdd(overflow, 1);
      continue;
    }
    {
      const double lp = log(kSisRecovery), l1p = log1p(-kSisRecovery);
      for (int i = threadIdx.x; i < nx; i += blockDim.x)
        px[i] = s == 0 ? 1.0 : exp(binom_logpmf(lf, s, xlo + i, lp, l1p));
      const bool deg = q <= 0.0 || N - s == 0;
      const double lq = deg ? 0.0 : log(q), l1q = deg ? 0.0 : log1p(-q);
      for (int i = threadIdx.x; i < ny; i += blockDim.x)
        py[i] = deg ? 1.0 : exp(binom_logpmf(lf, N - s, ylo + i, lq, l1q));
    }
    __syncthreads();
    // s' = s - x + y ranges over [s - xhi + ylo, s - xlo + yhi]
    const int k_lo = s - xhi + ylo, k_hi = s - xlo + yhi;
    const int nk = k_hi - k_lo + 1;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
      const int k = k_lo + i;
      double acc = 0.0;
      // y = k - s + x  in [ylo, yhi]
      int x0 = max(xlo, ylo + s - k), x1 = min(xhi, yhi + s - k);
      for (int x = x0; x <= x1; ++x) acc += px[x - xlo] * py[k - s + x - ylo];
      conv[i] = acc;
    }
    if (threadIdx.x == 0) {
      cnt_sh = 0;
      tot_sh = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int c = 0;
      double t = 0.0;
      for (int i = 0; i < nk; ++i)
        if (conv[i] >= kSisTrunc) {
          ++c;
          t += conv[i];
        }
      cnt_sh = c;
      tot_sh = t;
    }
    __syncthreads();
    if (pass == 1) {
      if (threadIdx.x == 0) row_ptr[r + 1] = cnt_sh;
    } else {
      if (threadIdx.x == 0) {
        int64_t o = row_ptr[r];
        for (int i = 0; i < nk; ++i)
          if (conv[i] >= kSisTrunc) {
            col[o] = k_lo + i;
            val[o] = conv[i] / tot_sh;
            ++o;
          }
        cost[r] = (double)s / (double)N + c_weights[a];
      }
    }
    __syncthreads();
  }
}

}  // namespace ipi

using namespace ipi;

extern "C" {

int ipi_gen_locality(int64_t n, int32_t m, int32_t K, int64_t window, uint64_t seed, int64_t state0,
                     int64_t n_states, int64_t* row_ptr, int32_t* col, double* val, double* cost,
                     void* stream) {
  if (K < 1 || K > kMaxK || K > n) return fail(IPI_EVALIDATION, "K must lie in [1, min(n, 128)]");
  if (state0 < 0 || state0 + n_states > n) return fail(IPI_EDIMENSION, "state range outside [0, n)");
  if (n_states == 0) return IPI_OK;
  const int64_t rows = n_states * m;
  int64_t blocks = (rows + kGenWarps - 1) / kGenWarps;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_locality_kernel<<<(int)blocks, kGenWarps * 32, 0, (cudaStream_t)stream>>>(
      n, m, K, window, seed, state0, n_states, row_ptr, col, val, cost);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

int ipi_gen_pendulum(int32_t N, int32_t n_actions, int64_t state0, int64_t n_states,
                     int64_t* row_ptr, int32_t* col, double* val, double* cost, void* stream) {
  if (N < 2 || n_actions < 1) return fail(IPI_EVALIDATION, "grid needs N >= 2 and >= 1 action");
  const int64_t rows = n_states * n_actions;
  if (rows == 0) return IPI_OK;
  int64_t blocks = (rows + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_pendulum_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(N, n_actions, state0, n_states,
                                                                      row_ptr, col, val, cost);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

int ipi_gen_sis(int32_t population, int32_t pass, int64_t* row_ptr, int32_t* col, double* val,
                double* cost, void* stream) {
  if (population < 1) return fail(IPI_EVALIDATION, "population must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  double* lf = nullptr;
  int* ovf = nullptr;
  IPI_CUDA_TRY(cudaMalloc(&lf, sizeof(double) * (population + 1)));
  IPI_CUDA_TRY(cudaMalloc(&ovf, sizeof(int)));
  cudaMemsetAsync(ovf, 0, sizeof(int), st);
  lfact_kernel<<<(population + 256) / 256, 256, 0, st>>>(population, lf);
  const int64_t rows = (int64_t)(population + 1) * 5;
  const int blocks = (int)std::min<int64_t>(rows, 148 * 8);
  IPI_CUDA_TRY(cudaFuncSetAttribute(gen_sis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSisSmem));
  gen_sis_kernel<<<blocks, kSisThreads, kSisSmem, st>>>(population, lf, pass, row_ptr, col, val, cost, ovf);
  int hovf = 0;
  cudaMemcpyAsync(&hovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(lf);
  cudaFree(ovf);
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("gen_sis: ") + cudaGetErrorString(e));
  if (hovf) return fail(IPI_ERESOURCE, "SIS pmf support exceeds the kernel's shared-memory tile");
  return IPI_OK;
}

}  // extern "C"
