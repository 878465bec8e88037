// policy.cu — K2: policy compaction (gather_policy_matrix / gather_policy_cost,
// sparse.py:243-269).
//
// Row s of P_pi is row s*m + pi[s] of the row-stacked matrix.  For uniform
// row length K the output row pointer is s*K and one fused copy kernel moves
// the rows (+ g_pi).  Otherwise a three-kernel reduce-then-scan over the
// selected row lengths builds the int64 row pointer, then the same copy
// kernel runs.  All integer work: results are exact and order-independent.
#include "handle.cuh"

namespace ipi {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t sel_len(const int64_t* rp, const int32_t* pi, int64_t s, int m) {
  const int64_t r = s * (int64_t)m + pi[s];
  return __ldg(rp + r + 1) - __ldg(rp + r);
}

// Block-wide exclusive scan of one int64 per thread; returns the block total.
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* excl, int64_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int64_t t = __shfl_up_sync(kFull, inc, off);
    if (lane >= off) inc += t;
  }
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int w = 0; w < nw; ++w) {
      int64_t t = sh[w];
      sh[w] = run;
      run += t;
    }
    sh[nw] = run;
  }
  __syncthreads();
  *excl = inc - v + sh[warp];
  const int64_t total = sh[nw];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kScanThreads) scan_partials(const int64_t* rp, const int32_t* pi,
                                                              int64_t n, int m, int64_t* part) {
  __shared__ int64_t sh[kScanThreads / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t t = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) t += sel_len(rp, pi, base + i, m);
  int64_t excl;
  const int64_t total = block_excl_scan(t, &excl, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = total;
}

// single block: in-place exclusive scan of part[0..nb), part[nb] = total
__global__ void __launch_bounds__(kScanThreads) scan_top(int64_t* part, int64_t nb) {
  __shared__ int64_t sh[kScanThreads / 32 + 1];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nb ? part[i] : 0;
    int64_t excl;
    const int64_t total = block_excl_scan(v, &excl, sh);
    if (i < nb) part[i] = carry + excl;
    carry += total;
  }
  if (threadIdx.x == 0) part[nb] = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_final(const int64_t* rp, const int32_t* pi,
                                                           int64_t n, int m, const int64_t* part,
                                                           int64_t nb, int64_t* rp_pi) {
  __shared__ int64_t sh[kScanThreads / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t len[kScanItems];
  int64_t t = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    len[i] = base + i < n ? sel_len(rp, pi, base + i, m) : 0;
    t += len[i];
  }
  int64_t excl;
  block_excl_scan(t, &excl, sh);
  int64_t run = part[blockIdx.x] + excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) rp_pi[base + i] = run;
    run += len[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) rp_pi[n] = part[nb];
}

__global__ void uniform_rowptr(int64_t* rp_pi, int64_t n, int64_t K) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    rp_pi[i] = i * K;
}

// G lanes per state copy the selected row; lane 0 also writes g_pi.
template <int G>
__global__ void __launch_bounds__(256) copy_rows(const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ cost,
                                                  const int32_t* __restrict__ pi, int64_t n, int m,
                                                  const int64_t* __restrict__ rp_pi,
                                                  int32_t* __restrict__ col_pi,
                                                  double* __restrict__ val_pi,
                                                  double* __restrict__ g_pi) {
  constexpr int GPW = 32 / G;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwt = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = wg * GPW + grp; s - grp < n; s += nwt * GPW) {
    if (s >= n) continue;
    const int64_t r = s * (int64_t)m + __ldg(pi + s);
    const int64_t p0 = __ldg(rp + r), p1 = __ldg(rp + r + 1);
    const int64_t d0 = __ldg(rp_pi + s);
    for (int64_t p = gl; p < p1 - p0; p += G) {
      col_pi[d0 + p] = ld_stream(col + p0 + p, pol);
      val_pi[d0 + p] = ld_stream(val + p0 + p, pol);
    }
    if (g_pi && gl == 0) g_pi[s] = __ldg(cost + r);
  }
}

// Uniform rows (length K = 4*G, 16-byte aligned arrays; C2/C5 K = 64, C3
// K = 4): the selected row of state s starts at (s*m + pi[s])*K, so no row
// pointers are read (for C3's 48-byte rows the random row-pointer pairs were
// most of the DRAM traffic), and each lane moves 4 entries with 16-byte loads
// and stores; P_pi rows land at s*K.
template <int G>
__global__ void __launch_bounds__(256) copy_rows_uniform(const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ cost,
                                                         const int32_t* __restrict__ pi, int64_t n,
                                                         int m, int32_t* __restrict__ col_pi,
                                                         double* __restrict__ val_pi,
                                                         double* __restrict__ g_pi) {
  constexpr int K = 4 * G, GPW = 32 / G;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwt = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s0 = wg * GPW; s0 < n; s0 += nwt * GPW) {
    const int64_t s = s0 + grp;
    if (s >= n) continue;
    const int64_t r = s * (int64_t)m + __ldg(pi + s);
    const int64_t src = r * K + 4 * gl, dst = s * K + 4 * gl;
    const double2 v0 = ld_stream_v2(val + src, pol), v1 = ld_stream_v2(val + src + 2, pol);
    const int2 c0 = ld_stream_v2(col + src, pol), c1 = ld_stream_v2(col + src + 2, pol);
    reinterpret_cast<double2*>(val_pi + dst)[0] = v0;
    reinterpret_cast<double2*>(val_pi + dst)[1] = v1;
    reinterpret_cast<int4*>(col_pi + dst)[0] = make_int4(c0.x, c0.y, c1.x, c1.y);
    if (g_pi && gl == 0) g_pi[s] = __ldg(cost + r);
  }
}

// warp per row of P_pi: the lane holding column s supplies the diagonal entry;
// absent diagonal -> 0 -> inv_diag = 1 (CsrMatrix.diagonal, sparse.py:102-109)
__global__ void jacobi_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double* __restrict__ val, int64_t n, double gamma,
                              double* __restrict__ invd, int64_t state0) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = wg; s < n; s += nw) {
    double d = 0.0;
    int found = 0;
    for (int64_t p = rp[s] + lane; p < rp[s + 1]; p += 32)
      if (col[p] == (int)(s + state0)) {  // row s of a row block is state state0 + s
        d = val[p];
        found = 1;
      }
    const unsigned who = __ballot_sync(kFull, found);
    const double dd = __shfl_sync(kFull, d, who ? __ffs(who) - 1 : 0);
    if (lane == 0) invd[s] = 1.0 / sub_rn(1.0, mul_rn(gamma, who ? dd : 0.0));
  }
}

int jacobi_inv_diag(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                    double gamma, double* inv_diag, cudaStream_t st, int64_t state0) {
  if (n <= 0) return IPI_OK;
  int64_t blocks = (n + 7) / 8;
  if (blocks > 148 * 32) blocks = 148 * 32;
  jacobi_kernel<<<(int)blocks, 256, 0, st>>>(rp_pi, col_pi, val_pi, n, gamma, inv_diag, state0);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

static int ensure_scan_tmp(ipi_mdp* h, int64_t nb) {
  if (h->scan_tmp_len >= nb + 1) return IPI_OK;
  if (h->scan_tmp) cudaFree(h->scan_tmp);
  h->scan_tmp = nullptr;
  IPI_CUDA_TRY(cudaMalloc(&h->scan_tmp, sizeof(int64_t) * (nb + 1)));
  h->scan_tmp_len = nb + 1;
  return IPI_OK;
}

// rp_pi may be null (count only); nnz_out (host) may be null (no sync).
static int build_rowptr(ipi_mdp* h, const int32_t* policy, int64_t* rp_pi, int64_t* nnz_out,
                        cudaStream_t st) {
  const int64_t n = h->n_local;
  if (h->plan.uniform_rows) {
    const int64_t K = h->plan.row_len_max;
    if (rp_pi) {
      int64_t blocks = (n + 1 + 255) / 256;
      if (blocks > 4096) blocks = 4096;
      uniform_rowptr<<<(int)blocks, 256, 0, st>>>(rp_pi, n, K);
      IPI_LAUNCH_CHECK();
    }
    if (nnz_out) *nnz_out = n * K;
    return IPI_OK;
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  int rc = ensure_scan_tmp(h, nb);
  if (rc) return rc;
  if (nb > 0) {
    scan_partials<<<(int)nb, kScanThreads, 0, st>>>(h->rp, policy, n, h->m, h->scan_tmp);
    IPI_LAUNCH_CHECK();
  }
  scan_top<<<1, kScanThreads, 0, st>>>(h->scan_tmp, nb);
  IPI_LAUNCH_CHECK();
  if (rp_pi) {
    if (nb > 0) {
      scan_final<<<(int)nb, kScanThreads, 0, st>>>(h->rp, policy, n, h->m, h->scan_tmp, nb, rp_pi);
    } else {
      cudaMemsetAsync(rp_pi, 0, sizeof(int64_t), st);
    }
    IPI_LAUNCH_CHECK();
  }
  if (nnz_out) {
    int64_t* hp = reinterpret_cast<int64_t*>(h->host_pinned);
    IPI_CUDA_TRY(cudaMemcpyAsync(hp, h->scan_tmp + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IPI_CUDA_TRY(cudaStreamSynchronize(st));
    *nnz_out = *hp;
  }
  return IPI_OK;
}

int policy_nnz(ipi_mdp* h, const int32_t* policy, int64_t* nnz_out, cudaStream_t st) {
  return build_rowptr(h, policy, nullptr, nnz_out, st);
}

int gather_policy(ipi_mdp* h, const int32_t* policy, const int32_t* /*len_pi*/, int64_t* rp_pi,
                  int32_t* col_pi, double* val_pi, double* g_pi, int64_t* nnz_out,
                  cudaStream_t st) {
  int rc = build_rowptr(h, policy, rp_pi, nnz_out, st);
  if (rc) return rc;
  const int64_t n = h->n_local;
  if (n == 0) return IPI_OK;
  const int K = h->plan.row_len_max;
  if (h->plan.uniform_rows && K % 4 == 0 && K >= 4 && K <= 128 && ((K / 4) & (K / 4 - 1)) == 0 &&
      (uintptr_t)h->val % 16 == 0 && (uintptr_t)h->col % 16 == 0 && (uintptr_t)val_pi % 16 == 0 &&
      (uintptr_t)col_pi % 16 == 0) {
    const int Gu = K / 4, GPWu = 32 / Gu;
    int64_t ub = ((n + GPWu - 1) / GPWu + 7) / 8;
    if (ub > (int64_t)h->num_sms * 32) ub = (int64_t)h->num_sms * 32;
    if (ub < 1) ub = 1;
#define IPI_UCOPY(GG)                                                                            \
  copy_rows_uniform<GG><<<(int)ub, 256, 0, st>>>(h->col, h->val, h->cost, policy, n, h->m, col_pi, \
                                                 val_pi, g_pi)
    switch (Gu) {
      case 1: IPI_UCOPY(1); break;
      case 2: IPI_UCOPY(2); break;
      case 4: IPI_UCOPY(4); break;
      case 8: IPI_UCOPY(8); break;
      case 16: IPI_UCOPY(16); break;
      default: IPI_UCOPY(32); break;
    }
#undef IPI_UCOPY
    IPI_LAUNCH_CHECK();
    return IPI_OK;
  }
  const int G = h->plan.lanes_per_row;
  const int GPW = 32 / G;
  int64_t blocks = ((n + GPW - 1) / GPW + 7) / 8;
  if (blocks > (int64_t)h->num_sms * 32) blocks = (int64_t)h->num_sms * 32;
  if (blocks < 1) blocks = 1;
#define IPI_COPY(GG)                                                                        \
  copy_rows<GG><<<(int)blocks, 256, 0, st>>>(h->rp, h->col, h->val, h->cost, policy, n, h->m, \
                                             rp_pi, col_pi, val_pi, g_pi)
  switch (G) {
    case 1: IPI_COPY(1); break;
    case 2: IPI_COPY(2); break;
    case 4: IPI_COPY(4); break;
    case 8: IPI_COPY(8); break;
    case 16: IPI_COPY(16); break;
    default: IPI_COPY(32); break;
  }
#undef IPI_COPY
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
