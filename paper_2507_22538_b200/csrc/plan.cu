// plan.cu — kernel planning for an instance (ipi_mdp_create).
//
// Stages, in order: row statistics + sampled locality histogram, the shared
// V window and the K1 grid, then the K1 variant (register-deep, uniform ring,
// generic-rows CTA autotune, flat ring).  Later stages may
// override earlier choices; each keeps the previous plan when its kernel does
// not fit.  Environment switches (IPI_K1_*, IPI_URING_*, IPI_RING_*) force
// shapes for A/B measurements.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "plan.cuh"

namespace ipi {

int k1_set_smem(int lanes, int smem);  // bellman.cu
int k1_occupancy(int lanes, int uniform_K, bool win, int smem);

// ---- planning kernels ------------------------------------------------------
__global__ void row_stats_kernel(const int64_t* rp, int64_t rows, unsigned long long* out) {
  // out[0] = min len, out[1] = max len (atomicMin/Max on u64)
  unsigned long long mn = ~0ull, mx = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long l = (unsigned long long)(rp[r + 1] - rp[r]);
    mn = l < mn ? l : mn;
    mx = l > mx ? l : mx;
  }
  for (int off = 16; off; off >>= 1) {
    unsigned long long a = __shfl_xor_sync(kFull, mn, off), b = __shfl_xor_sync(kFull, mx, off);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

// Contiguous rows: every row's columns are consecutive integers (banded
// birth-death transitions: each SIS row, C4, is the truncated convolution of
// two binomial pmfs, a log-concave pmf, so its support is an interval).  Then
// kernels read only the first column of a row (8 instead of 12 bytes per
// entry).  out[0] stays 1 unless some row breaks the rule.
__global__ void contiguous_rows_kernel(const int64_t* rp, const int32_t* col, int64_t rows,
                                       int* out) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool ok = true;
  for (int64_t r = wg; r < rows; r += nw) {
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    for (int64_t p = p0 + lane; p + 1 < p1; p += 32) ok = ok && (col[p + 1] == col[p] + 1);
  }
  if (!__all_sync(kFull, ok) && lane == 0) *out = 0;
}

// log2 histogram of |col - state| (locality profile, 40 buckets)
// Rows are sampled with a fixed stride (>= 2^17 sampled rows) so planning stays
// a few ms even at 2^31 nnz; the histogram only steers the window size.
__global__ void locality_hist_kernel(const int64_t* rp, const int32_t* col, int64_t rows, int m,
                                     int64_t state0, int64_t stride, unsigned long long* hist) {
  __shared__ unsigned long long sh[40];
  for (int i = threadIdx.x; i < 40; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t rs = wg; rs * stride < rows; rs += nw) {
    const int64_t r = rs * stride;
    const int64_t s = state0 + r / m;
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      int64_t d = (int64_t)col[p] - s;
      d = d < 0 ? -d : d;
      const int b = d == 0 ? 0 : 64 - __clzll((unsigned long long)d);  // d in [2^(b-1), 2^b)
      atomicAdd(&sh[b < 39 ? b : 39], 1ull);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 40; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// nnz-balanced state boundaries: bounds[c] = first state s with rp[s*m] >= c*nnz/nb
__global__ void bounds_kernel(const int64_t* rp, int64_t n, int m, int nb, int64_t* bounds) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nb) return;
  if (c == 0) {
    bounds[0] = 0;
    return;
  }
  if (c == nb) {
    bounds[nb] = n;
    return;
  }
  const int64_t nnz = rp[n * (int64_t)m];
  const int64_t key = (nnz * (int64_t)c) / nb;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rp[mid * (int64_t)m] < key) lo = mid + 1; else hi = mid;
  }
  bounds[c] = lo;
}


struct PlanCtx {
  ipi_mdp* h;
  cudaStream_t st;
  int64_t rows;
  unsigned long long hst[48];  // [0] min len, [1] max len, [8..47] locality histogram
};

// row statistics (min / max / mean length) and the sampled locality histogram
static int plan_row_stats(PlanCtx& c) {
  ipi_mdp* h = c.h;
  cudaStream_t st = c.st;
  ipi_plan& p = h->plan;
  [[maybe_unused]] const int64_t* row_ptr = h->rp;
  [[maybe_unused]] const int32_t* col = h->col;
  [[maybe_unused]] const double* values = h->val;
  [[maybe_unused]] const double* stage_cost = h->cost;
  [[maybe_unused]] const int64_t n_local = h->n_local, n_global = h->n_global, state0 = h->state0;
  [[maybe_unused]] const int32_t m = h->m;
  [[maybe_unused]] const int64_t rows = c.rows;
  // ---- row statistics + locality histogram --------------------------------
  unsigned long long* d_tmp = nullptr;
  if (cudaMalloc(&d_tmp, sizeof(unsigned long long) * 48) != cudaSuccess)
    return (fail(IPI_ECUDA, "cudaMalloc failed"));
  unsigned long long init[48];
  std::memset(init, 0, sizeof(init));
  init[0] = ~0ull;
  cudaMemcpyAsync(d_tmp, init, sizeof(init), cudaMemcpyHostToDevice, st);
  int64_t nnz = 0;
  if (rows > 0) {
    row_stats_kernel<<<grid_for(rows, 256, h->num_sms), 256, 0, st>>>(row_ptr, rows, d_tmp);
    const int64_t stride = std::max<int64_t>(1, rows >> 17);
    locality_hist_kernel<<<h->num_sms * 8, 256, 0, st>>>(row_ptr, col, rows, m, state0, stride,
                                                         d_tmp + 8);
  }
  unsigned long long* hst = c.hst;
  cudaMemcpyAsync(c.hst, d_tmp, sizeof(c.hst), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&nnz, row_ptr + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(d_tmp);
  if (e != cudaSuccess) return (fail(IPI_ECUDA, std::string("planning: ") + cudaGetErrorString(e)));
  p.nnz = nnz;
  p.row_len_min = rows > 0 ? (int32_t)hst[0] : 0;
  p.row_len_max = rows > 0 ? (int32_t)hst[1] : 0;
  p.row_len_mean = rows > 0 ? (double)nnz / (double)rows : 0.0;
  p.uniform_rows = rows > 0 && p.row_len_min == p.row_len_max;
  p.lanes_per_row = pick_lanes_per_row(p.row_len_mean);
  p.contiguous_rows = 0;
  if (rows > 0 && !p.uniform_rows && p.row_len_max > 1) {  // variable rows (C4): one more pass
    int* d_flag = nullptr;
    if (cudaMalloc(&d_flag, sizeof(int)) != cudaSuccess) return fail(IPI_ECUDA, "cudaMalloc failed");
    const int one = 1;
    int h_flag = 0;
    cudaMemcpyAsync(d_flag, &one, sizeof(int), cudaMemcpyHostToDevice, st);
    contiguous_rows_kernel<<<h->num_sms * 8, 256, 0, st>>>(row_ptr, col, rows, d_flag);
    cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    const cudaError_t e2 = cudaStreamSynchronize(st);
    cudaFree(d_flag);
    if (e2 != cudaSuccess) return fail(IPI_ECUDA, std::string("planning: ") + cudaGetErrorString(e2));
    static const bool allow = !(getenv("IPI_CONTIG") && getenv("IPI_CONTIG")[0] == '0');
    p.contiguous_rows = h_flag && allow;
  }
  p.k1_threads = kK1Threads;
  p.inner_threads = kInnerThreads;
  return IPI_OK;
}

// shared-memory V window (halo) from the locality profile; K1 grid and nnz-balanced bounds
static int plan_window_and_grid(PlanCtx& c) {
  ipi_mdp* h = c.h;
  cudaStream_t st = c.st;
  ipi_plan& p = h->plan;
  [[maybe_unused]] const int64_t* row_ptr = h->rp;
  [[maybe_unused]] const int32_t* col = h->col;
  [[maybe_unused]] const double* values = h->val;
  [[maybe_unused]] const double* stage_cost = h->cost;
  [[maybe_unused]] const int64_t n_local = h->n_local, n_global = h->n_global, state0 = h->state0;
  [[maybe_unused]] const int32_t m = h->m;
  [[maybe_unused]] const int64_t rows = c.rows;
  [[maybe_unused]] const int64_t nnz = p.nnz;
  // ---- shared-memory V window (halo) choice ---------------------------------
  // coverage(k) = fraction of nnz with |col - s| < 2^k.  Pick the largest k
  // whose window (own slice + 2*2^k, clipped to n_global) fits 100 KB (two
  // 512-thread CTAs per SM); use it only if it covers >= 50% of the gathers,
  // then shrink to the smallest k within 1% of that coverage.
  const int ctas_win = getenv("IPI_K1_GEN_CTAS") ? std::max(1, atoi(getenv("IPI_K1_GEN_CTAS"))) : 2;
  const int nb_win = h->num_sms * ctas_win;
  const int64_t own = (n_local + nb_win - 1) / std::max(nb_win, 1);
  const int64_t cap_doubles = 100 * 1024 / 8;
  double cum[41];
  cum[0] = 0.0;
  for (int b = 0; b < 40; ++b) cum[b + 1] = cum[b] + (double)c.hst[8 + b];
  auto coverage = [&](int k) {  // d < 2^k  <=> bucket <= k
    const int b = std::min(k, 39);
    return cum[40] > 0 ? cum[b + 1] / cum[40] : 1.0;
  };
  int kfit = -1;
  for (int k = 0; k <= 31; ++k) {
    const int64_t halo = 1ll << k;
    const int64_t wlen = std::min<int64_t>(n_global, own + 2 * halo);
    if (wlen <= cap_doubles) kfit = k;
  }
  p.halo = -1;
  if (kfit >= 0 && rows > 0) {
    const double best = coverage(kfit);
    if (best >= 0.5) {
      int k = kfit;
      while (k > 0 && coverage(k - 1) >= best - 0.01) --k;
      p.halo = (int32_t)std::min<int64_t>(1ll << k, n_global);
    }
  }
  // ---- K1 grid -------------------------------------------------------------
  int k1_blocks;
  if (p.halo >= 0) {
    k1_blocks = nb_win;
    const int64_t wlen = std::min<int64_t>(n_global, own + 2 * (int64_t)p.halo);
    p.k1_smem_bytes = (int32_t)(wlen * 8 + 1024);
    int rc = k1_set_smem(p.lanes_per_row, p.k1_smem_bytes);
    if (rc) return (rc);
  } else {
    p.k1_smem_bytes = 0;
    k1_blocks = h->num_sms * k1_occupancy(p.lanes_per_row, p.uniform_rows ? p.row_len_max : 0,
                                          false, 0);
  }
  // enough states per CTA: at least one per warp
  const int64_t max_blocks = std::max<int64_t>(1, (n_local + 15) / 16);
  k1_blocks = (int)std::min<int64_t>(k1_blocks, max_blocks);
  p.k1_blocks = k1_blocks;
  if (cudaMalloc(&h->k1_bounds, sizeof(int64_t) * (k1_blocks + 1)) != cudaSuccess)
    return (fail(IPI_ECUDA, "cudaMalloc bounds"));
  bounds_kernel<<<(k1_blocks + 1 + 127) / 128, 128, 0, st>>>(row_ptr, n_local, m, k1_blocks,
                                                            h->k1_bounds);
  if (p.halo >= 0) {
    // every K1 window must fit: check the realised nnz-balanced bounds
    std::vector<int64_t> hb(k1_blocks + 1);
    cudaMemcpyAsync(hb.data(), h->k1_bounds, sizeof(int64_t) * (k1_blocks + 1),
                    cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return (fail(IPI_ECUDA, "bounds sync"));
    int64_t worst = 0;
    for (int c = 0; c < k1_blocks; ++c) worst = std::max<int64_t>(worst, hb[c + 1] - hb[c]);
    const int64_t wlen = std::min<int64_t>(n_global, worst + 2 * (int64_t)p.halo);
    if (wlen * 8 + 1024 > 200 * 1024) {
      p.halo = -1;  // unbalanced slices: plain L1 gathers
      p.k1_smem_bytes = 0;
    } else if (wlen * 8 + 1024 > p.k1_smem_bytes) {
      p.k1_smem_bytes = (int32_t)(wlen * 8 + 1024);
      int rc = k1_set_smem(p.lanes_per_row, p.k1_smem_bytes);
      if (rc) return (rc);
    }
  }
  p.inner_blocks = 0;
  p.inner_smem_bytes = 0;
  int Gu = 0, Pu = 0;
  p.k1_variant = (p.uniform_rows && uniform_shape(p.row_len_max, &Gu, &Pu)) ? 1 : 0;
  return IPI_OK;
}

// register-deep uniform kernel (default when no V window fits, e.g. C5)
static int plan_deep(PlanCtx& c) {
  ipi_mdp* h = c.h;
  cudaStream_t st = c.st;
  ipi_plan& p = h->plan;
  [[maybe_unused]] const int64_t* row_ptr = h->rp;
  [[maybe_unused]] const int32_t* col = h->col;
  [[maybe_unused]] const double* values = h->val;
  [[maybe_unused]] const double* stage_cost = h->cost;
  [[maybe_unused]] const int64_t n_local = h->n_local, n_global = h->n_global, state0 = h->state0;
  [[maybe_unused]] const int32_t m = h->m;
  [[maybe_unused]] const int64_t rows = c.rows;
  [[maybe_unused]] const int64_t nnz = p.nnz;
  // ---- deep-pipeline uniform kernel: one 512-thread CTA per SM ---------------
  {
    // Default for uniform rows without a shared V window (C5: the +-65536 window
    // does not fit): every gather is an L2 access, and the register-deep kernel
    // beats the cp.async ring there (C5 rank proxy: 8.3 vs 11.3 ms,
    // scripts/c5_ab.sh).  IPI_K1_DEEP=1/0 forces it on/off.
    const char* env = getenv("IPI_K1_DEEP");
    const bool allow = env ? env[0] == '1' : p.halo < 0;
    if (allow && p.k1_variant == 1 && p.row_len_max > 4 && n_local > 0) {
      const int blocks = (int)std::min<int64_t>(h->num_sms, std::max<int64_t>(1, (n_local + 15) / 16));
      std::vector<int64_t> hb(blocks + 1);
      for (int c = 0; c <= blocks; ++c) hb[c] = (int64_t)((double)n_local * c / blocks);
      hb[blocks] = n_local;
      int64_t worst = 0;
      for (int c = 0; c < blocks; ++c) worst = std::max<int64_t>(worst, hb[c + 1] - hb[c]);
      int smem = 0;
      int halo = p.halo;
      if (halo >= 0) {
        const int64_t wlen = std::min<int64_t>(n_global, worst + 2 * (int64_t)halo);
        if (wlen * 8 + 1024 <= 200 * 1024) smem = (int)(wlen * 8 + 1024);
        else halo = -1;
      }
      int64_t* db = nullptr;
      if (cudaMalloc(&db, sizeof(int64_t) * (blocks + 1)) == cudaSuccess &&
          cudaMemcpy(db, hb.data(), sizeof(int64_t) * (blocks + 1), cudaMemcpyHostToDevice) ==
              cudaSuccess &&
          (smem == 0 || k1_set_smem(p.lanes_per_row, smem) == IPI_OK)) {
        cudaFree(h->k1_bounds);
        h->k1_bounds = db;
        p.k1_blocks = blocks;
        p.k1_smem_bytes = smem;
        p.halo = halo;
        p.k1_variant = 3;
      } else if (db) {
        cudaFree(db);
      }
    }
  }
  return IPI_OK;
}

// uniform rows K = 64: per-warp cp.async ring, CTA count autotuned on the instance
static int plan_uniform_ring(PlanCtx& c) {
  ipi_mdp* h = c.h;
  cudaStream_t st = c.st;
  ipi_plan& p = h->plan;
  [[maybe_unused]] const int64_t* row_ptr = h->rp;
  [[maybe_unused]] const int32_t* col = h->col;
  [[maybe_unused]] const double* values = h->val;
  [[maybe_unused]] const double* stage_cost = h->cost;
  [[maybe_unused]] const int64_t n_local = h->n_local, n_global = h->n_global, state0 = h->state0;
  [[maybe_unused]] const int32_t m = h->m;
  [[maybe_unused]] const int64_t rows = c.rows;
  [[maybe_unused]] const int64_t nnz = p.nnz;
  // ---- uniform rows, K = 64: cp.async ring per warp (bellman.cu) -------------
  // Shapes (warps, stages, waves): waves > 1 splits each SM's state range over
  // several CTAs so the V window per CTA shrinks and leaves room for the rings.
  if ((p.k1_variant == 1 || (p.k1_variant == 3 && getenv("IPI_URING_WARPS"))) && p.uniform_rows &&
      p.row_len_max == 64 && m % 4 == 0 && n_local > 0) {
    const char* env = getenv("IPI_K1_URING");
    const bool aligned = ((uintptr_t)values % 16 == 0) && ((uintptr_t)stage_cost % 16 == 0) &&
                         ((uintptr_t)col % 16 == 0);
    // (warps, stages, waves, lookahead); measured on C2 (scripts/uring_ab.sh,
    // profiles/r01_uring_shapes*.txt): 8 waves (small CTAs, even tail) with the
    // cp.async window are the most stable; 4 waves swing 0.70-0.89 across boxes
    int shapes[6][4] = {{12, 3, 8, 1}, {12, 3, 4, 1}, {10, 3, 2, 1}, {11, 3, 2, 1}, {10, 4, 2, 1}, {8, 4, 2, 1}};
    int nshape = 6;
    if (getenv("IPI_URING_WARPS") && getenv("IPI_URING_STAGES") && getenv("IPI_URING_WAVES")) {
      shapes[0][0] = atoi(getenv("IPI_URING_WARPS"));
      shapes[0][1] = atoi(getenv("IPI_URING_STAGES"));
      shapes[0][2] = atoi(getenv("IPI_URING_WAVES"));
      shapes[0][3] = getenv("IPI_URING_AHEAD") ? atoi(getenv("IPI_URING_AHEAD")) : 1;
      nshape = 1;
    }
    const int budget = 227 * 1024 - 256;  // one CTA per SM
    // install one (warps, stages, waves, lookahead) shape into the plan
    auto install = [&](int NW, int S, int waves, int D) -> bool {
      const int blocks = (int)std::min<int64_t>((int64_t)h->num_sms * waves,
                                                std::max<int64_t>(1, (n_local + 63) / 64));
      std::vector<int64_t> hb(blocks + 1);
      for (int c = 0; c <= blocks; ++c) hb[c] = (int64_t)((double)n_local * c / blocks);
      hb[blocks] = n_local;
      int64_t worst = 0;
      for (int c = 0; c < blocks; ++c) worst = std::max<int64_t>(worst, hb[c + 1] - hb[c]);
      int wbytes = 0;
      const bool nowin = getenv("IPI_K1_NOWIN") && atoi(getenv("IPI_K1_NOWIN")) != 0;
      if (p.halo >= 0 && !nowin) {  // + 2: the cp.async window start is rounded down to an even index
        const int64_t wlen = std::min<int64_t>(n_global, worst + 2 * (int64_t)p.halo) + 2;
        wbytes = (int)std::min<int64_t>(wlen * 8, INT32_MAX / 2);
        if (uniform_ring_smem(64, S, NW, wbytes) > budget) return false;  // keep the window
      }
      const int smem = uniform_ring_smem(64, S, NW, wbytes);
      if (smem > budget || !k1_uring_prepare(64, NW, S, D, wbytes > 0, smem)) {
        cudaGetLastError();
        return false;
      }
      int64_t* db = nullptr;
      if (cudaMalloc(&db, sizeof(int64_t) * (blocks + 1)) != cudaSuccess ||
          cudaMemcpy(db, hb.data(), sizeof(int64_t) * (blocks + 1), cudaMemcpyHostToDevice) !=
              cudaSuccess) {
        if (db) cudaFree(db);
        cudaGetLastError();
        return false;
      }
      cudaFree(h->k1_bounds);
      h->k1_bounds = db;
      h->ring_win_bytes = wbytes;
      p.k1_blocks = blocks;
      p.k1_threads = NW * 32;
      p.k1_smem_bytes = smem;
      p.k1_stages = S;
      h->uring_lookahead = D;
      p.k1_variant = 6;
      return true;
    };
    bool done = false;
    for (int si = 0; si < nshape && !(env && env[0] == '0') && aligned && !done; ++si)
      done = install(shapes[si][0], shapes[si][1], shapes[si][2], shapes[si][3]);
    // Autotune the CTA count on the instance itself.  The streaming rate of the
    // ring depends on the number of CTAs in a way that differs between B200
    // boards (C2, 12 warps x 3 stages: 4 waves 0.70 on one box and 0.89 on
    // another, 8 waves the reverse pattern less often; per-CTA rates are
    // uniform within a launch, so it is not a tail effect —
    // scripts/k1_trace.py, scripts/k1_offset.py).  For large instances time a
    // few wave counts (one warm + one timed launch each, ~30 ms once) and keep
    // the fastest.  IPI_K1_AUTOTUNE=0 keeps the static first choice.
    const char* at = getenv("IPI_K1_AUTOTUNE");
    if (done && nshape > 1 && !(at && at[0] == '0') && nnz >= (1ll << 28)) {
      // the rate also varies between processes on one board (fresh physical
      // placement of the CSR), so a broader set of wave counts is timed
      const int cand[8] = {8, 6, 4, 2, 10, 12, 3, 5};
      K1Scratch tmp(n_global, n_local, st);
      const int best = !tmp.ok ? -1 : autotune_pick(
          8, [&](int i) { return install(12, 3, cand[i], 1); },
          [&] { return launch_bellman(h, tmp.v, IPI_MODE_MIN, tmp.policy, tmp.applied, nullptr,
                                      nullptr, nullptr, st); }, st, 1, 3, 2);
      if (best >= 0) install(12, 3, cand[best], 1);
      else install(shapes[0][0], shapes[0][1], shapes[0][2], shapes[0][3]);
    }
  }
  return IPI_OK;
}

// generic rows: CTA count autotuned on the instance
static int plan_generic_autotune(PlanCtx& c) {
  ipi_mdp* h = c.h;
  cudaStream_t st = c.st;
  ipi_plan& p = h->plan;
  [[maybe_unused]] const int64_t* row_ptr = h->rp;
  [[maybe_unused]] const int32_t* col = h->col;
  [[maybe_unused]] const double* values = h->val;
  [[maybe_unused]] const double* stage_cost = h->cost;
  [[maybe_unused]] const int64_t n_local = h->n_local, n_global = h->n_global, state0 = h->state0;
  [[maybe_unused]] const int32_t m = h->m;
  [[maybe_unused]] const int64_t rows = c.rows;
  [[maybe_unused]] const int64_t nnz = p.nnz;
  // ---- generic rows: autotune the CTA count (C4: 2 CTAs/SM 0.200 ms, 8 CTAs/SM
  // 0.154 ms; the order is not monotone, scripts/c4_ab.sh).  One warm + one
  // timed launch per candidate; IPI_K1_GEN_CTAS forces the static choice.
  if (p.k1_variant == 0 && p.halo >= 0 && nnz >= (1ll << 24) && n_local > 0 &&
      !getenv("IPI_K1_GEN_CTAS") && !(getenv("IPI_K1_AUTOTUNE") && getenv("IPI_K1_AUTOTUNE")[0] == '0')) {
    const int64_t max_blocks_g = std::max<int64_t>(1, (n_local + 15) / 16);
    auto install_gen = [&](int ctas) -> bool {
      const int blocks = (int)std::min<int64_t>((int64_t)h->num_sms * ctas, max_blocks_g);
      int64_t* db = nullptr;
      if (cudaMalloc(&db, sizeof(int64_t) * (blocks + 1)) != cudaSuccess) return false;
      bounds_kernel<<<(blocks + 1 + 127) / 128, 128, 0, st>>>(row_ptr, n_local, m, blocks, db);
      std::vector<int64_t> hb(blocks + 1);
      if (cudaMemcpyAsync(hb.data(), db, sizeof(int64_t) * (blocks + 1), cudaMemcpyDeviceToHost, st) !=
              cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        cudaFree(db);
        return false;
      }
      int64_t worst = 0;
      for (int c2 = 0; c2 < blocks; ++c2) worst = std::max<int64_t>(worst, hb[c2 + 1] - hb[c2]);
      const int64_t wlen = std::min<int64_t>(n_global, worst + 2 * (int64_t)p.halo);
      const int smem = (int)(wlen * 8 + 1024);
      if (smem > 200 * 1024 || k1_set_smem(p.lanes_per_row, smem) != IPI_OK) {
        cudaFree(db);
        cudaGetLastError();
        return false;
      }
      cudaFree(h->k1_bounds);
      h->k1_bounds = db;
      p.k1_blocks = blocks;
      p.k1_smem_bytes = smem;
      return true;
    };
    const int cand[5] = {8, 2, 4, 12, 16};
    K1Scratch tmp(n_global, n_local, st);
    const int best = !tmp.ok ? -1 : autotune_pick(
        5, [&](int i) { return install_gen(cand[i]); },
        [&] { return launch_bellman(h, tmp.v, IPI_MODE_MIN, tmp.policy, tmp.applied, nullptr,
                                    nullptr, nullptr, st); }, st);
    if (best >= 0) install_gen(cand[best]);
  }
  return IPI_OK;
}

// flat rows (K <= 4): per-warp cp.async ring
static int plan_flat_ring(PlanCtx& c) {
  ipi_mdp* h = c.h;
  cudaStream_t st = c.st;
  ipi_plan& p = h->plan;
  [[maybe_unused]] const int64_t* row_ptr = h->rp;
  [[maybe_unused]] const int32_t* col = h->col;
  [[maybe_unused]] const double* values = h->val;
  [[maybe_unused]] const double* stage_cost = h->cost;
  [[maybe_unused]] const int64_t n_local = h->n_local, n_global = h->n_global, state0 = h->state0;
  [[maybe_unused]] const int32_t m = h->m;
  [[maybe_unused]] const int64_t rows = c.rows;
  [[maybe_unused]] const int64_t nnz = p.nnz;
  // ---- flat rows (K <= 4): cp.async ring per warp (bellman.cu) ---------------
  if (p.uniform_rows && p.row_len_max <= 4 && (p.row_len_max % 2) == 0 && n_local > 0) {
    p.k1_variant = 5;  // register-pipelined flat kernel unless a ring shape fits
    const char* env = getenv("IPI_K1_RING");
    const bool aligned = ((uintptr_t)values % 16 == 0) && ((uintptr_t)stage_cost % 16 == 0) &&
                         ((uintptr_t)col % (p.row_len_max == 4 ? 16 : 8) == 0);
    // (stages, warps): forced by IPI_RING_STAGES / IPI_RING_WARPS, else the first that fits
    int shapes[4][2] = {{4, 18}, {4, 16}, {6, 12}, {8, 8}};  // measured order on C3
    int nshape = 4;
    if (getenv("IPI_RING_STAGES") && getenv("IPI_RING_WARPS")) {
      shapes[0][0] = atoi(getenv("IPI_RING_STAGES"));
      shapes[0][1] = atoi(getenv("IPI_RING_WARPS"));
      nshape = 1;
    }
    const int budget = 227 * 1024 - 256;  // one CTA per SM
    for (int si = 0; si < nshape && !(env && env[0] == '0') && aligned && p.k1_variant == 5; ++si) {
      const int S = shapes[si][0], NW = shapes[si][1];
      const int blocks = (int)std::min<int64_t>(h->num_sms, std::max<int64_t>(1, (n_local + 31) / 32));
      std::vector<int64_t> hb(blocks + 1);
      for (int c = 0; c <= blocks; ++c) hb[c] = (int64_t)((double)n_local * c / blocks);
      hb[blocks] = n_local;
      int64_t worst = 0;
      for (int c = 0; c < blocks; ++c) worst = std::max<int64_t>(worst, hb[c + 1] - hb[c]);
      int wbytes = 0;
      if (p.halo >= 0) {
        const int64_t wlen = std::min<int64_t>(n_global, worst + 2 * (int64_t)p.halo);
        wbytes = (int)std::min<int64_t>(wlen * 8, INT32_MAX / 2);
        if (flat_ring_smem(p.row_len_max, S, NW, m, wbytes) > budget) wbytes = 0;  // L1 gathers
      }
      const int smem = flat_ring_smem(p.row_len_max, S, NW, m, wbytes);
      if (smem > budget || !k1_ring_prepare(p.row_len_max, S, NW, wbytes > 0, smem)) {
        cudaGetLastError();
        continue;
      }
      int64_t* db = nullptr;
      if (cudaMalloc(&db, sizeof(int64_t) * (blocks + 1)) == cudaSuccess &&
          cudaMemcpy(db, hb.data(), sizeof(int64_t) * (blocks + 1), cudaMemcpyHostToDevice) ==
              cudaSuccess) {
        cudaFree(h->k1_bounds);
        h->k1_bounds = db;
        h->ring_win_bytes = wbytes;
        p.k1_blocks = blocks;
        p.k1_threads = NW * 32;
        p.k1_smem_bytes = smem;  // p.halo stays: the inner solver plans its own window from it
        p.k1_stages = S;
        p.k1_variant = 4;
      } else {
        if (db) cudaFree(db);
        cudaGetLastError();
      }
    }
  }
  return IPI_OK;
}

int plan_instance(ipi_mdp* h, cudaStream_t st) {
  PlanCtx c{h, st, h->n_local * (int64_t)h->m, {}};
  int rc = plan_row_stats(c);
  if (!rc) rc = plan_window_and_grid(c);
  if (!rc) rc = plan_deep(c);
  if (!rc) rc = plan_uniform_ring(c);
  if (!rc) rc = plan_generic_autotune(c);
  if (!rc) rc = plan_flat_ring(c);
  if (rc) return rc;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("planning kernels: ") + cudaGetErrorString(e));
  return IPI_OK;
}

}  // namespace ipi
