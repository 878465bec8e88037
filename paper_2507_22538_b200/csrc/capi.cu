// capi.cu — extern "C" boundary (include/ipi_b200.h), planning, validation and
// the native outer iPI loop (driver.py:109-209).
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "plan.cuh"

namespace ipi {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

cudaError_t raise_smem_limit(const void* fn, int smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> limits;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& cur = limits[{fn, dev}];
  if (smem <= cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

int pick_lanes_per_row(double mean_len) {
  // ~4+ elements per lane: 4 independent loads in flight per row
  if (mean_len <= 6.0) return 1;
  if (mean_len <= 12.0) return 2;
  if (mean_len <= 24.0) return 4;
  if (mean_len <= 56.0) return 8;
  if (mean_len <= 112.0) return 16;
  return 32;
}

int k1_set_smem(int lanes, int smem);  // bellman.cu
int k1_occupancy(int lanes, int uniform_K, bool win, int smem);

// ---------------------------------------------------------------------------
// validation (model.py:148-194 + sparse.py:56-86)
// ---------------------------------------------------------------------------
struct VAcc {
  unsigned long long bad_rp, bad_range, bad_order, nonfinite, first_bad_prob, n_bad_sum,
      first_bad_sum_row, nonfinite_cost;
};

__global__ void validate_rowptr_kernel(const int64_t* rp, int64_t rows, VAcc* acc) {
  unsigned long long bad = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    bad += rp[r + 1] < rp[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) bad += rp[0] != 0;
  for (int off = 16; off; off >>= 1) bad += __shfl_xor_sync(kFull, bad, off);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&acc->bad_rp, bad);
}

// warp per row: column range/order, finiteness, [0,1], row sums.
// `after` restricts the bad-sum search to rows > after (used to list the first five).
__global__ void validate_rows_kernel(const int64_t* rp, const int32_t* col, const double* val,
                                     int64_t rows, int64_t ncols, long long after, VAcc* acc,
                                     int structural_only) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long br = 0, bo = 0, nf = 0;
  for (int64_t r = wg; r < rows; r += nw) {
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    double sum = 0.0;
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      const int c = col[p];
      br += (c < 0 || (int64_t)c >= ncols);
      if (p > p0) bo += col[p - 1] >= c;
      const double v = val[p];
      if (!isfinite(v)) nf += 1;
      if (!structural_only && (v < 0.0 || v > 1.0))
        atomicMin(&acc->first_bad_prob, (unsigned long long)p);
      sum = add_rn(sum, v);
    }
    if (!structural_only && (long long)r > after) {
      sum = warp_sum(sum);
      if (lane == 0 && fabs(sum - 1.0) > 1e-12) {
        atomicAdd(&acc->n_bad_sum, 1ull);
        atomicMin(&acc->first_bad_sum_row, (unsigned long long)r);
      }
    }
  }
  for (int off = 16; off; off >>= 1) {
    br += __shfl_xor_sync(kFull, br, off);
    bo += __shfl_xor_sync(kFull, bo, off);
    nf += __shfl_xor_sync(kFull, nf, off);
  }
  if (lane == 0) {
    if (br) atomicAdd(&acc->bad_range, br);
    if (bo) atomicAdd(&acc->bad_order, bo);
    if (nf) atomicAdd(&acc->nonfinite, nf);
  }
}

// Uniform rows of length K = 8*G (K % 4 == 0 and 16-byte aligned arrays: C2 /
// C5's K = 64): G lanes per row, 8 consecutive entries per lane read with
// 16-byte loads, 32/G rows per warp step and two steps in flight, so the
// 26 GB validation pass streams instead of waiting per row (the warp-per-row
// kernel above is latency-bound).  Same checks and counters; the row sum is
// lane partials then an xor tree (1e-12 tolerance, as the warp-per-row kernel).
template <int G>
__global__ void __launch_bounds__(256) validate_rows_uniform_kernel(
    const int32_t* __restrict__ col, const double* __restrict__ val, int64_t rows, int64_t ncols,
    VAcc* acc, int structural_only) {
  constexpr int K = 8 * G, RPW = 32 / G;
  const int lane = threadIdx.x & 31, grp = lane / G, gl = lane % G;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  unsigned long long br = 0, bo = 0, nf = 0;
  auto do_rows = [&](int64_t base) {
    const int64_t r = base + grp;
    const bool ok = r < rows;
    const int64_t p0 = (ok ? r : 0) * K + 8 * gl;
    double v[8];
    int c[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 t = ld_stream_v2(val + p0 + 2 * q, pol);
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int2 t = ld_stream_v2(col + p0 + 2 * q, pol);
      c[2 * q] = t.x;
      c[2 * q + 1] = t.y;
    }
    // previous column of this lane's first entry: last entry of lane gl-1 in the row
    const int prev = __shfl_up_sync(kFull, c[7], 1);
    double sum = 0.0;
    if (ok) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        br += (c[q] < 0 || (int64_t)c[q] >= ncols);
        if (q > 0) bo += c[q - 1] >= c[q];
        if (!isfinite(v[q])) nf += 1;
        if (!structural_only && (v[q] < 0.0 || v[q] > 1.0))
          atomicMin(&acc->first_bad_prob, (unsigned long long)(p0 + q));
        sum = add_rn(sum, v[q]);
      }
      if (gl > 0) bo += prev >= c[0];
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) sum = add_rn(sum, __shfl_xor_sync(kFull, sum, off));
    if (!structural_only && ok && gl == 0 && fabs(sum - 1.0) > 1e-12) {
      atomicAdd(&acc->n_bad_sum, 1ull);
      atomicMin(&acc->first_bad_sum_row, (unsigned long long)r);
    }
  };
  for (int64_t base = wg * RPW; base < rows; base += 2 * nw * RPW) {
    do_rows(base);
    if (base + nw * RPW < rows) do_rows(base + nw * RPW);
  }
  for (int off = 16; off; off >>= 1) {
    br += __shfl_xor_sync(kFull, br, off);
    bo += __shfl_xor_sync(kFull, bo, off);
    nf += __shfl_xor_sync(kFull, nf, off);
  }
  if (lane == 0) {
    if (br) atomicAdd(&acc->bad_range, br);
    if (bo) atomicAdd(&acc->bad_order, bo);
    if (nf) atomicAdd(&acc->nonfinite, nf);
  }
}

__global__ void uniform_rp_check_kernel(const int64_t* rp, int64_t rows, int64_t K,
                                        unsigned long long* bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= rows;
       r += (int64_t)gridDim.x * blockDim.x)
    if (rp[r] != r * K) atomicAdd(bad, 1ull);
}

// min / max column index of a CSR block (the V range a row-sharded rank reads)
__global__ void col_range_kernel(const int32_t* __restrict__ col, int64_t nnz, int* out) {
  int lo = INT32_MAX, hi = INT32_MIN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = col[i];
    lo = c < lo ? c : lo;
    hi = c > hi ? c : hi;
  }
  for (int off = 16; off; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, off));
    hi = max(hi, __shfl_xor_sync(kFull, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

__global__ void row_sum_kernel(const int64_t* rp, const double* val, int64_t r, double* out) {
  // same summation layout as validate_rows_kernel for one row
  const int lane = threadIdx.x;
  double sum = 0.0;
  for (int64_t p = rp[r] + lane; p < rp[r + 1]; p += 32) sum = add_rn(sum, val[p]);
  sum = warp_sum(sum);
  if (lane == 0) *out = sum;
}

__global__ void cost_finite_kernel(const double* cost, int64_t len, VAcc* acc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(cost[i])) atomicMin(&acc->nonfinite_cost, (unsigned long long)i);
}


int ensure_scratch(ipi_mdp* h) {
  if (h->pi) return IPI_OK;
  const int64_t n = std::max<int64_t>(h->n_local, 1);
  IPI_CUDA_TRY(cudaMalloc(&h->pi, sizeof(int32_t) * n));
  IPI_CUDA_TRY(cudaMalloc(&h->applied, sizeof(double) * n));
  IPI_CUDA_TRY(cudaMalloc(&h->gpi, sizeof(double) * n));
  IPI_CUDA_TRY(cudaMalloc(&h->lenpi, sizeof(int32_t) * n));
  IPI_CUDA_TRY(cudaMalloc(&h->res_bits, sizeof(unsigned long long) * 2));
  IPI_CUDA_TRY(cudaMalloc(&h->xbuf, sizeof(double) * n));
  IPI_CUDA_TRY(cudaMalloc(&h->d_report, sizeof(ipi_inner_report)));
  h->kry_len = krylov_workspace_doubles(n);
  IPI_CUDA_TRY(cudaMalloc(&h->kry, sizeof(double) * h->kry_len));
  const int64_t cap = std::max<int64_t>((int64_t)h->plan.row_len_max * h->n_local, 1);
  IPI_CUDA_TRY(cudaMalloc(&h->rp_pi, sizeof(int64_t) * (n + 1)));
  IPI_CUDA_TRY(cudaMalloc(&h->col_pi, sizeof(int32_t) * cap));
  IPI_CUDA_TRY(cudaMalloc(&h->val_pi, sizeof(double) * cap));
  h->cap_pi = cap;
  return IPI_OK;
}

}  // namespace ipi

using namespace ipi;

extern "C" {

const char* ipi_last_error(void) { return g_err.c_str(); }

const char* ipi_version(void) { return "ipi_b200 0.1 (sm_100a, fp64 CSR, persistent GMRES)"; }

int ipi_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int ipi_mdp_create(const int64_t* row_ptr, const int32_t* col, const double* values,
                   const double* stage_cost, int64_t n_local, int64_t n_global, int32_t m,
                   int64_t state0, double gamma, int32_t mode, void* stream, ipi_mdp** out) {
  if (!out) return fail(IPI_EVALIDATION, "null output handle");
  *out = nullptr;
  if (m < 1) return fail(IPI_EVALIDATION, "action count must be >= 1, got " + std::to_string(m));
  if (n_local < 0 || n_global < 1 || state0 < 0 || state0 + n_local > n_global)
    return fail(IPI_EDIMENSION, "inconsistent shard geometry");
  if (n_global > INT32_MAX) return fail(IPI_EDIMENSION, "state count exceeds int32 column range");
  cudaStream_t st = (cudaStream_t)stream;
  ipi_mdp* h = new ipi_mdp();
  h->rp = row_ptr;
  h->col = col;
  h->val = values;
  h->cost = stage_cost;
  h->n_local = n_local;
  h->n_global = n_global;
  h->state0 = state0;
  h->m = m;
  h->gamma = gamma;
  h->mode = mode;
  cudaGetDevice(&h->device);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  auto bail = [&](int code) {
    ipi_mdp_destroy(h);
    return code;
  };
  if (getenv("IPI_K1_WIN_ASYNC")) h->k1_win_async = atoi(getenv("IPI_K1_WIN_ASYNC")) != 0;
  if (getenv("IPI_K1_INTERLEAVE")) h->k1_interleave = atoi(getenv("IPI_K1_INTERLEAVE")) != 0;
  if (getenv("IPI_K1_ROTATE")) h->k1_rotate = atoi(getenv("IPI_K1_ROTATE")) != 0;
  if (cudaMallocHost(&h->host_pinned, 4096) != cudaSuccess)
    return bail(fail(IPI_ECUDA, "cudaMallocHost failed"));
  const int rc = plan_instance(h, st);
  if (rc) return bail(rc);
  *out = h;
  return IPI_OK;
}

void ipi_mdp_destroy(ipi_mdp* h) {
  if (!h) return;
  cudaFree(h->k1_bounds);
  cudaFree(h->pi);
  cudaFree(h->applied);
  cudaFree(h->gpi);
  cudaFree(h->lenpi);
  cudaFree(h->res_bits);
  cudaFree(h->rp_pi);
  cudaFree(h->col_pi);
  cudaFree(h->val_pi);
  cudaFree(h->xbuf);
  cudaFree(h->scan_tmp);
  cudaFree(h->d_report);
  cudaFree(h->kry);
  cudaFree(h->invd);
  cudaFree(h->vbuf);
  cudaFree(h->k1_trace);
  ipi_op_destroy(h->op_pi);
  if (h->host_pinned) cudaFreeHost(h->host_pinned);
  delete h;
}

int ipi_mdp_k1_trace(ipi_mdp* h, int32_t enable, uint64_t* out, int32_t cap) {
  if (!h) return fail(IPI_EVALIDATION, "null handle");
  const int64_t words = 3 * (int64_t)h->plan.k1_blocks;
  if (enable) {
    if (!h->k1_trace) IPI_CUDA_TRY(cudaMalloc(&h->k1_trace, sizeof(uint64_t) * words));
    IPI_CUDA_TRY(cudaMemset(h->k1_trace, 0, sizeof(uint64_t) * words));
    return IPI_OK;
  }
  if (h->k1_trace && out && cap > 0) {
    IPI_CUDA_TRY(cudaDeviceSynchronize());
    IPI_CUDA_TRY(cudaMemcpy(out, h->k1_trace, sizeof(uint64_t) * std::min<int64_t>(words, cap),
                            cudaMemcpyDeviceToHost));
  }
  cudaFree(h->k1_trace);
  h->k1_trace = nullptr;
  return IPI_OK;
}

int ipi_mdp_plan(const ipi_mdp* h, ipi_plan* out) {
  if (!h || !out) return fail(IPI_EVALIDATION, "null handle");
  *out = h->plan;
  return IPI_OK;
}

static int csr_check_impl(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                          int64_t cols, int64_t nnz_len, ipi_csr_report* out, bool probs,
                          const double* cost, int64_t cost_len, VAcc* res, cudaStream_t st) {
  std::memset(out, 0, sizeof(*out));
  VAcc init;
  std::memset(&init, 0, sizeof(init));
  init.first_bad_prob = ~0ull;
  init.first_bad_sum_row = ~0ull;
  init.nonfinite_cost = ~0ull;
  VAcc* d = nullptr;
  IPI_CUDA_TRY(cudaMalloc(&d, sizeof(VAcc)));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaMemcpyAsync(d, &init, sizeof(VAcc), cudaMemcpyHostToDevice, st);
  if (rows > 0) validate_rowptr_kernel<<<grid_for(rows, 256, sms), 256, 0, st>>>(rp, rows, d);
  if (cost && cost_len > 0) cost_finite_kernel<<<grid_for(cost_len, 256, sms), 256, 0, st>>>(cost, cost_len, d);
  int64_t last = 0;
  cudaMemcpyAsync(&last, rp + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(res, d, sizeof(VAcc), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(d);
    return fail(IPI_ECUDA, std::string("csr check: ") + cudaGetErrorString(e));
  }
  out->bad_row_ptr = (int64_t)res->bad_rp;
  out->nnz = last;
  out->nnz_mismatch = (last != nnz_len);
  if (out->bad_row_ptr == 0 && !out->nnz_mismatch && rows > 0 && last > 0) {
    // uniform K = 64 rows with 16-byte aligned arrays: the streaming kernel
    bool uniform64 = last == rows * 64 && (uintptr_t)val % 16 == 0 && (uintptr_t)col % 16 == 0;
    if (uniform64) {  // every row exactly 64 long <=> rp[r] == 64 r (checked on the device)
      unsigned long long* flag = nullptr;
      uniform64 = cudaMalloc(&flag, sizeof(unsigned long long)) == cudaSuccess;
      if (uniform64) {
        unsigned long long hflag = 0;
        cudaMemsetAsync(flag, 0, sizeof(unsigned long long), st);
        uniform_rp_check_kernel<<<grid_for(rows + 1, 256, sms), 256, 0, st>>>(rp, rows, 64, flag);
        cudaMemcpyAsync(&hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, st);
        uniform64 = cudaStreamSynchronize(st) == cudaSuccess && hflag == 0;
        cudaFree(flag);
      }
    }
    if (uniform64)
      validate_rows_uniform_kernel<8><<<sms * 8, 256, 0, st>>>(col, val, rows, cols, d, probs ? 0 : 1);
    else
      validate_rows_kernel<<<grid_for(rows * 32, 256, sms), 256, 0, st>>>(rp, col, val, rows, cols,
                                                                            probs ? -1 : (long long)rows, d, probs ? 0 : 1);
    cudaMemcpyAsync(res, d, sizeof(VAcc), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      cudaFree(d);
      return fail(IPI_ECUDA, std::string("csr check: ") + cudaGetErrorString(e));
    }
    out->bad_col_range = (int64_t)res->bad_range;
    out->bad_col_order = (int64_t)res->bad_order;
    out->nonfinite_values = (int64_t)res->nonfinite;
  }
  cudaFree(d);
  return IPI_OK;
}

int ipi_csr_check(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t rows,
                  int64_t cols, int64_t nnz_len, ipi_csr_report* out, void* stream) {
  if (!out) return fail(IPI_EVALIDATION, "null report");
  VAcc res;
  return csr_check_impl(row_ptr, col, val, rows, cols, nnz_len, out, false, nullptr, 0, &res,
                        (cudaStream_t)stream);
}

int ipi_validate(ipi_mdp* h, ipi_validation* out, void* stream) {
  if (!h || !out) return fail(IPI_EVALIDATION, "null handle");
  cudaStream_t st = (cudaStream_t)stream;
  std::memset(out, 0, sizeof(*out));
  out->first_bad_prob = -1;
  out->nonfinite_cost = -1;
  for (int i = 0; i < 5; ++i) out->bad_rows[i] = -1;
  const int64_t rows = h->n_local * (int64_t)h->m;
  ipi_csr_report cr;
  VAcc r;
  int rc = csr_check_impl(h->rp, h->col, h->val, rows, h->n_global, h->plan.nnz, &cr, true,
                          h->cost, rows, &r, st);
  if (rc) return rc;
  out->bad_row_ptr = cr.bad_row_ptr + (cr.nnz_mismatch ? 1 : 0);
  out->bad_col_range = cr.bad_col_range;
  out->bad_col_order = cr.bad_col_order;
  out->nonfinite_values = cr.nonfinite_values;
  out->nonfinite_cost = r.nonfinite_cost == ~0ull ? -1 : (int64_t)r.nonfinite_cost;
  if (out->bad_row_ptr) return IPI_OK;
  out->first_bad_prob = r.first_bad_prob == ~0ull ? -1 : (int64_t)r.first_bad_prob;
  if (r.first_bad_prob != ~0ull) {
    IPI_CUDA_TRY(cudaMemcpy(&out->first_bad_prob_value, h->val + r.first_bad_prob, sizeof(double),
                            cudaMemcpyDeviceToHost));
  }
  out->n_bad_row_sums = (int64_t)r.n_bad_sum;
  if (r.n_bad_sum > 0) {
    VAcc* d = nullptr;
    double* dsum = nullptr;
    IPI_CUDA_TRY(cudaMalloc(&d, sizeof(VAcc)));
    IPI_CUDA_TRY(cudaMalloc(&dsum, sizeof(double)));
    VAcc init;
    std::memset(&init, 0, sizeof(init));
    init.first_bad_prob = ~0ull;
    init.first_bad_sum_row = ~0ull;
    init.nonfinite_cost = ~0ull;
    unsigned long long row = r.first_bad_sum_row;
    for (int k = 0; k < 5 && row != ~0ull; ++k) {
      out->bad_rows[k] = (int64_t)row;
      row_sum_kernel<<<1, 32, 0, st>>>(h->rp, h->val, (int64_t)row, dsum);
      cudaMemcpyAsync(&out->bad_row_sums[k], dsum, sizeof(double), cudaMemcpyDeviceToHost, st);
      if (k == 4) break;
      cudaMemcpyAsync(d, &init, sizeof(VAcc), cudaMemcpyHostToDevice, st);
      validate_rows_kernel<<<grid_for(rows * 32, 256, h->num_sms), 256, 0, st>>>(
          h->rp, h->col, h->val, rows, h->n_global, (long long)row, d, 0);
      VAcc r2;
      cudaMemcpyAsync(&r2, d, sizeof(VAcc), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) break;
      row = r2.first_bad_sum_row;
    }
    cudaStreamSynchronize(st);
    cudaFree(d);
    cudaFree(dsum);
  }
  IPI_CUDA_TRY(cudaGetLastError());
  return IPI_OK;
}

int ipi_bellman(ipi_mdp* h, const double* v_full, int32_t mode, int32_t* policy, double* applied,
                double* g_pi, int32_t* len_pi, unsigned long long* res_inf_bits, void* stream) {
  if (!h) return fail(IPI_EVALIDATION, "null handle");
  if (res_inf_bits)  // zeroed here (a memset, not a kernel) so callers cannot forget
    IPI_CUDA_TRY(cudaMemsetAsync(res_inf_bits, 0, sizeof(unsigned long long), (cudaStream_t)stream));
  return launch_bellman(h, v_full, mode, policy, applied, g_pi, len_pi, res_inf_bits,
                        (cudaStream_t)stream);
}

int ipi_policy_nnz(ipi_mdp* h, const int32_t* policy, int64_t* nnz_out, void* stream) {
  if (!h || !nnz_out) return fail(IPI_EVALIDATION, "null argument");
  return policy_nnz(h, policy, nnz_out, (cudaStream_t)stream);
}

int ipi_gather_policy(ipi_mdp* h, const int32_t* policy, int64_t* rp_pi, int32_t* col_pi,
                      double* val_pi, double* g_pi, void* stream) {
  if (!h) return fail(IPI_EVALIDATION, "null handle");
  return gather_policy(h, policy, nullptr, rp_pi, col_pi, val_pi, g_pi, nullptr,
                       (cudaStream_t)stream);
}

int ipi_spmv(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t rows,
             int64_t cols, const double* x, double* y, void* stream) {
  (void)cols;
  if (rows < 0) return fail(IPI_EDIMENSION, "negative row count");
  if (rows == 0) return IPI_OK;
  int64_t nnz = 0;
  IPI_CUDA_TRY(cudaMemcpyAsync(&nnz, row_ptr + rows, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               (cudaStream_t)stream));
  IPI_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return launch_spmv(row_ptr, col, val, rows, x, nullptr, 0.0, 0, y,
                     pick_lanes_per_row((double)nnz / (double)rows), (cudaStream_t)stream);
}

int ipi_apply_J(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                double gamma, const double* x, const double* b, double* y, void* stream) {
  if (n <= 0) return IPI_OK;
  int64_t nnz = 0;
  IPI_CUDA_TRY(cudaMemcpyAsync(&nnz, rp_pi + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               (cudaStream_t)stream));
  IPI_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return launch_spmv(rp_pi, col_pi, val_pi, n, x, b, gamma, b ? 2 : 1, y,
                     pick_lanes_per_row((double)nnz / (double)n), (cudaStream_t)stream);
}

int ipi_apply_J_shard(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi,
                      int64_t n_local, int64_t state0, double gamma, const double* x_full,
                      const double* b, double* y, void* stream) {
  if (n_local <= 0) return IPI_OK;
  int64_t nnz = 0;
  IPI_CUDA_TRY(cudaMemcpyAsync(&nnz, rp_pi + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               (cudaStream_t)stream));
  IPI_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return launch_spmv(rp_pi, col_pi, val_pi, n_local, x_full, b, gamma, b ? 2 : 1, y,
                     pick_lanes_per_row((double)nnz / (double)n_local), (cudaStream_t)stream,
                     state0);
}

// ---- planned policy operator (K3) ------------------------------------------
int ipi_op_create(const int64_t* rp, const int32_t* col, const double* val, int64_t n_local,
                  int64_t n_global, int64_t state0, double gamma, void* stream, ipi_op** out) {
  if (!out) return fail(IPI_EVALIDATION, "null output operator");
  *out = nullptr;
  if (n_local < 0 || n_global < 1 || state0 < 0 || state0 + n_local > n_global)
    return fail(IPI_EDIMENSION, "inconsistent operator geometry");
  ipi_op* op = new ipi_op();
  op->rp = rp;
  op->col = col;
  op->val = val;
  op->n_local = n_local;
  op->n_global = n_global;
  op->state0 = state0;
  op->gamma = gamma;
  if (n_local == 0) {
    *out = op;
    return IPI_OK;
  }
  // row statistics + sampled locality profile: the planner of an m = 1 view
  ipi_mdp* view = nullptr;
  int rc = ipi_mdp_create(rp, col, val, val, n_local, n_global, 1, state0, gamma, IPI_MODE_MIN,
                          stream, &view);
  if (rc) {
    delete op;
    return rc;
  }
  const ipi_plan pl = view->plan;
  const int sms = view->num_sms;
  ipi_mdp_destroy(view);
  op->nnz = pl.nnz;
  op->lanes = pl.lanes_per_row;
  op->K = pl.uniform_rows ? pl.row_len_max : 0;
  op->variant = IPI_K3_GENERIC;
  const char* env = getenv("IPI_K3_RING");
  const bool allow = !(env && env[0] == '0');
  const int K = op->K;
  const bool aligned = ((uintptr_t)val % 16 == 0) && ((uintptr_t)col % (K == 2 ? 8 : 16) == 0);
  const int budget = 227 * 1024 - 256;
  // (warps, stages, CTAs per SM); IPI_K3_WARPS/STAGES/WAVES force one shape
  int shapes[4][3];
  int nshape = 0;
  int variant = IPI_K3_GENERIC;
  if (K == 64) {
    variant = IPI_K3_URING;
    const int sh[4][3] = {{11, 3, 1}, {12, 3, 4}, {16, 3, 2}, {8, 4, 4}};
    std::memcpy(shapes, sh, sizeof(sh));
    nshape = 4;
  } else if (K == 4 || K == 2) {
    variant = IPI_K3_FLAT;
    const int sh[4][3] = {{24, 4, 1}, {16, 4, 1}, {8, 6, 2}, {16, 4, 1}};
    std::memcpy(shapes, sh, sizeof(sh));
    nshape = 3;
  }
  if (nshape && getenv("IPI_K3_WARPS") && getenv("IPI_K3_STAGES") && getenv("IPI_K3_WAVES")) {
    shapes[0][0] = atoi(getenv("IPI_K3_WARPS"));
    shapes[0][1] = atoi(getenv("IPI_K3_STAGES"));
    shapes[0][2] = atoi(getenv("IPI_K3_WAVES"));
    nshape = 1;
  }
  const int align = variant == IPI_K3_FLAT ? 32 : 4;
  // nowin: no x window — gathers go through L1/L2 (x is L2-resident) and the
  // warps interleave 4-row steps so each CTA reads one contiguous stream; on
  // C2 this beats the windowed shapes (0.81 vs 0.72 of HBM: no window staging
  // before the first row, fewer concurrent DRAM streams).
  auto install = [&](int NW, int S, int waves, bool nowin = false, int ilv = -1) -> bool {
    const int64_t per_warp_min = variant == IPI_K3_FLAT ? 64 : 16;
    const int blocks = (int)std::min<int64_t>((int64_t)sms * waves,
                                              std::max<int64_t>(1, n_local / (NW * per_warp_min)));
    const int64_t worst = (n_local + blocks - 1) / blocks + 2 * align;
    int wbytes = 0;
    int halo = nowin ? -1 : pl.halo;
    if (halo >= 0 && getenv("IPI_K3_HALO")) halo = std::min(halo, std::max(-1, atoi(getenv("IPI_K3_HALO"))));
    if (halo >= 0) {  // + 2: the window start is rounded down to an even index
      const int64_t wlen = std::min<int64_t>(n_global, worst + 2 * (int64_t)halo) + 2;
      wbytes = (int)std::min<int64_t>(wlen * 8, INT32_MAX / 2);
    }
    int smem = variant == IPI_K3_FLAT ? k3_flat_smem(K, S, NW, wbytes) : k3_uring_smem(K, S, NW, wbytes);
    if (smem > budget && wbytes > 0) {  // drop the window rather than the ring
      wbytes = 0;
      smem = variant == IPI_K3_FLAT ? k3_flat_smem(K, S, NW, 0) : k3_uring_smem(K, S, NW, 0);
    }
    if (smem > budget || !k3_shape_prepare(variant, K, NW, S, wbytes > 0, smem)) return false;
    op->variant = variant;
    op->blocks = blocks;
    op->warps = NW;
    op->stages = S;
    op->smem = smem;
    op->win_bytes = wbytes;
    op->halo = wbytes > 0 ? halo : -1;
    op->pf = getenv("IPI_K3_PF") ? atoi(getenv("IPI_K3_PF")) : 0;
    op->interleave = ilv >= 0 ? ilv : wbytes == 0;
    if (getenv("IPI_K3_INTERLEAVE")) op->interleave = atoi(getenv("IPI_K3_INTERLEAVE")) != 0;
    if (variant != IPI_K3_URING) op->interleave = 0;  // the flat kernel has one row order
    return true;
  };
  bool done = false;
  for (int si = 0; si < nshape && allow && aligned && pl.uniform_rows && !done; ++si)
    done = install(shapes[si][0], shapes[si][1], shapes[si][2]);
  // Autotune the shape on the operator itself for large P_pi (same board
  // sensitivity as K1, see ipi_mdp_create): one warm + three timed applies per
  // candidate (~6 ms once per operator).  IPI_K3_AUTOTUNE=0 disables.
  const char* at = getenv("IPI_K3_AUTOTUNE");
  if (done && nshape > 1 && !(at && at[0] == '0') && op->nnz >= (1ll << 25)) {
    // (warps, stages, CTAs per SM, no window, interleaved warps)
    const int cu[11][5] = {{12, 3, 1, 1, 1}, {11, 3, 1, 1, 1}, {10, 3, 2, 1, 1}, {10, 4, 1, 1, 1},
                           {12, 3, 3, 1, 0}, {12, 3, 4, 1, 0}, {11, 3, 1, 0, 0}, {12, 3, 3, 0, 0},
                           {12, 3, 6, 0, 0}, {12, 3, 4, 0, 0}, {12, 3, 2, 0, 0}};
    const int cf[4][5] = {{24, 4, 1, 0, 0}, {28, 4, 1, 0, 0}, {16, 4, 1, 0, 0}, {16, 4, 2, 0, 0}};
    const int nc = variant == IPI_K3_FLAT ? 4 : 11;
    auto shape = [&](int i) { return variant == IPI_K3_FLAT ? cf[i] : cu[i]; };
    // The pick is cached per (device, geometry, halo) for the process: the
    // sharded driver re-plans P_pi every outer iteration with the same shape
    // (IPI_K3_AUTOTUNE_CACHE=0 re-times every operator).
    static std::mutex tune_mu;
    static std::map<std::vector<int64_t>, int> tune_cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const std::vector<int64_t> key = {dev, variant, K, n_local, n_global, state0, op->nnz, pl.halo};
    const char* cenv = getenv("IPI_K3_AUTOTUNE_CACHE");
    const bool use_cache = !(cenv && cenv[0] == '0');
    int best = -1;
    if (use_cache) {
      std::lock_guard<std::mutex> lk(tune_mu);
      auto it = tune_cache.find(key);
      if (it != tune_cache.end()) best = it->second;
    }
    if (best < 0) {
      cudaStream_t st = (cudaStream_t)stream;
      double* tx = nullptr;
      double* ty = nullptr;
      const bool ok = cudaMalloc(&tx, sizeof(double) * n_global) == cudaSuccess &&
                      cudaMalloc(&ty, sizeof(double) * n_local) == cudaSuccess &&
                      cudaMemsetAsync(tx, 0, sizeof(double) * n_global, st) == cudaSuccess;
      best = !ok ? -1 : autotune_pick(
          nc, [&](int i) { const int* c = shape(i); return install(c[0], c[1], c[2], c[3] != 0, c[4]); },
          [&] { return op_launch(op, tx, nullptr, 1, ty, st); }, st, 3, 3, 10);
      cudaFree(tx);
      cudaFree(ty);
      cudaGetLastError();
      if (best >= 0 && use_cache) {
        std::lock_guard<std::mutex> lk(tune_mu);
        tune_cache[key] = best;
      }
    }
    bool installed = false;
    if (best >= 0) {
      const int* c = shape(best);
      installed = install(c[0], c[1], c[2], c[3] != 0, c[4]);
    }
    if (!installed) install(shapes[0][0], shapes[0][1], shapes[0][2]);
  }
  *out = op;
  return IPI_OK;
}

void ipi_op_destroy(ipi_op* op) {
  if (op) cudaFree(op->trace);
  delete op;
}

int ipi_op_trace(ipi_op* op, int32_t enable, uint64_t* out, int32_t cap) {
  if (!op) return fail(IPI_EVALIDATION, "null operator");
  const int64_t words = 3 * (int64_t)std::max(op->blocks, 1);
  if (enable) {
    if (!op->trace) IPI_CUDA_TRY(cudaMalloc(&op->trace, sizeof(uint64_t) * words));
    IPI_CUDA_TRY(cudaMemset(op->trace, 0, sizeof(uint64_t) * words));
    return IPI_OK;
  }
  if (op->trace && out && cap > 0) {
    IPI_CUDA_TRY(cudaDeviceSynchronize());
    IPI_CUDA_TRY(cudaMemcpy(out, op->trace, sizeof(uint64_t) * std::min<int64_t>(words, cap),
                            cudaMemcpyDeviceToHost));
  }
  cudaFree(op->trace);
  op->trace = nullptr;
  return IPI_OK;
}

int ipi_op_get_plan(const ipi_op* op, ipi_op_plan* out) {
  if (!op || !out) return fail(IPI_EVALIDATION, "null operator");
  out->nnz = op->nnz;
  out->variant = op->variant;
  out->row_len = op->K;
  out->halo = op->halo;
  out->blocks = op->blocks;
  out->threads = op->warps * 32;
  out->smem_bytes = op->smem;
  out->stages = op->stages;
  out->lanes_per_row = op->lanes;
  out->interleave = op->interleave;
  return IPI_OK;
}

static int op_run(const ipi_op* op, const double* x_full, const double* b, int epi, double* y,
                  void* stream) {
  if (!op) return fail(IPI_EVALIDATION, "null operator");
  if (op->n_local > 0 && (!x_full || !y)) return fail(IPI_EVALIDATION, "null vector");
  if (op->variant != IPI_K3_GENERIC &&
      ((b && (uintptr_t)b % 16 != 0) || (op->win_bytes > 0 && (uintptr_t)x_full % 16 != 0))) {
    ipi_op generic = *op;  // b and window chunks are copied 16 bytes at a time
    generic.variant = IPI_K3_GENERIC;
    return op_launch(&generic, x_full, b, epi, y, (cudaStream_t)stream);
  }
  return op_launch(op, x_full, b, epi, y, (cudaStream_t)stream);
}

int ipi_op_apply(const ipi_op* op, const double* x_full, const double* b, double* y, void* stream) {
  return op_run(op, x_full, b, b ? 2 : 1, y, stream);
}

int ipi_op_spmv(const ipi_op* op, const double* x_full, double* y, void* stream) {
  return op_run(op, x_full, nullptr, 0, y, stream);
}

int ipi_op_apply_partial(const ipi_op* op, const double* x_full, const double* y_partial,
                         const double* b, double* y, void* stream) {
  if (!op) return fail(IPI_EVALIDATION, "null operator");
  if (op->n_local > 0 && (!x_full || !y || !y_partial)) return fail(IPI_EVALIDATION, "null vector");
  return op_launch(op, x_full, b, b ? 5 : 4, y, (cudaStream_t)stream, y_partial);
}

int ipi_csr_split_local(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                        int64_t lo, int64_t hi, int64_t* rp_loc, int32_t* col_loc, double* val_loc,
                        int64_t* rp_rem, int32_t* col_rem, double* val_rem, void* stream) {
  if (rows < 0 || lo < 0 || hi < lo || hi > INT32_MAX) return fail(IPI_EDIMENSION, "bad split geometry");
  if (!rp || !rp_loc || !rp_rem) return fail(IPI_EVALIDATION, "null row pointers");
  if ((col_loc == nullptr) != (col_rem == nullptr) || (col_loc && (!val_loc || !val_rem)))
    return fail(IPI_EVALIDATION, "split: pass 2 needs all output arrays");
  return split_local_remote(rp, col, val, rows, (int32_t)lo, (int32_t)hi, rp_loc, col_loc, val_loc,
                            rp_rem, col_rem, val_rem, (cudaStream_t)stream);
}

int ipi_col_range(const int32_t* col, int64_t nnz, int64_t* cmin, int64_t* cmax, void* stream) {
  if (!cmin || !cmax) return fail(IPI_EVALIDATION, "null output");
  *cmin = 0;
  *cmax = -1;
  if (nnz <= 0) return IPI_OK;
  if (!col) return fail(IPI_EVALIDATION, "null columns");
  cudaStream_t st = (cudaStream_t)stream;
  int* d = nullptr;
  IPI_CUDA_TRY(cudaMalloc(&d, 2 * sizeof(int)));
  const int init[2] = {INT32_MAX, INT32_MIN};
  cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  col_range_kernel<<<grid_for(nnz, 256, sms), 256, 0, st>>>(col, nnz, d);
  int h[2];
  cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(d);
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("col range: ") + cudaGetErrorString(e));
  *cmin = h[0];
  *cmax = h[1];
  return IPI_OK;
}

int ipi_jacobi_inv_diag(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi,
                        int64_t n, double gamma, double* inv_diag, void* stream) {
  if (!inv_diag) return fail(IPI_EVALIDATION, "null output");
  return jacobi_inv_diag(rp_pi, col_pi, val_pi, n, gamma, inv_diag, (cudaStream_t)stream);
}

int ipi_inner_solve(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                    double gamma, const double* b, double* x, double target_2norm,
                    int32_t max_it, int32_t kind, double richardson_scale,
                    const double* inv_diag, int32_t ortho, ipi_inner_report* report,
                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return fail(IPI_EDIMENSION, "empty system");
  int64_t nnz = 0;
  IPI_CUDA_TRY(cudaMemcpyAsync(&nnz, rp_pi + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  // plan the standalone operator like an m = 1 instance (row stats + locality
  // profile -> lanes per row, uniform rows, V-window halo)
  ipi_mdp* view = nullptr;
  int rc = ipi_mdp_create(rp_pi, col_pi, val_pi, b, n, n, 1, 0, gamma, IPI_MODE_MIN, stream, &view);
  if (rc) return rc;
  const ipi_plan pl = view->plan;
  ipi_mdp_destroy(view);
  // the planned K3 operator carries the stepped GMRES's SpMV (uniform rows)
  ipi_op* op = nullptr;
  if (pl.uniform_rows && kind == IPI_KSP_GMRES) {
    rc = ipi_op_create(rp_pi, col_pi, val_pi, n, n, 0, gamma, stream, &op);
    if (rc) return rc;
  }
  ipi_inner_report* d_rep = nullptr;
  if (cudaMalloc(&d_rep, sizeof(ipi_inner_report)) != cudaSuccess) {
    ipi_op_destroy(op);
    return fail(IPI_ECUDA, "cudaMalloc of the inner report failed");
  }
  rc = inner_solve(rp_pi, col_pi, val_pi, n, gamma, b, x, target_2norm, max_it, kind,
                   richardson_scale, pl.lanes_per_row, pl.halo,
                   pl.uniform_rows ? pl.row_len_max : 0, d_rep, st, nullptr, 0, inv_diag,
                   12.0 * (double)nnz + 8.0 * (double)(n + 1), ortho, op, pl.contiguous_rows);
  ipi_op_destroy(op);
  if (rc == IPI_OK && report) {
    cudaError_t e = cudaMemcpyAsync(report, d_rep, sizeof(*report), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(IPI_ECUDA, std::string("inner solve: ") + cudaGetErrorString(e));
  }
  cudaFree(d_rep);
  return rc;
}

int ipi_k4_ring_apply_test(const int32_t* col, const double* val, int64_t n, double gamma,
                           const double* x, double* y, int32_t reps, float* ms, void* stream) {
  return ring_apply_test(col, val, n, gamma, x, y, reps, ms, (cudaStream_t)stream);
}

int ipi_memcpy_sync(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return IPI_OK;
  if (!dst || !src) return fail(IPI_EVALIDATION, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  IPI_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  return IPI_OK;
}

int ipi_k4_trace(int32_t enable, uint64_t* out, int32_t cap) {
  return k4_trace(enable, reinterpret_cast<unsigned long long*>(out), cap);
}

// driver.py:109-209 — the outer loop, natively.  One host sync per outer
// iteration (the residual scalar that drives the stopping tests).
int ipi_solve(ipi_mdp* h, const ipi_opts* o, double* v, int32_t* policy, double* history,
              int32_t hist_cap, ipi_stats* stats, void* stream) {
  if (!h || !o || !v || !stats) return fail(IPI_EVALIDATION, "null argument");
  if (h->state0 != 0 || h->n_local != h->n_global)
    return fail(IPI_EVALIDATION, "ipi_solve drives a whole instance; sharded runs use the rank driver");
  if (!(o->tol > 0.0)) return fail(IPI_EVALIDATION, "tolerance must be > 0");
  if (!(o->alpha > 0.0 && o->alpha < 1.0)) return fail(IPI_EVALIDATION, "alpha must lie in (0, 1)");
  if (o->max_outer < 1 || o->max_inner < 1) return fail(IPI_EVALIDATION, "iteration caps must be >= 1");
  if (hist_cap < 1) return fail(IPI_EVALIDATION, "history capacity must be >= 1");
  if (o->pc_type != IPI_PC_NONE && o->pc_type != IPI_PC_JACOBI)
    return fail(IPI_EVALIDATION, "only the none and jacobi preconditioners run on the device");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_scratch(h);
  if (rc) return rc;
  const int64_t n = h->n_local;
  const auto t_start = std::chrono::steady_clock::now();
  // Phase timing with six reused events (greedy, assembly, inner).  The
  // residual read after every K1 synchronises the stream, so at that point
  // this iteration's greedy phase and the previous iteration's assembly and
  // inner phases are complete and can be accumulated; the events are then
  // recorded again.  The guard destroys them on every exit path.
  struct Events {
    cudaEvent_t e[6] = {};
    Events() {
      for (auto& x : e) cudaEventCreate(&x);
    }
    ~Events() {
      for (auto x : e) if (x) cudaEventDestroy(x);
    }
  } ev;
  cudaEvent_t g0 = ev.e[0], g1 = ev.e[1], a0 = ev.e[2], a1 = ev.e[3], i0 = ev.e[4], i1 = ev.e[5];
  double tg = 0, ta = 0, ti = 0;
  bool pending_phases = false;
  auto elapsed = [](cudaEvent_t x, cudaEvent_t y) {
    float ms = 0;
    cudaEventElapsedTime(&ms, x, y);
    return ms * 1e-3;
  };
  double* host = reinterpret_cast<double*>(h->host_pinned);
  ipi_inner_report* hrep = reinterpret_cast<ipi_inner_report*>(host + 8);
  std::vector<double> hist;
  int64_t inner_total = 0, basis_total = 0;
  int stall = 0;
  int k = 0;
  int status = IPI_CONVERGED;
  double* vcur = v;
  double* vnext = h->xbuf;
  bool pending_report = false;
  // IPI_R0_FROM_TV=0: every inner solve recomputes its initial residual by an SpMV
  static const bool r0_from_tv = !(getenv("IPI_R0_FROM_TV") && getenv("IPI_R0_FROM_TV")[0] == '0');
  while (true) {
    cudaEventRecord(g0, st);
    IPI_CUDA_TRY(cudaMemsetAsync(h->res_bits, 0, sizeof(unsigned long long), st));
    rc = launch_bellman(h, vcur, o->mode, h->pi, h->applied, h->gpi, nullptr, h->res_bits, st);
    if (rc) return rc;
    cudaEventRecord(g1, st);
    IPI_CUDA_TRY(cudaMemcpyAsync(host, h->res_bits, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (pending_report)
      IPI_CUDA_TRY(cudaMemcpyAsync(hrep, h->d_report, sizeof(ipi_inner_report), cudaMemcpyDeviceToHost, st));
    IPI_CUDA_TRY(cudaStreamSynchronize(st));
    tg += elapsed(g0, g1);
    if (pending_phases) {
      ta += elapsed(a0, a1);
      ti += elapsed(i0, i1);
      pending_phases = false;
    }
    if (pending_report) {
      inner_total += hrep->iterations;
      basis_total += hrep->basis_reads;
      pending_report = false;
    }
    const double res = host[0];
    hist.push_back(res);
    if (res <= o->tol) {
      status = IPI_CONVERGED;
      break;
    }
    if (k >= o->max_outer) {
      status = IPI_OUTER_CAP;
      break;
    }
    if (k > 0 && res >= hist[k - 1]) {
      if (++stall >= 50) {  // driver.py:38,146-153
        status = IPI_STALLED;
        break;
      }
    } else {
      stall = 0;
    }
    cudaEventRecord(a0, st);
    rc = gather_policy(h, h->pi, nullptr, h->rp_pi, h->col_pi, h->val_pi, nullptr, nullptr, st);
    if (rc) return rc;
    if (o->pc_type == IPI_PC_JACOBI) {
      if (!h->invd) IPI_CUDA_TRY(cudaMalloc(&h->invd, sizeof(double) * std::max<int64_t>(n, 1)));
      rc = jacobi_inv_diag(h->rp_pi, h->col_pi, h->val_pi, n, h->gamma, h->invd, st);
      if (rc) return rc;
    }
    cudaEventRecord(a1, st);
    double target;
    int cap;
    if (o->ksp_max_it > 0) {
      target = 0.0;
      cap = o->ksp_max_it;
    } else {
      target = o->alpha * res;
      cap = o->max_inner;
    }
    cudaEventRecord(i0, st);
    IPI_CUDA_TRY(cudaMemcpyAsync(vnext, vcur, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    if (!h->op_pi && h->plan.uniform_rows && o->ksp_type == IPI_KSP_GMRES) {
      // planned once per handle: P_pi always lives in the same scratch with the
      // same uniform geometry; only its contents change between iterations
      rc = ipi_op_create(h->rp_pi, h->col_pi, h->val_pi, n, n, 0, h->gamma, stream, &h->op_pi);
      if (rc) return rc;
    }
    rc = inner_solve(h->rp_pi, h->col_pi, h->val_pi, n, h->gamma, h->gpi, vnext, target, cap,
                     o->ksp_type, o->richardson_scale, h->plan.lanes_per_row, h->plan.halo,
                     h->plan.uniform_rows ? h->plan.row_len_max : 0, h->d_report, st, h->kry,
                     h->kry_len, o->pc_type == IPI_PC_JACOBI ? h->invd : nullptr,
                     (12.0 * h->plan.row_len_mean + 8.0) * (double)n,  // P_pi size estimate
                     o->gmres_ortho, h->op_pi, h->plan.contiguous_rows,
                     // K1 has just produced TV = g_pi + gamma P_pi V for this policy and this V
                     r0_from_tv ? h->applied : nullptr);
    if (rc) return rc;
    if (o->ksp_type == IPI_KSP_TFQMR || o->ksp_type == IPI_KSP_BICGSTAB) {
      // these kinds can break down: read the report now (driver.py:189-193)
      IPI_CUDA_TRY(cudaMemcpyAsync(hrep, h->d_report, sizeof(ipi_inner_report), cudaMemcpyDeviceToHost, st));
      IPI_CUDA_TRY(cudaStreamSynchronize(st));
      inner_total += hrep->iterations;
      basis_total += hrep->basis_reads;
      if (hrep->breakdown) {
        // one plain evaluation sweep from the pre-solve V: theta = g_pi + gamma * P_pi v
        rc = launch_spmv(h->rp_pi, h->col_pi, h->val_pi, n, vcur, h->gpi, h->gamma, 3, vnext,
                         h->plan.lanes_per_row, st);
        if (rc) return rc;
        inner_total += 1;
      }
    } else {
      pending_report = true;
    }
    cudaEventRecord(i1, st);
    pending_phases = true;
    std::swap(vcur, vnext);
    ++k;
  }
  if (vcur != v) IPI_CUDA_TRY(cudaMemcpyAsync(v, vcur, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (policy) IPI_CUDA_TRY(cudaMemcpyAsync(policy, h->pi, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  const auto t_end = std::chrono::steady_clock::now();
  const int nh = std::min<int>((int)hist.size(), hist_cap);
  if (history) std::memcpy(history, hist.data(), sizeof(double) * nh);
  stats->status = status;
  stats->outer_iterations = k;
  stats->inner_iterations_total = inner_total;
  stats->wall_time = std::chrono::duration<double>(t_end - t_start).count();
  stats->time_greedy = tg;
  stats->time_assembly = ta;
  stats->time_inner = ti;
  stats->basis_reads_total = basis_total;
  return IPI_OK;
}

}  // extern "C"
