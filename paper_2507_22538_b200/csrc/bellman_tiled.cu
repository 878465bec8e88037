// bellman_tiled.cu — K1 for uniform rows whose columns are too spread for a
// resident V window (C5: +-65 536 locality, 10% uniform columns).
//
// The register-deep kernel gathers every V entry from L2 with 32-byte sectors
// per 8-byte value: on a C5 rank block that is ~90 GB of L2->SM traffic per
// backup and the kernel runs L1TEX/L2-bound at ~0.48 of HBM.  Here the shard's
// entries are re-laid out once (plan time) per block of BS states: entries
// whose column lies in the block's near span [cs, ce) are stable-sorted by
// TW-column tile (the tile index is monotone along a sorted row, so a
// per-warp counting sort does it) and stored with a packed key
// (row_in_block << 13 | column_in_tile); the far entries follow in row order
// with their full columns in a side array.  Per (tile, warp) split points give
// every warp its own row range inside every tile, so row partial sums go to
// shared memory without atomics (deterministic).  The backup then stages one
// TW-double V tile at a time (cp.async, double-buffered): near gathers become
// shared-memory loads and only the far ones touch L2.
//
// Row sum order: per row, tile 0, 1, ... partials (segmented shuffle scans over
// 32-entry chunks, in chunk order), then the far partial — deterministic, 1e-13
// relative to numpy's reduceat like the register kernels.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <vector>

#include "handle.cuh"

namespace ipi {

constexpr int kTileW = 8192;  // columns per V tile (64 KB)
constexpr int kTiledNW = 32;  // warps per CTA (transform and backup)

struct TiledArgs {
  const double* tv;
  const uint32_t* tk;
  const int32_t* tfc;
  const int64_t* far_base;
  const int32_t* meta;  // per block: (T + 1) x (NW + 1) split offsets, relative to the block's entries
  const double* cost;
  const double* v;
  int64_t n_local, n_global, state0;
  int32_t m, K, bs, T;  // states per block, max tiles per block
  int64_t wt;           // near half-width
  int64_t nblocks;
  double gamma;
  int32_t maximize;
  int32_t* policy;
  double* applied;
  double* gpi;
  int32_t* lenpi;
  unsigned long long* res_bits;
};

__device__ __forceinline__ void block_span(const TiledArgs& a, int64_t b, int64_t& s0, int64_t& s1,
                                           int64_t& cs, int64_t& ce) {
  s0 = b * a.bs;
  s1 = s0 + a.bs < a.n_local ? s0 + a.bs : a.n_local;
  cs = a.state0 + s0 - a.wt;
  cs = cs < 0 ? 0 : cs;
  ce = a.state0 + s1 + a.wt;
  ce = ce > a.n_global ? a.n_global : ce;
}

// ---- plan-time transform ------------------------------------------------------
// pass 1: per (warp, tile) counts -> split offsets (meta) and the block's far count
__global__ void __launch_bounds__(kTiledNW * 32) tiled_count_kernel(const int32_t* __restrict__ col,
                                                                    TiledArgs a, int32_t* meta,
                                                                    int64_t* far_count) {
  extern __shared__ int tcnt[];  // [NW][T + 1]
  const int T1 = a.T + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = blockIdx.x;
  int64_t s0, s1, cs, ce;
  block_span(a, b, s0, s1, cs, ce);
  for (int i = threadIdx.x; i < kTiledNW * T1; i += blockDim.x) tcnt[i] = 0;
  __syncthreads();
  const int64_t r0 = s0 * a.m, nr = (s1 - s0) * a.m;
  const int64_t w0 = r0 + nr * warp / kTiledNW, w1 = r0 + nr * (warp + 1) / kTiledNW;
  for (int64_t e = w0 * a.K + lane; e < w1 * a.K; e += 32) {
    const int64_t c = col[e];
    const int t = (c >= cs && c < ce) ? (int)((c - cs) / kTileW) : a.T;
    atomicAdd(&tcnt[warp * T1 + t], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* mb = meta + b * (int64_t)T1 * (kTiledNW + 1);
    int off = 0;
    for (int t = 0; t < T1; ++t) {
      for (int w = 0; w < kTiledNW; ++w) {
        mb[t * (kTiledNW + 1) + w] = off;
        off += tcnt[w * T1 + t];
      }
      mb[t * (kTiledNW + 1) + kTiledNW] = off;
    }
    int far = 0;
    for (int w = 0; w < kTiledNW; ++w) far += tcnt[w * T1 + a.T];
    far_count[b] = far;
  }
}

// pass 2: stable scatter in (tile, warp, row, column) order
__global__ void __launch_bounds__(kTiledNW * 32) tiled_scatter_kernel(
    const int32_t* __restrict__ col, const double* __restrict__ val, TiledArgs a, double* tv,
    uint32_t* tk, int32_t* tfc) {
  extern __shared__ int tcur[];  // [NW][T + 1] cursors
  const int T1 = a.T + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = blockIdx.x;
  int64_t s0, s1, cs, ce;
  block_span(a, b, s0, s1, cs, ce);
  const int32_t* mb = a.meta + b * (int64_t)T1 * (kTiledNW + 1);
  for (int t = lane; t < T1; t += 32) tcur[warp * T1 + t] = mb[t * (kTiledNW + 1) + warp];
  __syncwarp();
  const int64_t r0 = s0 * a.m, nr = (s1 - s0) * a.m;
  const int64_t w0 = r0 + nr * warp / kTiledNW, w1 = r0 + nr * (warp + 1) / kTiledNW;
  const int64_t ebase = r0 * a.K;       // the block's first entry
  const int far0 = mb[a.T * (kTiledNW + 1)];
  const int64_t fbase = a.far_base[b];
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t r = w0; r < w1; ++r) {
    const uint32_t rib = (uint32_t)(r - r0);
    for (int64_t e0 = r * a.K; e0 < (r + 1) * a.K; e0 += 32) {
      const int64_t e = e0 + lane;
      const bool act = e < (r + 1) * a.K;
      const unsigned am = __ballot_sync(kFull, act);
      if (!act) continue;
      const int64_t c = col[e];
      const bool near = c >= cs && c < ce;
      const int t = near ? (int)((c - cs) / kTileW) : a.T;
      const unsigned peers = __match_any_sync(am, t);
      const int rank = __popc(peers & lt);
      const int pos = tcur[warp * T1 + t] + rank;
      tv[ebase + pos] = val[e];
      if (near) {
        tk[ebase + pos] = (rib << 13) | (uint32_t)(c - cs - (int64_t)t * kTileW);
      } else {
        tk[ebase + pos] = rib << 13;
        tfc[fbase + (pos - far0)] = (int32_t)c;
      }
      __syncwarp(am);
      if (rank == 0) tcur[warp * T1 + t] += __popc(peers);
      __syncwarp(am);
    }
  }
}

// ---- the backup ----------------------------------------------------------------
template <bool FAR>
__device__ __forceinline__ void tiled_segment(const TiledArgs& a, int64_t ebase, int e_lo, int e_hi,
                                              const double* vt, int64_t far_off, double* acc) {
  constexpr int U = 8;  // 32-entry chunks in flight per warp (loads issued before any reduction)
  const int lane = threadIdx.x & 31;
  for (int c0 = e_lo; c0 < e_hi; c0 += 32 * U) {
    uint32_t key[U];
    double vv[U], x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = c0 + 32 * u + lane;
      key[u] = 0xffffffffu;
      vv[u] = 0.0;
      if (e < e_hi) {
        key[u] = __ldg(a.tk + ebase + e);
        vv[u] = __ldg(a.tv + ebase + e);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = c0 + 32 * u + lane;
      x[u] = 0.0;
      if (e < e_hi) x[u] = FAR ? __ldg(a.v + __ldg(a.tfc + far_off + (e - e_lo))) : vt[key[u] & 8191u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // chunks in order: deterministic row partials
      const int e = c0 + 32 * u + lane;
      const bool act = e < e_hi;
      double p = act ? mul_rn(vv[u], x[u]) : 0.0;
      const uint32_t row = key[u] >> 13;
      // segmented inclusive scan over the chunk (rows are sorted within it)
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(kFull, p, d);
        const uint32_t orow = __shfl_up_sync(kFull, row, d);
        if (lane >= d && orow == row) p = add_rn(o, p);
      }
      const uint32_t nrow = __shfl_down_sync(kFull, row, 1);
      if (act && (lane == 31 || e + 1 >= e_hi || nrow != row)) acc[row] = add_rn(acc[row], p);
    }
  }
}

__global__ void __launch_bounds__(kTiledNW * 32, 1) k1_bellman_tiled(TiledArgs a) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ double red[32];
  double* vt = tsm;                       // 2 x kTileW
  double* acc = tsm + 2 * kTileW;         // bs * m row sums
  int32_t* sp = reinterpret_cast<int32_t*>(acc + (int64_t)a.bs * a.m);  // splits of the block
  const int T1 = a.T + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool mx = a.maximize != 0;
  const uint32_t vt_s = (uint32_t)__cvta_generic_to_shared(vt);
  double res = 0.0;
  for (int64_t b = blockIdx.x; b < a.nblocks; b += gridDim.x) {
    int64_t s0, s1, cs, ce;
    block_span(a, b, s0, s1, cs, ce);
    const int nrows = (int)((s1 - s0) * a.m);
    const int64_t ebase = s0 * a.m * (int64_t)a.K;
    const int nt = (int)((ce - cs + kTileW - 1) / kTileW);
    __syncthreads();  // previous block fully consumed
    for (int i = threadIdx.x; i < nrows; i += blockDim.x) acc[i] = 0.0;
    const int32_t* mb = a.meta + b * (int64_t)T1 * (kTiledNW + 1);
    for (int i = threadIdx.x; i < T1 * (kTiledNW + 1); i += blockDim.x) sp[i] = mb[i];
    auto issue_tile = [&](int t) {
      const int64_t c0 = cs + (int64_t)t * kTileW;
      const int64_t len = ce - c0 < kTileW ? ce - c0 : kTileW;
      const uint32_t dst = vt_s + (uint32_t)((t & 1) * kTileW * 8);
      for (int64_t i = threadIdx.x; i < len; i += blockDim.x) cp_async8(dst + (uint32_t)(8 * i), a.v + c0 + i);
      cp_async_commit();
    };
    if (nt > 0) issue_tile(0);
    __syncthreads();
    for (int t = 0; t < nt; ++t) {
      if (t + 1 < nt) {
        issue_tile(t + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();  // tile t staged by every thread
      tiled_segment<false>(a, ebase, sp[t * (kTiledNW + 1) + warp], sp[t * (kTiledNW + 1) + warp + 1],
                           vt + (t & 1) * kTileW, 0, acc);
      __syncthreads();  // tile t consumed before its buffer is refilled
    }
    const int f_lo = sp[a.T * (kTiledNW + 1) + warp], f_hi = sp[a.T * (kTiledNW + 1) + warp + 1];
    const int far0 = sp[a.T * (kTiledNW + 1)];
    tiled_segment<true>(a, ebase, f_lo, f_hi, nullptr, a.far_base[b] + (f_lo - far0), acc);
    __syncthreads();
    // first-index argmin / argmax over each state's m rows (bellman.py:58-62)
    for (int64_t s = s0 + warp; s < s1; s += kTiledNW) {
      const int64_t row0 = s * a.m;
      double bq = mx ? -INFINITY : INFINITY;
      int ba = INT_MAX;
      for (int act = lane; act < a.m; act += 32) {
        const double q = add_rn(__ldg(a.cost + row0 + act), mul_rn(a.gamma, acc[(s - s0) * a.m + act]));
        if (better(q, act, bq, ba, mx)) {
          bq = q;
          ba = act;
        }
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double oq = __shfl_xor_sync(kFull, bq, off);
        const int oa = __shfl_xor_sync(kFull, ba, off);
        if (better(oq, oa, bq, ba, mx)) {
          bq = oq;
          ba = oa;
        }
      }
      if (lane == 0) {
        const int pa = ba == INT_MAX ? 0 : ba;
        a.policy[s] = pa;
        a.applied[s] = bq;
        if (a.gpi) a.gpi[s] = __ldg(a.cost + row0 + pa);
        if (a.lenpi) a.lenpi[s] = a.K;
        res = fmax(res, fabs(sub_rn(__ldg(a.v + a.state0 + s), bq)));
      }
    }
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kTiledNW; ++w) t = fmax(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

static TiledArgs tiled_args(const ipi_mdp* h) {
  TiledArgs a{};
  a.tv = h->tl_val;
  a.tk = h->tl_key;
  a.tfc = h->tl_farcol;
  a.far_base = h->tl_farbase;
  a.meta = h->tl_meta;
  a.cost = h->cost;
  a.n_local = h->n_local;
  a.n_global = h->n_global;
  a.state0 = h->state0;
  a.m = h->m;
  a.K = h->plan.row_len_max;
  a.bs = h->tl_bs;
  a.T = h->tl_T;
  a.wt = h->tl_wt;
  a.nblocks = h->tl_nblocks;
  a.gamma = h->gamma;
  return a;
}

int k1_tiled_smem(const ipi_mdp* h) {
  return (2 * kTileW + h->tl_bs * h->m) * 8 + (h->tl_T + 1) * (kTiledNW + 1) * 4;
}

// Build the tiled layout for h (uniform rows, m * bs <= 8192).  Returns IPI_OK
// with h->tl_nblocks == 0 when it does not apply or memory is short.
int k1_tiled_build(ipi_mdp* h, int64_t wt, cudaStream_t st) {
  const int K = h->plan.row_len_max, m = h->m;
  if (!h->plan.uniform_rows || K <= 0 || m > 8192 || h->n_local <= 0) return IPI_OK;
  int bs = 8192 / m;
  bs = bs > 512 ? 512 : bs;
  const int64_t nblocks = (h->n_local + bs - 1) / bs;
  const int T = (int)((bs + 2 * wt + kTileW - 1) / kTileW);
  if (T > 64) return IPI_OK;
  const int64_t nnz = h->plan.nnz;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double need = 12.0 * nnz + 4.0 * nnz * 0.25 + 1e8;
  if (need > 0.9 * (double)fr) return IPI_OK;
  h->tl_bs = bs;
  h->tl_T = T;
  h->tl_wt = wt;
  IPI_CUDA_TRY(cudaMalloc(&h->tl_val, sizeof(double) * nnz));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_key, sizeof(uint32_t) * nnz));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_meta, sizeof(int32_t) * nblocks * (T + 1) * (kTiledNW + 1)));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_farbase, sizeof(int64_t) * (nblocks + 1)));
  h->tl_nblocks = nblocks;
  TiledArgs a = tiled_args(h);
  const int cnt_smem = kTiledNW * (T + 1) * 4;
  tiled_count_kernel<<<(int)nblocks, kTiledNW * 32, cnt_smem, st>>>(h->col, a, h->tl_meta, h->tl_farbase);
  IPI_LAUNCH_CHECK();
  // exclusive prefix of the per-block far counts (host: nblocks values)
  std::vector<int64_t> fc(nblocks);
  IPI_CUDA_TRY(cudaMemcpyAsync(fc.data(), h->tl_farbase, sizeof(int64_t) * nblocks, cudaMemcpyDeviceToHost, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int64_t> fb(nblocks + 1);
  fb[0] = 0;
  for (int64_t b = 0; b < nblocks; ++b) fb[b + 1] = fb[b] + fc[b];
  IPI_CUDA_TRY(cudaMemcpyAsync(h->tl_farbase, fb.data(), sizeof(int64_t) * (nblocks + 1), cudaMemcpyHostToDevice, st));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_farcol, sizeof(int32_t) * (fb[nblocks] > 0 ? fb[nblocks] : 1)));
  a = tiled_args(h);
  tiled_scatter_kernel<<<(int)nblocks, kTiledNW * 32, cnt_smem, st>>>(h->col, h->val, a, h->tl_val,
                                                                       h->tl_key, h->tl_farcol);
  IPI_LAUNCH_CHECK();
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  const int smem = k1_tiled_smem(h);
  if (smem > 227 * 1024 - 1024 || raise_smem_limit(k1_bellman_tiled, smem) != cudaSuccess) {
    cudaGetLastError();
    k1_tiled_free(h);
  }
  return IPI_OK;
}

void k1_tiled_free(ipi_mdp* h) {
  cudaFree(h->tl_val);
  cudaFree(h->tl_key);
  cudaFree(h->tl_meta);
  cudaFree(h->tl_farbase);
  cudaFree(h->tl_farcol);
  h->tl_val = nullptr;
  h->tl_key = nullptr;
  h->tl_meta = nullptr;
  h->tl_farbase = nullptr;
  h->tl_farcol = nullptr;
  h->tl_nblocks = 0;
}

int launch_bellman_tiled(ipi_mdp* h, const double* v_full, int32_t mode, int32_t* policy,
                         double* applied, double* g_pi, int32_t* len_pi,
                         unsigned long long* res_bits, cudaStream_t st) {
  TiledArgs a = tiled_args(h);
  a.v = v_full;
  a.maximize = mode == IPI_MODE_MAX;
  a.policy = policy;
  a.applied = applied;
  a.gpi = g_pi;
  a.lenpi = len_pi;
  a.res_bits = res_bits;
  const int grid = (int)std::min<int64_t>(h->tl_nblocks, (int64_t)h->num_sms);
  k1_bellman_tiled<<<grid, kTiledNW * 32, k1_tiled_smem(h), st>>>(a);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
