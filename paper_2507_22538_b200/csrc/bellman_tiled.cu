// bellman_tiled.cu — K1 for uniform rows whose columns are too spread for a
// resident V window (C5: +-65 536 locality, 10% uniform columns).
//
// The register-deep kernel gathers every V entry from L2 with 32-byte sectors
// per 8-byte value: on a C5 rank block that is ~90 GB of L2->SM traffic per
// backup and the kernel runs L1TEX/L2-bound at ~0.48 of HBM.  Here the shard's
// entries are re-laid out once (plan time) per block of BS states.  Thread i of
// the 1024-thread CTA owns block rows [i*rpl, i*rpl + rpl) (rpl <= 8).  Entries
// whose column lies in the block's near span [cs, ce) are grouped by 8192-column
// tile; per (tile, warp) the warp's entries form one jagged-diagonal segment —
// step k holds entry k of every lane with more than k entries in the tile, in
// lane order — so the warp-wide load of a step is contiguous.  Keys are 16 bits
// (row_in_thread << 13 | column_in_tile); far entries (tile T) keep their full
// column in a side array.  Per block, a split table (tile, warp) and uint16
// per-(tile, thread) counts drive the backup.  Entry bytes drop from 12 to ~10.4
// per nnz.  The backup stages one 64 KB V tile at a time (cp.async, double
// buffered): near gathers become shared-memory loads, only far ones touch L2.
//
// Measured on a C5 rank block (profiles/r01_k1_c5_tiled_jds.txt): 9.6 ms vs
// 8.0 ms for the deep kernel (13.7 ms for the earlier segmented-scan design),
// so the planner still only uses it on request (IPI_K1_TILED).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <vector>

#include "handle.cuh"

namespace ipi {

constexpr int kTileW = 8192;   // columns per V tile (64 KB)
#ifndef IPI_TILED_NW
#define IPI_TILED_NW 32
#endif
#ifndef IPI_TILED_NBUF
#define IPI_TILED_NBUF 2
#endif
constexpr int kTiledNW = IPI_TILED_NW;      // warps per CTA (transform and backup)
constexpr int kTiledNBuf = IPI_TILED_NBUF;  // V tile buffers (1: two CTAs per SM overlap instead)
constexpr int kTiledCTAs = 1024 / (kTiledNW * 32);  // resident CTAs per SM the kernel is built for
constexpr int kTiledNT = kTiledNW * 32;
#ifndef IPI_TILED_UN
#define IPI_TILED_UN 8
#endif
#ifndef IPI_TILED_UF
#define IPI_TILED_UF 4
#endif
#ifndef IPI_TILED_DIAG  // timing diagnostics only: 1 skips the far list, 2 the near tiles
#define IPI_TILED_DIAG 0
#endif
#ifndef IPI_TILED_FAR_SPREAD
#define IPI_TILED_FAR_SPREAD 0  // 1: far list spread over the tile phases — measured slower (10.1 vs 9.6 ms)
#endif
constexpr int kTiledUN = IPI_TILED_UN;  // JDS steps in flight per warp (near tiles)
constexpr int kTiledUF = IPI_TILED_UF;  // (far list: one more dependent load per step)

struct TiledArgs {
  const double* tv;
  const uint16_t* tk;
  const int32_t* tfc;
  const int64_t* far_base;
  const int32_t* meta;  // per block: split table (T + 1) x (NW + 1), then uint16 counts (T + 1) x NT
  const double* cost;
  const double* v;
  int64_t n_local, n_global, state0;
  int32_t m, K, bs, T;  // states per block, max tiles per block
  int32_t rpl;          // rows per thread (consecutive block rows)
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

__host__ __device__ __forceinline__ int64_t tiled_meta_stride(int T) {
  return (int64_t)(T + 1) * (kTiledNW + 1) + (int64_t)(T + 1) * (kTiledNT / 2);
}

__device__ __forceinline__ void block_span(const TiledArgs& a, int64_t b, int64_t& s0, int64_t& s1,
                                           int64_t& cs, int64_t& ce) {
  s0 = b * a.bs;
  s1 = s0 + a.bs < a.n_local ? s0 + a.bs : a.n_local;
  cs = a.state0 + s0 - a.wt;
  cs = cs < 0 ? 0 : cs;
  ce = a.state0 + s1 + a.wt;
  ce = ce > a.n_global ? a.n_global : ce;
}

__device__ __forceinline__ int tile_of(int64_t c, int64_t cs, int64_t ce, int T) {
  return (c >= cs && c < ce) ? (int)((c - cs) / kTileW) : T;
}

// ---- plan-time transform ------------------------------------------------------
// Layout per block of bs states: thread t of the CTA owns rows [t*rpl, t*rpl+rpl)
// of the block.  For every tile (and the far list, tile T) each warp's entries
// form one jagged-diagonal segment: step k holds entry k of every lane that has
// more than k entries in the tile, in lane order, so a warp-wide load at step k
// is contiguous.  A lane's entries in a tile are in (row, column) order; the
// 16-bit key is (row_in_thread << 13 | column_in_tile).
//
// pass 1: per (tile, thread) counts and per (tile, warp) split offsets
__global__ void __launch_bounds__(kTiledNT) tiled_count_kernel(const int32_t* __restrict__ col,
                                                               TiledArgs a, int32_t* meta,
                                                               int64_t* far_count) {
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  uint16_t* cnt = reinterpret_cast<uint16_t*>(tsm_raw);  // [T + 1][NT]
  const int T1 = a.T + 1;
  int* wtot = reinterpret_cast<int*>(tsm_raw + (size_t)T1 * kTiledNT * 2);  // [T + 1][NW]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x;
  int64_t s0, s1, cs, ce;
  block_span(a, b, s0, s1, cs, ce);
  for (int i = tid; i < T1 * kTiledNT; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int nrows = (int)((s1 - s0) * a.m);
  const int q0 = tid * a.rpl, q1 = min(nrows, q0 + a.rpl);
  for (int q = q0; q < q1; ++q) {
    const int64_t e0 = (s0 * a.m + q) * (int64_t)a.K;
    for (int k = 0; k < a.K; ++k) ++cnt[tile_of(col[e0 + k], cs, ce, a.T) * kTiledNT + tid];
  }
  __syncthreads();
  int32_t* mb = meta + b * tiled_meta_stride(a.T);
  uint16_t* cg = reinterpret_cast<uint16_t*>(mb + (int64_t)T1 * (kTiledNW + 1));
  for (int t = 0; t < T1; ++t) {
    const int c = cnt[t * kTiledNT + tid];
    cg[t * kTiledNT + tid] = (uint16_t)c;
    const int s = __reduce_add_sync(kFull, c);
    if (lane == 0) wtot[t * kTiledNW + warp] = s;
  }
  __syncthreads();
  if (tid == 0) {
    int off = 0;
    for (int t = 0; t < T1; ++t) {
      for (int w = 0; w < kTiledNW; ++w) {
        mb[t * (kTiledNW + 1) + w] = off;
        off += wtot[t * kTiledNW + w];
      }
      mb[t * (kTiledNW + 1) + kTiledNW] = off;
    }
    far_count[b] = off - mb[a.T * (kTiledNW + 1)];
  }
}

// pass 2: every thread walks its own rows; entry j of a lane in tile t goes to
// split(t, warp) + sum_l min(cnt_l, j) + #{l < lane : cnt_l > j}.
__global__ void __launch_bounds__(kTiledNT) tiled_scatter_kernel(
    const int32_t* __restrict__ col, const double* __restrict__ val, TiledArgs a, double* tv,
    uint16_t* tk, int32_t* tfc) {
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  const int T1 = a.T + 1;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(tsm_raw);  // [T + 1][NT]
  uint16_t* cur = cnt + (size_t)T1 * kTiledNT;           // [T + 1][NT]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x;
  int64_t s0, s1, cs, ce;
  block_span(a, b, s0, s1, cs, ce);
  const int32_t* mb = a.meta + b * tiled_meta_stride(a.T);
  const uint16_t* cg = reinterpret_cast<const uint16_t*>(mb + (int64_t)T1 * (kTiledNW + 1));
  for (int i = tid; i < T1 * kTiledNT; i += blockDim.x) {
    cnt[i] = cg[i];
    cur[i] = 0;
  }
  __syncthreads();
  const int nrows = (int)((s1 - s0) * a.m);
  const int q0 = tid * a.rpl, q1 = min(nrows, q0 + a.rpl);
  const int64_t ebase = s0 * a.m * (int64_t)a.K;
  const int far0 = mb[a.T * (kTiledNW + 1)];
  const int64_t fbase = a.far_base[b];
  for (int q = q0; q < q1; ++q) {
    const int64_t e0 = (s0 * a.m + q) * (int64_t)a.K;
    for (int k = 0; k < a.K; ++k) {
      const int64_t c = col[e0 + k];
      const int t = tile_of(c, cs, ce, a.T);
      const int j = cur[t * kTiledNT + tid]++;
      const uint16_t* cw = cnt + t * kTiledNT + warp * 32;
      int off = 0;
      for (int l = 0; l < 32; ++l) {
        const int cl = cw[l];
        off += cl < j ? cl : j;
        off += (l < lane && cl > j) ? 1 : 0;
      }
      const int pos = mb[t * (kTiledNW + 1) + warp] + off;
      tv[ebase + pos] = val[e0 + k];
      const uint32_t tag = (uint32_t)(q - q0) << 13;
      if (t < a.T) {
        tk[ebase + pos] = (uint16_t)(tag | (uint32_t)(c - cs - (int64_t)t * kTileW));
      } else {
        tk[ebase + pos] = (uint16_t)tag;
        tfc[fbase + (pos - far0)] = (int32_t)c;
      }
    }
  }
}

// ---- the backup ----------------------------------------------------------------
// Read-only loads with an L2 hint: the entry streams are evict-first, the far
// V gathers evict-last, so the 10% uniform columns find V in L2 more often.
__device__ __forceinline__ uint32_t ldg_u16_hint(const uint16_t* p, uint64_t pol) {
  unsigned short v;
  asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_f64_hint(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ldg_s32_hint(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// One warp walks its jagged-diagonal segment of tile t, kTiledU steps in flight,
// branch-free: lanes past their count re-load the segment's first entry and add
// nothing.  A lane's entries in a tile come in row runs; each run is summed in a
// register and added to the row's thread-private shared-memory slot, so a row's
// sum is tile 0, 1, ... run sums (each sequential in column order), then the
// far run — deterministic, 1e-13 relative to numpy's reduceat like the
// register kernels.
template <bool FAR, int kTiledU>
__device__ __forceinline__ void tiled_segment(const TiledArgs& a, int64_t ebase, int seg, int cnt,
                                              const double* vt, int64_t far_off, double* rs,
                                              uint64_t pol_s, uint64_t pol_v, int k_lo = 0,
                                              int k_hi = INT_MAX) {
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int maxc = min((int)__reduce_max_sync(kFull, (unsigned)cnt), k_hi);
  const uint16_t* __restrict__ tkw = a.tk + ebase + seg;
  const double* __restrict__ tvw = a.tv + ebase + seg;
  const int32_t* __restrict__ fcw = FAR ? a.tfc + far_off : nullptr;
  double* rst = rs + tid;
  int off = k_lo > 0 ? (int)__reduce_add_sync(kFull, (unsigned)min(cnt, k_lo)) : 0;
  int cur = -1;
  double acc = 0.0;
  for (int k0 = k_lo; k0 < maxc; k0 += kTiledU) {
    uint32_t key[kTiledU];
    int32_t fcol[kTiledU];
    double vv[kTiledU];
#pragma unroll
    for (int u = 0; u < kTiledU; ++u) {
      const bool act = k0 + u < cnt;
      const unsigned bal = __ballot_sync(kFull, act);
      const int o = act ? off + __popc(bal & lt) : 0;
      off += __popc(bal);
      key[u] = ldg_u16_hint(tkw + o, pol_s);
      vv[u] = ldg_f64_hint(tvw + o, pol_s);
      if (FAR) fcol[u] = ldg_s32_hint(fcw + o, pol_s);
    }
#pragma unroll
    for (int u = 0; u < kTiledU; ++u) {
      // a run of one row's entries accumulates in a register; the run's sum
      // goes to the row's shared-memory slot when the row tag changes
      const bool act = k0 + u < cnt;
      const double x = FAR ? ldg_f64_hint(a.v + fcol[u], pol_v) : vt[key[u] & 8191u];
      const double p = mul_rn(vv[u], x);
      const int r = act ? (int)(key[u] >> 13) : cur;
      const bool sw = r != cur;
      if (sw && cur >= 0) rst[cur * kTiledNT] = add_rn(rst[cur * kTiledNT], acc);
      acc = sw ? p : (act ? add_rn(acc, p) : acc);
      cur = r;
    }
  }
  if (cur >= 0) rst[cur * kTiledNT] = add_rn(rst[cur * kTiledNT], acc);
}

__global__ void __launch_bounds__(kTiledNT, kTiledCTAs) k1_bellman_tiled(TiledArgs a) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ double red[32];
  double* vt = tsm;                        // 2 x kTileW
  double* rs = tsm + kTiledNBuf * kTileW;  // [rpl][NT] row sums (row q = tid * rpl + r)
  int32_t* sp = reinterpret_cast<int32_t*>(rs + (int64_t)a.rpl * kTiledNT);  // splits of the block
  const int T1 = a.T + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool mx = a.maximize != 0;
  const uint32_t vt_s = (uint32_t)__cvta_generic_to_shared(vt);
  const uint64_t pol_s = policy_evict_first(), pol_v = policy_evict_last();
  double res = 0.0;
  for (int64_t b = blockIdx.x; b < a.nblocks; b += gridDim.x) {
    int64_t s0, s1, cs, ce;
    block_span(a, b, s0, s1, cs, ce);
    const int64_t ebase = s0 * a.m * (int64_t)a.K;
    const int nt = (int)((ce - cs + kTileW - 1) / kTileW);
    __syncthreads();  // previous block fully consumed
    for (int i = tid; i < a.rpl * kTiledNT; i += blockDim.x) rs[i] = 0.0;
    const int32_t* mb = a.meta + b * tiled_meta_stride(a.T);
    const uint16_t* cg = reinterpret_cast<const uint16_t*>(mb + (int64_t)T1 * (kTiledNW + 1));
    for (int i = tid; i < T1 * (kTiledNW + 1); i += blockDim.x) sp[i] = mb[i];
    auto issue_tile = [&](int t) {
      const int64_t c0 = cs + (int64_t)t * kTileW;
      const int64_t len = ce - c0 < kTileW ? ce - c0 : kTileW;
      const uint32_t dst = vt_s + (uint32_t)((t % kTiledNBuf) * kTileW * 8);
      for (int64_t i = tid; i < len; i += blockDim.x) cp_async8(dst + (uint32_t)(8 * i), a.v + c0 + i);
      cp_async_commit();
    };
    if (nt > 0) issue_tile(0);
    __syncthreads();
    // The far list is spread over the tile phases (chunk t of its steps in phase
    // t, before or after the near segment by warp parity) so its L2/DRAM
    // gathers overlap the near tiles instead of forming a tail.
    const int f_lo = sp[a.T * (kTiledNW + 1) + warp];
    const int far0 = sp[a.T * (kTiledNW + 1)];
    const int fcnt = IPI_TILED_DIAG == 1 ? 0 : __ldg(cg + a.T * kTiledNT + tid);
    const int64_t foff = a.far_base[b] + (f_lo - far0);
    const int fmx = (int)__reduce_max_sync(kFull, (unsigned)fcnt);
    const int fchunk = IPI_TILED_FAR_SPREAD && nt > 0 ? ((fmx + nt - 1) / nt + kTiledUF - 1) / kTiledUF * kTiledUF : 0;
    for (int t = 0; t < nt; ++t) {
      const int c = IPI_TILED_DIAG == 2 ? 0 : __ldg(cg + t * kTiledNT + tid);
      if (kTiledNBuf == 2 && t + 1 < nt) {
        issue_tile(t + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();  // tile t staged by every thread
      const bool far_first = (warp & 1) == 0;
      if (fchunk && far_first)
        tiled_segment<true, kTiledUF>(a, ebase, f_lo, fcnt, nullptr, foff, rs, pol_s, pol_v, t * fchunk, (t + 1) * fchunk);
      tiled_segment<false, kTiledUN>(a, ebase, sp[t * (kTiledNW + 1) + warp], c, vt + (t % kTiledNBuf) * kTileW, 0, rs, pol_s, pol_v);
      if (fchunk && !far_first)
        tiled_segment<true, kTiledUF>(a, ebase, f_lo, fcnt, nullptr, foff, rs, pol_s, pol_v, t * fchunk, (t + 1) * fchunk);
      __syncthreads();  // tile t consumed before its buffer is refilled
      if (kTiledNBuf == 1 && t + 1 < nt) issue_tile(t + 1);
    }
    if (!fchunk) tiled_segment<true, kTiledUF>(a, ebase, f_lo, fcnt, nullptr, foff, rs, pol_s, pol_v);
    __syncthreads();
    // first-index argmin / argmax over each state's m rows (bellman.py:58-62)
    for (int64_t s = s0 + warp; s < s1; s += kTiledNW) {
      const int64_t row0 = s * a.m;
      double bq = mx ? -INFINITY : INFINITY;
      int ba = INT_MAX;
      for (int act = lane; act < a.m; act += 32) {
        const int q = (int)((s - s0) * a.m + act);
        const double q_sa = add_rn(__ldg(a.cost + row0 + act), mul_rn(a.gamma, rs[(q % a.rpl) * kTiledNT + q / a.rpl]));
        if (better(q_sa, act, bq, ba, mx)) {
          bq = q_sa;
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
  a.rpl = (h->tl_bs * h->m + kTiledNT - 1) / kTiledNT;
  a.wt = h->tl_wt;
  a.nblocks = h->tl_nblocks;
  a.gamma = h->gamma;
  return a;
}

int k1_tiled_smem(const ipi_mdp* h) {
  const int rpl = (h->tl_bs * h->m + kTiledNT - 1) / kTiledNT;
  return (kTiledNBuf * kTileW + rpl * kTiledNT) * 8 + (h->tl_T + 1) * (kTiledNW + 1) * 4;
}

// Build the tiled layout for h (uniform rows, m * bs <= 8192).  Returns IPI_OK
// with h->tl_nblocks == 0 when it does not apply or memory is short.
int k1_tiled_build(ipi_mdp* h, int64_t wt, cudaStream_t st) {
  const int K = h->plan.row_len_max, m = h->m;
  if (!h->plan.uniform_rows || K <= 0 || m > 8 * kTiledNT || h->n_local <= 0) return IPI_OK;
  int bs = 8 * kTiledNT / m;  // rpl <= 8
  bs = bs > 512 ? 512 : bs;
  const int rpl = (bs * m + kTiledNT - 1) / kTiledNT;  // <= 8: a 3-bit row tag
  if (rpl * K >= 65536) return IPI_OK;                  // uint16 per-(tile, thread) counts
  const int64_t nblocks = (h->n_local + bs - 1) / bs;
  const int T = (int)((bs + 2 * wt + kTileW - 1) / kTileW);
  if (T > 48) return IPI_OK;
  const int64_t nnz = h->plan.nnz;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double need = 10.0 * nnz + 4.0 * nnz * 0.25 + 1e8;
  if (need > 0.9 * (double)fr) return IPI_OK;
  const int cnt_smem = (T + 1) * kTiledNT * 2 + (T + 1) * kTiledNW * 4;
  const int sct_smem = (T + 1) * kTiledNT * 4;
  if (raise_smem_limit(tiled_count_kernel, cnt_smem) != cudaSuccess ||
      raise_smem_limit(tiled_scatter_kernel, sct_smem) != cudaSuccess) {
    cudaGetLastError();
    return IPI_OK;
  }
  h->tl_bs = bs;
  h->tl_T = T;
  h->tl_wt = wt;
  IPI_CUDA_TRY(cudaMalloc(&h->tl_val, sizeof(double) * nnz));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_key, sizeof(uint16_t) * nnz));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_meta, sizeof(int32_t) * nblocks * tiled_meta_stride(T)));
  IPI_CUDA_TRY(cudaMalloc(&h->tl_farbase, sizeof(int64_t) * (nblocks + 1)));
  h->tl_nblocks = nblocks;
  TiledArgs a = tiled_args(h);
  tiled_count_kernel<<<(int)nblocks, kTiledNT, cnt_smem, st>>>(h->col, a, h->tl_meta, h->tl_farbase);
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
  tiled_scatter_kernel<<<(int)nblocks, kTiledNT, sct_smem, st>>>(h->col, h->val, a, h->tl_val,
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
  const int grid = (int)std::min<int64_t>(h->tl_nblocks, (int64_t)h->num_sms * kTiledCTAs);
  k1_bellman_tiled<<<grid, kTiledNT, k1_tiled_smem(h), st>>>(a);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
