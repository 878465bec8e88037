// bellman.cu — K1: the fused Bellman backup.
//
// Replaces greedy_policy (bellman.py:44-68: one SpMV over the row-stacked
// (n*m) x n matrix, q = g + gamma*PV, first-index argmin/argmax, applied =
// q[pi]) plus the outer residual norm(v - applied, inf) (driver.py:136) with
// ONE pass over the CSR stream.
//
// Mapping: a warp owns one state at a time; its 32 lanes are
// split into 32/G groups of G lanes, one group per (s,a) row, so a state's m
// rows are swept in ceil(m*G/32) steps.  Each lane walks its row with stride
// G and keeps 4 independent (value, column) loads in flight.  Row sums reduce
// over the group with xor shuffles; the per-state argmin is a shuffle merge
// across groups (first index wins ties), so the kernel needs no shared-memory
// q buffer and no block barrier.  Values/columns stream with
// ld.global.nc.L1::no_allocate + L2 evict_first; V is gathered either from a
// shared-memory window [state0+s_lo-halo, state0+s_hi+halo) staged once per
// CTA (locality configs: 10x fewer L1 wavefronts than 32-way divergent LDGs)
// or through the read-only L1 path.  Each CTA owns a contiguous, nnz-balanced
// state range so the window is compact and the L1 working set is local.
#include <cfloat>
#include <climits>

#include "handle.cuh"

namespace ipi {

struct K1Args {
  const int64_t* rp;
  const int32_t* col;
  const double* val;
  const double* cost;
  const double* v;          // full V (n_global)
  const int64_t* bounds;    // per-CTA local state range
  int64_t n_global;
  int64_t state0;
  int32_t m;
  int32_t halo;
  double gamma;
  int32_t maximize;
  int32_t* policy;
  double* applied;
  double* gpi;
  int32_t* lenpi;
  unsigned long long* res_bits;
};

template <int G, bool WIN>
__global__ void __launch_bounds__(kK1Threads) k1_bellman(K1Args a) {
  extern __shared__ double win[];
  __shared__ double red[32];
  const int64_t s_lo = a.bounds[blockIdx.x], s_hi = a.bounds[blockIdx.x + 1];
  int64_t w_lo = 0, w_len = 0;
  if (WIN) {
    int64_t lo = a.state0 + s_lo - a.halo;
    int64_t hi = a.state0 + s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n_global ? a.n_global : hi;
    w_lo = lo;
    w_len = hi > lo ? hi - lo : 0;
    for (int64_t i = threadIdx.x; i < w_len; i += blockDim.x) win[i] = __ldg(a.v + lo + i);
    __syncthreads();
  }
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  constexpr int GPW = 32 / G;
  const int grp = lane / G, gl = lane % G;
  const bool mx = a.maximize != 0;
  const int m = a.m;
  double res = 0.0;

  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint64_t off = (uint64_t)((int64_t)c - w_lo);
      if (off < (uint64_t)w_len) return win[off];
    }
    return __ldg(a.v + c);
  };

  for (int64_t s = s_lo + warp; s < s_hi; s += nwarps) {
    const int64_t row0 = s * (int64_t)m;
    double bq = mx ? -INFINITY : INFINITY;
    int ba = INT_MAX;
    for (int a0 = 0; a0 < m; a0 += GPW) {
      const int act = a0 + grp;
      double acc = 0.0;
      if (act < m) {
        const int64_t p0 = __ldg(a.rp + row0 + act), p1 = __ldg(a.rp + row0 + act + 1);
        for (int64_t p = p0 + gl; p < p1; p += 4 * G) {
          double vv[4];
          int cc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t q = p + (int64_t)u * G;
            if (q < p1) {
              vv[u] = ld_stream(a.val + q, pol);
              cc[u] = ld_stream(a.col + q, pol);
            } else {
              vv[u] = 0.0;
              cc[u] = -1;
            }
          }
          double xx[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) xx[u] = cc[u] >= 0 ? gather(cc[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cc[u] >= 0) acc = add_rn(acc, mul_rn(vv[u], xx[u]));
        }
      }
      acc = group_sum<G>(acc);
      if (act < m) {
        // bellman.py:58: q = stage_cost + gamma * pv (gamma applied first)
        const double q = add_rn(__ldg(a.cost + row0 + act), mul_rn(a.gamma, acc));
        if (better(q, act, bq, ba, mx)) {
          bq = q;
          ba = act;
        }
      }
    }
#pragma unroll
    for (int off = 16; off >= G; off >>= 1) {
      const double oq = __shfl_xor_sync(kFull, bq, off);
      const int oa = __shfl_xor_sync(kFull, ba, off);
      if (better(oq, oa, bq, ba, mx)) {
        bq = oq;
        ba = oa;
      }
    }
    if (ba == INT_MAX) ba = 0;  // unreachable for finite inputs (validated)
    if (lane == 0) {
      a.policy[s] = ba;
      a.applied[s] = bq;
      if (a.gpi) a.gpi[s] = __ldg(a.cost + row0 + ba);
      if (a.lenpi) a.lenpi[s] = (int32_t)(__ldg(a.rp + row0 + ba + 1) - __ldg(a.rp + row0 + ba));
      const double vs = WIN ? gather((int)(a.state0 + s)) : __ldg(a.v + a.state0 + s);
      res = fmax(res, fabs(sub_rn(vs, bq)));
    }
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t = fmax(t, red[w]);
      // |v - Tv| >= 0: IEEE bit patterns of non-negative doubles are ordered,
      // so an integer max is an exact, order-independent max.
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

template <int G>
static void launch_g(const K1Args& a, bool win, int blocks, int smem, cudaStream_t st) {
  if (win)
    k1_bellman<G, true><<<blocks, kK1Threads, smem, st>>>(a);
  else
    k1_bellman<G, false><<<blocks, kK1Threads, 0, st>>>(a);
}

template <int G>
static cudaError_t set_smem_attr(int smem) {
  return cudaFuncSetAttribute(k1_bellman<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem);
}

int k1_set_smem(int lanes, int smem) {
  cudaError_t e = cudaSuccess;
  switch (lanes) {
    case 1: e = set_smem_attr<1>(smem); break;
    case 2: e = set_smem_attr<2>(smem); break;
    case 4: e = set_smem_attr<4>(smem); break;
    case 8: e = set_smem_attr<8>(smem); break;
    case 16: e = set_smem_attr<16>(smem); break;
    default: e = set_smem_attr<32>(smem); break;
  }
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("k1 smem attr: ") + cudaGetErrorString(e));
  return IPI_OK;
}

int launch_bellman(ipi_mdp* h, const double* v_full, int32_t mode, int32_t* policy,
                   double* applied, double* g_pi, int32_t* len_pi,
                   unsigned long long* res_bits, cudaStream_t st) {
  if (h->n_local == 0) return IPI_OK;
  K1Args a;
  a.rp = h->rp;
  a.col = h->col;
  a.val = h->val;
  a.cost = h->cost;
  a.v = v_full;
  a.bounds = h->k1_bounds;
  a.n_global = h->n_global;
  a.state0 = h->state0;
  a.m = h->m;
  a.halo = h->plan.halo;
  a.gamma = h->gamma;
  a.maximize = mode == IPI_MODE_MAX;
  a.policy = policy;
  a.applied = applied;
  a.gpi = g_pi;
  a.lenpi = len_pi;
  a.res_bits = res_bits;
  const bool win = h->plan.halo >= 0;
  const int blocks = h->plan.k1_blocks, smem = h->plan.k1_smem_bytes;
  switch (h->plan.lanes_per_row) {
    case 1: launch_g<1>(a, win, blocks, smem, st); break;
    case 2: launch_g<2>(a, win, blocks, smem, st); break;
    case 4: launch_g<4>(a, win, blocks, smem, st); break;
    case 8: launch_g<8>(a, win, blocks, smem, st); break;
    case 16: launch_g<16>(a, win, blocks, smem, st); break;
    default: launch_g<32>(a, win, blocks, smem, st); break;
  }
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
