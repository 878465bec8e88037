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
#include <cstdlib>

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
  int32_t win_async;   // uniform ring: stage the V window with cp.async
  int32_t interleave;  // uniform ring: warps take interleaved states
  int32_t rotate;      // uniform ring: per-CTA rotated start in the warp's state sequence
  unsigned long long* trace;  // diagnostics: per-CTA (smid, t_start, t_end) or nullptr
  int32_t contig;             // generic rows: columns consecutive within each row (plan)
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// CONTIG: every row's columns are consecutive (plan.contiguous_rows, C4's
// banded rows): entry q's column is c0 + (q - p0), so the column stream is not
// read (8 instead of 12 bytes per entry).
template <int G, bool WIN, bool CONTIG = false, int UL = (G == 32 ? 8 : 4)>
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
    window_load8(win, a.v, lo, w_len);
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
        int c0 = 0;
        if constexpr (CONTIG) c0 = p1 > p0 ? __ldg(a.col + p0) : 0;
        // long rows (G = 32, e.g. C4's ~570-entry rows): 8 loads in flight per lane
        constexpr int U = UL;
        for (int64_t p = p0 + gl; p < p1; p += U * G) {
          double vv[U];
          int cc[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t q = p + (int64_t)u * G;
            if (q < p1) {
              vv[u] = ld_stream(a.val + q, pol);
              if constexpr (CONTIG) cc[u] = c0 + (int)(q - p0);
              else cc[u] = ld_stream(a.col + q, pol);
            } else {
              vv[u] = 0.0;
              cc[u] = -1;
            }
          }
          double xx[U];
#pragma unroll
          for (int u = 0; u < U; ++u) xx[u] = cc[u] >= 0 ? gather(cc[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u)
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
      res = res_max(res, fabs(sub_rn(vs, bq)));
    }
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t = res_max(t, red[w]);
      // |v - Tv| >= 0: IEEE bit patterns of non-negative doubles are ordered,
      // so an integer max is an exact, order-independent max.
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

// ---------------------------------------------------------------------------
// Uniform-row fast path (every row has the same even length K; rows start at
// r*K so value pairs are 16-byte aligned).  Each lane owns P value pairs per
// row (16-byte ld.v2.f64 + 8-byte ld.v2.s32); the warp's (state, row-step)
// batches are flattened into one stream and software-pipelined: batch b+1's
// loads are issued before batch b's gathers/shuffles, so every warp keeps two
// batches of CSR bytes in flight (Little's law: ~52 KB/SM at 6.4 TB/s).
// ---------------------------------------------------------------------------
template <int G, int P, bool WIN>
__global__ void __launch_bounds__(kK1Threads) k1_bellman_uniform(K1Args a, int K) {
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
    window_load8(win, a.v, lo, w_len);
  }
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  constexpr int GPW = 32 / G;
  const int grp = lane / G, gl = lane % G;
  const bool mx = a.maximize != 0;
  const int m = a.m;
  const int nit = (m + GPW - 1) / GPW;
  const int pairs = K >> 1;
  double res = 0.0;

  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint64_t off = (uint64_t)((int64_t)c - w_lo);
      if (off < (uint64_t)w_len) return win[off];
    }
    return __ldg(a.v + c);
  };
  auto load = [&](int64_t s, int it, Batch<P>& b) {
    const int act = it * GPW + grp;
    const int64_t base = (s * (int64_t)m + act) * (int64_t)K;
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const int j = gl + G * t;
      if (act < m && j < pairs) {
        b.v[t] = ld_stream_v2(a.val + base + 2 * j, pol);
        b.c[t] = ld_stream_v2(a.col + base + 2 * j, pol);
      } else {
        b.v[t] = make_double2(0.0, 0.0);
        b.c[t] = make_int2(-1, -1);
      }
    }
  };

  int64_t s = s_lo + warp;
  if (s < s_hi) {
    int it = 0;
    Batch<P> cur, nxt;
    load(s, 0, cur);
    double bq = mx ? -INFINITY : INFINITY;
    int ba = INT_MAX;
    while (true) {
      int it_n = it + 1;
      int64_t s_n = s;
      if (it_n == nit) {
        it_n = 0;
        s_n = s + nwarps;
      }
      const bool has_next = s_n < s_hi;
      if (has_next) load(s_n, it_n, nxt);
      // gathers + row sum for the current batch
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < P; ++t) {
        if (cur.c[t].x >= 0) {
          const double x0 = gather(cur.c[t].x), x1 = gather(cur.c[t].y);
          acc = add_rn(acc, mul_rn(cur.v[t].x, x0));
          acc = add_rn(acc, mul_rn(cur.v[t].y, x1));
        }
      }
      acc = group_sum<G>(acc);
      const int act = it * GPW + grp;
      const int64_t row0 = s * (int64_t)m;
      if (act < m) {
        const double q = add_rn(__ldg(a.cost + row0 + act), mul_rn(a.gamma, acc));
        if (better(q, act, bq, ba, mx)) {
          bq = q;
          ba = act;
        }
      }
      if (it == nit - 1) {
#pragma unroll
        for (int off = 16; off >= G; off >>= 1) {
          const double oq = __shfl_xor_sync(kFull, bq, off);
          const int oa = __shfl_xor_sync(kFull, ba, off);
          if (better(oq, oa, bq, ba, mx)) {
            bq = oq;
            ba = oa;
          }
        }
        if (ba == INT_MAX) ba = 0;
        if (lane == 0) {
          a.policy[s] = ba;
          a.applied[s] = bq;
          if (a.gpi) a.gpi[s] = __ldg(a.cost + row0 + ba);
          if (a.lenpi) a.lenpi[s] = K;
          const double vs = WIN ? gather((int)(a.state0 + s)) : __ldg(a.v + a.state0 + s);
          res = res_max(res, fabs(sub_rn(vs, bq)));
        }
        bq = mx ? -INFINITY : INFINITY;
        ba = INT_MAX;
      }
      if (!has_next) break;
      cur = nxt;
      s = s_n;
      it = it_n;
    }
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t = res_max(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

// ---------------------------------------------------------------------------
// Flat-rows fast path for very short uniform rows (K <= 4, e.g. C3's bilinear
// rows): one (s,a) row per lane over a warp-contiguous row range that ignores
// state boundaries, so no lane idles when 32 is not a multiple of m (C3:
// m = 21).  The per-state first-index argmin is a segmented shuffle scan keyed
// by state id, with the partial best of a state that straddles two batches
// carried in registers.  Loads of batch b+1 are issued before batch b is
// reduced.
// ---------------------------------------------------------------------------
struct FlatBatch {
  double2 v0, v1;
  int2 c0, c1;
  double g;
};

template <bool WIN>
__global__ void __launch_bounds__(kK1Threads, 2) k1_bellman_flat(K1Args a, int K) {
  extern __shared__ double win[];
  __shared__ double red[32];
  const int64_t s_lo = a.bounds[blockIdx.x], s_hi = a.bounds[blockIdx.x + 1];
  int w_lo = 0;
  uint32_t w_len = 0;
  if (WIN) {
    int64_t lo = a.state0 + s_lo - a.halo;
    int64_t hi = a.state0 + s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n_global ? a.n_global : hi;
    w_lo = (int)lo;
    w_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
    window_load8(win, a.v, lo, w_len);
  }
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const bool mx = a.maximize != 0;
  const int m = a.m;
  double res = 0.0;
  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) return win[off];
    }
    return __ldg(a.v + c);
  };
  // this warp's contiguous state range -> row range
  const int64_t ns = s_hi - s_lo;
  const int64_t ws0 = s_lo + ns * warp / nwarps, ws1 = s_lo + ns * (warp + 1) / nwarps;
  const int64_t r_beg = ws0 * m, r_end = ws1 * m;
  const int pairs = K >> 1;
  auto load = [&](int64_t base, FlatBatch& b) {
    const int64_t r = base + lane;
    const bool ok = r < r_end;
    const double* vp = a.val + r * K;
    const int* cp = a.col + r * K;
    b.v0 = ok ? ld_stream_v2(vp, pol) : make_double2(0.0, 0.0);
    b.c0 = ok ? ld_stream_v2(cp, pol) : make_int2(-1, -1);
    const bool ok1 = ok && pairs > 1;
    b.v1 = ok1 ? ld_stream_v2(vp + 2, pol) : make_double2(0.0, 0.0);
    b.c1 = ok1 ? ld_stream_v2(cp + 2, pol) : make_int2(-1, -1);
    b.g = ok ? __ldg(a.cost + r) : 0.0;
  };
  double carry_q = mx ? -INFINITY : INFINITY;
  int carry_a = INT_MAX;
  int64_t carry_s = -1;
  if (r_beg < r_end) {
    FlatBatch cur, nxt;
    load(r_beg, cur);
    for (int64_t base = r_beg; base < r_end; base += 32) {
      const bool has_next = base + 32 < r_end;
      if (has_next) load(base + 32, nxt);
      const int64_t r = base + lane;
      const bool ok = r < r_end;
      double acc = 0.0;
      if (ok) {  // reduceat order: p0 + (((0 + p1) + p2) + p3)
        acc = add_rn(0.0, mul_rn(cur.v0.y, gather(cur.c0.y)));
        if (pairs > 1) {
          acc = add_rn(acc, mul_rn(cur.v1.x, gather(cur.c1.x)));
          acc = add_rn(acc, mul_rn(cur.v1.y, gather(cur.c1.y)));
        }
        acc = add_rn(mul_rn(cur.v0.x, gather(cur.c0.x)), acc);
      }
      // state id and action of this lane's row
      const int64_t sb = base / m;
      const int rem = (int)(base - sb * m);
      const int t = rem + lane;
      const int ds = t / m;
      int64_t sid = ok ? sb + ds : INT64_MAX;
      int act = t - ds * m;
      double q = ok ? add_rn(cur.g, mul_rn(a.gamma, acc)) : (mx ? -INFINITY : INFINITY);
      int aa = ok ? act : INT_MAX;
      // merge the carried partial of a state begun in the previous batch
      if (lane == 0 && sid == carry_s && better(carry_q, carry_a, q, aa, mx)) {
        q = carry_q;
        aa = carry_a;
      }
      // segmented inclusive scan (first-index argmin) by state id
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double oq = __shfl_up_sync(kFull, q, off);
        const int oa = __shfl_up_sync(kFull, aa, off);
        const long long os = __shfl_up_sync(kFull, (long long)sid, off);
        if (lane >= off && os == sid && better(oq, oa, q, aa, mx)) {
          q = oq;
          aa = oa;
        }
      }
      if (ok && act == m - 1) {  // last row of a state: its best is final
        const int64_t s = sid;
        const int ba = aa == INT_MAX ? 0 : aa;
        a.policy[s] = ba;
        a.applied[s] = q;
        if (a.gpi) a.gpi[s] = __ldg(a.cost + s * m + ba);
        if (a.lenpi) a.lenpi[s] = K;
        res = res_max(res, fabs(sub_rn(gather((int)(a.state0 + s)), q)));
      }
      carry_q = __shfl_sync(kFull, q, 31);
      carry_a = __shfl_sync(kFull, aa, 31);
      carry_s = __shfl_sync(kFull, (long long)sid, 31);
      if (has_next) cur = nxt;
    }
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t = res_max(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

// ---------------------------------------------------------------------------
// Flat rows, shared-memory ring (K <= 4, C3: n = 4.2M, m = 21, K = 4).
//
// The register-pipelined flat kernel above spends ~390 instructions per
// 32-row batch, 2/3 of them in the segmented argmin scan (5 shuffle rounds on
// q, action and state id), and waits on V gathers issued one batch ahead, so
// it is issue/latency-bound at ~50% of HBM.  This kernel:
//   * streams each warp's contiguous row range through a private S-stage
//     shared-memory ring with cp.async: every instruction moves 512
//     contiguous bytes (lane l copies 16-byte chunk l), nothing occupies
//     registers while in flight, and S-3..S-2 batches stay outstanding;
//   * issues the V gathers of batch i+2 while batch i is reduced (three
//     rotating register sets, loop unrolled by 3 so no register copy waits
//     on an outstanding load);
//   * lane = row for the products (q = g + gamma*acc, numpy reduceat order
//     p0 + (((0 + p1) + p2) + p3), so Q is bitwise the reference's), q goes to
//     a per-warp shared buffer of 32 states, and after every m batches
//     (= 32 states) lane = state runs the first-index argmin/argmax over its
//     m entries sequentially: no shuffles, and the policy / applied / g_pi /
//     residual traffic becomes coalesced.
// ---------------------------------------------------------------------------
template <int K>
struct RingLayout {
  static constexpr int kVal = 32 * K * 8;             // values of 32 rows
  static constexpr int kCol = 32 * K * 4;             // columns of 32 rows
  static constexpr int kCost = 17 * 16;               // 16-byte chunks covering 32 (+1) costs
  static constexpr int kStage = kVal + kCol + kCost;  // multiple of 16
};

// dynamic shared memory: [V window][NW rings of S stages][NW q buffers of 32*m]
int flat_ring_smem(int K, int stages, int warps, int m, int window_bytes) {
  const int st = K == 2 ? RingLayout<2>::kStage : RingLayout<4>::kStage;
  return ((window_bytes + 15) & ~15) + warps * (stages * st + 32 * m * 8);
}

template <int K, int S, int NW, bool WIN>
__global__ void __launch_bounds__(NW * 32, 1) k1_bellman_ring(K1Args a, int win_bytes) {
  static_assert(K == 2 || K == 4, "flat ring handles K = 2 or 4");
  static_assert(S >= 4, "ring needs >= 4 stages (gathers run two batches ahead)");
  using L = RingLayout<K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  double* win = reinterpret_cast<double*>(smem_raw);
  const int64_t s_lo = a.bounds[blockIdx.x], s_hi = a.bounds[blockIdx.x + 1];
  int w_lo = 0;
  uint32_t w_len = 0;
  if (WIN) {
    int64_t lo = a.state0 + s_lo - a.halo;
    int64_t hi = a.state0 + s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n_global ? a.n_global : hi;
    w_lo = (int)lo;
    w_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
    window_load8(win, a.v, lo, w_len);
  }
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = a.m;
  unsigned char* rings = smem_raw + (((WIN ? win_bytes : 0) + 15) & ~15);
  unsigned char* ring = rings + warp * S * L::kStage;
  double* qb = reinterpret_cast<double*>(rings + NW * S * L::kStage) + warp * 32 * m;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const bool mx = a.maximize != 0;
  double res = 0.0;
  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) return win[off];
    }
    return __ldg(a.v + c);
  };
  const int64_t ns = s_hi - s_lo;
  const int64_t ws0 = s_lo + ns * warp / NW, ws1 = s_lo + ns * (warp + 1) / NW;
  const int64_t r_beg = ws0 * m, r_end = ws1 * m;
  const int64_t r_valid = s_hi * (int64_t)m;  // rows < r_valid exist in the arrays
  const int64_t nb = (r_end - r_beg + 31) >> 5;

  // batch i -> stage stg: values, columns, costs (one commit group, maybe empty)
  auto issue = [&](int64_t i, int stg) {
    if (i < nb) {
      const int64_t base = r_beg + (i << 5);
      const int64_t left = r_end - base;
      const int nr = left < 32 ? (int)left : 32;
      const uint32_t st = ring_s + (uint32_t)(stg * L::kStage);
      const double* vp = a.val + base * K;
#pragma unroll
      for (int c = lane; c < 32 * K / 2; c += 32)  // 16-byte value chunks
        if (c < nr * K / 2) cp_async16(st + 16 * c, vp + 2 * c, 16, pol);
      if (K == 4) {
        if (lane < nr) cp_async16(st + L::kVal + 16 * lane, a.col + (base + lane) * 4, 16, pol);
      } else {
        if (lane < nr) cp_async8(st + L::kVal + 8 * lane, a.col + (base + lane) * 2);
      }
      const int64_t c0 = base & ~(int64_t)1;  // 16-byte aligned cost chunk start
      const int nch = (int)((base + nr - c0 + 1) >> 1);
      if (lane < nch) {
        const int64_t lo = c0 + 2 * lane;
        const uint32_t bytes = lo + 1 < r_valid ? 16u : 8u;
        cp_async16(st + L::kVal + L::kCol + 16 * lane, a.cost + lo, bytes, pol);
      }
    }
    cp_async_commit();
  };
  // V gathers of batch i (its columns must have landed)
  auto fetch = [&](int64_t i, int stg, double (&x)[K]) {
    if (i < nb && r_beg + (i << 5) + lane < r_end) {
      const unsigned char* st = ring + stg * L::kStage;
      if (K == 4) {
        const int4 c = *reinterpret_cast<const int4*>(st + L::kVal + 16 * lane);
        x[0] = gather(c.x);
        x[1] = gather(c.y);
        x[2 % K] = gather(c.z);
        x[3 % K] = gather(c.w);
      } else {
        const int2 c = *reinterpret_cast<const int2*>(st + L::kVal + 8 * lane);
        x[0] = gather(c.x);
        x[1 % K] = gather(c.y);
      }
    }
  };
  int bi = 0;        // batch index inside the current 32-state group
  int64_t gs0 = ws0;  // first state of the current group
  // q of batch i's rows -> q buffer; after the group's last batch, lane = state
  auto compute = [&](int64_t i, int stg, const double (&x)[K]) {
    const int64_t base = r_beg + (i << 5);
    const unsigned char* st = ring + stg * L::kStage;
    if (base + lane < r_end) {
      const double2 v0 = *reinterpret_cast<const double2*>(st + lane * K * 8);
      double acc = add_rn(0.0, mul_rn(v0.y, x[1 % K]));
      if (K == 4) {
        const double2 v1 = *reinterpret_cast<const double2*>(st + lane * K * 8 + 16);
        acc = add_rn(acc, mul_rn(v1.x, x[2 % K]));
        acc = add_rn(acc, mul_rn(v1.y, x[3 % K]));
      }
      acc = add_rn(mul_rn(v0.x, x[0]), acc);
      const double g = reinterpret_cast<const double*>(st + L::kVal + L::kCol)[(base & 1) + lane];
      qb[bi * 32 + lane] = add_rn(g, mul_rn(a.gamma, acc));
    }
    ++bi;
    if (bi == m || i + 1 == nb) {  // group complete: 32 states (fewer in the tail)
      __syncwarp();
      const int64_t left = ws1 - gs0;
      const int nst = left < 32 ? (int)left : 32;
      if (lane < nst) {
        const double* q = qb + lane * m;
        double bq = q[0];
        int ba = 0;
        if (mx) {
          for (int t = 1; t < m; ++t) {
            const double v = q[t];
            if (v > bq) { bq = v; ba = t; }
          }
        } else {
          for (int t = 1; t < m; ++t) {
            const double v = q[t];
            if (v < bq) { bq = v; ba = t; }
          }
        }
        const int64_t s = gs0 + lane;
        a.policy[s] = ba;
        a.applied[s] = bq;
        if (a.gpi) a.gpi[s] = __ldg(a.cost + s * m + ba);
        if (a.lenpi) a.lenpi[s] = K;
        res = res_max(res, fabs(sub_rn(gather((int)(a.state0 + s)), bq)));
      }
      __syncwarp();
      bi = 0;
      gs0 += 32;
    }
  };
  // step i: batch i+2's gathers go out, batch i is reduced, stage i % S is
  // refilled with batch i+S
  int stg = 0;
  auto step = [&](int64_t i, const double (&cur)[K], double (&ahead)[K]) {
    const int s2 = stg + 2 >= S ? stg + 2 - S : stg + 2;
    cp_async_wait<S - 3>();  // batch i+2 landed (this lane's copies)
    __syncwarp();            // ... and every lane's
    fetch(i + 2, s2, ahead);
    compute(i, stg, cur);
    __syncwarp();  // stage i fully consumed
    issue(i + S, stg);
    stg = stg + 1 == S ? 0 : stg + 1;
  };

  if (nb > 0) {
#pragma unroll 1
    for (int j = 0; j < S; ++j) issue(j, j);
    double x0[K], x1[K], x2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) x0[k] = x1[k] = x2[k] = 0.0;
    cp_async_wait<S - 2>();  // batches 0 and 1 landed
    __syncwarp();
    fetch(0, 0, x0);
    fetch(1, 1, x1);
#pragma unroll 1
    for (int64_t i = 0; i < nb; i += 3) {
      step(i, x0, x2);
      if (i + 1 < nb) step(i + 1, x1, x0);
      if (i + 2 < nb) step(i + 2, x2, x1);
    }
  }
  cp_async_wait<0>();
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t = res_max(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

template <int K, int S, int NW, bool WIN>
static cudaError_t ring_attr(int smem) {
  return raise_smem_limit(k1_bellman_ring<K, S, NW, WIN>, smem);
}

template <int K, int S, int NW>
static void ring_go(const K1Args& a, bool win, int blocks, int smem, int win_bytes, cudaStream_t st) {
  if (win)
    k1_bellman_ring<K, S, NW, true><<<blocks, NW * 32, smem, st>>>(a, win_bytes);
  else
    k1_bellman_ring<K, S, NW, false><<<blocks, NW * 32, smem, st>>>(a, 0);
}

// (stages, warps) shapes with an instance: deeper rings for fewer warps
#define IPI_RING_SHAPES(K, MACRO) \
  MACRO(K, 4, 18) MACRO(K, 4, 16) MACRO(K, 6, 12) MACRO(K, 5, 12) MACRO(K, 8, 8)
#define IPI_DISPATCH_RING(K, S, W, MACRO)                           \
  do {                                                              \
    ok = false;                                                     \
    if ((K) == 2) { IPI_RING_SHAPES(2, MACRO) }                     \
    else if ((K) == 4) { IPI_RING_SHAPES(4, MACRO) }                \
  } while (0)

bool k1_ring_prepare(int K, int S, int NW, bool win, int smem) {
  bool ok = false;
  cudaError_t e = cudaSuccess;
#define IPI_R_ATTR(KK, SS, WW)                                                             \
  if (!ok && K == KK && S == SS && NW == WW) {                                             \
    ok = true;                                                                             \
    e = win ? ring_attr<KK, SS, WW, true>(smem) : ring_attr<KK, SS, WW, false>(smem);      \
  }
  IPI_DISPATCH_RING(K, S, NW, IPI_R_ATTR);
#undef IPI_R_ATTR
  return ok && e == cudaSuccess;
}

// ---------------------------------------------------------------------------
// Uniform rows, shared-memory ring (9 <= K <= 129, K % 4 == 0, m % 4 == 0;
// C2/C5: K = 64, m = 32).
//
// Same streaming scheme as the flat ring above: each warp moves its
// contiguous row range through a private S-stage cp.async ring (4 rows per
// stage), so the CSR stream costs no registers in flight and every copy
// instruction moves 512 contiguous bytes.  A stage is one warp step: 8 lanes
// per row, 4 rows.  The row sum restates numpy's reduceat arithmetic exactly
// (a[0] + pairwise(a[1:]); for 8 <= K-1 <= 128 pairwise keeps 8 running sums
// r[j] = a[1+j] + a[9+j] + ..., folds them as ((r0+r1)+(r2+r3))+((r4+r5)+
// (r6+r7)) and adds the (K-1) % 8 leftover terms in order): lane j of a row
// owns r[j], the fold is three xor shuffles, the leftovers are added in
// order from shuffles -- so Q is bitwise the reference's.  Shared-memory
// stage rows are XOR-swizzled at 16-byte granularity so the 4 rows of a
// step hit disjoint banks.  V gathers of step i+1 are issued before step i
// is reduced.  The argmin keeps one running (q, a) per row group (actions
// a = g mod 4) and merges the 4 groups with two xor shuffles per state.
// ---------------------------------------------------------------------------
template <int K>
struct URingLayout {
  static constexpr int kVal = 4 * K * 8;   // 4 rows of values
  static constexpr int kCol = 4 * K * 4;   // 4 rows of columns
  static constexpr int kStage = kVal + kCol + 32;  // + 4 costs
};

int uniform_ring_smem(int K, int stages, int warps, int window_bytes) {
  const int st = 4 * K * 12 + 32;
  return ((window_bytes + 15) & ~15) + warps * (stages * st + 256);
}

// D = gather lookahead in steps (1 or 2): V gathers of step i+D are issued
// before step i is reduced, so the ~10% that miss the window and go to L2
// have D steps to land.
template <int K, int NW, int S, int D, bool WIN>
__global__ void __launch_bounds__(NW * 32, 1) k1_bellman_uring(K1Args a, int win_bytes) {
  constexpr int N1 = K - 1;       // pairwise runs over a[1 .. K-1]
  constexpr int NC = N1 / 8;      // terms per running sum
  constexpr int TAIL = N1 % 8;    // leftover terms added in order
  static_assert(N1 >= 8 && N1 <= 128 && K % 4 == 0, "uniform ring: 9 <= K <= 129, K % 4 == 0");
  static_assert(D == 1 || D == 2, "gather lookahead is 1 or 2 steps");
  static_assert(S >= D + 2, "ring needs D + 2 stages");
  using L = URingLayout<K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  double* win = reinterpret_cast<double*>(smem_raw);
  if (a.trace && threadIdx.x == 0) {
    a.trace[3 * blockIdx.x] = sm_id();
    a.trace[3 * blockIdx.x + 1] = global_ns();
  }
  const int64_t s_lo = a.bounds[blockIdx.x], s_hi = a.bounds[blockIdx.x + 1];
  int w_lo = 0;
  uint32_t w_len = 0;
  // the V window goes out as one cp.async group together with the first ring
  // stages (a scalar window loop stalled every CTA wave's start)
  if (WIN && a.win_async)
    window_issue_async(a.v, a.state0 + s_lo - a.halo, a.state0 + s_hi + a.halo, a.n_global,
                       smem_raw, w_lo, w_len);
  if (WIN && !a.win_async) {  // scalar window loop (A/B: IPI_K1_WIN_ASYNC=0)
    int64_t lo = a.state0 + s_lo - a.halo;
    int64_t hi = a.state0 + s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n_global ? a.n_global : hi;
    w_lo = (int)lo;
    w_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
    for (uint32_t i = threadIdx.x; i < w_len; i += blockDim.x) win[i] = __ldg(a.v + lo + i);
    __syncthreads();
  }
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, j = lane & 7;  // row of the step, lane within the row
  const int m = a.m;
  unsigned char* base_s = smem_raw + (((WIN ? win_bytes : 0) + 15) & ~15) + warp * (S * L::kStage + 256);
  unsigned char* ring = base_s;
  double* tb = reinterpret_cast<double*>(base_s + S * L::kStage);  // 32 tail products
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const double sgn = a.maximize != 0 ? -1.0 : 1.0;  // argmax(q) == argmin(-q), ties alike
  const double* __restrict__ vg = a.v;
  double res = 0.0;
  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) return win[off];
    }
    return __ldg(vg + c);
  };
  const int64_t ns = s_hi - s_lo;
  // State order.  Interleaved (default): warp w takes states s_lo + w, + NW, ...
  // so the CTA's warps stream NW consecutive states (one contiguous region per
  // CTA).  Contiguous (IPI_K1_INTERLEAVE=0): warp w owns a contiguous state
  // range; its NW*grid concurrent streams sit at regular strides and, for some
  // wave counts, collide in the DRAM channel hash (0.70 vs 0.88 of HBM).
  const bool inter = a.interleave != 0;
  const int64_t ws0 = inter ? s_lo + warp : s_lo + ns * warp / NW;
  const int64_t ws1 = inter ? s_hi : s_lo + ns * (warp + 1) / NW;
  const int64_t s_step = inter ? NW : 1;  // state stride of this warp
  const int64_t n_states = inter ? (ns > warp ? (ns - warp + NW - 1) / NW : 0) : ws1 - ws0;
  const int spm = m >> 2;                  // steps per state (m % 4 == 0)
  const int64_t nb = n_states * spm;
  // Rotation (interleaved order): this warp starts at state index `rot` of its
  // sequence and wraps, so the grid's concurrent streams do not advance in
  // lock-step at fixed strides (IPI_K1_ROTATE=0 disables).
  const int64_t rot = (inter && a.rotate && n_states > 0)
                          ? (int64_t)(((uint64_t)blockIdx.x * 2654435761ull) % (uint64_t)n_states) : 0;
  auto state_of = [&](int64_t k) -> int64_t {  // k-th state this warp processes
    int64_t kk = k + rot;
    if (kk >= n_states) kk -= n_states;
    return ws0 + kk * s_step;
  };
  int64_t ik = 0;                          // state index of the next issue
  int64_t irow = state_of(0) * m;          // next row to issue
  int ist = 0;                             // steps issued in the current state

  // 16-byte chunk cc of row r lives at chunk cc ^ swz(r): rows of a step on disjoint banks
  // values: LDS.64 half-warp = rows {0,1} / {2,3}: flip 64 B for odd rows
  // columns: LDS.32 full warp = rows 0..3: flip 32 B * r
  // issue() is called once per step, in step order
  auto issue = [&](int64_t i, int stg) {
    if (i < nb) {
      const int64_t row0 = irow;
      irow += 4;
      if (++ist == spm) {
        ist = 0;
        irow = state_of(++ik) * m;
      }
      const uint32_t st = ring_s + (uint32_t)(stg * L::kStage);
      const double* vp = a.val + row0 * K;
      const int* cp = a.col + row0 * K;
#pragma unroll
      for (int c = lane; c < 4 * K / 2; c += 32) {  // value chunks (2 doubles)
        const int r = c / (K / 2), cc = c % (K / 2);
        cp_async16(st + r * K * 8 + 16 * (cc ^ ((r & 1) << 2)), vp + 2 * c, 16, pol);
      }
#pragma unroll
      for (int c = lane; c < 4 * K / 4; c += 32) {  // column chunks (4 ints)
        const int r = c / (K / 4), cc = c % (K / 4);
        cp_async16(st + L::kVal + r * K * 4 + 16 * (cc ^ (r << 1)), cp + 4 * c, 16, pol);
      }
      if (lane < 2) cp_async16(st + L::kVal + L::kCol + 16 * lane, a.cost + row0 + 2 * lane, 16, pol);
    }
    cp_async_commit();
  };
  auto vaddr = [&](int r, int e) {  // byte offset of value e of row r
    return r * K * 8 + ((((e >> 1) ^ ((r & 1) << 2))) << 4) + ((e & 1) << 3);
  };
  auto caddr = [&](int r, int e) {  // byte offset of column e of row r
    return L::kVal + r * K * 4 + ((((e >> 2) ^ (r << 1))) << 4) + ((e & 3) << 2);
  };
  // gathers of one step: NC chain terms a[1+j+8k] and one leftover/first term
  constexpr int NG = NC + 1;
  const bool has_last = j < TAIL || j == 7;
  const int e_last = j < TAIL ? 1 + 8 * NC + j : 0;  // leftover term, lane 7: a[0]
  auto fetch = [&](int stg, double (&x)[NG]) {
    const unsigned char* st = ring + stg * L::kStage;
#pragma unroll
    for (int k = 0; k < NC; ++k) x[k] = gather(*reinterpret_cast<const int*>(st + caddr(grp, 1 + j + 8 * k)));
    if (has_last) x[NC] = gather(*reinterpret_cast<const int*>(st + caddr(grp, e_last)));
  };
  int t_in_state = 0;
  int64_t kc = 0;  // state index of the step being reduced
  int64_t s_cur = state_of(0);
  double bq = INFINITY;
  int ba = INT_MAX;
  auto compute = [&](int stg, const double (&x)[NG]) {
    const unsigned char* st = ring + stg * L::kStage;
    auto val = [&](int e) { return *reinterpret_cast<const double*>(st + vaddr(grp, e)); };
    tb[lane] = has_last ? mul_rn(val(e_last), x[NC]) : 0.0;
    double r = mul_rn(val(1 + j), x[0]);
#pragma unroll
    for (int k = 1; k < NC; ++k) r = add_rn(r, mul_rn(val(1 + j + 8 * k), x[k]));
    r = add_rn(r, __shfl_xor_sync(kFull, r, 1));
    r = add_rn(r, __shfl_xor_sync(kFull, r, 2));
    r = add_rn(r, __shfl_xor_sync(kFull, r, 4));
    __syncwarp();
    const double2* t2 = reinterpret_cast<const double2*>(tb + (grp << 3));
    double t[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 u = t2[q];
      t[2 * q] = u.x;
      t[2 * q + 1] = u.y;
    }
#pragma unroll
    for (int q = 0; q < TAIL; ++q) r = add_rn(r, t[q]);
    const double total = add_rn(t[7], r);
    const double g = reinterpret_cast<const double*>(st + L::kVal + L::kCol)[grp];
    const double q = mul_rn(sgn, add_rn(g, mul_rn(a.gamma, total)));
    const int act = 4 * t_in_state + grp;
    if (q < bq) {  // actions of a group arrive in increasing order
      bq = q;
      ba = act;
    }
    if (++t_in_state == (m >> 2)) {  // state complete: merge the 4 groups
#pragma unroll
      for (int off = 8; off <= 16; off <<= 1) {
        const double oq = __shfl_xor_sync(kFull, bq, off);
        const int oa = __shfl_xor_sync(kFull, ba, off);
        if (oq < bq || (oq == bq && oa < ba)) {
          bq = oq;
          ba = oa;
        }
      }
      if (lane == 0) {
        const int64_t s = s_cur;
        const double ap = mul_rn(sgn, bq);
        const int pa = ba == INT_MAX ? 0 : ba;
        a.policy[s] = pa;
        a.applied[s] = ap;
        if (a.gpi) a.gpi[s] = __ldg(a.cost + s * m + pa);
        if (a.lenpi) a.lenpi[s] = K;
        res = res_max(res, fabs(sub_rn(gather((int)(a.state0 + s)), ap)));
      }
      t_in_state = 0;
      s_cur = state_of(++kc);
      bq = INFINITY;
      ba = INT_MAX;
    }
  };
  int stg = 0;
  auto step = [&](int64_t i, const double (&cur)[NG], double (&ahead)[NG]) {
    const int sd = stg + D >= S ? stg + D - S : stg + D;
    cp_async_wait<S - 1 - D>();  // step i+D landed (this lane's copies)
    __syncwarp();                // ... and every lane's
    if (i + D < nb) fetch(sd, ahead);
    compute(stg, cur);
    __syncwarp();  // stage i and the tail buffer fully consumed
    issue(i + S, stg);
    stg = stg + 1 == S ? 0 : stg + 1;
  };
#pragma unroll 1
  for (int q = 0; q < S; ++q) issue(q, q);
  if (WIN && a.win_async) {
    cp_async_wait<S>();  // the window group landed (this thread's copies)
    __syncthreads();     // ... and every thread's
  }
  if (nb > 0) {
    double x0[NG], x1[NG], x2[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) x0[k] = x1[k] = x2[k] = 0.0;
    cp_async_wait<S - D>();  // steps 0 .. D-1 landed
    __syncwarp();
    fetch(0, x0);
    if (D == 2 && nb > 1) fetch(1, x1);
    if (D == 1) {
#pragma unroll 1
      for (int64_t i = 0; i < nb; i += 2) {
        step(i, x0, x1);
        if (i + 1 < nb) step(i + 1, x1, x0);
      }
    } else {
#pragma unroll 1
      for (int64_t i = 0; i < nb; i += 3) {
        step(i, x0, x2);
        if (i + 1 < nb) step(i + 1, x1, x0);
        if (i + 2 < nb) step(i + 2, x2, x1);
      }
    }
  }
  cp_async_wait<0>();
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) a.trace[3 * blockIdx.x + 2] = global_ns();
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t = res_max(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

template <int K, int NW, int S, int D, bool WIN>
static cudaError_t uring_attr(int smem) {
  return raise_smem_limit(k1_bellman_uring<K, NW, S, D, WIN>, smem);
}

template <int K, int NW, int S, int D>
static void uring_go(const K1Args& a, bool win, int blocks, int smem, int win_bytes, cudaStream_t st) {
  if (win)
    k1_bellman_uring<K, NW, S, D, true><<<blocks, NW * 32, smem, st>>>(a, win_bytes);
  else
    k1_bellman_uring<K, NW, S, D, false><<<blocks, NW * 32, smem, st>>>(a, 0);
}

// (K, warps, stages, lookahead) instances
#define IPI_URING_SHAPES(MACRO)                                                           \
  MACRO(64, 12, 3, 1) MACRO(64, 10, 3, 1) MACRO(64, 11, 3, 1) MACRO(64, 10, 4, 1)        \
  MACRO(64, 12, 4, 1) MACRO(64, 11, 4, 1) MACRO(64, 11, 4, 2) MACRO(64, 16, 4, 2)        \
  MACRO(64, 16, 3, 1) MACRO(64, 14, 4, 2) MACRO(64, 12, 5, 2) MACRO(64, 14, 3, 1)        \
  MACRO(64, 15, 3, 1)                                                                    \
  MACRO(64, 8, 4, 1) MACRO(64, 8, 3, 1) MACRO(64, 10, 4, 2) MACRO(64, 8, 4, 2)           \
  MACRO(64, 8, 5, 2) MACRO(64, 12, 4, 2) MACRO(64, 6, 6, 2)

bool k1_uring_prepare(int K, int NW, int S, int D, bool win, int smem) {
  bool ok = false;
  cudaError_t e = cudaSuccess;
#define IPI_U_ATTR(KK, WW, SS, DD)                                                               \
  if (!ok && K == KK && NW == WW && S == SS && D == DD) {                                        \
    ok = true;                                                                                   \
    e = win ? uring_attr<KK, WW, SS, DD, true>(smem) : uring_attr<KK, WW, SS, DD, false>(smem);  \
  }
  IPI_URING_SHAPES(IPI_U_ATTR)
#undef IPI_U_ATTR
  return ok && e == cudaSuccess;
}

// ---------------------------------------------------------------------------
// Deep-pipeline uniform kernel: 16 warps per SM with up to 128 registers each
// (one 512-thread CTA per SM, one V window per SM).  Bytes in flight are
// bounded by registers, so fewer warps with deeper rings beat many shallow
// warps: a ring of 4 CSR batches (values/columns/cost of batch b+3 are issued
// while b is reduced) and a ring of 2 gather batches (V gathers of b+1 are
// issued before b is reduced), indices resolved at compile time (loop unrolled
// by 4) so no register copy waits on an outstanding load.
// ---------------------------------------------------------------------------
template <int P>
struct DeepCsr {
  double2 v[P];
  int2 c[P];
  double g;
};

template <int G, int P, bool WIN>
__global__ void __launch_bounds__(kK1Threads, 1) k1_bellman_deep(K1Args a, int K) {
  extern __shared__ double win[];
  __shared__ double red[32];
  const int64_t s_lo = a.bounds[blockIdx.x], s_hi = a.bounds[blockIdx.x + 1];
  int w_lo = 0;
  uint32_t w_len = 0;
  if (WIN) {
    int64_t lo = a.state0 + s_lo - a.halo;
    int64_t hi = a.state0 + s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n_global ? a.n_global : hi;
    w_lo = (int)lo;
    w_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
    window_load8(win, a.v, lo, w_len);
  }
  const uint32_t win_s = (uint32_t)__cvta_generic_to_shared(win);
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  constexpr int GPW = 32 / G;
  const int grp = lane / G, gl = lane % G;
  const bool mx = a.maximize != 0;
  const int m = a.m;
  const int nit = (m + GPW - 1) / GPW;
  const int pairs = K >> 1;
  double res = 0.0;

  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) {
        double x;
        // volatile: the window is filled in this kernel (ordered by the barrier)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(win_s + off * 8u));
        return x;
      }
    }
    return __ldg(a.v + c);
  };
  auto load = [&](int64_t s, int it, DeepCsr<P>& b) {
    const int act = it * GPW + grp;
    const bool ok = s < s_hi && act < m;
    const int64_t row = s * (int64_t)m + act;
    const double* vp = a.val + row * K;
    const int* cp = a.col + row * K;
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const int j = gl + G * t;
      if (ok && j < pairs) {
        b.v[t] = ld_stream_v2(vp + 2 * j, pol);
        b.c[t] = ld_stream_v2(cp + 2 * j, pol);
      } else {
        b.v[t] = make_double2(0.0, 0.0);
        b.c[t] = make_int2(-1, -1);
      }
    }
    b.g = ok ? __ldg(a.cost + row) : 0.0;
  };
  auto gather_batch = [&](const DeepCsr<P>& b, double2 (&x)[P]) {
#pragma unroll
    for (int t = 0; t < P; ++t)
      x[t] = make_double2(b.c[t].x >= 0 ? gather(b.c[t].x) : 0.0,
                          b.c[t].y >= 0 ? gather(b.c[t].y) : 0.0);
  };
  // flattened (state, row-step) coordinates of batch k after the current one
  auto advance = [&](int64_t& s, int& it) {
    if (++it == nit) {
      it = 0;
      s += nwarps;
    }
  };

  int64_t sC = s_lo + warp;
  if (sC < s_hi) {
    int itC = 0;
    // coordinates of batches b+1 (gather stage) and b+3 (load stage)
    int64_t s1 = sC, s3;
    int it1 = 0, it3;
    advance(s1, it1);
    s3 = s1;
    it3 = it1;
    advance(s3, it3);
    DeepCsr<P> R[4];
    double2 X[2][P];
    {
      int64_t s2 = s3;
      int i2 = it3;
      load(sC, itC, R[0]);
      load(s1, it1, R[1]);
      load(s2, i2, R[2]);
      advance(s3, it3);
    }
    gather_batch(R[0], X[0]);
    double bq = mx ? -INFINITY : INFINITY;
    int ba = INT_MAX;
    bool live = true;
    while (live) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (live) {
          load(s3, it3, R[(u + 3) & 3]);                // predicated off past s_hi
          const bool has1 = s1 < s_hi;
          if (has1) gather_batch(R[(u + 1) & 3], X[(u + 1) & 1]);
          double acc = 0.0;
#pragma unroll
          for (int t = 0; t < P; ++t) {
            acc = add_rn(acc, mul_rn(R[u].v[t].x, X[u & 1][t].x));
            acc = add_rn(acc, mul_rn(R[u].v[t].y, X[u & 1][t].y));
          }
          acc = group_sum<G>(acc);
          const int act = itC * GPW + grp;
          if (act < m) {
            const double q = add_rn(R[u].g, mul_rn(a.gamma, acc));
            if (better(q, act, bq, ba, mx)) {
              bq = q;
              ba = act;
            }
          }
          if (itC == nit - 1) {
#pragma unroll
            for (int off = 16; off >= G; off >>= 1) {
              const double oq = __shfl_xor_sync(kFull, bq, off);
              const int oa = __shfl_xor_sync(kFull, ba, off);
              if (better(oq, oa, bq, ba, mx)) {
                bq = oq;
                ba = oa;
              }
            }
            if (ba == INT_MAX) ba = 0;
            if (lane == 0) {
              const int64_t row0 = sC * (int64_t)m;
              a.policy[sC] = ba;
              a.applied[sC] = bq;
              if (a.gpi) a.gpi[sC] = __ldg(a.cost + row0 + ba);
              if (a.lenpi) a.lenpi[sC] = K;
              res = res_max(res, fabs(sub_rn(gather((int)(a.state0 + sC)), bq)));
            }
            bq = mx ? -INFINITY : INFINITY;
            ba = INT_MAX;
          }
          live = has1;
          sC = s1;
          itC = it1;
          advance(s1, it1);
          advance(s3, it3);
        }
      }
    }
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t = res_max(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

// (G, P) for the uniform path: pairs = K/2 <= P*G, P = 2 (or 4 for very long rows)
bool uniform_shape(int K, int* G, int* P) {
  if (K <= 0 || (K & 1)) return false;
  const int pairs = K / 2;
  const int gs[6] = {1, 2, 4, 8, 16, 32};
  for (int g : gs)
    if (pairs <= 2 * g) {
      *G = g;
      *P = 2;
      return true;
    }
  return false;  // rows longer than 128: generic path
}

template <int G, int P>
static void launch_u(const K1Args& a, int K, bool win, int blocks, int smem, cudaStream_t st) {
  if (win)
    k1_bellman_uniform<G, P, true><<<blocks, kK1Threads, smem, st>>>(a, K);
  else
    k1_bellman_uniform<G, P, false><<<blocks, kK1Threads, 0, st>>>(a, K);
}

template <int G, int P>
static cudaError_t set_smem_attr_u(int smem) {
  cudaError_t e = raise_smem_limit(k1_bellman_deep<G, P, true>, smem);
  if (e != cudaSuccess) return e;
  return raise_smem_limit(k1_bellman_uniform<G, P, true>, smem);
}

static cudaError_t uniform_smem(int G, int P, int smem) {
  cudaError_t e = cudaSuccess;
#define IPI_U_SMEM(GG, PP) e = set_smem_attr_u<GG, PP>(smem)
  IPI_DISPATCH_UNIFORM(G, P, IPI_U_SMEM);
#undef IPI_U_SMEM
  return e;
}

template <int G>
static void launch_g(const K1Args& a, bool win, int blocks, int smem, cudaStream_t st) {
  if (G == 32 && a.contig) {  // banded rows (C4)
    if (win) k1_bellman<G, true, true><<<blocks, kK1Threads, smem, st>>>(a);
    else k1_bellman<G, false, true><<<blocks, kK1Threads, 0, st>>>(a);
    return;
  }
  if (win)
    k1_bellman<G, true><<<blocks, kK1Threads, smem, st>>>(a);
  else
    k1_bellman<G, false><<<blocks, kK1Threads, 0, st>>>(a);
}

template <int G>
static cudaError_t set_smem_attr(int smem) {
  cudaError_t e = raise_smem_limit(k1_bellman<G, true>, smem);
  if (G == 32 && e == cudaSuccess) e = raise_smem_limit(k1_bellman<G, true, true>, smem);
  return e;
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
  e = raise_smem_limit(k1_bellman_flat<true>, smem);
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("k1 smem attr: ") + cudaGetErrorString(e));
  for (int K = 2; K <= 256; K *= 2) {  // make every uniform instance launchable too
    int G, P;
    if (uniform_shape(K, &G, &P)) {
      e = uniform_smem(G, P, smem);
      if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("k1 smem attr: ") + cudaGetErrorString(e));
    }
  }
  return IPI_OK;
}

// Resident CTAs per SM of the K1 variant the plan selects.
int k1_occupancy(int lanes, int uniform_K, bool win, int smem) {
  int G = 0, P = 0, nb = 0;
  const void* fn = nullptr;
  if (uniform_K > 0 && uniform_K <= 4 && uniform_K % 2 == 0) {
    fn = win ? (const void*)k1_bellman_flat<true> : (const void*)k1_bellman_flat<false>;
  } else if (uniform_K > 0 && uniform_shape(uniform_K, &G, &P)) {
#define U_FN(GG, PP) fn = (win ? (const void*)k1_bellman_uniform<GG, PP, true> \
                           : (const void*)k1_bellman_uniform<GG, PP, false>)
    IPI_DISPATCH_UNIFORM(G, P, U_FN);
#undef U_FN
  } else {
#define G_FN(GG) (win ? (const void*)k1_bellman<GG, true> : (const void*)k1_bellman<GG, false>)
    switch (lanes) {
      case 1: fn = G_FN(1); break;
      case 2: fn = G_FN(2); break;
      case 4: fn = G_FN(4); break;
      case 8: fn = G_FN(8); break;
      case 16: fn = G_FN(16); break;
      default: fn = G_FN(32); break;
    }
#undef G_FN
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kK1Threads, win ? smem : 0) != cudaSuccess)
    return 1;
  return nb < 1 ? 1 : nb;
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
  a.win_async = h->k1_win_async;
  a.interleave = h->k1_interleave;
  a.rotate = h->k1_rotate;
  a.trace = h->k1_trace;
  a.contig = h->plan.contiguous_rows;
  const bool win = h->plan.halo >= 0;
  const int blocks = h->plan.k1_blocks, smem = h->plan.k1_smem_bytes;
  int G = 0, P = 0;
  if (h->plan.k1_variant == 3 && uniform_shape(h->plan.row_len_max, &G, &P)) {
    const int K = h->plan.row_len_max;
#define IPI_D_LAUNCH(GG, PP)                                                             \
  (win ? k1_bellman_deep<GG, PP, true><<<blocks, kK1Threads, smem, st>>>(a, K)            \
       : k1_bellman_deep<GG, PP, false><<<blocks, kK1Threads, 0, st>>>(a, K))
    IPI_DISPATCH_UNIFORM(G, P, IPI_D_LAUNCH);
#undef IPI_D_LAUNCH
    IPI_LAUNCH_CHECK();
    return IPI_OK;
  }
  if (h->plan.k1_variant == 6) {
    if (a.win_async && h->ring_win_bytes > 0 && (uintptr_t)v_full % 16 != 0) {
      // the window is staged in 16-byte cp.async chunks: realign V once
      if (!h->vbuf) IPI_CUDA_TRY(cudaMalloc(&h->vbuf, sizeof(double) * h->n_global));
      IPI_CUDA_TRY(cudaMemcpyAsync(h->vbuf, v_full, sizeof(double) * h->n_global,
                                   cudaMemcpyDeviceToDevice, st));
      a.v = h->vbuf;
    }
    bool ok = false;
    const int K = h->plan.row_len_max, S = h->plan.k1_stages, NW = h->plan.k1_threads / 32;
    const int D = h->uring_lookahead;
    const bool rw = h->ring_win_bytes > 0;
#define IPI_U_LAUNCH(KK, WW, SS, DD)                                                 \
  if (!ok && K == KK && NW == WW && S == SS && D == DD) {                            \
    ok = true;                                                                       \
    uring_go<KK, WW, SS, DD>(a, rw, blocks, smem, h->ring_win_bytes, st);            \
  }
    IPI_URING_SHAPES(IPI_U_LAUNCH)
#undef IPI_U_LAUNCH
    if (!ok) return fail(IPI_ECUDA, "k1 uniform ring: no instance for this (K, warps, stages)");
    IPI_LAUNCH_CHECK();
    return IPI_OK;
  }
  if (h->plan.k1_variant == 4) {
    bool ok = false;
    const int K = h->plan.row_len_max, S = h->plan.k1_stages, NW = h->plan.k1_threads / 32;
    const bool rw = h->ring_win_bytes > 0;
#define IPI_R_LAUNCH(KK, SS, WW)                                                     \
  if (!ok && K == KK && S == SS && NW == WW) {                                       \
    ok = true;                                                                       \
    ring_go<KK, SS, WW>(a, rw, blocks, smem, h->ring_win_bytes, st);                 \
  }
    IPI_DISPATCH_RING(K, S, NW, IPI_R_LAUNCH);
#undef IPI_R_LAUNCH
    if (!ok) return fail(IPI_ECUDA, "k1 ring: no instance for this (K, stages, warps)");
    IPI_LAUNCH_CHECK();
    return IPI_OK;
  }
  if (h->plan.uniform_rows && h->plan.row_len_max <= 4 && (h->plan.row_len_max % 2) == 0) {
    const int K = h->plan.row_len_max;
    if (win)
      k1_bellman_flat<true><<<blocks, kK1Threads, smem, st>>>(a, K);
    else
      k1_bellman_flat<false><<<blocks, kK1Threads, 0, st>>>(a, K);
    IPI_LAUNCH_CHECK();
    return IPI_OK;
  }
  if (h->plan.uniform_rows && uniform_shape(h->plan.row_len_max, &G, &P)) {
    const int K = h->plan.row_len_max;
#define IPI_U_LAUNCH(GG, PP) launch_u<GG, PP>(a, K, win, blocks, smem, st)
    IPI_DISPATCH_UNIFORM(G, P, IPI_U_LAUNCH);
#undef IPI_U_LAUNCH
    IPI_LAUNCH_CHECK();
    return IPI_OK;
  }
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
