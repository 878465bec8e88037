// bellman_tma.cu — K1 on uniform-row instances with a TMA producer/consumer
// pipeline (the B200-native form of the fused Bellman backup).
//
// Why: K1 streams 12 B/nnz of CSR once and gathers V.  Keeping enough bytes in
// flight to cover HBM latency through registers costs registers per byte;
// 1-D bulk copies (cp.async.bulk, TMA engine) into a shared-memory ring do it
// for free: one elected producer thread keeps NS chunk-stages (~25 KB each)
// in flight per SM while 16 consumer warps compute from shared memory.
//
// CTA = 1 per SM (persistent), contiguous nnz-balanced state range,
//   16 consumer warps + 1 producer warp.
// Shared memory:  [mbarriers][V window][NS stages: values | columns | costs][q buffers]
//   * V window: V[s0 - halo, s0 + SUPER + halo) for the current super-chunk of
//     SUPER states, reloaded by the consumers at super-chunk boundaries (the
//     producer keeps streaming CSR meanwhile), so the window costs 2*halo +
//     SUPER doubles instead of the whole CTA range.
//   * stage c%NS holds chunk c = SC states: their m*SC rows of values (fp64),
//     columns (int32) and stage costs, filled by 3 bulk copies that complete
//     on full[c%NS] (expect_tx); consumers release it on empty[c%NS].
// Consumers: G lanes per row (P = 2 pairs per lane, 16-byte LDS), rows of the
// chunk round-robin over warps, q = cost + gamma*(PV) into a per-chunk q
// buffer; one named barrier per chunk, then a warp per state does the
// first-index argmin, writes pi / TV / g_pi / len and the residual max.
// Tail chunks whose byte counts are not 16-byte multiples are read straight
// from global memory (uniform per-chunk branch).
#include <cfloat>
#include <climits>

#include "handle.cuh"

namespace ipi {

constexpr int kTmaConsumers = 16;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;

struct K1TmaArgs {
  const int64_t* bounds;
  const int32_t* col;
  const double* val;
  const double* cost;
  const double* v;
  int64_t n_global;
  int64_t state0;
  int32_t m;
  int32_t K;
  int32_t halo;        // < 0: no window (gathers through L1)
  int32_t SC;          // states per chunk
  int32_t NS;          // stages
  int32_t super_states;
  int32_t win_cap;     // doubles
  int32_t stage_bytes;
  double gamma;
  int32_t maximize;
  int32_t* policy;
  double* applied;
  double* gpi;
  int32_t* lenpi;
  unsigned long long* res_bits;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers * 32) : "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 lds_v2f64(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ int2 lds_v2s32(uint32_t addr) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

template <int G, bool WIN>
__global__ void __launch_bounds__(kTmaThreads, 1) k1_bellman_tma(K1TmaArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int NS = a.NS, SC = a.SC, m = a.m, K = a.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- shared-memory carve-up --------------------------------------------
  const uint32_t bar_full = smem_u32(smem);                 // NS x 8 B
  const uint32_t bar_empty = bar_full + 8u * NS;            // NS x 8 B
  unsigned char* p = smem + ((16 * NS + 127) / 128) * 128;
  double* win = reinterpret_cast<double*>(p);
  p += (size_t)a.win_cap * 8;
  unsigned char* stages = p;
  p += (size_t)NS * a.stage_bytes;
  double* qbuf = reinterpret_cast<double*>(p);               // (NS+2) x SC*m doubles + counters
  __shared__ double red[32];
  const uint32_t win_s = smem_u32(win);
  const uint32_t stages_s = smem_u32(stages);
  const int rows_c = SC * m;                                 // rows per full chunk
  const uint32_t val_bytes_c = (uint32_t)rows_c * K * 8, col_bytes_c = (uint32_t)rows_c * K * 4;

  const int64_t s_lo = a.bounds[blockIdx.x], s_hi = a.bounds[blockIdx.x + 1];
  const int64_t n_states = s_hi - s_lo;
  const int64_t nchunks = (n_states + SC - 1) / SC;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(bar_full + 8u * i, 1);
      mbar_init(bar_empty + 8u * i, kTmaConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();

  if (warp == kTmaConsumers) {
    // ======================= producer warp ===================================
    if (lane == 0) {
      int st = 0;
      uint32_t eparity = 0;  // parity of the empty-barrier phase to wait for
      for (int64_t c = 0; c < nchunks; ++c) {
        if (c >= NS) mbar_wait(bar_empty + 8u * st, eparity);
        const int64_t s0 = s_lo + c * SC;
        const int ns = (int)((s_hi - s0) < SC ? (s_hi - s0) : SC);
        const int rows = ns * m;
        const uint32_t vb = (uint32_t)rows * K * 8, cb = (uint32_t)rows * K * 4,
                       gb = (uint32_t)rows * 8;
        const uint32_t bar = bar_full + 8u * st;
        const bool aligned = (vb % 16 == 0) && (cb % 16 == 0) && (gb % 16 == 0);
        if (aligned) {
          mbar_expect_tx(bar, vb + cb + gb);
          const uint32_t dst = stages_s + (uint32_t)st * a.stage_bytes;
          const int64_t row0 = s0 * m;
          bulk_g2s(dst, a.val + row0 * K, vb, bar, pol);
          bulk_g2s(dst + val_bytes_c, a.col + row0 * K, cb, bar, pol);
          bulk_g2s(dst + val_bytes_c + col_bytes_c, a.cost + row0, gb, bar, pol);
        } else {
          mbar_arrive(bar);  // tail chunk: consumers read it from global memory
        }
        if (++st == NS) {
          st = 0;
          if (c >= NS - 1) eparity ^= (c >= NS) ? 1u : 0u;
        }
      }
    }
    return;
  }

  // ========================= consumers =======================================
  // Warps drift independently through the chunk stream (no per-chunk CTA
  // barrier): each warp computes its rows of a chunk into q, releases the stage,
  // and bumps the chunk's arrival counter; the LAST warp to arrive performs the
  // per-state argmin.  Two chunks are in flight per warp (their loads and
  // gathers are issued before either is reduced) to overlap the L2 latency of
  // out-of-window gathers.  Warps can drift by at most NS chunks (the producer
  // refills a stage only after all 16 warps released it), so NS+2 q buffers
  // suffice.
  constexpr int GPW = 32 / G;
  const int grp = lane / G, gl = lane % G;
  const int pairs = K >> 1;
  const bool mx = a.maximize != 0;
  const double gamma = a.gamma;
  const int QB = NS + 2;
  int* cnt = reinterpret_cast<int*>(qbuf + (size_t)QB * rows_c);   // QB counters
  int w_lo = 0;
  uint32_t w_len = 0;
  double res = 0.0;

  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) return lds_f64(win_s + off * 8u);
    }
    return __ldg(a.v + c);
  };

  // Row sums of one row-group pass of a chunk (rows rb.. of chunk at s0);
  // returns the lane's partial (before the group reduction).
  auto row_partial = [&](int r, int rows, bool in_smem, uint32_t sv, uint32_t sc_,
                         int64_t row0) -> double {
    double acc = 0.0;
    if (r < rows) {
#pragma unroll 2
      for (int j = gl; j < pairs; j += G) {
        double2 v2;
        int2 c2;
        const int e = r * K + 2 * j;
        if (in_smem) {
          v2 = lds_v2f64(sv + (uint32_t)e * 8u);
          c2 = lds_v2s32(sc_ + (uint32_t)e * 4u);
        } else {
          v2 = *reinterpret_cast<const double2*>(a.val + row0 * K + e);
          c2 = *reinterpret_cast<const int2*>(a.col + row0 * K + e);
        }
        const double x0 = gather(c2.x), x1 = gather(c2.y);
        acc = add_rn(acc, mul_rn(v2.x, x0));
        acc = add_rn(acc, mul_rn(v2.y, x1));
      }
    }
    return acc;
  };

  auto finish_chunk = [&](int64_t c, int64_t s0, int ns, double* q) {
    // caller: q of all rows visible (last arriver)
    for (int t = 0; t < ns; ++t) {
      double bq = mx ? -INFINITY : INFINITY;
      int ba = INT_MAX;
      for (int a0 = lane; a0 < m; a0 += 32) {
        const double qq = q[t * m + a0];
        if (better(qq, a0, bq, ba, mx)) {
          bq = qq;
          ba = a0;
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
      if (ba == INT_MAX) ba = 0;
      if (lane == 0) {
        const int64_t s = s0 + t;
        a.policy[s] = ba;
        a.applied[s] = bq;
        if (a.gpi) a.gpi[s] = __ldg(a.cost + s * m + ba);
        if (a.lenpi) a.lenpi[s] = K;
        const double vs = gather((int)(a.state0 + s));
        res = fmax(res, fabs(sub_rn(vs, bq)));
      }
    }
    (void)c;
  };

  for (int i = tid; i < QB; i += kTmaConsumers * 32) cnt[i] = 0;
  consumer_sync();

  int st = 0;             // stage of chunk c
  uint32_t parity = 0;    // full-barrier parity of chunk c
  int qb = 0;             // q buffer of chunk c
  int64_t next_reload = 0;
  for (int64_t c = 0; c < nchunks; c += 2) {
    const int64_t s0 = s_lo + c * SC;
    // super-chunk boundary: reload the V window (consumers only; rare)
    if (WIN && c * SC >= next_reload) {
      consumer_sync();
      int64_t lo = a.state0 + s0 - a.halo;
      int64_t send = s0 + a.super_states;
      if (send > s_hi) send = s_hi;
      int64_t hi = a.state0 + send + a.halo;
      lo = lo < 0 ? 0 : lo;
      hi = hi > a.n_global ? a.n_global : hi;
      w_lo = (int)lo;
      w_len = (uint32_t)(hi - lo);
      for (uint32_t i = tid; i < w_len; i += kTmaConsumers * 32) win[i] = __ldg(a.v + lo + i);
      next_reload = c * SC + a.super_states;
      consumer_sync();
    }
    // ---- two chunks: A = c, B = c+1 (if any and inside the same super-chunk)
    const bool hasB = (c + 1 < nchunks) && (!WIN || (c + 1) * SC < next_reload);
    const int stA = st, stB = (st + 1 == NS) ? 0 : st + 1;
    const uint32_t parA = parity, parB = (stB == 0) ? parity ^ 1u : parity;
    const int qbA = qb, qbB = (qb + 1 == QB) ? 0 : qb + 1;
    const int64_t s0B = s0 + SC;
    const int nsA = (int)((s_hi - s0) < SC ? (s_hi - s0) : SC);
    const int nsB = hasB ? (int)((s_hi - s0B) < SC ? (s_hi - s0B) : SC) : 0;
    const int rowsA = nsA * m, rowsB = nsB * m;
    mbar_wait(bar_full + 8u * stA, parA);
    if (hasB) mbar_wait(bar_full + 8u * stB, parB);
    const uint32_t svA = stages_s + (uint32_t)stA * a.stage_bytes, svB = stages_s + (uint32_t)stB * a.stage_bytes;
    auto aligned = [&](int rows) {
      return ((uint32_t)rows * K * 8) % 16 == 0 && ((uint32_t)rows * K * 4) % 16 == 0 &&
             ((uint32_t)rows * 8) % 16 == 0;
    };
    const bool smA = aligned(rowsA), smB = aligned(rowsB);
    const int64_t row0A = s0 * m, row0B = s0B * m;
    double* qA = qbuf + (size_t)qbA * rows_c;
    double* qB = qbuf + (size_t)qbB * rows_c;
    const int rmax = rowsA > rowsB ? rowsA : rowsB;
    for (int rb = warp * GPW; rb < rmax; rb += kTmaConsumers * GPW) {
      const int r = rb + grp;
      double accA = row_partial(r, rowsA, smA, svA, svA + val_bytes_c, row0A);
      double accB = hasB ? row_partial(r, rowsB, smB, svB, svB + val_bytes_c, row0B) : 0.0;
      accA = group_sum<G>(accA);
      accB = group_sum<G>(accB);
      if (gl == 0) {
        if (r < rowsA) {
          const double g = smA ? lds_f64(svA + val_bytes_c + col_bytes_c + (uint32_t)r * 8u)
                               : __ldg(a.cost + row0A + r);
          qA[r] = add_rn(g, mul_rn(gamma, accA));
        }
        if (r < rowsB) {
          const double g = smB ? lds_f64(svB + val_bytes_c + col_bytes_c + (uint32_t)r * 8u)
                               : __ldg(a.cost + row0B + r);
          qB[r] = add_rn(g, mul_rn(gamma, accB));
        }
      }
    }
    __syncwarp();
    // release the stages and count arrivals; the last warp finishes the chunk
    int lastA = 0, lastB = 0;
    if (lane == 0) {
      mbar_arrive(bar_empty + 8u * stA);
      if (hasB) mbar_arrive(bar_empty + 8u * stB);
      __threadfence_block();
      lastA = atomicAdd(&cnt[qbA], 1) == kTmaConsumers - 1;
      if (hasB) lastB = atomicAdd(&cnt[qbB], 1) == kTmaConsumers - 1;
    }
    lastA = __shfl_sync(kFull, lastA, 0);
    lastB = __shfl_sync(kFull, lastB, 0);
    if (lastA) {
      __threadfence_block();
      finish_chunk(c, s0, nsA, qA);
      if (lane == 0) cnt[qbA] = 0;
    }
    if (lastB) {
      __threadfence_block();
      finish_chunk(c + 1, s0B, nsB, qB);
      if (lane == 0) cnt[qbB] = 0;
    }
    // advance by the number of chunks consumed (1 or 2)
    const int step = hasB ? 2 : 1;
    for (int k = 0; k < step; ++k) {
      if (++st == NS) {
        st = 0;
        parity ^= 1u;
      }
      if (++qb == QB) qb = 0;
    }
    if (!hasB) c -= 1;  // consumed only chunk c
  }
  if (a.res_bits) {
    res = warp_max(res);
    if (lane == 0) red[warp] = res;
    consumer_sync();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kTmaConsumers; ++w) t = fmax(t, red[w]);
      atomicMax(a.res_bits, (unsigned long long)__double_as_longlong(t));
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
template <int G, bool WIN>
static int launch_tma_t(const K1TmaArgs& a, int blocks, int smem, cudaStream_t st) {
  auto fn = k1_bellman_tma<G, WIN>;
  cudaError_t e = raise_smem_limit(fn, smem);
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("k1 tma smem attr: ") + cudaGetErrorString(e));
  fn<<<blocks, kTmaThreads, smem, st>>>(a);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

// Plan: chunk size SC (states), stages NS, super-chunk size, window capacity.
// Returns false when the TMA path does not apply (non-uniform or odd K).
bool k1_tma_plan(int64_t n_states_max_cta, int m, int K, int halo, int64_t n_global, int* SC,
                 int* NS, int* super_states, int* win_cap, int* stage_bytes, int* smem_bytes) {
  if (K <= 0 || (K & 1)) return false;
  const int budget = 225 * 1024;
  const int row_bytes = K * 12 + 8;
  // chunk: >= 8 KB and >= 2 states, 16-byte friendly (even rows)
  int sc = 1;
  while ((int64_t)sc * m * row_bytes < 12 * 1024) sc *= 2;
  if (sc * m % 4) sc *= 4;
  const int stage = ((sc * m * row_bytes + 127) / 128) * 128;
  int wcap = 0, sup = 1 << 30;
  if (halo >= 0) {
    sup = 1024;
    int64_t w = (int64_t)sup + 2 * (int64_t)halo;
    if (w > n_global) w = n_global;
    if (n_states_max_cta + 2 * (int64_t)halo <= w) w = std::min<int64_t>(n_global, n_states_max_cta + 2 * (int64_t)halo);
    wcap = (int)w;
    sup = std::max(sc, (int)((wcap - 2 * (int64_t)halo) / sc) * sc);
    if (wcap >= n_global) sup = 1 << 30;  // whole V resident: never reload
    if (sup < sc) return false;
  }
  wcap = (wcap + 15) / 16 * 16;  // keep the stage ring 128-byte aligned (TMA dst)
  const int fixed = 256 + wcap * 8 + 12 * sc * m * 8 + 1024;  // q buffers: NS+2 <= 10
  int ns = (budget - fixed) / stage;
  if (ns > 8) ns = 8;
  if (ns < 2) return false;
  *SC = sc;
  *NS = ns;
  *super_states = sup;
  *win_cap = wcap;
  *stage_bytes = stage;
  *smem_bytes = fixed + ns * stage;
  return true;
}

int launch_bellman_tma(ipi_mdp* h, const double* v_full, int32_t mode, int32_t* policy,
                       double* applied, double* g_pi, int32_t* len_pi,
                       unsigned long long* res_bits, cudaStream_t st) {
  const ipi_plan& p = h->plan;
  K1TmaArgs a;
  a.bounds = h->tma_bounds;
  a.col = h->col;
  a.val = h->val;
  a.cost = h->cost;
  a.v = v_full;
  a.n_global = h->n_global;
  a.state0 = h->state0;
  a.m = h->m;
  a.K = p.row_len_max;
  a.halo = h->tma_halo;
  a.SC = h->tma_sc;
  a.NS = h->tma_ns;
  a.super_states = h->tma_super;
  a.win_cap = h->tma_wcap;
  a.stage_bytes = h->tma_stage;
  a.gamma = h->gamma;
  a.maximize = mode == IPI_MODE_MAX;
  a.policy = policy;
  a.applied = applied;
  a.gpi = g_pi;
  a.lenpi = len_pi;
  a.res_bits = res_bits;
  int G = 0, P = 0;
  if (!uniform_shape(a.K, &G, &P)) return fail(IPI_EVALIDATION, "tma path needs uniform even rows");
  const bool win = a.halo >= 0;
#define IPI_TMA(GG) return win ? launch_tma_t<GG, true>(a, h->tma_blocks, h->tma_smem, st) \
                              : launch_tma_t<GG, false>(a, h->tma_blocks, h->tma_smem, st)
  switch (G) {
    case 1: IPI_TMA(1);
    case 2: IPI_TMA(2);
    case 4: IPI_TMA(4);
    case 8: IPI_TMA(8);
    case 16: IPI_TMA(16);
    default: IPI_TMA(32);
  }
#undef IPI_TMA
}

}  // namespace ipi
