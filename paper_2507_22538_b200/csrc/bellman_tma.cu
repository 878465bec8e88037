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
  double* qbuf = reinterpret_cast<double*>(p);               // 2 x SC*m doubles
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
      for (int64_t c = 0; c < nchunks; ++c) {
        const int st = (int)(c % NS);
        if (c >= NS) mbar_wait(bar_empty + 8u * st, (uint32_t)(((c / NS) - 1) & 1));
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
      }
    }
    return;
  }

  // ========================= consumers =======================================
  constexpr int GPW = 32 / G;
  const int grp = lane / G, gl = lane % G;
  const int pairs = K >> 1;
  const bool mx = a.maximize != 0;
  const double gamma = a.gamma;
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

  for (int64_t c = 0; c < nchunks; ++c) {
    const int st = (int)(c % NS);
    const int64_t s0 = s_lo + c * SC;
    const int ns = (int)((s_hi - s0) < SC ? (s_hi - s0) : SC);
    const int rows = ns * m;
    // super-chunk boundary: reload the V window (consumers only)
    if (WIN && (c * SC) % a.super_states == 0) {
      consumer_sync();  // nobody still gathers from the old window
      int64_t lo = a.state0 + s0 - a.halo;
      int64_t send = s0 + a.super_states;
      if (send > s_hi) send = s_hi;
      int64_t hi = a.state0 + send + a.halo;
      lo = lo < 0 ? 0 : lo;
      hi = hi > a.n_global ? a.n_global : hi;
      w_lo = (int)lo;
      w_len = (uint32_t)(hi - lo);
      for (uint32_t i = tid; i < w_len; i += kTmaConsumers * 32) win[i] = __ldg(a.v + lo + i);
      consumer_sync();
    }
    mbar_wait(bar_full + 8u * st, (uint32_t)((c / NS) & 1));
    const uint32_t vb = (uint32_t)rows * K * 8, cb = (uint32_t)rows * K * 4, gb = (uint32_t)rows * 8;
    const bool in_smem = (vb % 16 == 0) && (cb % 16 == 0) && (gb % 16 == 0);
    const uint32_t sv = stages_s + (uint32_t)st * a.stage_bytes;
    const uint32_t sc = sv + val_bytes_c, sg = sc + col_bytes_c;
    const int64_t row0 = s0 * m;
    double* q = qbuf + (size_t)(c & 1) * rows_c;
    // ---- rows: q = cost + gamma * (P V) ------------------------------------
    for (int rb = warp * GPW; rb < rows; rb += kTmaConsumers * GPW) {
      const int r = rb + grp;
      double acc = 0.0;
      if (r < rows) {
        for (int j = gl; j < pairs; j += G) {
          double2 v2;
          int2 c2;
          const int e = r * K + 2 * j;
          if (in_smem) {
            v2 = lds_v2f64(sv + (uint32_t)e * 8u);
            c2 = lds_v2s32(sc + (uint32_t)e * 4u);
          } else {
            v2 = *reinterpret_cast<const double2*>(a.val + row0 * K + e);
            c2 = *reinterpret_cast<const int2*>(a.col + row0 * K + e);
          }
          acc = add_rn(acc, mul_rn(v2.x, gather(c2.x)));
          acc = add_rn(acc, mul_rn(v2.y, gather(c2.y)));
        }
      }
      acc = group_sum<G>(acc);
      if (r < rows && gl == 0) {
        const double g = in_smem ? lds_f64(sg + (uint32_t)r * 8u) : __ldg(a.cost + row0 + r);
        q[r] = add_rn(g, mul_rn(gamma, acc));
      }
    }
    consumer_sync();  // all rows of the chunk are in q; the stage is free
    if (lane == 0) mbar_arrive(bar_empty + 8u * st);
    // ---- per-state first-index argmin (warp per state) ---------------------
    for (int t = warp; t < ns; t += kTmaConsumers) {
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
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
  const int fixed = 256 + wcap * 8 + 2 * sc * m * 8 + 1024;
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
