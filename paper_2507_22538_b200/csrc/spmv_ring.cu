// spmv_ring.cu — K3 fast paths: the policy operator J_pi = I - gamma*P_pi
// applied to a vector (PolicyOperator.apply, sparse.py:272-295; spmv,
// sparse.py:189-215) for P_pi with uniform row length, which is what K2
// produces from every BASELINE instance except C4.
//
// Same streaming scheme as K1's rings (bellman.cu): every warp owns a
// contiguous row range and moves it through a private S-stage shared-memory
// ring with cp.async (16-byte chunks, lane l copies chunk l, L2 evict-first),
// so nothing in flight occupies registers.  Two shapes:
//
//   * k3_uring (9 <= K <= 129, K % 4 == 0; C2/C5: K = 64): a step is 4 rows x
//     8 lanes.  The row sum restates numpy's reduceat arithmetic exactly
//     (a[0] + pairwise(a[1:]); 8 running sums folded ((r0+r1)+(r2+r3))+
//     ((r4+r5)+(r6+r7)), leftovers in order), so P x is bitwise the
//     reference's spmv and apply() is bitwise x - gamma*spmv(x), the
//     identity test_sparse.py:191-196 asserts.  V gathers of step i+1 are
//     issued before step i is reduced; x[s] for the identity term is one of
//     them.
//   * k3_flat (K in {2, 4}; C3: K = 4): lane = row, 32 rows per stage, rows
//     summed as p0 + (((0 + p1) + p2) + p3) (numpy's order for segments
//     shorter than 9), gathers two batches ahead, coalesced y / b traffic.
//
// Optional shared-memory window of x ([state0+r_lo-halo, state0+r_hi+halo)),
// staged with cp.async alongside the first ring stages, for locality
// instances (C2: halo 4096 covers 90% of the gathers).
// Epilogues (EPI): 0 y = P x; 1 y = x - gamma*(P x); 2 y = b - (x - gamma*(P x));
// 3 y = b + gamma*(P x) — the same four as spmv.cu.
#include <string>

#include "handle.cuh"

namespace ipi {

struct K3Args {
  const int32_t* col;
  const double* val;
  int64_t rows;      // local rows; row r is state state0 + r
  int64_t state0;    // x index of row 0 (identity term, window centre)
  int64_t n_global;  // length of x
  const double* x;
  const double* b;
  double gamma;
  double* y;
  int halo;
  int pf;  // uniform ring: L2 bulk prefetch distance in steps beyond the ring (0 = off)
  unsigned long long* trace;  // diagnostics: per-CTA (smid, start ns, end ns) or nullptr
  int interleave;  // uniform ring: warp w takes 4-row steps w, w+NW, ... of its CTA (else a contiguous range)
  const int* active;  // stepped GMRES (krylov_step.cu): skip the launch when *active == 0 (nullable)
  int pdl;  // launched with programmatic stream serialization: x, b and *active are read only
            // after griddep_wait(); the first ring stages (P_pi, never written here) go out before it
};

__device__ __forceinline__ unsigned long long k3_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void k3_trace_begin(const K3Args& a) {
  if (a.trace && threadIdx.x == 0) {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    a.trace[3 * blockIdx.x] = r;
    a.trace[3 * blockIdx.x + 1] = k3_ns();
  }
}
__device__ __forceinline__ void k3_trace_end(const K3Args& a) {
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) a.trace[3 * blockIdx.x + 2] = k3_ns();
  }
}

template <int EPI>
__device__ __forceinline__ double k3_epi(double px, double xd, double bb, double gamma) {
  if (EPI == 0) return px;
  if (EPI == 3) return add_rn(bb, mul_rn(gamma, px));
  const double ax = sub_rn(xd, mul_rn(gamma, px));
  return EPI == 1 ? ax : sub_rn(bb, ax);
}

// Contiguous row range of CTA c, rounded to multiples of `align` rows so every
// warp step starts on an aligned row (16-byte b chunks).
__device__ __forceinline__ int64_t k3_split(int64_t rows, int64_t c, int64_t parts, int64_t align) {
  if (c >= parts) return rows;
  const int64_t r = (rows * c / parts) / align * align;
  return r < rows ? r : rows;
}

// Issue the x window of rows [r_lo, r_hi) into shared memory as ONE cp.async
// commit group (16-byte chunks, every thread's copies in flight at once; the
// window start is rounded down to an even index so chunks are aligned).  The
// caller waits for the group and barriers before the first gather.
__device__ __forceinline__ void k3_window_issue(const K3Args& a, unsigned char* win, int64_t r_lo,
                                                int64_t r_hi, int& w_lo, uint32_t& w_len) {
  int64_t lo = a.state0 + r_lo - a.halo;
  int64_t hi = a.state0 + r_hi + a.halo;
  lo = lo < 0 ? 0 : lo;
  hi = hi > a.n_global ? a.n_global : hi;
  lo &= ~(int64_t)1;
  w_lo = (int)lo;
  w_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
  const uint64_t keep = policy_evict_last();
  const uint32_t win_s = (uint32_t)__cvta_generic_to_shared(win);
  const uint32_t nch = (w_len + 1) >> 1;
  for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x)
    cp_async16(win_s + 16 * c, a.x + lo + 2 * c, 2 * c + 1 < w_len ? 16u : 8u, keep);
  cp_async_commit();
}

// ---------------------------------------------------------------------------
// uniform rows, 4 rows x 8 lanes per step
// ---------------------------------------------------------------------------
template <int K>
struct K3URing {
  static constexpr int kVal = 4 * K * 8;
  static constexpr int kCol = 4 * K * 4;
  static constexpr int kStage = kVal + kCol + 32;  // + 4 b entries
};

int k3_uring_smem(int K, int stages, int warps, int window_bytes) {
  const int st = 4 * K * 12 + 32;
  return ((window_bytes + 15) & ~15) + warps * (stages * st + 256);
}

template <int K, int NW, int S, int EPI, bool WIN>
__global__ void __launch_bounds__(NW * 32, 1) k3_uring(K3Args a, int win_bytes) {
  constexpr int N1 = K - 1, NC = N1 / 8, TAIL = N1 % 8;
  static_assert(N1 >= 8 && N1 <= 128 && K % 4 == 0, "uniform ring: 9 <= K <= 129, K % 4 == 0");
  static_assert(S >= 3, "ring needs 3 stages (one-step gather lookahead)");
  using L = K3URing<K>;
  constexpr bool NEED_B = EPI >= 2, NEED_XD = EPI == 1 || EPI == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const bool early = a.pdl && !WIN && !NEED_B;  // prologue before the predecessor has finished
  if (a.pdl && !early) griddep_wait();
  if (!early && a.active && *a.active == 0) return;  // stepped GMRES: the cycle already ended
  k3_trace_begin(a);
  double* win = reinterpret_cast<double*>(smem_raw);
  const int64_t r_lo = k3_split(a.rows, blockIdx.x, gridDim.x, 4);
  const int64_t r_hi = k3_split(a.rows, blockIdx.x + 1, gridDim.x, 4);
  int w_lo = 0;
  uint32_t w_len = 0;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, j = lane & 7;
  unsigned char* ring = smem_raw + (((WIN ? win_bytes : 0) + 15) & ~15) + warp * (S * L::kStage + 256);
  double* tb = reinterpret_cast<double*>(ring + S * L::kStage);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const double* __restrict__ xg = a.x;
  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) return win[off];
    }
    return __ldg(xg + c);
  };
  const int64_t nr = r_hi - r_lo;
  // rows of step i: [w0 + 4*rs*i, +4) clipped to w1
  int64_t w0, w1, nb, rs;
  if (a.interleave) {  // the CTA's warps read one contiguous stream
    const int64_t groups = (nr + 3) >> 2;
    w0 = r_lo + 4 * warp;
    w1 = r_hi;
    nb = groups > warp ? (groups - warp + NW - 1) / NW : 0;
    rs = NW;
  } else {
    w0 = r_lo + (nr * warp / NW) / 4 * 4;
    w1 = warp + 1 == NW ? r_hi : r_lo + (nr * (warp + 1) / NW) / 4 * 4;
    nb = (w1 - w0 + 3) >> 2;
    rs = 1;
  }

  auto issue = [&](int64_t i, int stg) {
    if (i < nb) {
      const int64_t row0 = w0 + 4 * rs * i;
      const int64_t left = w1 - row0;
      const int nrow = left < 4 ? (int)left : 4;
      const uint32_t st = ring_s + (uint32_t)(stg * L::kStage);
      const double* vp = a.val + row0 * K;
      const int* cp = a.col + row0 * K;
#pragma unroll
      for (int c = lane; c < 4 * K / 2; c += 32) {
        const int r = c / (K / 2), cc = c % (K / 2);
        const bool ok = r < nrow;
        cp_async16(st + r * K * 8 + 16 * (cc ^ ((r & 1) << 2)), ok ? vp + 2 * c : vp, ok ? 16 : 0, pol);
      }
#pragma unroll
      for (int c = lane; c < 4 * K / 4; c += 32) {
        const int r = c / (K / 4), cc = c % (K / 4);
        const bool ok = r < nrow;
        cp_async16(st + L::kVal + r * K * 4 + 16 * (cc ^ (r << 1)), ok ? cp + 4 * c : cp, ok ? 16 : 0, pol);
      }
      if (a.pf > 0 && lane < 2 && i + a.pf < nb) {  // DRAM -> L2 ahead of the ring
        const int64_t rp0 = row0 + 4 * rs * (int64_t)a.pf;
        const int64_t lp = w1 - rp0;
        const int np = lp < 4 ? (int)lp : 4;
        if (lane == 0) l2_prefetch(a.val + rp0 * K, (uint32_t)(np * K * 8));
        else l2_prefetch(a.col + rp0 * K, (uint32_t)(np * K * 4));
      }
      if (NEED_B && lane < 2) {
        const int have = nrow - 2 * lane;  // rows of this 16-byte chunk present
        const uint32_t bytes = have >= 2 ? 16u : (have == 1 ? 8u : 0u);
        cp_async16(st + L::kVal + L::kCol + 16 * lane, a.b + row0 + (bytes ? 2 * lane : 0), bytes, pol);
      }
    }
    cp_async_commit();
  };
  auto caddr = [&](int r, int e) {
    return L::kVal + r * K * 4 + ((((e >> 2) ^ (r << 1))) << 4) + ((e & 3) << 2);
  };
  auto vaddr = [&](int r, int e) {
    return r * K * 8 + ((((e >> 1) ^ ((r & 1) << 2))) << 4) + ((e & 1) << 3);
  };
  constexpr int NG = NC + 2;  // chain terms, the leftover / first term, x[s]
  const bool has_last = j < TAIL || j == 7;
  const int e_last = j < TAIL ? 1 + 8 * NC + j : 0;
  auto fetch = [&](int64_t i, int stg, double (&x)[NG]) {
    const unsigned char* st = ring + stg * L::kStage;
#pragma unroll
    for (int k = 0; k < NC; ++k) x[k] = gather(*reinterpret_cast<const int*>(st + caddr(grp, 1 + j + 8 * k)));
    if (has_last) x[NC] = gather(*reinterpret_cast<const int*>(st + caddr(grp, e_last)));
    if (NEED_XD && j == 0) {
      const int64_t row = w0 + 4 * rs * i + grp;
      if (row < w1) x[NC + 1] = gather((int)(a.state0 + row));
    }
  };
  auto compute = [&](int64_t i, int stg, const double (&x)[NG]) {
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
    if (j == 0) {
      const int64_t row = w0 + 4 * rs * i + grp;
      if (row < w1) {
        const double* t = tb + (grp << 3);
#pragma unroll
        for (int q = 0; q < TAIL; ++q) r = add_rn(r, t[q]);
        const double px = add_rn(t[7], r);
        const double bb = NEED_B ? reinterpret_cast<const double*>(st + L::kVal + L::kCol)[grp] : 0.0;
        a.y[row] = k3_epi<EPI>(px, x[NC + 1], bb, a.gamma);
      }
    }
  };
  int stg = 0;
  auto step = [&](int64_t i, const double (&cur)[NG], double (&ahead)[NG]) {
    const int sd = stg + 1 >= S ? stg + 1 - S : stg + 1;
    cp_async_wait<S - 2>();  // step i+1 landed (this lane's copies)
    __syncwarp();            // ... and every lane's
    if (i + 1 < nb) fetch(i + 1, sd, ahead);
    compute(i, stg, cur);
    __syncwarp();  // stage i and the tail buffer consumed
    issue(i + S, stg);
    stg = stg + 1 == S ? 0 : stg + 1;
  };
  // window copies (one group) and the first S ring stages go out together
  if (WIN) k3_window_issue(a, smem_raw, r_lo, r_hi, w_lo, w_len);
#pragma unroll 1
  for (int q = 0; q < S; ++q) issue(q, q);
  if (early) {  // P_pi's first stages are in flight; x and *active need the predecessor
    griddep_wait();
    if (a.active && *a.active == 0) {
      cp_async_wait<0>();
      return;
    }
  }
  if (a.pdl) griddep_launch_dependents();
  if (WIN) {
    cp_async_wait<S>();  // the window group landed (this thread's copies)
    __syncthreads();     // ... and every thread's
  }
  if (nb > 0) {
    double x0[NG], x1[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) x0[k] = x1[k] = 0.0;
    cp_async_wait<S - 1>();
    __syncwarp();
    fetch(0, 0, x0);
#pragma unroll 1
    for (int64_t i = 0; i < nb; i += 2) {
      step(i, x0, x1);
      if (i + 1 < nb) step(i + 1, x1, x0);
    }
  }
  cp_async_wait<0>();
  k3_trace_end(a);
}

// ---------------------------------------------------------------------------
// flat rows (K in {2, 4}): lane = row, 32 rows per stage
// ---------------------------------------------------------------------------
template <int K>
struct K3Flat {
  static constexpr int kVal = 32 * K * 8;
  static constexpr int kCol = 32 * K * 4;
  static constexpr int kStage = kVal + kCol + 256;  // + 32 b entries
};

int k3_flat_smem(int K, int stages, int warps, int window_bytes) {
  const int st = 32 * K * 12 + 256;
  return ((window_bytes + 15) & ~15) + warps * stages * st;
}

template <int K, int NW, int S, int EPI, bool WIN>
__global__ void __launch_bounds__(NW * 32, 1) k3_flat(K3Args a, int win_bytes) {
  static_assert(K == 2 || K == 4, "flat ring handles K = 2 or 4");
  static_assert(S >= 4, "ring needs 4 stages (gathers two batches ahead)");
  using L = K3Flat<K>;
  if (a.pdl) {
    griddep_wait();
    griddep_launch_dependents();
  }
  constexpr bool NEED_B = EPI >= 2, NEED_XD = EPI == 1 || EPI == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (a.active && *a.active == 0) return;  // stepped GMRES: the cycle already ended
  k3_trace_begin(a);
  double* win = reinterpret_cast<double*>(smem_raw);
  const int64_t r_lo = k3_split(a.rows, blockIdx.x, gridDim.x, 32);
  const int64_t r_hi = k3_split(a.rows, blockIdx.x + 1, gridDim.x, 32);
  int w_lo = 0;
  uint32_t w_len = 0;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = smem_raw + (((WIN ? win_bytes : 0) + 15) & ~15) + warp * S * L::kStage;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint32_t off = (uint32_t)(c - w_lo);
      if (off < w_len) return win[off];
    }
    return __ldg(a.x + c);
  };
  const int64_t nr = r_hi - r_lo;
  const int64_t w0 = r_lo + (nr * warp / NW) / 32 * 32;
  const int64_t w1 = warp + 1 == NW ? r_hi : r_lo + (nr * (warp + 1) / NW) / 32 * 32;
  const int64_t nb = (w1 - w0 + 31) >> 5;

  auto issue = [&](int64_t i, int stg) {
    if (i < nb) {
      const int64_t base = w0 + (i << 5);
      const int64_t left = w1 - base;
      const int nrow = left < 32 ? (int)left : 32;
      const uint32_t st = ring_s + (uint32_t)(stg * L::kStage);
      const double* vp = a.val + base * K;
#pragma unroll
      for (int c = lane; c < 32 * K / 2; c += 32)
        if (c < nrow * K / 2) cp_async16(st + 16 * c, vp + 2 * c, 16, pol);
      if (K == 4) {
        if (lane < nrow) cp_async16(st + L::kVal + 16 * lane, a.col + (base + lane) * 4, 16, pol);
      } else {
        if (lane < nrow) cp_async8(st + L::kVal + 8 * lane, a.col + (base + lane) * 2);
      }
      if (NEED_B && lane < 16) {
        const int have = nrow - 2 * lane;
        const uint32_t bytes = have >= 2 ? 16u : (have == 1 ? 8u : 0u);
        cp_async16(st + L::kVal + L::kCol + 16 * lane, a.b + base + (bytes ? 2 * lane : 0), bytes, pol);
      }
    }
    cp_async_commit();
  };
  constexpr int NG = K + 1;  // K gathers + x[s]
  auto fetch = [&](int64_t i, int stg, double (&x)[NG]) {
    const int64_t row = w0 + (i << 5) + lane;
    if (i < nb && row < w1) {
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
      if (NEED_XD) x[K] = gather((int)(a.state0 + row));
    }
  };
  auto compute = [&](int64_t i, int stg, const double (&x)[NG]) {
    const int64_t row = w0 + (i << 5) + lane;
    if (row < w1) {
      const unsigned char* st = ring + stg * L::kStage;
      const double2 v0 = *reinterpret_cast<const double2*>(st + lane * K * 8);
      double acc = add_rn(0.0, mul_rn(v0.y, x[1 % K]));
      if (K == 4) {
        const double2 v1 = *reinterpret_cast<const double2*>(st + lane * K * 8 + 16);
        acc = add_rn(acc, mul_rn(v1.x, x[2 % K]));
        acc = add_rn(acc, mul_rn(v1.y, x[3 % K]));
      }
      acc = add_rn(mul_rn(v0.x, x[0]), acc);
      const double bb = NEED_B ? reinterpret_cast<const double*>(st + L::kVal + L::kCol)[lane] : 0.0;
      a.y[row] = k3_epi<EPI>(acc, x[K], bb, a.gamma);
    }
  };
  int stg = 0;
  auto step = [&](int64_t i, const double (&cur)[NG], double (&ahead)[NG]) {
    const int s2 = stg + 2 >= S ? stg + 2 - S : stg + 2;
    cp_async_wait<S - 3>();
    __syncwarp();
    fetch(i + 2, s2, ahead);
    compute(i, stg, cur);
    __syncwarp();
    issue(i + S, stg);
    stg = stg + 1 == S ? 0 : stg + 1;
  };
  if (WIN) k3_window_issue(a, smem_raw, r_lo, r_hi, w_lo, w_len);
#pragma unroll 1
  for (int q = 0; q < S; ++q) issue(q, q);
  if (WIN) {
    cp_async_wait<S>();
    __syncthreads();
  }
  if (nb > 0) {
    double x0[NG], x1[NG], x2[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) x0[k] = x1[k] = x2[k] = 0.0;
    cp_async_wait<S - 2>();
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
  k3_trace_end(a);
}

// ---------------------------------------------------------------------------
// instances and dispatch
// ---------------------------------------------------------------------------
// (warps, stages) shapes with an instance
#define IPI_K3U_SHAPES(M) M(64, 12, 3) M(64, 16, 3) M(64, 8, 4) M(64, 10, 3) M(64, 14, 3) M(64, 15, 3) M(64, 11, 3) M(64, 13, 3) M(64, 12, 4) M(64, 13, 4) M(64, 10, 4)
#define IPI_K3F_SHAPES(M) M(4, 16, 4) M(4, 8, 6) M(4, 24, 4) M(4, 28, 4) M(4, 20, 5) M(2, 16, 4) M(2, 24, 4)

template <class F>
static cudaError_t k3_attr(F fn, int smem) {
  return raise_smem_limit(fn, smem);
}

template <int K, int NW, int S, bool WIN>
static cudaError_t k3u_attr_all(int smem) {
  cudaError_t e = k3_attr(k3_uring<K, NW, S, 0, WIN>, smem);
  if (e == cudaSuccess) e = k3_attr(k3_uring<K, NW, S, 1, WIN>, smem);
  if (e == cudaSuccess) e = k3_attr(k3_uring<K, NW, S, 2, WIN>, smem);
  if (e == cudaSuccess) e = k3_attr(k3_uring<K, NW, S, 3, WIN>, smem);
  return e;
}
template <int K, int NW, int S, bool WIN>
static cudaError_t k3f_attr_all(int smem) {
  cudaError_t e = k3_attr(k3_flat<K, NW, S, 0, WIN>, smem);
  if (e == cudaSuccess) e = k3_attr(k3_flat<K, NW, S, 1, WIN>, smem);
  if (e == cudaSuccess) e = k3_attr(k3_flat<K, NW, S, 2, WIN>, smem);
  if (e == cudaSuccess) e = k3_attr(k3_flat<K, NW, S, 3, WIN>, smem);
  return e;
}

bool k3_shape_prepare(int variant, int K, int NW, int S, bool win, int smem) {
  bool ok = false;
  cudaError_t e = cudaSuccess;
#define IPI_K3U_ATTR(KK, WW, SS)                                                          \
  if (!ok && variant == IPI_K3_URING && K == KK && NW == WW && S == SS) {                  \
    ok = true;                                                                            \
    e = win ? k3u_attr_all<KK, WW, SS, true>(smem) : k3u_attr_all<KK, WW, SS, false>(smem); \
  }
#define IPI_K3F_ATTR(KK, WW, SS)                                                          \
  if (!ok && variant == IPI_K3_FLAT && K == KK && NW == WW && S == SS) {                   \
    ok = true;                                                                            \
    e = win ? k3f_attr_all<KK, WW, SS, true>(smem) : k3f_attr_all<KK, WW, SS, false>(smem); \
  }
  IPI_K3U_SHAPES(IPI_K3U_ATTR)
  IPI_K3F_SHAPES(IPI_K3F_ATTR)
#undef IPI_K3U_ATTR
#undef IPI_K3F_ATTR
  if (e != cudaSuccess) cudaGetLastError();
  return ok && e == cudaSuccess;
}

template <class Kern>
static void k3_go(Kern kern, const ipi_op* op, int threads, const K3Args& a, int wb, cudaStream_t st) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(op->blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = (size_t)op->smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, a, wb);
}

template <int EPI>
static bool k3_launch_epi(const ipi_op* op, const K3Args& a, cudaStream_t st) {
  bool ok = false;
  const bool win = op->win_bytes > 0;
  const int wb = op->win_bytes;
#define IPI_K3U_GO(KK, WW, SS)                                                                   \
  if (!ok && op->variant == IPI_K3_URING && op->K == KK && op->warps == WW && op->stages == SS) { \
    ok = true;                                                                                   \
    if (win) k3_go(k3_uring<KK, WW, SS, EPI, true>, op, WW * 32, a, wb, st);                      \
    else k3_go(k3_uring<KK, WW, SS, EPI, false>, op, WW * 32, a, 0, st);                          \
  }
#define IPI_K3F_GO(KK, WW, SS)                                                                  \
  if (!ok && op->variant == IPI_K3_FLAT && op->K == KK && op->warps == WW && op->stages == SS) { \
    ok = true;                                                                                  \
    if (win) k3_go(k3_flat<KK, WW, SS, EPI, true>, op, WW * 32, a, wb, st);                      \
    else k3_go(k3_flat<KK, WW, SS, EPI, false>, op, WW * 32, a, 0, st);                          \
  }
  IPI_K3U_SHAPES(IPI_K3U_GO)
  IPI_K3F_SHAPES(IPI_K3F_GO)
#undef IPI_K3U_GO
#undef IPI_K3F_GO
  return ok;
}

// y = epi(P x) over the operator's rows; generic rows use spmv.cu's kernel.
int op_launch(const ipi_op* op, const double* x_full, const double* b, int epi, double* y,
              cudaStream_t st, const double* y_partial, const int* active, int pdl) {
  if (op->n_local <= 0) return IPI_OK;
  if (op->variant == IPI_K3_GENERIC || epi >= 4)  // split halves: generic rows
    return launch_spmv(op->rp, op->col, op->val, op->n_local, x_full, b, op->gamma, epi, y,
                       op->lanes, st, op->state0, y_partial);
  K3Args a{op->col, op->val, op->n_local, op->state0, op->n_global, x_full, b, op->gamma, y, op->halo,
            op->pf, op->trace, op->interleave, active, pdl};
  bool ok = false;
  switch (epi) {
    case 0: ok = k3_launch_epi<0>(op, a, st); break;
    case 1: ok = k3_launch_epi<1>(op, a, st); break;
    case 2: ok = k3_launch_epi<2>(op, a, st); break;
    default: ok = k3_launch_epi<3>(op, a, st); break;
  }
  if (!ok) return fail(IPI_ECUDA, "K3: no kernel instance for the planned shape");
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
