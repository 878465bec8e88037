// krylov.cuh — persistent policy-evaluation kernel shared by the krylov*.cu units.
#pragma once
// K4: policy evaluation (I - gamma P_pi) x = b as ONE persistent
// cooperative kernel per inner solve (inner.py:163-292).
//
// Why persistent: GMRES(30) with modified Gram-Schmidt needs j+1 dependent
// grid-wide reductions per Arnoldi step.  Launch-per-op would pay a kernel
// launch plus a host round trip per dot (C1/C4 vectors are 80-160 KB, i.e.
// microsecond kernels).  Here every CTA owns a contiguous, nnz-balanced slice
// of rows/vector entries; reductions are two-level and deterministic (fixed
// intra-CTA tree -> per-CTA partial -> every CTA sums all partials in the
// same fixed order), so every CTA holds bit-identical scalars and runs the
// reference's control logic (Givens, est_target tightening, caps) redundantly
// without any broadcast.  Grid barriers are cooperative-groups grid syncs.
//
// Semantics mirrored exactly (inner.py line refs):
//   eff = max(target, 1e-14*max(1,||b||))           :189
//   Richardson: r=b-A th; stop if rn<=eff|it>=cap|!finite; th += scale*r   :216-226
//   GMRES: restart 30, MGS, Givens, break on |g_j|<=est or hnorm==0,
//          true residual per cycle, est_target = |g_j|*(eff/rn)*0.5       :229-283
//   back substitution with zero-pivot -> 0                                 :286-292
// Every vector op uses separate mul/add roundings like numpy (no FMA).
#include <cooperative_groups.h>

#include <algorithm>
#include <string>

#include "handle.cuh"

namespace cg = cooperative_groups;

namespace ipi {

constexpr int R = kGmresRestart;
constexpr int kKindGmresCgs = 4;  // inner_kernel KIND of GMRES with CGS2 orthogonalisation

struct KArgs {
  const int64_t* rp;
  const int32_t* col;
  const double* val;
  int64_t n;
  double gamma;
  const double* b;
  double* x;
  double* V;         // (R+1) * n Krylov basis
  double* w;         // n
  double* r;         // n
  double* partials;  // [2 slots][kPartStride values][grid]: value-major, so the CTA
                     // partials of one value are contiguous for the reducing warp
  double target;
  int max_it;
  int kind;
  double scale;
  int halo;
  int win_cap;   // doubles of the shared-memory window (0 = none)
  int own_cap;   // doubles of the shared-memory w slice (0 = w in global)
  int K;         // uniform row length of P_pi (0 = variable)
  const double* invd;  // Jacobi: 1 / (1 - gamma diag(P_pi)); nullptr = identity (inner.py:113-118)
  ipi_inner_report* rep;
  unsigned* bar;       // grid barrier counter, zeroed before every launch
  int bar_mode;        // GridBarrier::mode (IPI_K4_BARRIER)
  float keep_frac;     // fraction of P_pi accesses marked L2 evict-last (0 = evict-first)
  int xwin;            // stage the SpMV input window (else the window space only holds MGS slices)
  int contig;          // generic rows: columns consecutive within each row (CONTIG instances)
  int ortho;           // GMRES Arnoldi orthogonalisation (resolved): IPI_ORTHO_MGS / IPI_ORTHO_CGS2
  unsigned long long* trace;  // diagnostics (ipi_k4_trace): phase timestamps or nullptr
  int trace_cap;
};

// Diagnostics: CTA 0 records %globaltimer at phase boundaries (trace[1..]);
// trace[0] counts the records.
__device__ __forceinline__ void k4_mark_raw(unsigned long long* trace, int cap) {
  if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    const unsigned long long k = trace[0];
    if ((int)k + 1 < cap) {
      trace[k + 1] = t;
      trace[0] = k + 1;
    }
  }
}
__device__ __forceinline__ void k4_mark(const KArgs& a) { k4_mark_raw(a.trace, a.trace_cap); }
// the buffer ipi_k4_trace enabled (nullptr when off)
unsigned long long* k4_trace_buffer(int* cap);

// doubles per CTA and slot in the all-reduce partials (the CGS dot vector:
// up to R projections + one norm)
constexpr int kPartStride = 32;

// Grid barrier for the co-resident (cooperatively launched) CTAs: one release
// add per CTA on a monotone counter + an acquire spin by the CTA's leader.
// Measured on B200 (scripts/micro/barrier_micro.cu, 148 x 1024 threads):
// 2.4 us per deterministic all-reduce vs 4.1 us with cooperative-groups
// grid.sync().  `epoch` advances in every thread so all agree on the target.
struct GridBarrier {
  unsigned* ctr;
  unsigned epoch;
  int mode;  // 0: release add + acquire spin, 1: cooperative-groups grid.sync(),
            // 2: as 0 with backoff, 3: as 0 plus full fences
  __device__ __forceinline__ void arrive_and_wait(bool leader) {
    ++epoch;
    if (mode == 1) {
      cg::this_grid().sync();
      return;
    }
    if (leader) {
      // red.release (MEMBAR.ALL.GPU + RED) and ld.acquire (LDG.STRONG.GPU +
      // CCTL.IVALL: the SM's L1 is invalidated, so the CTA's later plain loads
      // cannot hit stale lines) carry the ordering; the CTA's own writes are
      // ordered before the leader by __syncthreads.  Mode 3 adds full SC fences
      // around them (C4 GMRES step 0.098 vs 0.089 ms without).
      if (mode == 3) __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
      const unsigned target = epoch * gridDim.x;
      unsigned seen;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
        if (seen >= target) break;
        if (mode == 2) __nanosleep(64);
      }
      if (mode == 3) __threadfence();
    }
  }
  __device__ __forceinline__ void sync() {
    __syncthreads();
    arrive_and_wait(threadIdx.x == 0);
    __syncthreads();
  }
};

struct KShared {
  double red[64];
  double bc[4];
  double red8[8 * 32];           // block level of an 8-wide chunk (vector all-reduce)
  double vpart[kPartStride];     // this CTA's partials of a vector all-reduce
  double cv[kPartStride];        // CGS: first projection  c = V^T w  (+ ||w||^2)
  double dv[kPartStride];        // CGS: re-orthogonalisation  d = V^T w1
  double H[(R + 1) * R];
  double cs[R], sn[R], g[R + 1], y[R];
  int iflag[4];
};

// Two-level deterministic all-reduce of NV doubles; result in every thread.
// Block level: warp xor trees, one shared-memory exchange for all NV values,
// warp 0 xor tree; grid level: per-CTA partials, the grid barrier, every CTA
// sums all partials in the same order.  Four CTA barriers per call (the
// broadcast slot sh.bc is next written only after two barriers of the next call).
template <int NV>
__device__ __forceinline__ void grid_allreduce(double (&v)[NV], const KArgs& a, int& slot,
                                               GridBarrier& gb, KShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double t[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) t[k] = warp_sum(v[k]);
  __syncthreads();  // sh.red free (previous call's warp 0 finished reading it)
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sh.red[k * 32 + warp] = t[k];
  }
  __syncthreads();
  const int nblk = gridDim.x;
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) t[k] = warp_sum(lane < nw ? sh.red[k * 32 + lane] : 0.0);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) a.partials[((int64_t)slot * kPartStride + k) * nblk + blockIdx.x] = t[k];
    }
  }
  gb.arrive_and_wait(threadIdx.x == 0);
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int i = lane; i < nblk; i += 32)
        s = add_rn(s, __ldcg(a.partials + ((int64_t)slot * kPartStride + k) * nblk + i));
      s = warp_sum(s);
      if (lane == 0) sh.bc[k] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sh.bc[k];
  slot ^= 1;
}

// Block level of a vector all-reduce: the block sums of acc[0..7] (fixed xor
// trees: warp, then warp 0..7 over the per-warp values) go to
// sh.vpart[base + k] for base + k < cnt.
__device__ __forceinline__ void block_accumulate8(const double (&acc)[8], int base, int cnt,
                                                  KShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) t[k] = warp_sum(acc[k]);
  __syncthreads();  // sh.red8 free (previous chunk's readers done)
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) sh.red8[k * 32 + warp] = t[k];
  }
  __syncthreads();
  if (warp < 8 && base + warp < cnt) {
    const double v = warp_sum(lane < nw ? sh.red8[warp * 32 + lane] : 0.0);
    if (lane == 0) sh.vpart[base + warp] = v;
  }
}

// Grid level of a vector all-reduce of sh.vpart[0..cnt) (cnt <= kPartStride):
// per-CTA partials, the grid barrier, then value k is summed over the CTAs in
// CTA order by warp k % nwarps (fixed order: every CTA gets bit-identical
// results) into out[k] (shared memory).  Ends with a CTA barrier.
__device__ __forceinline__ void grid_allreduce_vec(int cnt, double* out, const KArgs& a, int& slot,
                                                   GridBarrier& gb, KShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nblk = gridDim.x;
  __syncthreads();  // sh.vpart complete
  if ((int)threadIdx.x < cnt)
    a.partials[((int64_t)slot * kPartStride + threadIdx.x) * nblk + blockIdx.x] = sh.vpart[threadIdx.x];
  __syncthreads();  // every lane's partial ordered before the leader's release
  gb.arrive_and_wait(threadIdx.x == 0);
  __syncthreads();
  for (int k = warp; k < cnt; k += nw) {
    double s = 0.0;
    for (int i = lane; i < nblk; i += 32)
      s = add_rn(s, __ldcg(a.partials + ((int64_t)slot * kPartStride + k) * nblk + i));
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
  __syncthreads();
  slot ^= 1;
}

// CGS projections of this CTA's slice of w onto the basis: out[l] = <V_l, w>
// for l < nv and, when with_norm, out[nv] = <w, w>.  One coalesced pass over
// the nv basis slices (8 in flight per thread), then one vector all-reduce.
__device__ __forceinline__ void cgs_dots(const KArgs& a, int nv, bool with_norm, const double* wl,
                                         int64_t s_lo, int64_t s_hi, uint64_t pol, double* out,
                                         int& slot, GridBarrier& gb, KShared& sh) {
  const int cnt = nv + (with_norm ? 1 : 0);
  const int64_t n = a.n;
  for (int l0 = 0; l0 < cnt; l0 += 8) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 2
    for (int64_t i = s_lo + threadIdx.x; i < s_hi; i += blockDim.x) {
      const double wi = wl[i - s_lo];
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = l0 + u < nv ? ld_hint(a.V + (int64_t)(l0 + u) * n + i, pol) : wi;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (l0 + u < cnt) acc[u] = add_rn(acc[u], mul_rn(v[u], wi));
    }
    block_accumulate8(acc, l0, cnt, sh);
  }
  grid_allreduce_vec(cnt, out, a, slot, gb, sh);
}

// w <- w - sum_{l < nv} coef[l] V_l over this CTA's slice (l ascending, separate
// roundings); returns this thread's share of ||w||^2.
__device__ __forceinline__ double cgs_update(const KArgs& a, int nv, const double* coef, double* wl,
                                             int64_t s_lo, int64_t s_hi, uint64_t pol) {
  const int64_t n = a.n;
  double q = 0.0;
  for (int64_t i = s_lo + threadIdx.x; i < s_hi; i += blockDim.x) {
    double t = wl[i - s_lo];
    for (int l0 = 0; l0 < nv; l0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = l0 + u < nv ? ld_hint(a.V + (int64_t)(l0 + u) * n + i, pol) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (l0 + u < nv) t = sub_rn(t, mul_rn(coef[l0 + u], v[u]));
    }
    wl[i - s_lo] = t;
    q = add_rn(q, mul_rn(t, t));
  }
  return q;
}

// Row sums of P_pi over this CTA's rows with an optional shared-memory window
// of the input vector; epi(s, Px_s, x_s) is called by one lane per row, x_s
// being the input's own entry (from the window when it is resident).  P == 0:
// generic rows (G lanes strided over the row, 4 loads in flight); P > 0:
// uniform even-length rows, P 16-byte value pairs per lane, batches
// software-pipelined across row groups (same scheme as K1's fast path).
template <int G, int P, bool WIN, bool CONTIG, class Epi>
__device__ __forceinline__ void spmv_rows(const KArgs& a, const double* xin, int64_t s_lo,
                                          int64_t s_hi, double* win, uint64_t pol, Epi&& epi) {
  int64_t w_lo = 0, w_len = 0;
  if (WIN) {
    int64_t lo = s_lo - a.halo, hi = s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n ? a.n : hi;
    __syncthreads();
    if (a.xwin && hi - lo <= a.win_cap) {  // all copies in flight at once (8-byte cp.async)
      w_lo = lo;
      w_len = hi - lo;
      const uint32_t ws = (uint32_t)__cvta_generic_to_shared(win);
      for (int64_t i = threadIdx.x; i < w_len; i += blockDim.x) cp_async8(ws + (uint32_t)(8 * i), xin + lo + i);
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();
  }
  auto gather = [&](int c) -> double {
    if (WIN) {
      const uint64_t off = (uint64_t)((int64_t)c - w_lo);
      if (off < (uint64_t)w_len) return win[off];
    }
    return xin[c];
  };
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / G, gl = lane % G;
  if constexpr (P == 0) {
    for (int64_t base = s_lo + (int64_t)warp * GPW; base < s_hi; base += (int64_t)nwarps * GPW) {
      const int64_t s = base + grp;
      double acc = 0.0;
      if (s < s_hi) {
        const int64_t p0 = __ldg(a.rp + s), p1 = __ldg(a.rp + s + 1);
        int c0 = 0;  // CONTIG: consecutive columns, entry q's column is c0 + (q - p0)
        if constexpr (CONTIG) c0 = p1 > p0 ? __ldg(a.col + p0) : 0;
        for (int64_t p = p0 + gl; p < p1; p += 4 * G) {
          double vv[4];
          int cc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
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
          double xx[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) xx[u] = cc[u] >= 0 ? gather(cc[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cc[u] >= 0) acc = add_rn(acc, mul_rn(vv[u], xx[u]));
        }
      }
      acc = group_sum<G>(acc);
      if (s < s_hi && gl == 0) epi(s, acc, gather((int)s));
    }
  } else {
    const int K = a.K, pairs = K >> 1;
    auto load = [&](int64_t base, Batch<P>& b) {
      const int64_t s = base + grp;
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const int j = gl + G * t;
        if (s < s_hi && j < pairs) {
          b.v[t] = ld_stream_v2(a.val + s * K + 2 * j, pol);
          b.c[t] = ld_stream_v2(a.col + s * K + 2 * j, pol);
        } else {
          b.v[t] = make_double2(0.0, 0.0);
          b.c[t] = make_int2(-1, -1);
        }
      }
    };
    int64_t base = s_lo + (int64_t)warp * GPW;
    if (base < s_hi) {
      Batch<P> cur, nxt;
      load(base, cur);
      while (true) {
        const int64_t nb = base + (int64_t)nwarps * GPW;
        const bool has_next = nb < s_hi;
        if (has_next) load(nb, nxt);
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
        const int64_t s = base + grp;
        if (s < s_hi && gl == 0) epi(s, acc, gather((int)s));
        if (!has_next) break;
        cur = nxt;
        base = nb;
      }
    }
  }
}

// KIND: 0 = GMRES (MGS) + Richardson (runtime a.kind), 4 = GMRES (CGS2) +
// Richardson, 2 = BiCGStab, 3 = TFQMR.  Each
// solver family is its own instantiation (and translation unit) so the hot
// GMRES kernel does not carry the register pressure of the others.
template <int G, int P, bool WIN, int KIND, bool CONTIG = false>
__global__ void __launch_bounds__(kInnerThreads, 1) inner_kernel(KArgs a) {
  GridBarrier gb{a.bar, 0u, a.bar_mode};
  extern __shared__ double win[];
  __shared__ KShared sh;
  // P_pi is re-read by every SpMV of the solve: when it is not much larger than
  // L2, mark that fraction of its lines evict-last so repeated SpMVs hit L2
  // (C4: 137 MB P_pi vs 126 MB L2); large P_pi streams evict-first.
  uint64_t pol;
  if (a.keep_frac > 0.f)
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;"
                 : "=l"(pol) : "f"(a.keep_frac));
  else
    pol = policy_evict_first();
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nblk = gridDim.x;
  const int64_t n = a.n;
  const int64_t nnz = a.rp[n];
  // nnz-balanced contiguous row slice (identical rule in every CTA)
  const int64_t s_lo =
      blockIdx.x == 0 ? 0 : lower_bound_i64(a.rp, n + 1, (nnz * (int64_t)blockIdx.x) / nblk);
  const int64_t s_hi = blockIdx.x == nblk - 1
                           ? n
                           : lower_bound_i64(a.rp, n + 1, (nnz * (int64_t)(blockIdx.x + 1)) / nblk);
  const double gam = a.gamma;
  const double* b = a.b;
  double* x = a.x;
  double* r = a.r;
  // this CTA's slice of w: shared memory when it fits, else its global rows
  const bool w_shared = (s_hi - s_lo) <= a.own_cap;
  double* wl = w_shared ? (win + a.win_cap) : (a.w + s_lo);
  // GMRES MGS passes on shared-memory copies of the basis slices (see below)
  const bool staged = WIN && w_shared && 2 * (s_hi - s_lo) <= (int64_t)a.win_cap;
  int slot = 0;

  // ---- r = b - (x - gamma P x), ||b||, ||r|| --------------------------------
  double acc2[2] = {0.0, 0.0};
  for (int64_t i = s_lo + tid; i < s_hi; i += nthr) acc2[0] = add_rn(acc2[0], mul_rn(b[i], b[i]));
  spmv_rows<G, P, WIN, CONTIG>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
    const double ri = sub_rn(b[s], sub_rn(xs, mul_rn(gam, px)));
    r[s] = ri;
    acc2[1] = add_rn(acc2[1], mul_rn(ri, ri));
  });
  grid_allreduce<2>(acc2, a, slot, gb, sh);
  const double bnorm = sqrt(acc2[0]);
  const double rr0 = acc2[1];
  double rn = sqrt(rr0);
  int brk = 0;
  // true residual r = b - A x (x complete after a grid sync); returns ||r||
  auto true_residual = [&]() -> double {
    gb.sync();
    double q[1] = {0.0};
    spmv_rows<G, P, WIN, CONTIG>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
      const double ri = sub_rn(b[s], sub_rn(xs, mul_rn(gam, px)));
      r[s] = ri;
      q[0] = add_rn(q[0], mul_rn(ri, ri));
    });
    grid_allreduce<1>(q, a, slot, gb, sh);
    return sqrt(q[0]);
  };
  const double eff = fmax(a.target, 1e-14 * fmax(1.0, bnorm));
  int it = 0;
  // left preconditioner pc(v)[s] (identity or Jacobi: elementwise multiply)
  const double* invd = a.invd;
  auto pcv = [&](int64_t s, double v) -> double { return invd ? mul_rn(v, invd[s]) : v; };
  // z = pc(r) on own rows into dst; returns ||z||^2 (the same sum rn^2 when pc = I)
  auto precond_residual = [&](double* dst) -> double {
    double q[1] = {0.0};
    for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
      const double z = pcv(i, r[i]);
      dst[i] = z;
      q[0] = add_rn(q[0], mul_rn(z, z));
    }
    if (!invd) return -1.0;  // caller reuses rn^2
    grid_allreduce<1>(q, a, slot, gb, sh);
    return q[0];
  };

  if constexpr (KIND == IPI_KSP_TFQMR) {
    // ---- TFQMR (inner.py:376-450) ------------------------------
    double* r0 = a.V;
    double* wv = a.V + n;
    double* yv = a.V + 2 * n;
    double* dv = a.V + 3 * n;
    double* uv = a.V + 4 * n;
    double* vv = a.V + 5 * n;
    double* vt = a.V + 6 * n;
    bool stale = false;
    if (!(rn <= eff)) {
      const double zz = precond_residual(r0);     // r0 = pc(r_true)
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
        const double ri = r0[i];
        wv[i] = ri;
        yv[i] = ri;
        dv[i] = 0.0;
      }
      gb.sync();
      double p2[2] = {0.0, 0.0};
      spmv_rows<G, P, WIN, CONTIG>(a, yv, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
        const double u = pcv(s, sub_rn(xs, mul_rn(gam, px)));
        uv[s] = u;
        vv[s] = u;
        p2[0] = add_rn(p2[0], mul_rn(r0[s], u));
        p2[1] = add_rn(p2[1], mul_rn(u, u));
      });
      const double r0nn = invd ? sqrt(zz) : rn;
      double tau = r0nn, thq = 0.0, eta = 0.0, rho = invd ? zz : rr0, est_target = eff;
      const double r0n = r0nn;
      while (it < a.max_it) {
        grid_allreduce<2>(p2, a, slot, gb, sh);
        const double sigma = p2[0], vn = sqrt(p2[1]);
        if (fabs(sigma) <= mul_rn(mul_rn(1e-14, r0n), vn)) { brk = 1; break; }
        const double alpha = rho / sigma;
        if (alpha == 0.0 || !isfinite(alpha)) { brk = 1; break; }
        bool conv = false;
        double pw[2] = {0.0, 0.0};
        for (int half = 1; half <= 2; ++half) {
          const double coef = mul_rn(mul_rn(thq, thq), eta) / alpha;
          pw[0] = pw[1] = 0.0;
          if (half == 1) {
            for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
              const double w = sub_rn(wv[i], mul_rn(alpha, uv[i]));
              wv[i] = w;
              dv[i] = add_rn(yv[i], mul_rn(coef, dv[i]));
              pw[0] = add_rn(pw[0], mul_rn(w, w));
            }
          } else {
            for (int64_t i = s_lo + tid; i < s_hi; i += nthr) yv[i] = sub_rn(yv[i], mul_rn(alpha, vv[i]));
            gb.sync();
            spmv_rows<G, P, WIN, CONTIG>(a, yv, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
              const double u = pcv(s, sub_rn(xs, mul_rn(gam, px)));
              uv[s] = u;
              const double w = sub_rn(wv[s], mul_rn(alpha, u));
              wv[s] = w;
              dv[s] = add_rn(xs, mul_rn(coef, dv[s]));
              pw[0] = add_rn(pw[0], mul_rn(w, w));
              pw[1] = add_rn(pw[1], mul_rn(r0[s], w));
            });
          }
          if (tau == 0.0) { brk = 1; break; }
          if (half == 1) {
            double q1[1] = {pw[0]};
            grid_allreduce<1>(q1, a, slot, gb, sh);
            pw[0] = q1[0];
          } else {
            grid_allreduce<2>(pw, a, slot, gb, sh);
          }
          thq = sqrt(pw[0]) / tau;
          const double c = 1.0 / sqrt(add_rn(1.0, mul_rn(thq, thq)));
          tau = mul_rn(mul_rn(tau, thq), c);
          eta = mul_rn(mul_rn(c, c), alpha);
          for (int64_t i = s_lo + tid; i < s_hi; i += nthr) x[i] = add_rn(x[i], mul_rn(eta, dv[i]));
          stale = true;
          const double est = mul_rn(tau, sqrt(add_rn(add_rn(mul_rn(2.0, (double)it), (double)half), 1.0)));
          if (est <= est_target) {
            rn = true_residual();
            stale = false;
            if (rn <= eff) { conv = true; break; }
            if (est == 0.0) { brk = 1; break; }
            est_target = fmin(est_target, mul_rn(mul_rn(est, eff / rn), 0.5));
          }
        }
        ++it;
        if (conv || brk) break;
        const double rho_new = pw[1], wn = sqrt(pw[0]);
        if (fabs(rho_new) <= mul_rn(mul_rn(1e-14, r0n), wn)) { brk = 1; break; }
        const double beta = rho_new / rho;
        rho = rho_new;
        const double b2 = mul_rn(beta, beta);
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
          yv[i] = add_rn(wv[i], mul_rn(beta, yv[i]));
          vt[i] = add_rn(mul_rn(beta, uv[i]), mul_rn(b2, vv[i]));
        }
        gb.sync();
        p2[0] = p2[1] = 0.0;
        spmv_rows<G, P, WIN, CONTIG>(a, yv, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
          const double u = pcv(s, sub_rn(xs, mul_rn(gam, px)));
          uv[s] = u;
          const double v = add_rn(vt[s], u);
          vv[s] = v;
          p2[0] = add_rn(p2[0], mul_rn(r0[s], v));
          p2[1] = add_rn(p2[1], mul_rn(v, v));
        });
      }
      if (stale || brk) rn = true_residual();
    }
  } else if constexpr (KIND == IPI_KSP_BICGSTAB) {
    // ---- BiCGStab (inner.py:295-373) ---------------------------
    double* rv = a.V;          // recurrence residual
    double* rt = a.V + n;      // shadow residual
    double* pv = a.V + 2 * n;
    double* vv = a.V + 3 * n;
    double* sv = a.V + 4 * n;
    double* tv = a.V + 5 * n;
    bool stale = false;
    if (!(rn <= eff)) {
      double zz = precond_residual(rv);           // r = pc(r_true)
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
        const double ri = rv[i];
        rt[i] = ri;
        pv[i] = ri;
      }
      double rtn = invd ? sqrt(zz) : rn, rho = invd ? zz : rr0, est = rtn, est_target = eff;
      while (it < a.max_it) {
        if (fabs(rho) <= mul_rn(mul_rn(1e-14, rtn), est)) { brk = 1; break; }
        gb.sync();
        double p2[2] = {0.0, 0.0};
        spmv_rows<G, P, WIN, CONTIG>(a, pv, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
          const double v = pcv(s, sub_rn(xs, mul_rn(gam, px)));
          vv[s] = v;
          p2[0] = add_rn(p2[0], mul_rn(rt[s], v));
          p2[1] = add_rn(p2[1], mul_rn(v, v));
        });
        grid_allreduce<2>(p2, a, slot, gb, sh);
        const double sigma = p2[0];
        if (fabs(sigma) <= mul_rn(mul_rn(1e-14, rtn), sqrt(p2[1]))) { brk = 1; break; }
        const double alpha = rho / sigma;
        double q1[1] = {0.0};
        __syncthreads();
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
          const double sval = sub_rn(rv[i], mul_rn(alpha, vv[i]));
          sv[i] = sval;
          q1[0] = add_rn(q1[0], mul_rn(sval, sval));
        }
        grid_allreduce<1>(q1, a, slot, gb, sh);
        const double s_norm = sqrt(q1[0]);
        if (s_norm <= est_target) {
          for (int64_t i = s_lo + tid; i < s_hi; i += nthr) x[i] = add_rn(x[i], mul_rn(alpha, pv[i]));
          ++it;
          gb.sync();
          double q[1] = {0.0};
          spmv_rows<G, P, WIN, CONTIG>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
            const double ri = sub_rn(b[s], sub_rn(xs, mul_rn(gam, px)));
            r[s] = ri;
            q[0] = add_rn(q[0], mul_rn(ri, ri));
          });
          grid_allreduce<1>(q, a, slot, gb, sh);
          rn = sqrt(q[0]);
          stale = false;
          if (rn <= eff) break;
          est_target = fmin(est_target, mul_rn(mul_rn(s_norm, eff / rn), 0.5));
          zz = precond_residual(rv);
          for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
            const double ri = rv[i];
            rt[i] = ri;
            pv[i] = ri;
          }
          rtn = invd ? sqrt(zz) : rn;
          rho = invd ? zz : q[0];
          est = rtn;
          continue;
        }
        gb.sync();
        double p3[2] = {0.0, 0.0};
        spmv_rows<G, P, WIN, CONTIG>(a, sv, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
          const double t = pcv(s, sub_rn(xs, mul_rn(gam, px)));
          tv[s] = t;
          p3[0] = add_rn(p3[0], mul_rn(t, t));
          p3[1] = add_rn(p3[1], mul_rn(t, sv[s]));
        });
        grid_allreduce<2>(p3, a, slot, gb, sh);
        const double tt = p3[0];
        if (tt == 0.0) { brk = 1; break; }
        const double omega = p3[1] / tt;
        if (omega == 0.0 || !isfinite(omega)) { brk = 1; break; }
        double p4[2] = {0.0, 0.0};
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
          x[i] = add_rn(add_rn(x[i], mul_rn(alpha, pv[i])), mul_rn(omega, sv[i]));
          const double rnew = sub_rn(sv[i], mul_rn(omega, tv[i]));
          rv[i] = rnew;
          p4[0] = add_rn(p4[0], mul_rn(rnew, rnew));
          p4[1] = add_rn(p4[1], mul_rn(rt[i], rnew));
        }
        ++it;
        stale = true;
        grid_allreduce<2>(p4, a, slot, gb, sh);
        est = sqrt(p4[0]);
        if (est <= est_target) {
          rn = true_residual();
          stale = false;
          if (rn <= eff) break;
          if (est == 0.0) break;
          est_target = fmin(est_target, mul_rn(mul_rn(est, eff / rn), 0.5));
        }
        const double rho_new = p4[1];
        const double beta = mul_rn(rho_new / rho, alpha / omega);
        if (!isfinite(beta)) { brk = 1; break; }
        rho = rho_new;
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr)
          pv[i] = add_rn(rv[i], mul_rn(beta, sub_rn(pv[i], mul_rn(omega, vv[i]))));
      }
      if (stale || brk) rn = true_residual();
    }
  } else   if (a.kind == IPI_KSP_RICHARDSON) {
    while (true) {
      if (rn <= eff || it >= a.max_it || !isfinite(rn)) break;
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr)
        x[i] = add_rn(x[i], mul_rn(a.scale, pcv(i, r[i])));
      ++it;
      gb.sync();
      double acc1[1] = {0.0};
      spmv_rows<G, P, WIN, CONTIG>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
        const double ri = sub_rn(b[s], sub_rn(xs, mul_rn(gam, px)));
        r[s] = ri;
        acc1[0] = add_rn(acc1[0], mul_rn(ri, ri));
      });
      grid_allreduce<1>(acc1, a, slot, gb, sh);
      rn = sqrt(acc1[0]);
    }
  } else {  // GMRES(30)
    double est_target = eff;
    while (rn > eff && it < a.max_it) {
      // z = pc(r); beta = ||z|| (with pc = I: same vector and reduction as rn)
      const double zz = precond_residual(a.V);
      const double beta = invd ? sqrt(zz) : rn;
      if (beta == 0.0 || !isfinite(beta)) break;
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) a.V[i] = a.V[i] / beta;
      __syncthreads();  // every thread has read the previous cycle's sh.g
      if (tid == 0) {
        for (int k = 0; k < (R + 1) * R; ++k) sh.H[k] = 0.0;
        for (int k = 0; k < R; ++k) sh.cs[k] = sh.sn[k] = 0.0;
        for (int k = 0; k <= R; ++k) sh.g[k] = 0.0;
        sh.g[0] = beta;
      }
      int j = 0;
      gb.sync();
      while (j < R && it < a.max_it) {
        const double* Vj = a.V + (int64_t)j * n;
        const double* V0 = a.V;
        double p[1] = {0.0};
        if constexpr (KIND == kKindGmresCgs) k4_mark(a);
        spmv_rows<G, P, WIN, CONTIG>(a, Vj, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
          wl[s - s_lo] = pcv(s, sub_rn(xs, mul_rn(gam, px)));
        });
        ++it;
        __syncthreads();  // w rows written by group leaders, read per-thread below
        if constexpr (KIND == kKindGmresCgs) {
          if (a.trace) gb.sync();  // diagnostics: every CTA's SpMV done
          k4_mark(a);
          // Classical Gram-Schmidt with one re-orthogonalisation when needed
          // (DGKS test, ||w1|| < ||w||/sqrt(2)): 2 all-reduces per step instead of
          // MGS's j+2 (inner.py:251-253 uses MGS; the projections agree to rounding).
          cgs_dots(a, j + 1, true, wl, s_lo, s_hi, pol_last, sh.cv, slot, gb, sh);
          k4_mark(a);
          const double nw = sh.cv[j + 1];
          double q1[1] = {cgs_update(a, j + 1, sh.cv, wl, s_lo, s_hi, pol_last)};
          grid_allreduce<1>(q1, a, slot, gb, sh);
          k4_mark(a);
          double nw1 = q1[0];
          const bool reorth = nw1 < 0.5 * nw;  // uniform across the grid
          if (reorth) {
            cgs_dots(a, j + 1, false, wl, s_lo, s_hi, pol_last, sh.dv, slot, gb, sh);
            double q2[1] = {cgs_update(a, j + 1, sh.dv, wl, s_lo, s_hi, pol_first)};
            grid_allreduce<1>(q2, a, slot, gb, sh);
            nw1 = q2[0];
          }
          k4_mark(a);
          if (tid == 0) {
            for (int l = 0; l <= j; ++l) sh.H[l * R + j] = reorth ? add_rn(sh.cv[l], sh.dv[l]) : sh.cv[l];
          }
          p[0] = nw1;
        } else if (staged) {
          // MGS with the basis slices staged in shared memory (the V window is
          // idle until the next SpMV): V_{l+1} is copied with cp.async before
          // the all-reduce that produces h_l, so each pass costs one barrier
          // and shared-memory arithmetic.  Same per-thread element order and
          // roundings as the global-memory passes below (bit-identical).
          const int64_t own_n = s_hi - s_lo;
          const uint32_t vb_s = (uint32_t)__cvta_generic_to_shared(win);
          auto stage = [&](int l, int buf) {
            const double* Vs = a.V + (int64_t)l * n + s_lo;
            const uint32_t dst = vb_s + (uint32_t)(buf * own_n * 8);
            for (int64_t i = tid; i < own_n; i += nthr) cp_async8(dst + (uint32_t)(i * 8), Vs + i);
            cp_async_commit();
          };
          stage(0, 0);
          cp_async_wait<0>();
          for (int64_t i = tid; i < own_n; i += nthr) p[0] = add_rn(p[0], mul_rn(win[i], wl[i]));
          for (int l = 0; l <= j; ++l) {
            if (l < j) stage(l + 1, (l + 1) & 1);
            grid_allreduce<1>(p, a, slot, gb, sh);
            const double hlj = p[0];
            if (tid == 0) sh.H[l * R + j] = hlj;
            if (l < j) cp_async_wait<0>();
            const double* vl = win + (l & 1) * own_n;
            const double* vn = win + ((l + 1) & 1) * own_n;
            double q = 0.0;
            if (l < j) {
              for (int64_t i = tid; i < own_n; i += nthr) {
                const double wi = sub_rn(wl[i], mul_rn(hlj, vl[i]));
                wl[i] = wi;
                q = add_rn(q, mul_rn(vn[i], wi));
              }
            } else {
              for (int64_t i = tid; i < own_n; i += nthr) {
                const double wi = sub_rn(wl[i], mul_rn(hlj, vl[i]));
                wl[i] = wi;
                q = add_rn(q, mul_rn(wi, wi));
              }
            }
            p[0] = q;
          }
        } else {
          // h_0 partial in a coalesced pass (keeps dependent V0 loads out of the SpMV)
          for (int64_t i = s_lo + tid; i < s_hi; i += nthr)
            p[0] = add_rn(p[0], mul_rn(ld_hint(V0 + i, pol_last), wl[i - s_lo]));
          for (int l = 0; l <= j; ++l) {
            grid_allreduce<1>(p, a, slot, gb, sh);
            const double hlj = p[0];
            if (tid == 0) sh.H[l * R + j] = hlj;
            const double* Vl = a.V + (int64_t)l * n;
            const double* Vn = a.V + (int64_t)(l + 1) * n;
            double q = 0.0;
            // L2 reuse: V_{l+1} is read here and again as V_l by the next pass
            // (evict-last); this is V_l's last read in the step (evict-first).
            // w never aliases the basis: restrict + unroll batch the loads.
            double* __restrict__ wr = wl - s_lo;
            if (l < j && !w_shared) {  // w in global: keep it L2-resident too
  #pragma unroll 4
              for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
                const double wi = sub_rn(ld_hint(wr + i, pol_last), mul_rn(hlj, ld_hint(Vl + i, pol_first)));
                st_hint(wr + i, wi, pol_last);
                q = add_rn(q, mul_rn(ld_hint(Vn + i, pol_last), wi));
              }
            } else if (l < j) {
  #pragma unroll 4
              for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
                const double wi = sub_rn(wr[i], mul_rn(hlj, ld_hint(Vl + i, pol_first)));
                wr[i] = wi;
                q = add_rn(q, mul_rn(ld_hint(Vn + i, pol_last), wi));
              }
            } else {
  #pragma unroll 4
              for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
                const double wi = sub_rn(wr[i], mul_rn(hlj, ld_hint(Vl + i, pol_first)));
                wr[i] = wi;
                q = add_rn(q, mul_rn(wi, wi));
              }
            }
            p[0] = q;
          }
        }
        if constexpr (KIND != kKindGmresCgs) grid_allreduce<1>(p, a, slot, gb, sh);
        const double hnorm = sqrt(p[0]);
        if (tid == 0) {
          double* H = sh.H;
          H[(j + 1) * R + j] = hnorm;
          for (int l = 0; l < j; ++l) {
            const double hl = H[l * R + j], hl1 = H[(l + 1) * R + j];
            const double t = add_rn(mul_rn(sh.cs[l], hl), mul_rn(sh.sn[l], hl1));
            H[(l + 1) * R + j] = add_rn(mul_rn(-sh.sn[l], hl), mul_rn(sh.cs[l], hl1));
            H[l * R + j] = t;
          }
          const double denom = hypot(H[j * R + j], H[(j + 1) * R + j]);
          int brk = 0;
          if (denom == 0.0) {
            brk = 1;
          } else {
            sh.cs[j] = H[j * R + j] / denom;
            sh.sn[j] = H[(j + 1) * R + j] / denom;
            H[j * R + j] = denom;
            H[(j + 1) * R + j] = 0.0;
            sh.g[j + 1] = mul_rn(-sh.sn[j], sh.g[j]);
            sh.g[j] = mul_rn(sh.cs[j], sh.g[j]);
            if (fabs(sh.g[j + 1]) <= est_target || hnorm == 0.0) brk = 2;
          }
          sh.iflag[0] = brk;
        }
        __syncthreads();
        const int brk = sh.iflag[0];
        if (brk == 1) break;  // denom == 0: j not advanced
        ++j;
        if (brk == 2) break;  // estimated convergence / invariant subspace
        double* Vnew = a.V + (int64_t)j * n;
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr)  // next SpMV input: keep in L2
          st_hint(Vnew + i, wl[i - s_lo] / hnorm, pol_last);
        gb.sync();
        if constexpr (KIND == kKindGmresCgs) k4_mark(a);
      }
      if (j == 0) break;
      if (tid == 0) {  // back substitution (inner.py:286-292)
        for (int i = j - 1; i >= 0; --i) {
          double dacc = 0.0;
          for (int k = i + 1; k < j; ++k) dacc = add_rn(dacc, mul_rn(sh.H[i * R + k], sh.y[k]));
          const double t = sub_rn(sh.g[i], dacc);
          const double d = sh.H[i * R + i];
          sh.y[i] = d != 0.0 ? t / d : 0.0;
        }
      }
      __syncthreads();
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
        double t = 0.0;
        for (int l = 0; l < j; ++l) t = add_rn(t, mul_rn(a.V[(int64_t)l * n + i], sh.y[l]));
        x[i] = add_rn(x[i], t);
      }
      gb.sync();
      double acc1[1] = {0.0};
      spmv_rows<G, P, WIN, CONTIG>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px, double xs) {
        const double ri = sub_rn(b[s], sub_rn(xs, mul_rn(gam, px)));
        r[s] = ri;
        acc1[0] = add_rn(acc1[0], mul_rn(ri, ri));
      });
      grid_allreduce<1>(acc1, a, slot, gb, sh);
      rn = sqrt(acc1[0]);
      const double gj = fabs(sh.g[j]);
      if (rn > eff && gj <= est_target) {
        if (gj == 0.0) break;
        est_target = mul_rn(mul_rn(gj, eff / rn), 0.5);
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    a.rep->iterations = it;
    a.rep->basis_reads = 0;  // not counted by the persistent kernels
    a.rep->final_linear_residual_2norm = rn;
    a.rep->converged = (rn <= eff && !brk) ? 1 : 0;
    a.rep->breakdown = brk;
    a.rep->target_2norm = eff;
  }
}

template <int G, int P, bool WIN, int KIND, bool CONTIG = false>
static int launch_inner_t(KArgs& a, int smem, int blocks, cudaStream_t st) {
  auto fn = inner_kernel<G, P, WIN, KIND, CONTIG>;
  cudaError_t e = raise_smem_limit(fn, smem);
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("inner smem attr: ") + cudaGetErrorString(e));
  int per_sm = 0;
  IPI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kInnerThreads, smem));
  if (per_sm < 1) return fail(IPI_ECUDA, "inner kernel cannot be resident (smem/regs)");
  void* args[] = {(void*)&a};
  IPI_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(blocks), dim3(kInnerThreads), args,
                                           (size_t)smem, st));
  return IPI_OK;
}

// Launch the KIND family for the planned shape (uniform (G, P) or generic lanes).
template <int KIND>
static int dispatch_inner(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                          cudaStream_t st) {
  int rc = IPI_OK;
#define IPI_INNER_LAUNCH(GG, PP)                                                    \
  rc = win ? launch_inner_t<GG, PP, true, KIND>(a, smem, blocks, st)                \
           : launch_inner_t<GG, PP, false, KIND>(a, smem, blocks, st)
  if (P > 0) {
    IPI_DISPATCH_UNIFORM(G, P, IPI_INNER_LAUNCH);
    return rc;
  }
  if (lanes >= 32 && a.contig) {  // banded rows (C4): no column stream
    rc = win ? launch_inner_t<32, 0, true, KIND, true>(a, smem, blocks, st)
             : launch_inner_t<32, 0, false, KIND, true>(a, smem, blocks, st);
    return rc;
  }
  switch (lanes) {
    case 1: IPI_INNER_LAUNCH(1, 0); break;
    case 2: IPI_INNER_LAUNCH(2, 0); break;
    case 4: IPI_INNER_LAUNCH(4, 0); break;
    case 8: IPI_INNER_LAUNCH(8, 0); break;
    case 16: IPI_INNER_LAUNCH(16, 0); break;
    default: IPI_INNER_LAUNCH(32, 0); break;
  }
#undef IPI_INNER_LAUNCH
  return rc;
}

int dispatch_inner_gmres(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                         cudaStream_t st);
// krylov_ring.cu: uniform rows (K = 64 class) with the per-warp cp.async ring SpMV
int ring_inner_smem(int K, int NW, int S);
int ring_mgs_elems(int NW);  // slice elements per thread the ring kernel's MGS keeps in registers
bool ring_inner_has(int K, int NW, int S);
int dispatch_inner_ring(KArgs& a, int K, int NW, int S, int smem, int blocks, cudaStream_t st);
int dispatch_inner_gmres_cgs(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                             cudaStream_t st);
int dispatch_inner_bicgstab(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                            cudaStream_t st);
int dispatch_inner_tfqmr(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                         cudaStream_t st);

}  // namespace ipi
