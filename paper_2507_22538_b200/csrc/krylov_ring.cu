// krylov_ring.cu — K4 for uniform-row P_pi (9 <= K <= 129, K % 4 == 0; C2/C5:
// K = 64): the persistent GMRES(30) / Richardson kernel of krylov.cuh with
// its SpMV replaced by K3's per-warp cp.async ring (spmv_ring.cu) and the
// Arnoldi step orthogonalised by CGS2 (two grid all-reduces per step).
//
// Why a second kernel: the 1024-thread K4 (krylov.cuh) is capped at 64
// registers and streams P_pi through a register pipeline (0.65-0.72 of HBM
// per SpMV on C2).  Here NW warps (12-16) each own a private S-stage ring in
// shared memory, so nothing in flight occupies registers and the SpMV runs
// at the standalone K3 rate; the vector phases (CGS projections, updates)
// keep 8-16 independent loads in flight per thread with the registers the
// smaller CTA leaves free (<= 168 per thread).
//
// Semantics: inner.py:163-292 as in krylov.cuh (floor, it counting, Givens,
// |g_j| <= est_target break, true residual per cycle, est_target
// tightening, zero-pivot back substitution); rows are summed in numpy's
// reduceat order (a[0] + pairwise(a[1:])) exactly like K3, so one SpMV
// here equals ipi_op_apply bit for bit.  Orthogonalisation: classical
// Gram-Schmidt with DGKS re-orthogonalisation (krylov.cuh cgs_*), the
// IPI_ORTHO_CGS2 choice; MGS requests run the 1024-thread kernel.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "krylov.cuh"

namespace ipi {

// MGS keeps mgs_elems<NW> slice elements of w per thread in registers (C2:
// 7092 rows per CTA over 384 threads = 19) and stages two basis slices in the
// ring area; longer slices fall back to CGS2 (host side).
template <int NW>
constexpr int mgs_elems() { return NW >= 16 ? 14 : NW >= 12 ? 19 : NW >= 10 ? 23 : 28; }

int ring_mgs_elems(int NW) {
  return NW >= 16 ? mgs_elems<16>() : NW >= 12 ? mgs_elems<12>() : NW >= 10 ? mgs_elems<10>() : mgs_elems<8>();
}

template <int K, int NW, int S>
struct RingGeom {
  static constexpr int kVal = 4 * K * 8;
  static constexpr int kCol = 4 * K * 4;
  static constexpr int kStage = kVal + kCol;
  static constexpr int kWarp = S * kStage + 256;  // + the per-warp leftover buffer
  static constexpr int kBytes = NW * kWarp;
};

// y-row epilogue for rows [r_lo, r_hi) of P_pi (row r is state r): warps take
// interleaved 4-row steps (warp w: steps w, w + NW, ...), so the CTA reads
// one contiguous stream.  epi(row, px, x_row) is called by one lane per row.
// x is read with plain (coherent) loads: it was written earlier in this
// kernel by other CTAs, ordered by the grid barrier's release/acquire.
#ifndef IPI_K4_NOINLINE
#define IPI_K4_NOINLINE 1
#endif
#if IPI_K4_NOINLINE
#define IPI_RING_INLINE __noinline__
#else
#define IPI_RING_INLINE __forceinline__
#endif
// Returns this thread's sum of epi's return values.  Compiled as its own
// function (IPI_K4_NOINLINE): inlined into the persistent kernel the same
// loop ran 20-25% slower than as a standalone kernel (SASS of the two loops
// is the same instruction mix; the difference is the surrounding kernel's
// register and scheduling context).
template <int K, int NW, int S, bool NEED_XD, class Epi>
__device__ IPI_RING_INLINE double ring_rows(const int32_t* __restrict__ colp,
                                            const double* __restrict__ valp, const double* x,
                                            const double* __restrict__ bvec, int64_t r_lo,
                                            int64_t r_hi, unsigned char* smem_ring, uint64_t pol,
                                            Epi epi) {
  double acc = 0.0;
  using L = RingGeom<K, NW, S>;
  constexpr int N1 = K - 1, NC = N1 / 8, TAIL = N1 % 8;
  static_assert(N1 >= 8 && N1 <= 128 && K % 4 == 0, "uniform ring: 9 <= K <= 129, K % 4 == 0");
  static_assert(S >= 3, "ring needs 3 stages (one-step gather lookahead)");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, j = lane & 7;
  unsigned char* ring = smem_ring + warp * L::kWarp;
  double* tb = reinterpret_cast<double*>(ring + S * L::kStage);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const int64_t groups = (r_hi - r_lo + 3) >> 2;
  const int64_t w0 = r_lo + 4 * warp;
  const int64_t nb = groups > warp ? (groups - warp + NW - 1) / NW : 0;
  auto issue = [&](int64_t i, int stg) {
    if (i < nb) {
      const int64_t row0 = w0 + 4 * (int64_t)NW * i;
      const int64_t left = r_hi - row0;
      const int nrow = left < 4 ? (int)left : 4;
      const uint32_t st = ring_s + (uint32_t)(stg * L::kStage);
      const double* vp = valp + row0 * K;
      const int* cp = colp + row0 * K;
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
    }
    cp_async_commit();
  };
  auto caddr = [&](int r, int e) {
    return L::kVal + r * K * 4 + ((((e >> 2) ^ (r << 1))) << 4) + ((e & 3) << 2);
  };
  auto vaddr = [&](int r, int e) {
    return r * K * 8 + ((((e >> 1) ^ ((r & 1) << 2))) << 4) + ((e & 1) << 3);
  };
  constexpr int NG = NC + 3;  // chain terms, the leftover / first term, x[row], b[row]
  const bool has_last = j < TAIL || j == 7;
  const int e_last = j < TAIL ? 1 + 8 * NC + j : 0;
#ifndef IPI_K4_LDG
#define IPI_K4_LDG 1
#endif
  // Gathers through the read-only path (LDG.CONSTANT), as K3 does.  x was
  // written earlier in this launch, which .nc loads may only read after every
  // SM's L1 has dropped its older lines: the grid barrier before every SpMV
  // ends with the leader's ld.acquire.gpu, which invalidates the SM's unified
  // L1 / texture cache (CCTL.IVALL), so no line of x cached before the
  // barrier survives into this pass (the reruns in test_gpu_k4_ring.py check
  // the results bit for bit against the coherent-load build).
  auto gx = [&](int64_t c) -> double {
#if IPI_K4_LDG
    return __ldg(x + c);
#else
    return x[c];
#endif
  };
  auto fetch = [&](int64_t i, int stg, double (&xv)[NG]) {
    const unsigned char* st = ring + stg * L::kStage;
#pragma unroll
    for (int k = 0; k < NC; ++k) xv[k] = gx(*reinterpret_cast<const int*>(st + caddr(grp, 1 + j + 8 * k)));
    if (has_last) xv[NC] = gx(*reinterpret_cast<const int*>(st + caddr(grp, e_last)));
    if (NEED_XD && j == 0) {
      const int64_t row = w0 + 4 * (int64_t)NW * i + grp;
      if (row < r_hi) {
        xv[NC + 1] = gx(row);
        if (bvec) xv[NC + 2] = __ldg(bvec + row);  // b is an input: never written in-kernel
      }
    }
  };
  auto compute = [&](int64_t i, int stg, const double (&xv)[NG]) {
    const unsigned char* st = ring + stg * L::kStage;
    auto val = [&](int e) { return *reinterpret_cast<const double*>(st + vaddr(grp, e)); };
    tb[lane] = has_last ? mul_rn(val(e_last), xv[NC]) : 0.0;
    double r = mul_rn(val(1 + j), xv[0]);
#pragma unroll
    for (int k = 1; k < NC; ++k) r = add_rn(r, mul_rn(val(1 + j + 8 * k), xv[k]));
    r = add_rn(r, __shfl_xor_sync(kFull, r, 1));
    r = add_rn(r, __shfl_xor_sync(kFull, r, 2));
    r = add_rn(r, __shfl_xor_sync(kFull, r, 4));
    __syncwarp();
    if (j == 0) {
      const int64_t row = w0 + 4 * (int64_t)NW * i + grp;
      if (row < r_hi) {
        const double* t = tb + (grp << 3);
#pragma unroll
        for (int q = 0; q < TAIL; ++q) r = add_rn(r, t[q]);
        acc = add_rn(acc, epi(row, add_rn(t[7], r), xv[NC + 1], xv[NC + 2]));
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
    __syncwarp();  // stage i and the leftover buffer consumed
    issue(i + S, stg);
    stg = stg + 1 == S ? 0 : stg + 1;
  };
#pragma unroll 1
  for (int q = 0; q < S; ++q) issue(q, q);
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
  __syncwarp();
  return acc;
}

#ifdef IPI_K4_MAXNREG
#define IPI_K4_REGS(NW) __maxnreg__(IPI_K4_MAXNREG)
#else
#define IPI_K4_REGS(NW) __launch_bounds__(NW * 32, 1)
#endif
template <int K, int NW, int S>
__global__ void IPI_K4_REGS(NW) inner_ring_kernel(KArgs a) {
  using L = RingGeom<K, NW, S>;
  GridBarrier gb{a.bar, 0u, a.bar_mode};
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ KShared sh;
  const uint64_t pol = a.keep_frac > 0.f ? policy_evict_last() : policy_evict_first();
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nblk = gridDim.x;
  const int64_t n = a.n;
  // row-balanced contiguous slices, boundaries on multiples of 4 rows
  auto split = [&](int64_t c) -> int64_t {
    if (c >= nblk) return n;
    const int64_t r = (n * c / nblk) / 4 * 4;
    return r < n ? r : n;
  };
  const int64_t s_lo = split(blockIdx.x), s_hi = split(blockIdx.x + 1);
  const double gam = a.gamma;
  const double* b = a.b;
  double* x = a.x;
  double* r = a.r;
  const bool w_shared = (s_hi - s_lo) <= a.own_cap;
  double* wl = w_shared ? reinterpret_cast<double*>(smem_raw + L::kBytes) : (a.w + s_lo);
  const double* invd = a.invd;
  auto pcv = [&](int64_t s, double v) -> double { return invd ? mul_rn(v, invd[s]) : v; };
  int slot = 0;

  // ---- r = b - (x - gamma P x), ||b||, ||r|| --------------------------------
  double acc2[2] = {0.0, 0.0};
  for (int64_t i = s_lo + tid; i < s_hi; i += nthr) acc2[0] = add_rn(acc2[0], mul_rn(b[i], b[i]));
  auto residual_pass = [&](double& q) {
    q = add_rn(q, ring_rows<K, NW, S, true>(a.col, a.val, x, b, s_lo, s_hi, smem_raw, pol,
                                            [=](int64_t s, double px, double xs, double bs) {
      const double ri = sub_rn(bs, sub_rn(xs, mul_rn(gam, px)));
      r[s] = ri;
      return mul_rn(ri, ri);
    }));
  };
  k4_mark(a);
  residual_pass(acc2[1]);
  __syncthreads();
  k4_mark(a);
  grid_allreduce<2>(acc2, a, slot, gb, sh);
  k4_mark(a);
  const double bnorm = sqrt(acc2[0]);
  double rn = sqrt(acc2[1]);
  const double eff = fmax(a.target, 1e-14 * fmax(1.0, bnorm));
  int it = 0;

  if (a.kind == IPI_KSP_RICHARDSON) {
    while (true) {
      if (rn <= eff || it >= a.max_it || !isfinite(rn)) break;
      {
        double* __restrict__ xr = x;
        const double* __restrict__ rr = r;
#pragma unroll 4
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr) xr[i] = add_rn(xr[i], mul_rn(a.scale, pcv(i, rr[i])));
      }
      ++it;
      gb.sync();
      k4_mark(a);
      double q[1] = {0.0};
      residual_pass(q[0]);
      __syncthreads();
      if (a.trace) gb.sync();
      k4_mark(a);
      grid_allreduce<1>(q, a, slot, gb, sh);
      rn = sqrt(q[0]);
      k4_mark(a);
    }
  } else {  // GMRES(30): MGS (register slices) or CGS2
    double est_target = eff;
    const int64_t own = s_hi - s_lo;
    // host guarantees own <= kMgsE * nthr and two slices fit the ring area
    const bool mgs = a.ortho == IPI_ORTHO_MGS;
    constexpr int kMgsE = mgs_elems<NW>();
    double wv[kMgsE];
    while (rn > eff && it < a.max_it) {
      // z = pc(r); beta = ||z||
      double q0[1] = {0.0};
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
        const double z = pcv(i, r[i]);
        a.V[i] = z;
        q0[0] = add_rn(q0[0], mul_rn(z, z));
      }
      double beta = rn;
      if (invd) {
        grid_allreduce<1>(q0, a, slot, gb, sh);
        beta = sqrt(q0[0]);
      }
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
        k4_mark(a);
        ring_rows<K, NW, S, true>(a.col, a.val, Vj, nullptr, s_lo, s_hi, smem_raw, pol,
                                  [=](int64_t s, double px, double xs, double) {
          const double v = sub_rn(xs, mul_rn(gam, px));
          wl[s - s_lo] = invd ? mul_rn(v, invd[s]) : v;
          return 0.0;
        });
        ++it;
        __syncthreads();  // w rows written by group leaders, read per-thread below
        if (a.trace) gb.sync();  // diagnostics: mark when every CTA's SpMV is done
        k4_mark(a);
        double nw1;
        bool reorth = false;
        if (mgs) {
          // Modified Gram-Schmidt (inner.py:251-253).  w's slice stays in
          // registers; the basis slices are staged in the (now idle) ring
          // area with 8-byte cp.async, V_{l+1} issued before the all-reduce
          // that produces h_l, so a pass costs one all-reduce plus
          // shared-memory arithmetic.
          const uint32_t vb = (uint32_t)__cvta_generic_to_shared(smem_raw);
          const int64_t own_pad = (own + 1) & ~(int64_t)1;
          const double* sv = reinterpret_cast<const double*>(smem_raw);
          auto stage = [&](int l, int buf) {
            const double* src = a.V + (int64_t)l * n + s_lo;
            const uint32_t dst = vb + (uint32_t)(buf * own_pad * 8);
            for (int64_t e = tid; e < own; e += nthr) cp_async8(dst + (uint32_t)(8 * e), src + e);
            cp_async_commit();
          };
          stage(0, 0);
#pragma unroll
          for (int k = 0; k < kMgsE; ++k) {
            const int64_t e = tid + (int64_t)k * nthr;
            wv[k] = e < own ? wl[e] : 0.0;
          }
          cp_async_wait<0>();
          __syncthreads();
          double p[1] = {0.0};
#pragma unroll
          for (int k = 0; k < kMgsE; ++k) {
            const int64_t e = tid + (int64_t)k * nthr;
            if (e < own) p[0] = add_rn(p[0], mul_rn(sv[e], wv[k]));
          }
          for (int l = 0; l <= j; ++l) {
            __syncthreads();  // every thread is done with the buffer V_{l+1} goes to
            if (l < j) stage(l + 1, (l + 1) & 1);
            grid_allreduce<1>(p, a, slot, gb, sh);
            const double hlj = p[0];
            if (tid == 0) sh.H[l * R + j] = hlj;
            if (l < j) {
              cp_async_wait<0>();
              __syncthreads();
            }
            const double* vl = sv + (l & 1) * own_pad;
            const double* vn = sv + ((l + 1) & 1) * own_pad;
            double q = 0.0;
#pragma unroll
            for (int k = 0; k < kMgsE; ++k) {
              const int64_t e = tid + (int64_t)k * nthr;
              if (e < own) {
                wv[k] = sub_rn(wv[k], mul_rn(hlj, vl[e]));
                q = l < j ? add_rn(q, mul_rn(vn[e], wv[k])) : add_rn(q, mul_rn(wv[k], wv[k]));
              }
            }
            p[0] = q;
          }
          grid_allreduce<1>(p, a, slot, gb, sh);
          nw1 = p[0];
          k4_mark(a);
          k4_mark(a);
        } else {
          cgs_dots(a, j + 1, true, wl, s_lo, s_hi, pol_last, sh.cv, slot, gb, sh);
          k4_mark(a);
          const double nw = sh.cv[j + 1];
          double q1[1] = {cgs_update(a, j + 1, sh.cv, wl, s_lo, s_hi, pol_last)};
          grid_allreduce<1>(q1, a, slot, gb, sh);
          k4_mark(a);
          nw1 = q1[0];
          reorth = nw1 < 0.5 * nw;  // DGKS: ||w1|| < ||w|| / sqrt(2)
          if (reorth) {
            cgs_dots(a, j + 1, false, wl, s_lo, s_hi, pol_last, sh.dv, slot, gb, sh);
            double q2[1] = {cgs_update(a, j + 1, sh.dv, wl, s_lo, s_hi, pol_first)};
            grid_allreduce<1>(q2, a, slot, gb, sh);
            nw1 = q2[0];
          }
        }
        const double hnorm = sqrt(nw1);
        if (tid == 0) {
          double* H = sh.H;
          if (!mgs)
            for (int l = 0; l <= j; ++l) H[l * R + j] = reorth ? add_rn(sh.cv[l], sh.dv[l]) : sh.cv[l];
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
        if (mgs) {
#pragma unroll
          for (int k = 0; k < kMgsE; ++k) {  // next SpMV input: keep in L2
            const int64_t e = tid + (int64_t)k * nthr;
            if (e < own) st_hint(Vnew + s_lo + e, wv[k] / hnorm, pol_last);
          }
        } else {
          for (int64_t i = s_lo + tid; i < s_hi; i += nthr)
            st_hint(Vnew + i, wl[i - s_lo] / hnorm, pol_last);
        }
        gb.sync();
        k4_mark(a);
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
        for (int l = 0; l < j; ++l) t = add_rn(t, mul_rn(ld_hint(a.V + (int64_t)l * n + i, pol_first), sh.y[l]));
        x[i] = add_rn(x[i], t);
      }
      gb.sync();
      double q[1] = {0.0};
      residual_pass(q[0]);
      grid_allreduce<1>(q, a, slot, gb, sh);
      rn = sqrt(q[0]);
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
    a.rep->converged = rn <= eff ? 1 : 0;
    a.rep->breakdown = 0;
    a.rep->target_2norm = eff;
  }
}

// Diagnostics: ring_rows alone as a regular kernel (y = x - gamma P x), to
// compare the persistent kernel's SpMV with the standalone K3 launch.
template <int K, int NW, int S, bool STATIC>
__global__ void __launch_bounds__(NW * 32, 1) ring_apply_kernel(KArgs a, double* y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (STATIC) {  // the persistent kernel's static shared memory, to A/B its effect
    __shared__ KShared sh;
    if (threadIdx.x == 0 && a.n < 0) sh.red[0] = 1.0, y[0] = sh.red[1];
  }
  const int64_t n = a.n;
  const int nblk = gridDim.x;
  auto split = [&](int64_t c) -> int64_t {
    if (c >= nblk) return n;
    const int64_t r = (n * c / nblk) / 4 * 4;
    return r < n ? r : n;
  };
  const int64_t s_lo = split(blockIdx.x), s_hi = split(blockIdx.x + 1);
  const double gam = a.gamma;
  if (a.kind == 0) {
    ring_rows<K, NW, S, true>(a.col, a.val, a.x, nullptr, s_lo, s_hi, smem_raw, policy_evict_first(),
                              [=](int64_t s, double px, double xs, double) {
                                y[s] = sub_rn(xs, mul_rn(gam, px));
                                return 0.0;
                              });
  } else {  // the persistent kernel's residual pass: b.b first, then r = b - Ax and ||r||^2
    const double* b = a.b;
    double bb = 0.0;
    for (int64_t i = s_lo + threadIdx.x; i < s_hi; i += blockDim.x) bb = add_rn(bb, mul_rn(b[i], b[i]));
    double q = ring_rows<K, NW, S, true>(a.col, a.val, a.x, b, s_lo, s_hi, smem_raw, policy_evict_first(),
                                         [=](int64_t s, double px, double xs, double bs) {
                                           const double ri = sub_rn(bs, sub_rn(xs, mul_rn(gam, px)));
                                           y[s] = ri;
                                           return mul_rn(ri, ri);
                                         });
    if (q + bb == -1.0) y[0] = 0.0;  // keep the sums live
  }
}

int ring_apply_test(const int32_t* col, const double* val, int64_t n, double gamma, const double* x,
                    double* y, int reps, float* ms, cudaStream_t st) {
  KArgs a{};
  a.col = col;
  a.val = val;
  a.n = n;
  a.gamma = gamma;
  a.x = const_cast<double*>(x);
  a.b = x;
  a.kind = getenv("IPI_K4_TEST_RESID") ? 1 : 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = ring_inner_smem(64, 12, 3);
  auto fn = getenv("IPI_K4_TEST_STATIC") ? ring_apply_kernel<64, 12, 3, true> : ring_apply_kernel<64, 12, 3, false>;
  IPI_CUDA_TRY(raise_smem_limit(fn, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const bool coop = getenv("IPI_K4_TEST_COOP") != nullptr;
  void* args[] = {(void*)&a, (void*)&y};
  auto go = [&] {
    if (coop) cudaLaunchCooperativeKernel((const void*)fn, dim3(sms), dim3(384), args, (size_t)smem, st);
    else fn<<<sms, 384, smem, st>>>(a, y);
  };
  go();
  cudaEventRecord(e0, st);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

// (K, warps, stages) instances
#define IPI_K4R_SHAPES(M) M(64, 12, 3) M(64, 16, 3) M(64, 12, 4) M(64, 8, 4) M(64, 10, 4)

int ring_inner_smem(int K, int NW, int S) {
  return NW * (S * 4 * K * 12 + 256);
}

bool ring_inner_has(int K, int NW, int S) {
#define IPI_K4R_HAS(KK, WW, SS) if (K == KK && NW == WW && S == SS) return true;
  IPI_K4R_SHAPES(IPI_K4R_HAS)
#undef IPI_K4R_HAS
  return false;
}

template <int K, int NW, int S>
static int launch_ring_t(KArgs& a, int smem, int blocks, cudaStream_t st) {
  auto fn = inner_ring_kernel<K, NW, S>;
  cudaError_t e = raise_smem_limit(fn, smem);
  if (getenv("IPI_K4_CARVEOUT"))
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(getenv("IPI_K4_CARVEOUT")));
  if (getenv("IPI_K4_ATTR")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, fn);
    fprintf(stderr, "ring inner: regs %d static smem %zu local %zu maxdyn %d carveout %d\n", fa.numRegs,
            fa.sharedSizeBytes, fa.localSizeBytes, fa.maxDynamicSharedSizeBytes, fa.preferredShmemCarveout);
  }
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("ring inner smem attr: ") + cudaGetErrorString(e));
  int per_sm = 0;
  IPI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NW * 32, smem));
  if (per_sm < 1) return fail(IPI_ECUDA, "ring inner kernel cannot be resident (smem/regs)");
  void* args[] = {(void*)&a};
  IPI_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(blocks), dim3(NW * 32), args,
                                           (size_t)smem, st));
  return IPI_OK;
}

int dispatch_inner_ring(KArgs& a, int K, int NW, int S, int smem, int blocks, cudaStream_t st) {
#define IPI_K4R_GO(KK, WW, SS) \
  if (K == KK && NW == WW && S == SS) return launch_ring_t<KK, WW, SS>(a, smem, blocks, st);
  IPI_K4R_SHAPES(IPI_K4R_GO)
#undef IPI_K4R_GO
  return fail(IPI_ECUDA, "ring inner kernel: no instance for (K, warps, stages)");
}

}  // namespace ipi
