// krylov.cu — K4: policy evaluation (I - gamma P_pi) x = b as ONE persistent
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
#include <mutex>

#include "handle.cuh"

namespace cg = cooperative_groups;

namespace ipi {

constexpr int R = kGmresRestart;

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
  double* partials;  // [2 slots][grid][2]
  double target;
  int max_it;
  int kind;
  double scale;
  int halo;
  int win_cap;   // doubles of the shared-memory window (0 = none)
  int own_cap;   // doubles of the shared-memory w slice (0 = w in global)
  int K;         // uniform row length of P_pi (0 = variable)
  ipi_inner_report* rep;
};

struct KShared {
  double red[32];
  double bc[4];
  double H[(R + 1) * R];
  double cs[R], sn[R], g[R + 1], y[R];
  int iflag[4];
};

// Two-level deterministic all-reduce of NV doubles; result in every thread.
template <int NV>
__device__ __forceinline__ void grid_allreduce(double (&v)[NV], const KArgs& a, int& slot,
                                               cg::grid_group& grid, KShared& sh) {
  double t[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) t[k] = block_sum(v[k], sh.red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) a.partials[((int64_t)slot * nblk + blockIdx.x) * 2 + k] = t[k];
  }
  grid.sync();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int i = lane; i < nblk; i += 32) s = add_rn(s, a.partials[((int64_t)slot * nblk + i) * 2 + k]);
      s = warp_sum(s);
      if (lane == 0) sh.bc[k] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sh.bc[k];
  slot ^= 1;
  __syncthreads();
}

// Row sums of P_pi over this CTA's rows with an optional shared-memory window
// of the input vector; epi(s, Px_s) is called by one lane per row.  P == 0:
// generic rows (G lanes strided over the row, 4 loads in flight); P > 0:
// uniform even-length rows, P 16-byte value pairs per lane, batches
// software-pipelined across row groups (same scheme as K1's fast path).
template <int G, int P, bool WIN, class Epi>
__device__ __forceinline__ void spmv_rows(const KArgs& a, const double* xin, int64_t s_lo,
                                          int64_t s_hi, double* win, uint64_t pol, Epi&& epi) {
  int64_t w_lo = 0, w_len = 0;
  if (WIN) {
    int64_t lo = s_lo - a.halo, hi = s_hi + a.halo;
    lo = lo < 0 ? 0 : lo;
    hi = hi > a.n ? a.n : hi;
    __syncthreads();
    if (hi - lo <= a.win_cap) {
      w_lo = lo;
      w_len = hi - lo;
      for (int64_t i = threadIdx.x; i < w_len; i += blockDim.x) win[i] = xin[lo + i];
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
      if (s < s_hi && gl == 0) epi(s, acc);
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
        if (s < s_hi && gl == 0) epi(s, acc);
        if (!has_next) break;
        cur = nxt;
        base = nb;
      }
    }
  }
}

template <int G, int P, bool WIN>
__global__ void __launch_bounds__(kInnerThreads, 1) inner_kernel(KArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double win[];
  __shared__ KShared sh;
  const uint64_t pol = policy_evict_first();
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
  int slot = 0;

  // ---- r = b - (x - gamma P x), ||b||, ||r|| --------------------------------
  double acc2[2] = {0.0, 0.0};
  for (int64_t i = s_lo + tid; i < s_hi; i += nthr) acc2[0] = add_rn(acc2[0], mul_rn(b[i], b[i]));
  spmv_rows<G, P, WIN>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px) {
    const double ri = sub_rn(b[s], sub_rn(x[s], mul_rn(gam, px)));
    r[s] = ri;
    acc2[1] = add_rn(acc2[1], mul_rn(ri, ri));
  });
  grid_allreduce<2>(acc2, a, slot, grid, sh);
  const double bnorm = sqrt(acc2[0]);
  double rn = sqrt(acc2[1]);
  const double eff = fmax(a.target, 1e-14 * fmax(1.0, bnorm));
  int it = 0;

  if (a.kind == IPI_KSP_RICHARDSON) {
    while (true) {
      if (rn <= eff || it >= a.max_it || !isfinite(rn)) break;
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) x[i] = add_rn(x[i], mul_rn(a.scale, r[i]));
      ++it;
      grid.sync();
      double acc1[1] = {0.0};
      spmv_rows<G, P, WIN>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px) {
        const double ri = sub_rn(b[s], sub_rn(x[s], mul_rn(gam, px)));
        r[s] = ri;
        acc1[0] = add_rn(acc1[0], mul_rn(ri, ri));
      });
      grid_allreduce<1>(acc1, a, slot, grid, sh);
      rn = sqrt(acc1[0]);
    }
  } else {  // GMRES(30)
    double est_target = eff;
    while (rn > eff && it < a.max_it) {
      const double beta = rn;  // ||pc(r)|| with pc = identity: same vector, same reduction
      if (beta == 0.0 || !isfinite(beta)) break;
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) a.V[i] = r[i] / beta;
      if (tid == 0) {
        for (int k = 0; k < (R + 1) * R; ++k) sh.H[k] = 0.0;
        for (int k = 0; k < R; ++k) sh.cs[k] = sh.sn[k] = 0.0;
        for (int k = 0; k <= R; ++k) sh.g[k] = 0.0;
        sh.g[0] = beta;
      }
      int j = 0;
      grid.sync();
      while (j < R && it < a.max_it) {
        const double* Vj = a.V + (int64_t)j * n;
        const double* V0 = a.V;
        double p[1] = {0.0};
        spmv_rows<G, P, WIN>(a, Vj, s_lo, s_hi, win, pol, [&](int64_t s, double px) {
          const double wi = sub_rn(Vj[s], mul_rn(gam, px));
          wl[s - s_lo] = wi;
          p[0] = add_rn(p[0], mul_rn(V0[s], wi));
        });
        ++it;
        __syncthreads();  // w rows written by group leaders, read per-thread below
        for (int l = 0; l <= j; ++l) {
          grid_allreduce<1>(p, a, slot, grid, sh);
          const double hlj = p[0];
          if (tid == 0) sh.H[l * R + j] = hlj;
          const double* Vl = a.V + (int64_t)l * n;
          const double* Vn = a.V + (int64_t)(l + 1) * n;
          double q = 0.0;
          if (l < j) {
            for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
              const double wi = sub_rn(wl[i - s_lo], mul_rn(hlj, Vl[i]));
              wl[i - s_lo] = wi;
              q = add_rn(q, mul_rn(Vn[i], wi));
            }
          } else {
            for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
              const double wi = sub_rn(wl[i - s_lo], mul_rn(hlj, Vl[i]));
              wl[i - s_lo] = wi;
              q = add_rn(q, mul_rn(wi, wi));
            }
          }
          p[0] = q;
        }
        grid_allreduce<1>(p, a, slot, grid, sh);
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
        for (int64_t i = s_lo + tid; i < s_hi; i += nthr) Vnew[i] = wl[i - s_lo] / hnorm;
        grid.sync();
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
      grid.sync();
      double acc1[1] = {0.0};
      spmv_rows<G, P, WIN>(a, x, s_lo, s_hi, win, pol, [&](int64_t s, double px) {
        const double ri = sub_rn(b[s], sub_rn(x[s], mul_rn(gam, px)));
        r[s] = ri;
        acc1[0] = add_rn(acc1[0], mul_rn(ri, ri));
      });
      grid_allreduce<1>(acc1, a, slot, grid, sh);
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
    a.rep->final_linear_residual_2norm = rn;
    a.rep->converged = rn <= eff ? 1 : 0;
    a.rep->breakdown = 0;
    a.rep->target_2norm = eff;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static std::mutex g_ws_mu;
static double* g_ws = nullptr;
static int64_t g_ws_len = 0;
static int g_ws_dev = -1;

double* krylov_workspace(int64_t /*n*/, int64_t doubles_needed) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_ws && g_ws_dev == dev && g_ws_len >= doubles_needed) return g_ws;
  if (g_ws) {
    cudaDeviceSynchronize();
    cudaFree(g_ws);
    g_ws = nullptr;
  }
  if (cudaMalloc(&g_ws, sizeof(double) * doubles_needed) != cudaSuccess) {
    g_ws = nullptr;
    g_ws_len = 0;
    return nullptr;
  }
  g_ws_len = doubles_needed;
  g_ws_dev = dev;
  return g_ws;
}

template <int G, int P, bool WIN>
static int launch_inner_t(KArgs& a, int smem, int blocks, cudaStream_t st) {
  auto fn = inner_kernel<G, P, WIN>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return fail(IPI_ECUDA, std::string("inner smem attr: ") + cudaGetErrorString(e));
  int per_sm = 0;
  IPI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kInnerThreads, smem));
  if (per_sm < 1) return fail(IPI_ECUDA, "inner kernel cannot be resident (smem/regs)");
  void* args[] = {(void*)&a};
  IPI_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(blocks), dim3(kInnerThreads), args,
                                           (size_t)smem, st));
  return IPI_OK;
}

template <int G, int P>
static int launch_inner_gp(KArgs& a, bool win, int smem, int blocks, cudaStream_t st) {
  return win ? launch_inner_t<G, P, true>(a, smem, blocks, st)
             : launch_inner_t<G, P, false>(a, smem, blocks, st);
}

int inner_solve(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                double gamma, const double* b, double* x, double target, int32_t max_it,
                int32_t kind, double scale, int lanes, int halo, int uniform_K,
                ipi_inner_report* d_report, cudaStream_t st) {
  if (kind != IPI_KSP_GMRES && kind != IPI_KSP_RICHARDSON)
    return fail(IPI_EVALIDATION, "inner solver kind not built on the device path yet");
  if (max_it < 1) return fail(IPI_EVALIDATION, "iteration cap must be >= 1, got " + std::to_string(max_it));
  if (target < 0.0) return fail(IPI_EVALIDATION, "residual target must be >= 0");
  if (n == 0) return fail(IPI_EDIMENSION, "empty system");
  int dev = 0, sms = 148;
  IPI_CUDA_TRY(cudaGetDevice(&dev));
  IPI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // one 1024-thread CTA per SM (fewer for tiny systems: >= 32 rows per CTA)
  int blocks = sms;
  if ((int64_t)blocks * 32 > n) blocks = (int)std::max<int64_t>(1, n / 32);
  const int64_t need = (int64_t)(R + 1) * n + 2 * n + 4 * (int64_t)blocks;
  double* ws = krylov_workspace(n, need);
  if (!ws) return fail(IPI_ERESOURCE, "cannot allocate Krylov workspace of " + std::to_string(need * 8) + " bytes");
  KArgs a;
  a.rp = rp_pi;
  a.col = col_pi;
  a.val = val_pi;
  a.n = n;
  a.gamma = gamma;
  a.b = b;
  a.x = x;
  a.V = ws;
  a.w = ws + (int64_t)(R + 1) * n;
  a.r = a.w + n;
  a.partials = a.r + n;
  a.target = target;
  a.max_it = max_it;
  a.kind = kind;
  a.scale = scale;
  a.rep = d_report;
  int G = lanes, P = 0;
  a.K = 0;
  if (uniform_K > 0 && uniform_shape(uniform_K, &G, &P)) a.K = uniform_K;
  else P = 0;
  // shared memory: [window: own + 2*halo][w slice: own]; budget ~200 KB
  const int64_t budget = 200 * 1024 / 8;
  const int64_t own_est = (n + blocks - 1) / blocks;
  int64_t own_cap = a.K ? own_est + 1 : std::min<int64_t>(n, 2 * own_est + 32);
  int64_t win_cap = 0;
  if (halo >= 0) win_cap = std::min<int64_t>(n, own_cap + 2 * (int64_t)halo);
  if (win_cap + own_cap > budget) own_cap = 0;      // keep the window, w in global
  if (win_cap > budget) win_cap = 0;                // window does not fit either
  if (win_cap + own_cap > budget) own_cap = 0;
  a.halo = win_cap > 0 ? halo : -1;
  a.win_cap = (int)win_cap;
  a.own_cap = (int)own_cap;
  const bool win = win_cap > 0;
  const int smem = (int)((win_cap + own_cap) * 8);
  if (P > 0) {
    int rc = IPI_OK;
#define IPI_INNER_LAUNCH(GG, PP) rc = launch_inner_gp<GG, PP>(a, win, smem, blocks, st)
    IPI_DISPATCH_UNIFORM(G, P, IPI_INNER_LAUNCH);
#undef IPI_INNER_LAUNCH
    return rc;
  }
  switch (lanes) {
    case 1: return launch_inner_gp<1, 0>(a, win, smem, blocks, st);
    case 2: return launch_inner_gp<2, 0>(a, win, smem, blocks, st);
    case 4: return launch_inner_gp<4, 0>(a, win, smem, blocks, st);
    case 8: return launch_inner_gp<8, 0>(a, win, smem, blocks, st);
    case 16: return launch_inner_gp<16, 0>(a, win, smem, blocks, st);
    default: return launch_inner_gp<32, 0>(a, win, smem, blocks, st);
  }
}

}  // namespace ipi
