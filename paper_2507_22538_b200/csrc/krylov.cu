// krylov.cu — K4 host side: workspace, planning of the persistent inner kernel, launch.
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
// without any broadcast.  Grid barriers: a release counter + acquire spin
// (GridBarrier, krylov.cuh) over cooperatively launched (co-resident) CTAs.
//
// Semantics mirrored exactly (inner.py line refs):
//   eff = max(target, 1e-14*max(1,||b||))           :189
//   Richardson: r=b-A th; stop if rn<=eff|it>=cap|!finite; th += scale*r   :216-226
//   GMRES: restart 30, MGS, Givens, break on |g_j|<=est or hnorm==0,
//          true residual per cycle, est_target = |g_j|*(eff/rn)*0.5       :229-283
//   back substitution with zero-pivot -> 0                                 :286-292
// Every vector op uses separate mul/add roundings like numpy (no FMA).
#include <cstdlib>
#include <mutex>

#include "krylov.cuh"

namespace ipi {

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// one arena per device (the standalone ipi_inner_solve; handles own theirs)
static std::mutex g_ws_mu;
static double* g_ws[64] = {};
static int64_t g_ws_len[64] = {};

double* krylov_workspace(int64_t /*n*/, int64_t doubles_needed) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (g_ws[dev] && g_ws_len[dev] >= doubles_needed) return g_ws[dev];
  if (g_ws[dev]) {
    cudaDeviceSynchronize();  // the arena may still be in use by queued solves
    cudaFree(g_ws[dev]);
    g_ws[dev] = nullptr;
    g_ws_len[dev] = 0;
  }
  if (cudaMalloc(&g_ws[dev], sizeof(double) * doubles_needed) != cudaSuccess) {
    g_ws[dev] = nullptr;
    cudaGetLastError();
    return nullptr;
  }
  g_ws_len[dev] = doubles_needed;
  return g_ws[dev];
}

int inner_solve(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                double gamma, const double* b, double* x, double target, int32_t max_it,
                int32_t kind, double scale, int lanes, int halo, int uniform_K,
                ipi_inner_report* d_report, cudaStream_t st, double* workspace,
                int64_t workspace_doubles, const double* inv_diag, double pi_bytes) {
  if (kind < IPI_KSP_RICHARDSON || kind > IPI_KSP_TFQMR)
    return fail(IPI_EVALIDATION, "unknown inner solver kind " + std::to_string(kind));
  if (max_it < 1) return fail(IPI_EVALIDATION, "iteration cap must be >= 1, got " + std::to_string(max_it));
  if (target < 0.0) return fail(IPI_EVALIDATION, "residual target must be >= 0");
  if (n == 0) return fail(IPI_EDIMENSION, "empty system");
  int dev = 0, sms = 148;
  IPI_CUDA_TRY(cudaGetDevice(&dev));
  IPI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // one 1024-thread CTA per SM (fewer for tiny systems: >= 32 rows per CTA)
  int blocks = sms;
  if ((int64_t)blocks * 32 > n) blocks = (int)std::max<int64_t>(1, n / 32);
  const int64_t need = (int64_t)(R + 1) * n + 2 * n + 4 * (int64_t)blocks + 8;
  // caller-owned workspace (per handle, so concurrent handles never share it)
  // or the per-device arena used by the standalone API
  double* ws = (workspace && workspace_doubles >= need) ? workspace : krylov_workspace(n, need);
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
  a.bar = reinterpret_cast<unsigned*>(a.partials + 4 * (int64_t)blocks);
  IPI_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 64, st));
  a.bar_mode = getenv("IPI_K4_BARRIER") ? atoi(getenv("IPI_K4_BARRIER")) : 0;
  a.xwin = getenv("IPI_K4_XWIN") ? atoi(getenv("IPI_K4_XWIN")) != 0 : 1;
  {  // L2 residency of P_pi across the solve's SpMVs (IPI_K4_KEEP overrides the fraction)
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    double bytes = pi_bytes;
    if (bytes <= 0.0) {  // unknown: read nnz (one sync)
      int64_t nnz_h = 0;
      cudaMemcpyAsync(&nnz_h, rp_pi + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      bytes = 12.0 * (double)nnz_h + 8.0 * (double)(n + 1);
    }
    const double budget = 0.6 * (double)l2;
    // whole P_pi when it fits; a fractional hint helped C4's SpMV (-9%) but not its
    // MGS-bound GMRES step and slowed C3's (IPI_K4_KEEP=<fraction> to experiment)
    double f = bytes <= budget ? 1.0 : 0.0;
    if (getenv("IPI_K4_KEEP")) f = atof(getenv("IPI_K4_KEEP"));
    a.keep_frac = (float)std::min(1.0, std::max(0.0, f));
  }
  a.target = target;
  a.max_it = max_it;
  a.kind = kind;
  a.scale = scale;
  a.rep = d_report;
  a.invd = inv_diag;
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
  switch (kind) {
    case IPI_KSP_TFQMR: return dispatch_inner_tfqmr(a, G, P, lanes, win, smem, blocks, st);
    case IPI_KSP_BICGSTAB: return dispatch_inner_bicgstab(a, G, P, lanes, win, smem, blocks, st);
    default: return dispatch_inner_gmres(a, G, P, lanes, win, smem, blocks, st);
  }
}

int dispatch_inner_gmres(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                         cudaStream_t st) {
  return dispatch_inner<0>(a, G, P, lanes, win, smem, blocks, st);
}

}  // namespace ipi
