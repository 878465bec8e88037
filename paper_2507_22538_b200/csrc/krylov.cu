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
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "krylov.cuh"

namespace ipi {

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// One arena per (device, stream) for the standalone ipi_inner_solve (handles
// own theirs).  Growth frees and allocates stream-ordered, so work already
// queued on the stream keeps its arena and nothing else is synchronised;
// solves on different streams never share a basis, partials or barrier.
static std::mutex g_ws_mu;
static std::map<std::pair<int, cudaStream_t>, std::pair<double*, int64_t>> g_ws;

double* krylov_workspace(int64_t doubles_needed, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto& slot = g_ws[{dev, st}];
  if (slot.first && slot.second >= doubles_needed) return slot.first;
  if (slot.first) {
    cudaFreeAsync(slot.first, st);
    slot = {nullptr, 0};
  }
  double* p = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(double) * doubles_needed, st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  slot = {p, doubles_needed};
  return p;
}

// diagnostics: phase timestamps of the next persistent launches (ipi_k4_trace)
static unsigned long long* g_k4_trace = nullptr;
static int g_k4_trace_cap = 0;

unsigned long long* k4_trace_buffer(int* cap) {
  *cap = g_k4_trace_cap;
  return g_k4_trace;
}

int k4_trace(int enable, unsigned long long* out, int cap) {
  if (enable) {
    if (!g_k4_trace) {
      IPI_CUDA_TRY(cudaMalloc(&g_k4_trace, sizeof(unsigned long long) * 8192));
      IPI_CUDA_TRY(cudaMemset(g_k4_trace, 0, sizeof(unsigned long long)));
      g_k4_trace_cap = 8192;
    }
    return IPI_OK;
  }
  if (g_k4_trace && out && cap > 0) {
    IPI_CUDA_TRY(cudaDeviceSynchronize());
    IPI_CUDA_TRY(cudaMemcpy(out, g_k4_trace, sizeof(unsigned long long) * std::min(cap, g_k4_trace_cap),
                            cudaMemcpyDeviceToHost));
  }
  cudaFree(g_k4_trace);
  g_k4_trace = nullptr;
  g_k4_trace_cap = 0;
  return IPI_OK;
}

// environment switches (A/B experiments), read once per process
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

int inner_solve(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                double gamma, const double* b, double* x, double target, int32_t max_it,
                int32_t kind, double scale, int lanes, int halo, int uniform_K,
                ipi_inner_report* d_report, cudaStream_t st, double* workspace,
                int64_t workspace_doubles, const double* inv_diag, double pi_bytes, int ortho,
                const ipi_op* op, int contig, const double* tv) {
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
  if (ortho != IPI_ORTHO_AUTO && ortho != IPI_ORTHO_CGS2 && ortho != IPI_ORTHO_MGS)
    return fail(IPI_EVALIDATION, "unknown GMRES orthogonalisation " + std::to_string(ortho));
  // AUTO: a grid all-reduce costs ~2-3 us; an MGS pass over a CTA's slice of
  // one basis vector costs about the same once the slice exceeds a few
  // thousand rows, below which CGS2's 2 reductions per step beat MGS's j+2
  // (C4: 0.062 vs 0.089 ms per step; C2: MGS).
  if (ortho == IPI_ORTHO_AUTO) ortho = n / blocks >= 1024 ? IPI_ORTHO_MGS : IPI_ORTHO_CGS2;
  const int64_t need = (int64_t)(R + 1) * n + 2 * n + 2 * kPartStride * (int64_t)blocks + 64;
  // caller-owned workspace (per handle, so concurrent handles never share it)
  // or the per-device arena used by the standalone API
  double* ws = (workspace && workspace_doubles >= need) ? workspace : krylov_workspace(need, st);
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
  a.bar = reinterpret_cast<unsigned*>(a.partials + 2 * kPartStride * (int64_t)blocks);
  a.ortho = ortho;
  a.contig = contig;
  a.trace = g_k4_trace;
  a.trace_cap = g_k4_trace_cap;
  if (a.trace) IPI_CUDA_TRY(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long), st));
  IPI_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 64, st));
  static const int bar_mode = env_int("IPI_K4_BARRIER", 0);
  static const int xwin = env_int("IPI_K4_XWIN", 1);
  static const double keep_env = getenv("IPI_K4_KEEP") ? atof(getenv("IPI_K4_KEEP")) : -1.0;
  a.bar_mode = bar_mode;
  a.xwin = xwin != 0;
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
    // contiguous rows stream 8 B per entry (values) instead of 12: C4's 137 MB
    // P_pi becomes ~92 MB, of which half marked evict-last measured best
    // (C4 iPI 53.0 ms at 0.5 vs 57.0 at 0 and 58.0 at 1: all of it evicts the
    // basis and K1's working set); a larger P_pi streams evict-first
    if (contig) bytes *= 8.0 / 12.0;
    const double budget = 0.6 * (double)l2;
    double f = bytes <= budget ? 1.0 : (contig && bytes <= (double)l2 ? 0.5 : 0.0);
    if (keep_env >= 0.0) f = keep_env;
    a.keep_frac = (float)std::min(1.0, std::max(0.0, f));
  }
  a.target = target;
  a.max_it = max_it;
  a.kind = kind;
  a.scale = scale;
  a.rep = d_report;
  a.invd = inv_diag;
  // Large uniform K = 64-class rows with GMRES/MGS: stepped launches (K3 ring
  // operator + one cooperative MGS/Givens kernel per Arnoldi step,
  // krylov_step.cu).  IPI_K4_STEPPED=0 keeps the persistent kernels.
  static const int stepped_env = env_int("IPI_K4_STEPPED", 1);
  if (stepped_env && op && op->variant == IPI_K3_URING && op->n_local == n && op->state0 == 0 &&
      kind == IPI_KSP_GMRES && ortho == IPI_ORTHO_MGS && stepped_gmres_fits(n, sms)) {
    const int64_t sneed = stepped_gmres_workspace(n, sms);
    double* sws = (workspace && workspace_doubles >= sneed) ? workspace : krylov_workspace(sneed, st);
    if (!sws) return fail(IPI_ERESOURCE, "cannot allocate the stepped GMRES workspace");
    return stepped_gmres(op, n, b, x, target, max_it, inv_diag, d_report, sws,
                         sws == workspace ? workspace_doubles : sneed, st, tv);
  }
  // Uniform K = 64-class rows with GMRES/CGS2 or Richardson: the ring kernel
  // (krylov_ring.cu).  IPI_K4_RING=0 keeps the 1024-thread kernel;
  // IPI_K4_RING_SHAPE=<warps>x<stages> forces a ring shape.
  static const int ring_env = env_int("IPI_K4_RING", 1);
  static const char* shape_env = getenv("IPI_K4_RING_SHAPE");
  if (ring_env && uniform_K > 0 && (kind == IPI_KSP_RICHARDSON || kind == IPI_KSP_GMRES)) {
    int NW = 12, S = 3;
    if (shape_env) sscanf(shape_env, "%dx%d", &NW, &S);
    if (ring_inner_has(uniform_K, NW, S) && n >= 64 * (int64_t)blocks) {
      a.K = uniform_K;
      a.halo = -1;
      a.win_cap = 0;
      const int ring = ring_inner_smem(uniform_K, NW, S);
      const int budget_b = 227 * 1024 - (int)sizeof(KShared) - 1024;
      const int64_t own_max = (n + blocks - 1) / blocks + 8;
      // w slice in shared memory only on request: the ring plus a 57 KB slice
      // leave L1 too small for the gathered x's neighbourhood (IPI_K4_RING_WSMEM=1)
      static const int wsmem = env_int("IPI_K4_RING_WSMEM", 0);
      a.own_cap = wsmem && ring + own_max * 8 <= budget_b ? (int)own_max : 0;
      const int smem = ring + a.own_cap * 8;
      if (a.ortho == IPI_ORTHO_MGS && (own_max > (int64_t)ring_mgs_elems(NW) * NW * 32 ||
                                       2 * (own_max + 1) * 8 > ring))
        a.ortho = IPI_ORTHO_CGS2;  // slices too long for the staged MGS
      return dispatch_inner_ring(a, uniform_K, NW, S, smem, blocks, st);
    }
  }
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
    default:
      if (kind == IPI_KSP_GMRES && ortho == IPI_ORTHO_CGS2)
        return dispatch_inner_gmres_cgs(a, G, P, lanes, win, smem, blocks, st);
      return dispatch_inner_gmres(a, G, P, lanes, win, smem, blocks, st);
  }
}

int dispatch_inner_gmres(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                         cudaStream_t st) {
  return dispatch_inner<0>(a, G, P, lanes, win, smem, blocks, st);
}

}  // namespace ipi
