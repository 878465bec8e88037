// krylov_step.cu — stepped GMRES(30) for large uniform-row P_pi (C2: n = 2^20,
// K = 64): every Arnoldi step is two launches on the caller's stream,
//
//   1. the planned K3 operator (spmv_ring.cu, ring kernel): w = V_j - gamma P V_j;
//   2. step_ortho: one cooperative kernel that applies the preconditioner,
//      runs modified Gram-Schmidt (inner.py:251-253, j+2 grid all-reduces,
//      each CTA's slices of w, V_l and the prefetched V_{l+1} in registers),
//      the Givens update and break test (:256-270) and writes V_{j+1},
//
// instead of the single persistent kernel of krylov.cuh / krylov_ring.cu.
// Why: inlined into a persistent kernel the same ring SpMV runs 15-25%
// slower than as its own launch (C2: 0.165-0.185 vs 0.145 ms; DESIGN.md
// §4.4), and the SpMV is three quarters of a step.  The price is two launch
// gaps per step (~2-3 us) against ~0.2 ms of work.
//
// Control stays on the device: the Hessenberg column, Givens rotations,
// est_target and the cycle flags live in a StepState in HBM; every kernel
// of a step that the previous step ended skips itself (K3 reads
// state.active).  The host stays one step ahead: it enqueues step k+1, then
// waits for step k's event and reads the flags CTA 0 mirrors into mapped
// host memory, so the GPU never waits on the host and at most one launched
// step per cycle is a no-op.  Cycle ends (back substitution :286-292, x
// update, true residual, est_target tightening :274-282, restart) are three
// more launches and one host synchronisation per cycle.
//
// Numerics are the reference's MGS with separate mul/add roundings; sums
// are two-level deterministic (fixed intra-CTA trees, CTA partials added in
// CTA order), so reruns are bit-identical.
#include <algorithm>
#include <string>

#include "krylov.cuh"

namespace ipi {

struct StepState {
  double H[(R + 1) * R];
  double cs[R], sn[R], g[R + 1];
  double eff, est_target, rn, target;
  int j, it, active, done, basis_reads;
};

// Host-mapped mirror of the flags the host loop reads (written by CTA 0).
struct StepFlags {
  int active, j, it, done;
  double rn;
};

struct StepArgs {
  int64_t n;
  const double* b;
  double* x;
  double* V;  // (R+1) x ldv basis (ldv even: every slice start 16-byte aligned)
  int64_t ldv;
  double* w;
  double* r;
  double* partials;
  unsigned* bar;  // two grid-barrier counters, used alternately by successive launches
  int parity;
  const double* invd;  // Jacobi inverse diagonal or nullptr
  StepState* s;
  StepFlags* hf;  // host-mapped (device pointer)
  int max_it;
  int first;  // step_cycle_start: first call of the solve
  unsigned long long* trace;  // diagnostics (ipi_k4_trace): step_ortho start / MGS done / end
  int trace_cap;
};

constexpr int kStepThreads = 512;
constexpr int kStepE = 16;  // slice elements per worker thread: n <= 148 * 480 * 16 = 1.14M
// Warp 0 owns no slice elements: thread 0 leads the grid barriers, and a
// release (red.release.gpu) waits for the leader's own outstanding loads, so
// a leader holding V_{l+1} prefetches would serialise them into every
// all-reduce (3.9 vs ~2.5 us per MGS pass on C2).
constexpr int kStepWorkers = kStepThreads - 32;

// CTA c's slice of the vectors, boundaries even (16-byte aligned bulk copies)
__device__ __forceinline__ void step_slice(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t c = blockIdx.x, nb = gridDim.x;
  lo = c == 0 ? 0 : ((n * c / nb) & ~(int64_t)1);
  hi = c + 1 == nb ? n : ((n * (c + 1) / nb) & ~(int64_t)1);
}

// grid_allreduce (krylov.cuh) reads only KArgs::partials; wrap ours.
__device__ __forceinline__ KArgs step_kargs(const StepArgs& a) {
  KArgs k{};
  k.partials = a.partials;
  return k;
}

__device__ __forceinline__ void publish_flags(const StepArgs& a, const StepState& s) {
  volatile StepFlags* f = a.hf;
  f->active = s.active;
  f->j = s.j;
  f->it = s.it;
  f->done = s.done;
  f->rn = s.rn;
  __threadfence_system();
}

// One Arnoldi step after the K3 launch wrote w = V_j - gamma P V_j: MGS with
// this CTA's slice of w in registers and V_{l+1}'s slice loaded into
// registers while the all-reduce producing h_l is in flight, so a pass costs
// one grid all-reduce plus register arithmetic (C2: ~3.5 us per pass).
// (Streaming the slices through shared memory with 1-D bulk copies two
// passes ahead measured slower: 4.5 us per pass.)
__global__ void __launch_bounds__(kStepThreads, 1) step_ortho(StepArgs a) {
  __shared__ KShared sh;
  __shared__ double hcol[R + 1], cs_s[R], sn_s[R], gj_s, est_s;
  __shared__ int brk_s;
  StepState* st = a.s;
  const int tid = threadIdx.x;
  // the next cooperative launch's barrier counter (its previous user, two
  // launches back, has retired); reset even when this launch is a no-op
  if (blockIdx.x == 0 && tid == 0) a.bar[a.parity ^ 1] = 0u;
  if (!st->active) return;  // uniform: the previous launch ended the cycle
  k4_mark_raw(a.trace, a.trace_cap);
  GridBarrier gb{a.bar + a.parity, 0u, 0};
  const KArgs ka = step_kargs(a);
  int slot = 0;
  const int j = st->j;
  const int64_t n = a.n, ldv = a.ldv;
  int64_t s_lo, s_hi;
  step_slice(n, s_lo, s_hi);
  const int64_t own = s_hi - s_lo;
  const uint64_t pol_keep = policy_evict_last(), pol_first = policy_evict_first();
  if (tid == 0) {  // snapshot the rotation state before the first grid barrier:
    for (int l = 0; l < j; ++l) {  // CTA 0 updates g[j] after the last one
      cs_s[l] = st->cs[l];
      sn_s[l] = st->sn[l];
    }
    gj_s = st->g[j];
    est_s = st->est_target;
  }
  double wv[kStepE], vc[kStepE];
  const int64_t wt = tid - 32;  // worker index (< 0: the control warp)
  auto elem = [&](int k) -> int64_t { return wt < 0 ? own : wt + (int64_t)k * kStepWorkers; };
#pragma unroll
  for (int k = 0; k < kStepE; ++k) {
    const int64_t e = elem(k);
    double wi = 0.0, v0 = 0.0;
    if (e < own) {
      wi = a.w[s_lo + e];
      if (a.invd) wi = mul_rn(wi, a.invd[s_lo + e]);  // w = pc(A v_j)  (inner.py:249)
      v0 = ld_hint(a.V + s_lo + e, j > 0 ? pol_keep : pol_first);
    }
    wv[k] = wi;
    vc[k] = v0;
  }
  double p[1] = {0.0};
#pragma unroll
  for (int k = 0; k < kStepE; ++k) p[0] = add_rn(p[0], mul_rn(vc[k], wv[k]));
  for (int l = 0; l <= j; ++l) {
    double vn[kStepE];
    if (l < j) {  // V_{l+1} in flight while h_l is reduced
      const double* Vn = a.V + (int64_t)(l + 1) * ldv + s_lo;
      const uint64_t pol = l + 1 < j ? pol_keep : pol_first;
#pragma unroll
      for (int k = 0; k < kStepE; ++k) {
        const int64_t e = elem(k);
        vn[k] = e < own ? ld_hint(Vn + e, pol) : 0.0;
      }
    }
    grid_allreduce<1>(p, ka, slot, gb, sh);
    const double h = p[0];
    if (tid == 0) hcol[l] = h;
    double q = 0.0;
#pragma unroll
    for (int k = 0; k < kStepE; ++k) wv[k] = sub_rn(wv[k], mul_rn(h, vc[k]));
    if (l < j) {
#pragma unroll
      for (int k = 0; k < kStepE; ++k) {
        q = add_rn(q, mul_rn(vn[k], wv[k]));
        vc[k] = vn[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < kStepE; ++k) q = add_rn(q, mul_rn(wv[k], wv[k]));
    }
    p[0] = q;
  }
  grid_allreduce<1>(p, ka, slot, gb, sh);
  const double hnorm = sqrt(p[0]);
  k4_mark_raw(a.trace, a.trace_cap);
  // Givens update (inner.py:256-270), redundantly in every CTA; CTA 0 stores.
  if (tid == 0) {
    hcol[j + 1] = hnorm;
    for (int l = 0; l < j; ++l) {
      const double hl = hcol[l], hl1 = hcol[l + 1];
      const double cs = cs_s[l], sn = sn_s[l];
      hcol[l] = add_rn(mul_rn(cs, hl), mul_rn(sn, hl1));
      hcol[l + 1] = add_rn(mul_rn(-sn, hl), mul_rn(cs, hl1));
    }
    const double denom = hypot(hcol[j], hcol[j + 1]);
    int brk = 0;
    double csj = 0.0, snj = 0.0, gj = gj_s, gj1 = 0.0;
    if (denom == 0.0) {
      brk = 1;
    } else {
      csj = hcol[j] / denom;
      snj = hcol[j + 1] / denom;
      hcol[j] = denom;
      hcol[j + 1] = 0.0;
      gj1 = mul_rn(-snj, gj);
      gj = mul_rn(csj, gj);
      if (fabs(gj1) <= est_s || hnorm == 0.0) brk = 2;
    }
    brk_s = brk;
    // every CTA took its snapshot of st before its first grid barrier, so
    // CTA 0 may update the state now
    if (blockIdx.x == 0) {
      for (int l = 0; l <= j + 1; ++l) st->H[l * R + j] = hcol[l];
      if (brk != 1) {
        st->cs[j] = csj;
        st->sn[j] = snj;
        st->g[j] = gj;
        st->g[j + 1] = gj1;
      }
      const int jn = brk == 1 ? j : j + 1;
      const int itn = st->it + 1;
      st->j = jn;
      st->it = itn;
      st->basis_reads += j + 1;
      st->active = (brk == 0 && jn < R && itn < a.max_it) ? 1 : 0;
      publish_flags(a, *st);
    }
  }
  __syncthreads();
  if (brk_s == 0) {  // V_{j+1} = w / hnorm: the next K3 launch's input, keep it in L2
    double* Vnew = a.V + (int64_t)(j + 1) * ldv + s_lo;
#pragma unroll
    for (int k = 0; k < kStepE; ++k) {
      const int64_t e = elem(k);
      if (e < own) st_hint(Vnew + e, wv[k] / hnorm, pol_keep);
    }
  }
  k4_mark_raw(a.trace, a.trace_cap);
}

// Cycle end (inner.py:272-276): y = H^-1 g by back substitution (:286-292,
// zero pivot -> 0), x += V y.  Every CTA solves the j x j system itself.
__global__ void __launch_bounds__(kStepThreads) step_cycle_end(StepArgs a) {
  __shared__ double y[R];
  const StepState* st = a.s;
  const int j = st->j;
  if (j == 0) return;
  if (threadIdx.x == 0) {
    for (int i = j - 1; i >= 0; --i) {
      double dacc = 0.0;
      for (int k = i + 1; k < j; ++k) dacc = add_rn(dacc, mul_rn(st->H[i * R + k], y[k]));
      const double t = sub_rn(st->g[i], dacc);
      const double d = st->H[i * R + i];
      y[i] = d != 0.0 ? t / d : 0.0;
    }
  }
  __syncthreads();
  const int64_t n = a.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int l = 0; l < j; ++l) t = add_rn(t, mul_rn(a.V[(int64_t)l * a.ldv + i], y[l]));
    a.x[i] = add_rn(a.x[i], t);
  }
}

// After a residual launch wrote r = b - A x: ||r|| (and ||b||, eff on the
// first call), the est_target rule of the finished cycle (:277-282), the
// loop test (:235) and the next cycle's start z = pc(r), beta = ||z||,
// V_0 = z / beta (:236-247).
__global__ void __launch_bounds__(kStepThreads, 1) step_cycle_start(StepArgs a) {
  __shared__ KShared sh;
  StepState* st = a.s;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (blockIdx.x == 0 && tid == 0) a.bar[a.parity ^ 1] = 0u;
  GridBarrier gb{a.bar + a.parity, 0u, 0};
  const KArgs ka = step_kargs(a);
  int slot = 0;
  const int64_t n = a.n;
  int64_t s_lo, s_hi;
  step_slice(n, s_lo, s_hi);
  // snapshot everything this kernel reads from st before the first barrier
  const int first = a.first, it = first ? 0 : st->it, jprev = first ? 0 : st->j;
  const double gj = first ? 0.0 : fabs(st->g[jprev]);
  double eff = first ? 0.0 : st->eff, est_target = first ? 0.0 : st->est_target;
  double q[2] = {0.0, 0.0};
  for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
    const double ri = a.r[i];
    q[0] = add_rn(q[0], mul_rn(ri, ri));
    if (first) q[1] = add_rn(q[1], mul_rn(a.b[i], a.b[i]));
  }
  grid_allreduce<2>(q, ka, slot, gb, sh);
  const double rn = sqrt(q[0]);
  bool done = false;
  if (first) {
    eff = fmax(st->target, 1e-14 * fmax(1.0, sqrt(q[1])));  // inner.py:189
    est_target = eff;
  } else if (rn > eff && gj <= est_target) {
    if (gj == 0.0) done = true;
    else est_target = mul_rn(mul_rn(gj, eff / rn), 0.5);
  }
  if (!(rn > eff && it < a.max_it)) done = true;
  double beta = rn;
  if (!done) {
    double z2[1] = {0.0};
    for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
      const double z = a.invd ? mul_rn(a.r[i], a.invd[i]) : a.r[i];
      a.V[i] = z;
      z2[0] = add_rn(z2[0], mul_rn(z, z));
    }
    if (a.invd) {
      grid_allreduce<1>(z2, ka, slot, gb, sh);
      beta = sqrt(z2[0]);
    }
    if (beta == 0.0 || !isfinite(beta)) done = true;
    else
      for (int64_t i = s_lo + tid; i < s_hi; i += nthr) a.V[i] = a.V[i] / beta;
  }
  if (blockIdx.x == 0 && tid == 0) {
    st->rn = rn;
    st->eff = eff;
    st->est_target = est_target;
    st->done = done ? 1 : 0;
    st->it = it;
    if (!done) {
      for (int k = 0; k < (R + 1) * R; ++k) st->H[k] = 0.0;
      for (int k = 0; k < R; ++k) st->cs[k] = st->sn[k] = 0.0;
      for (int k = 0; k <= R; ++k) st->g[k] = 0.0;
      st->g[0] = beta;
      st->j = 0;
      st->active = 1;
    } else {
      st->active = 0;
    }
    publish_flags(a, *st);
  }
}

bool stepped_gmres_fits(int64_t n, int sms) {
  return (n + sms - 1) / sms + 2 <= (int64_t)kStepWorkers * kStepE;
}

int64_t stepped_gmres_workspace(int64_t n, int blocks) {
  const int64_t ldv = (n + 1) & ~(int64_t)1;
  return (int64_t)(R + 1) * ldv + 2 * n + 2 + 2 * kPartStride * (int64_t)blocks + 64 +
         (int64_t)(sizeof(StepState) + 7) / 8;
}

// Host loop (inner.py:229-283).  `op` is the planned K3 operator of P_pi.
int stepped_gmres(const ipi_op* op, int64_t n, const double* b, double* x, double target,
                  int32_t max_it, const double* inv_diag, ipi_inner_report* d_report,
                  double* ws, int64_t ws_doubles, cudaStream_t st) {
  int dev = 0, sms = 148;
  IPI_CUDA_TRY(cudaGetDevice(&dev));
  IPI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms;
  if (ws_doubles < stepped_gmres_workspace(n, blocks))
    return fail(IPI_ERESOURCE, "stepped GMRES: workspace too small");
  // mapped host flags, one block per device (pinned allocations are slow to make)
  static StepFlags* h_flags[64] = {};
  if (dev < 0 || dev >= 64) return fail(IPI_ECUDA, "device index out of range");
  if (!h_flags[dev]) IPI_CUDA_TRY(cudaHostAlloc(&h_flags[dev], sizeof(StepFlags), cudaHostAllocMapped));
  volatile StepFlags* hf = h_flags[dev];
  StepFlags* hf_dev = nullptr;
  IPI_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hf_dev), h_flags[dev], 0));
  StepArgs a{};
  a.n = n;
  a.b = b;
  a.x = x;
  a.ldv = (n + 1) & ~(int64_t)1;
  a.V = ws;
  a.w = ws + (int64_t)(R + 1) * a.ldv;
  a.r = a.w + n + 2;
  a.partials = a.r + n;
  a.bar = reinterpret_cast<unsigned*>(a.partials + 2 * kPartStride * (int64_t)blocks);
  a.s = reinterpret_cast<StepState*>(a.partials + 2 * kPartStride * (int64_t)blocks + 64);
  a.invd = inv_diag;
  a.hf = hf_dev;
  a.max_it = max_it;
  a.trace = k4_trace_buffer(&a.trace_cap);
  if (a.trace) IPI_CUDA_TRY(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long), st));
  IPI_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned), st));
  {
    StepState init{};
    init.target = target;
    IPI_CUDA_TRY(cudaMemcpyAsync(a.s, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  const int* active = &a.s->active;
  {
    int per_sm = 0;
    IPI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_ortho, kStepThreads, 0));
    if (per_sm < 1) return fail(IPI_ECUDA, "step_ortho cannot be resident");
  }
  auto coop = [&](const void* fn, int smem = 0) -> int {
    void* args[] = {(void*)&a};
    IPI_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kStepThreads), args, (size_t)smem, st));
    a.parity ^= 1;
    return IPI_OK;
  };
  cudaEvent_t ev[2];
  IPI_CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  if (cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess) {
    cudaEventDestroy(ev[0]);
    return fail(IPI_ECUDA, "event create");
  }
  struct Guard {
    cudaEvent_t* e;
    ~Guard() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } guard{ev};
  auto read_flags = [&](StepFlags& f) {
    f.active = hf->active;
    f.j = hf->j;
    f.it = hf->it;
    f.done = hf->done;
    f.rn = hf->rn;
  };
  int rc;
  // r = b - A x, then ||r||, ||b||, eff, the first cycle's start
  if ((rc = op_launch(op, x, b, 2, a.r, st))) return rc;
  a.first = 1;
  if ((rc = coop((const void*)step_cycle_start))) return rc;
  a.first = 0;
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  StepFlags f{};
  read_flags(f);
  while (!f.done) {
    // Arnoldi steps, one enqueued ahead of the one the host waits for
    int issued = 0, waited = 0;
    auto issue = [&]() -> int {
      int e;
      if ((e = op_launch(op, a.V + (int64_t)issued * a.ldv, nullptr, 1, a.w, st, nullptr, active))) return e;
      if ((e = coop((const void*)step_ortho))) return e;
      IPI_CUDA_TRY(cudaEventRecord(ev[issued & 1], st));
      ++issued;
      return IPI_OK;
    };
    if ((rc = issue())) return rc;
    while (true) {
      // the host's view of the cycle: steps beyond j + 1 are launched only
      // while the device says the cycle is active
      if (issued < R && issued == waited + 1 && (rc = issue())) return rc;
      IPI_CUDA_TRY(cudaEventSynchronize(ev[waited & 1]));
      ++waited;
      read_flags(f);
      if (!f.active) break;  // steps already issued beyond it skip themselves
      if (waited >= issued) break;  // R steps issued and all done
    }
    IPI_CUDA_TRY(cudaStreamSynchronize(st));  // the no-op tail step (if any) retired
    read_flags(f);
    if (f.j == 0) break;  // inner.py:271-272
    // x += V y, r = b - A x, est_target / loop test / next cycle start
    step_cycle_end<<<blocks * 2, kStepThreads, 0, st>>>(a);
    IPI_LAUNCH_CHECK();
    if ((rc = op_launch(op, x, b, 2, a.r, st))) return rc;
    if ((rc = coop((const void*)step_cycle_start))) return rc;
    IPI_CUDA_TRY(cudaStreamSynchronize(st));
    read_flags(f);
  }
  ipi_inner_report rep{};
  rep.iterations = f.it;
  rep.final_linear_residual_2norm = f.rn;
  StepState fin;
  IPI_CUDA_TRY(cudaMemcpyAsync(&fin, a.s, sizeof(fin), cudaMemcpyDeviceToHost, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  rep.iterations = fin.it;
  rep.final_linear_residual_2norm = fin.rn;
  rep.converged = fin.rn <= fin.eff ? 1 : 0;
  rep.breakdown = 0;
  rep.basis_reads = fin.basis_reads;
  rep.target_2norm = fin.eff;
  IPI_CUDA_TRY(cudaMemcpyAsync(d_report, &rep, sizeof(rep), cudaMemcpyHostToDevice, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  return IPI_OK;
}

}  // namespace ipi
