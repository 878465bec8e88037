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
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <utility>

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
  const double* tv;  // first call: r = tv - x instead of reading a.r (the caller's b + gamma P x), or nullptr
  unsigned long long* trace;  // diagnostics (ipi_k4_trace): step_ortho start / MGS done / end
  int trace_cap;
  unsigned long long* board;  // LL all-reduce mailboxes + result slots (ll_allreduce)
  unsigned call_base;         // first LL call number of this launch (unique per launch)
  int pf;                     // step_ortho: basis vectors prefetched into L2 ahead of the MGS pass
  int pdl;                    // step_ortho*: launched with programmatic stream serialization
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

// step_ortho: CTA 0 is the all-reduce's reducer and owns no elements; the
// worker CTAs 1..nb-1 split the vectors.
__device__ __forceinline__ void ortho_slice(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t c = (int64_t)blockIdx.x - 1, nb = (int64_t)gridDim.x - 1;
  if (c < 0) {
    lo = hi = 0;
    return;
  }
  lo = c == 0 ? 0 : ((n * c / nb) & ~(int64_t)1);
  hi = c + 1 == nb ? n : ((n * (c + 1) / nb) & ~(int64_t)1);
}

// ---------------------------------------------------------------------------
// LL all-reduce: a deterministic grid all-reduce of NV <= 3 doubles without a
// counter barrier or fences.  A message is two 8-byte words, each carrying 32
// data bits and the 32-bit call number, so every word validates itself and no
// ordering between words is needed (relaxed gpu-scope accesses; the protocol
// NCCL's LL uses).  Worker CTAs post their block partial to their mailbox;
// CTA 0 gathers with one polling lane per mailbox (warp 5 v + q takes value v
// of CTAs 32 q + lane: with a single polling warp the fan-in cost 1.4 us more,
// scripts/micro/allreduce_ll2.cu), adds them in CTA order (lane-wise over q,
// then the fixed xor tree) and posts the sums to the result slots every worker
// polls.  Measured 1.64 us per call on 148 CTAs against 2.3 us for the counter
// barrier + ordered partial reads of grid_allreduce.  Call numbers never repeat
// within a solve (the board is zeroed per solve; numbers start at 1), so a
// stale mailbox can never match.
// ---------------------------------------------------------------------------
constexpr int kLLVals = 3;
constexpr int kLLChunks = 5;  // reducer lanes cover up to 160 CTAs

struct LLShared {
  double red[kLLVals * 32];
  double xs[kLLVals][kLLChunks][32];
  double bc[4];
};

__device__ __forceinline__ void ll_store(unsigned long long* dst, double v, unsigned call) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = (bits & 0xffffffffull) | ((unsigned long long)call << 32);
  const unsigned long long w1 = (bits >> 32) | ((unsigned long long)call << 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ double ll_wait(const unsigned long long* src, unsigned call) {
  unsigned long long w0, w1;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(src) : "memory");
  } while ((unsigned)(w0 >> 32) != call || (unsigned)(w1 >> 32) != call);
  return __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
}

int64_t ll_board_words(int blocks) { return 2 * ((int64_t)kLLVals * blocks + kLLVals + 5); }

// Named CTA barriers of the split all-reduce: the worker warps arrive on
// kBarPosted without waiting (their partials are in shared memory), issue
// whatever loads they want in flight during the exchange, and wait on
// kBarResult, which the control warp (warp 0) arrives on once the sums are in
// sh.bc.  (With the loads issued before a blocking barrier the workers only
// reached it after the load queue had drained: +0.8 us per MGS pass.)
constexpr int kBarPosted = 1, kBarResult = 2, kBarGo = 3;

// NV warp sums with their shuffle levels interleaved (independent chains: the
// latency of one level is paid once, not NV times); same xor tree as warp_sum.
template <int NV>
__device__ __forceinline__ void warp_sum_n(double (&t)[NV]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double o[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) o[k] = __shfl_xor_sync(kFull, t[k], off);
#pragma unroll
    for (int k = 0; k < NV; ++k) t[k] = add_rn(t[k], o[k]);
  }
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// First half, every thread of every CTA: `v` holds the thread's partials
// (ignored in CTA 0).  Worker threads return at once; warp 0 of a worker CTA
// returns after posting the block's partial; CTA 0 returns after publishing.
template <int NV>
__device__ __forceinline__ void ll_post(const double (&v)[NV], unsigned long long* board, unsigned& call,
                                        LLShared& sh) {
  static_assert(NV <= kLLVals, "LL all-reduce carries up to kLLVals values");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nb = gridDim.x;
  const int nthr = blockDim.x;
  unsigned long long* pub = board + 2 * (int64_t)kLLVals * nb;
  ++call;
  if (blockIdx.x != 0) {
    if (warp != 0) {
      double t[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) t[k] = v[k];
      warp_sum_n<NV>(t);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sh.red[k * 32 + warp] = t[k];
      }
      bar_arrive(kBarPosted, nthr);
      // the block's post enters the memory pipeline ahead of the callers' loads:
      // behind a 57 KB load burst it left the SM ~1500 cycles late
      bar_sync(kBarGo, nthr);
    } else {
      bar_sync(kBarPosted, nthr);
      const int nw = nthr >> 5;
      double t[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k)  // warp 0 holds no elements: lanes 1.. carry the workers
        t[k] = lane >= 1 && lane < nw ? sh.red[k * 32 + lane] : 0.0;
      warp_sum_n<NV>(t);
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (lane == k) ll_store(board + 2 * ((int64_t)k * nb + blockIdx.x), t[k], call);
      bar_arrive(kBarGo, nthr);
    }
  } else {
    if (warp < kLLChunks * NV) {
      const int k = warp / kLLChunks, q = warp % kLLChunks, c = lane + 32 * q;
      sh.xs[k][q][lane] = c >= 1 && c < nb ? ll_wait(board + 2 * ((int64_t)k * nb + c), call) : 0.0;
    }
    __syncthreads();
    if (warp < NV) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kLLChunks; ++q)
        if (lane + 32 * q < nb) s = add_rn(s, sh.xs[warp][q][lane]);
      s = warp_sum(s);
      if (lane == 0) {
        ll_store(pub + 2 * warp, s, call);
        sh.bc[warp] = s;
      }
    }
  }
}

// Second half: on return every thread of the grid holds the sums in `v`.
template <int NV>
__device__ __forceinline__ void ll_wait_result(double (&v)[NV], unsigned long long* board, unsigned call,
                                               LLShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nb = gridDim.x;
  const int nthr = blockDim.x;
  const unsigned long long* pub = board + 2 * (int64_t)kLLVals * nb;
  if (blockIdx.x != 0) {
    if (warp == 0) {
      if (lane < NV) sh.bc[lane] = ll_wait(pub + 2 * lane, call);
      bar_arrive(kBarResult, nthr);
    } else {
      bar_sync(kBarResult, nthr);
    }
  } else {
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sh.bc[k];
}

template <int NV>
__device__ __forceinline__ void ll_allreduce(double (&v)[NV], unsigned long long* board, unsigned& call,
                                             LLShared& sh) {
  ll_post<NV>(v, board, call, sh);
  ll_wait_result<NV>(v, board, call, sh);
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
  // no system fence: the host reads the mirror only after synchronising on an
  // event recorded behind this launch, which makes the kernel's writes visible
}

// Givens update of the new Hessenberg column (inner.py:256-270), run by
// thread 0 of every CTA on identical inputs; CTA 0 stores the state.  Every
// CTA took its snapshot of the state before its first all-reduce of the
// launch, so CTA 0 may update it here.
__device__ __forceinline__ void step_givens(const StepArgs& a, StepState* st, int j, double hnorm,
                                            double* hcol, const double* cs_s, const double* sn_s,
                                            double gj_s, double est_s, int& brk_s) {
  if (threadIdx.x != 0) return;
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

// One Arnoldi step after the K3 launch wrote w = V_j - gamma P V_j: MGS with
// this CTA's slice of w in registers and V_{l+1}'s slice loaded into
// registers while the all-reduce producing h_l is in flight, so a pass costs
// one grid all-reduce plus register arithmetic (C2: ~3.5 us per pass).
// (Streaming the slices through shared memory with 1-D bulk copies two
// passes ahead measured slower: 4.5 us per pass.)
__global__ void __launch_bounds__(kStepThreads, 1) step_ortho(StepArgs a) {
  __shared__ LLShared sh;
  __shared__ double hcol[R + 1], cs_s[R], sn_s[R], gj_s, est_s;
  __shared__ int brk_s;
  StepState* st = a.s;
  const int tid = threadIdx.x;
  if (a.pdl) {
    griddep_wait();
    griddep_launch_dependents();
  }
  // the next cooperative launch's barrier counter (its previous user, two
  // launches back, has retired); reset even when this launch is a no-op
  if (blockIdx.x == 0 && tid == 0) a.bar[a.parity ^ 1] = 0u;
  if (!st->active) return;  // uniform: the previous launch ended the cycle
  k4_mark_raw(a.trace, a.trace_cap);
  unsigned call = a.call_base;
  const int j = st->j;
  const int64_t n = a.n, ldv = a.ldv;
  int64_t s_lo, s_hi;
  ortho_slice(n, s_lo, s_hi);
  const int64_t own = s_hi - s_lo;
  const uint64_t pol_keep = policy_evict_last(), pol_first = policy_evict_first();
  if (tid == 0) {  // snapshot the rotation state before the first all-reduce:
    for (int l = 0; l < j; ++l) {  // CTA 0 updates g[j] after the last one
      cs_s[l] = st->cs[l];
      sn_s[l] = st->sn[l];
    }
    gj_s = st->g[j];
    est_s = st->est_target;
  }
  // The basis does not stay in L2 across the K3 launches (P_pi streams 822 MB
  // per step), and with only V_{l+1} in flight a pass waits one DRAM round
  // trip (3.3 us per pass on C2).  The control warp therefore pulls this CTA's
  // slices of the next a.pf vectors into L2 with bulk prefetches; the register
  // loads below then hit L2.
  const uint32_t pf_bytes = (uint32_t)((own * 8) & ~(int64_t)15);
  if (tid < a.pf && tid + 1 <= j && pf_bytes)
    l2_prefetch(a.V + (int64_t)(tid + 1) * ldv + s_lo, pf_bytes);
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
    ll_post<1>(p, a.board, call, sh);
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
    if (tid == 0 && l + 1 + a.pf <= j && pf_bytes)
      l2_prefetch(a.V + (int64_t)(l + 1 + a.pf) * ldv + s_lo, pf_bytes);
    ll_wait_result<1>(p, a.board, call, sh);
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
  ll_allreduce<1>(p, a.board, call, sh);
  const double hnorm = sqrt(p[0]);
  k4_mark_raw(a.trace, a.trace_cap);
  // V_{j+1} = w / hnorm (the next K3 launch's input: keep it in L2) goes out
  // while thread 0 runs the Givens update; when that update ends the cycle the
  // vector is simply not used (slot j + 1 <= R exists).  hnorm == 0 is the
  // breakdown case (inner.py:268-270): nothing is written.
  if (hnorm != 0.0) {
    double* Vnew = a.V + (int64_t)(j + 1) * ldv + s_lo;
#pragma unroll
    for (int k = 0; k < kStepE; ++k) {
      const int64_t e = elem(k);
      if (e < own) st_hint(Vnew + e, wv[k] / hnorm, pol_keep);
    }
  }
  step_givens(a, st, j, hnorm, hcol, cs_s, sn_s, gj_s, est_s, brk_s);
  k4_mark_raw(a.trace, a.trace_cap);
}

// Pair-blocked MGS: the same Arnoldi step with the basis taken two vectors per
// all-reduce, so a step makes ceil((j+1)/2) + 1 dependent grid exchanges
// instead of j + 2.  For the pair (V_l, V_{l+1}) one exchange carries
//   d0 = <V_l, w_l>,  d1 = <V_{l+1}, w_l>,  G = <V_{l+1}, V_l>
// and h_l = d0, h_{l+1} = d1 - h_l G, which is MGS's <V_{l+1}, w_l - h_l V_l>
// expanded by linearity: identical in exact arithmetic, and it keeps MGS's
// correction for a basis that has lost orthogonality (G is the measured
// inner product, ~1e-16 here, not assumed zero).  w is then updated as MGS
// does, (w - h_l V_l) - h_{l+1} V_{l+1}.  h_l is bitwise MGS's; h_{l+1}
// differs from it by rounding of order eps |w|.  Inner products and updates use
// fused multiply-adds: the reference's dots are BLAS dots, whose rounding order
// is not specified, so the h_l are not bitwise the reference's in any case, and
// the FP64 pipe is what the compute phase of a pass waits for (7 -> 5
// instructions per element and pair).  IPI_STEP_PAIR=0 keeps numpy's separate
// mul / add roundings throughout.
//
// Data movement: the pair in use lives in registers (va, vb); the next pair is
// copied into shared memory with cp.async (16-byte chunks, every thread copies
// exactly the elements it owns, so it waits only on its own groups) while the
// exchange of the current pair is in flight.  After the w update has released
// va / vb, the dots of the next pair read the stage once and leave that pair
// in the registers, so the stage is free again at the next exchange.
constexpr int kPairChunks = kStepE / 2;                          // 16-byte chunks per thread and vector
constexpr int kPairSmem = 2 * kPairChunks * kStepWorkers * 16;   // two vectors staged

__global__ void __launch_bounds__(kStepThreads, 1) step_ortho_pair(StepArgs a) {
  extern __shared__ __align__(16) unsigned char stage_raw[];
  __shared__ LLShared sh;
  __shared__ double hcol[R + 1], cs_s[R], sn_s[R], gj_s, est_s;
  __shared__ int brk_s;
  StepState* st = a.s;
  const int tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) a.bar[a.parity ^ 1] = 0u;
  if (!st->active) return;  // uniform: the previous launch ended the cycle
  if (a.pdl) griddep_launch_dependents();  // the next K3 launch may stage its first P_pi rows
  k4_mark_raw(a.trace, a.trace_cap);
  unsigned call = a.call_base;
  const int j = st->j;
  const int64_t n = a.n, ldv = a.ldv;
  int64_t s_lo, s_hi;
  ortho_slice(n, s_lo, s_hi);
  const int own = (int)(s_hi - s_lo);  // <= kStepWorkers * kStepE: 32-bit slice indices
  const uint64_t pol_keep = policy_evict_last(), pol_first = policy_evict_first();
  if (tid == 0) {
    for (int l = 0; l < j; ++l) {
      cs_s[l] = st->cs[l];
      sn_s[l] = st->sn[l];
    }
    gj_s = st->g[j];
    est_s = st->est_target;
  }
  const int wt = tid - 32;  // worker index (< 0: the control warp owns nothing)
  // element k of this thread: chunk k/2 (16 bytes), half k%2
  auto elem = [&](int k) -> int {
    return wt < 0 ? own : 2 * (wt + (k >> 1) * kStepWorkers) + (k & 1);
  };
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage_raw);
  auto slot = [&](int v, int c) -> uint32_t {  // byte offset of chunk c of staged vector v
    return (uint32_t)(((v * kPairChunks + c) * kStepWorkers + (int)(wt < 0 ? 0 : wt)) * 16);
  };
  // stage vectors l, l+1 (those <= j) of the basis: this thread's chunks only
  auto stage_pair = [&](int l) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      if (l + v <= j) {
        const double* Vl = a.V + (int64_t)(l + v) * ldv + s_lo;
        const uint64_t pol = l + v < j ? pol_keep : pol_first;
#pragma unroll
        for (int c = 0; c < kPairChunks; ++c) {
          const int e = elem(2 * c);
          if (e < own) cp_async16(stage_s + slot(v, c), Vl + e, e + 1 < own ? 16u : 8u, pol);
        }
      }
    }
    cp_async_commit();
  };
  auto staged = [&](int v, int c) -> double2 {
    return *reinterpret_cast<const double2*>(stage_raw + slot(v, c));
  };
  // The basis and the solver state were written by launches that finished
  // before the K3 launch ahead of this one started: under programmatic
  // dependent launch they are read while that K3 launch drains; only w waits.
  double wv[kStepE], va[kStepE], vb[kStepE];
#pragma unroll
  for (int k = 0; k < kStepE; ++k) {
    const int e = elem(k);
    double v0 = 0.0, v1 = 0.0;
    if (e < own) {
      v0 = ld_hint(a.V + s_lo + e, j > 0 ? pol_keep : pol_first);
      if (j >= 1) v1 = ld_hint(a.V + ldv + s_lo + e, j > 1 ? pol_keep : pol_first);
    }
    va[k] = v0;
    vb[k] = v1;
  }
  if (j >= 2) stage_pair(2);
  if (a.pdl) griddep_wait();
#pragma unroll
  for (int k = 0; k < kStepE; ++k) {
    const int e = elem(k);
    double wi = 0.0;
    if (e < own) {
      wi = a.w[s_lo + e];
      if (a.invd) wi = mul_rn(wi, a.invd[s_lo + e]);  // w = pc(A v_j)  (inner.py:249)
    }
    wv[k] = wi;
  }
  double p[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < kStepE; ++k) {
    p[0] = fma(va[k], wv[k], p[0]);
    p[1] = fma(vb[k], wv[k], p[1]);
    p[2] = fma(vb[k], va[k], p[2]);
  }
  for (int l = 0; l <= j; l += 2) {
    const bool two = l + 1 <= j, more = l + 2 <= j;
    ll_post<3>(p, a.board, call, sh);
    // the pair being exchanged is already in va / vb (the dots below left it
    // there), so the stage is free: it takes the next pair during the exchange
    if (l > 0 && more) stage_pair(l + 2);
    ll_wait_result<3>(p, a.board, call, sh);
    const double h0 = p[0];
    const double h1 = two ? sub_rn(p[1], mul_rn(h0, p[2])) : 0.0;
    if (tid == 0) {
      hcol[l] = h0;
      if (two) hcol[l + 1] = h1;
    }
#pragma unroll
    for (int k = 0; k < kStepE; ++k) {  // (w - h_l V_l) - h_{l+1} V_{l+1}, one rounding per term
      wv[k] = fma(-h0, va[k], wv[k]);
      if (two) wv[k] = fma(-h1, vb[k], wv[k]);
    }
    double q0 = 0.0, q1 = 0.0, q2 = 0.0;
    if (more) {
      const bool two_n = l + 3 <= j;
      cp_async_wait<0>();  // this thread's chunks of the next pair
      // the update above released va / vb: the next pair moves into them here
#pragma unroll
      for (int c = 0; c < kPairChunks; ++c) {
        // chunks past the slice were never staged; a chunk's second half is
        // zero-filled past the slice end (8-byte copy)
        const bool ok = elem(2 * c) < own;
        const double2 x = ok ? staged(0, c) : make_double2(0.0, 0.0);
        const double2 y = ok && two_n ? staged(1, c) : make_double2(0.0, 0.0);
        va[2 * c] = x.x;
        va[2 * c + 1] = x.y;
        vb[2 * c] = y.x;
        vb[2 * c + 1] = y.y;
        q0 = fma(x.x, wv[2 * c], q0);
        q0 = fma(x.y, wv[2 * c + 1], q0);
        q1 = fma(y.x, wv[2 * c], q1);
        q1 = fma(y.y, wv[2 * c + 1], q1);
        q2 = fma(y.x, x.x, q2);
        q2 = fma(y.y, x.y, q2);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kStepE; ++k) q0 = fma(wv[k], wv[k], q0);
    }
    p[0] = q0;
    p[1] = q1;
    p[2] = q2;
  }
  double pn[1] = {p[0]};
  ll_allreduce<1>(pn, a.board, call, sh);
  const double hnorm = sqrt(pn[0]);
  k4_mark_raw(a.trace, a.trace_cap);
  // V_{j+1} = w / hnorm (the next K3 launch's input: keep it in L2) goes out
  // while thread 0 runs the Givens update; when that update ends the cycle the
  // vector is simply not used (slot j + 1 <= R exists).  hnorm == 0 is the
  // breakdown case (inner.py:268-270): nothing is written.
  if (hnorm != 0.0) {
    double* Vnew = a.V + (int64_t)(j + 1) * ldv + s_lo;
#pragma unroll
    for (int k = 0; k < kStepE; ++k) {
      const int e = elem(k);
      if (e < own) st_hint(Vnew + e, wv[k] / hnorm, pol_keep);
    }
  }
  step_givens(a, st, j, hnorm, hcol, cs_s, sn_s, gj_s, est_s, brk_s);
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
  // r0 = (b + gamma P x0) - x0 when the caller already holds b + gamma P x0 (the
  // outer loop's TV): the same residual as b - (x0 - gamma P x0) up to the
  // rounding of the last two operations, and one SpMV less per inner solve
  const bool from_tv = first && a.tv != nullptr;
  auto resid = [&](int64_t i) -> double { return from_tv ? sub_rn(a.tv[i], a.x[i]) : a.r[i]; };
  double q[2] = {0.0, 0.0};
  for (int64_t i = s_lo + tid; i < s_hi; i += nthr) {
    const double ri = resid(i);
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
      const double ri = resid(i);
      const double z = a.invd ? mul_rn(ri, a.invd[i]) : ri;
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
  const int64_t workers = sms - 1;  // CTA 0 is the all-reduce's reducer
  return sms >= 2 && sms <= 32 * kLLChunks && (n + workers - 1) / workers + 2 <= (int64_t)kStepWorkers * kStepE;
}

int64_t stepped_gmres_workspace(int64_t n, int blocks) {
  const int64_t ldv = (n + 1) & ~(int64_t)1;
  return (int64_t)(R + 1) * ldv + 2 * n + 2 + 2 * kPartStride * (int64_t)blocks + 64 +
         (((int64_t)(sizeof(StepState) + 7) / 8 + 1) & ~(int64_t)1) + ll_board_words(blocks);
}

// Host loop (inner.py:229-283).  `op` is the planned K3 operator of P_pi.
int stepped_gmres(const ipi_op* op, int64_t n, const double* b, double* x, double target,
                  int32_t max_it, const double* inv_diag, ipi_inner_report* d_report,
                  double* ws, int64_t ws_doubles, cudaStream_t st, const double* tv) {
  int dev = 0, sms = 148;
  IPI_CUDA_TRY(cudaGetDevice(&dev));
  IPI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms;
  if (ws_doubles < stepped_gmres_workspace(n, blocks))
    return fail(IPI_ERESOURCE, "stepped GMRES: workspace too small");
  // mapped host flags, one block per (device, stream): pinned allocations are
  // slow to make, and two solves on two streams must not share a mirror
  static std::mutex flags_mu;
  static std::map<std::pair<int, cudaStream_t>, StepFlags*> flags_of;
  StepFlags* h_flags = nullptr;
  {
    std::lock_guard<std::mutex> lk(flags_mu);
    StepFlags*& slot = flags_of[{dev, st}];
    if (!slot) IPI_CUDA_TRY(cudaHostAlloc(&slot, sizeof(StepFlags), cudaHostAllocMapped));
    h_flags = slot;
  }
  volatile StepFlags* hf = h_flags;
  StepFlags* hf_dev = nullptr;
  IPI_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hf_dev), h_flags, 0));
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
  a.board = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<double*>(a.s) + (((int64_t)(sizeof(StepState) + 7) / 8 + 1) & ~(int64_t)1));
  a.call_base = 0;
  static const int pf_env = getenv("IPI_STEP_PF") ? atoi(getenv("IPI_STEP_PF")) : 4;
  a.pf = std::min(std::max(pf_env, 0), 32);
  a.invd = inv_diag;
  a.hf = hf_dev;
  a.max_it = max_it;
  a.trace = k4_trace_buffer(&a.trace_cap);
  if (a.trace) IPI_CUDA_TRY(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long), st));
  IPI_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned), st));
  IPI_CUDA_TRY(cudaMemsetAsync(a.board, 0, ll_board_words(blocks) * sizeof(unsigned long long), st));
  {
    StepState init{};
    init.target = target;
    IPI_CUDA_TRY(cudaMemcpyAsync(a.s, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  const int* active = &a.s->active;
  // IPI_STEP_PAIR=0: one basis vector per grid exchange (bitwise MGS) instead of the pair-blocked kernel
  static const int pair = getenv("IPI_STEP_PAIR") ? atoi(getenv("IPI_STEP_PAIR")) : 1;
  if (pair) IPI_CUDA_TRY(raise_smem_limit(step_ortho_pair, kPairSmem));
  {
    int per_sm = 0;
    IPI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_ortho, kStepThreads, 0));
    if (per_sm < 1) return fail(IPI_ECUDA, "step_ortho cannot be resident");
  }
  // IPI_STEP_PDL=0: plain stream order between the K3 and step_ortho launches
  static std::atomic<int> pdl_ok{getenv("IPI_STEP_PDL") ? atoi(getenv("IPI_STEP_PDL")) : 1};
  auto coop = [&](const void* fn, int smem = 0, bool pdl = false) -> int {
    void* args[] = {(void*)&a};
    a.pdl = pdl && pdl_ok ? 1 : 0;
    if (a.pdl) {
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(kStepThreads);
      cfg.dynamicSmemBytes = (size_t)smem;
      cfg.stream = st;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
      if (e == cudaSuccess) {
        a.parity ^= 1;
        return IPI_OK;
      }
      cudaGetLastError();  // the combination is refused: fall back to stream order for good
      pdl_ok = 0;
      a.pdl = 0;
    }
    IPI_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kStepThreads), args, (size_t)smem, st));
    a.parity ^= 1;
    return IPI_OK;
  };
  cudaEvent_t ev[3] = {};  // two step events (alternating) and the cycle-start event
  struct Guard {
    cudaEvent_t* e;
    ~Guard() {
      for (int i = 0; i < 3; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  for (int i = 0; i < 3; ++i) IPI_CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  auto read_flags = [&](StepFlags& f) {
    f.active = hf->active;
    f.j = hf->j;
    f.it = hf->it;
    f.done = hf->done;
    f.rn = hf->rn;
  };
  int rc;
  // r = b - A x (or tv - x), then ||r||, ||b||, eff, the first cycle's start
  a.tv = tv;
  if (!tv && (rc = op_launch(op, x, b, 2, a.r, st))) return rc;
  a.first = 1;
  if ((rc = coop((const void*)step_cycle_start))) return rc;
  a.first = 0;
  a.tv = nullptr;
  IPI_CUDA_TRY(cudaEventRecord(ev[2], st));
  // Arnoldi steps, one enqueued ahead of the one the host waits for.  The first
  // step of a cycle is enqueued right behind step_cycle_start, before the host
  // knows whether the solve is done: a launched step skips itself when the
  // device state says so, and the GPU has work while the host wakes up.
  int issued = 0, waited = 0;
  auto issue = [&]() -> int {
    int e;
    if ((e = op_launch(op, a.V + (int64_t)issued * a.ldv, nullptr, 1, a.w, st, nullptr, active, pdl_ok.load()))) return e;
    if ((e = pair ? coop((const void*)step_ortho_pair, kPairSmem, true) : coop((const void*)step_ortho, 0, true)))
      return e;
    a.call_base += R + 2;  // a launch makes at most R + 1 calls
    IPI_CUDA_TRY(cudaEventRecord(ev[issued & 1], st));
    ++issued;
    return IPI_OK;
  };
  if ((rc = issue())) return rc;
  IPI_CUDA_TRY(cudaEventSynchronize(ev[2]));  // step_cycle_start's flags; the speculative step runs on
  StepFlags f{};
  read_flags(f);
  // f.done is set only by step_cycle_start (steps republish it unchanged); when
  // it is set the speculative step is a no-op
  while (!f.done) {
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
    // a no-op tail step (if any) changes nothing: the flags read above are the
    // cycle's last, and the launches below follow it in stream order
    if (f.j == 0) break;  // inner.py:271-272
    // x += V y, r = b - A x, est_target / loop test / next cycle start
    step_cycle_end<<<blocks * 2, kStepThreads, 0, st>>>(a);
    IPI_LAUNCH_CHECK();
    if ((rc = op_launch(op, x, b, 2, a.r, st))) return rc;
    if ((rc = coop((const void*)step_cycle_start))) return rc;
    IPI_CUDA_TRY(cudaEventRecord(ev[2], st));
    issued = waited = 0;
    if ((rc = issue())) return rc;  // speculative first step of the next cycle
    IPI_CUDA_TRY(cudaEventSynchronize(ev[2]));
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
  IPI_CUDA_TRY(cudaMemcpyAsync(d_report, &rep, sizeof(rep), cudaMemcpyHostToDevice, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  return IPI_OK;
}

}  // namespace ipi
