// sharded.cu — the row-sharded iPI driver (one process per GPU), natively:
// driver.py:109-209 across ranks with the inner GMRES(30) / Richardson on the
// rank's rows, every scalar on the device, and the two exchanges the path has
// going through the caller's collectives (ipi_comm):
//
//   * the value vector: every SpMV (K1's V, the Krylov vectors, the iterate)
//     needs the full vector, assembled from the ranks' blocks
//     (allgather_blocks: NCCL broadcasts of each rank's block in one group);
//   * scalars: each rank's partial dots are all-gathered (R x cnt doubles) and
//     every rank adds them in rank order, so every rank holds bit-identical
//     scalars and takes the same decisions (parallel.py:21-33 tree_reduce
//     semantics, deterministic at fixed R).
//
// Arnoldi orthogonalisation is CGS2 (classical Gram-Schmidt with one full
// re-orthogonalisation): 3 all-gathers of partials per step whatever j,
// against MGS's j+2 (inner.py:251-253), the choice SURVEY §8(e) names for
// multi-GPU runs.  The host stays one Arnoldi step ahead of the device: it
// enqueues step j+1 (kernels and collectives) and only then waits for step
// j's event and reads the break decision from mapped flags; a step the
// previous one ended skips itself on the device (every kernel reads
// state.active; the collectives still run, on every rank alike, and move stale
// partials nobody reads).  One more synchronisation per outer iteration (the
// Bellman residual).  All vector work runs in the kernels below and the
// K1/K2/K3 kernels of the single-GPU path on the rank's rows.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "krylov.cuh"

namespace ipi {

constexpr int kShT = 256;

struct ShState {
  double H[(R + 1) * R];
  double cs[R], sn[R], g[R + 1];
  double eff, est_target, rn, hnorm, target;
  int j, it, active, done, brk;
};

struct ShFlags {  // host-mapped mirror read after every step
  int active, j, it, done, brk, pad;
  double rn;
};

struct ShArgs {
  int64_t n;     // local rows
  int64_t ldv;   // basis leading dimension
  double* V;     // (R+1) x ldv local basis
  double* w;
  double* r;
  double* x;        // local iterate
  const double* b;  // g_pi (local)
  const double* invd;
  const double* parts;  // world x cnt gathered partials (rank-major)
  int world;
  double* part_out;  // this rank's cnt partials
  double* blk;       // kPartStride x nblk block partials
  unsigned* ticket;
  ShState* s;
  ShFlags* hf;
  int max_it;
};

// Sum of gathered partials for value k in rank order (rank_ordered_sum).
__device__ __forceinline__ double rank_sum(const double* parts, int world, int cnt, int k) {
  double s = parts[k];
  for (int r = 1; r < world; ++r) s = add_rn(s, parts[(int64_t)r * cnt + k]);
  return s;
}

// Block-reduce acc[0..7] into bs[base + k]; fixed trees.
__device__ __forceinline__ void sh_block8(const double (&acc)[8], int base, int cnt, double* bs,
                                          double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) t[k] = warp_sum(acc[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 8; ++k) red[k * 32 + warp] = t[k];
  __syncthreads();
  if (warp < 8 && base + warp < cnt) {
    const double v = warp_sum(lane < nw ? red[warp * 32 + lane] : 0.0);
    if (lane == 0) bs[base + warp] = v;
  }
}

// Block sums bs[0..cnt) -> the last block to finish adds every block's sums in
// block order (fixed lanes + xor tree) into out[0..cnt).  Returns true in the
// last block (every block has arrived, i.e. finished everything before its
// call), false elsewhere.
__device__ __forceinline__ bool sh_finish(const double* bs, int cnt, double* blk, unsigned* ticket,
                                          double* out) {
  __shared__ bool last;
  __syncthreads();
  const int nblk = gridDim.x;
  if ((int)threadIdx.x < cnt) blk[(int64_t)threadIdx.x * nblk + blockIdx.x] = bs[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (unsigned)nblk - 1;
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = warp; k < cnt; k += nw) {
    double s = 0.0;
    for (int i = lane; i < nblk; i += 32) s = add_rn(s, __ldcg(blk + (int64_t)k * nblk + i));
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// The sweeps below take two consecutive elements per thread and step (16-byte
// loads: ldv is even and every vector starts 16-byte aligned); an odd last
// element is handled by the grid's first thread.  sh_elems(a, f) calls
// f(i, pair) for this thread's elements in a fixed order.
template <class F>
__device__ __forceinline__ void sh_elems(const ShArgs& a, F&& f) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n2 = a.n >> 1;
  for (int64_t p = gtid; p < n2; p += stride) f(2 * p, true);
  if ((a.n & 1) && gtid == 0) f(a.n - 1, false);
}
__device__ __forceinline__ double2 sh_ld2(const double* p, bool pair) {
  return pair ? *reinterpret_cast<const double2*>(p) : make_double2(*p, 0.0);
}
__device__ __forceinline__ void sh_st2(double* p, double2 v, bool pair) {
  if (pair) *reinterpret_cast<double2*>(p) = v;
  else *p = v.x;
}

// Pass 1 of a CGS2 step: (optionally w <- pc(w)), partials <V_l, w> (l <= j), <w, w>.
__global__ void __launch_bounds__(kShT) sh_dots1(ShArgs a, int j, int apply_pc) {
  __shared__ double red[8 * 32], bs[kPartStride];
  if (!a.s->active) return;  // uniform: the previous step ended the cycle
  const int cnt = j + 2;
  for (int l0 = 0; l0 < cnt; l0 += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    sh_elems(a, [&](int64_t i, bool pair) {
      double2 wi = sh_ld2(a.w + i, pair);
      if (l0 == 0 && apply_pc && a.invd) {  // w = pc(A v_j) (inner.py:249), once
        const double2 d = sh_ld2(a.invd + i, pair);
        wi.x = mul_rn(wi.x, d.x);
        wi.y = mul_rn(wi.y, d.y);
        sh_st2(a.w + i, wi, pair);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int l = l0 + u;
        if (l <= j) {
          const double2 v = sh_ld2(a.V + (int64_t)l * a.ldv + i, pair);
          acc[u] = add_rn(add_rn(acc[u], mul_rn(v.x, wi.x)), mul_rn(v.y, wi.y));
        } else if (l == j + 1) {
          acc[u] = add_rn(add_rn(acc[u], mul_rn(wi.x, wi.x)), mul_rn(wi.y, wi.y));
        }
      }
    });
    sh_block8(acc, l0, cnt, bs, red);
  }
  sh_finish(bs, cnt, a.blk, a.ticket, a.part_out);
}

// CGS update: coef = rank sums of the gathered partials (cnt_in values, the
// first j+1 are projections); w <- w - sum_l coef_l V_l; H[:, j] (+)= coef.
// mode 1 then computes partials <V_l, w> (l <= j) and <w, w> (the
// re-orthogonalisation pass); mode 2 only <w, w>.
__global__ void __launch_bounds__(kShT) sh_update(ShArgs a, int j, int cnt_in, int mode) {
  __shared__ double red[8 * 32], bs[kPartStride], coef[kPartStride];
  if (!a.s->active) return;  // uniform: the previous step ended the cycle
  if ((int)threadIdx.x <= j) coef[threadIdx.x] = rank_sum(a.parts, a.world, cnt_in, threadIdx.x);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int l = 0; l <= j; ++l)
      a.s->H[l * R + j] = mode == 1 ? coef[l] : add_rn(a.s->H[l * R + j], coef[l]);
  }
  const int cnt = mode == 1 ? j + 2 : 1;
  for (int l0 = 0; l0 < cnt; l0 += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    sh_elems(a, [&](int64_t i, bool pair) {
      double2 wi = sh_ld2(a.w + i, pair);
      if (l0 == 0) {  // the update, once per element (l ascending, separate roundings)
        for (int l = 0; l <= j; ++l) {
          const double2 v = sh_ld2(a.V + (int64_t)l * a.ldv + i, pair);
          wi.x = sub_rn(wi.x, mul_rn(coef[l], v.x));
          wi.y = sub_rn(wi.y, mul_rn(coef[l], v.y));
        }
        sh_st2(a.w + i, wi, pair);
      }
      if (mode == 1) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = l0 + u;
          if (l <= j) {
            const double2 v = sh_ld2(a.V + (int64_t)l * a.ldv + i, pair);
            acc[u] = add_rn(add_rn(acc[u], mul_rn(v.x, wi.x)), mul_rn(v.y, wi.y));
          } else if (l == j + 1) {
            acc[u] = add_rn(add_rn(acc[u], mul_rn(wi.x, wi.x)), mul_rn(wi.y, wi.y));
          }
        }
      } else {
        acc[0] = add_rn(add_rn(acc[0], mul_rn(wi.x, wi.x)), mul_rn(wi.y, wi.y));
      }
    });
    sh_block8(acc, l0, cnt, bs, red);
  }
  sh_finish(bs, cnt, a.blk, a.ticket, a.part_out);
}

__device__ __forceinline__ void sh_publish(const ShArgs& a, const ShState& s) {
  volatile ShFlags* f = a.hf;
  f->active = s.active;
  f->j = s.j;
  f->it = s.it;
  f->done = s.done;
  f->brk = s.brk;
  f->rn = s.rn;
  // no system fence: the host reads the mirror only after synchronising on an
  // event (or the stream) behind this launch
}

// Givens update and break test (inner.py:255-270) on the completed column j.
// One warp: the column and the rotations are loaded and stored by 32 lanes
// (thread 0 alone paid one dependent global round trip per operand: ~10 us per
// step), the recurrence itself runs in thread 0 on shared memory.
__global__ void sh_givens(ShArgs a, int j) {
  __shared__ double hc[R + 2], cs_s[R], sn_s[R];
  ShState* st = a.s;
  const int t = threadIdx.x;
  if (!st->active) {  // a step enqueued past the cycle's end: nothing to normalise either
    if (t == 0) st->brk = 3;
    return;
  }
  if (t <= j) hc[t] = st->H[t * R + j];
  if (t < j) {
    cs_s[t] = st->cs[t];
    sn_s[t] = st->sn[t];
  }
  __syncwarp();
  if (t == 0) {
    const double hnorm = sqrt(rank_sum(a.parts, a.world, 1, 0));
    hc[j + 1] = hnorm;
    for (int l = 0; l < j; ++l) {
      const double hl = hc[l], hl1 = hc[l + 1];
      hc[l] = add_rn(mul_rn(cs_s[l], hl), mul_rn(sn_s[l], hl1));
      hc[l + 1] = add_rn(mul_rn(-sn_s[l], hl), mul_rn(cs_s[l], hl1));
    }
    const double denom = hypot(hc[j], hc[j + 1]);
    int brk = 0;
    if (denom == 0.0) {
      brk = 1;
    } else {
      const double csj = hc[j] / denom, snj = hc[j + 1] / denom;
      st->cs[j] = csj;
      st->sn[j] = snj;
      hc[j] = denom;
      hc[j + 1] = 0.0;
      const double gj = st->g[j];
      const double gj1 = mul_rn(-snj, gj);
      st->g[j + 1] = gj1;
      st->g[j] = mul_rn(csj, gj);
      if (fabs(gj1) <= st->est_target || hnorm == 0.0) brk = 2;
    }
    st->hnorm = hnorm;
    st->brk = brk;
    st->it += 1;
    st->j = brk == 1 ? j : j + 1;
    st->active = (brk == 0 && st->j < R && st->it < a.max_it) ? 1 : 0;
    sh_publish(a, *st);
  }
  __syncwarp();
  if (t <= j + 1) st->H[t * R + j] = hc[t];
}

// V_{j+1} = w / hnorm (only when the step ran and did not break)
__global__ void __launch_bounds__(kShT) sh_normalize(ShArgs a) {
  const ShState* st = a.s;
  if (st->brk != 0) return;
  double* Vn = a.V + (int64_t)st->j * a.ldv;
  const double h = st->hnorm;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x)
    Vn[i] = a.w[i] / h;
}

// x += V y, y from back substitution (inner.py:272-276, 286-292)
__global__ void __launch_bounds__(kShT) sh_cycle_end(ShArgs a) {
  __shared__ double y[R];
  const ShState* st = a.s;
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
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int l = 0; l < j; ++l) t = add_rn(t, mul_rn(a.V[(int64_t)l * a.ldv + i], y[l]));
    a.x[i] = add_rn(a.x[i], t);
  }
}

// partials of ||r||^2 (and ||b||^2 when first) for the cycle test
__global__ void __launch_bounds__(kShT) sh_rnorm(ShArgs a, int first) {
  __shared__ double red[8 * 32], bs[kPartStride];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    acc[0] = add_rn(acc[0], mul_rn(a.r[i], a.r[i]));
    if (first) acc[1] = add_rn(acc[1], mul_rn(a.b[i], a.b[i]));
  }
  sh_block8(acc, 0, first ? 2 : 1, bs, red);
  sh_finish(bs, first ? 2 : 1, a.blk, a.ticket, a.part_out);
}

// After a cycle (or at the start): rn, eff / est_target (inner.py:189, 277-282),
// the loop test (:235); when continuing, z = pc(r) -> V_0 (unnormalised) and
// the partial of ||z||^2.  Every block derives the scalars from the gathered
// partials and the state; the last block to finish (all blocks have read the
// state by then) stores them.
__global__ void __launch_bounds__(kShT) sh_cycle_start(ShArgs a, int first) {
  __shared__ double red[8 * 32], bs[kPartStride], sc[3];
  __shared__ int sci[2];
  ShState* st = a.s;
  if (threadIdx.x == 0) {
    const int cnt = first ? 2 : 1;
    const double rn = sqrt(rank_sum(a.parts, a.world, cnt, 0));
    double eff = st->eff, est = st->est_target;
    bool done = false;
    if (first) {
      eff = fmax(st->target, 1e-14 * fmax(1.0, sqrt(rank_sum(a.parts, a.world, cnt, 1))));
      est = eff;
    } else {
      const double gj = fabs(st->g[st->j]);
      if (rn > eff && gj <= est) {
        if (gj == 0.0) done = true;
        else est = mul_rn(mul_rn(gj, eff / rn), 0.5);
      }
    }
    const int it = first ? 0 : st->it;
    if (!(rn > eff && it < a.max_it)) done = true;
    sc[0] = rn;
    sc[1] = eff;
    sc[2] = est;
    sci[0] = it;
    sci[1] = done;
  }
  __syncthreads();
  const bool done = sci[1] != 0;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (!done) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const double z = a.invd ? mul_rn(a.r[i], a.invd[i]) : a.r[i];
      a.V[i] = z;
      acc[0] = add_rn(acc[0], mul_rn(z, z));
    }
  }
  sh_block8(acc, 0, 1, bs, red);
  if (sh_finish(bs, 1, a.blk, a.ticket, a.part_out) && threadIdx.x == 0) {
    st->rn = sc[0];
    st->eff = sc[1];
    st->est_target = sc[2];
    st->it = sci[0];
    st->done = done ? 1 : 0;
    st->active = 0;
    sh_publish(a, *st);
  }
}

// V_0 /= beta (beta = ||z||, :236-241); reset the cycle's rotations.
__global__ void __launch_bounds__(kShT) sh_cycle_begin(ShArgs a) {
  ShState* st = a.s;
  if (st->done) return;
  const double beta = sqrt(rank_sum(a.parts, a.world, 1, 0));
  if (beta == 0.0 || !isfinite(beta)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->done = 1;
      sh_publish(a, *st);
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x)
    a.V[i] = a.V[i] / beta;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < (R + 1) * R; ++k) st->H[k] = 0.0;
    for (int k = 0; k < R; ++k) st->cs[k] = st->sn[k] = 0.0;
    for (int k = 0; k <= R; ++k) st->g[k] = 0.0;
    st->g[0] = beta;
    st->j = 0;
    st->brk = 0;
    st->active = 1;
    sh_publish(a, *st);
  }
}

// Richardson (inner.py:216-226): x += scale * pc(r)
__global__ void __launch_bounds__(kShT) sh_richardson_update(ShArgs a, double scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double z = a.invd ? mul_rn(a.r[i], a.invd[i]) : a.r[i];
    a.x[i] = add_rn(a.x[i], mul_rn(scale, z));
  }
}

// the rank's K1 residual (IEEE bits of a non-negative double or NaN) as a double
__global__ void sh_res_to_double(const unsigned long long* bits, double* out) {
  *out = __longlong_as_double((long long)*bits);
}

}  // namespace ipi

using namespace ipi;

namespace {

struct ShWork {
  double *V = nullptr, *w = nullptr, *r = nullptr, *x = nullptr, *xfull = nullptr;
  double *parts = nullptr, *part_out = nullptr, *blk = nullptr;
  unsigned* ticket = nullptr;
  ShState* s = nullptr;
  double* res = nullptr;
  void* base = nullptr;
};

int comm_check(int rc, const char* what) {
  return rc ? fail(IPI_ECUDA, std::string("collective failed: ") + what + ": " + ipi_last_error()) : IPI_OK;
}

}  // namespace

extern "C" {

int ipi_solve_sharded(ipi_mdp* h, const ipi_comm* comm, const ipi_opts* o, double* v_local,
                      int32_t* policy, double* history, int32_t hist_cap, ipi_stats* stats,
                      void* stream) {
  if (!h || !comm || !o || !v_local || !stats) return fail(IPI_EVALIDATION, "null argument");
  if (!comm->allgather || !comm->allgather_blocks) return fail(IPI_EVALIDATION, "incomplete ipi_comm");
  if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world)
    return fail(IPI_EVALIDATION, "bad rank / world");
  if (!(o->tol > 0.0)) return fail(IPI_EVALIDATION, "tolerance must be > 0");
  if (!(o->alpha > 0.0 && o->alpha < 1.0)) return fail(IPI_EVALIDATION, "alpha must lie in (0, 1)");
  if (o->max_outer < 1 || o->max_inner < 1) return fail(IPI_EVALIDATION, "iteration caps must be >= 1");
  if (hist_cap < 1) return fail(IPI_EVALIDATION, "history capacity must be >= 1");
  if (o->pc_type != IPI_PC_NONE && o->pc_type != IPI_PC_JACOBI)
    return fail(IPI_EVALIDATION, "only the none and jacobi preconditioners run on the device");
  if (o->ksp_type != IPI_KSP_GMRES && o->ksp_type != IPI_KSP_RICHARDSON)
    return fail(IPI_EVALIDATION, "the sharded driver runs GMRES and Richardson inner solves "
                                 "(BiCGStab / TFQMR: single GPU only)");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_scratch(h);
  if (rc) return rc;
  const int64_t n = h->n_local, N = h->n_global;
  const int world = comm->world;
  int dev = 0, sms = 148;
  IPI_CUDA_TRY(cudaGetDevice(&dev));
  IPI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static const int nblk_mult = getenv("IPI_SH_NBLK") ? atoi(getenv("IPI_SH_NBLK")) : 4;  // blocks per SM of the vector sweeps: 4 measured best (C2, world 1: 51.7 / 41.1 / 43.9 ms of inner
  // time at 2 / 4 / 6; occupancy, not per-thread loads in flight, is what these sweeps need: a
  // register-resident single-sweep variant of the re-orthogonalisation pass measured 42.8-47.3 ms)
  const int nblk = nblk_mult * sms;
  const auto t_start = std::chrono::steady_clock::now();
  // ---- workspace (stream-ordered) -----------------------------------------
  ShWork W;
  const int64_t ldv = (std::max<int64_t>(n, 1) + 1) & ~(int64_t)1;
  const int64_t doubles = (int64_t)(R + 1) * ldv + 3 * ldv + N + 2 + (int64_t)world * kPartStride +
                          kPartStride + (int64_t)kPartStride * nblk + 16 +
                          (int64_t)(sizeof(ShState) + 7) / 8 + 4;
  IPI_CUDA_TRY(cudaMallocAsync(&W.base, sizeof(double) * doubles, st));
  struct Free {
    void* p;
    cudaStream_t s;
    ~Free() {
      if (p) cudaFreeAsync(p, s);
    }
  } free_guard{W.base, st};
  double* p = static_cast<double*>(W.base);
  W.V = p; p += (int64_t)(R + 1) * ldv;
  W.w = p; p += ldv;
  W.r = p; p += ldv;
  W.x = p; p += ldv;
  W.xfull = p; p += N + 2;
  W.parts = p; p += (int64_t)world * kPartStride;
  W.part_out = p; p += kPartStride;
  W.blk = p; p += (int64_t)kPartStride * nblk;
  W.ticket = reinterpret_cast<unsigned*>(p); p += 16;
  W.res = p; p += 2;
  W.s = reinterpret_cast<ShState*>(p);
  IPI_CUDA_TRY(cudaMemsetAsync(W.ticket, 0, 64, st));
  // mapped host flags, one block per (device, stream)
  static std::mutex flags_mu;
  static std::map<std::pair<int, cudaStream_t>, ShFlags*> flags_of;
  ShFlags* h_flags = nullptr;
  {
    std::lock_guard<std::mutex> lk(flags_mu);
    ShFlags*& slot = flags_of[{dev, st}];
    if (!slot) IPI_CUDA_TRY(cudaHostAlloc(&slot, sizeof(ShFlags), cudaHostAllocMapped));
    h_flags = slot;
  }
  volatile ShFlags* hf = h_flags;
  ShFlags* hf_dev = nullptr;
  IPI_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hf_dev), h_flags, 0));
  cudaEvent_t step_ev[2] = {};
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } ev_guard{step_ev};
  for (int i = 0; i < 2; ++i) IPI_CUDA_TRY(cudaEventCreateWithFlags(&step_ev[i], cudaEventDisableTiming));
  ShArgs a{};
  a.n = n;
  a.ldv = ldv;
  a.V = W.V;
  a.w = W.w;
  a.r = W.r;
  a.x = W.x;
  a.b = h->gpi;
  a.invd = nullptr;
  a.parts = W.parts;
  a.world = world;
  a.part_out = W.part_out;
  a.blk = W.blk;
  a.ticket = W.ticket;
  a.s = W.s;
  a.hf = hf_dev;
  // ---- collectives ------------------------------------------------------
  auto gather_parts = [&](int cnt) -> int {
    return comm_check(comm->allgather(comm->ctx, W.part_out, W.parts, cnt, stream), "allgather");
  };
  auto gather_vec = [&](const double* local) -> int {
    return comm_check(comm->allgather_blocks(comm->ctx, local, W.xfull, stream), "allgather_blocks");
  };
  auto sync = [&]() -> int {
    IPI_CUDA_TRY(cudaStreamSynchronize(st));
    return IPI_OK;
  };
  // ---- outer loop (driver.py:109-209) --------------------------------------
  std::vector<double> hist;
  int64_t inner_total = 0;
  int stall = 0, k = 0, status = IPI_CONVERGED;
  double tg = 0, ta = 0, ti = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto x, auto y) { return std::chrono::duration<double>(y - x).count(); };
  std::vector<double> res_all(world);
  IPI_CUDA_TRY(cudaMemcpyAsync(W.x, v_local, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  while (true) {
    const auto t0 = now();
    if ((rc = gather_vec(W.x))) return rc;
    IPI_CUDA_TRY(cudaMemsetAsync(h->res_bits, 0, sizeof(unsigned long long), st));
    if ((rc = launch_bellman(h, W.xfull, o->mode, h->pi, h->applied, h->gpi, nullptr, h->res_bits, st)))
      return rc;
    sh_res_to_double<<<1, 1, 0, st>>>(h->res_bits, W.part_out);
    if ((rc = gather_parts(1))) return rc;
    IPI_CUDA_TRY(cudaMemcpyAsync(res_all.data(), W.parts, sizeof(double) * world, cudaMemcpyDeviceToHost, st));
    if ((rc = sync())) return rc;
    double res = 0.0;
    for (int q = 0; q < world; ++q) {  // NaN-propagating max (driver.py:136)
      const double x = res_all[q];
      if (x != x || res != res) res = NAN;
      else res = std::max(res, x);
    }
    tg += secs(t0, now());
    hist.push_back(res);
    if (res <= o->tol) { status = IPI_CONVERGED; break; }
    if (k >= o->max_outer) { status = IPI_OUTER_CAP; break; }
    if (k > 0 && res >= hist[k - 1]) {
      if (++stall >= 50) { status = IPI_STALLED; break; }
    } else {
      stall = 0;
    }
    const auto t1 = now();
    if ((rc = gather_policy(h, h->pi, nullptr, h->rp_pi, h->col_pi, h->val_pi, nullptr, nullptr, st)))
      return rc;
    if (o->pc_type == IPI_PC_JACOBI) {
      if (!h->invd) IPI_CUDA_TRY(cudaMalloc(&h->invd, sizeof(double) * std::max<int64_t>(n, 1)));
      if ((rc = jacobi_inv_diag(h->rp_pi, h->col_pi, h->val_pi, n, h->gamma, h->invd, st, h->state0)))
        return rc;
      a.invd = h->invd;
    }
    if (!h->op_pi) {  // the planned K3 operator over this rank's P_pi rows (global columns),
                      // planned on its first contents; later iterations reuse the scratch
      if ((rc = ipi_op_create(h->rp_pi, h->col_pi, h->val_pi, n, N, h->state0, h->gamma, stream, &h->op_pi)))
        return rc;
    }
    if ((rc = sync())) return rc;
    ta += secs(t1, now());
    const auto t2 = now();
    double target;
    int cap;
    if (o->ksp_max_it > 0) {
      target = 0.0;
      cap = o->ksp_max_it;
    } else {
      target = o->alpha * res;
      cap = o->max_inner;
    }
    a.max_it = cap;
    {
      ShState init{};
      init.target = target;
      IPI_CUDA_TRY(cudaMemcpyAsync(W.s, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    }
    // r = b - A x, ||r||, ||b||, eff (inner.py:189)
    if ((rc = gather_vec(W.x))) return rc;
    if ((rc = op_launch(h->op_pi, W.xfull, h->gpi, 2, W.r, st))) return rc;
    sh_rnorm<<<nblk, kShT, 0, st>>>(a, 1);
    IPI_LAUNCH_CHECK();
    if ((rc = gather_parts(2))) return rc;
    int its = 0;
    if (o->ksp_type == IPI_KSP_RICHARDSON) {
      // inner.py:216-226: stop on rn <= eff | it >= cap | !finite
      sh_cycle_start<<<nblk, kShT, 0, st>>>(a, 1);  // rn, eff
      IPI_LAUNCH_CHECK();
      if ((rc = sync())) return rc;
      ShState s_h;
      while (true) {
        IPI_CUDA_TRY(cudaMemcpy(&s_h, W.s, sizeof(ShState), cudaMemcpyDeviceToHost));
        if (s_h.rn <= s_h.eff || its >= cap || !std::isfinite(s_h.rn)) break;
        sh_richardson_update<<<nblk, kShT, 0, st>>>(a, o->richardson_scale);
        ++its;
        if ((rc = gather_vec(W.x))) return rc;
        if ((rc = op_launch(h->op_pi, W.xfull, h->gpi, 2, W.r, st))) return rc;
        sh_rnorm<<<nblk, kShT, 0, st>>>(a, 0);
        if ((rc = gather_parts(1))) return rc;
        // rn only: a cycle_start with the converged eff kept
        sh_cycle_start<<<nblk, kShT, 0, st>>>(a, 0);
        IPI_LAUNCH_CHECK();
        if ((rc = sync())) return rc;
      }
    } else {
      // GMRES(30) with CGS2 (inner.py:229-283)
      sh_cycle_start<<<nblk, kShT, 0, st>>>(a, 1);
      IPI_LAUNCH_CHECK();
      if ((rc = gather_parts(1))) return rc;
      sh_cycle_begin<<<nblk, kShT, 0, st>>>(a);
      IPI_LAUNCH_CHECK();
      if ((rc = sync())) return rc;
      const int* active = &W.s->active;
      while (!hf->done) {
        // Arnoldi steps, one enqueued ahead of the one the host waits for
        int issued = 0, waited = 0;
        auto issue = [&]() -> int {
          const int j = issued;
          int e;
          // w = A V_j on the rank's rows (the Krylov vector assembled first)
          if ((e = gather_vec(W.V + (int64_t)j * ldv))) return e;
          if ((e = op_launch(h->op_pi, W.xfull, nullptr, 1, W.w, st, nullptr, active))) return e;
          sh_dots1<<<nblk, kShT, 0, st>>>(a, j, 1);
          if ((e = gather_parts(j + 2))) return e;
          sh_update<<<nblk, kShT, 0, st>>>(a, j, j + 2, 1);
          if ((e = gather_parts(j + 2))) return e;
          sh_update<<<nblk, kShT, 0, st>>>(a, j, j + 2, 2);
          if ((e = gather_parts(1))) return e;
          sh_givens<<<1, 32, 0, st>>>(a, j);
          sh_normalize<<<nblk, kShT, 0, st>>>(a);
          IPI_LAUNCH_CHECK();
          IPI_CUDA_TRY(cudaEventRecord(step_ev[issued & 1], st));
          ++issued;
          return IPI_OK;
        };
        if ((rc = issue())) return rc;
        while (true) {
          if (issued < R && issued == waited + 1 && (rc = issue())) return rc;
          IPI_CUDA_TRY(cudaEventSynchronize(step_ev[waited & 1]));
          ++waited;
          if (!hf->active) break;       // steps enqueued beyond it skip themselves
          if (waited >= issued) break;  // R steps issued and all done
        }
        its = hf->it;
        if (hf->j == 0) break;  // inner.py:271-272
        sh_cycle_end<<<nblk, kShT, 0, st>>>(a);
        if ((rc = gather_vec(W.x))) return rc;
        if ((rc = op_launch(h->op_pi, W.xfull, h->gpi, 2, W.r, st))) return rc;
        sh_rnorm<<<nblk, kShT, 0, st>>>(a, 0);
        if ((rc = gather_parts(1))) return rc;
        sh_cycle_start<<<nblk, kShT, 0, st>>>(a, 0);
        if ((rc = gather_parts(1))) return rc;
        sh_cycle_begin<<<nblk, kShT, 0, st>>>(a);
        IPI_LAUNCH_CHECK();
        if ((rc = sync())) return rc;
      }
      its = hf->it;
    }
    inner_total += its;
    ti += secs(t2, now());
    ++k;
  }
  IPI_CUDA_TRY(cudaMemcpyAsync(v_local, W.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (policy) IPI_CUDA_TRY(cudaMemcpyAsync(policy, h->pi, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  IPI_CUDA_TRY(cudaStreamSynchronize(st));
  const int nh = std::min<int>((int)hist.size(), hist_cap);
  if (history) std::memcpy(history, hist.data(), sizeof(double) * nh);
  stats->status = status;
  stats->outer_iterations = k;
  stats->inner_iterations_total = inner_total;
  stats->wall_time = secs(t_start, now());
  stats->time_greedy = tg;
  stats->time_assembly = ta;
  stats->time_inner = ti;
  stats->basis_reads_total = 0;
  return IPI_OK;
}

}  // extern "C"
