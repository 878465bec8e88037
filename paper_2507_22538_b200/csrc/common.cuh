// common.cuh — shared device helpers for the sm_100a iPI kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/ipi_b200.h"

namespace ipi {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, returned codes)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// Raise (never lower) a kernel's dynamic shared-memory limit.  The attribute is
// per function and process-wide, so a later plan with a smaller footprint (a
// second instance, an m = 1 operator view) must not break the launches of an
// earlier plan that needs more.
cudaError_t raise_smem_limit(const void* fn, int smem);
template <class F>
inline cudaError_t raise_smem_limit(F* fn, int smem) {
  return raise_smem_limit(reinterpret_cast<const void*>(fn), smem);
}

#define IPI_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      return ::ipi::fail(IPI_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    }                                                                             \
  } while (0)

#define IPI_LAUNCH_CHECK()                                                        \
  do {                                                                            \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess) {                                                      \
      return ::ipi::fail(IPI_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    }                                                                             \
  } while (0)

// ---------------------------------------------------------------------------
// loads.  CSR streams are read once per pass: bypass L1 (keep it for the
// gathered V) and mark them evict-first in L2 so V stays L2-resident.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Coherent (non-.nc) load with an L2 eviction hint, for data written earlier in
// the same kernel (Krylov basis, w).  Volatile with a memory clobber: a plain
// asm without one is a pure function of its operands to the compiler, which
// may then hoist it above the barrier or the stores that produce the data (it
// did, in a 384-thread K4 build: GMRES diverged until this was added; the
// committed 1024-thread kernels measured the same before and after).
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}

__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ long long ld_stream(const long long* p, uint64_t pol) {
  long long v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;"
               : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ld_stream_i64(const int64_t* p, uint64_t pol) {
  return (int64_t)ld_stream(reinterpret_cast<const long long*>(p), pol);
}

__device__ __forceinline__ double2 ld_stream_v2(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ld_stream_v2(const int* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}

// cp.async (Ampere-style async copies into shared memory): the per-warp
// streaming rings of K1 (bellman.cu) and K3 (spmv_ring.cu).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes,
                                           uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst),
               "l"(src), "r"(src_bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Stage the window x[lo, hi) (clipped to [0, n)) into shared memory as ONE
// cp.async commit group: 16-byte chunks, every thread's copies in flight at
// once, the start rounded down to an even index so chunks are aligned (the
// buffer needs 2 doubles of slack).  The caller waits for the group and
// barriers before the first read; x must be 16-byte aligned.
__device__ __forceinline__ void window_issue_async(const double* x, int64_t lo, int64_t hi, int64_t n,
                                                   unsigned char* win, int& w_lo, uint32_t& w_len) {
  lo = lo < 0 ? 0 : lo;
  hi = hi > n ? n : hi;
  lo &= ~(int64_t)1;
  w_lo = (int)lo;
  w_len = hi > lo ? (uint32_t)(hi - lo) : 0u;
  uint64_t keep;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  const uint32_t win_s = (uint32_t)__cvta_generic_to_shared(win);
  const uint32_t nch = (w_len + 1) >> 1;
  for (uint32_t c = threadIdx.x; c < nch; c += blockDim.x)
    cp_async16(win_s + 16 * c, x + lo + 2 * c, 2 * c + 1 < w_len ? 16u : 8u, keep);
  cp_async_commit();
}

// Stage x[lo, lo+len) into shared memory with 8-byte cp.async (every copy in
// flight at once; only 8-byte alignment needed), then wait and barrier.  A
// scalar load/store loop here waits one L2 round trip per few elements and
// stalled the start of every CTA.
__device__ __forceinline__ void window_load8(double* win, const double* x, int64_t lo, int64_t len) {
  const uint32_t ws = (uint32_t)__cvta_generic_to_shared(win);
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) cp_async8(ws + (uint32_t)(8 * i), x + lo + i);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
}

// mbarrier + bulk-copy (TMA engine, 1-D) helpers: one thread arms a barrier
// with the expected bytes and issues the copy; consumers wait on the phase.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
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
// global -> shared bulk copy completing on `bar` (16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
// order this thread's generic-proxy shared accesses before later async-proxy
// (bulk copy) writes to the same shared memory
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Bulk L2 prefetch of a contiguous byte range (16-byte aligned, multiple of 16).
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-stream-serialization attribute may start while its predecessor
// in the stream is still running; griddep_wait() blocks until the predecessor
// has completed and its writes are visible (a no-op for a normal launch), and
// griddep_launch_dependents() lets the successor's CTAs be scheduled as soon
// as every CTA of this grid has called it (or exited).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Register batch of P value pairs + column pairs (uniform-row fast paths).
template <int P>
struct Batch {
  double2 v[P];
  int2 c[P];
};

// Exact two-step rounding as numpy does it (no FMA contraction):
// prod = a*b rounded, then sum rounded.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// ---------------------------------------------------------------------------
// warp / group reductions (fixed xor trees -> deterministic)
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) v = add_rn(v, __shfl_xor_sync(kFull, v, off));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) { return group_sum<32>(v); }

// NaN-propagating max for the Bellman residual: the reference's
// np.max(np.abs(v - applied)) (driver.py:136) returns NaN when any entry is
// NaN, so a diverged iterate can never read as converged.  fmax would drop it.
// Non-negative doubles and a positive NaN order correctly as unsigned IEEE
// bits (NaN > +inf), so the integer atomicMax that combines CTAs keeps it.
__device__ __forceinline__ double res_max(double a, double b) {
  return a != a ? a : (b != b ? fabs(b) : fmax(a, b));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = res_max(v, __shfl_xor_sync(kFull, v, off));
  return v;
}

// Argmin/argmax merge with first-index tie break (bellman.py:59-60):
// prefer strictly better q, on equal q the smaller action.
__device__ __forceinline__ bool better(double q, int a, double bq, int ba, bool maximize) {
  if (maximize) return q > bq || (q == bq && a < ba);
  return q < bq || (q == bq && a < ba);
}

// Block reduction of one double per thread: warp trees, then warp 0 reduces
// the per-warp values with the same fixed xor tree (deterministic).  Result
// valid in warp 0 (thread 0 is the one callers use).
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {  // the per-warp values through the same fixed xor tree
    t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace ipi
