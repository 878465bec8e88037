// shard_ops.cu — vector kernels of the row-sharded inner solve (parallel.py).
//
// In a sharded GMRES step every MGS pass is one cross-rank reduction
// (inner.py:251-253: h_lj = <V_l, w>; w -= h_lj V_l).  The host driver keeps
// all scalars on the device: each pass is ONE kernel here plus one all-gather
// of the R per-rank partials (NCCL), and the host synchronises once per
// Arnoldi step (to read the Hessenberg column for the Givens update).
//
//   ipi_dot_partial:  out = <a, b> over this rank's rows;
//   ipi_mgs_pass:     h = sum_r partials[r] in rank order (rank_ordered_sum,
//                     parallel.py), w -= h v, out = <v_next, w> (or <w, w>).
//
// Reductions are deterministic: fixed grid, per-thread grid-stride sums,
// fixed block trees, and the last block to finish (ticket) adds the block
// partials in block order.  Same separate mul/add roundings as numpy.
#include <map>
#include <mutex>

#include "handle.cuh"

namespace ipi {

constexpr int kShardThreads = 256;

struct ShardScratch {
  double* blk = nullptr;      // block partials
  unsigned* ticket = nullptr;  // last-block counter (self-resetting)
  int blocks = 0;
};

// One scratch (block partials + last-block ticket) per (device, stream): the
// ticket protocol is only safe for launches that run one after another, which
// stream order guarantees; two streams get two scratches.
static std::mutex g_shard_mu;
static std::map<std::pair<int, cudaStream_t>, ShardScratch> g_shard;

static int shard_scratch(cudaStream_t st, ShardScratch** out) {
  int dev = 0;
  IPI_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_shard_mu);
  ShardScratch& s = g_shard[{dev, st}];
  if (!s.blk) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    s.blocks = 2 * sms;
    IPI_CUDA_TRY(cudaMalloc(&s.blk, sizeof(double) * s.blocks));
    IPI_CUDA_TRY(cudaMalloc(&s.ticket, sizeof(unsigned)));
    IPI_CUDA_TRY(cudaMemset(s.ticket, 0, sizeof(unsigned)));
  }
  *out = &s;
  return IPI_OK;
}

// Block-sum `v`, then the last block to arrive sums the block partials in
// block order into *out and re-arms the ticket.
__device__ __forceinline__ void finish_reduction(double v, double* blk, unsigned* ticket,
                                                 double* out) {
  __shared__ double red[32];
  __shared__ bool last;
  const double t = block_sum(v, red);
  if (threadIdx.x == 0) {
    blk[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < 32) {
    __threadfence();
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) s = add_rn(s, __ldcg(blk + i));
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      *out = s;
      *ticket = 0u;
    }
  }
}

__global__ void __launch_bounds__(kShardThreads) dot_partial_kernel(const double* __restrict__ a,
                                                                    const double* __restrict__ b,
                                                                    int64_t n, double* blk,
                                                                    unsigned* ticket, double* out) {
  double q = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    q = add_rn(q, mul_rn(a[i], b[i]));
  finish_reduction(q, blk, ticket, out);
}

__global__ void __launch_bounds__(kShardThreads) mgs_pass_kernel(
    const double* __restrict__ partials, int R, double* h_out, double* __restrict__ w,
    const double* __restrict__ v, const double* __restrict__ v_next, int64_t n, double* blk,
    unsigned* ticket, double* out) {
  // h = parts[0] + parts[1] + ... in rank order (parallel.rank_ordered_sum)
  double h = partials[0];
  for (int r = 1; r < R; ++r) h = add_rn(h, partials[r]);
  if (blockIdx.x == 0 && threadIdx.x == 0) *h_out = h;
  double q = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = sub_rn(w[i], mul_rn(h, v[i]));
    w[i] = wi;
    q = v_next ? add_rn(q, mul_rn(v_next[i], wi)) : add_rn(q, mul_rn(wi, wi));
  }
  finish_reduction(q, blk, ticket, out);
}

}  // namespace ipi

using namespace ipi;

extern "C" {

int ipi_dot_partial(const double* a, const double* b, int64_t n, double* out, void* stream) {
  if (!out || (n > 0 && (!a || !b))) return fail(IPI_EVALIDATION, "null argument");
  if (n < 0) return fail(IPI_EDIMENSION, "negative length");
  ShardScratch* s = nullptr;
  int rc = shard_scratch((cudaStream_t)stream, &s);
  if (rc) return rc;
  dot_partial_kernel<<<s->blocks, kShardThreads, 0, (cudaStream_t)stream>>>(a, b, n, s->blk,
                                                                            s->ticket, out);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

int ipi_mgs_pass(const double* partials, int32_t R, double* h_out, double* w, const double* v,
                 const double* v_next, int64_t n, double* out_partial, void* stream) {
  if (!partials || !h_out || !out_partial || (n > 0 && (!w || !v)))
    return fail(IPI_EVALIDATION, "null argument");
  if (R < 1) return fail(IPI_EVALIDATION, "rank count must be >= 1");
  if (n < 0) return fail(IPI_EDIMENSION, "negative length");
  ShardScratch* s = nullptr;
  int rc = shard_scratch((cudaStream_t)stream, &s);
  if (rc) return rc;
  mgs_pass_kernel<<<s->blocks, kShardThreads, 0, (cudaStream_t)stream>>>(
      partials, R, h_out, w, v, v_next, n, s->blk, s->ticket, out_partial);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // extern "C"
