// spmv.cu — K3 standalone SpMV family (sparse.py:189-215, 294-295).
//
// G lanes per CSR row (G chosen from the mean row length), 32/G rows per
// warp step, grid-stride over row groups; 4 loads in flight per lane.
// Epilogues: 0: y = A x;  1: y = x - gamma*(A x) (PolicyOperator.apply, exact
// two-step rounding);  2: y = b - (x - gamma*(A x)) (inner.py:220/232/276);
// 3: y = b + gamma*(A x) (breakdown sweep g_pi + gamma*P_pi v, driver.py:190-193).
// Used by the Python API mirror (spmv / PolicyOperator.apply) and tests; the
// inner solver has its own fused copy of this loop inside the persistent
// kernel (krylov.cu).
#include "handle.cuh"

namespace ipi {

template <int G, int EPI>
__global__ void __launch_bounds__(256) spmv_kernel(const int64_t* __restrict__ rp,
                                                    const int32_t* __restrict__ col,
                                                    const double* __restrict__ val, int64_t rows,
                                                    const double* __restrict__ x,
                                                    const double* __restrict__ b, double gamma,
                                                    double* __restrict__ y,
                                                    const double* __restrict__ x_diag) {
  constexpr int GPW = 32 / G;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int64_t warp_global = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp_global * GPW; base < rows; base += nwarps_total * GPW) {
    const int64_t r = base + grp;
    double acc = 0.0;
    if (r < rows) {
      const int64_t p0 = __ldg(rp + r), p1 = __ldg(rp + r + 1);
      for (int64_t p = p0 + gl; p < p1; p += 4 * G) {
        double vv[4];
        int cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t q = p + (int64_t)u * G;
          if (q < p1) {
            vv[u] = ld_stream(val + q, pol);
            cc[u] = ld_stream(col + q, pol);
          } else {
            vv[u] = 0.0;
            cc[u] = -1;
          }
        }
        double xx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xx[u] = cc[u] >= 0 ? __ldg(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (cc[u] >= 0) acc = add_rn(acc, mul_rn(vv[u], xx[u]));
      }
    }
    acc = group_sum<G>(acc);
    if (r < rows && gl == 0) {
      if (EPI == 0) {
        y[r] = acc;
      } else if (EPI == 3) {
        y[r] = add_rn(__ldg(b + r), mul_rn(gamma, acc));
      } else {
        const double ax = sub_rn(__ldg(x_diag + r), mul_rn(gamma, acc));
        y[r] = EPI == 1 ? ax : sub_rn(__ldg(b + r), ax);
      }
    }
  }
}

template <int G>
static void launch_spmv_g(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                          const double* x, const double* b, double gamma, int epi, double* y,
                          int blocks, const double* xd, cudaStream_t st) {
  if (epi == 0)
    spmv_kernel<G, 0><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd);
  else if (epi == 1)
    spmv_kernel<G, 1><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd);
  else if (epi == 2)
    spmv_kernel<G, 2><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd);
  else
    spmv_kernel<G, 3><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd);
}

int launch_spmv(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                const double* x, const double* b, double gamma, int epi, double* y, int lanes,
                cudaStream_t st, int64_t diag_offset) {
  if (rows <= 0) return IPI_OK;
  const double* xd = x + diag_offset;  // identity term of row r reads x[diag_offset + r]
  const int GPW = 32 / lanes;
  int64_t warps = (rows + GPW - 1) / GPW;
  int64_t blocks = (warps + 7) / 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (blocks > (int64_t)sms * 64) blocks = (int64_t)sms * 64;
  if (blocks < 1) blocks = 1;
  switch (lanes) {
    case 1: launch_spmv_g<1>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, st); break;
    case 2: launch_spmv_g<2>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, st); break;
    case 4: launch_spmv_g<4>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, st); break;
    case 8: launch_spmv_g<8>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, st); break;
    case 16: launch_spmv_g<16>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, st); break;
    default: launch_spmv_g<32>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, st); break;
  }
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
