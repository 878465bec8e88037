// spmv.cu — K3 standalone SpMV family (sparse.py:189-215, 294-295).
//
// G lanes per CSR row (G chosen from the mean row length), 32/G rows per
// warp step, grid-stride over row groups; 4 loads in flight per lane.
// Epilogues: 0: y = A x;  1: y = x - gamma*(A x) (PolicyOperator.apply, exact
// two-step rounding);  2: y = b - (x - gamma*(A x)) (inner.py:220/232/276);
// 3: y = b + gamma*(A x) (breakdown sweep g_pi + gamma*P_pi v, driver.py:190-193);
// 4/5: like 1/2 with a precomputed partial row sum added first,
//      y = x - gamma*(yp + A x) — the remote-column half of a split apply
//      (parallel.py: local-column SpMV overlapped with the V all-gather).
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
                                                    const double* __restrict__ x_diag,
                                                    const double* __restrict__ yp) {
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
      // long rows (G = 32: C4's ~570-entry P_pi rows): 8 loads in flight per lane
      constexpr int U = G == 32 ? 8 : 4;
      for (int64_t p = p0 + gl; p < p1; p += U * G) {
        double vv[U];
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t q = p + (int64_t)u * G;
          if (q < p1) {
            vv[u] = ld_stream(val + q, pol);
            cc[u] = ld_stream(col + q, pol);
          } else {
            vv[u] = 0.0;
            cc[u] = -1;
          }
        }
        double xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) xx[u] = cc[u] >= 0 ? __ldg(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (cc[u] >= 0) acc = add_rn(acc, mul_rn(vv[u], xx[u]));
      }
    }
    acc = group_sum<G>(acc);
    if (r < rows && gl == 0) {
      if (EPI == 4 || EPI == 5) acc = add_rn(__ldg(yp + r), acc);
      if (EPI == 0) {
        y[r] = acc;
      } else if (EPI == 3) {
        y[r] = add_rn(__ldg(b + r), mul_rn(gamma, acc));
      } else {
        const double ax = sub_rn(__ldg(x_diag + r), mul_rn(gamma, acc));
        y[r] = (EPI == 1 || EPI == 4) ? ax : sub_rn(__ldg(b + r), ax);
      }
    }
  }
}

template <int G>
static void launch_spmv_g(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                          const double* x, const double* b, double gamma, int epi, double* y,
                          int blocks, const double* xd, const double* yp, cudaStream_t st) {
  switch (epi) {
    case 0: spmv_kernel<G, 0><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd, yp); break;
    case 1: spmv_kernel<G, 1><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd, yp); break;
    case 2: spmv_kernel<G, 2><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd, yp); break;
    case 3: spmv_kernel<G, 3><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd, yp); break;
    case 4: spmv_kernel<G, 4><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd, yp); break;
    default: spmv_kernel<G, 5><<<blocks, 256, 0, st>>>(rp, col, val, rows, x, b, gamma, y, xd, yp); break;
  }
}

int launch_spmv(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                const double* x, const double* b, double gamma, int epi, double* y, int lanes,
                cudaStream_t st, int64_t diag_offset, const double* y_partial) {
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
    case 1: launch_spmv_g<1>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, y_partial, st); break;
    case 2: launch_spmv_g<2>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, y_partial, st); break;
    case 4: launch_spmv_g<4>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, y_partial, st); break;
    case 8: launch_spmv_g<8>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, y_partial, st); break;
    case 16: launch_spmv_g<16>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, y_partial, st); break;
    default: launch_spmv_g<32>(rp, col, val, rows, x, b, gamma, epi, y, (int)blocks, xd, y_partial, st); break;
  }
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

// ---------------------------------------------------------------------------
// split of a row block's CSR into local columns [lo, hi) (re-indexed to col-lo)
// and remote columns: pass 1 (cols == nullptr) writes per-row counts to
// rp_loc[r+1] / rp_rem[r+1]; the caller scans; pass 2 scatters in row order
// (each part keeps the row's column order).
// ---------------------------------------------------------------------------
__global__ void split_rows_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, int64_t rows, int32_t lo, int32_t hi,
                                  int64_t* rp_loc, int32_t* col_loc, double* val_loc, int64_t* rp_rem,
                                  int32_t* col_rem, double* val_rem, int fill) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = wg; r < rows; r += nw) {
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    int64_t nl = 0, nr = 0;  // entries written so far (fill) / counted
    const int64_t ol = fill ? rp_loc[r] : 0, orr = fill ? rp_rem[r] : 0;
    for (int64_t base = p0; base < p1; base += 32) {
      const int64_t p = base + lane;
      const bool in = p < p1;
      const int c = in ? col[p] : 0;
      const bool loc = in && c >= lo && c < hi;
      const unsigned ml = __ballot_sync(kFull, loc), mr = __ballot_sync(kFull, in && !loc);
      if (fill && in) {
        const unsigned below = (1u << lane) - 1u;
        if (loc) {
          const int64_t q = ol + nl + __popc(ml & below);
          col_loc[q] = c - lo;
          val_loc[q] = val[p];
        } else {
          const int64_t q = orr + nr + __popc(mr & below);
          col_rem[q] = c;
          val_rem[q] = val[p];
        }
      }
      nl += __popc(ml);
      nr += __popc(mr);
    }
    if (!fill && lane == 0) {
      rp_loc[r + 1] = nl;
      rp_rem[r + 1] = nr;
    }
  }
}

int split_local_remote(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                       int32_t lo, int32_t hi, int64_t* rp_loc, int32_t* col_loc, double* val_loc,
                       int64_t* rp_rem, int32_t* col_rem, double* val_rem, cudaStream_t st) {
  if (rows <= 0) return IPI_OK;
  const int fill = col_loc != nullptr;
  int64_t blocks = (rows + 7) / 8;
  if (blocks > 148 * 32) blocks = 148 * 32;
  split_rows_kernel<<<(int)blocks, 256, 0, st>>>(rp, col, val, rows, lo, hi, rp_loc, col_loc, val_loc,
                                                 rp_rem, col_rem, val_rem, fill);
  IPI_LAUNCH_CHECK();
  return IPI_OK;
}

}  // namespace ipi
