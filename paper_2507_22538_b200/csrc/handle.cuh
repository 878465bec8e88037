// handle.cuh — the ipi_mdp handle and cross-file launcher declarations.
#pragma once

#include "common.cuh"

struct ipi_mdp {
  // borrowed instance arrays (device)
  const int64_t* rp = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
  const double* cost = nullptr;
  int64_t n_local = 0, n_global = 0, state0 = 0;
  int32_t m = 0;
  double gamma = 0.0;
  int32_t mode = IPI_MODE_MIN;

  ipi_plan plan{};
  int num_sms = 0;
  int device = 0;
  int64_t* k1_bounds = nullptr;  // k1_blocks + 1 local state boundaries (device)

  // owned scratch (device), allocated on first use
  int32_t* pi = nullptr;
  double* applied = nullptr;
  double* gpi = nullptr;
  int32_t* lenpi = nullptr;
  unsigned long long* res_bits = nullptr;
  int64_t* rp_pi = nullptr;
  int32_t* col_pi = nullptr;
  double* val_pi = nullptr;
  int64_t cap_pi = 0;
  double* xbuf = nullptr;
  int64_t* scan_tmp = nullptr;
  double* kry = nullptr;        // per-handle Krylov workspace (ipi_solve)
  ipi_op* op_pi = nullptr;      // planned K3 operator over the P_pi scratch (stepped GMRES)
  double* invd = nullptr;       // Jacobi inverse diagonal (ipi_solve with pc = jacobi)
  int64_t kry_len = 0;
  int64_t scan_tmp_len = 0;
  ipi_inner_report* d_report = nullptr;
  void* host_pinned = nullptr;  // small pinned staging area

  // K1 flat-row cp.async ring (variant 4): window bytes in front of the rings
  int ring_win_bytes = 0;
  int uring_lookahead = 1;  // variant 6: V gathers issued this many steps ahead
  double* vbuf = nullptr;   // 16-byte-aligned copy of a misaligned V (cp.async window)
  int k1_win_async = 1;     // variant 6: cp.async V window (IPI_K1_WIN_ASYNC=0: scalar loop)
  int k1_interleave = 1;    // variant 6: interleaved state order (IPI_K1_INTERLEAVE=0: contiguous)
  int k1_rotate = 1;        // variant 6: rotated per-CTA start (IPI_K1_ROTATE=0: none)
  unsigned long long* k1_trace = nullptr;  // diagnostics (ipi_mdp_k1_trace)
};

// A planned policy operator (K3): borrowed P_pi rows + the kernel shape.
struct ipi_op {
  const int64_t* rp = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
  int64_t n_local = 0, n_global = 0, state0 = 0, nnz = 0;
  double gamma = 0.0;
  int variant = IPI_K3_GENERIC;
  int K = 0;          // uniform row length (0 = variable)
  int lanes = 1;      // generic variant: lanes per row
  int halo = -1;      // x window half-width (-1 = none)
  int win_bytes = 0;  // window bytes in front of the rings
  int blocks = 0, warps = 0, stages = 0, smem = 0;
  int pf = 0;         // uniform ring: L2 prefetch distance (steps)
  int interleave = 0; // uniform ring: warps interleave 4-row steps (one stream per CTA)
  unsigned long long* trace = nullptr;  // diagnostics (ipi_op_trace)
};

namespace ipi {

constexpr int kK1Threads = 512;
constexpr int kInnerThreads = 1024;
constexpr int kGmresRestart = 30;  // inner.py:40

int pick_lanes_per_row(double mean_len);
bool uniform_shape(int K, int* G, int* P);

// Dispatch a uniform-row (G, P) shape chosen by uniform_shape() to a template
// instance: P = 1 with G in {1..32}, or (G, P) = (32, 2).
#define IPI_DISPATCH_UNIFORM(G_, P_, FN)                 \
  do {                                                   \
    if ((P_) == 2) {                                     \
      switch (G_) {                                      \
        case 1: FN(1, 2); break;                         \
        case 2: FN(2, 2); break;                         \
        case 4: FN(4, 2); break;                         \
        case 8: FN(8, 2); break;                         \
        case 16: FN(16, 2); break;                       \
        default: FN(32, 2); break;                       \
      }                                                  \
    } else {                                             \
      switch (G_) {                                      \
        case 1: FN(1, 1); break;                         \
        case 2: FN(2, 1); break;                         \
        case 4: FN(4, 1); break;                         \
        case 8: FN(8, 1); break;                         \
        case 16: FN(16, 1); break;                       \
        default: FN(32, 1); break;                       \
      }                                                  \
    }                                                    \
  } while (0)

// bellman.cu
int launch_bellman(ipi_mdp* h, const double* v_full, int32_t mode, int32_t* policy,
                   double* applied, double* g_pi, int32_t* len_pi,
                   unsigned long long* res_bits, cudaStream_t st);

// bellman.cu: flat-row cp.async ring (variant 4)
int flat_ring_smem(int K, int stages, int warps, int m, int window_bytes);
bool k1_ring_prepare(int K, int S, int NW, bool win, int smem);
int uniform_ring_smem(int K, int stages, int warps, int window_bytes);
bool k1_uring_prepare(int K, int NW, int S, int D, bool win, int smem);

// policy.cu
int gather_policy(ipi_mdp* h, const int32_t* policy, const int32_t* len_pi, int64_t* rp_pi,
                  int32_t* col_pi, double* val_pi, double* g_pi, int64_t* nnz_out,
                  cudaStream_t st);
int policy_nnz(ipi_mdp* h, const int32_t* policy, int64_t* nnz_out, cudaStream_t st);

// spmv.cu
int launch_spmv(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                const double* x, const double* b, double gamma, int epi, double* y,
                int lanes, cudaStream_t st, int64_t diag_offset = 0,
                const double* y_partial = nullptr);
int split_local_remote(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                       int32_t lo, int32_t hi, int64_t* rp_loc, int32_t* col_loc, double* val_loc,
                       int64_t* rp_rem, int32_t* col_rem, double* val_rem, cudaStream_t st);

// spmv_ring.cu: K3 ring kernels for a planned operator
int k3_uring_smem(int K, int stages, int warps, int window_bytes);
int k3_flat_smem(int K, int stages, int warps, int window_bytes);
bool k3_shape_prepare(int variant, int K, int NW, int S, bool win, int smem);
int op_launch(const ipi_op* op, const double* x_full, const double* b, int epi, double* y,
              cudaStream_t st, const double* y_partial = nullptr, const int* active = nullptr,
              int pdl = 0);

// krylov.cu
int inner_solve(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                double gamma, const double* b, double* x, double target, int32_t max_it,
                int32_t kind, double scale, int lanes, int halo, int uniform_K,
                ipi_inner_report* d_report, cudaStream_t st, double* workspace = nullptr,
                int64_t workspace_doubles = 0, const double* inv_diag = nullptr,
                double pi_bytes = 0.0,   // bytes of P_pi (L2-residency choice; <= 0: read nnz)
                int ortho = IPI_ORTHO_AUTO,
                const ipi_op* op = nullptr,   // planned K3 operator of P_pi: stepped GMRES
                int contig = 0,               // P_pi rows have consecutive columns
                const double* tv = nullptr);  // b + gamma P_pi x0 when the caller already has it
                                              // (K1's TV in the outer loop): r0 = tv - x0
// krylov_step.cu
bool stepped_gmres_fits(int64_t n, int sms);
int64_t stepped_gmres_workspace(int64_t n, int blocks);
int stepped_gmres(const ipi_op* op, int64_t n, const double* b, double* x, double target,
                  int32_t max_it, const double* inv_diag, ipi_inner_report* d_report,
                  double* ws, int64_t ws_doubles, cudaStream_t st, const double* tv = nullptr);
// Jacobi: inv_diag[s] = 1 / (1 - gamma * P_pi[s, s])  (inner.py:115-118)
int jacobi_inv_diag(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                    double gamma, double* inv_diag, cudaStream_t st, int64_t state0 = 0);
// capi.cu: the handle's per-solve scratch (policy, P_pi, Krylov arena), allocated once
int ensure_scratch(ipi_mdp* h);
// doubles of Krylov workspace inner_solve needs for an n-row system
inline int64_t krylov_workspace_doubles(int64_t n) {
  return (int64_t)(kGmresRestart + 1) * n + 2 * n + 2 * 32 * 1024 + 64;
}

// diagnostics: record K4 phase timestamps (enable = 1) / copy them out and stop (0)
int k4_trace(int enable, unsigned long long* out, int cap);
int ring_apply_test(const int32_t* col, const double* val, int64_t n, double gamma, const double* x,
                    double* y, int reps, float* ms, cudaStream_t st);

// device scratch arena for the standalone inner solver (per device and
// stream, grown stream-ordered on demand)
double* krylov_workspace(int64_t doubles_needed, cudaStream_t st);

}  // namespace ipi
