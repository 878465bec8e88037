/*
 * ipi_b200.h — C ABI of the B200-native iPI hot path (libipi_b200.so).
 *
 * Drop-in boundary for the reference's Python API (mdpsolve / mdpsolve_frontend,
 * /root/reference/pkg).  The reference has no FFI: its boundary is a Python
 * API whose numeric core is numpy.  Every entry point below replaces one
 * reference function (cited file:line, relative to /root/reference/pkg/src/mdpsolve)
 * and is bound from Python with ctypes (paper_2507_22538_b200/_lib.py);
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers borrowed from the caller (torch
 *    tensors); the caller owns them and keeps them alive for the call (for
 *    ipi_mdp_* handles: for the handle's lifetime).
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered.
 *    Calls that return host scalars synchronise that stream.
 *  - Layout (model.py:112-131): row-stacked (n*m) x n CSR, row s*m+a;
 *    row_ptr int64, col int32, values fp64; stage cost fp64 (n, m) row-major.
 *  - Return codes: IPI_OK, or an error whose message ipi_last_error() returns
 *    (thread-local).  Python maps 1 -> ValidationError (model.py:24),
 *    2 -> DimensionError (sparse.py:22), 4 -> ResourceLimitError (sparse.py:26),
 *    3 -> RuntimeError.
 *  - A handle is used by one host thread at a time (SPEC: one solve owns its workers).
 */
#ifndef IPI_B200_H
#define IPI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IPI_OK 0
#define IPI_EVALIDATION 1
#define IPI_EDIMENSION 2
#define IPI_ECUDA 3
#define IPI_ERESOURCE 4

#define IPI_MODE_MIN 0
#define IPI_MODE_MAX 1

/* inner solver kinds (inner.py:48-54) */
#define IPI_KSP_RICHARDSON 0
#define IPI_KSP_GMRES 1
#define IPI_KSP_BICGSTAB 2
#define IPI_KSP_TFQMR 3

/* preconditioners on the device path (inner.py:65-84, 113-118) */
#define IPI_PC_NONE 0
#define IPI_PC_JACOBI 1

/* GMRES Arnoldi orthogonalisation.  The reference uses modified Gram-Schmidt
 * (inner.py:251-253): j+2 dependent reductions per step, one pass over the
 * basis.  CGS2 is classical Gram-Schmidt with one re-orthogonalisation when
 * the DGKS test asks for it (PETSc's KSPGMRESClassicalGramSchmidtOrthogonalization
 * with refine_ifneeded, the library madupite runs on): 2 reductions per step
 * but 2-4 passes over the basis.  AUTO picks MGS where a pass over the basis
 * costs more than a grid reduction (large systems) and CGS2 where the
 * reductions dominate (small systems). */
#define IPI_ORTHO_AUTO 0 /* default */
#define IPI_ORTHO_MGS 1
#define IPI_ORTHO_CGS2 2

/* outer status (driver.py:41-44) */
#define IPI_CONVERGED 0
#define IPI_OUTER_CAP 1
#define IPI_STALLED 2

typedef struct ipi_mdp ipi_mdp;
typedef struct ipi_op ipi_op;

/* K3 kernel variants of a planned policy operator (ipi_op_create) */
#define IPI_K3_GENERIC 0 /* G lanes per row through the row pointers (spmv.cu)       */
#define IPI_K3_URING 1   /* uniform rows 9..129 (K % 4 == 0): cp.async ring, 4 rows/step */
#define IPI_K3_FLAT 2    /* uniform rows K in {2, 4}: cp.async ring, lane = row        */

/* Inner-solve report (inner.py:87-95 InnerSolveReport). */
typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t breakdown;
  int32_t basis_reads; /* GMRES: basis-vector passes of the orthogonalisation (sum of j+1 over
                          steps, MGS), for the roofline byte count; 0 where not counted */
  double final_linear_residual_2norm;
  double target_2norm; /* effective target after the floor (inner.py:189) */
} ipi_inner_report;

/* Solve options (driver.py:47-68 SolveOptions, pc = NONE). */
typedef struct {
  double tol;              /* -atol_pi   */
  double alpha;            /* -alpha     */
  int32_t max_outer;       /* -max_iter_pi  */
  int32_t max_inner;       /* -max_iter_ksp */
  int32_t ksp_type;        /* IPI_KSP_*  */
  int32_t ksp_max_it;      /* -ksp_max_it, <=0 = unset */
  double richardson_scale; /* -ksp_richardson_scale */
  int32_t mode;            /* IPI_MODE_* */
  int32_t pc_type;         /* -pc_type: IPI_PC_NONE or IPI_PC_JACOBI */
  int32_t gmres_ortho;     /* IPI_ORTHO_* (-ksp_gmres_modifiedgramschmidt / _classicalgramschmidt) */
  int32_t reserved;
} ipi_opts;

/* Solve statistics (driver.py:93-106 SolveResult minus the arrays). */
typedef struct {
  int32_t status;
  int32_t outer_iterations;
  int64_t inner_iterations_total;
  double wall_time;
  double time_greedy;
  double time_assembly;
  double time_inner;
  int64_t basis_reads_total; /* sum of the inner reports' basis_reads */
} ipi_stats;

/* Kernel plan chosen at ipi_mdp_create: exposed for reports/tests. */
typedef struct {
  int64_t nnz;
  int32_t row_len_min;
  int32_t row_len_max;
  double row_len_mean;
  int32_t lanes_per_row;   /* G: lanes of a warp that share one CSR row        */
  int32_t halo;            /* shared-memory V window half-width (states), -1 = none */
  int32_t k1_blocks;
  int32_t k1_threads;
  int32_t k1_smem_bytes;
  int32_t inner_blocks;
  int32_t inner_threads;
  int32_t inner_smem_bytes;
  int32_t uniform_rows;    /* all rows have the same length: P_pi row_ptr is s*K */
  int32_t k1_variant;      /* 0 generic rows, 1 uniform rows (registers), 2 uniform rows (TMA ring),
                              3 uniform rows (deep registers), 4 flat rows (cp.async ring),
                              5 flat rows (registers), 6 uniform rows (cp.async ring) */
  int32_t k1_stages;       /* shared-memory ring stages (variants 2, 4, 6) */
  int32_t k1_tma_chunk_states; /* states per TMA stage (variant 2) */
  int32_t contiguous_rows; /* every row's columns are consecutive (banded rows, C4): the
                              generic kernels read one column per row */
} ipi_plan;

/* Plan of a policy operator (ipi_op_create): exposed for reports/tests. */
typedef struct {
  int64_t nnz;
  int32_t variant;   /* IPI_K3_* */
  int32_t row_len;   /* uniform row length K (0 = variable) */
  int32_t halo;      /* shared-memory x window half-width, -1 = none */
  int32_t blocks;
  int32_t threads;
  int32_t smem_bytes;
  int32_t stages;
  int32_t lanes_per_row; /* generic variant */
  int32_t interleave;    /* uniform ring: warps take interleaved 4-row steps */
} ipi_op_plan;

/* Validation summary (model.py:148-194 validate; sparse.py:56-86 check). */
typedef struct {
  int64_t bad_row_ptr;       /* count of row_ptr decreases (+1 if rp[0]!=0)   */
  int64_t bad_col_range;     /* count of cols outside [0, n)                  */
  int64_t bad_col_order;     /* count of non-increasing pairs inside a row    */
  int64_t nonfinite_values;  /* count of non-finite transition values         */
  int64_t first_bad_prob;    /* first entry index outside [0,1], -1 if none   */
  double first_bad_prob_value;
  int64_t n_bad_row_sums;    /* rows whose |sum-1| > 1e-12                    */
  int64_t bad_rows[5];       /* first five such rows (ascending)              */
  double bad_row_sums[5];
  int64_t nonfinite_cost;    /* first flat index of a non-finite cost, -1 none */
} ipi_validation;

/* Structural CSR check (sparse.py:56-86 CsrMatrix.check). */
typedef struct {
  int64_t nnz;               /* row_ptr[rows]                                  */
  int64_t nnz_mismatch;      /* row_ptr[rows] != length of col/val arrays       */
  int64_t bad_row_ptr;       /* decreases in row_ptr (+1 if row_ptr[0] != 0)    */
  int64_t bad_col_range;
  int64_t bad_col_order;
  int64_t nonfinite_values;
} ipi_csr_report;

const char* ipi_last_error(void);
int ipi_device_count(void);
/* Build information string (arch, git-free version). */
const char* ipi_version(void);

/* CsrMatrix construction check; runs only the row-pointer pass when that fails. */
int ipi_csr_check(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t rows,
                  int64_t cols, int64_t nnz_len, ipi_csr_report* out, void* stream);

/* ---- instance handle -------------------------------------------------- */
/* Borrow an MDP that lives in HBM and plan the kernels for it.
 * n_local states owned by this rank starting at global state `state0`
 * (model.py:95-109 make_partition); n_global columns.  Replaces
 * MdpInstance (model.py:112-141) as the device-side carrier. */
int ipi_mdp_create(const int64_t* row_ptr, const int32_t* col, const double* values,
                   const double* stage_cost, int64_t n_local, int64_t n_global, int32_t m,
                   int64_t state0, double gamma, int32_t mode, void* stream, ipi_mdp** out);
void ipi_mdp_destroy(ipi_mdp* h);
int ipi_mdp_plan(const ipi_mdp* h, ipi_plan* out);
/* Diagnostics: enable != 0 starts recording (smid, start ns, end ns) per K1
 * CTA (uniform-ring kernel) of later ipi_bellman calls; enable == 0 copies up
 * to cap words of the last launch's record to host `out` and stops. */
int ipi_mdp_k1_trace(ipi_mdp* h, int32_t enable, uint64_t* out, int32_t cap);

/* validate (model.py:148-194, sparse.py:56-86) on device. */
int ipi_validate(ipi_mdp* h, ipi_validation* out, void* stream);

/* ---- K1: fused Bellman backup ---------------------------------------- */
/* greedy_policy (bellman.py:44-68) + residual norm(v - applied, inf)
 * (driver.py:136).  v_full: n_global values.  policy int32[n_local],
 * applied f64[n_local]; g_pi / len_pi / res_inf_bits nullable.  res_inf_bits
 * is an 8-byte device word receiving the max via integer atomicMax on the
 * IEEE bits of |v-applied| (>= 0); ipi_bellman zeroes it first (memset). */
int ipi_bellman(ipi_mdp* h, const double* v_full, int32_t mode, int32_t* policy, double* applied,
                double* g_pi, int32_t* len_pi, unsigned long long* res_inf_bits, void* stream);

/* ---- K2: policy compaction (sparse.py:243-269) ------------------------ */
int ipi_policy_nnz(ipi_mdp* h, const int32_t* policy, int64_t* nnz_out, void* stream);
int ipi_gather_policy(ipi_mdp* h, const int32_t* policy, int64_t* rp_pi, int32_t* col_pi,
                      double* val_pi, double* g_pi, void* stream);

/* ---- K3: SpMV family (sparse.py:189-215, 294-295) --------------------- */
/* y = A x for a general CSR (rows x cols). */
int ipi_spmv(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t rows,
             int64_t cols, const double* x, double* y, void* stream);
/* PolicyOperator.apply: y = x - gamma*(P x); with b != NULL: y = b - (x - gamma*(P x)). */
int ipi_apply_J(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                double gamma, const double* x, const double* b, double* y, void* stream);

/* Row-sharded PolicyOperator.apply for rank-local rows [state0, state0+n_local):
 * y = x_full[state0+r] - gamma*(P x_full)[r]  (b == NULL)  or  b[r] - that.
 * x_full holds all n_global entries (the all-gathered vector). */
int ipi_apply_J_shard(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi,
                      int64_t n_local, int64_t state0, double gamma, const double* x_full,
                      const double* b, double* y, void* stream);

/* Planned policy operator J_pi = I - gamma*P_pi over a row block (PolicyOperator,
 * sparse.py:272-295).  Rows [0, n_local) of (rp, col, val) are the states
 * state0 .. state0+n_local-1 of an n_global-state system (state0 = 0,
 * n_local = n_global for an unsharded operator).  Planning reads the row
 * statistics and a sampled locality profile (one host sync); the applies
 * below never synchronise.  The arrays are borrowed for the operator's life. */
int ipi_op_create(const int64_t* rp, const int32_t* col, const double* val, int64_t n_local,
                  int64_t n_global, int64_t state0, double gamma, void* stream, ipi_op** out);
void ipi_op_destroy(ipi_op* op);
/* Diagnostics: per-CTA (smid, start ns, end ns) of the ring kernels' later launches
 * (enable != 0 starts recording; enable == 0 copies up to cap words to host and stops). */
int ipi_op_trace(ipi_op* op, int32_t enable, uint64_t* out, int32_t cap);
int ipi_op_get_plan(const ipi_op* op, ipi_op_plan* out);
/* apply (sparse.py:294-295): y = x - gamma*(P x) (b == NULL) or y = b - (x - gamma*(P x))
 * (inner.py:220/232/276); x_full holds all n_global entries, y and b n_local. */
int ipi_op_apply(const ipi_op* op, const double* x_full, const double* b, double* y, void* stream);
/* spmv (sparse.py:189-215): y = P x_full. */
int ipi_op_spmv(const ipi_op* op, const double* x_full, double* y, void* stream);
/* Remote half of a split apply (parallel.py, all-gather overlap): y = x_full[state0+r]
 * - gamma*(y_partial[r] + (P x_full)[r]) (b == NULL) or b[r] - that, where
 * y_partial is the local-column half P_loc x_local computed while V was gathered. */
int ipi_op_apply_partial(const ipi_op* op, const double* x_full, const double* y_partial,
                         const double* b, double* y, void* stream);
/* Split a row block's CSR into columns in [lo, hi) (stored as col - lo) and the
 * rest, each keeping the row's column order.  Pass 1 (col_loc == NULL): per-row
 * counts into rp_loc[r+1] / rp_rem[r+1] (caller sets [0] = 0 and scans);
 * pass 2: scatter.  Used per outer iteration on the rank's P_pi rows. */
int ipi_csr_split_local(const int64_t* rp, const int32_t* col, const double* val, int64_t rows,
                        int64_t lo, int64_t hi, int64_t* rp_loc, int32_t* col_loc, double* val_loc,
                        int64_t* rp_rem, int32_t* col_rem, double* val_rem, void* stream);

/* ---- row-sharded inner solve: device-resident MGS (parallel.py) ------- */
/* out[0] = <a, b> over n entries (this rank's partial; sparse.py:218-226).
 * Deterministic (fixed grid, ordered block partials); one stream per device. */
int ipi_dot_partial(const double* a, const double* b, int64_t n, double* out, void* stream);
/* One MGS pass of a sharded Arnoldi step (inner.py:251-253):
 * h = partials[0] + ... + partials[R-1] (rank order), h_out[0] = h,
 * w -= h*v, out_partial[0] = <v_next, w> (v_next == NULL: <w, w>). */
int ipi_mgs_pass(const double* partials, int32_t R, double* h_out, double* w, const double* v,
                 const double* v_next, int64_t n, double* out_partial, void* stream);

/* Min / max column index of a CSR block's nnz entries (the V range a
 * row-sharded rank's rows read; parallel.py uses it to pick a halo exchange
 * instead of the all-gather when column locality allows).  One sync. */
int ipi_col_range(const int32_t* col, int64_t nnz, int64_t* cmin, int64_t* cmax, void* stream);

/* ---- K4: policy evaluation (inner.py:163-292) ------------------------- */
/* Jacobi preconditioner of I - gamma P_pi: inv_diag[s] = 1/(1 - gamma P_pi[s,s])
 * (build_preconditioner JACOBI, inner.py:115-118). */
int ipi_jacobi_inv_diag(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi,
                        int64_t n, double gamma, double* inv_diag, void* stream);
/* Diagnostics: enable = 1 makes later persistent inner solves record CTA 0's
 * %globaltimer at phase boundaries (out[0] = count, out[1..] = ns); enable = 0
 * copies up to cap entries into out (host) and stops recording. */
int ipi_k4_trace(int32_t enable, uint64_t* out, int32_t cap);
/* Diagnostics: the uniform ring SpMV of the persistent kernel as a plain
 * kernel, y = x - gamma P x (K = 64 rows), timed over reps launches. */
int ipi_k4_ring_apply_test(const int32_t* col, const double* val, int64_t n, double gamma,
                           const double* x, double* y, int32_t reps, float* ms, void* stream);
/* ---- row-sharded iPI (one process per GPU) ------------ */
/* The two exchanges of the sharded path, supplied by the caller: NCCL over
 * NVLink (ipi_comm_nccl) in production, host-staged gloo callbacks in the CPU
 * tests.  Both are stream-ordered on `stream` and return IPI_OK or an error. */
typedef struct {
  void* ctx;
  int32_t rank, world;
  /* every rank's block of the state vector (rank r: block_start[r] ..
   * block_start[r+1], make_partition, model.py:95-109) into `full` */
  int (*allgather_blocks)(void* ctx, const double* local, double* full, void* stream);
  /* each rank's `count` doubles -> out (world x count, rank-major) */
  int (*allgather)(void* ctx, const double* send, double* out, int64_t count, void* stream);
} ipi_comm;
/* An ipi_comm over an existing NCCL communicator (ncclComm_t, e.g. torch's
 * ProcessGroupNCCL._comm_ptr()); block_start (world+1 entries) is copied.
 * libnccl.so.2 is resolved at run time (the one the process already loaded). */
int ipi_comm_nccl(void* nccl_comm, int32_t rank, int32_t world, const int64_t* block_start,
                  ipi_comm* out);
void ipi_comm_nccl_destroy(ipi_comm* c);
/* Synchronous copy between any two (UVA) pointers on `stream`: the staging of
 * host-side collectives (gloo test callbacks). */
int ipi_memcpy_sync(void* dst, const void* src, int64_t bytes, void* stream);
/* driver.py:109-209 across ranks: `h` is this rank's shard (ipi_mdp_create with
 * state0 / n_global), v_local its block of V0 (in) and of the final V (out),
 * policy its block of the final greedy policy.  Inner solves: GMRES(30) with
 * CGS2 orthogonalisation (3 all-gathers of partial dots per Arnoldi step) or
 * Richardson; preconditioner none or jacobi; opts->mode overrides the
 * shard's.  Every rank returns the same history, counts and status. */
int ipi_solve_sharded(ipi_mdp* h, const ipi_comm* comm, const ipi_opts* opts, double* v_local,
                      int32_t* policy, double* history, int32_t hist_cap, ipi_stats* stats,
                      void* stream);

/* Solve (I - gamma P_pi) x = b from x (in/out) to the floored 2-norm target
 * or max_it iterations, device-resident: one persistent cooperative kernel
 * per call, or (GMRES/MGS on large uniform K = 64-class rows) the stepped
 * solver of krylov_step.cu, two launches per Arnoldi step.
 * inv_diag == NULL: pc = identity; else left Jacobi preconditioning.
 * ortho: IPI_ORTHO_* (GMRES only).  The Krylov workspace is one arena per
 * (device, stream): concurrent calls must use different streams. */
int ipi_inner_solve(const int64_t* rp_pi, const int32_t* col_pi, const double* val_pi, int64_t n,
                    double gamma, const double* b, double* x, double target_2norm,
                    int32_t max_it, int32_t kind, double richardson_scale,
                    const double* inv_diag, int32_t ortho, ipi_inner_report* report,
                    void* stream);

/* ---- outer iPI loop (driver.py:109-209) ------------------------------- */
/* v (device, n) holds V0 on entry and the final V on exit; policy (device,
 * int32 n) the greedy policy of the final V; history (host) receives
 * residual_history (capacity hist_cap >= max_outer + 1). */
int ipi_solve(ipi_mdp* h, const ipi_opts* opts, double* v, int32_t* policy, double* history,
              int32_t hist_cap, ipi_stats* stats, void* stream);

/* ---- device generators for the BASELINE configs ----------------------- */
/* C2/C5 locality random rows [row0, row0+rows) of an (n*m) x n instance. */
int ipi_gen_locality(int64_t n, int32_t m, int32_t K, int64_t window, uint64_t seed,
                     int64_t state0, int64_t n_states, int64_t* row_ptr, int32_t* col,
                     double* val, double* cost, void* stream);
/* C3 pendulum (N x N grid, n_actions torques) for states [state0, state0+n_states). */
int ipi_gen_pendulum(int32_t N, int32_t n_actions, int64_t state0, int64_t n_states,
                     int64_t* row_ptr, int32_t* col, double* val, double* cost, void* stream);
/* C4 SIS convolution rows: two-pass.  Pass 1 (col == NULL): row lengths into
 * row_ptr[1..] (caller scans).  Pass 2: fill col/val/cost. */
int ipi_gen_sis(int32_t population, int32_t pass, int64_t* row_ptr, int32_t* col, double* val,
                double* cost, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* IPI_B200_H */
