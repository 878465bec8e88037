// plan.cuh — planning helpers shared by plan.cu (instances) and capi.cu (operators).
#pragma once

#include "handle.cuh"

namespace ipi {

inline int grid_for(int64_t work, int threads, int sms) {
  int64_t b = (work + threads - 1) / threads;
  b = std::min<int64_t>(b, (int64_t)sms * 32);
  return (int)std::max<int64_t>(b, 1);
}

// Plan-time autotuning: for each candidate that `install(i)` accepts, run
// `launch()` once warm and `reps` times timed (CUDA events on `st`) and return the
// index of the fastest (-1 if none ran).  The kernels' streaming rate depends on
// the CTA count in a board-dependent way, so large instances are
// planned by measurement; callers install the winner afterwards.
template <class Install, class Launch>
inline int autotune_pick(int ncand, Install&& install, Launch&& launch, cudaStream_t st,
                         int reps = 1, int refine = 0, int refine_reps = 0) {
  // One warm + `reps` timed launches per candidate; then, when refine > 0, the
  // `refine` fastest are timed again with `refine_reps` launches each and the
  // fastest of that round wins (a single short timing picked a 10% slower K3
  // shape in about one process out of four).
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    if (e0) cudaEventDestroy(e0);
    cudaGetLastError();
    return -1;
  }
  auto time_one = [&](int i, int n, float* ms_per) -> bool {
    if (!install(i)) return false;
    if (launch()) return false;
    cudaEventRecord(e0, st);
    for (int r = 0; r < n; ++r)
      if (launch() != 0) return false;
    cudaEventRecord(e1, st);
    float ms = 0.f;
    if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) return false;
    *ms_per = ms / (float)n;
    return true;
  };
  float t[64];
  const int nc = ncand < 64 ? ncand : 64;
  int best = -1;
  for (int i = 0; i < nc; ++i) {
    t[i] = 1e30f;
    float ms;
    if (time_one(i, reps, &ms)) t[i] = ms;
    if (t[i] < 1e30f && (best < 0 || t[i] < t[best])) best = i;
  }
  if (best >= 0 && refine > 1 && refine_reps > 0) {
    int top[8];
    const int nt = refine < 8 ? refine : 8;
    bool used[64] = {};
    int got = 0;
    for (int k = 0; k < nt; ++k) {
      int b = -1;
      for (int i = 0; i < nc; ++i)
        if (!used[i] && t[i] < 1e30f && (b < 0 || t[i] < t[b])) b = i;
      if (b < 0) break;
      used[b] = true;
      top[got++] = b;
    }
    float best_ms = 1e30f;
    for (int k = 0; k < got; ++k) {
      float ms;
      if (time_one(top[k], refine_reps, &ms) && ms < best_ms) {
        best_ms = ms;
        best = top[k];
      }
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGetLastError();
  return best;
}

// Zeroed V plus output buffers for timing K1 candidates at plan time.
struct K1Scratch {
  double* v = nullptr;
  double* applied = nullptr;
  int32_t* policy = nullptr;
  bool ok = false;
  K1Scratch(int64_t n_global, int64_t n_local, cudaStream_t st) {
    ok = cudaMalloc(&v, sizeof(double) * n_global) == cudaSuccess &&
         cudaMalloc(&applied, sizeof(double) * n_local) == cudaSuccess &&
         cudaMalloc(&policy, sizeof(int32_t) * n_local) == cudaSuccess &&
         cudaMemsetAsync(v, 0, sizeof(double) * n_global, st) == cudaSuccess;
    if (!ok) cudaGetLastError();
  }
  ~K1Scratch() {
    cudaFree(v);
    cudaFree(applied);
    cudaFree(policy);
  }
};

// plan.cu: every kernel choice for an instance (row statistics, V window,
// K1 variant and grid, autotuning).  Called by ipi_mdp_create.
int plan_instance(ipi_mdp* h, cudaStream_t st);

}  // namespace ipi
