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
                         int reps = 1) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    if (e0) cudaEventDestroy(e0);
    cudaGetLastError();
    return -1;
  }
  float best_ms = 1e30f;
  int best = -1;
  for (int i = 0; i < ncand; ++i) {
    if (!install(i)) continue;
    if (launch()) break;
    cudaEventRecord(e0, st);
    bool bad = false;
    for (int r = 0; r < reps && !bad; ++r) bad = launch() != 0;
    if (bad) break;
    cudaEventRecord(e1, st);
    float ms = 0.f;
    if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) break;
    if (ms < best_ms) {
      best_ms = ms;
      best = i;
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
