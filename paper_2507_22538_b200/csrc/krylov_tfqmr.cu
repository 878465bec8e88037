// krylov_tfqmr.cu — TFQMR instantiations of the persistent inner kernel
// (separate translation unit: compiled in parallel, keeps register pressure
// of the GMRES kernel unaffected).
#include "krylov.cuh"

namespace ipi {

int dispatch_inner_tfqmr(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                          cudaStream_t st) {
  return dispatch_inner<3>(a, G, P, lanes, win, smem, blocks, st);
}

}  // namespace ipi
