// krylov_cgs.cu — GMRES(30) with CGS2 orthogonalisation: instantiations of the
// 1024-thread persistent inner kernel (krylov.cuh) for the rows the ring
// kernel (krylov_ring.cu) does not take: variable-length (C4) and short or
// odd uniform rows (C1, C3).  A separate translation unit and template
// instance, so the MGS kernel keeps its own register allocation (the CGS
// passes' accumulators would otherwise spill into it).
#include "krylov.cuh"

namespace ipi {

int dispatch_inner_gmres_cgs(KArgs& a, int G, int P, int lanes, bool win, int smem, int blocks,
                             cudaStream_t st) {
  return dispatch_inner<kKindGmresCgs>(a, G, P, lanes, win, smem, blocks, st);
}

}  // namespace ipi
