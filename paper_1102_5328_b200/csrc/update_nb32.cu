// update_nb32.cu -- instantiation of the DMMA update kernels and of the
// dataflow DAG kernel for NB = 32 (one translation unit per NB so the build
// compiles them in parallel).
#include "dag.cuh"
#include "update_dmma.cuh"
#include "update_v2.cuh"

namespace tileqr {
int launch_update_nb32(bool trans, bool larfb, int IB, int batch, const double* const* V,
                        const double* const* T, double* const* C1, double* const* C2, int ncols,
                        cudaStream_t s) {
  return upd::launch_update_dmma<32>(trans, larfb, IB, batch, V, T, C1, C2, ncols, s);
}
int launch_dag_nb32(int IB, const dag::Item* items, int nitems, int* next, int* done, int nsm,
                     unsigned long long* prof, cudaStream_t s, int* grid_out, const dag::DagIO* io,
                     int mode) {
  return dag::launch_dag_nb<32>(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
}
int launch_update_pk_nb32(bool larfb, int IB, int batch, const double* const* Pk, double* const* C1,
                          double* const* C2, cudaStream_t s) {
  return v2::launch_update_v2<32>(larfb, IB, batch, Pk, C1, C2, s);
}
int launch_pack_nb32(bool larfb, int IB, int batch, const double* const* V, const double* const* T,
                     double* const* Pk, cudaStream_t s) {
  return v2::launch_pack<32>(larfb, IB, batch, V, T, Pk, s);
}
}  // namespace tileqr
