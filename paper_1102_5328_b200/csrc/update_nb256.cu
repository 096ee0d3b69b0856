// update_nb256.cu -- instantiation of the DMMA update kernels for NB = 256
// (one translation unit per NB so the build compiles them in parallel).
#include "update_dmma.cuh"

namespace tileqr {
int launch_update_nb256(bool trans, bool larfb, int IB, int batch, const double* const* V,
                        const double* const* T, double* const* C1, double* const* C2, int ncols,
                        cudaStream_t s) {
  return upd::launch_update_dmma<256>(trans, larfb, IB, batch, V, T, C1, C2, ncols, s);
}
}  // namespace tileqr
