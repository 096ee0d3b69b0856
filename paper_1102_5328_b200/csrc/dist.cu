// dist.cu -- multi-GPU tile QR (placeholder until the NCCL path lands).
#include "internal.h"

using namespace tileqr;

extern "C" {
int tileqr_dist_unique_id(void* h_id) { (void)h_id; set_error("dist: not built"); return TILEQR_ERR_NOT_INIT; }
int tileqr_dist_init(int nranks, int rank, const void* id, int device) {
  (void)nranks; (void)rank; (void)id; (void)device;
  set_error("dist: not built");
  return TILEQR_ERR_NOT_INIT;
}
int tileqr_dist_local_cols(int64_t N, int NB, int* n_local) { (void)N; (void)NB; (void)n_local; return TILEQR_ERR_NOT_INIT; }
int tileqr_dist_fill_uniform(int64_t N, int NB, double* A_local, uint64_t seed, tileqr_stream_t s) {
  (void)N; (void)NB; (void)A_local; (void)seed; (void)s;
  return TILEQR_ERR_NOT_INIT;
}
int tileqr_dist_factor(int64_t N, double* A_local, int NB, int IB, double* T_local, int* d_info,
                       tileqr_stream_t s) {
  (void)N; (void)A_local; (void)NB; (void)IB; (void)T_local; (void)d_info; (void)s;
  return TILEQR_ERR_NOT_INIT;
}
void tileqr_dist_finalize(void) {}
}
