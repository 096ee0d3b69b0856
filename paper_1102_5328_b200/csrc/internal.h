// internal.h -- shared declarations of libtileqr's CUDA kernels and host runtime.
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Boundary").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/tileqr.h"

namespace tileqr {

// ---- error plumbing (api.cu) --------------------------------------------
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define TQ_CUDA(call)                                                         \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) return ::tileqr::cuda_fail(e_, #call, __FILE__, __LINE__); \
  } while (0)
#define TQ_LAUNCH_CHECK()                                                     \
  do {                                                                        \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) return ::tileqr::cuda_fail(e_, "kernel launch", __FILE__, __LINE__); \
  } while (0)

// ---- argument validation shared by entry points ---------------------------
inline bool valid_nb_ib(int NB, int IB) {
  return NB >= 1 && NB <= 512 && IB >= 1 && IB <= NB && NB % IB == 0;
}

// ---- layout / utility kernels (kernels_layout.cu) --------------------------
// A (M x N, lda) -> padded tile buffer (MT*NT tiles of NB*NB, tile (m,n) at
// (m + n*MT)*NB*NB); sets *d_info = 1 when A holds a non-finite value.
int launch_layout_to_tiles(int64_t M, int64_t N, const double* A, int64_t lda, int NB, int64_t MT,
                           int64_t NT, double* tiles, int* d_info, cudaStream_t s);
int launch_t_assemble(bool ts, int NB, int IBe, int IB, int batch, const double* const* V,
                      const double* const* Tin, double* const* Tout, cudaStream_t s);
int effective_ib(int NB, int IB);
int launch_t_extract_ptrs(const double* const* Tin, int IBi, double* const* Tout, int IBo, int NB, int batch,
                          cudaStream_t s);
int launch_t_assemble_big(const double* tiles, const double* Ts, double* T, int NB, int IB, int IBs, int64_t MT,
                          int64_t NTl, int64_t KT, int P, int r, int nsm, cudaStream_t s);
int launch_t_extract(const double* Te, int IBe, double* T, int IB, int NB, int64_t ntiles, cudaStream_t s);
int launch_tiles_to_layout(int64_t M, int64_t N, double* A, int64_t lda, int NB, int64_t MT,
                           int64_t NT, const double* tiles, cudaStream_t s);
// Copy the V part of A (M x K) into a tile buffer (rows >= M zero, columns >= K zero).
int launch_v_to_tiles(int64_t M, int64_t K, const double* A, int64_t lda, int NB, int64_t MT,
                      int64_t KT, double* tiles, cudaStream_t s);
int launch_rng_uniform(int64_t M, int64_t N, double* A, int64_t lda, uint64_t seed, uint64_t offset,
                       cudaStream_t s);
int launch_zero_int(int* p, cudaStream_t s);
// out[i] = base + i*stride, i < n (device pointer arrays for batched calls)
int launch_fill_ptrs(double** out, double* base, size_t stride, int n, cudaStream_t s);

// ---- tile kernels ---------------------------------------------------------
// All take device arrays of device pointers (tiles NB x NB, ld NB; T IB x NB, ld IB).
// Pk (nullable): per task, a packed copy of the reflector tile (V_p, T_p) for
// the barrier-free update (update_v2.cuh; written when v2_supported(NB, IB)).
int launch_geqrt(int NB, int IB, int batch, double* const* A, double* const* T, cudaStream_t s,
                 double* const* Pk = nullptr);
int launch_tsqrt(int NB, int IB, int batch, double* const* R, double* const* A2, double* const* T,
                 cudaStream_t s, double* const* Pk = nullptr);
int launch_larfb(bool trans, int NB, int IB, int batch, const double* const* V,
                 const double* const* T, double* const* C, int ncols, cudaStream_t s);
int launch_ssrfb(bool trans, int NB, int IB, int batch, const double* const* V2,
                 const double* const* T, double* const* C1, double* const* C2, int ncols,
                 cudaStream_t s);

// Packed-reflector update path (update_v2.cuh): Q^T form, full tiles,
// NB in {32, 64, 96, 128}, IB in {8, 16, 24, 32}, IB | NB.
bool v2_supported(int NB, int IB);
size_t v2_pk_doubles(int NB, int IB);  // doubles per packed reflector tile
int launch_update_pk(bool larfb, int NB, int IB, int batch, const double* const* Pk, double* const* C1,
                     double* const* C2, cudaStream_t s);
// standard V (GEQRT form if larfb) / T tiles -> packed tiles
int launch_pack(bool larfb, int NB, int IB, int batch, const double* const* V, const double* const* T,
                double* const* Pk, cudaStream_t s);

// Which SSRFB implementation a (NB, IB) pair uses ("dmma" or "simt").
const char* ssrfb_impl_name(int NB, int IB);
// Decision-table lookup (table.cu): (NB, IB) for an M x N factorization on
// ngpus GPUs; the built-in default when no table is installed (*from_table false).
int lookup_pair(int64_t M, int64_t N, int ngpus, int* NB, int* IB, bool* from_table);
// ---- dataflow kernel (dag.cuh, launched through api.cu) ----------------------
namespace dag { struct Item; struct DagIO; }
int launch_dag(int NB, int IB, const dag::Item* items, int nitems, int* next, int* done, int nsm,
               unsigned long long* prof, cudaStream_t s, int* grid_out, const dag::DagIO* io, int mode);
int panel_sub_cols(int NB, int IB);       // columns of one GEQRT / TSQRT sub-task
bool dag_path_supported(int NB, int IB);  // the dataflow kernel with packed reflector tiles runs (NB, IB)
// ---- multi-GPU helpers (dist.cu) for tileqr_tune with ngpus > 1 -----------------
int dist_ranks(int* nranks, int* rank);
int dist_host_collective(double* h, int n, int op);  // op 0: broadcast from rank 0, 1: max over ranks
// Stream-ordered scratch (cudaMallocAsync) from the device's default pool,
// which is told once per device to keep freed memory (release threshold =
// max): the batched / apply entry points allocate per call, and a pool that
// returns memory to the driver at every synchronisation made each such call
// pay a fresh allocation (~0.3-2 ms, measured on the wide-panel launches).
int stream_alloc(void** p, size_t bytes, cudaStream_t s);
// Free the cached tileqr_factor workspace of one shape (api.cu; waits for its last use).
void release_ws(int dev, int64_t M, int64_t N, int NB, int IB);

}  // namespace tileqr
