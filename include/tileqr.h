/*
 * tileqr.h -- C ABI of the B200-native (sm_100a) FP64 tile Householder QR
 * library libtileqr.so (package paper_1102_5328_b200).
 *
 * The method is the PLASMA-style tile QR of arxiv 1102.5328 (INRIA RR-7526):
 * "split the initial matrix of order N into NT x NT smaller square pieces of
 * order NB, called tiles", factored by four serial kernels
 * "DGEQRT and DTSQRT ... DLARFB and DSSRFB" whose DAG is
 * executed level by level; (NB, IB) are the tunable parameters of Problem 1
 * and tileqr_tune applies the paper's Step-1/Step-2
 * pruning.  Kernel internals follow the compact-WY
 * formulation adopted by SPEC.md:125 (readings listed in DESIGN.md).
 *
 * Conventions (all entry points):
 *   - Matrices are FP64, column-major.  Pointers are DEVICE pointers on the
 *     current CUDA device unless the name starts with h_ (host).
 *   - Work is stream-ordered on `stream` (0 = legacy default stream); the
 *     library never synchronizes the stream except where stated (tune).
 *   - The caller owns A, T, B and every batched operand; the library owns a
 *     workspace (padded tile buffer, task lists, CUDA graphs, NCCL comm)
 *     cached per (device, shape) -- at most TILEQR_WS_CACHE shapes (default
 *     4; the least recently used is freed after its last use) -- and released
 *     by tileqr_finalize().
 *   - Return value: 0 = success; -i = the i-th argument is illegal (LAPACK
 *     xerbla style, nothing is launched); > 0 = TILEQR_ERR_* (message from
 *     tileqr_last_error()).  NB must satisfy 1 <= NB <= 512 (the paper bounds
 *     tiles by 512) and 1 <= IB <= NB with IB dividing NB
 *     (PAPER.md:366-367).
 *   - Results are deterministic: bitwise identical run to run (and across
 *     GPU counts in tileqr_dist_factor) for the same (NB, IB).
 *   - No CPU fallback exists: without a CUDA device every compute call returns
 *     TILEQR_ERR_CUDA.
 *   - Supported input range: the reflectors form plain sums of squares with no
 *     LAPACK-style safmin/safmax rescaling (R1), so entries must
 *     satisfy 2^-450 <= |a_ij| <= 2^450 (or be 0) for every sum to stay in
 *     the normal FP64 range; scaling A by a power of two inside that range
 *     scales R exactly and leaves V and T unchanged (tests).
 *   - Concurrency: calls of the same shape share one cached workspace; each
 *     call's stream waits for the previous call's last operation on it (an
 *     event), so same-shape calls on different streams or host threads are
 *     serialised on the device, not corrupted.
 */
#ifndef TILEQR_H_
#define TILEQR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tileqr_stream_t; /* == cudaStream_t */

enum {
  TILEQR_OK = 0,
  TILEQR_ERR_CUDA = 1,     /* a CUDA runtime call or kernel launch failed  */
  TILEQR_ERR_NCCL = 2,     /* an NCCL call failed                           */
  TILEQR_ERR_ALLOC = 3,    /* device or host allocation failed              */
  TILEQR_ERR_NOT_INIT = 4, /* tileqr_dist_* before tileqr_dist_init         */
  TILEQR_ERR_INTERNAL = 5
};

/* Library version string, e.g. "tileqr 0.1 sm_100a". */
const char* tileqr_version(void);

/* Thread-local text of the last error (empty string when none). */
const char* tileqr_last_error(void);

/* Number of doubles of the T buffer of an M x N factorization:
 * MT*NT*IB*NB with MT = ceil(M/NB), NT = ceil(N/NB).
 * T tile (m,k), m >= k, starts at offset (m + k*MT)*IB*NB and is IB x NB with
 * ld = IB: block p (columns [p*IB,(p+1)*IB)) is the IB x IB upper-triangular
 * compact-WY factor of inner panel p; its strictly-lower part is 0.
 * Errors: -1..-4 for M < 0, N < 0, bad NB, bad IB; -5 for n_doubles == NULL. */
int tileqr_t_size(int64_t M, int64_t N, int NB, int IB, size_t* n_doubles);

/* ------------------------------------------------------------------------
 * tileqr_lookup -- (NB, IB) from the installed decision table of the
 * autotuner: "the pre-built decision tree is used" when the user calls the
 * library, by nearest-point interpolation on the tuned
 * grid.  The table (tools/autotune.py -> tileqr_tune over
 * the (N, ngpus) grid) is read from $TILEQR_TUNED_TABLE, else from
 * tuned_table.json beside libtileqr.so.  Axes: the order of the problem (for
 * M x N the square order with the same useful flop count, (3/4 *
 * flops)^(1/3); R19) and ngpus; per-axis nearest grid value, ties
 * toward the larger one.
 *   Returns 0 (pair from the table) or TILEQR_ERR_NOT_INIT when no table is
 *   installed -- *h_NB, *h_IB then hold the built-in default (128, 16).
 *   Errors: -1 M < 0, -2 N < 0, -3 ngpus < 1, -4/-5 NULL outputs.
 * Every entry point taking (NB, IB) -- tileqr_t_size, tileqr_factor,
 * tileqr_factor_host, tileqr_apply_qt, tileqr_dist_factor -- accepts
 * NB = IB = 0 as "the pair tileqr_lookup returns for this shape" (with the
 * default when no table is installed).
 * ------------------------------------------------------------------------ */
int tileqr_lookup(int64_t M, int64_t N, int ngpus, int* h_NB, int* h_IB);

/* ------------------------------------------------------------------------
 * tileqr_factor -- tile QR of the M x N matrix A (Fig. 1).
 *
 *   A  [in/out] device, M x N, leading dimension lda >= max(1, M).
 *      On return (PLASMA convention): R in the upper triangle
 *      of A[0:min(M,N), 0:N]; V_kk strictly below the diagonal of tile (k,k)
 *      (unit diagonal implicit); the full V2_mk in tile (m,k), m > k.
 *      Non-dividing sizes are padded internally (reading R5).
 *   T  [out] device, tileqr_t_size() doubles (layout above); overwritten.
 *   d_info [out] device int (may be NULL): 0 = ok, 1 = A held a non-finite
 *      entry (the factorization still runs; its output is then unspecified).
 *   Workspace: (MT*NB) x (NT*NB) doubles plus task lists, cached.
 *   Inner blocking (R23): an IB that is not a multiple of 8 runs
 *   at IBe = lcm(IB, 8) when IBe <= 64 divides NB, an IB > 64 at the largest
 *   of 32, 24, 16, 8 dividing it; R and V are the IB-blocked reflectors (to
 *   rounding) and T is returned at IB (diagonal blocks of T at IBe, or
 *   assembled from the factored tiles).
 *   Errors: -1 M<0, -2 N<0, -3 A==NULL (M,N>0), -4 lda<max(1,M), -5 NB,
 *   -6 IB, -7 T==NULL.  Quick return for M == 0 or N == 0.
 * ------------------------------------------------------------------------ */
int tileqr_factor(int64_t M, int64_t N, double* A, int64_t lda, int NB, int IB, double* T,
                  int* d_info, tileqr_stream_t stream);

/* ------------------------------------------------------------------------
 * tileqr_factor_host -- tileqr_factor for a matrix in HOST memory, with the
 * host<->device transfers overlapped with the factorization (the user-facing
 * end-to-end call).
 *
 *   h_A [in]  host, M x N, lda >= max(1, M); read column tile by column tile
 *             by the copy engine while the factorization runs (the dataflow
 *             kernel's LOAD items convert each column tile as it lands).
 *   h_R [out] host, M x N, ldr >= max(1, M): the tileqr_factor output (R and
 *             V as there); may alias h_A (each column is read before it is
 *             written).  Column tiles are copied back as soon as the
 *             factorization has finished them (STORE items + stream waits).
 *   h_T [out] host, tileqr_t_size() doubles, the T factors.
 *   d_info [out] device int (may be NULL), as tileqr_factor.
 *   Stream-ordered: the host buffers must stay valid until `stream` completes;
 *   page-locked buffers give the full overlap (pageable ones serialise the
 *   copies with the host thread).  (NB, IB) outside the dataflow set: copy
 *   in, tileqr_factor, copy out, without overlap.
 *   Errors: -1 M, -2 N, -3 h_A, -4 lda, -5 NB, -6 IB, -7 h_R, -8 ldr, -9 h_T.
 * ------------------------------------------------------------------------ */
int tileqr_factor_host(int64_t M, int64_t N, const double* h_A, int64_t lda, int NB, int IB, double* h_R,
                       int64_t ldr, double* h_T, int* d_info, tileqr_stream_t stream);

/* ------------------------------------------------------------------------
 * tileqr_apply_qt -- B <- Q^T B (trans = 'T') or B <- Q B (trans = 'N') with
 * the Q of a tileqr_factor output:
 *   'T': k ascending: LARFB(k) on B's row-tile k, then SSRFB(k,m) on row-tiles
 *        (k, m) for m ascending;
 *   'N': k descending: SSRFB(k,m) for m descending, then LARFB(k); panels in
 *        reverse order and T not transposed.
 *   M x K is the shape that was factored (A, lda, T as returned, same NB/IB);
 *   B is M x NRHS, ldb >= max(1, M).
 *   Errors: -1 trans, -2 M, -3 NRHS, -4 K, -5 A, -6 lda, -7 T, -8 NB, -9 IB,
 *   -10 B, -11 ldb.
 * ------------------------------------------------------------------------ */
int tileqr_apply_qt(char trans, int64_t M, int64_t NRHS, int64_t K, const double* A, int64_t lda,
                    const double* T, int NB, int IB, double* B, int64_t ldb,
                    tileqr_stream_t stream);

/* ------------------------------------------------------------------------
 * Batched tile kernels.  Each takes DEVICE arrays of
 * `batch` DEVICE pointers; every tile is NB x NB with ld = NB, every T is
 * IB x NB with ld = IB.  Tiles within one call must not alias (except as
 * stated).  batch == 0 is a no-op.  Errors: -1 NB, -2 IB, -3 batch < 0,
 * -4.. NULL arrays (numbered in argument order), -(last) ncols out of range.
 * ------------------------------------------------------------------------ */

/* GEQRT: QR of each tile A[i] (R upper, V strictly lower), writes T[i]. */
int tileqr_geqrt_batched(int NB, int IB, int batch, double* const* A, double* const* T,
                         tileqr_stream_t stream);

/* TSQRT: QR of [R[i]; A2[i]] with R[i] upper triangular: updates the upper
 * triangle of R[i] only (its strict lower part is neither read nor written),
 * overwrites A2[i] with V2, writes T[i]. */
int tileqr_tsqrt_batched(int NB, int IB, int batch, double* const* R, double* const* A2,
                         double* const* T, tileqr_stream_t stream);

/* LARFB: C[i] <- Q^T C[i] ('T') or Q C[i] ('N') with Q from a GEQRT
 * (V[i] strictly-lower part read, T[i]); C[i] is NB x ncols (ld = NB),
 * 1 <= ncols <= NB. */
int tileqr_larfb_batched(char trans, int NB, int IB, int batch, const double* const* V,
                         const double* const* T, double* const* C, int ncols,
                         tileqr_stream_t stream);

/* SSRFB (TSMQR): [C1[i]; C2[i]] <- Q^T [C1; C2] ('T') or Q [C1; C2] ('N')
 * with Q from a TSQRT (V2[i], T[i]); C1, C2 are NB x ncols (ld = NB),
 * 1 <= ncols <= NB.  This is the dominant kernel. */
int tileqr_ssrfb_batched(char trans, int NB, int IB, int batch, const double* const* V2,
                         const double* const* T, double* const* C1, double* const* C2,
                         int ncols, tileqr_stream_t stream);

/* Packed reflector tiles -- the operand format of the factorization's
 * trailing-update kernel for NB % 32 == 0, NB <= 256, and IB | NB with
 * IB in {8, 16, 24, 32} or a wide IB in {40, 48, 56, 64} whose column group
 * plus T_p fits one shared-memory ring stage (every such pair of the tuning
 * grid): the V_p / T_p of a tile in the shared-memory image the
 * barrier-free DMMA update loads with TMA bulk copies (layout: DESIGN.md §5,
 * csrc/update_v2.cuh).  tileqr_factor writes them itself from its GEQRT /
 * TSQRT kernels; these entry points expose the same kernels for tests and
 * for the tuner's Step-1 timing.
 *   tileqr_packed_size: doubles per packed tile (0 if (NB, IB) unsupported).
 *   tileqr_pack_batched: Pk[i] <- pack(V[i], T[i]); larfb != 0 reads V as a
 *     GEQRT tile (unit lower trapezoid implied), else as a full TSQRT V2.
 *   tileqr_update_packed_batched: the Q^T update ('T' only, full NB x NB
 *     tiles): larfb != 0: C2[i] <- Q^T C2[i] (C1 ignored, may be NULL);
 *     else [C1[i]; C2[i]] <- Q^T [C1[i]; C2[i]].
 * Errors: -1 NB/IB unsupported, -3 batch < 0, -4.. NULL arrays. */
int tileqr_packed_size(int NB, int IB, size_t* n_doubles);
int tileqr_pack_batched(int larfb, int NB, int IB, int batch, const double* const* V,
                        const double* const* T, double* const* Pk, tileqr_stream_t stream);
int tileqr_update_packed_batched(int larfb, int NB, int IB, int batch, const double* const* Pk,
                                 double* const* C1, double* const* C2, tileqr_stream_t stream);

/* ------------------------------------------------------------------------
 * tileqr_tune -- the paper's two-step empirical tuning:
 *   Step 1: time tileqr_ssrfb_batched for every (NB, IB)
 *     of the grid NB in {64,96,...,256}, IB | NB (IB >= 8 unless
 *     TILEQR_TUNE_SMALL_IB=1), 50 back-to-back launches on the same buffers
 *     ("No Flush"); rate = 50*batch*4*NB^3/t.
 *   Pre-selection: Property 1, upper convex hull (Property 2), then Heuristic
 *     0/1/2, cap 8.  Property 1 counts the IB values
 *     whose Step-1 rate is within 0.5 % of the NB's best as tied and keeps
 *     the largest (R13/R18: closer rates are below the timing's
 *     repeatability; env TILEQR_TUNE_TIE sets the relative width).
 *   Step 2: for N' on a ladder ascending to N, time
 *     tileqr_factor 6x per surviving candidate (median), then drop NB2 when
 *     some NB1 > NB2 is strictly faster (Property 3, if payg != 0).
 *   Returns the best (NB, IB) at N in *h_NB, *h_IB.  Synchronizes the current
 *   device.  report_json_path (nullable) receives the Step-1 data set, the
 *   candidate set and every Step-2 sample as JSON.
 *   ngpus > 1: collective over the nranks == ngpus ranks of tileqr_dist_init
 *     (square problems): every rank runs Step 1, all decide on rank 0's
 *     Step-1 data set (NCCL broadcast), and Step 2 times tileqr_dist_factor,
 *     each run's time the max over ranks (PAPER.md:620-623 tunes per core
 *     count; here per GPU count).  TILEQR_TUNE_DIST=1 takes that path on one
 *     rank too.
 *   Errors: -1 M, -2 N, -3 ngpus (< 1, or != the dist ranks, or M != N),
 *   -4 heuristic not in {0,1,2}, -6/-7 NULL outputs.
 * ------------------------------------------------------------------------ */
int tileqr_tune(int64_t M, int64_t N, int ngpus, int heuristic, int payg, int* h_NB, int* h_IB,
                const char* report_json_path);

/* Pure host pieces of the tuner (no GPU needed), exported for testing:
 * Property 1 + upper hull + heuristic on n samples (nb[i], ib[i], gflops[i]);
 * writes at most `cap` (heuristic 1/2) or n (heuristic 0) selected points to
 * out_nb/out_ib/out_gflops (capacity n) and their count to *n_out. */
int tileqr_preselect(int n, const int* h_nb, const int* h_ib, const double* h_gflops, int heuristic,
                     int cap, int* h_out_nb, int* h_out_ib, double* h_out_gflops, int* n_out);
/* Same with a Property-1 tie width: per NB, every IB whose rate is
 * >= (1 - tie_rel) * the NB's best rate is tied and the largest is kept
 * (tie_rel = 0: exact ties only, as tileqr_preselect).  Errors: as
 * tileqr_preselect, -7 tie_rel not in [0, 1), -8 NULL outputs. */
int tileqr_preselect_tie(int n, const int* h_nb, const int* h_ib, const double* h_gflops, int heuristic,
                         int cap, double tie_rel, int* h_out_nb, int* h_out_ib, double* h_out_gflops,
                         int* n_out);
/* Property 3 prune: keep[i] = 0 when some j has nb[j] > nb[i] and
 * gflops[j] > gflops[i]; else 1. */
int tileqr_payg_prune(int n, const int* h_nb, const double* h_gflops, int* h_keep);
/* ASAP level of each task kind (G,L,T,S) in the tile DAG: the launcher's
 * closed form (G(k)=3k, L(k,n)=3k+1, T(k,m)=2k+m, S(k,m,n)=2k+m+1);
 * returns the number of levels of an MT x NT tile matrix in *n_levels. */
int tileqr_num_levels(int64_t MT, int64_t NT, int64_t* n_levels);

/* ------------------------------------------------------------------------
 * Multi-GPU: one process per GPU, tile columns 1D
 * block-cyclic -- tile column n lives on rank n mod nranks, stored locally
 * (local column j <-> global n = rank + j*nranks).  GEQRT(k) and the TSQRT
 * chain of panel k run on the owner of column k; LARFB(k,n) / SSRFB(k,m,n)
 * on the owner of column n.  Two schedules:
 *  - dataflow (default for NB % 32 == 0, NB <= 256, IB in {8,16,24,32}):
 *    each rank runs its share of the DAG in the persistent dataflow kernel;
 *    the panel broadcast is fused into it -- the owner pushes every packed
 *    reflector tile (V and T) over peer memory (NVLink, buffers mapped with
 *    cudaIpc, handles exchanged over NCCL) into each consumer's slot and
 *    raises the consumer's arrival counter, which its update items acquire
 *    at system scope.  No collective on the data path, no level barriers.
 *  - levels (TILEQR_DIST_SCHED=levels or other (NB, IB); square only): the
 *    level-synchronous launcher with one grouped ncclBroadcast of the level's
 *    panel tiles per DAG level (the NCCL baseline).
 * Both are bitwise equal to tileqr_factor for the same (NB, IB).
 * ------------------------------------------------------------------------ */
/* h_nccl_unique_id: 128-byte ncclUniqueId from rank 0 (e.g. via
 * torch.distributed); device: CUDA ordinal this rank uses. */
int tileqr_dist_init(int nranks, int rank, const void* h_nccl_unique_id, int device);
/* Writes a fresh ncclUniqueId (128 bytes) into h_id (rank 0 only). */
int tileqr_dist_unique_id(void* h_id);
/* Local tile storage of an M x N factorization (padded as tileqr_factor):
 * n_local = number of tile columns owned by this rank; A_local holds them in
 * tile layout: local column j (global n = rank + j*nranks) has its MT tiles
 * (MT = ceil(M/NB)) at A_local + (m + j*MT)*NB*NB, column-major within a
 * tile (ld = NB).  T_local: tile (m, j) at (m + j*MT)*IB*NB. */
int tileqr_dist_local_cols(int64_t N, int NB, int* n_local);
/* Fill this rank's local tile columns with the synthetic generator below
 * (global idx = i + j*M of the M x N matrix), zero / identity padding as
 * tileqr_factor does.  Errors: -1 M, -2 N, -3 NB, -4 A_local NULL. */
int tileqr_dist_fill_uniform(int64_t M, int64_t N, int NB, double* A_local, uint64_t seed,
                             tileqr_stream_t stream);
/* Host-only schedule of one DAG level of the LEVEL-SYNCHRONOUS path for
 * `rank` of `nranks` (square MT x MT tiles), exported so the multi-GPU plan
 * can be tested without GPUs.  Writes 5-tuples (kind, k, m, n, root) to h_out
 * (capacity `cap` int64s): first the rank's panel tasks (kind 0 GEQRT(k), 1
 * TSQRT(k,m)), then the level's broadcast items (kind 4: V/T of tile (m,k)
 * from root = k mod nranks, same list and order on every rank), then the
 * rank's update tasks (2 LARFB(k,n), 3 SSRFB(k,m,n), n = local columns);
 * h_counts[3] = the three counts.
 * Errors: -1..-4 bad MT/nranks/rank/level, -6 capacity too small, -7 NULL. */
int tileqr_dist_plan_level(int64_t MT, int nranks, int rank, int64_t level, int64_t* h_out,
                           int64_t cap, int64_t* h_counts);
/* Host-only work list of one rank under the DATAFLOW schedule (the items its
 * persistent kernel claims, in claim order), for CPU tests of the plan:
 * per item 10 int64 (kind, k, m, n, s, task, ndep, dep0, dep1, dep2) with kind
 * 0 GEQRT, 1 TSQRT, 2 LARFB, 3 SSRFB, 7 COPY; s = the panel sub-task (inner
 * panels [s*sub_cols, (s+1)*sub_cols)), the update slab, or for COPY the
 * destination rank; task / dep = global task ids (a dependency on an id of
 * kind 6 ARRIVE is the arrival of the COPY of reflector tile (k, m) at this
 * rank).  workers: resident CTAs per rank in the schedule simulation;
 * sub_cols: columns per panel sub-task (IB | sub_cols | NB).  *h_count
 * receives the item count; h_out (capacity cap int64s) may be NULL.
 * Errors: -1 M, -2 N, -3 NB/IB, -5 nranks, -6 rank, -7 workers, -8 sub_cols,
 * -10 capacity too small, -11 h_count NULL. */
int tileqr_dist_plan_items(int64_t M, int64_t N, int NB, int IB, int nranks, int rank, int workers,
                           int sub_cols, int64_t* h_out, int64_t cap, int64_t* h_count);
/* Factor the distributed M x N matrix in place (NB = IB = 0: the decision
 * table at (order, nranks)); d_info as tileqr_factor.  Collective: every rank
 * calls it with the same arguments.  Errors: -1 M, -2 N, -3 A_local NULL,
 * -4 NB, -5 IB, -6 T_local NULL; -1 also for M != N on the levels path. */
int tileqr_dist_factor(int64_t M, int64_t N, double* A_local, int NB, int IB, double* T_local, int* d_info,
                       tileqr_stream_t stream);
void tileqr_dist_finalize(void);
/* B <- Q^T B on this rank's local tile columns (layout of A_local, padded as
 * tileqr_dist_fill_uniform pads) with the Q of the most recent DATAFLOW
 * tileqr_dist_factor of this (M, N, NB, IB) on this rank: panels k <= n on
 * local column n, from the packed reflector tiles the rank's slots hold (its
 * own panels, the pushed ones).  For the P > 1 residual check: Q^T A = R on
 * every rank's columns, ||Q^T A - R||_F = ||A - QR||_F, sums of squares
 * all-reduced (bench.py --verify).  Not collective.  Errors: -1 M, -2 N,
 * -3 B_local NULL, TILEQR_ERR_NOT_INIT without such a factorization. */
int tileqr_dist_apply_qt_local(int64_t M, int64_t N, double* B_local, int NB, int IB, tileqr_stream_t stream);
/* The dataflow multi-rank factorization with nranks EMULATED ranks on the
 * current GPU (one process, no NCCL): rank r's local columns in
 * h_A_local[r] / h_T_local[r] (device pointers, layout as above), the
 * packed-tile pushes of the COPY items going to the other ranks' buffers on
 * the same device.  Same work lists and kernel code as tileqr_dist_factor,
 * all ranks' items in one launch -- the way the multi-rank path is tested on
 * a single GPU.  Errors: -1 nranks, -2 M, -3 N, -4 NULL buffers, -5 NB/IB,
 * -6 (NB, IB) outside the dataflow set, -7 h_T_local NULL. */
int tileqr_dist_emulate(int nranks, int64_t M, int64_t N, double* const* h_A_local, int NB, int IB,
                        double* const* h_T_local, int* d_info, tileqr_stream_t stream);

/* ------------------------------------------------------------------------
 * Tall-skinny / communication-avoiding variant (
 * PAPER.md:840-850): the flat TSQRT chain of every panel is replaced by a
 * reduction tree -- tile rows in domains of BS consecutive rows [d*BS,
 * (d+1)*BS); per panel k each domain's first row >= k (its head) is factored
 * by GEQRT and joined by the domain's other rows through the flat TSQRT
 * chain; the heads are merged pairwise along a binary tree (distance 1, 2,
 * 4, ...) by TTQRT ("triangle on triangle"), applied to the trailing tiles
 * by TTMQRT (R20).  BS >= ceil(M/NB) is the flat tree.  Runs on the
 * persistent dataflow kernel: (NB, IB) in its set (NB % 32 == 0, NB <= 256,
 * IB in {8,16,24,32}).
 *   tileqr_factor_tree: as tileqr_factor; output A holds R, the GEQRT V of
 *     every head strictly below its diagonal, TSQRT V2 in full tiles, and the
 *     TTQRT V2 of a merged head in the upper triangle (diagonal included) of
 *     its tile; T holds tileqr_t_size_tree() = 2*MT*NT*IB*NB doubles: the
 *     GEQRT / TSQRT factors (tileqr_factor layout), then the TTQRT factors
 *     T2 (same offsets, tile (b,k) for the merged head b).
 *     Errors: -1 M, -2 N, -3 A, -4 lda, -5 NB/IB, -6 (NB, IB) outside the
 *     dataflow set, -7 BS < 1, -8 T.
 *   tileqr_apply_qt_tree: B <- Q^T B / Q B for that factorization (same NB,
 *     IB, BS): the operations replayed in order ('T') or backwards ('N').
 *     Errors: -1 trans, -2 M, -3 NRHS, -4 K, -5 A, -6 lda, -7 T, -8 NB/IB,
 *     -10 BS, -11 B, -12 ldb.
 *   tileqr_ttqrt_batched: QR of [R[i]; A2[i]], both upper triangular (LAPACK
 *     dtpqrt with L = NB): R's upper triangle updated, V2 in A2's upper
 *     triangle, T[i] (IB x NB); the strict lower parts of R[i] and A2[i] are
 *     neither read nor written.  Errors: -1 (NB, IB) unsupported, -3 batch,
 *     -4..-6 NULL arrays.
 * ------------------------------------------------------------------------ */
int tileqr_factor_tree(int64_t M, int64_t N, double* A, int64_t lda, int NB, int IB, int64_t BS, double* T,
                       int* d_info, tileqr_stream_t stream);
int tileqr_t_size_tree(int64_t M, int64_t N, int NB, int IB, size_t* n_doubles);
int tileqr_apply_qt_tree(char trans, int64_t M, int64_t NRHS, int64_t K, const double* A, int64_t lda,
                         const double* T, int NB, int IB, int64_t BS, double* B, int64_t ldb,
                         tileqr_stream_t stream);
int tileqr_ttqrt_batched(int NB, int IB, int batch, double* const* R, double* const* A2, double* const* T,
                         tileqr_stream_t stream);
/* The domain size BS as a tunable ("p domains"): times
 * tileqr_factor_tree on a seeded M x N matrix for BS = 1, 2, 4, ... and the
 * flat tree (BS = MT), 1 warm-up + 6 timed runs each, and returns the BS with
 * the smallest median in *h_BS (its median ms in *h_ms, nullable); the
 * report (nullable path) lists every median.  Synchronizes the device.
 * Errors: -1 M, -2 N, -3 (NB, IB) outside the dataflow set, -5 h_BS NULL. */
int tileqr_tune_tree(int64_t M, int64_t N, int NB, int IB, int64_t* h_BS, double* h_ms,
                     const char* report_json_path);
/* Host-only work list of the tree variant's dataflow kernel (its claim
 * order), for CPU tests of the derived task graph: per item 11 int64 (kind,
 * a, b, k, n, s, task, ndep, dep0, dep1, dep2) with kind 0 GEQRT(tile a; panel
 * k), 1 TSQRT(a <- b), 8 TTQRT(a <- b), 2 LARFB(a; column n), 3 SSRFB(a, b;
 * column n), 9 TTMQRT(a, b; column n); s = panel sub-task (inner panels of
 * columns [s*sub_cols, (s+1)*sub_cols)) or update slab.  workers: resident
 * CTAs in the schedule simulation.  *h_count = item count; h_out may be
 * NULL.  Errors: -1 M, -2 N, -3 NB/IB, -5 BS, -6 workers, -7 sub_cols,
 * -9 capacity, -10 h_count NULL. */
int tileqr_tree_plan_items(int64_t M, int64_t N, int NB, int IB, int64_t BS, int workers, int sub_cols,
                           int64_t* h_out, int64_t cap, int64_t* h_count);
/* Release the tree variant's cached workspaces. */
void tileqr_tree_finalize(void);

/* ------------------------------------------------------------------------
 * Utilities.
 * ------------------------------------------------------------------------ */
/* Synthetic input generator (same counter-based
 * generator as synth_inputs.uniform):
 *   A[i + j*lda] = (splitmix64(splitmix64(seed) + offset + i + j*M) >> 11)
 *                  * 2^-53 - 0.5 */
int tileqr_rng_uniform(int64_t M, int64_t N, double* A, int64_t lda, uint64_t seed,
                       uint64_t offset, tileqr_stream_t stream);

/* Name of the implementation tileqr_ssrfb_batched / tileqr_larfb_batched use
 * for this (NB, IB): "dmma" (FP64 tensor-core mma.sync path, NB % 32 == 0,
 * 32 <= NB <= 256) or "simt" (any NB <= 512). */
const char* tileqr_ssrfb_impl(int NB, int IB);

/* Static plan of tileqr_factor(M, N, NB, IB): h_out[8] = {levels, kernel
 * launches per call, #GEQRT, #TSQRT, #LARFB, #SSRFB tasks, MT, NT}. */
/* How tileqr_factor executes the DAG for this (NB, IB): "dag" = one
 * persistent dataflow kernel (NB % 32 == 0, NB <= 256, IB in {8,16,24,32};
 * environment TILEQR_SCHED=levels forces the other), "levels" = one batched
 * launch per kernel kind and DAG level, captured in a CUDA graph. */
const char* tileqr_factor_schedule(int NB, int IB);
int tileqr_factor_plan(int64_t M, int64_t N, int NB, int IB, int64_t* h_out);

/* Kernel timing for measurement (bench.py): bit k of `mask` (k = 0 GEQRT,
 * 1 TSQRT, 2 LARFB, 3 SSRFB) makes tileqr_factor bracket every batched launch
 * of that kind with CUDA events on the stream it is launched on (captured
 * into the CUDA graph as event-record nodes); 0 turns timing off.  Bit 4:
 * CUDA events around every dataflow-kernel launch only (no device-clock
 * trace), accumulated until read with kind 5 below. */
void tileqr_set_kernel_timing(int mask);
/* After the stream of a timed tileqr_factor(M, N, NB, IB) completed: sum of
 * the launch durations of kernel kind (0 GEQRT, 1 TSQRT, 2 LARFB, 3 SSRFB) in
 * the most recent run, the number of launches and of tasks.  Dataflow
 * schedule ("dag", tileqr_factor_schedule): kinds 0-3 give the busy time of
 * that kind's work items summed over CTAs (inputs ready -> completion), the
 * number of items and of tasks; kind 4 gives the dataflow kernel's duration
 * (CUDA events around its launch), h_launches = its resident CTAs and
 * h_tasks = the DAG's task count.  Kind 5 (timing bit 4): the summed
 * durations and the number of dataflow-kernel launches recorded since the
 * last kind-5 read (which resets them). */
int tileqr_kernel_times(int64_t M, int64_t N, int NB, int IB, int kind, double* h_total_ms,
                        int64_t* h_launches, int64_t* h_tasks);

/* Launch trace of the most recent timed tileqr_factor(M, N, NB, IB): for
 * up to max_recs timed launches, start/end in ms relative to the first timed
 * launch's start event, kernel kind, DAG level and task count (host arrays,
 * each nullable except h_count, which receives the number of records).
 * Dataflow schedule ("dag"): one record per work item in claim order, start
 * = inputs ready, end = completion published (device ns clock, relative to
 * the first claim), h_tasks = the item's claim time in ns. */
int tileqr_kernel_trace(int64_t M, int64_t N, int NB, int IB, int64_t max_recs, double* h_t0_ms,
                        double* h_t1_ms, int* h_kind, int64_t* h_level, int64_t* h_tasks,
                        int64_t* h_count);

/* Release all cached workspaces, graphs and communicators. */
void tileqr_finalize(void);

#ifdef __cplusplus
}
#endif

#endif /* TILEQR_H_ */
