// dag_item.h -- work-item descriptor of the dataflow DAG kernel (dag.cuh),
// built on the host by api.cu.
#pragma once

namespace tileqr {
namespace dag {

// CTA geometry of the DAG kernel.  NB <= 128 (packed-reflector update with a
// shared-memory ring): 2 CTAs of 4 warps per SM, so one CTA's item prologue,
// epilogue and dependency waits overlap the other's DMMA work.  NB > 128:
// 1 CTA of 8 warps per SM.
#ifdef TILEQR_DAG_ONE_CTA  // build variant: one 8-warp CTA per SM for every NB
__host__ __device__ constexpr int dag_warps(int) { return 8; }
__host__ __device__ constexpr int dag_ctas_per_sm(int) { return 1; }
#else
__host__ __device__ constexpr int dag_warps(int NB) { return NB <= 128 ? 4 : 8; }
__host__ __device__ constexpr int dag_ctas_per_sm(int NB) { return NB <= 128 ? 2 : 1; }
#endif

enum Kind { kGeqrt = 0, kTsqrt = 1, kLarfb = 2, kSsrfb = 3, kLoad = 4, kStore = 5,
            kArrive = 6,  // host-only pseudo task: completed by a copy engine / a peer, not by a CTA
            kCopy = 7,    // multi-rank dataflow: push a packed reflector tile to a peer rank
            kTtqrt = 8,   // tree variant (f3): TTQRT sub-task (p: R_a, R_b, T2)
            kTtmqr = 9 }; // tree variant: TTMQRT column slab (p: -, -, C1, C2)

// Kernel instantiations of the dataflow kernel (dag.cuh): the device-only
// factorization, the host-buffer pipeline (LOAD / STORE items) and the
// multi-rank dataflow factorization (COPY items, system-scope signals).
enum Mode { kModePlain = 0, kModeIO = 1, kModeDist = 2, kModeTree = 3,
            kModePlainRetire = 4 };  // kModePlain + tail retirement (dag.cuh), for DAGs whose tail is a visible share

// One work item: a whole panel task, or a column slab of an update task.
struct Item {
  int kind;
  int task;      // completion counter index
  int col0;      // LARFB / SSRFB: first column of the slab; GEQRT / TSQRT: the
                 // sub-task's inner-panel columns [col0 & 0xffff, col0 >> 16)
  int ndep;
  int dep[3];    // tasks whose counters must reach need[] before the item runs
  int need[3];   // required counts; negative (-count) in the multi-rank kernel: the counter
                 // is written by a peer GPU, so it is acquired at system scope
  double* p[4];  // GEQRT: A, -, T; TSQRT: R, A2, T; LARFB: V, T, C; SSRFB: V2, T, C1, C2
  double* pk;    // packed reflector tile (NB <= 128): written by GEQRT/TSQRT, read by LARFB/SSRFB
  int aux[4];    // COPY: aux[0] = doubles to push from p[0] to p[1], then +1 on the peer counter (int*)p[2];
                 // LOAD / STORE (host-buffer pipeline): tile column n, tile rows [aux[1], aux[2]);
                 // LARFB / SSRFB: aux[0] = column limit in the tile (N - n*NB, at most NB):
                 // the columns past it are padding, which every update leaves exactly as is;
                 // SSRFB: aux[1] = rows of C2's tile above M when that tile holds padding
                 // rows (V2 is zero there: those rows are skipped), else 0 (all NB rows)
};

// aux[1] of SSRFB(k, m, n): rows of tile row m that are inside the matrix, or
// 0 when all NB are
inline int ssrfb_rows(long long M, long long m, int NB) {
  const long long r = M - m * NB;
  return (r > 0 && r < NB) ? (int)r : 0;
}

// Host-buffer pipeline of tileqr_factor_host: LOAD items convert a tile
// column that the copy engine has landed in a column-major staging buffer
// into tiles; STORE items convert a finished tile column back for the
// device-to-host copy.
struct DagIO {
  long long M, N, ld;   // matrix and staging leading dimension
  const double* in;     // column-major input staging (device)
  double* out;          // column-major output staging (device)
  int* info;            // non-finite flag
  long long MT;         // tile rows of the workspace
  double* tiles;        // tile workspace
};

// Update columns per item for tile order NB: warps x 8*MB columns.
__host__ __device__ constexpr int dag_mb(int NB) { return (NB == 96 || NB == 128) ? 2 : 1; }
__host__ __device__ constexpr int dag_cols(int NB) { return dag_warps(NB) * 8 * dag_mb(NB); }

// DAG kernel supported for these (NB, IB): the fast panel set.
inline bool dag_supported(int NB, int IB) {
  return NB % 32 == 0 && NB >= 32 && NB <= 256 && IB % 8 == 0 && IB >= 8 && IB <= 32;
}

}  // namespace dag
}  // namespace tileqr
