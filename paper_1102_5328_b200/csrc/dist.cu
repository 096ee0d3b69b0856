// dist.cu -- multi-GPU tile QR: tile columns 1D block-cyclic over the ranks
// (one process per GPU), panel V/T tiles broadcast with NCCL over NVLink
// (J:north_star).
//
// Tile column n lives on rank n mod P, stored locally as MT tiles per local
// column (local column j <-> global n = rank + j*P).  The DAG levels are the
// single-GPU closed form (api.cu).  Per level t:
//   panel stream : GEQRT(k) [3k == t] and TSQRT(k,m) [2k+m == t] on owner(k)
//                  (their inputs are local: column k is owned by owner(k));
//                  the owner copies V_kk (whose upper part the next TSQRT
//                  rewrites) into its panel buffer.
//   comm stream  : after the level's panel kernels, ONE grouped set of
//                  ncclBroadcast calls, one per new V tile and T tile, from
//                  owner(k) into every rank's per-panel receive buffer
//                  pbuf[k][m-k] / pT[k][m-k] (written exactly once).
//   update stream: LARFB(k,n) [3k+1 == t] and SSRFB(k,m,n) [2k+m+1 == t] for
//                  the LOCAL columns n, reading V/T from the panel buffers;
//                  it waits for the broadcasts of level t-1, the panel stream
//                  of level t waits for the updates of level t-1.
// Every tile sees the same kernel sequence with the same inputs as in
// tileqr_factor, so R, V and T are bitwise identical for any P.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "dag_item.h"
#include "dist_dag.h"
#include "internal.h"

namespace tileqr {

int launch_dist_fill(int64_t M, int64_t N, int NB, int64_t MT, int nranks, int rank, int64_t nloc, double* A,
                     uint64_t seed, cudaStream_t s);
int launch_nonfinite_check(const double* A, int64_t n, int* d_info, cudaStream_t s);

namespace {

#define TQ_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      char b_[256];                                                                     \
      snprintf(b_, sizeof b_, "NCCL error %s in %s", ncclGetErrorString(r_), #call);    \
      set_error(b_);                                                                    \
      return TILEQR_ERR_NCCL;                                                           \
    }                                                                                   \
  } while (0)

// A planned task of one rank at one level.  kind: 0 GEQRT(k), 1 TSQRT(k,m),
// 2 LARFB(k,n), 3 SSRFB(k,m,n), 4 broadcast of V/T (k,m) from root.
struct Task {
  int kind;
  int64_t k, m, n;
  int root;
};

int64_t dist_levels(int64_t MT) { return MT <= 0 ? 0 : 3 * MT - 2; }

// Host plan of level t for `rank` (square MT x MT tile matrix).
void plan_level(int64_t MT, int P, int rank, int64_t t, std::vector<Task>& panel,
                std::vector<Task>& bcast, std::vector<Task>& update) {
  panel.clear();
  bcast.clear();
  update.clear();
  // panel tasks and the broadcasts they feed (same order on every rank)
  if (t % 3 == 0 && t / 3 < MT) {
    const int64_t k = t / 3;
    if ((int)(k % P) == rank) panel.push_back({0, k, k, k, (int)(k % P)});
    bcast.push_back({4, k, k, -1, (int)(k % P)});
  }
  for (int64_t k = 0; k < MT; ++k) {
    const int64_t m = t - 2 * k;
    if (m <= k) break;
    if (m >= MT) continue;
    if ((int)(k % P) == rank) panel.push_back({1, k, m, k, (int)(k % P)});
    bcast.push_back({4, k, m, -1, (int)(k % P)});
  }
  // update tasks on local columns
  if ((t - 1) % 3 == 0 && t >= 1) {
    const int64_t k = (t - 1) / 3;
    if (k < MT)
      for (int64_t n = k + 1; n < MT; ++n)
        if ((int)(n % P) == rank) update.push_back({2, k, k, n, -1});
  }
  for (int64_t k = 0; k < MT; ++k) {
    const int64_t m = t - 1 - 2 * k;
    if (m <= k) break;
    if (m >= MT) continue;
    for (int64_t n = k + 1; n < MT; ++n)
      if ((int)(n % P) == rank) update.push_back({3, k, m, n, -1});
  }
}

struct LevelPlan {
  // offsets into the device pointer array and counts, per level
  size_t oG, oT, oL, oS;
  int nG, nT, nL, nS;
  std::vector<Task> panel, bcast;  // host copies (owner snapshots + broadcasts)
};

struct DistState {
  bool init = false;
  int nranks = 0, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t sp = nullptr, su = nullptr, sc = nullptr;
  cudaEvent_t ep = nullptr, eu = nullptr, ec = nullptr, e0 = nullptr;
  // cached workspace of one shape
  int64_t N = -1;
  int NB = 0, IB = 0;
  double* A_cached = nullptr;
  double* T_cached = nullptr;
  double* pbuf = nullptr;  // V tiles of every panel: slot(k, m) = off(k) + (m - k)
  double* pT = nullptr;    // T tiles of every panel
  double* ppk = nullptr;   // packed reflector tiles (update_v2.cuh) of every panel, same slots
  bool v2 = false;
  size_t pk_dbl = 0;
  void** dptr = nullptr;   // all levels' pointer arrays
  std::vector<LevelPlan> plan;
};

DistState g_d;

// Multi-rank dataflow path (dist_dag.cu): this rank's work list, its slot and
// counter buffers, and the peers' slot / counter buffers mapped with cudaIpc.
struct DistDag {
  int64_t M = -1, N = -1;
  int NB = 0, IB = 0, SC = 0;
  double* A = nullptr;
  double* T = nullptr;
  std::shared_ptr<dd::Plan> plan;
  double* slots = nullptr;
  int* ctr = nullptr;   // [claim cursor | 256 | ntask counters]
  int* red = nullptr;   // barrier scratch
  std::vector<double*> peer_slots;
  std::vector<int*> peer_ctr;
  dag::Item* d_items = nullptr;
  int nitems = 0, nsm = 0;
  void release() {
    for (size_t r = 0; r < peer_slots.size(); ++r)
      if ((int)r != g_d.rank) {
        if (peer_slots[r]) cudaIpcCloseMemHandle(peer_slots[r]);
        if (peer_ctr[r]) cudaIpcCloseMemHandle(peer_ctr[r]);
      }
    peer_slots.clear();
    peer_ctr.clear();
    cudaFree(slots);
    cudaFree(ctr);
    cudaFree(red);
    cudaFree(d_items);
    slots = nullptr;
    ctr = red = nullptr;
    d_items = nullptr;
    plan.reset();
    M = N = -1;
  }
};
DistDag g_dd;

// Build (or reuse) this rank's dataflow work list for (M, N, NB, IB).
int dd_prepare(int64_t M, int64_t N, double* A_local, int NB, int IB, double* T_local, cudaStream_t s) {
  const int SC = panel_sub_cols(NB, IB);
  if (g_dd.plan && g_dd.M == M && g_dd.N == N && g_dd.NB == NB && g_dd.IB == IB && g_dd.SC == SC &&
      g_dd.A == A_local && g_dd.T == T_local)
    return 0;
  g_dd.release();
  const int P = g_d.nranks, me = g_d.rank;
  TQ_CUDA(cudaDeviceGetAttribute(&g_dd.nsm, cudaDevAttrMultiProcessorCount, g_d.device));
  int rc = dd::build_plan(M, N, NB, IB, P, g_dd.nsm * dag::dag_ctas_per_sm(NB), SC, &g_dd.plan);
  if (rc) return rc;
  const dd::Plan& p = *g_dd.plan;
  const size_t pkd = v2_pk_doubles(NB, IB);
  if (cudaMalloc(&g_dd.slots, std::max<size_t>(1, (size_t)p.nslots() * pkd) * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&g_dd.ctr, (size_t)(257 + p.ntask) * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&g_dd.red, 64 * P) != cudaSuccess) {
    cudaGetLastError();
    g_dd.release();
    set_error("tileqr_dist_factor: workspace allocation failed");
    return TILEQR_ERR_ALLOC;
  }
  g_dd.peer_slots.assign(P, nullptr);
  g_dd.peer_ctr.assign(P, nullptr);
  g_dd.peer_slots[me] = g_dd.slots;
  g_dd.peer_ctr[me] = g_dd.ctr;
  if (P > 1) {  // exchange the slot / counter buffers: cudaIpc handles all-gathered over NCCL
    cudaIpcMemHandle_t h[2];
    TQ_CUDA(cudaIpcGetMemHandle(&h[0], g_dd.slots));
    TQ_CUDA(cudaIpcGetMemHandle(&h[1], g_dd.ctr));
    char* d_h = nullptr;
    TQ_CUDA(cudaMalloc(&d_h, sizeof h * P));
    TQ_CUDA(cudaMemcpy(d_h + sizeof h * me, h, sizeof h, cudaMemcpyHostToDevice));
    ncclResult_t nr = ncclAllGather(d_h + sizeof h * me, d_h, sizeof h, ncclChar, g_d.comm, s);
    std::vector<cudaIpcMemHandle_t> all(2 * P);
    cudaError_t ce = nr == ncclSuccess ? cudaStreamSynchronize(s) : cudaSuccess;
    if (nr == ncclSuccess && ce == cudaSuccess)
      ce = cudaMemcpy(all.data(), d_h, sizeof h * P, cudaMemcpyDeviceToHost);
    cudaFree(d_h);
    if (nr != ncclSuccess) {
      g_dd.release();
      set_error(std::string("tileqr_dist_factor: handle exchange failed: ") + ncclGetErrorString(nr));
      return TILEQR_ERR_NCCL;
    }
    if (ce != cudaSuccess) { g_dd.release(); return cuda_fail(ce, "handle exchange", __FILE__, __LINE__); }
    for (int r = 0; r < P; ++r) {
      if (r == me) continue;
      void* ps = nullptr;
      void* pc = nullptr;
      cudaError_t e1 = cudaIpcOpenMemHandle(&ps, all[2 * r], cudaIpcMemLazyEnablePeerAccess);
      cudaError_t e2 = e1 == cudaSuccess ? cudaIpcOpenMemHandle(&pc, all[2 * r + 1], cudaIpcMemLazyEnablePeerAccess)
                                         : e1;
      g_dd.peer_slots[r] = static_cast<double*>(ps);
      g_dd.peer_ctr[r] = static_cast<int*>(pc);
      if (e2 != cudaSuccess) {
        g_dd.release();
        return cuda_fail(e2, "cudaIpcOpenMemHandle (peer slots / counters)", __FILE__, __LINE__);
      }
    }
  }
  std::vector<dd::RankBufs> bufs(P);
  for (int r = 0; r < P; ++r)
    bufs[r] = {r == me ? A_local : nullptr, r == me ? T_local : nullptr, g_dd.peer_slots[r], g_dd.peer_ctr[r] + 257};
  std::vector<dag::Item> items;
  rc = dd::emit_items(p, me, bufs, false, &items);
  if (rc) { g_dd.release(); return rc; }
  g_dd.nitems = (int)items.size();
  if (cudaMalloc(&g_dd.d_items, std::max<size_t>(1, items.size()) * sizeof(dag::Item)) != cudaSuccess) {
    cudaGetLastError();
    g_dd.release();
    set_error("tileqr_dist_factor: work list allocation failed");
    return TILEQR_ERR_ALLOC;
  }
  TQ_CUDA(cudaMemcpy(g_dd.d_items, items.data(), items.size() * sizeof(dag::Item), cudaMemcpyHostToDevice));
  g_dd.M = M; g_dd.N = N; g_dd.NB = NB; g_dd.IB = IB; g_dd.SC = SC;
  g_dd.A = A_local; g_dd.T = T_local;
  return 0;
}

// The dataflow factorization of this rank's columns: counters zeroed, a
// barrier (every rank's counters are zero before any peer pushes into them),
// then the persistent kernel.  No collective on the data path.
int dd_factor(int64_t M, int64_t N, double* A_local, int NB, int IB, double* T_local, int* d_info, cudaStream_t s) {
  int rc = dd_prepare(M, N, A_local, NB, IB, T_local, s);
  if (rc) return rc;
  const dd::Plan& p = *g_dd.plan;
  const int64_t nloc = dd::local_cols(p.NT, g_d.nranks, g_d.rank);
  if (nloc > 0 && d_info) {
    rc = launch_nonfinite_check(A_local, nloc * p.MT * NB * (int64_t)NB, d_info, s);
    if (rc) return rc;
  }
  TQ_CUDA(cudaMemsetAsync(g_dd.ctr, 0, (size_t)(257 + p.ntask) * sizeof(int), s));
  if (g_d.nranks > 1) TQ_NCCL(ncclAllReduce(g_dd.red, g_dd.red, 1, ncclInt, ncclSum, g_d.comm, s));
  int grid = 0;
  return launch_dag(NB, IB, g_dd.d_items, g_dd.nitems, g_dd.ctr, g_dd.ctr + 257, g_dd.nsm, nullptr, s, &grid,
                    nullptr, dag::kModeDist);
}

bool dist_dataflow(int NB, int IB) {
  const char* e = getenv("TILEQR_DIST_SCHED");
  if (e && strcmp(e, "levels") == 0) return false;
  return dag_path_supported(NB, IB);
}

int64_t slot_off(int64_t MT, int64_t k) { return k * MT - k * (k - 1) / 2; }

void free_shape() {
  cudaFree(g_d.pbuf);
  cudaFree(g_d.pT);
  cudaFree(g_d.ppk);
  g_d.ppk = nullptr;
  cudaFree(g_d.dptr);
  g_d.pbuf = nullptr;
  g_d.pT = nullptr;
  g_d.dptr = nullptr;
  g_d.plan.clear();
  g_d.N = -1;
}

}  // namespace

// ---- collectives for tileqr_tune (ngpus > 1), over the library's comm -----
int dist_ranks(int* nranks, int* rank) {
  if (!g_d.init) {
    set_error("tileqr_dist_init not called");
    return TILEQR_ERR_NOT_INIT;
  }
  *nranks = g_d.nranks;
  *rank = g_d.rank;
  return 0;
}

// op 0: broadcast h[0:n] from rank 0; op 1: element-wise max over ranks.
int dist_host_collective(double* h, int n, int op) {
  if (!g_d.init) return TILEQR_ERR_NOT_INIT;
  if (n <= 0) return 0;
  double* d = nullptr;
  TQ_CUDA(cudaMalloc(&d, n * sizeof(double)));
  cudaStream_t s = g_d.sc;
  int rc = 0;
  cudaError_t e = cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, s);
  ncclResult_t r = ncclSuccess;
  if (e == cudaSuccess)
    r = op == 0 ? ncclBroadcast(d, d, n, ncclDouble, 0, g_d.comm, s)
                : ncclAllReduce(d, d, n, ncclDouble, ncclMax, g_d.comm, s);
  if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (r != ncclSuccess) {
    set_error(std::string("tileqr_tune: NCCL collective failed: ") + ncclGetErrorString(r));
    rc = TILEQR_ERR_NCCL;
  } else if (e != cudaSuccess) {
    rc = cuda_fail(e, "tileqr_tune collective", __FILE__, __LINE__);
  }
  return rc;
}

}  // namespace tileqr

using namespace tileqr;

extern "C" {

int tileqr_dist_unique_id(void* h_id) {
  if (!h_id) return -1;
  ncclUniqueId id;
  TQ_NCCL(ncclGetUniqueId(&id));
  memcpy(h_id, &id, sizeof id);
  return 0;
}

int tileqr_dist_init(int nranks, int rank, const void* h_nccl_unique_id, int device) {
  if (nranks < 1) return -1;
  if (rank < 0 || rank >= nranks) return -2;
  if (!h_nccl_unique_id) return -3;
  if (device < 0) return -4;
  if (g_d.init) tileqr_dist_finalize();
  TQ_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, h_nccl_unique_id, sizeof id);
  TQ_NCCL(ncclCommInitRank(&g_d.comm, nranks, id, rank));
  int lo = 0, hi = 0;
  TQ_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  TQ_CUDA(cudaStreamCreateWithPriority(&g_d.sp, cudaStreamNonBlocking, hi));
  TQ_CUDA(cudaStreamCreateWithPriority(&g_d.su, cudaStreamNonBlocking, lo));
  TQ_CUDA(cudaStreamCreateWithPriority(&g_d.sc, cudaStreamNonBlocking, hi));
  for (cudaEvent_t* e : {&g_d.ep, &g_d.eu, &g_d.ec, &g_d.e0})
    TQ_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  g_d.nranks = nranks;
  g_d.rank = rank;
  g_d.device = device;
  g_d.init = true;
  return 0;
}

int tileqr_dist_local_cols(int64_t N, int NB, int* n_local) {
  if (N < 0) return -1;
  if (NB < 1 || NB > 512) return -2;
  if (!n_local) return -3;
  if (!g_d.init) {
    set_error("tileqr_dist_local_cols: tileqr_dist_init not called");
    return TILEQR_ERR_NOT_INIT;
  }
  const int64_t NT = (N + NB - 1) / NB;
  *n_local = (int)((NT - g_d.rank + g_d.nranks - 1) / g_d.nranks);
  if (NT <= g_d.rank) *n_local = 0;
  return 0;
}

int tileqr_dist_fill_uniform(int64_t M, int64_t N, int NB, double* A_local, uint64_t seed,
                             tileqr_stream_t stream) {
  if (M < 0) return -1;
  if (N < 0) return -2;
  if (NB < 1 || NB > 512) return -3;
  if (!g_d.init) {
    set_error("tileqr_dist_fill_uniform: tileqr_dist_init not called");
    return TILEQR_ERR_NOT_INIT;
  }
  int nloc = 0;
  int rc = tileqr_dist_local_cols(N, NB, &nloc);
  if (rc) return rc;
  if (nloc == 0 || N == 0 || M == 0) return 0;
  if (!A_local) return -4;
  const int64_t MT = (M + NB - 1) / NB;
  return launch_dist_fill(M, N, NB, MT, g_d.nranks, g_d.rank, nloc, A_local, seed,
                          reinterpret_cast<cudaStream_t>(stream));
}

// Host-only plan of one level, exported for CPU tests of the schedule:
// writes tuples (kind, k, m, n, root) for the panel tasks, then the broadcast
// items, then the update tasks of `rank`; counts in h_counts[3].
int tileqr_dist_plan_level(int64_t MT, int nranks, int rank, int64_t level, int64_t* h_out,
                           int64_t cap, int64_t* h_counts) {
  if (MT < 0) return -1;
  if (nranks < 1) return -2;
  if (rank < 0 || rank >= nranks) return -3;
  if (level < 0) return -4;
  if (!h_counts) return -7;
  std::vector<Task> p, b, u;
  plan_level(MT, nranks, rank, level, p, b, u);
  h_counts[0] = (int64_t)p.size();
  h_counts[1] = (int64_t)b.size();
  h_counts[2] = (int64_t)u.size();
  const int64_t need = 5 * (int64_t)(p.size() + b.size() + u.size());
  if (need > cap || (!h_out && need > 0)) return -6;
  int64_t o = 0;
  for (auto* v : {&p, &b, &u})
    for (const Task& t : *v) {
      h_out[o++] = t.kind;
      h_out[o++] = t.k;
      h_out[o++] = t.m;
      h_out[o++] = t.n;
      h_out[o++] = t.root;
    }
  return 0;
}

int tileqr_dist_factor(int64_t M, int64_t N, double* A_local, int NB, int IB, double* T_local, int* d_info,
                       tileqr_stream_t stream) {
  if (M < 0) return -1;
  if (N < 0) return -2;
  if (!g_d.init) {
    set_error("tileqr_dist_factor: tileqr_dist_init not called");
    return TILEQR_ERR_NOT_INIT;
  }
  if (NB == 0 && IB == 0) {  // the installed decision table at (order, nranks)
    bool f = false;
    lookup_pair(M, N, g_d.nranks, &NB, &IB, &f);
  }
  if (NB < 1 || NB > 512) return -4;
  if (IB < 1 || IB > NB || NB % IB) return -5;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_info) {
    int rc = launch_zero_int(d_info, s);
    if (rc) return rc;
  }
  if (M == 0 || N == 0) return 0;
  int nloc0 = 0;
  tileqr_dist_local_cols(N, NB, &nloc0);
  if (nloc0 > 0 && !A_local) return -3;
  if (nloc0 > 0 && !T_local) return -6;
  // the inner blocking tileqr_factor runs (R23), so that the result
  // is bitwise the single-GPU one: the factorization at IBe into a scratch T,
  // then T at IB (its diagonal blocks, or assembled from the local V tiles)
  if (const int IBe = effective_ib(NB, IB); IBe != IB) {
    const int64_t MTl = (M + NB - 1) / NB, KT = std::min(MTl, (N + NB - 1) / NB);
    double* te = nullptr;
    if (int rc = stream_alloc(reinterpret_cast<void**>(&te), (size_t)std::max(1, nloc0) * MTl * IBe * NB * sizeof(double), s))
      return rc;
    int rc = tileqr_dist_factor(M, N, A_local, NB, IBe, te, d_info, stream);
    if (!rc && IBe > IB) rc = launch_t_extract(te, IBe, T_local, IB, NB, MTl * nloc0, s);
    if (!rc && IBe < IB) {
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      if (cudaMemsetAsync(T_local, 0, (size_t)MTl * nloc0 * IB * NB * sizeof(double), s) != cudaSuccess) {
        rc = TILEQR_ERR_CUDA;
        set_error("tileqr_dist_factor: memset failed");
      } else {
        rc = launch_t_assemble_big(A_local, te, T_local, NB, IB, IBe, MTl, nloc0, KT, g_d.nranks, g_d.rank, nsm, s);
      }
    }
    cudaFreeAsync(te, s);
    return rc;
  }
  if (dist_dataflow(NB, IB)) return dd_factor(M, N, A_local, NB, IB, T_local, d_info, s);
  if (M != N) {
    set_error("tileqr_dist_factor: the level-synchronous (NCCL broadcast) path is square only");
    return -1;
  }
  const int P = g_d.nranks, me = g_d.rank;
  const int64_t MT = (N + NB - 1) / NB;
  int nloc = 0;
  tileqr_dist_local_cols(N, NB, &nloc);
  const size_t tile = (size_t)NB * NB, ttile = (size_t)IB * NB;
  auto loc = [&](int64_t m, int64_t n) { return A_local + (size_t)(m + (n / P) * MT) * tile; };
  auto locT = [&](int64_t m, int64_t n) { return T_local + (size_t)(m + (n / P) * MT) * ttile; };
  auto pv = [&](int64_t k, int64_t m) { return g_d.pbuf + (size_t)(slot_off(MT, k) + (m - k)) * tile; };
  auto pt = [&](int64_t k, int64_t m) { return g_d.pT + (size_t)(slot_off(MT, k) + (m - k)) * ttile; };
  auto pp = [&](int64_t k, int64_t m) { return g_d.ppk + (size_t)(slot_off(MT, k) + (m - k)) * g_d.pk_dbl; };
  const int64_t nlev = dist_levels(MT);

  // ---- per-shape workspace: panel buffers and every level's pointer arrays ----
  if (g_d.N != N || g_d.NB != NB || g_d.IB != IB || g_d.A_cached != A_local || g_d.T_cached != T_local) {
    free_shape();
    const int64_t nslots = slot_off(MT, MT);
    // packed path (as tileqr_factor): panel kernels write the packed reflector
    // tile into the slot, which is what gets broadcast and what updates read
    g_d.v2 = v2_supported(NB, IB);
    g_d.pk_dbl = g_d.v2 ? v2_pk_doubles(NB, IB) : 0;
    if ((g_d.v2 && cudaMalloc(&g_d.ppk, nslots * g_d.pk_dbl * sizeof(double)) != cudaSuccess) ||
        (!g_d.v2 && cudaMalloc(&g_d.pbuf, nslots * tile * sizeof(double)) != cudaSuccess) ||
        (!g_d.v2 && cudaMalloc(&g_d.pT, nslots * ttile * sizeof(double)) != cudaSuccess)) {
      cudaGetLastError();
      free_shape();
      set_error("tileqr_dist_factor: panel buffer allocation failed");
      return TILEQR_ERR_ALLOC;
    }
    std::vector<void*> hp;
    std::vector<Task> panel, bc, upd;
    g_d.plan.resize(nlev);
    for (int64_t t = 0; t < nlev; ++t) {
      plan_level(MT, P, me, t, panel, bc, upd);
      LevelPlan& L = g_d.plan[t];
      L.panel = panel;
      L.bcast = bc;
      std::vector<void*> gA, gT, gP, tR, tA, tT, tP, lV, lT, lC, lP, sV, sT, s1, s2, sP;
      const bool v2 = g_d.v2;
      for (const Task& q : panel) {
        if (q.kind == 0) {
          gA.push_back(loc(q.k, q.k)); gT.push_back(locT(q.k, q.k)); gP.push_back(v2 ? pp(q.k, q.k) : nullptr);
        } else {
          tR.push_back(loc(q.k, q.k)); tA.push_back(loc(q.m, q.k)); tT.push_back(locT(q.m, q.k));
          tP.push_back(v2 ? pp(q.k, q.m) : nullptr);
        }
      }
      for (const Task& q : upd) {
        if (q.kind == 2) {
          lV.push_back(v2 ? nullptr : pv(q.k, q.k)); lT.push_back(v2 ? nullptr : pt(q.k, q.k));
          lC.push_back(loc(q.k, q.n)); lP.push_back(v2 ? pp(q.k, q.k) : nullptr);
        } else {
          sV.push_back(v2 ? nullptr : pv(q.k, q.m)); sT.push_back(v2 ? nullptr : pt(q.k, q.m));
          s1.push_back(loc(q.k, q.n)); s2.push_back(loc(q.m, q.n)); sP.push_back(v2 ? pp(q.k, q.m) : nullptr);
        }
      }
      auto put = [&](std::vector<void*>& v) { size_t o = hp.size(); hp.insert(hp.end(), v.begin(), v.end()); return o; };
      L.nG = (int)gA.size(); L.oG = put(gA); put(gT); put(gP);
      L.nT = (int)tR.size(); L.oT = put(tR); put(tA); put(tT); put(tP);
      L.nL = (int)lV.size(); L.oL = put(lV); put(lT); put(lC); put(lP);
      L.nS = (int)sV.size(); L.oS = put(sV); put(sT); put(s1); put(s2); put(sP);
    }
    if (cudaMalloc(&g_d.dptr, std::max<size_t>(hp.size(), 1) * sizeof(void*)) != cudaSuccess) {
      cudaGetLastError();
      free_shape();
      set_error("tileqr_dist_factor: task list allocation failed");
      return TILEQR_ERR_ALLOC;
    }
    TQ_CUDA(cudaMemcpy(g_d.dptr, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice));
    g_d.N = N;
    g_d.NB = NB;
    g_d.IB = IB;
    g_d.A_cached = A_local;
    g_d.T_cached = T_local;
  }
  if (nloc > 0 && d_info) {
    int rc = launch_nonfinite_check(A_local, (int64_t)nloc * MT * tile, d_info, s);
    if (rc) return rc;
  }

  // the three internal streams start after the caller's prior work
  TQ_CUDA(cudaEventRecord(g_d.e0, s));
  for (cudaStream_t st : {g_d.sp, g_d.su, g_d.sc}) TQ_CUDA(cudaStreamWaitEvent(st, g_d.e0, 0));
  double** d = reinterpret_cast<double**>(g_d.dptr);
  for (int64_t t = 0; t < nlev; ++t) {
    const LevelPlan& L = g_d.plan[t];
    // panel(t) after update(t-1); update(t) after the broadcasts of level t-1
    if (t > 0) {
      TQ_CUDA(cudaEventRecord(g_d.eu, g_d.su));
      TQ_CUDA(cudaStreamWaitEvent(g_d.sp, g_d.eu, 0));
      TQ_CUDA(cudaEventRecord(g_d.ec, g_d.sc));
      TQ_CUDA(cudaStreamWaitEvent(g_d.su, g_d.ec, 0));
    }
    int rc;
    // ---- panel kernels on the owner, snapshot of V_kk into its panel slot ----
    const bool v2 = g_d.v2;
    if (L.nG && (rc = launch_geqrt(NB, IB, L.nG, d + L.oG, d + L.oG + L.nG, g_d.sp, v2 ? d + L.oG + 2 * L.nG : nullptr)))
      return rc;
    if (L.nT && (rc = launch_tsqrt(NB, IB, L.nT, d + L.oT, d + L.oT + L.nT, d + L.oT + 2 * L.nT, g_d.sp,
                                   v2 ? d + L.oT + 3 * L.nT : nullptr)))
      return rc;
    if (!v2)
      for (const Task& q : L.panel)
        if (q.kind == 0)  // before TSQRT(k, k+1) rewrites the upper part of tile (k, k)
          TQ_CUDA(cudaMemcpyAsync(pv(q.k, q.k), loc(q.k, q.k), tile * sizeof(double),
                                  cudaMemcpyDeviceToDevice, g_d.sp));
    // ---- one grouped broadcast of this level's new V/T tiles -----------------
    if (!L.bcast.empty()) {
      TQ_CUDA(cudaEventRecord(g_d.ep, g_d.sp));
      TQ_CUDA(cudaStreamWaitEvent(g_d.sc, g_d.ep, 0));
      TQ_NCCL(ncclGroupStart());
      for (const Task& q : L.bcast) {
        if (v2) {  // the packed tile (V and T) in its slot, in place on the root
          TQ_NCCL(ncclBroadcast(pp(q.k, q.m), pp(q.k, q.m), g_d.pk_dbl, ncclDouble, q.root, g_d.comm, g_d.sc));
          continue;
        }
        const bool root = q.root == me;
        const double* sv = root ? (q.m == q.k ? pv(q.k, q.k) : loc(q.m, q.k)) : pv(q.k, q.m);
        const double* st = root ? locT(q.m, q.k) : pt(q.k, q.m);
        TQ_NCCL(ncclBroadcast(sv, pv(q.k, q.m), tile, ncclDouble, q.root, g_d.comm, g_d.sc));
        TQ_NCCL(ncclBroadcast(st, pt(q.k, q.m), ttile, ncclDouble, q.root, g_d.comm, g_d.sc));
      }
      TQ_NCCL(ncclGroupEnd());
    }
    // ---- update kernels on the local columns ---------------------------------
    if (v2) {
      if (L.nL && (rc = launch_update_pk(true, NB, IB, L.nL, d + L.oL + 3 * L.nL, nullptr, d + L.oL + 2 * L.nL,
                                         g_d.su)))
        return rc;
      if (L.nS && (rc = launch_update_pk(false, NB, IB, L.nS, d + L.oS + 4 * L.nS, d + L.oS + 2 * L.nS,
                                         d + L.oS + 3 * L.nS, g_d.su)))
        return rc;
      continue;
    }
    if (L.nL && (rc = launch_larfb(true, NB, IB, L.nL, d + L.oL, d + L.oL + L.nL, d + L.oL + 2 * L.nL, NB, g_d.su)))
      return rc;
    if (L.nS && (rc = launch_ssrfb(true, NB, IB, L.nS, d + L.oS, d + L.oS + L.nS, d + L.oS + 2 * L.nS,
                                   d + L.oS + 3 * L.nS, NB, g_d.su)))
      return rc;
  }
  // join into the caller's stream
  for (cudaStream_t st : {g_d.sp, g_d.su, g_d.sc}) {
    TQ_CUDA(cudaEventRecord(g_d.e0, st));
    TQ_CUDA(cudaStreamWaitEvent(s, g_d.e0, 0));
  }
  return 0;
}

// B <- Q^T B for this rank's local tile columns of an M x N matrix (same
// layout as A_local), with the Q of the most recent dataflow
// tileqr_dist_factor of that shape: panels k <= n applied to local column n
// (LARFB(k, n), then SSRFB(k, m, n) for m ascending), reading the packed
// reflector tiles this rank's slots hold after the factorization (its own
// panels and the pushed ones).  Panels k > n act on rows where Q^T a_n is
// zero and are not applied.  Used for the P > 1 residual check
// ||Q^T A - R||_F (= ||A - QR||_F): every rank applies Q^T to its pristine
// columns and compares with its R tiles; the sum of squares is all-reduced.
int tileqr_dist_apply_qt_local(int64_t M, int64_t N, double* B_local, int NB, int IB, tileqr_stream_t stream) {
  if (M < 1) return -1;
  if (N < 1) return -2;
  if (!g_d.init) {
    set_error("tileqr_dist_apply_qt_local: tileqr_dist_init not called");
    return TILEQR_ERR_NOT_INIT;
  }
  if (!g_dd.plan || g_dd.M != M || g_dd.N != N || g_dd.NB != NB || g_dd.IB != IB) {
    set_error("tileqr_dist_apply_qt_local: no dataflow factorization of this shape on this rank");
    return TILEQR_ERR_NOT_INIT;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const dd::Plan& p = *g_dd.plan;
  const int P = g_d.nranks, me = g_d.rank;
  const int64_t MT = p.MT, NT = p.NT, KT = p.KT;
  const size_t tile = (size_t)NB * NB, pkd = v2_pk_doubles(NB, IB);
  if (dd::local_cols(NT, P, me) == 0) return 0;
  if (!B_local) return -3;
  auto bt = [&](int64_t m, int64_t n) { return (void*)(B_local + (size_t)(m + (n / P) * MT) * tile); };
  auto sl = [&](int64_t k, int64_t m) { return (void*)(g_dd.slots + (size_t)p.slot(k, m) * pkd); };
  struct L { bool larfb; size_t off; int cnt; };
  std::vector<L> seq;
  std::vector<void*> hp;
  for (int64_t k = 0; k < KT; ++k) {
    std::vector<int64_t> cols;
    for (int64_t n = k; n < NT; ++n)
      if (p.owner(n) == me) cols.push_back(n);
    if (cols.empty()) continue;
    const int c = (int)cols.size();
    seq.push_back({true, hp.size(), c});  // [Pk | C1 (unused) | C2]
    for (int64_t n : cols) hp.push_back(sl(k, k));
    for (int64_t n : cols) hp.push_back(nullptr), (void)n;
    for (int64_t n : cols) hp.push_back(bt(k, n));
    for (int64_t m = k + 1; m < MT; ++m) {
      seq.push_back({false, hp.size(), c});
      for (int64_t n : cols) hp.push_back(sl(k, m)), (void)n;
      for (int64_t n : cols) hp.push_back(bt(k, n));
      for (int64_t n : cols) hp.push_back(bt(m, n));
    }
  }
  void** dp = nullptr;
  if (int rc = stream_alloc(reinterpret_cast<void**>(&dp), std::max<size_t>(1, hp.size()) * sizeof(void*), s)) return rc;
  TQ_CUDA(cudaMemcpyAsync(dp, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice, s));
  TQ_CUDA(cudaStreamSynchronize(s));  // hp is a host temporary
  int rc = 0;
  double** d = reinterpret_cast<double**>(dp);
  for (const L& l : seq) {
    rc = launch_update_pk(l.larfb, NB, IB, l.cnt, (const double* const*)(d + l.off), d + l.off + l.cnt,
                          d + l.off + 2 * l.cnt, s);
    if (rc) break;
  }
  cudaFreeAsync(dp, s);
  return rc;
}

void tileqr_dist_finalize(void) {
  if (!g_d.init) return;
  cudaDeviceSynchronize();
  g_dd.release();
  free_shape();
  if (g_d.comm) ncclCommDestroy(g_d.comm);
  for (cudaStream_t st : {g_d.sp, g_d.su, g_d.sc})
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t e : {g_d.ep, g_d.eu, g_d.ec, g_d.e0})
    if (e) cudaEventDestroy(e);
  g_d.comm = nullptr;
  g_d.sp = g_d.su = g_d.sc = nullptr;
  g_d.ep = g_d.eu = g_d.ec = g_d.e0 = nullptr;
  g_d.A_cached = g_d.T_cached = nullptr;
  g_d.init = false;
}

}  // extern "C"
