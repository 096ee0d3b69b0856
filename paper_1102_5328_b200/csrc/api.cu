// api.cu -- C ABI of libtileqr (include/tileqr.h): argument checking, error
// model, per-shape workspaces, and the wavefront (DAG-level) launcher of the
// tile QR factorization.
//
// The DAG of the flat-tree tile QR (Fig. 1b) is executed
// level by level.  Every task is placed at its ASAP level, which has the
// closed form (checked against an explicit dependency DP in
// tests): GEQRT(k) = 3k, LARFB(k,n) = 3k+1, TSQRT(k,m) = 2k+m,
// SSRFB(k,m,n) = 2k+m+1, so an MT x NT matrix has 3*min(MT,NT)-2 (+ the tail
// of a tall matrix) levels.  All tasks of one kind at one level are
// independent and run as ONE batched launch; the panel kernels (GEQRT, TSQRT)
// and the update kernels (LARFB, SSRFB) of a level run concurrently on two
// streams.  The whole level sequence is captured once per shape into a CUDA
// graph and replayed (the GPU counterpart of PLASMA's static schedule,
// PAPER.md:163-164).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "dag_item.h"
#include "internal.h"
#include "sched.h"

namespace tileqr {

#define TQ_DECL_DAG(nb)                                                                        \
  int launch_dag_nb##nb(int IB, const dag::Item* items, int nitems, int* next, int* done, int nsm, \
                        unsigned long long* prof, cudaStream_t s, int* grid_out, const dag::DagIO* io, int mode);
TQ_DECL_DAG(32) TQ_DECL_DAG(64) TQ_DECL_DAG(96) TQ_DECL_DAG(128) TQ_DECL_DAG(160) TQ_DECL_DAG(192)
TQ_DECL_DAG(224) TQ_DECL_DAG(256)
#undef TQ_DECL_DAG

int launch_dag(int NB, int IB, const dag::Item* items, int nitems, int* next, int* done, int nsm,
               unsigned long long* prof, cudaStream_t s, int* grid_out, const dag::DagIO* io, int mode) {
  switch (NB) {
    case 32: return launch_dag_nb32(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 64: return launch_dag_nb64(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 96: return launch_dag_nb96(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 128: return launch_dag_nb128(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 160: return launch_dag_nb160(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 192: return launch_dag_nb192(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 224: return launch_dag_nb224(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 256: return launch_dag_nb256(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    default: return TILEQR_ERR_CUDA;
  }
}

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
           cudaGetErrorString(e), what, file, line);
  set_error(buf);
  return TILEQR_ERR_CUDA;
}

int stream_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  TQ_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), dev) == done.end()) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
      done.push_back(dev);
    }
  }
  TQ_CUDA(cudaMallocAsync(p, bytes, s));
  return 0;
}

static int arg_error(int i, const char* fn, const char* what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: illegal argument %d (%s)", fn, i, what);
  set_error(buf);
  return -i;
}

// ---------------------------------------------------------------------------
// Level schedule (closed form) and task lists
// ---------------------------------------------------------------------------
struct LevelLists {
  int64_t nlev = 0;
  // per level: offset/count into each kind's flat arrays; the first lc_cnt /
  // sc_cnt LARFB / SSRFB tasks of a level are "critical" (they update tile
  // column k+1, the next panel) and run on the panel stream
  std::vector<int64_t> g_off, g_cnt, t_off, t_cnt, l_off, l_cnt, s_off, s_cnt, lc_cnt, sc_cnt;
};

static int64_t num_levels(int64_t MT, int64_t NT) {
  const int64_t KT = std::min(MT, NT);
  if (KT <= 0) return 0;
  int64_t last = 0;
  for (int64_t k = 0; k < KT; ++k) {
    last = std::max(last, 3 * k);                              // G
    if (NT > k + 1) last = std::max(last, 3 * k + 1);          // L
    if (MT > k + 1) last = std::max(last, 2 * k + MT - 1);     // T(k, MT-1)
    if (MT > k + 1 && NT > k + 1) last = std::max(last, 2 * k + MT);  // S(k, MT-1, .)
  }
  return last + 1;
}

// Host-side task lists in tile-index form; materialised to device pointers.
struct HostTasks {
  std::vector<std::vector<int64_t>> G, T, L, S;  // per level: flattened tuples
  std::vector<int64_t> Lc, Sc;                   // per level: leading critical tasks
};

// Tasks per level; within a level the critical LARFB/SSRFB tasks (column
// n == k+1, read by the next panel) come first.
static void build_tasks(int64_t MT, int64_t NT, HostTasks& h, int64_t nlev) {
  h.G.assign(nlev, {});
  h.T.assign(nlev, {});
  h.L.assign(nlev, {});
  h.S.assign(nlev, {});
  h.Lc.assign(nlev, 0);
  h.Sc.assign(nlev, 0);
  std::vector<std::vector<int64_t>> Sb(nlev);
  const int64_t KT = std::min(MT, NT);
  for (int64_t k = 0; k < KT; ++k) {
    h.G[3 * k].push_back(k);
    for (int64_t n = k + 1; n < NT; ++n) {  // n = k+1 first: the critical one
      h.L[3 * k + 1].push_back(k);
      h.L[3 * k + 1].push_back(n);
      if (n == k + 1) ++h.Lc[3 * k + 1];
    }
    for (int64_t m = k + 1; m < MT; ++m) {
      h.T[2 * k + m].push_back(k);
      h.T[2 * k + m].push_back(m);
      for (int64_t n = k + 1; n < NT; ++n) {
        const int64_t t = 2 * k + m + 1;
        auto& v = (n == k + 1) ? h.S[t] : Sb[t];
        v.push_back(k);
        v.push_back(m);
        v.push_back(n);
        if (n == k + 1) ++h.Sc[t];
      }
    }
  }
  for (int64_t t = 0; t < nlev; ++t) h.S[t].insert(h.S[t].end(), Sb[t].begin(), Sb[t].end());
}

// One work list of the dataflow kernel (items in claim order + counters).
struct DagList {
  dag::Item* d_items = nullptr;
  int nitems = 0, ntasks = 0, nio = 0;
  int64_t id_ld = 0, id_st = 0, id_ar = 0;  // first LOAD / STORE / ARRIVE task (host pipeline)
  int* d_ctr = nullptr;                     // [claim cursor | 256 reserved | one per task]
  std::vector<unsigned char> item_kind;     // host copies for the diagnostics
  std::vector<int> item_info;               // per item: kind, k, m, n, sub-task / slab column
  std::vector<int> item_level;
  std::vector<std::pair<int, int>> st_order;  // STORE groups (column, group) in claim order
  int io_tiles = 8;
  bool retire = false;  // tail items flagged: run the kModePlainRetire instantiation
  int launch_nsm = 0;  // > 0: SM count handed to the launch (one resident CTA per SM for small DAGs)
  ~DagList() {
    cudaFree(d_items);
    cudaFree(d_ctr);
  }
};

// ---------------------------------------------------------------------------
// Workspace of one factorization shape
// ---------------------------------------------------------------------------
struct FactorWS {
  int dev = -1;
  int64_t M = 0, N = 0, MT = 0, NT = 0;
  int NB = 0, IB = 0;
  double* tiles = nullptr;  // (MT*NB) x (NT*NB) in tile layout
  double* Tws = nullptr;    // MT*NT*IB*NB
  void** dptr = nullptr;    // all pointer arrays
  LevelLists lv;
  // device pointer arrays per kind
  double** gA = nullptr; double** gT = nullptr;
  double** tR = nullptr; double** tA = nullptr; double** tT = nullptr;
  double** lV = nullptr; double** lT = nullptr; double** lC = nullptr;
  double** sV = nullptr; double** sT = nullptr; double** sC1 = nullptr; double** sC2 = nullptr;
  double** gP = nullptr; double** tP = nullptr; double** lP = nullptr; double** sP = nullptr;  // packed tiles
  bool v2 = false;          // packed-reflector update path (update_v2.cuh)
  double* Vpk = nullptr;    // MT x KT packed reflector tiles
  size_t pk_dbl = 0;
  cudaStream_t s_panel = nullptr, s_update = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaGraphExec_t graph = nullptr;
  int graph_timed = 0;
  // dataflow DAG kernel (dag.cuh): two work lists -- device input
  // (tileqr_factor) and host input with LOAD/STORE items (tileqr_factor_host)
  DagList dag_plain, dag_io;
  DagList* dag_last = nullptr;           // list of the most recent run (diagnostics)
  int nsm = 0;
  unsigned long long* d_prof = nullptr;  // per-item claim/start/end (tileqr_set_kernel_timing)
  size_t prof_cap = 0;
  cudaEvent_t dag_ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> acc_ev;  // timing bit 4: event pairs around every dataflow-kernel launch
  size_t acc_n = 0;                 // launches recorded since the last read
  bool use_dag = false, dag_timed = false;
  int dag_grid = 0;  // resident CTAs of the last DAG launch
  // host pipeline (tileqr_factor_host): column-major staging, copy streams
  double* st_in = nullptr;
  double* st_out = nullptr;
  dag::DagIO* d_io = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t io_ev[3] = {nullptr, nullptr, nullptr};
  bool io_ready = false;  // st_in/st_out, copy streams and io_ev all created
  // Ordering across callers: the workspace (tiles, T, packed tiles, DAG
  // counters, staging) is shared by every call of this shape, so each call's
  // stream waits for the previous call's last operation (this event) before
  // touching it, whatever stream or host thread that call came from.
  cudaEvent_t last_use = nullptr;
  bool used = false;
  uint64_t stamp = 0;  // LRU
  // kernel timing (tileqr_set_kernel_timing): one event pair per launch
  struct Rec { int kind; int64_t tasks; int64_t level; cudaEvent_t a, b; };
  int64_t cur_level = 0;
  std::vector<Rec> recs;
  size_t rec_used = 0;
  ~FactorWS() {
    if (graph) cudaGraphExecDestroy(graph);
    for (auto& r : recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ev) cudaEventDestroy(e);
    if (s_panel) cudaStreamDestroy(s_panel);
    if (s_update) cudaStreamDestroy(s_update);
    cudaFree(tiles);
    cudaFree(Tws);
    cudaFree(dptr);
    cudaFree(Vpk);
    cudaFree(d_prof);
    cudaFree(st_in);
    cudaFree(st_out);
    cudaFree(d_io);
    for (auto e : dag_ev) if (e) cudaEventDestroy(e);
    for (auto e : acc_ev) if (e) cudaEventDestroy(e);
    for (auto e : io_ev) if (e) cudaEventDestroy(e);
    if (last_use) cudaEventDestroy(last_use);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
  }
};

static std::mutex g_mu;
static std::map<std::tuple<int, int64_t, int64_t, int, int>, std::unique_ptr<FactorWS>> g_ws;
static uint64_t g_ws_clock = 0;  // LRU stamps of the cached workspaces

// Cap on cached factorization workspaces (each is the padded tile buffer, T,
// the packed reflector tiles and the DAG lists: ~3.4 GB at 10000^2): the
// least recently used one is freed (after its last use completes) when a new
// shape would exceed TILEQR_WS_CACHE (default 4).  Call with g_mu held.
static void evict_workspaces() {
  size_t cap = 4;
  if (const char* e = getenv("TILEQR_WS_CACHE")) cap = std::max(1, atoi(e));
  while (g_ws.size() >= cap) {
    auto lru = g_ws.begin();
    for (auto it = g_ws.begin(); it != g_ws.end(); ++it)
      if (it->second->stamp < lru->second->stamp) lru = it;
    if (lru->second->used) cudaEventSynchronize(lru->second->last_use);
    g_ws.erase(lru);
  }
}

static int g_timing = 0;  // bit k: time launches of kernel kind k

static bool use_graph() {
  const char* e = getenv("TILEQR_NO_GRAPH");
  return !(e && e[0] == '1');
}

// ---------------------------------------------------------------------------
// Dataflow DAG: tasks, dependencies, priority order, work items (dag.cuh)
// ---------------------------------------------------------------------------
static bool dag_enabled(int NB, int IB) {
  const char* e = getenv("TILEQR_SCHED");
  if (e && strcmp(e, "levels") == 0) return false;
  // the DAG kernel's update items for NB <= 128 are the packed-reflector body
  return dag::dag_supported(NB, IB) && (NB > 128 || v2_supported(NB, IB));
}

bool dag_path_supported(int NB, int IB) { return dag::dag_supported(NB, IB) && v2_supported(NB, IB); }

// Columns of one GEQRT / TSQRT sub-task (a multiple of IB): 16 for NB <= 64,
// else 32 (same-box sweep of 16 / 32 / 64 / NB, profiles/r02ad_panel_sub_ab.log:
// at NB = 64 16 columns give 2048^2 -7 %, 1024^2 -8 %, 4096^2 -2 %; at
// NB = 128 16 columns are neutral at 2048^2 and slower at 4096^2 / 10000^2).
int panel_sub_cols(int NB, int IB) {
  const char* e = getenv("TILEQR_PANEL_SUB");
  int sc = e ? atoi(e) : (NB <= 64 ? 16 : 32);
  if (sc <= 0 || sc >= NB) sc = NB;
  sc = std::max(IB, sc / IB * IB);
  while (NB % sc) sc += IB;
  return sc;
}

// Tasks of the flat-tree tile QR with their dependencies.
// GEQRT(k) and TSQRT(k,m) are split into NS sub-tasks s of consecutive inner
// panels: inner panel c0 of a TSQRT reads and writes only the R rows
// [c0, c0+IB) of tile (k,k) (and its own tile (m,k)), and GEQRT(k)'s inner
// panel c0 is the last to touch those rows, so the flat TSQRT chain of step
// k pipelines at sub-task granularity instead of running tile after tile:
//   G(k,s) <- G(k,s-1) | S(k-1,k,k);         L(k,n) <- G(k,NS-1), S(k-1,k,n);
//   T(k,m,s) <- T(k,m,s-1) | S(k-1,m,k),  (m == k+1 ? G(k,s) : T(k,m-1,s));
//   S(k,m,n) <- T(k,m,NS-1), (m == k+1 ? L(k,n) : S(k,m-1,n)), S(k-1,m,n).
// ("a | b": a for s > 0, b for s == 0.)  Claim order: bottom level (longest
// weighted path to the end of the DAG) descending -- a topological order,
// since a task's bottom level exceeds each successor's -- ties by ASAP level,
// then task id.
static int build_dag(FactorWS* ws, bool io) {
  const int64_t MT = ws->MT, NT = ws->NT, KT = std::min(MT, NT), N = ws->N, M = ws->M;
  const int NB = ws->NB, IB = ws->IB;
  const int SC = panel_sub_cols(NB, IB), NS = NB / SC;
  std::vector<int64_t> offL(KT + 1), offT(KT + 1), offS(KT + 1);
  int64_t nG = KT * NS, nL = 0, nT = 0, nS = 0;
  for (int64_t k = 0; k < KT; ++k) {
    offL[k] = nL; nL += NT - k - 1;
    offT[k] = nT; nT += (MT - k - 1) * NS;
    offS[k] = nS; nS += (MT - k - 1) * (NT - k - 1);
  }
  const int64_t ntask0 = nG + nL + nT + nS;        // the factorization's tasks
  // host pipeline: LOAD(n), STORE(n), ARRIVE(n) per tile column n (the copy
  // engine lands the input column block by column block: contiguous copies
  // run at the link's rate, strided row blocks of NB doubles measured ~30 %
  // slower in total)
  int kIoTiles = 8;  // tiles per LOAD / STORE item
  if (const char* e = getenv("TILEQR_DAG_IOTILES")) kIoTiles = std::max(1, atoi(e));  // diagnostics
  const int nld = (int)((MT + kIoTiles - 1) / kIoTiles), nst = nld;
  // STORE tasks per (tile column n, group g of kIoTiles tile rows): a group
  // is copied back as soon as ITS tiles are final -- the R rows of a column
  // long before the column's own panel -- so the device-to-host traffic is
  // spread over the factorization instead of bunching at its end
  const int64_t ntask = ntask0 + (io ? (2 + nst) * NT : 0);
  if (ntask > (int64_t)1 << 30) {
    set_error("tileqr_factor: DAG too large for the dataflow kernel");
    return TILEQR_ERR_ALLOC;
  }
  auto idG = [&](int64_t k, int s) { return k * NS + s; };
  auto idL = [&](int64_t k, int64_t n) { return nG + offL[k] + (n - k - 1); };
  auto idT = [&](int64_t k, int64_t m, int s) { return nG + nL + offT[k] + (m - k - 1) * NS + s; };
  auto idS = [&](int64_t k, int64_t m, int64_t n) {
    return nG + nL + nT + offS[k] + (m - k - 1) * (NT - k - 1) + (n - k - 1);
  };
  auto idLD = [&](int64_t n) { return ntask0 + n; };
  auto idST = [&](int64_t n, int g) { return ntask0 + NT + n * nst + g; };
  auto idAR = [&](int64_t n) { return ntask0 + NT + NT * nst + n; };
  constexpr int kArrive = dag::kArrive;  // host-only pseudo kind: set by the copy stream
  using Task = sched::Task;
  std::vector<Task> tk(ntask);
  for (int64_t k = 0; k < KT; ++k) {
    for (int sub = 0; sub < NS; ++sub) {
      Task g{dag::kGeqrt, (int)k, (int)k, (int)k, (int)(3 * k), 0, {0, 0, 0}, sub};
      if (sub > 0) g.dep[g.ndep++] = (int)idG(k, sub - 1);
      else if (k > 0) g.dep[g.ndep++] = (int)idS(k - 1, k, k);
      else if (io) g.dep[g.ndep++] = (int)idLD(0);
      tk[idG(k, sub)] = g;
    }
    for (int64_t n = k + 1; n < NT; ++n) {
      Task l{dag::kLarfb, (int)k, (int)k, (int)n, (int)(3 * k + 1), 0, {0, 0, 0}, 0};
      l.dep[l.ndep++] = (int)idG(k, NS - 1);
      if (k > 0) l.dep[l.ndep++] = (int)idS(k - 1, k, n);
      else if (io) l.dep[l.ndep++] = (int)idLD(n);
      tk[idL(k, n)] = l;
    }
    for (int64_t m = k + 1; m < MT; ++m) {
      for (int sub = 0; sub < NS; ++sub) {
        Task t{dag::kTsqrt, (int)k, (int)m, (int)k, (int)(2 * k + m), 0, {0, 0, 0}, sub};
        if (sub > 0) t.dep[t.ndep++] = (int)idT(k, m, sub - 1);
        else if (k > 0) t.dep[t.ndep++] = (int)idS(k - 1, m, k);
        t.dep[t.ndep++] = (int)(m == k + 1 ? idG(k, sub) : idT(k, m - 1, sub));
        tk[idT(k, m, sub)] = t;
      }
      for (int64_t n = k + 1; n < NT; ++n) {
        Task u{dag::kSsrfb, (int)k, (int)m, (int)n, (int)(2 * k + m + 1), 0, {0, 0, 0}, 0};
        u.dep[u.ndep++] = (int)idT(k, m, NS - 1);
        u.dep[u.ndep++] = (int)(m == k + 1 ? idL(k, n) : idS(k, m - 1, n));
        if (k > 0) u.dep[u.ndep++] = (int)idS(k - 1, m, n);
        tk[idS(k, m, n)] = u;
      }
    }
  }
  if (io) {
    const int last_level = (int)num_levels(MT, NT);
    for (int64_t n = 0; n < NT; ++n) {
      tk[idAR(n)] = Task{kArrive, 0, 0, (int)n, 0, 0, {0, 0, 0}, 0};
      Task ld{dag::kLoad, 0, 0, (int)n, 0, 0, {0, 0, 0}, 0};
      ld.dep[ld.ndep++] = (int)idAR(n);
      tk[idLD(n)] = ld;
      for (int g = 0; g < nst; ++g) {
        // the last task writing tile rows [r0, r1) of column n (its chain
        // implies every earlier writer): the column's panel when the group
        // reaches the diagonal tile, else step r1-1's last update of the column
        const int64_t r1 = std::min<int64_t>(MT, (int64_t)(g + 1) * kIoTiles);
        int64_t last;
        if (n < KT && r1 - 1 >= n) {
          last = (MT > n + 1) ? idT(n, MT - 1, NS - 1) : idG(n, NS - 1);
        } else {
          const int64_t k = r1 - 1;
          last = (MT > k + 1) ? idS(k, MT - 1, n) : idL(k, n);
        }
        Task st{dag::kStore, 0, 0, (int)n, last_level, 0, {0, 0, 0}, g};
        st.dep[st.ndep++] = (int)last;
        tk[idST(n, g)] = st;
      }
    }
  }
  const int cols = dag::dag_cols(NB);
  const int nslab = (NB + cols - 1) / cols;
  auto parts = [&](int kind) {
    if (kind == dag::kLarfb || kind == dag::kSsrfb) return nslab;
    if (kind == dag::kLoad) return nld;
    return 1;  // GEQRT / TSQRT sub-tasks, STORE groups
  };
  // bottom levels (priority of ready items in the simulation below)
  // panel weight: twice the earlier 1200 ns per column (same-box sweep of
  // TILEQR_DAG_WP at 10000^2: x2 -0.9 % (IB=16) / -1.2 % (IB=32), x0.5 and
  // x3 slower)
  double wS = 4.0 * NB * NB * NB / 150.0, wP = 2400.0 * NB / NS;
  if (const char* e = getenv("TILEQR_DAG_WS")) wS *= atof(e);  // diagnostics: priority weights
  if (const char* e = getenv("TILEQR_DAG_WP")) wP *= atof(e);
  double wL = wS / 2;
  const double wIO = 10000.0;
  if (const char* e = getenv("TILEQR_DAG_WL")) wL *= atof(e);  // diagnostics
  auto weight = [&](int kind) {
    return kind == dag::kSsrfb ? wS : kind == dag::kLarfb ? wL : kind == kArrive ? 0.0
         : (kind == dag::kLoad || kind == dag::kStore) ? wIO : wP;
  };
  sched::Params prm;
  prm.parts = parts;
  prm.weight = weight;
  // LOAD / STORE items start as soon as they are ready: they gate everything
  // downstream (LOAD) or the device-to-host copy (STORE) and are cheap
  prm.bl_override.assign(ntask, -1.0);
  for (int64_t i = ntask0; i < ntask; ++i)
    if (tk[i].kind == dag::kLoad || tk[i].kind == dag::kStore) prm.bl_override[i] = 1e30;

  // Claim order: a list schedule simulated on the host (sched.h) -- P workers
  // (the resident CTAs), rough per-item durations, ready items started in
  // bottom-level order -- and the items sorted by their simulated start time.
  // A CTA that claims an item blocks until its inputs are final, so claiming
  // in an order the DAG can actually keep up with avoids head-of-line
  // blocking (pure bottom-level order parks hundreds of CTAs on far-future
  // items while the first panels run).  ARRIVE pseudo-tasks (host pipeline)
  // complete at the time their column's copy is expected to land.
  int dev0 = 0, nsm0 = 0;
  TQ_CUDA(cudaGetDevice(&dev0));
  TQ_CUDA(cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, dev0));
  // Small DAGs are bound by the panel chain, and a GEQRT/TSQRT item runs at
  // about half speed while an update CTA shares its SM: with at most
  // kOneCtaTiles tile updates in the widest step, one CTA per SM is resident.
  // Same-box sweeps (profiles/r02s4_one_cta*.log): NB = 64 gains 3-8 % up to
  // 2048^2 (961 tiles) and loses 12 % at 2500^2 (1521); NB = 128 gains 6-14 %
  // up to 4000^2 (961) and loses 5 % at 5000^2 (1444); NB = 96 +3 % at 961,
  // -16 % at 1681.  The results do not depend on the resident CTA count.
  int ctas_per_sm = dag::dag_ctas_per_sm(NB);
  {
    long kOneCtaTiles = 1200;
    if (const char* e = getenv("TILEQR_DAG_ONE_CTA_TILES")) kOneCtaTiles = atol(e);  // diagnostics
    const long widest = (long)(MT - 1) * (long)(NT - 1);
    if (!io && ctas_per_sm == 2 && widest <= kOneCtaTiles) ctas_per_sm = 1;
  }
  const int P = std::max(1, nsm0 * ctas_per_sm);
  double cta_gflops = 220.0 / ctas_per_sm;                          // update rate per CTA
  if (const char* e = getenv("TILEQR_DAG_CTAGF")) cta_gflops *= atof(e);  // diagnostics
  const double dS = 4.0 * NB * NB * cols / cta_gflops;               // ns per SSRFB slab
  // measured in the dataflow kernel at NB = 128 (10000^2): TSQRT and GEQRT
  // sub-tasks ~2-3 us per column (sharing their SM with an update CTA), LARFB
  // slab ~0.77 of an SSRFB slab; plus ~3 us of hand-off (release -> acquire
  // -> operand loads) per item.  The values below are the best of a sweep
  // (tools/sim_sweep.sh; +-40 % moves the factorization by ~1 %)
  double sT = 3000.0, sG = 3000.0, hand = 5000.0;
  if (ctas_per_sm == 1) sT = sG = 1500.0;  // a panel item has its SM alone
  if (const char* e = getenv("TILEQR_DAG_SIM")) sscanf(e, "%lf,%lf,%lf", &sT, &sG, &hand);  // diagnostics
  const double dL = 0.77 * dS + hand, dT = sT * SC + hand, dG = sG * SC + hand;
  const double dIO = 1.0e3 + (double)kIoTiles * NB * NB * 16 / 50.0;  // ~50 GB/s per CTA
  double h2d_gbs = 54.0;  // host link, measured while the kernel runs (54 GB/s; 30-100 in the sim: +-3 %)
  if (const char* e = getenv("TILEQR_DAG_H2D_GBS")) h2d_gbs = atof(e);  // diagnostics
  const double tcol = (double)MT * NB * NB * 8 / h2d_gbs;
  for (int64_t i = ntask0; i < ntask; ++i)
    if (tk[i].kind == kArrive) {
      tk[i].worker = false;
      tk[i].fixed = tcol * (tk[i].n + 1);
    }
  prm.dur = [&](int kind) {
    switch (kind) {
      case dag::kSsrfb: return dS + hand;
      case dag::kLarfb: return dL;
      case dag::kTsqrt: return dT;
      case dag::kGeqrt: return dG;
      case kArrive: return 0.0;
      default: return dIO;
    }
  };
  prm.npools = 1;
  prm.workers = P;
  std::vector<sched::Slot> sched;
  const char* ord = getenv("TILEQR_DAG_ORDER");  // diagnostics: "bl" = pure bottom-level order
  const int src = sched::simulate(tk, prm, &sched, ord && strcmp(ord, "bl") == 0);
  if (src == -1) {
    set_error("tileqr_factor: internal error: the task graph has a cycle");
    return TILEQR_ERR_CUDA;
  }
  if (src) {
    set_error("tileqr_factor: internal error in the DAG schedule simulation");
    return TILEQR_ERR_CUDA;
  }
  const size_t tile = (size_t)NB * NB;
  double* A = ws->tiles;
  double* Tw = ws->Tws;
  auto tp = [&](int64_t m, int64_t n) { return A + (size_t)(m + n * MT) * tile; };
  auto tt = [&](int64_t m, int64_t k) { return Tw + (size_t)(m + k * MT) * IB * NB; };
  auto pkp = [&](int64_t m, int64_t k) { return ws->Vpk ? ws->Vpk + (size_t)(m + k * MT) * ws->pk_dbl : nullptr; };
  DagList& L = io ? ws->dag_io : ws->dag_plain;
  const bool rowlim = !getenv("TILEQR_DAG_NO_ROWLIM");  // diagnostics: SSRFB over the padding rows too
  // Tail retirement (dag.cuh): the items of the last panel steps -- those
  // with at most kTailTiles tile updates, where the panel chain and not the
  // CTA slots bounds the run -- are flagged, as a count at the end of the
  // claim order; from there on one CTA per SM keeps claiming.  Same-box sweep
  // (profiles/r02s4_retire*.log): 6000^2 (128, 16) -3.1 %, (128, 32) -2.4 %,
  // 10000^2 -0.1 %; a tail three times as long costs 2 % at 10000^2.
  int64_t retire_from = INT64_MAX;
  // Only where the tail is a visible share of the run (widest step of at most
  // kRetireMaxTiles tile updates: up to 8000^2 at NB = 128): the retirement
  // code costs the kernel 0.2-0.4 % at 10000^2 (same-box A/B of builds,
  // profiles/r02s4_retire_build_ab.log), more than it gains there.
  long kRetireMaxTiles = 4000;
  if (const char* e = getenv("TILEQR_DAG_RETIRE_MAX_TILES")) kRetireMaxTiles = atol(e);  // diagnostics
  if (!io && dag::dag_ctas_per_sm(NB) == 2 && ctas_per_sm == 2 && (MT - 1) * (NT - 1) <= kRetireMaxTiles) {
    long kTailTiles = 500;
    if (const char* e = getenv("TILEQR_DAG_RETIRE_TILES")) kTailTiles = atol(e);  // diagnostics; 0: off
    int64_t tail = 0;
    for (int64_t i = 0; i < ntask0; ++i)
      if ((MT - tk[i].k - 1) * (NT - tk[i].k - 1) <= kTailTiles) tail += parts(tk[i].kind);
    if (const char* e = getenv("TILEQR_DAG_RETIRE")) tail = atol(e);  // diagnostics: the count itself
    if (kTailTiles > 0 && tail > 0) retire_from = std::max<int64_t>(0, (int64_t)sched.size() - tail);
  }
  std::vector<dag::Item> items;
  items.reserve(sched.size());
  L.item_kind.clear();
  L.item_level.clear();
  L.item_info.clear();
  L.st_order.clear();
  for (const sched::Slot& sl : sched) {
    const int i = sl.task;
    const Task& t = tk[i];
    dag::Item it{};
    it.kind = t.kind;
    it.task = i;
    if (t.kind == dag::kGeqrt || t.kind == dag::kTsqrt) it.col0 = (t.s * SC) | ((t.s + 1) * SC) << 16;
    else it.col0 = sl.slab * cols;
    it.ndep = t.ndep;
    for (int d = 0; d < t.ndep; ++d) {
      it.dep[d] = t.dep[d];
      it.need[d] = parts(tk[t.dep[d]].kind);
    }
    switch (t.kind) {
      case dag::kGeqrt: it.p[0] = tp(t.k, t.k); it.p[2] = tt(t.k, t.k); it.pk = pkp(t.k, t.k); break;
      case dag::kTsqrt:
        it.p[0] = tp(t.k, t.k); it.p[1] = tp(t.m, t.k); it.p[2] = tt(t.m, t.k); it.pk = pkp(t.m, t.k);
        break;
      case dag::kLarfb:
        it.p[0] = tp(t.k, t.k); it.p[1] = tt(t.k, t.k); it.p[2] = tp(t.k, t.n); it.pk = pkp(t.k, t.k);
        break;
      case dag::kLoad:   // tiles (m, n), m in the item's row range
      case dag::kStore: {
        const int g = t.kind == dag::kStore ? t.s : sl.slab;
        it.aux[0] = t.n;
        it.aux[1] = t.n + 1;
        it.aux[2] = g * kIoTiles;
        it.aux[3] = (int)std::min<int64_t>(MT, (int64_t)(g + 1) * kIoTiles);
        if (t.kind == dag::kStore) L.st_order.push_back({t.n, g});
        break;
      }
      default:
        it.p[0] = tp(t.m, t.k); it.p[1] = tt(t.m, t.k); it.p[2] = tp(t.k, t.n); it.p[3] = tp(t.m, t.n);
        it.pk = pkp(t.m, t.k);
        break;
    }
    if (t.kind == dag::kLarfb || t.kind == dag::kSsrfb)  // padded columns (e_j or 0) are invariant
      it.aux[0] = (int)std::min<int64_t>(NB, std::max<int64_t>(0, N - (int64_t)t.n * NB));
    if (t.kind == dag::kSsrfb && rowlim) it.aux[1] = dag::ssrfb_rows(M, t.m, NB);
    if (!io && (int64_t)items.size() >= retire_from) it.aux[3] = 1;  // tail item (dag.cuh: tail retirement)
    items.push_back(it);
    L.item_kind.push_back((unsigned char)t.kind);
    L.item_level.push_back(t.level);
    for (int v : {t.kind, t.k, t.m, t.n, (t.kind >= dag::kLarfb) ? it.col0 : t.s}) L.item_info.push_back(v);
  }
  L.nitems = (int)items.size();
  L.ntasks = (int)ntask;
  L.nio = nst;
  L.io_tiles = kIoTiles;
  L.retire = retire_from != INT64_MAX;
  L.launch_nsm = ctas_per_sm < dag::dag_ctas_per_sm(NB) ? std::max(1, nsm0 / dag::dag_ctas_per_sm(NB)) : 0;
  L.id_ld = ntask0;
  L.id_st = ntask0 + NT;
  L.id_ar = ntask0 + NT + NT * nst;
  int dev = 0;
  TQ_CUDA(cudaGetDevice(&dev));
  TQ_CUDA(cudaDeviceGetAttribute(&ws->nsm, cudaDevAttrMultiProcessorCount, dev));
  if (cudaMalloc(&L.d_items, std::max<size_t>(items.size(), 1) * sizeof(dag::Item)) != cudaSuccess ||
      cudaMalloc(&L.d_ctr, (size_t)(ntask + 257) * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    set_error("tileqr_factor: device allocation of the DAG work list failed");
    return TILEQR_ERR_ALLOC;
  }
  TQ_CUDA(cudaMemcpy(L.d_items, items.data(), items.size() * sizeof(dag::Item), cudaMemcpyHostToDevice));
  if (!ws->dag_ev[0])
    for (auto& e : ws->dag_ev) TQ_CUDA(cudaEventCreate(&e));
  return 0;
}

static int run_dag_list(FactorWS* ws, DagList& L, const dag::DagIO* io, cudaStream_t stream) {
  unsigned long long* prof = nullptr;
  const bool acc = (g_timing & 16) != 0;  // launch events only (no device-clock trace)
  if (acc) {
    while (ws->acc_ev.size() < 2 * (ws->acc_n + 1)) {
      cudaEvent_t e;
      TQ_CUDA(cudaEventCreate(&e));
      ws->acc_ev.push_back(e);
    }
    TQ_CUDA(cudaEventRecord(ws->acc_ev[2 * ws->acc_n], stream));
  }
  if (g_timing & 15) {
    if (ws->prof_cap < (size_t)L.nitems) {
      cudaFree(ws->d_prof);
      ws->d_prof = nullptr;
      TQ_CUDA(cudaMalloc(&ws->d_prof, (size_t)L.nitems * 3 * sizeof(unsigned long long)));
      ws->prof_cap = L.nitems;
    }
    prof = ws->d_prof;
    TQ_CUDA(cudaEventRecord(ws->dag_ev[0], stream));
  }
  int nitems = L.nitems;
  if (const char* e = getenv("TILEQR_DAG_NITEMS")) {  // diagnostics: run a prefix of the claim order
    const long v = atol(e);
    if (v >= 0 && v < nitems) nitems = (int)v;
  }
  int rc = launch_dag(ws->NB, ws->IB, L.d_items, nitems, L.d_ctr, L.d_ctr + 257, L.launch_nsm > 0 ? L.launch_nsm : ws->nsm, prof, stream,
                      &ws->dag_grid, io, io ? dag::kModeIO : L.retire ? dag::kModePlainRetire : dag::kModePlain);
  if (rc) return rc;
  if (g_timing & 15) TQ_CUDA(cudaEventRecord(ws->dag_ev[1], stream));
  if (acc) TQ_CUDA(cudaEventRecord(ws->acc_ev[2 * ws->acc_n++ + 1], stream));
  ws->dag_timed = (g_timing & 15) != 0;
  ws->dag_last = &L;
  return 0;
}

static int run_dag(FactorWS* ws, cudaStream_t stream) {
  DagList& L = ws->dag_plain;
  // counters: [claim cursor | 256 reserved | one per task]
  TQ_CUDA(cudaMemsetAsync(L.d_ctr, 0, (size_t)(L.ntasks + 257) * sizeof(int), stream));
  return run_dag_list(ws, L, nullptr, stream);
}

static int create_ws(int dev, int64_t M, int64_t N, int NB, int IB, FactorWS** out) {
  auto ws = std::make_unique<FactorWS>();
  ws->dev = dev;
  ws->M = M;
  ws->N = N;
  ws->NB = NB;
  ws->IB = IB;
  ws->MT = (M + NB - 1) / NB;
  ws->NT = (N + NB - 1) / NB;
  const int64_t MT = ws->MT, NT = ws->NT;
  const size_t tile = (size_t)NB * NB;
  if (cudaMalloc(&ws->tiles, tile * MT * NT * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ws->Tws, (size_t)MT * NT * IB * NB * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    set_error("tileqr_factor: device allocation of the tile workspace failed");
    return TILEQR_ERR_ALLOC;
  }
  // T tiles (m, k) with m < k are never written: keep them 0 in the output
  TQ_CUDA(cudaMemset(ws->Tws, 0, (size_t)MT * NT * IB * NB * sizeof(double)));
  const int64_t nlev = num_levels(MT, NT);
  HostTasks h;
  build_tasks(MT, NT, h, nlev);
  LevelLists& lv = ws->lv;
  lv.nlev = nlev;
  int64_t nG = 0, nT = 0, nL = 0, nS = 0;
  for (int64_t t = 0; t < nlev; ++t) {
    lv.g_off.push_back(nG); lv.g_cnt.push_back((int64_t)h.G[t].size()); nG += h.G[t].size();
    lv.t_off.push_back(nT); lv.t_cnt.push_back((int64_t)h.T[t].size() / 2); nT += h.T[t].size() / 2;
    lv.l_off.push_back(nL); lv.l_cnt.push_back((int64_t)h.L[t].size() / 2); nL += h.L[t].size() / 2;
    lv.s_off.push_back(nS); lv.s_cnt.push_back((int64_t)h.S[t].size() / 3); nS += h.S[t].size() / 3;
    lv.lc_cnt.push_back(h.Lc[t]);
    lv.sc_cnt.push_back(h.Sc[t]);
  }
  // packed reflector tiles (update_v2.cuh): one per (m, k), m >= k
  ws->v2 = v2_supported(NB, IB);
  const int64_t KT = std::min(MT, NT);
  if (ws->v2) {
    ws->pk_dbl = v2_pk_doubles(NB, IB);
    if (cudaMalloc(&ws->Vpk, ws->pk_dbl * MT * KT * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      set_error("tileqr_factor: device allocation of the packed reflector tiles failed");
      return TILEQR_ERR_ALLOC;
    }
  }
  const size_t total = 3 * nG + 4 * nT + 4 * nL + 5 * nS;
  std::vector<void*> hp(std::max<size_t>(total, 1));
  double* A = ws->tiles;
  double* T = ws->Tws;
  auto tp = [&](int64_t m, int64_t n) { return A + (size_t)(m + n * MT) * tile; };
  auto tt = [&](int64_t m, int64_t k) { return T + (size_t)(m + k * MT) * IB * NB; };
  auto pk = [&](int64_t m, int64_t k) -> void* {
    return ws->Vpk ? ws->Vpk + (size_t)(m + k * MT) * ws->pk_dbl : nullptr;
  };
  size_t o = 0;
  const size_t oG = o; o += 3 * nG;
  const size_t oT = o; o += 4 * nT;
  const size_t oL = o; o += 4 * nL;
  const size_t oS = o; o += 5 * nS;
  {
    size_t i = 0;
    for (int64_t t = 0; t < nlev; ++t)
      for (int64_t k : h.G[t]) {
        hp[oG + i] = tp(k, k);
        hp[oG + nG + i] = tt(k, k);
        hp[oG + 2 * nG + i] = pk(k, k);
        ++i;
      }
    i = 0;
    for (int64_t t = 0; t < nlev; ++t)
      for (size_t q = 0; q < h.T[t].size(); q += 2) {
        const int64_t k = h.T[t][q], m = h.T[t][q + 1];
        hp[oT + i] = tp(k, k);
        hp[oT + nT + i] = tp(m, k);
        hp[oT + 2 * nT + i] = tt(m, k);
        hp[oT + 3 * nT + i] = pk(m, k);
        ++i;
      }
    i = 0;
    for (int64_t t = 0; t < nlev; ++t)
      for (size_t q = 0; q < h.L[t].size(); q += 2) {
        const int64_t k = h.L[t][q], n = h.L[t][q + 1];
        hp[oL + i] = tp(k, k);
        hp[oL + nL + i] = tt(k, k);
        hp[oL + 2 * nL + i] = tp(k, n);
        hp[oL + 3 * nL + i] = pk(k, k);
        ++i;
      }
    i = 0;
    for (int64_t t = 0; t < nlev; ++t)
      for (size_t q = 0; q < h.S[t].size(); q += 3) {
        const int64_t k = h.S[t][q], m = h.S[t][q + 1], n = h.S[t][q + 2];
        hp[oS + i] = tp(m, k);
        hp[oS + nS + i] = tt(m, k);
        hp[oS + 2 * nS + i] = tp(k, n);
        hp[oS + 3 * nS + i] = tp(m, n);
        hp[oS + 4 * nS + i] = pk(m, k);
        ++i;
      }
  }
  if (cudaMalloc(&ws->dptr, hp.size() * sizeof(void*)) != cudaSuccess) {
    cudaGetLastError();
    set_error("tileqr_factor: device allocation of the task lists failed");
    return TILEQR_ERR_ALLOC;
  }
  TQ_CUDA(cudaMemcpy(ws->dptr, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice));
  double** d = reinterpret_cast<double**>(ws->dptr);
  ws->gA = d + oG; ws->gT = d + oG + nG; ws->gP = d + oG + 2 * nG;
  ws->tR = d + oT; ws->tA = d + oT + nT; ws->tT = d + oT + 2 * nT; ws->tP = d + oT + 3 * nT;
  ws->lV = d + oL; ws->lT = d + oL + nL; ws->lC = d + oL + 2 * nL; ws->lP = d + oL + 3 * nL;
  ws->sV = d + oS; ws->sT = d + oS + nS; ws->sC1 = d + oS + 2 * nS; ws->sC2 = d + oS + 3 * nS;
  ws->sP = d + oS + 4 * nS;
  // The panel kernels (GEQRT/TSQRT) are the DAG's critical path: their stream
  // gets the highest priority so their CTAs are dispatched ahead of queued
  // update CTAs whenever an SM frees up (kept per node in the CUDA graph).
  int prio_lo = 0, prio_hi = 0;
  TQ_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  TQ_CUDA(cudaStreamCreateWithPriority(&ws->s_panel, cudaStreamNonBlocking, prio_hi));
  TQ_CUDA(cudaStreamCreateWithPriority(&ws->s_update, cudaStreamNonBlocking, prio_lo));
  ws->ev.resize(9);
  for (auto& e : ws->ev) TQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TQ_CUDA(cudaEventCreateWithFlags(&ws->last_use, cudaEventDisableTiming));
  ws->use_dag = dag_enabled(NB, IB);
  if (ws->use_dag) {
    int rc = build_dag(ws.get(), false);
    if (rc) return rc;
  }
  *out = ws.get();
  evict_workspaces();
  g_ws[std::make_tuple(dev, M, N, NB, IB)] = std::move(ws);
  return 0;
}

// Issue the level sequence: s_panel runs GEQRT/TSQRT, s_update LARFB/SSRFB.
// With kernel timing on, every launch is bracketed by two events (captured as
// event-record nodes when the sequence is captured into the graph).
static int timed_begin(FactorWS* ws, int kind, int64_t tasks, cudaStream_t st, size_t* slot) {
  *slot = (size_t)-1;
  if (!(g_timing & (1 << kind))) return 0;
  if (ws->rec_used == ws->recs.size()) {
    FactorWS::Rec r{kind, tasks, 0, nullptr, nullptr};
    TQ_CUDA(cudaEventCreate(&r.a));
    TQ_CUDA(cudaEventCreate(&r.b));
    ws->recs.push_back(r);
  }
  *slot = ws->rec_used++;
  ws->recs[*slot].kind = kind;
  ws->recs[*slot].tasks = tasks;
  ws->recs[*slot].level = ws->cur_level;
  TQ_CUDA(cudaEventRecordWithFlags(ws->recs[*slot].a, st, cudaEventRecordExternal));
  return 0;
}
static int timed_end(FactorWS* ws, size_t slot, cudaStream_t st) {
  if (slot == (size_t)-1) return 0;
  TQ_CUDA(cudaEventRecordWithFlags(ws->recs[slot].b, st, cudaEventRecordExternal));
  return 0;
}

// Critical-first schedule.  Level t:
//   panel stream  : waits for the bulk updates of level t-2 (the last writers
//                   of every tile its tasks touch), then the critical updates
//                   of level t (LARFB(k,k+1), SSRFB(k,m,k+1): they feed the
//                   next panel), then GEQRT/TSQRT of level t;
//   update stream : waits for the panel stream of level t-1 (the V/T tiles
//                   read at level t), then the bulk LARFB/SSRFB of level t.
// Every task still runs at its ASAP level and every tile sees the same
// sequence of operations (bitwise identical to the level-synchronous order);
// the panel chain just never waits for a whole update batch.
static int issue_levels(FactorWS* ws, cudaStream_t sp, cudaStream_t su) {
  const LevelLists& lv = ws->lv;
  const int NB = ws->NB, IB = ws->IB;
  cudaEvent_t* pdone = &ws->ev[4];  // ring of 2: panel stream done with level t
  cudaEvent_t* bdone = &ws->ev[6];  // ring of 3: update stream done with level t
  ws->rec_used = 0;
  auto larfb = [&](int64_t off, int64_t cnt, cudaStream_t st) -> int {
    if (cnt <= 0) return 0;
    size_t slot = 0;
    int rc;
    if ((rc = timed_begin(ws, 2, cnt, st, &slot))) return rc;
    if (ws->v2) rc = launch_update_pk(true, NB, IB, (int)cnt, ws->lP + off, nullptr, ws->lC + off, st);
    else rc = launch_larfb(true, NB, IB, (int)cnt, ws->lV + off, ws->lT + off, ws->lC + off, NB, st);
    if (rc) return rc;
    return timed_end(ws, slot, st);
  };
  auto ssrfb = [&](int64_t off, int64_t cnt, cudaStream_t st) -> int {
    if (cnt <= 0) return 0;
    size_t slot = 0;
    int rc;
    if ((rc = timed_begin(ws, 3, cnt, st, &slot))) return rc;
    if (ws->v2)
      rc = launch_update_pk(false, NB, IB, (int)cnt, ws->sP + off, ws->sC1 + off, ws->sC2 + off, st);
    else
      rc = launch_ssrfb(true, NB, IB, (int)cnt, ws->sV + off, ws->sT + off, ws->sC1 + off, ws->sC2 + off, NB, st);
    if (rc) return rc;
    return timed_end(ws, slot, st);
  };
  const char* cf = getenv("TILEQR_CRITICAL_FIRST");
  const bool critical_first = cf && cf[0] == '1';
  for (int64_t t = 0; t < lv.nlev; ++t) {
    int rc;
    ws->cur_level = t;
    if (!critical_first) {
      // level-synchronous (default): level t after everything of level t-1
      if (t > 0) {
        TQ_CUDA(cudaEventRecord(ws->ev[1], su));
        TQ_CUDA(cudaStreamWaitEvent(sp, ws->ev[1], 0));
        TQ_CUDA(cudaEventRecord(ws->ev[0], sp));
        TQ_CUDA(cudaStreamWaitEvent(su, ws->ev[0], 0));
      }
      size_t slot = 0;
      if (lv.g_cnt[t] > 0) {
        if ((rc = timed_begin(ws, 0, lv.g_cnt[t], sp, &slot))) return rc;
        if ((rc = launch_geqrt(NB, IB, (int)lv.g_cnt[t], ws->gA + lv.g_off[t], ws->gT + lv.g_off[t], sp,
                              ws->v2 ? ws->gP + lv.g_off[t] : nullptr)))
          return rc;
        if ((rc = timed_end(ws, slot, sp))) return rc;
      }
      if (lv.t_cnt[t] > 0) {
        if ((rc = timed_begin(ws, 1, lv.t_cnt[t], sp, &slot))) return rc;
        if ((rc = launch_tsqrt(NB, IB, (int)lv.t_cnt[t], ws->tR + lv.t_off[t], ws->tA + lv.t_off[t],
                               ws->tT + lv.t_off[t], sp, ws->v2 ? ws->tP + lv.t_off[t] : nullptr)))
          return rc;
        if ((rc = timed_end(ws, slot, sp))) return rc;
      }
      if ((rc = larfb(lv.l_off[t], lv.l_cnt[t], su))) return rc;
      if ((rc = ssrfb(lv.s_off[t], lv.s_cnt[t], su))) return rc;
      continue;
    }
    // ---- panel stream ----------------------------------------------------
    if (t >= 2) TQ_CUDA(cudaStreamWaitEvent(sp, bdone[(t - 2) % 3], 0));
    if ((rc = larfb(lv.l_off[t], lv.lc_cnt[t], sp))) return rc;
    if ((rc = ssrfb(lv.s_off[t], lv.sc_cnt[t], sp))) return rc;
    size_t slot = 0;
    if (lv.g_cnt[t] > 0) {
      if ((rc = timed_begin(ws, 0, lv.g_cnt[t], sp, &slot))) return rc;
      if ((rc = launch_geqrt(NB, IB, (int)lv.g_cnt[t], ws->gA + lv.g_off[t], ws->gT + lv.g_off[t], sp,
                              ws->v2 ? ws->gP + lv.g_off[t] : nullptr)))
        return rc;
      if ((rc = timed_end(ws, slot, sp))) return rc;
    }
    if (lv.t_cnt[t] > 0) {
      if ((rc = timed_begin(ws, 1, lv.t_cnt[t], sp, &slot))) return rc;
      if ((rc = launch_tsqrt(NB, IB, (int)lv.t_cnt[t], ws->tR + lv.t_off[t], ws->tA + lv.t_off[t],
                             ws->tT + lv.t_off[t], sp, ws->v2 ? ws->tP + lv.t_off[t] : nullptr)))
        return rc;
      if ((rc = timed_end(ws, slot, sp))) return rc;
    }
    TQ_CUDA(cudaEventRecord(pdone[t % 2], sp));
    // ---- update stream ---------------------------------------------------
    if (t >= 1) TQ_CUDA(cudaStreamWaitEvent(su, pdone[(t - 1) % 2], 0));
    if ((rc = larfb(lv.l_off[t] + lv.lc_cnt[t], lv.l_cnt[t] - lv.lc_cnt[t], su))) return rc;
    if ((rc = ssrfb(lv.s_off[t] + lv.sc_cnt[t], lv.s_cnt[t] - lv.sc_cnt[t], su))) return rc;
    TQ_CUDA(cudaEventRecord(bdone[t % 3], su));
  }
  // the caller joins both streams (run_levels)
  return 0;
}

// Run the level sequence ordered after `stream` and before subsequent work on it.
static int run_levels(FactorWS* ws, cudaStream_t stream) {
  if (ws->use_dag) return run_dag(ws, stream);
  if (use_graph()) {
    if (ws->graph && ws->graph_timed != g_timing) {
      cudaGraphExecDestroy(ws->graph);
      ws->graph = nullptr;
    }
    if (!ws->graph) {
      ws->graph_timed = g_timing;
      cudaStream_t cs = ws->s_panel;
      TQ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
      TQ_CUDA(cudaEventRecord(ws->ev[2], cs));
      TQ_CUDA(cudaStreamWaitEvent(ws->s_update, ws->ev[2], 0));
      int rc = issue_levels(ws, cs, ws->s_update);
      cudaEventRecord(ws->ev[3], ws->s_update);
      cudaStreamWaitEvent(cs, ws->ev[3], 0);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(cs, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      TQ_CUDA(e);
      e = cudaGraphInstantiate(&ws->graph, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      TQ_CUDA(e);
    }
    TQ_CUDA(cudaGraphLaunch(ws->graph, stream));
    return 0;
  }
  // eager: fork/join the two internal streams around the caller's stream
  TQ_CUDA(cudaEventRecord(ws->ev[2], stream));
  TQ_CUDA(cudaStreamWaitEvent(ws->s_panel, ws->ev[2], 0));
  TQ_CUDA(cudaStreamWaitEvent(ws->s_update, ws->ev[2], 0));
  int rc = issue_levels(ws, ws->s_panel, ws->s_update);
  if (rc) return rc;
  TQ_CUDA(cudaEventRecord(ws->ev[2], ws->s_panel));
  TQ_CUDA(cudaStreamWaitEvent(stream, ws->ev[2], 0));
  TQ_CUDA(cudaEventRecord(ws->ev[3], ws->s_update));
  TQ_CUDA(cudaStreamWaitEvent(stream, ws->ev[3], 0));
  return 0;
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline (tileqr_factor_host)
// ---------------------------------------------------------------------------
using PFN_streamValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_streamValue32 g_wait_value = nullptr, g_write_value = nullptr;

// cuStreamWaitValue32 / cuStreamWriteValue32 through the runtime's driver
// entry points (no link dependency on libcuda).
static int stream_value_ops() {
  if (g_wait_value && g_write_value) return 0;
  void* f1 = nullptr;
  void* f2 = nullptr;
  cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = q1;
  TQ_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &f1, cudaEnableDefault, &q1));
  TQ_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &f2, cudaEnableDefault, &q2));
  if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !f1 || !f2) {
    set_error("tileqr_factor_host: stream memory operations unavailable");
    return TILEQR_ERR_CUDA;
  }
  g_wait_value = reinterpret_cast<PFN_streamValue32>(f1);
  g_write_value = reinterpret_cast<PFN_streamValue32>(f2);
  return 0;
}

#define TQ_CU(call)                                                         \
  do {                                                                      \
    CUresult r_ = (call);                                                   \
    if (r_ != CUDA_SUCCESS) {                                               \
      set_error("tileqr_factor_host: stream memory operation failed");      \
      return TILEQR_ERR_CUDA;                                               \
    }                                                                       \
  } while (0)

static int factor_host_dag(FactorWS* ws, const double* hA, int64_t lda, double* hR, int64_t ldr, double* hT,
                           int* d_info, cudaStream_t s) {
  const int64_t M = ws->M, N = ws->N, MT = ws->MT, NT = ws->NT;
  const int NB = ws->NB, IB = ws->IB;
  DagList& L = ws->dag_io;
  if (!L.d_items) {
    int rc = build_dag(ws, true);
    if (rc) return rc;
  }
  if (int rc = stream_value_ops()) return rc;
  if (!ws->io_ready) {
    // every resource of the host pipeline, or none: a partial set is freed
    // again so the next call retries from scratch
    auto release = [&]() {
      cudaFree(ws->st_in);
      cudaFree(ws->st_out);
      ws->st_in = ws->st_out = nullptr;
      if (ws->s_h2d) cudaStreamDestroy(ws->s_h2d);
      if (ws->s_d2h) cudaStreamDestroy(ws->s_d2h);
      ws->s_h2d = ws->s_d2h = nullptr;
      for (auto& e : ws->io_ev) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
      }
    };
    release();
    bool ok = cudaMalloc(&ws->st_in, (size_t)M * N * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ws->st_out, (size_t)M * N * sizeof(double)) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      release();
      set_error("tileqr_factor_host: device allocation of the staging buffers failed");
      return TILEQR_ERR_ALLOC;
    }
    ok = cudaStreamCreateWithFlags(&ws->s_h2d, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&ws->s_d2h, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& e : ws->io_ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      cudaError_t e = cudaGetLastError();
      release();
      return cuda_fail(e, "tileqr_factor_host pipeline setup", __FILE__, __LINE__);
    }
    ws->io_ready = true;
  }
  int* ctr = L.d_ctr;
  TQ_CUDA(cudaMemsetAsync(ctr, 0, (size_t)(L.ntasks + 257) * sizeof(int), s));
  TQ_CUDA(cudaEventRecord(ws->io_ev[0], s));
  TQ_CUDA(cudaStreamWaitEvent(ws->s_h2d, ws->io_ev[0], 0));
  TQ_CUDA(cudaStreamWaitEvent(ws->s_d2h, ws->io_ev[0], 0));
  auto counter = [&](int64_t task) { return (CUdeviceptr)(uintptr_t)(ctr + 257 + task); };
  // copy engine, host -> device: one tile column at a time (contiguous when
  // lda == M), each followed by its ARRIVE counter (the LOAD items of that
  // column wait on it)
  for (int64_t n = 0; n < NT; ++n) {
    const int64_t c0 = n * NB, nc = std::min<int64_t>(NB, N - c0);
    if (lda == M)
      TQ_CUDA(cudaMemcpyAsync(ws->st_in + c0 * M, hA + c0 * lda, (size_t)M * nc * sizeof(double),
                              cudaMemcpyHostToDevice, ws->s_h2d));
    else
      TQ_CUDA(cudaMemcpy2DAsync(ws->st_in + c0 * M, M * sizeof(double), hA + c0 * lda, lda * sizeof(double),
                                M * sizeof(double), nc, cudaMemcpyHostToDevice, ws->s_h2d));
    TQ_CU(g_write_value((CUstream)ws->s_h2d, counter(L.id_ar + n), 1, CU_STREAM_WRITE_VALUE_DEFAULT));
  }
  // the factorization, with LOAD / STORE items
  // the LOAD / STORE items read their parameters from device memory (a
  // by-value kernel argument would cost every item registers)
  const dag::DagIO io{M, N, M, ws->st_in, ws->st_out, d_info, MT, ws->tiles};
  if (!ws->d_io) TQ_CUDA(cudaMalloc(&ws->d_io, sizeof(dag::DagIO)));
  TQ_CUDA(cudaMemcpyAsync(ws->d_io, &io, sizeof io, cudaMemcpyHostToDevice, s));
  if (int rc = run_dag_list(ws, L, ws->d_io, s)) return rc;
  // copy engine, device -> host: each STORE group (tile rows [r0, r1) of a
  // column) as soon as its STORE item is done, in the simulated claim order;
  // a column's T with the group holding its diagonal tile (final with the
  // panel)
  const int64_t KT = std::min(MT, NT);
  for (const auto& sg : L.st_order) {
    const int64_t n = sg.first, g = sg.second;
    const int64_t c0 = n * NB, nc = std::min<int64_t>(NB, N - c0);
    const int64_t r0 = g * L.io_tiles * NB, r1 = std::min<int64_t>(M, (g + 1) * L.io_tiles * NB);
    TQ_CU(g_wait_value((CUstream)ws->s_d2h, counter(L.id_st + n * L.nio + g), 1, CU_STREAM_WAIT_VALUE_GEQ));
    if (r1 > r0) {
      if (r0 == 0 && r1 == M && ldr == M)
        TQ_CUDA(cudaMemcpyAsync(hR + c0 * ldr, ws->st_out + c0 * M, (size_t)M * nc * sizeof(double),
                                cudaMemcpyDeviceToHost, ws->s_d2h));
      else
        TQ_CUDA(cudaMemcpy2DAsync(hR + r0 + c0 * ldr, ldr * sizeof(double), ws->st_out + r0 + c0 * M,
                                  M * sizeof(double), (r1 - r0) * sizeof(double), nc, cudaMemcpyDeviceToHost,
                                  ws->s_d2h));
    }
    const int64_t gd = std::min<int64_t>(n < KT ? n : MT - 1, MT - 1) / L.io_tiles;
    if (g == gd) {
      const size_t tcol = (size_t)MT * IB * NB;
      TQ_CUDA(cudaMemcpyAsync(hT + n * tcol, ws->Tws + n * tcol, tcol * sizeof(double), cudaMemcpyDeviceToHost,
                              ws->s_d2h));
    }
  }
  TQ_CUDA(cudaEventRecord(ws->io_ev[1], ws->s_h2d));
  TQ_CUDA(cudaEventRecord(ws->io_ev[2], ws->s_d2h));
  TQ_CUDA(cudaStreamWaitEvent(s, ws->io_ev[1], 0));
  TQ_CUDA(cudaStreamWaitEvent(s, ws->io_ev[2], 0));
  return 0;
}

}  // namespace tileqr

namespace tileqr {
int panel_prof_read(unsigned long long* out, int reset);
int panel_prof_read_dag128(unsigned long long* out, int reset);
}
using namespace tileqr;

namespace tileqr {
bool panel_fast_supported(int NB, int IB);  // kernels_panel_fast.cu
bool panel_wide_supported(int NB, int IB);  // kernels_panel.cu

// Inner blocking the factorization runs at (R23): IB itself when
// the register-resident panels and the packed DMMA update take it, else
// lcm(IB, 8) when they take that (IB in {1, 2, 4} -> 8, 3, 6, 12 -> 24, 5,
// 10, 20 -> 40, 7, 14, 28 -> 56, where it divides NB): the same reflectors
// (applying the IBe-blocks of a panel in order is applying its IB-blocks in
// order, R22), with T returned at IB as the diagonal blocks of T at IBe.
// IB > 64 (whole-tile blockings such as IB = NB/2, NB): the largest of 32,
// 24, 16, 8 dividing IB (the dataflow kernel's inner blockings), with T at IB
// assembled afterwards from the factored tiles (its diagonal IBs-blocks are T
// at IBs).  Else IB (the generic panels and update).  TILEQR_NO_IB_LCM=1:
// always IB.
int effective_ib(int NB, int IB) {
  auto fast = [&](int ib) {
    return ib <= NB && NB % ib == 0 &&
           (panel_fast_supported(NB, ib) || (panel_wide_supported(NB, ib) && v2_supported(NB, ib)));
  };
  if (fast(IB)) return IB;
  const char* e = getenv("TILEQR_NO_IB_LCM");
  if (e && e[0] == '1') return IB;
  if (IB > 64) {
    for (int d : {32, 24, 16, 8})
      if (IB % d == 0 && fast(d)) return d;
    return IB;
  }
  const int l = std::lcm(IB, 8);
  return (l <= 64 && fast(l)) ? l : IB;
}
}  // namespace tileqr

extern "C" {

const char* tileqr_version(void) { return "tileqr 0.1 sm_100a (FP64 DMMA tile QR)"; }

const char* tileqr_last_error(void) { return g_last_error.c_str(); }

int tileqr_t_size(int64_t M, int64_t N, int NB, int IB, size_t* n_doubles) {
  if (M < 0) return arg_error(1, "tileqr_t_size", "M < 0");
  if (N < 0) return arg_error(2, "tileqr_t_size", "N < 0");
  if (NB == 0 && IB == 0) {  // "use the installed decision table" (table.cu)
    bool from_table = false;
    lookup_pair(M, N, 1, &NB, &IB, &from_table);
  }
  if (NB < 1 || NB > 512) return arg_error(3, "tileqr_t_size", "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(4, "tileqr_t_size", "IB must divide NB");
  if (!n_doubles) return arg_error(5, "tileqr_t_size", "NULL output");
  const int64_t MT = (M + NB - 1) / NB, NT = (N + NB - 1) / NB;
  *n_doubles = (size_t)(MT * NT) * IB * NB;
  return 0;
}

int tileqr_num_levels(int64_t MT, int64_t NT, int64_t* n_levels) {
  if (MT < 0) return arg_error(1, "tileqr_num_levels", "MT < 0");
  if (NT < 0) return arg_error(2, "tileqr_num_levels", "NT < 0");
  if (!n_levels) return arg_error(3, "tileqr_num_levels", "NULL output");
  *n_levels = num_levels(MT, NT);
  return 0;
}

int tileqr_factor(int64_t M, int64_t N, double* A, int64_t lda, int NB, int IB, double* T,
                  int* d_info, tileqr_stream_t stream) {
  static const char* fn = "tileqr_factor";
  if (M < 0) return arg_error(1, fn, "M < 0");
  if (N < 0) return arg_error(2, fn, "N < 0");
  if (!A && M > 0 && N > 0) return arg_error(3, fn, "A is NULL");
  if (lda < std::max<int64_t>(1, M)) return arg_error(4, fn, "lda < max(1,M)");
  if (NB == 0 && IB == 0) {  // "use the installed decision table" (table.cu)
    bool from_table = false;
    lookup_pair(M, N, 1, &NB, &IB, &from_table);
  }
  if (NB < 1 || NB > 512) return arg_error(5, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(6, fn, "IB must divide NB");
  if (!T && M > 0 && N > 0) return arg_error(7, fn, "T is NULL");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_info) {
    int rc = launch_zero_int(d_info, s);
    if (rc) return rc;
  }
  if (M == 0 || N == 0) return 0;
  int dev;
  TQ_CUDA(cudaGetDevice(&dev));
  const int IBe = effective_ib(NB, IB);
  std::lock_guard<std::mutex> lock(g_mu);
  FactorWS* ws = nullptr;
  auto it = g_ws.find(std::make_tuple(dev, M, N, NB, IBe));
  if (it != g_ws.end()) {
    ws = it->second.get();
  } else {
    int rc = create_ws(dev, M, N, NB, IBe, &ws);
    if (rc) return rc;
  }
  if (ws->used) TQ_CUDA(cudaStreamWaitEvent(s, ws->last_use, 0));  // previous user of the workspace
  ws->stamp = ++g_ws_clock;
  int rc = launch_layout_to_tiles(M, N, A, lda, NB, ws->MT, ws->NT, ws->tiles, d_info, s);
  if (rc) return rc;
  if ((rc = run_levels(ws, s))) return rc;
  if ((rc = launch_tiles_to_layout(M, N, A, lda, NB, ws->MT, ws->NT, ws->tiles, s))) return rc;
  if (IBe == IB) {
    TQ_CUDA(cudaMemcpyAsync(T, ws->Tws, (size_t)ws->MT * ws->NT * IB * NB * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  } else if (IBe > IB) {
    if ((rc = launch_t_extract(ws->Tws, IBe, T, IB, NB, ws->MT * ws->NT, s))) return rc;
  } else {
    TQ_CUDA(cudaMemsetAsync(T, 0, (size_t)ws->MT * ws->NT * IB * NB * sizeof(double), s));
    int nsm = 148;
    TQ_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t KT = std::min(ws->MT, ws->NT);
    if ((rc = launch_t_assemble_big(ws->tiles, ws->Tws, T, NB, IB, IBe, ws->MT, KT, KT, 1, 0, nsm, s)))
      return rc;
  }
  TQ_CUDA(cudaEventRecord(ws->last_use, s));
  ws->used = true;
  return 0;
}

int tileqr_factor_host(int64_t M, int64_t N, const double* h_A, int64_t lda, int NB, int IB, double* h_R,
                       int64_t ldr, double* h_T, int* d_info, tileqr_stream_t stream) {
  static const char* fn = "tileqr_factor_host";
  if (M < 0) return arg_error(1, fn, "M < 0");
  if (N < 0) return arg_error(2, fn, "N < 0");
  if (!h_A && M > 0 && N > 0) return arg_error(3, fn, "h_A is NULL");
  if (lda < std::max<int64_t>(1, M)) return arg_error(4, fn, "lda < max(1,M)");
  if (NB == 0 && IB == 0) {  // "use the installed decision table" (table.cu)
    bool from_table = false;
    lookup_pair(M, N, 1, &NB, &IB, &from_table);
  }
  if (NB < 1 || NB > 512) return arg_error(5, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(6, fn, "IB must divide NB");
  if (!h_R && M > 0 && N > 0) return arg_error(7, fn, "h_R is NULL");
  if (ldr < std::max<int64_t>(1, M)) return arg_error(8, fn, "ldr < max(1,M)");
  if (!h_T && M > 0 && N > 0) return arg_error(9, fn, "h_T is NULL");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_info) {
    int rc = launch_zero_int(d_info, s);
    if (rc) return rc;
  }
  if (M == 0 || N == 0) return 0;
  int dev;
  TQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  FactorWS* ws = nullptr;
  auto it = g_ws.find(std::make_tuple(dev, M, N, NB, IB));
  if (it != g_ws.end()) {
    ws = it->second.get();
  } else {
    int rc = create_ws(dev, M, N, NB, IB, &ws);
    if (rc) return rc;
  }
  if (ws->used) TQ_CUDA(cudaStreamWaitEvent(s, ws->last_use, 0));  // previous user of the workspace
  ws->stamp = ++g_ws_clock;
  if (ws->use_dag) {
    const int rc = factor_host_dag(ws, h_A, lda, h_R, ldr, h_T, d_info, s);
    if (rc) return rc;
    TQ_CUDA(cudaEventRecord(ws->last_use, s));
    ws->used = true;
    return 0;
  }
  // level-synchronous schedule: copy in, factor, copy out (no overlap)
  if (!ws->st_in) {
    if (cudaMalloc(&ws->st_in, (size_t)M * N * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      set_error("tileqr_factor_host: device allocation of the staging buffer failed");
      return TILEQR_ERR_ALLOC;
    }
  }
  TQ_CUDA(cudaMemcpy2DAsync(ws->st_in, M * sizeof(double), h_A, lda * sizeof(double), M * sizeof(double), N,
                            cudaMemcpyHostToDevice, s));
  int rc = launch_layout_to_tiles(M, N, ws->st_in, M, NB, ws->MT, ws->NT, ws->tiles, d_info, s);
  if (rc) return rc;
  if ((rc = run_levels(ws, s))) return rc;
  if ((rc = launch_tiles_to_layout(M, N, ws->st_in, M, NB, ws->MT, ws->NT, ws->tiles, s))) return rc;
  TQ_CUDA(cudaMemcpy2DAsync(h_R, ldr * sizeof(double), ws->st_in, M * sizeof(double), M * sizeof(double), N,
                            cudaMemcpyDeviceToHost, s));
  TQ_CUDA(cudaMemcpyAsync(h_T, ws->Tws, (size_t)ws->MT * ws->NT * IB * NB * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
  TQ_CUDA(cudaEventRecord(ws->last_use, s));
  ws->used = true;
  return 0;
}

int tileqr_apply_qt(char trans, int64_t M, int64_t NRHS, int64_t K, const double* A, int64_t lda,
                    const double* T, int NB, int IB, double* B, int64_t ldb,
                    tileqr_stream_t stream) {
  static const char* fn = "tileqr_apply_qt";
  if (trans != 'T' && trans != 'N' && trans != 't' && trans != 'n')
    return arg_error(1, fn, "trans not 'T' or 'N'");
  if (M < 0) return arg_error(2, fn, "M < 0");
  if (NRHS < 0) return arg_error(3, fn, "NRHS < 0");
  if (K < 0) return arg_error(4, fn, "K < 0");
  if (!A && M > 0 && K > 0) return arg_error(5, fn, "A is NULL");
  if (lda < std::max<int64_t>(1, M)) return arg_error(6, fn, "lda < max(1,M)");
  if (!T && M > 0 && K > 0) return arg_error(7, fn, "T is NULL");
  if (NB == 0 && IB == 0) {  // "use the installed decision table" (table.cu)
    bool from_table = false;
    lookup_pair(M, K, 1, &NB, &IB, &from_table);
  }
  if (NB < 1 || NB > 512) return arg_error(8, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(9, fn, "IB must divide NB");
  if (!B && M > 0 && NRHS > 0) return arg_error(10, fn, "B is NULL");
  if (ldb < std::max<int64_t>(1, M)) return arg_error(11, fn, "ldb < max(1,M)");
  if (M == 0 || NRHS == 0 || K == 0) return 0;
  const bool tr = (trans == 'T' || trans == 't');
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t MT = (M + NB - 1) / NB, KTt = (K + NB - 1) / NB, BT = (NRHS + NB - 1) / NB;
  const int64_t KT = std::min(MT, KTt);
  const size_t tile = (size_t)NB * NB;
  double *Vt = nullptr, *Bt = nullptr;
  void** dp = nullptr;
  // per launch: LARFB tasks (k, n) n < BT; SSRFB tasks (k, m, n) n < BT
  const int64_t nlaunch_s = KT * MT;  // upper bound
  const size_t nptr = (size_t)KT * BT * 3 + (size_t)nlaunch_s * BT * 4;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&Vt), tile * MT * KT * sizeof(double), s)) return rc_;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&Bt), tile * MT * BT * sizeof(double), s)) return rc_;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&dp), nptr * sizeof(void*), s)) return rc_;
  int rc = launch_v_to_tiles(M, K, A, lda, NB, MT, KT, Vt, s);
  if (!rc) rc = launch_layout_to_tiles(M, NRHS, B, ldb, NB, MT, BT, Bt, nullptr, s);
  std::vector<void*> hp(nptr);
  auto vt = [&](int64_t m, int64_t k) { return (void*)(Vt + (size_t)(m + k * MT) * tile); };
  auto bt = [&](int64_t m, int64_t n) { return (void*)(Bt + (size_t)(m + n * MT) * tile); };
  auto tt = [&](int64_t m, int64_t k) { return (void*)(T + (size_t)(m + k * MT) * IB * NB); };
  struct L { bool larfb; size_t off; int64_t cnt; };
  std::vector<L> seq;
  size_t o = 0;
  for (int64_t kk = 0; kk < KT; ++kk) {
    const int64_t k = tr ? kk : KT - 1 - kk;
    auto add_larfb = [&]() {
      seq.push_back({true, o, BT});
      for (int64_t n = 0; n < BT; ++n) {
        hp[o + n] = vt(k, k);
        hp[o + BT + n] = tt(k, k);
        hp[o + 2 * BT + n] = bt(k, n);
      }
      o += 3 * BT;
    };
    if (tr) add_larfb();
    for (int64_t mm = k + 1; mm < MT; ++mm) {
      const int64_t m = tr ? mm : MT - 1 - (mm - (k + 1));
      seq.push_back({false, o, BT});
      for (int64_t n = 0; n < BT; ++n) {
        hp[o + n] = vt(m, k);
        hp[o + BT + n] = tt(m, k);
        hp[o + 2 * BT + n] = bt(k, n);
        hp[o + 3 * BT + n] = bt(m, n);
      }
      o += 4 * BT;
    }
    if (!tr) add_larfb();
  }
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(dp, hp.data(), o * sizeof(void*), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync", __FILE__, __LINE__);
  }
  double** d = reinterpret_cast<double**>(dp);
  for (const L& l : seq) {
    if (rc) break;
    if (l.larfb)
      rc = launch_larfb(tr, NB, IB, (int)l.cnt, (const double* const*)(d + l.off),
                        (const double* const*)(d + l.off + l.cnt), d + l.off + 2 * l.cnt, NB, s);
    else
      rc = launch_ssrfb(tr, NB, IB, (int)l.cnt, (const double* const*)(d + l.off),
                        (const double* const*)(d + l.off + l.cnt), d + l.off + 2 * l.cnt,
                        d + l.off + 3 * l.cnt, NB, s);
  }
  if (!rc) rc = launch_tiles_to_layout(M, NRHS, B, ldb, NB, MT, BT, Bt, s);
  cudaFreeAsync(Vt, s);
  cudaFreeAsync(Bt, s);
  cudaFreeAsync(dp, s);
  return rc;
}

// Batched Q^T update through the factorization's packed-reflector kernel:
// pack (V, T) into stream-ordered scratch, then run update_v2.
// IB the batched LARFB / SSRFB entry points run through lcm(IB, 8) (R23): the
// T assembly at IBe (wide_t_kernel, a sequential recurrence per tile) costs
// about as much as the update itself, which pays only against the 4-8x slower
// generic kernels of IB < 8 (4096-pair SSRFB at (128, 4): 12.9 -> 16.7
// TFLOP/s; at (160, 10) it would fall from 15.1 to 10.3, so IB >= 8 keeps the
// staged DMMA update).  tileqr_factor and Step 1 run IBe directly (no assembly).
// IB > 64: T at IBs (a divisor of IB) is the caller's T's diagonal blocks.
static int batched_ib(int NB, int IB) { return (IB < 8 || IB > 64) ? effective_ib(NB, IB) : IB; }

static int packed_update(bool larfb, int NB, int IB, int batch, const double* const* V, const double* const* T,
                         double* const* C1, double* const* C2, cudaStream_t s) {
  const int IBe = batched_ib(NB, IB);
  if (IBe != IB) {  // R23: T at IBe from V and tau (IBe > IB) or T's diagonal blocks (IBe < IB), then the IBe update
    double* tb = nullptr;
    double** tp = nullptr;
    if (int rc_ = stream_alloc(reinterpret_cast<void**>(&tb), (size_t)batch * IBe * NB * sizeof(double), s)) return rc_;
    if (int rc_ = stream_alloc(reinterpret_cast<void**>(&tp), (size_t)batch * sizeof(double*), s)) return rc_;
    int rc = launch_fill_ptrs(tp, tb, (size_t)IBe * NB, batch, s);
    if (!rc) rc = IBe > IB ? launch_t_assemble(!larfb, NB, IBe, IB, batch, V, T, tp, s)
                           : launch_t_extract_ptrs(T, IB, tp, IBe, NB, batch, s);
    if (!rc) rc = packed_update(larfb, NB, IBe, batch, V, tp, C1, C2, s);
    cudaFreeAsync(tb, s);
    cudaFreeAsync(tp, s);
    return rc;
  }
  const size_t pd = v2_pk_doubles(NB, IB);
  double* buf = nullptr;
  double** ptr = nullptr;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&buf), pd * batch * sizeof(double), s)) return rc_;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&ptr), (size_t)batch * sizeof(double*), s)) return rc_;
  int rc = launch_fill_ptrs(ptr, buf, pd, batch, s);
  if (!rc) rc = launch_pack(larfb, NB, IB, batch, V, T, ptr, s);
  if (!rc) rc = launch_update_pk(larfb, NB, IB, batch, ptr, C1, C2, s);
  cudaFreeAsync(buf, s);
  cudaFreeAsync(ptr, s);
  return rc;
}

static int check_batched(const char* fn, int NB, int IB, int batch) {
  if (NB < 1 || NB > 512) return arg_error(1, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(2, fn, "IB must divide NB");
  if (batch < 0) return arg_error(3, fn, "batch < 0");
  return 0;
}

int tileqr_geqrt_batched(int NB, int IB, int batch, double* const* A, double* const* T,
                         tileqr_stream_t stream) {
  static const char* fn = "tileqr_geqrt_batched";
  if (int rc = check_batched(fn, NB, IB, batch)) return rc;
  if (batch == 0) return 0;
  if (!A) return arg_error(4, fn, "A is NULL");
  if (!T) return arg_error(5, fn, "T is NULL");
  return launch_geqrt(NB, IB, batch, A, T, reinterpret_cast<cudaStream_t>(stream));
}

int tileqr_tsqrt_batched(int NB, int IB, int batch, double* const* R, double* const* A2,
                         double* const* T, tileqr_stream_t stream) {
  static const char* fn = "tileqr_tsqrt_batched";
  if (int rc = check_batched(fn, NB, IB, batch)) return rc;
  if (batch == 0) return 0;
  if (!R) return arg_error(4, fn, "R is NULL");
  if (!A2) return arg_error(5, fn, "A2 is NULL");
  if (!T) return arg_error(6, fn, "T is NULL");
  return launch_tsqrt(NB, IB, batch, R, A2, T, reinterpret_cast<cudaStream_t>(stream));
}

int tileqr_larfb_batched(char trans, int NB, int IB, int batch, const double* const* V,
                         const double* const* T, double* const* C, int ncols,
                         tileqr_stream_t stream) {
  static const char* fn = "tileqr_larfb_batched";
  if (trans != 'T' && trans != 'N' && trans != 't' && trans != 'n')
    return arg_error(1, fn, "trans not 'T' or 'N'");
  if (NB < 1 || NB > 512) return arg_error(2, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(3, fn, "IB must divide NB");
  if (batch < 0) return arg_error(4, fn, "batch < 0");
  if (batch == 0) return 0;
  if (!V) return arg_error(5, fn, "V is NULL");
  if (!T) return arg_error(6, fn, "T is NULL");
  if (!C) return arg_error(7, fn, "C is NULL");
  if (ncols < 1 || ncols > NB) return arg_error(8, fn, "ncols not in [1, NB]");
  const bool tr = trans == 'T' || trans == 't';
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (tr && ncols == NB && v2_supported(NB, batched_ib(NB, IB)))  // the factorization's kernel: pack, then update
    return packed_update(true, NB, IB, batch, V, T, nullptr, C, s);
  return launch_larfb(tr, NB, IB, batch, V, T, C, ncols, s);
}

int tileqr_ssrfb_batched(char trans, int NB, int IB, int batch, const double* const* V2,
                         const double* const* T, double* const* C1, double* const* C2, int ncols,
                         tileqr_stream_t stream) {
  static const char* fn = "tileqr_ssrfb_batched";
  if (trans != 'T' && trans != 'N' && trans != 't' && trans != 'n')
    return arg_error(1, fn, "trans not 'T' or 'N'");
  if (NB < 1 || NB > 512) return arg_error(2, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(3, fn, "IB must divide NB");
  if (batch < 0) return arg_error(4, fn, "batch < 0");
  if (batch == 0) return 0;
  if (!V2) return arg_error(5, fn, "V2 is NULL");
  if (!T) return arg_error(6, fn, "T is NULL");
  if (!C1) return arg_error(7, fn, "C1 is NULL");
  if (!C2) return arg_error(8, fn, "C2 is NULL");
  if (ncols < 1 || ncols > NB) return arg_error(9, fn, "ncols not in [1, NB]");
  const bool tr = trans == 'T' || trans == 't';
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (tr && ncols == NB && v2_supported(NB, batched_ib(NB, IB)))
    return packed_update(false, NB, IB, batch, V2, T, C1, C2, s);
  return launch_ssrfb(tr, NB, IB, batch, V2, T, C1, C2, ncols, s);
}

int tileqr_packed_size(int NB, int IB, size_t* n_doubles) {
  if (!n_doubles) return arg_error(3, "tileqr_packed_size", "NULL output");
  *n_doubles = (valid_nb_ib(NB, IB) && v2_supported(NB, IB)) ? v2_pk_doubles(NB, IB) : 0;
  return 0;
}

int tileqr_pack_batched(int larfb, int NB, int IB, int batch, const double* const* V, const double* const* T,
                        double* const* Pk, tileqr_stream_t stream) {
  static const char* fn = "tileqr_pack_batched";
  if (!valid_nb_ib(NB, IB) || !v2_supported(NB, IB)) return arg_error(1, fn, "(NB, IB) has no packed form");
  if (batch < 0) return arg_error(3, fn, "batch < 0");
  if (batch == 0) return 0;
  if (!V) return arg_error(4, fn, "V is NULL");
  if (!T) return arg_error(5, fn, "T is NULL");
  if (!Pk) return arg_error(6, fn, "Pk is NULL");
  return launch_pack(larfb != 0, NB, IB, batch, V, T, Pk, reinterpret_cast<cudaStream_t>(stream));
}

int tileqr_update_packed_batched(int larfb, int NB, int IB, int batch, const double* const* Pk,
                                 double* const* C1, double* const* C2, tileqr_stream_t stream) {
  static const char* fn = "tileqr_update_packed_batched";
  if (!valid_nb_ib(NB, IB) || !v2_supported(NB, IB)) return arg_error(1, fn, "(NB, IB) has no packed form");
  if (batch < 0) return arg_error(3, fn, "batch < 0");
  if (batch == 0) return 0;
  if (!Pk) return arg_error(4, fn, "Pk is NULL");
  if (!larfb && !C1) return arg_error(5, fn, "C1 is NULL");
  if (!C2) return arg_error(6, fn, "C2 is NULL");
  return launch_update_pk(larfb != 0, NB, IB, batch, Pk, C1, C2, reinterpret_cast<cudaStream_t>(stream));
}

int tileqr_rng_uniform(int64_t M, int64_t N, double* A, int64_t lda, uint64_t seed,
                       uint64_t offset, tileqr_stream_t stream) {
  static const char* fn = "tileqr_rng_uniform";
  if (M < 0) return arg_error(1, fn, "M < 0");
  if (N < 0) return arg_error(2, fn, "N < 0");
  if (!A && M > 0 && N > 0) return arg_error(3, fn, "A is NULL");
  if (lda < std::max<int64_t>(1, M)) return arg_error(4, fn, "lda < max(1,M)");
  return launch_rng_uniform(M, N, A, lda, seed, offset, reinterpret_cast<cudaStream_t>(stream));
}

const char* tileqr_ssrfb_impl(int NB, int IB) { return ssrfb_impl_name(NB, IB); }

// Diagnostic (not in the header): item idx of the dataflow work list of a cached
// shape -> out[5] = {kind, k, m, n, sub-task or slab column}.
int tileqr_debug_dag_item(int64_t M, int64_t N, int NB, int IB, int64_t idx, int* out) {
  int dev;
  TQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_ws.find(std::make_tuple(dev, M, N, NB, effective_ib(NB, IB)));
  if (it == g_ws.end() || !it->second->use_dag) return TILEQR_ERR_NOT_INIT;
  FactorWS* ws = it->second.get();
  const DagList& L = ws->dag_last ? *ws->dag_last : ws->dag_plain;
  if (idx < 0 || idx >= L.nitems) return -5;
  for (int q = 0; q < 5; ++q) out[q] = L.item_info[5 * idx + q];
  return 0;
}

// Diagnostic (not in the header): accumulated phase cycles of the fast panel kernel.
int tileqr_debug_panel_prof(unsigned long long* out, int reset) { return tileqr::panel_prof_read(out, reset); }
// Diagnostic: the same counters of the panel bodies inside the NB=128 DAG kernel.
int tileqr_debug_dag_panel_prof(unsigned long long* out, int reset) {
  return tileqr::panel_prof_read_dag128(out, reset);
}

const char* tileqr_factor_schedule(int NB, int IB) {
  if (!valid_nb_ib(NB, IB)) return "invalid";
  return dag_enabled(NB, IB) ? "dag" : "levels";
}

int tileqr_factor_plan(int64_t M, int64_t N, int NB, int IB, int64_t* h_out) {
  static const char* fn = "tileqr_factor_plan";
  if (M < 0) return arg_error(1, fn, "M < 0");
  if (N < 0) return arg_error(2, fn, "N < 0");
  if (NB < 1 || NB > 512) return arg_error(3, fn, "NB not in [1, 512]");
  if (IB < 1 || IB > NB || NB % IB) return arg_error(4, fn, "IB must divide NB");
  if (!h_out) return arg_error(5, fn, "NULL output");
  const int64_t MT = (M + NB - 1) / NB, NT = (N + NB - 1) / NB;
  const int64_t nlev = (M == 0 || N == 0) ? 0 : num_levels(MT, NT);
  HostTasks h;
  build_tasks(MT, NT, h, nlev);
  int64_t launches = 0, cnt[4] = {0, 0, 0, 0};
  for (int64_t t = 0; t < nlev; ++t) {
    const int64_t c[4] = {(int64_t)h.G[t].size(), (int64_t)h.T[t].size() / 2,
                          (int64_t)h.L[t].size() / 2, (int64_t)h.S[t].size() / 3};
    for (int q = 0; q < 4; ++q) cnt[q] += c[q];
    const char* cf = getenv("TILEQR_CRITICAL_FIRST");
    if (cf && cf[0] == '1')  // panel stream: G, T, critical L/S; update stream: bulk L/S
      launches += (c[0] > 0) + (c[1] > 0) + (h.Lc[t] > 0) + (h.Sc[t] > 0) + (c[2] > h.Lc[t]) +
                  (c[3] > h.Sc[t]);
    else
      launches += (c[0] > 0) + (c[1] > 0) + (c[2] > 0) + (c[3] > 0);
  }
  if (dag_enabled(NB, IB)) launches = nlev > 0 ? 1 : 0;  // one persistent dataflow kernel
  h_out[0] = nlev;
  h_out[1] = launches + ((M == 0 || N == 0) ? 0 : 3);  // + zero-info, layout in, layout out
  for (int q = 0; q < 4; ++q) h_out[2 + q] = cnt[q];
  h_out[6] = MT;
  h_out[7] = NT;
  return 0;
}

void tileqr_set_kernel_timing(int mask) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_timing = mask & 31;
}

int tileqr_kernel_times(int64_t M, int64_t N, int NB, int IB, int kind, double* h_total_ms,
                        int64_t* h_launches, int64_t* h_tasks) {
  static const char* fn = "tileqr_kernel_times";
  if (kind < 0 || kind > 5) return arg_error(5, fn, "kind not in 0..5");
  if (!h_total_ms || !h_launches || !h_tasks) return arg_error(6, fn, "NULL output");
  int dev;
  TQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_ws.find(std::make_tuple(dev, M, N, NB, effective_ib(NB, IB)));
  if (it == g_ws.end()) {
    set_error("tileqr_kernel_times: no factorization of this shape has run");
    return TILEQR_ERR_NOT_INIT;
  }
  FactorWS* ws = it->second.get();
  double tot = 0.0;
  int64_t nl = 0, nt = 0;
  if (kind == 5) {  // timing bit 4: dataflow-kernel launches since the last read (sum, count); resets
    double t = 0.0;
    for (size_t i = 0; i < ws->acc_n; ++i) {
      float ms = 0.f;
      TQ_CUDA(cudaEventElapsedTime(&ms, ws->acc_ev[2 * i], ws->acc_ev[2 * i + 1]));
      t += ms;
    }
    *h_total_ms = t;
    *h_launches = (int64_t)ws->acc_n;
    *h_tasks = ws->dag_last ? ws->dag_last->ntasks : 0;
    ws->acc_n = 0;
    return 0;
  }
  if (ws->use_dag) {
    // dataflow kernel: busy time of the items of this kind summed over CTAs
    // (inputs ready -> completion published); kind 4 = the whole DAG kernel
    if (!ws->dag_timed) {
      set_error("tileqr_kernel_times: the last run was not timed");
      return TILEQR_ERR_NOT_INIT;
    }
    if (kind == 4) {  // the kernel: duration, launches = resident CTAs (work-item slots), tasks
      float ms = 0.f;
      TQ_CUDA(cudaEventElapsedTime(&ms, ws->dag_ev[0], ws->dag_ev[1]));
      *h_total_ms = ms;
      *h_launches = ws->dag_grid;
      *h_tasks = ws->dag_last ? ws->dag_last->ntasks : 0;
      return 0;
    }
    const DagList& L = *ws->dag_last;
    std::vector<unsigned long long> pr((size_t)L.nitems * 3);
    TQ_CUDA(cudaMemcpy(pr.data(), ws->d_prof, pr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    const int cols = dag::dag_cols(ws->NB);
    const int nslab = (ws->NB + cols - 1) / cols;
    for (int i = 0; i < L.nitems; ++i) {
      if (L.item_kind[i] != kind) continue;
      tot += (double)(pr[3 * i + 2] - pr[3 * i + 1]) * 1e-6;
      ++nl;
    }
    nt = (kind >= 2) ? nl / nslab : nl;
    *h_total_ms = tot;
    *h_launches = nl;
    *h_tasks = nt;
    return 0;
  }
  for (size_t i = 0; i < ws->rec_used; ++i) {
    const FactorWS::Rec& r = ws->recs[i];
    if (r.kind != kind) continue;
    float ms = 0.f;
    TQ_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    tot += ms;
    ++nl;
    nt += r.tasks;
  }
  *h_total_ms = tot;
  *h_launches = nl;
  *h_tasks = nt;
  return 0;
}

int tileqr_kernel_trace(int64_t M, int64_t N, int NB, int IB, int64_t max_recs, double* h_t0_ms,
                        double* h_t1_ms, int* h_kind, int64_t* h_level, int64_t* h_tasks,
                        int64_t* h_count) {
  static const char* fn = "tileqr_kernel_trace";
  if (max_recs < 0) return arg_error(5, fn, "max_recs < 0");
  if (!h_count) return arg_error(11, fn, "NULL output");
  int dev;
  TQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_ws.find(std::make_tuple(dev, M, N, NB, effective_ib(NB, IB)));
  if (it == g_ws.end()) {
    set_error("tileqr_kernel_trace: no factorization of this shape has run");
    return TILEQR_ERR_NOT_INIT;
  }
  FactorWS* ws = it->second.get();
  if (ws->use_dag) {
    // per work item: start = inputs ready, end = completion published (ns
    // clock of the device), relative to the earliest claim
    if (!ws->dag_timed) {
      set_error("tileqr_kernel_trace: the last run was not timed");
      return TILEQR_ERR_NOT_INIT;
    }
    const DagList& L = *ws->dag_last;
    std::vector<unsigned long long> pr((size_t)L.nitems * 3);
    TQ_CUDA(cudaMemcpy(pr.data(), ws->d_prof, pr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < L.nitems; ++i) t0 = std::min(t0, pr[3 * i]);
    *h_count = L.nitems;
    for (int64_t i = 0; i < L.nitems && i < max_recs; ++i) {
      if (h_t0_ms) h_t0_ms[i] = (double)(pr[3 * i + 1] - t0) * 1e-6;
      if (h_t1_ms) h_t1_ms[i] = (double)(pr[3 * i + 2] - t0) * 1e-6;
      if (h_kind) h_kind[i] = L.item_kind[i];
      if (h_level) h_level[i] = L.item_level[i];
      // DAG: claim time (ns from origin, 1024 ns resolution), the low 10 bits
      // the item's tag (SM id | C2 staged << 9, dag.cuh)
      if (h_tasks) h_tasks[i] = (int64_t)(((pr[3 * i] - t0) & ~0x3ffull) | (pr[3 * i] & 0x3ffull));
    }
    return 0;
  }
  *h_count = (int64_t)ws->rec_used;
  if (ws->rec_used == 0) return 0;
  const cudaEvent_t origin = ws->recs[0].a;
  for (size_t i = 0; i < ws->rec_used && (int64_t)i < max_recs; ++i) {
    const FactorWS::Rec& r = ws->recs[i];
    float a = 0.f, b = 0.f;
    TQ_CUDA(cudaEventElapsedTime(&a, origin, r.a));
    TQ_CUDA(cudaEventElapsedTime(&b, origin, r.b));
    if (h_t0_ms) h_t0_ms[i] = a;
    if (h_t1_ms) h_t1_ms[i] = b;
    if (h_kind) h_kind[i] = r.kind;
    if (h_level) h_level[i] = r.level;
    if (h_tasks) h_tasks[i] = r.tasks;
  }
  return 0;
}

}  // extern "C"

namespace tileqr {
// Free the cached workspace of one shape once its last use has completed
// (the tuner calls this after timing a Step-2 candidate, so tuning does not
// keep one workspace per candidate resident).
void release_ws(int dev, int64_t M, int64_t N, int NB, int IB) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_ws.find(std::make_tuple(dev, M, N, NB, effective_ib(NB, IB)));
  if (it == g_ws.end()) return;
  if (it->second->used) cudaEventSynchronize(it->second->last_use);
  g_ws.erase(it);
}
}  // namespace tileqr

extern "C" {

void tileqr_finalize(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_ws.clear();
}

}  // extern "C"
