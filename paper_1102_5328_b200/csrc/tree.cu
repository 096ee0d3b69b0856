// tree.cu -- the tall-skinny / communication-avoiding variant of the tile QR
// ("tall and skinny" matrices,
// communication-avoiding QR with p domains as an added tunable).
//
// The flat TSQRT chain of each panel (sequential in m) is
// replaced by a reduction tree (R20, the oracle's
// oracle_tileqr_factor_tree): tile rows are split into domains of BS rows
// [d*BS, (d+1)*BS); at panel k each domain's first row >= k is its head,
// factored by GEQRT, the domain's other rows join it by the flat TSQRT chain,
// and the heads are merged pairwise by TTQRT (triangle on triangle) along a
// binary tree (distance 1, 2, 4, ...).  The trailing tiles see LARFB, the
// SSRFB chain and TTMQRT in the same order.  The critical path of a panel
// drops from MT - k TSQRT steps to BS + log2(MT/BS) steps: for a tall
// matrix (MT >> NT) this is what bounds the factorization.
//
// Execution: the persistent dataflow kernel (dag.cuh, mode kModeTree) on a
// task graph whose dependencies are derived here by tracking, in the
// sequential order of the algorithm, the last writer of every tile (updates)
// and of every sub-task's R rows (panel tasks); claim order from the same
// list-schedule simulation as the flat tree (sched.h).  TTQRT items are the
// register-resident panel kernel with the TT flag (panel_fast.cuh), TTMQRT
// items the packed-reflector update with the TT flag (update_v2.cuh, zero row
// blocks skipped).  Every tile (m, k) has two packed-reflector slots: its
// GEQRT / TSQRT reflectors and, for a merged head, its TTQRT reflectors.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <functional>
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

int launch_ttqrt_fast(int NB, int IB, int batch, double* const* R, double* const* A2, double* const* T,
                      cudaStream_t s, double* const* Pk);

namespace {

// heads of panel k (R20)
std::vector<int64_t> heads_of(int64_t MT, int64_t k, int64_t BS) {
  std::vector<int64_t> h;
  for (int64_t d = k / BS; d * BS < MT; ++d) h.push_back(std::max(d * BS, k));
  return h;
}
int64_t domain_end(int64_t h, int64_t BS, int64_t MT) { return std::min((h / BS + 1) * BS, MT); }

struct TreeWS {
  int64_t M = 0, N = 0, MT = 0, NT = 0, BS = 1;
  int NB = 0, IB = 0;
  double* tiles = nullptr;
  double* Tws = nullptr;   // 2 * MT*NT*IB*NB: T then T2
  double* Vpk = nullptr;   // 2 slots per tile (m, k), k < KT: [GEQRT/TSQRT | TTQRT]
  size_t pk_dbl = 0;
  dag::Item* d_items = nullptr;
  int nitems = 0, ntasks = 0, nsm = 0;
  int* d_ctr = nullptr;
  cudaEvent_t last_use = nullptr;
  bool used = false;
  ~TreeWS() {
    cudaFree(tiles);
    cudaFree(Tws);
    cudaFree(Vpk);
    cudaFree(d_items);
    cudaFree(d_ctr);
    if (last_use) cudaEventDestroy(last_use);
  }
};

std::mutex g_tree_mu;
std::map<std::tuple<int, int64_t, int64_t, int, int, int64_t>, std::unique_ptr<TreeWS>> g_tree;

struct TTask {
  int kind;
  int64_t a, b, k, n;  // GEQRT: a = head; TSQRT: a = head, b = member; TTQRT: a <- b; updates: + column n
  int s;
};

// The tree variant's task graph (dependencies by last-writer tracking) and
// its claim order (list-schedule simulation over `workers` CTAs); host only.
struct TreePlan {
  std::vector<sched::Task> tk;
  std::vector<TTask> info;
  std::vector<sched::Slot> order;
  int SC = 0, NS = 1, cols = 0, nslab = 1;
  std::function<int(int)> parts;
};

int build_tree_plan(int64_t MT, int64_t NT, int NB, int IB, int64_t BS, int SC, int workers, TreePlan* out) {
  const int64_t KT = std::min(MT, NT);
  const int NS = NB / SC;
  const int cols = dag::dag_cols(NB), nslab = (NB + cols - 1) / cols;
  std::vector<sched::Task>& tk = out->tk;
  std::vector<TTask>& info = out->info;
  tk.clear();
  info.clear();
  auto add = [&](int kind, int64_t a, int64_t b, int64_t k, int64_t n, int s, int level,
                 std::initializer_list<int64_t> deps) {
    sched::Task t{kind, (int)k, (int)b, (int)n, level, 0, {0, 0, 0}, s};
    for (int64_t d : deps)  // -1: no producer (the input / no earlier sub-task)
      if (d != -1) t.dep[t.ndep++] = (int)d;
    tk.push_back(t);
    info.push_back({kind, a, b, k, n, s});
    return (int64_t)tk.size() - 1;
  };
  // last writer of tile (m, n) (-1: the input), and of the R rows of
  // sub-task s of tile (m, k) during panel k
  std::vector<int64_t> U((size_t)MT * NT, -1), lastR((size_t)MT * NS, -1);
  auto u = [&](int64_t m, int64_t n) -> int64_t& { return U[(size_t)m + (size_t)n * MT]; };
  for (int64_t k = 0; k < KT; ++k) {
    const std::vector<int64_t> H = heads_of(MT, k, BS);
    std::vector<int64_t> gdone(MT, -1), tdone(MT, -1), ttdone(MT, -1);  // reflectors ready, per row
    std::fill(lastR.begin(), lastR.end(), -1);
    const int lvl = (int)(3 * k);
    for (int64_t h : H) {
      for (int s = 0; s < NS; ++s) {
        const int64_t g = add(dag::kGeqrt, h, h, k, k, s, lvl, {s > 0 ? lastR[h * NS + s - 1] : u(h, k)});
        lastR[h * NS + s] = g;
      }
      gdone[h] = lastR[h * NS + NS - 1];
      for (int64_t m = h + 1; m < domain_end(h, BS, MT); ++m) {
        int64_t prev = -1;
        for (int s = 0; s < NS; ++s) {
          const int64_t t = add(dag::kTsqrt, h, m, k, k, s, lvl + 1, {s > 0 ? prev : u(m, k), lastR[h * NS + s]});
          lastR[h * NS + s] = t;
          prev = t;
        }
        tdone[m] = prev;
      }
    }
    std::vector<std::pair<int64_t, int64_t>> merges;
    for (size_t st = 1; st < H.size(); st *= 2)
      for (size_t i = 0; i + st < H.size(); i += 2 * st) merges.push_back({H[i], H[i + st]});
    for (const auto& mg : merges) {
      const int64_t a = mg.first, b = mg.second;
      int64_t prev = -1;
      for (int s = 0; s < NS; ++s) {
        const int64_t t = add(dag::kTtqrt, a, b, k, k, s, lvl + 2,
                              {prev, lastR[a * NS + s], lastR[b * NS + s]});
        lastR[a * NS + s] = t;
        lastR[b * NS + s] = t;
        prev = t;
      }
      ttdone[b] = prev;
    }
    for (int64_t m = k; m < MT; ++m) u(m, k) = -2;  // column k is done: a later reader is a bug (checked)
    // updates of every column n > k, in the same order
    for (int64_t n = k + 1; n < NT; ++n) {
      for (int64_t h : H) {
        u(h, n) = add(dag::kLarfb, h, h, k, n, 0, lvl + 1, {gdone[h], u(h, n)});
        for (int64_t m = h + 1; m < domain_end(h, BS, MT); ++m) {
          const int64_t t = add(dag::kSsrfb, h, m, k, n, 0, lvl + 2, {tdone[m], u(h, n), u(m, n)});
          u(h, n) = u(m, n) = t;
        }
      }
      for (const auto& mg : merges) {
        const int64_t t = add(dag::kTtmqr, mg.first, mg.second, k, n, 0, lvl + 3,
                              {ttdone[mg.second], u(mg.first, n), u(mg.second, n)});
        u(mg.first, n) = u(mg.second, n) = t;
      }
    }
  }
  for (auto& t : tk)  // -2 (a finished column) never appears as a dependency
    for (int d = 0; d < t.ndep; ++d)
      if (t.dep[d] < 0) {
        set_error("tileqr_factor_tree: internal error (dependency)");
        return TILEQR_ERR_INTERNAL;
      }
  const int64_t ntask = (int64_t)tk.size();
  if (ntask > ((int64_t)1 << 30)) {
    set_error("tileqr_factor_tree: DAG too large for the dataflow kernel");
    return TILEQR_ERR_ALLOC;
  }
  // claim order: the flat tree's simulation model (api.cu build_dag)
  const int cps = dag::dag_ctas_per_sm(NB);
  const double cta_gflops = 220.0 / cps, hand = 5000.0, sPan = cps == 1 ? 1500.0 : 3000.0;
  const double dS = 4.0 * NB * NB * cols / cta_gflops;
  const double wS = 4.0 * NB * NB * NB / 150.0, wP = 2400.0 * NB / NS;
  sched::Params prm;
  prm.parts = [&](int kind) { return (kind == dag::kLarfb || kind == dag::kSsrfb || kind == dag::kTtmqr) ? nslab : 1; };
  prm.weight = [&](int kind) {
    return kind == dag::kSsrfb ? wS : kind == dag::kLarfb || kind == dag::kTtmqr ? wS / 2 : wP;
  };
  prm.dur = [&](int kind) {
    switch (kind) {
      case dag::kSsrfb: return dS + hand;
      case dag::kLarfb: case dag::kTtmqr: return 0.77 * dS + hand;
      default: return sPan * SC + hand;
    }
  };
  prm.workers = std::max(1, workers);
  if (sched::simulate(tk, prm, &out->order)) {
    set_error("tileqr_factor_tree: internal error in the DAG schedule simulation");
    return TILEQR_ERR_INTERNAL;
  }
  out->SC = SC;
  out->NS = NS;
  out->cols = cols;
  out->nslab = nslab;
  out->parts = prm.parts;
  return 0;
}

int build_tree(TreeWS* ws) {
  const int64_t MT = ws->MT, NT = ws->NT;
  const int NB = ws->NB, IB = ws->IB;
  int dev = 0;
  TQ_CUDA(cudaGetDevice(&dev));
  TQ_CUDA(cudaDeviceGetAttribute(&ws->nsm, cudaDevAttrMultiProcessorCount, dev));
  TreePlan pl;
  int rc = build_tree_plan(MT, NT, NB, IB, ws->BS, panel_sub_cols(NB, IB), ws->nsm * dag::dag_ctas_per_sm(NB), &pl);
  if (rc) return rc;
  const std::vector<sched::Task>& tk = pl.tk;
  const std::vector<TTask>& info = pl.info;
  const std::vector<sched::Slot>& order = pl.order;
  const int SC = pl.SC, cols = pl.cols;
  const int64_t ntask = (int64_t)tk.size();
  auto parts = pl.parts;
  const size_t tile = (size_t)NB * NB, ttile = (size_t)IB * NB, tsz = (size_t)MT * NT * ttile;
  auto tp = [&](int64_t m, int64_t n) { return ws->tiles + (size_t)(m + n * MT) * tile; };
  auto T1 = [&](int64_t m, int64_t k) { return ws->Tws + (size_t)(m + k * MT) * ttile; };
  auto T2 = [&](int64_t m, int64_t k) { return ws->Tws + tsz + (size_t)(m + k * MT) * ttile; };
  auto pk = [&](int64_t m, int64_t k, int sl) { return ws->Vpk + ((size_t)(m + k * MT) * 2 + sl) * ws->pk_dbl; };
  std::vector<dag::Item> items;
  items.reserve(order.size());
  for (const sched::Slot& sl : order) {
    const sched::Task& t = tk[sl.task];
    const TTask& x = info[sl.task];
    dag::Item it{};
    it.kind = t.kind;
    it.task = sl.task;
    it.ndep = t.ndep;
    for (int d = 0; d < t.ndep; ++d) {
      it.dep[d] = t.dep[d];
      it.need[d] = parts(tk[t.dep[d]].kind);
    }
    const int64_t k = x.k;
    switch (t.kind) {
      case dag::kGeqrt:
        it.col0 = (x.s * SC) | ((x.s + 1) * SC) << 16;
        it.p[0] = tp(x.a, k); it.p[2] = T1(x.a, k); it.pk = pk(x.a, k, 0);
        break;
      case dag::kTsqrt:
        it.col0 = (x.s * SC) | ((x.s + 1) * SC) << 16;
        it.p[0] = tp(x.a, k); it.p[1] = tp(x.b, k); it.p[2] = T1(x.b, k); it.pk = pk(x.b, k, 0);
        break;
      case dag::kTtqrt:
        it.col0 = (x.s * SC) | ((x.s + 1) * SC) << 16;
        it.p[0] = tp(x.a, k); it.p[1] = tp(x.b, k); it.p[2] = T2(x.b, k); it.pk = pk(x.b, k, 1);
        break;
      case dag::kLarfb:
        it.col0 = sl.slab * cols;
        it.p[2] = tp(x.a, x.n); it.pk = pk(x.a, k, 0);
        break;
      case dag::kSsrfb:
        it.col0 = sl.slab * cols;
        it.p[2] = tp(x.a, x.n); it.p[3] = tp(x.b, x.n); it.pk = pk(x.b, k, 0);
        break;
      default:  // TTMQRT
        it.col0 = sl.slab * cols;
        it.p[2] = tp(x.a, x.n); it.p[3] = tp(x.b, x.n); it.pk = pk(x.b, k, 1);
        break;
    }
    if (t.kind == dag::kLarfb || t.kind == dag::kSsrfb || t.kind == dag::kTtmqr)
      it.aux[0] = (int)std::min<int64_t>(NB, std::max<int64_t>(0, ws->N - x.n * NB));
    items.push_back(it);
  }
  ws->nitems = (int)items.size();
  ws->ntasks = (int)ntask;
  if (cudaMalloc(&ws->d_items, std::max<size_t>(1, items.size()) * sizeof(dag::Item)) != cudaSuccess ||
      cudaMalloc(&ws->d_ctr, (size_t)(257 + ntask) * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    set_error("tileqr_factor_tree: work list allocation failed");
    return TILEQR_ERR_ALLOC;
  }
  TQ_CUDA(cudaMemcpy(ws->d_items, items.data(), items.size() * sizeof(dag::Item), cudaMemcpyHostToDevice));
  return 0;
}

int get_ws(int64_t M, int64_t N, int NB, int IB, int64_t BS, TreeWS** out) {
  int dev = 0;
  TQ_CUDA(cudaGetDevice(&dev));
  auto key = std::make_tuple(dev, M, N, NB, IB, BS);
  auto it = g_tree.find(key);
  if (it != g_tree.end()) {
    *out = it->second.get();
    return 0;
  }
  auto ws = std::make_unique<TreeWS>();
  ws->M = M; ws->N = N; ws->NB = NB; ws->IB = IB; ws->BS = BS;
  ws->MT = (M + NB - 1) / NB;
  ws->NT = (N + NB - 1) / NB;
  const int64_t MT = ws->MT, NT = ws->NT, KT = std::min(MT, NT);
  ws->pk_dbl = v2_pk_doubles(NB, IB);
  const size_t tsz = (size_t)MT * NT * IB * NB;
  if (cudaMalloc(&ws->tiles, (size_t)NB * NB * MT * NT * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ws->Tws, 2 * tsz * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ws->Vpk, 2 * (size_t)MT * KT * ws->pk_dbl * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    set_error("tileqr_factor_tree: workspace allocation failed");
    return TILEQR_ERR_ALLOC;
  }
  TQ_CUDA(cudaMemset(ws->Tws, 0, 2 * tsz * sizeof(double)));
  TQ_CUDA(cudaEventCreateWithFlags(&ws->last_use, cudaEventDisableTiming));
  int rc = build_tree(ws.get());
  if (rc) return rc;
  *out = ws.get();
  size_t cap = 4;  // cached shapes, as tileqr_factor (TILEQR_WS_CACHE)
  if (const char* e = getenv("TILEQR_WS_CACHE")) cap = std::max(1, atoi(e));
  while (g_tree.size() >= cap) {  // drop the oldest entry after its last use
    auto it = g_tree.begin();
    if (it->second->used) cudaEventSynchronize(it->second->last_use);
    g_tree.erase(it);
  }
  g_tree[key] = std::move(ws);
  return 0;
}

// upper triangle (diagonal included) of `count` tiles, zero below
__global__ void triu_tiles_kernel(const double* __restrict__ src, double* __restrict__ dst, int NB) {
  const size_t t = blockIdx.x;
  const double* s = src + t * NB * NB;
  double* d = dst + t * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int j = e / NB, i = e - j * NB;
    d[e] = i <= j ? s[e] : 0.0;
  }
}

}  // namespace
}  // namespace tileqr

using namespace tileqr;

extern "C" {

int tileqr_factor_tree(int64_t M, int64_t N, double* A, int64_t lda, int NB, int IB, int64_t BS, double* T,
                       int* d_info, tileqr_stream_t stream) {
  static const char* fn = "tileqr_factor_tree";
  char msg[256];
  auto bad = [&](int i, const char* what) {
    snprintf(msg, sizeof msg, "%s: illegal argument %d (%s)", fn, i, what);
    set_error(msg);
    return -i;
  };
  if (M < 0) return bad(1, "M < 0");
  if (N < 0) return bad(2, "N < 0");
  if (!A && M > 0 && N > 0) return bad(3, "A is NULL");
  if (lda < std::max<int64_t>(1, M)) return bad(4, "lda < max(1,M)");
  if (!valid_nb_ib(NB, IB)) return bad(5, "NB / IB");
  if (!dag_path_supported(NB, IB))
    return bad(6, "(NB, IB) outside the dataflow set (NB % 32 == 0, NB <= 256, IB in {8,16,24,32})");
  if (BS < 1) return bad(7, "BS < 1");
  if (!T && M > 0 && N > 0) return bad(8, "T is NULL");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_info) {
    int rc = launch_zero_int(d_info, s);
    if (rc) return rc;
  }
  if (M == 0 || N == 0) return 0;
  std::lock_guard<std::mutex> lock(g_tree_mu);
  TreeWS* ws = nullptr;
  int rc = get_ws(M, N, NB, IB, BS, &ws);
  if (rc) return rc;
  if (ws->used) TQ_CUDA(cudaStreamWaitEvent(s, ws->last_use, 0));
  if ((rc = launch_layout_to_tiles(M, N, A, lda, NB, ws->MT, ws->NT, ws->tiles, d_info, s))) return rc;
  TQ_CUDA(cudaMemsetAsync(ws->d_ctr, 0, (size_t)(257 + ws->ntasks) * sizeof(int), s));
  int grid = 0;
  if ((rc = launch_dag(NB, IB, ws->d_items, ws->nitems, ws->d_ctr, ws->d_ctr + 257, ws->nsm, nullptr, s, &grid,
                       nullptr, dag::kModeTree)))
    return rc;
  if ((rc = launch_tiles_to_layout(M, N, A, lda, NB, ws->MT, ws->NT, ws->tiles, s))) return rc;
  TQ_CUDA(cudaMemcpyAsync(T, ws->Tws, 2 * (size_t)ws->MT * ws->NT * IB * NB * sizeof(double),
                          cudaMemcpyDeviceToDevice, s));
  TQ_CUDA(cudaEventRecord(ws->last_use, s));
  ws->used = true;
  return 0;
}

int tileqr_t_size_tree(int64_t M, int64_t N, int NB, int IB, size_t* n_doubles) {
  if (M < 0) return -1;
  if (N < 0) return -2;
  if (!valid_nb_ib(NB, IB)) return -3;
  if (!n_doubles) return -5;
  const int64_t MT = (M + NB - 1) / NB, NT = (N + NB - 1) / NB;
  *n_doubles = 2 * (size_t)(MT * NT) * IB * NB;
  return 0;
}

int tileqr_apply_qt_tree(char trans, int64_t M, int64_t NRHS, int64_t K, const double* A, int64_t lda,
                         const double* T, int NB, int IB, int64_t BS, double* B, int64_t ldb,
                         tileqr_stream_t stream) {
  static const char* fn = "tileqr_apply_qt_tree";
  char msg[256];
  auto bad = [&](int i, const char* what) {
    snprintf(msg, sizeof msg, "%s: illegal argument %d (%s)", fn, i, what);
    set_error(msg);
    return -i;
  };
  if (trans != 'T' && trans != 'N' && trans != 't' && trans != 'n') return bad(1, "trans");
  if (M < 0) return bad(2, "M < 0");
  if (NRHS < 0) return bad(3, "NRHS < 0");
  if (K < 0) return bad(4, "K < 0");
  if (!A && M > 0 && K > 0) return bad(5, "A is NULL");
  if (lda < std::max<int64_t>(1, M)) return bad(6, "lda");
  if (!T && M > 0 && K > 0) return bad(7, "T is NULL");
  if (!valid_nb_ib(NB, IB)) return bad(8, "NB / IB");
  if (BS < 1) return bad(10, "BS < 1");
  if (!B && M > 0 && NRHS > 0) return bad(11, "B is NULL");
  if (ldb < std::max<int64_t>(1, M)) return bad(12, "ldb");
  if (M == 0 || NRHS == 0 || K == 0) return 0;
  const bool tr = (trans == 'T' || trans == 't');
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t MT = (M + NB - 1) / NB, KTt = (K + NB - 1) / NB, BT = (NRHS + NB - 1) / NB;
  const int64_t KT = std::min(MT, KTt);
  const size_t tile = (size_t)NB * NB, ttile = (size_t)IB * NB, tsz = (size_t)MT * KTt * ttile;
  double *Vt = nullptr, *Ut = nullptr, *Bt = nullptr;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&Vt), tile * MT * KT * sizeof(double), s)) return rc_;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&Ut), tile * MT * KT * sizeof(double), s)) return rc_;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&Bt), tile * MT * BT * sizeof(double), s)) return rc_;
  int rc = launch_v_to_tiles(M, K, A, lda, NB, MT, KT, Vt, s);
  if (!rc) {
    triu_tiles_kernel<<<(unsigned)(MT * KT), 256, 0, s>>>(Vt, Ut, NB);  // TTQRT V2 (upper triangles)
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "triu_tiles_kernel", __FILE__, __LINE__);
  }
  if (!rc) rc = launch_layout_to_tiles(M, NRHS, B, ldb, NB, MT, BT, Bt, nullptr, s);
  auto vt = [&](int64_t m, int64_t k) { return (void*)(Vt + (size_t)(m + k * MT) * tile); };
  auto ut = [&](int64_t m, int64_t k) { return (void*)(Ut + (size_t)(m + k * MT) * tile); };
  auto bt = [&](int64_t m, int64_t n) { return (void*)(Bt + (size_t)(m + n * MT) * tile); };
  auto t1 = [&](int64_t m, int64_t k) { return (void*)(T + (size_t)(m + k * MT) * ttile); };
  auto t2 = [&](int64_t m, int64_t k) { return (void*)(T + tsz + (size_t)(m + k * MT) * ttile); };
  // the operation sequence (one batched launch over B's column tiles each)
  struct Op { bool larfb; void* v; void* t; int64_t r1, r2; };
  std::vector<Op> ops;
  for (int64_t kk = 0; kk < KT; ++kk) {
    const int64_t k = tr ? kk : KT - 1 - kk;
    const std::vector<int64_t> H = heads_of(MT, k, BS);
    std::vector<Op> seq;
    for (int64_t h : H) {
      seq.push_back({true, vt(h, k), t1(h, k), h, -1});
      for (int64_t m = h + 1; m < domain_end(h, BS, MT); ++m) seq.push_back({false, vt(m, k), t1(m, k), h, m});
    }
    for (size_t st = 1; st < H.size(); st *= 2)
      for (size_t i = 0; i + st < H.size(); i += 2 * st)
        seq.push_back({false, ut(H[i + st], k), t2(H[i + st], k), H[i], H[i + st]});
    if (!tr) std::reverse(seq.begin(), seq.end());  // Q B: every operation backwards, trans 'N'
    ops.insert(ops.end(), seq.begin(), seq.end());
  }
  void** dp = nullptr;
  const size_t per = 4 * (size_t)BT;
  if (!rc) {
    rc = stream_alloc(reinterpret_cast<void**>(&dp), std::max<size_t>(1, ops.size() * per) * sizeof(void*), s);
  }
  std::vector<void*> hp(ops.size() * per);
  for (size_t o = 0; o < ops.size(); ++o)
    for (int64_t n = 0; n < BT; ++n) {
      hp[o * per + n] = ops[o].v;
      hp[o * per + BT + n] = ops[o].t;
      hp[o * per + 2 * BT + n] = bt(ops[o].r1, n);
      hp[o * per + 3 * BT + n] = ops[o].r2 >= 0 ? bt(ops[o].r2, n) : nullptr;
    }
  if (!rc && !hp.empty()) {
    cudaError_t e = cudaMemcpyAsync(dp, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync", __FILE__, __LINE__);
    if (!rc) e = cudaStreamSynchronize(s);  // hp is a host temporary
    if (e != cudaSuccess && !rc) rc = cuda_fail(e, "cudaStreamSynchronize", __FILE__, __LINE__);
  }
  double** d = reinterpret_cast<double**>(dp);
  for (size_t o = 0; o < ops.size() && !rc; ++o) {
    double** q = d + o * per;
    if (ops[o].larfb)
      rc = launch_larfb(tr, NB, IB, (int)BT, (const double* const*)q, (const double* const*)(q + BT), q + 2 * BT,
                        NB, s);
    else
      rc = launch_ssrfb(tr, NB, IB, (int)BT, (const double* const*)q, (const double* const*)(q + BT), q + 2 * BT,
                        q + 3 * BT, NB, s);
  }
  if (!rc) rc = launch_tiles_to_layout(M, NRHS, B, ldb, NB, MT, BT, Bt, s);
  cudaFreeAsync(Vt, s);
  cudaFreeAsync(Ut, s);
  cudaFreeAsync(Bt, s);
  if (dp) cudaFreeAsync(dp, s);
  return rc;
}

// Batched TTQRT (the tree's merge kernel, f3): [R[i]; A2[i]] with both upper
// triangular; R's strict lower part and A2's strict lower part untouched.
int tileqr_ttqrt_batched(int NB, int IB, int batch, double* const* R, double* const* A2, double* const* T,
                         tileqr_stream_t stream) {
  if (!valid_nb_ib(NB, IB) || !dag_path_supported(NB, IB)) {
    set_error("tileqr_ttqrt_batched: (NB, IB) outside the register-resident panel set");
    return -1;
  }
  if (batch < 0) return -3;
  if (batch == 0) return 0;
  if (!R) return -4;
  if (!A2) return -5;
  if (!T) return -6;
  return launch_ttqrt_fast(NB, IB, batch, R, A2, T, reinterpret_cast<cudaStream_t>(stream), nullptr);
}

// The domain size as a tunable ("p domains"): time
// tileqr_factor_tree for BS = 1, 2, 4, ... (and the flat tree, BS >= MT) on a
// seeded M x N matrix, 1 warm-up + 6 timed runs each, and
// return the fastest BS (median).  Synchronizes the current device.
int tileqr_tune_tree(int64_t M, int64_t N, int NB, int IB, int64_t* h_BS, double* h_ms,
                     const char* report_json_path) {
  if (M < 1) return -1;
  if (N < 1) return -2;
  if (!valid_nb_ib(NB, IB) || !dag_path_supported(NB, IB)) return -3;
  if (!h_BS) return -5;
  const int64_t MT = (M + NB - 1) / NB;
  double *A0 = nullptr, *A = nullptr, *T = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  size_t tn = 0;
  tileqr_t_size_tree(M, N, NB, IB, &tn);
  auto cleanup = [&]() {
    if (s) cudaStreamSynchronize(s);
    cudaFree(A0); cudaFree(A); cudaFree(T);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
  };
  if (cudaMalloc(&A0, (size_t)M * N * 8) != cudaSuccess || cudaMalloc(&A, (size_t)M * N * 8) != cudaSuccess ||
      cudaMalloc(&T, tn * 8) != cudaSuccess || cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    set_error("tileqr_tune_tree: allocation failed");
    return TILEQR_ERR_ALLOC;
  }
  int rc = launch_rng_uniform(M, N, A0, M, 3, 0, s);
  std::vector<int64_t> cand;
  for (int64_t bs = 1; bs < MT; bs *= 2) cand.push_back(bs);
  cand.push_back(MT);  // one domain: the flat tree
  std::string rep = "[";
  double best_ms = 1e300;
  int64_t best = MT;
  for (int64_t bs : cand) {
    std::vector<float> t;
    for (int r = 0; r < 7 && !rc; ++r) {
      cudaMemcpyAsync(A, A0, (size_t)M * N * 8, cudaMemcpyDeviceToDevice, s);
      cudaEventRecord(e0, s);
      rc = tileqr_factor_tree(M, N, A, M, NB, IB, bs, T, nullptr, (tileqr_stream_t)s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) t.push_back(ms);
    }
    if (rc) break;
    std::sort(t.begin(), t.end());
    const double med = 0.5 * (t[2] + t[3]);
    char b[128];
    snprintf(b, sizeof b, "%s{\"bs\": %lld, \"median_ms\": %.6f}", rep.size() > 1 ? ", " : "", (long long)bs, med);
    rep += b;
    if (med < best_ms) {
      best_ms = med;
      best = bs;
    }
    std::lock_guard<std::mutex> lock(g_tree_mu);  // this shape's workspace is not needed again
    int dev = 0;
    cudaGetDevice(&dev);
    g_tree.erase(std::make_tuple(dev, M, N, NB, IB, bs));
  }
  rep += "]";
  cleanup();
  if (rc) return rc;
  *h_BS = best;
  if (h_ms) *h_ms = best_ms;
  if (report_json_path) {
    FILE* f = fopen(report_json_path, "w");
    if (f) {
      fprintf(f, "{\"M\": %lld, \"N\": %lld, \"NB\": %d, \"IB\": %d, \"runs\": %s, \"best_bs\": %lld}\n",
              (long long)M, (long long)N, NB, IB, rep.c_str(), (long long)best);
      fclose(f);
    }
  }
  return 0;
}

// Host-only work list of the tree variant (claim order), for CPU tests of the
// task graph: per item 11 int64 (kind, a, b, k, n, s, task, ndep, dep0, dep1,
// dep2): kind 0 GEQRT(a; k), 1 TSQRT(a <- b; k), 8 TTQRT(a <- b; k), 2 LARFB(a;
// k, n), 3 SSRFB(a, b; k, n), 9 TTMQRT(a, b; k, n); s = panel sub-task
// (columns [s*sub_cols, (s+1)*sub_cols)) or update slab; task / deps = task
// ids.  Errors: -1 M, -2 N, -3 NB/IB, -5 BS, -6 workers, -7 sub_cols, -9
// capacity, -10 h_count NULL.
int tileqr_tree_plan_items(int64_t M, int64_t N, int NB, int IB, int64_t BS, int workers, int sub_cols,
                           int64_t* h_out, int64_t cap, int64_t* h_count) {
  if (M < 1) return -1;
  if (N < 1) return -2;
  if (!valid_nb_ib(NB, IB)) return -3;
  if (BS < 1) return -5;
  if (workers < 1) return -6;
  if (sub_cols < IB || NB % sub_cols || sub_cols % IB) return -7;
  if (!h_count) return -10;
  TreePlan pl;
  int rc = build_tree_plan((M + NB - 1) / NB, (N + NB - 1) / NB, NB, IB, BS, sub_cols, workers, &pl);
  if (rc) return rc;
  const int64_t n = (int64_t)pl.order.size();
  *h_count = n;
  if (!h_out) return 0;
  if (cap < 11 * n) return -9;
  for (int64_t i = 0; i < n; ++i) {
    const sched::Slot& sl = pl.order[i];
    const sched::Task& t = pl.tk[sl.task];
    const TTask& x = pl.info[sl.task];
    int64_t* o = h_out + 11 * i;
    o[0] = t.kind; o[1] = x.a; o[2] = x.b; o[3] = x.k; o[4] = x.n;
    o[5] = (t.kind == dag::kLarfb || t.kind == dag::kSsrfb || t.kind == dag::kTtmqr) ? sl.slab : x.s;
    o[6] = sl.task; o[7] = t.ndep;
    for (int d = 0; d < 3; ++d) o[8 + d] = d < t.ndep ? t.dep[d] : -1;
  }
  return 0;
}

void tileqr_tree_finalize(void) {
  std::lock_guard<std::mutex> lock(g_tree_mu);
  g_tree.clear();
}

}  // extern "C"
