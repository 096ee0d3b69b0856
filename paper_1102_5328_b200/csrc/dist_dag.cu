// dist_dag.cu -- multi-rank dataflow tile QR: the whole DAG of every rank in
// the persistent dataflow kernel (dag.cuh), the panel broadcast fused into it
// as COPY items that push each packed reflector tile over peer memory
// (J:north_star "panel V/T tiles broadcast over
// NVLink"; PAPER.md:852-864 future work on distributed memory).
//
// Partition: tile column n lives on rank owner(n) = n mod P.
//   GEQRT(k, s), TSQRT(k, m, s)      on owner(k)   (column k is local there)
//   LARFB(k, n), SSRFB(k, m, n)      on owner(n)
//   COPY(k, m, d)                    on owner(k): after the last panel
//       sub-task that writes reflector tile (k, m), push its packed image
//       (V_p and T_p of every inner panel, update_v2.cuh) into the same slot
//       of rank d, then +1 on d's ARRIVE(k, m) counter (system-scope release)
//   ARRIVE(k, m, d)                  the counter on rank d (no CTA runs it)
// for every rank d != owner(k) that owns a column n > k.  An update on rank
// d waits on ARRIVE(k, m, d) (system-scope acquire) where the single-GPU
// DAG waits on the panel task; everything else is the single-GPU DAG (api.cu
// build_dag), so every tile sees the same kernels with the same operands in
// the same order: R, V and T are bitwise those of tileqr_factor.
//
// Claim order: ONE list schedule simulated over all ranks (sched.h, one pool
// of resident CTAs per rank, cross-rank edges through COPY + ARRIVE), each
// rank claiming its own items in that global start-time order -- deadlock
// free across ranks (sched.h).  No per-level synchronisation, no NCCL on the
// data path: lookahead is whatever the dependencies allow.
//
// Emulation (tileqr_dist_emulate): all ranks' items in one launch on one GPU,
// each rank with its own tile, T, slot and counter buffers, COPY items
// writing into another rank's buffers of the same device -- the same kernel
// code and item lists as the multi-GPU run (which differs only in the peer
// pointers, cudaIpc-mapped, see dist.cu).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dag_item.h"
#include "dist_dag.h"
#include "internal.h"
#include "sched.h"

namespace tileqr {

int launch_nonfinite_check(const double* A, int64_t n, int* d_info, cudaStream_t s);
int launch_dist_fill(int64_t M, int64_t N, int NB, int64_t MT, int nranks, int rank, int64_t nloc, double* A,
                     uint64_t seed, cudaStream_t s);

namespace dd {

int64_t Plan::slot(int64_t k, int64_t m) const { return k * MT - k * (k - 1) / 2 + (m - k); }
int64_t Plan::nslots() const { return slot(KT, KT); }

int64_t local_cols(int64_t NT, int P, int rank) {
  return NT > rank ? (NT - rank + P - 1) / P : 0;
}

int build_plan(int64_t M, int64_t N, int NB, int IB, int P, int workers, int SC, std::shared_ptr<Plan>* out) {
  auto pl = std::make_shared<Plan>();
  Plan& p = *pl;
  p.M = M;
  p.N = N;
  p.NB = NB;
  p.IB = IB;
  p.P = P;
  p.MT = (M + NB - 1) / NB;
  p.NT = (N + NB - 1) / NB;
  p.KT = std::min(p.MT, p.NT);
  p.SC = SC;
  p.NS = NB / SC;
  p.cols = dag::dag_cols(NB);
  p.nslab = (NB + p.cols - 1) / p.cols;
  const int64_t MT = p.MT, NT = p.NT, KT = p.KT;
  const int NS = p.NS;
  p.offL.assign(KT + 1, 0);
  p.offT.assign(KT + 1, 0);
  p.offS.assign(KT + 1, 0);
  p.nG = KT * NS;
  p.nL = p.nT = p.nS = 0;
  for (int64_t k = 0; k < KT; ++k) {
    p.offL[k] = p.nL; p.nL += NT - k - 1;
    p.offT[k] = p.nT; p.nT += (MT - k - 1) * NS;
    p.offS[k] = p.nS; p.nS += (MT - k - 1) * (NT - k - 1);
  }
  // destinations of panel k: ranks other than owner(k) owning a column n > k
  p.dests.assign(KT, {});
  p.cpo.assign(KT + 1, 0);
  int64_t ncp = 0;
  for (int64_t k = 0; k < KT; ++k) {
    for (int d = 0; d < P; ++d) {
      if (d == p.owner(k)) continue;
      bool has = false;
      for (int64_t n = k + 1; n < NT && !has; ++n) has = p.owner(n) == d;
      if (has) p.dests[k].push_back(d);
    }
    p.cpo[k] = ncp;
    ncp += (MT - k) * (int64_t)p.dests[k].size();
  }
  p.cpo[KT] = ncp;
  p.base_cp = p.nG + p.nL + p.nT + p.nS;
  p.base_ar = p.base_cp + ncp;
  p.ntask = p.base_ar + ncp;
  if (p.ntask > ((int64_t)1 << 30) / std::max(1, P)) {
    set_error("tileqr_dist: DAG too large for the dataflow kernel");
    return TILEQR_ERR_ALLOC;
  }
  using Task = sched::Task;
  std::vector<Task> tk(p.ntask);
  auto panel_done = [&](int64_t k, int64_t m) {  // the last sub-task writing reflector tile (k, m)
    return m == k ? p.idG(k, NS - 1) : p.idT(k, m, NS - 1);
  };
  // the reflector tile (k, m) as seen by an update on rank r: the panel task
  // itself on its owner, the arrival of its copy elsewhere
  auto refl = [&](int64_t k, int64_t m, int r) {
    if (r == p.owner(k)) return panel_done(k, m);
    const auto& ds = p.dests[k];
    const int di = (int)(std::find(ds.begin(), ds.end(), r) - ds.begin());
    return p.idAR(k, m, di);
  };
  for (int64_t k = 0; k < KT; ++k) {
    const int ok = p.owner(k);
    for (int s = 0; s < NS; ++s) {
      Task g{dag::kGeqrt, (int)k, (int)k, (int)k, (int)(3 * k), 0, {0, 0, 0}, s};
      if (s > 0) g.dep[g.ndep++] = (int)p.idG(k, s - 1);
      else if (k > 0) g.dep[g.ndep++] = (int)p.idS(k - 1, k, k);
      g.pool = ok;
      tk[p.idG(k, s)] = g;
    }
    for (int64_t n = k + 1; n < NT; ++n) {
      Task l{dag::kLarfb, (int)k, (int)k, (int)n, (int)(3 * k + 1), 0, {0, 0, 0}, 0};
      l.dep[l.ndep++] = (int)refl(k, k, p.owner(n));
      if (k > 0) l.dep[l.ndep++] = (int)p.idS(k - 1, k, n);
      l.pool = p.owner(n);
      tk[p.idL(k, n)] = l;
    }
    for (int64_t m = k + 1; m < MT; ++m) {
      for (int s = 0; s < NS; ++s) {
        Task t{dag::kTsqrt, (int)k, (int)m, (int)k, (int)(2 * k + m), 0, {0, 0, 0}, s};
        if (s > 0) t.dep[t.ndep++] = (int)p.idT(k, m, s - 1);
        else if (k > 0) t.dep[t.ndep++] = (int)p.idS(k - 1, m, k);
        t.dep[t.ndep++] = (int)(m == k + 1 ? p.idG(k, s) : p.idT(k, m - 1, s));
        t.pool = ok;
        tk[p.idT(k, m, s)] = t;
      }
      for (int64_t n = k + 1; n < NT; ++n) {
        Task u{dag::kSsrfb, (int)k, (int)m, (int)n, (int)(2 * k + m + 1), 0, {0, 0, 0}, 0};
        u.dep[u.ndep++] = (int)refl(k, m, p.owner(n));
        u.dep[u.ndep++] = (int)(m == k + 1 ? p.idL(k, n) : p.idS(k, m - 1, n));
        if (k > 0) u.dep[u.ndep++] = (int)p.idS(k - 1, m, n);
        u.pool = p.owner(n);
        tk[p.idS(k, m, n)] = u;
      }
    }
    for (int64_t m = k; m < MT; ++m)
      for (int di = 0; di < (int)p.dests[k].size(); ++di) {
        const int lvl = (int)(m == k ? 3 * k : 2 * k + m);
        Task c{dag::kCopy, (int)k, (int)m, (int)k, lvl, 1, {(int)panel_done(k, m), 0, 0}, p.dests[k][di]};
        c.pool = ok;
        tk[p.idCP(k, m, di)] = c;
        Task a{dag::kArrive, (int)k, (int)m, (int)k, lvl, 1, {(int)p.idCP(k, m, di), 0, 0}, p.dests[k][di]};
        a.pool = p.dests[k][di];
        a.worker = false;
        tk[p.idAR(k, m, di)] = a;
      }
  }
  // simulated durations (api.cu build_dag's constants) plus the push: ~50
  // GB/s per CTA over NVLink and ~3 us from the release to the peer's acquire
  const int cps = dag::dag_ctas_per_sm(NB);
  const double cta_gflops = 220.0 / cps;
  const double dS = 4.0 * NB * NB * p.cols / cta_gflops, hand = 5000.0;
  const double sPan = cps == 1 ? 1500.0 : 3000.0;
  const double pkb = (double)v2_pk_doubles(NB, IB) * 8.0;
  const double wS = 4.0 * NB * NB * NB / 150.0, wP = 2400.0 * NB / NS;
  sched::Params prm;
  prm.parts = [&](int kind) { return (kind == dag::kLarfb || kind == dag::kSsrfb) ? p.nslab : 1; };
  prm.weight = [&](int kind) {
    return kind == dag::kSsrfb ? wS : kind == dag::kLarfb ? wS / 2 : kind == dag::kArrive ? 3000.0
         : kind == dag::kCopy ? pkb / 50.0 : wP;
  };
  prm.dur = [&](int kind) {
    switch (kind) {
      case dag::kSsrfb: return dS + hand;
      case dag::kLarfb: return 0.77 * dS + hand;
      case dag::kCopy: return pkb / 50.0 + 1000.0;
      case dag::kArrive: return 3000.0;
      default: return sPan * SC + hand;
    }
  };
  prm.npools = P;
  prm.workers = std::max(1, workers);
  const int rc = sched::simulate(tk, prm, &p.order);
  if (rc) {
    set_error("tileqr_dist: internal error in the multi-rank DAG schedule");
    return TILEQR_ERR_INTERNAL;
  }
  p.tasks = std::move(tk);
  *out = pl;
  return 0;
}

int emit_items(const Plan& p, int rank, const std::vector<RankBufs>& bufs, bool emul,
               std::vector<dag::Item>* items) {
  const int NB = p.NB, IB = p.IB, P = p.P;
  const size_t tile = (size_t)NB * NB, ttile = (size_t)IB * NB;
  const size_t pkd = v2_pk_doubles(NB, IB);
  const int64_t MT = p.MT;
  auto A = [&](int64_t m, int64_t n) { return bufs[p.owner(n)].A + (size_t)(m + (n / P) * MT) * tile; };
  auto Tt = [&](int64_t m, int64_t k) { return bufs[p.owner(k)].T + (size_t)(m + (k / P) * MT) * ttile; };
  auto slot = [&](int r, int64_t k, int64_t m) { return bufs[r].slots + (size_t)p.slot(k, m) * pkd; };
  auto cidx = [&](int r, int64_t id) { return (int)((emul ? (int64_t)r * p.ntask : 0) + id); };
  items->clear();
  for (const sched::Slot& sl : p.order) {
    const sched::Task& t = p.tasks[sl.task];
    if (rank >= 0 && t.pool != rank) continue;
    const int r = t.pool;
    dag::Item it{};
    it.kind = t.kind;
    it.task = cidx(r, sl.task);
    if (t.kind == dag::kGeqrt || t.kind == dag::kTsqrt) it.col0 = (t.s * p.SC) | ((t.s + 1) * p.SC) << 16;
    else it.col0 = sl.slab * p.cols;
    it.ndep = t.ndep;
    for (int d = 0; d < t.ndep; ++d) {
      const sched::Task& dt = p.tasks[t.dep[d]];
      it.dep[d] = cidx(r, t.dep[d]);
      const int need = dt.worker ? ((dt.kind == dag::kLarfb || dt.kind == dag::kSsrfb) ? p.nslab : 1) : 1;
      it.need[d] = dt.kind == dag::kArrive ? -need : need;  // peer-written: system scope
    }
    switch (t.kind) {
      case dag::kGeqrt:
        it.p[0] = A(t.k, t.k); it.p[2] = Tt(t.k, t.k); it.pk = slot(r, t.k, t.k);
        break;
      case dag::kTsqrt:
        it.p[0] = A(t.k, t.k); it.p[1] = A(t.m, t.k); it.p[2] = Tt(t.m, t.k); it.pk = slot(r, t.k, t.m);
        break;
      case dag::kLarfb:
        it.p[2] = A(t.k, t.n); it.pk = slot(r, t.k, t.k);
        it.aux[0] = (int)std::min<int64_t>(NB, std::max<int64_t>(0, p.N - (int64_t)t.n * NB));
        break;
      case dag::kSsrfb:
        it.p[2] = A(t.k, t.n); it.p[3] = A(t.m, t.n); it.pk = slot(r, t.k, t.m);
        it.aux[0] = (int)std::min<int64_t>(NB, std::max<int64_t>(0, p.N - (int64_t)t.n * NB));
        it.aux[1] = dag::ssrfb_rows(p.M, t.m, NB);
        break;
      case dag::kCopy: {
        const int d = t.s;
        const auto& ds = p.dests[t.k];
        const int di = (int)(std::find(ds.begin(), ds.end(), d) - ds.begin());
        it.p[0] = slot(r, t.k, t.m);
        it.p[1] = slot(d, t.k, t.m);
        it.p[2] = reinterpret_cast<double*>(bufs[d].done + p.idAR(t.k, t.m, di));
        it.aux[0] = (int)pkd;
        break;
      }
      default:
        set_error("tileqr_dist: internal error (item kind)");
        return TILEQR_ERR_INTERNAL;
    }
    items->push_back(it);
  }
  return 0;
}

}  // namespace dd

namespace {

// Emulated ranks: cached plan, slot and counter buffers, item list.
struct EmuState {
  int64_t M = -1, N = -1;
  int NB = 0, IB = 0, P = 0, SC = 0;
  std::vector<double*> A, T;
  std::shared_ptr<dd::Plan> plan;
  double* slots = nullptr;
  int* ctr = nullptr;
  dag::Item* d_items = nullptr;
  int nitems = 0;
  int nsm = 0;
  ~EmuState() {
    cudaFree(slots);
    cudaFree(ctr);
    cudaFree(d_items);
  }
};
std::mutex g_emu_mu;
std::unique_ptr<EmuState> g_emu;

}  // namespace
}  // namespace tileqr

using namespace tileqr;

extern "C" {

int tileqr_dist_emulate(int nranks, int64_t M, int64_t N, double* const* h_A_local, int NB, int IB,
                        double* const* h_T_local, int* d_info, tileqr_stream_t stream) {
  static const char* fn = "tileqr_dist_emulate";
  char msg[256];
  auto bad = [&](int i, const char* what) {
    snprintf(msg, sizeof msg, "%s: illegal argument %d (%s)", fn, i, what);
    set_error(msg);
    return -i;
  };
  if (nranks < 1) return bad(1, "nranks < 1");
  if (M < 0) return bad(2, "M < 0");
  if (N < 0) return bad(3, "N < 0");
  if (!h_A_local) return bad(4, "NULL pointer array");
  if (NB == 0 && IB == 0) {
    bool f = false;
    lookup_pair(M, N, nranks, &NB, &IB, &f);
  }
  if (!valid_nb_ib(NB, IB)) return bad(5, "NB");
  if (!dag_path_supported(NB, IB))
    return bad(6, "(NB, IB) outside the dataflow set (NB % 32 == 0, NB <= 256, IB in {8,16,24,32})");
  if (!h_T_local) return bad(7, "NULL pointer array");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_info) {
    int rc = launch_zero_int(d_info, s);
    if (rc) return rc;
  }
  if (M == 0 || N == 0) return 0;
  const int64_t MT = (M + NB - 1) / NB, NT = (N + NB - 1) / NB;
  for (int r = 0; r < nranks; ++r)
    if (dd::local_cols(NT, nranks, r) > 0 && (!h_A_local[r] || !h_T_local[r])) return bad(4, "NULL local buffer");
  std::lock_guard<std::mutex> lock(g_emu_mu);
  const int SC = panel_sub_cols(NB, IB);
  EmuState* e = g_emu.get();
  bool same = e && e->M == M && e->N == N && e->NB == NB && e->IB == IB && e->P == nranks && e->SC == SC;
  for (int r = 0; same && r < nranks; ++r) same = e->A[r] == h_A_local[r] && e->T[r] == h_T_local[r];
  if (!same) {
    g_emu.reset();
    auto ne = std::make_unique<EmuState>();
    ne->M = M; ne->N = N; ne->NB = NB; ne->IB = IB; ne->P = nranks; ne->SC = SC;
    ne->A.assign(h_A_local, h_A_local + nranks);
    ne->T.assign(h_T_local, h_T_local + nranks);
    int dev = 0;
    TQ_CUDA(cudaGetDevice(&dev));
    TQ_CUDA(cudaDeviceGetAttribute(&ne->nsm, cudaDevAttrMultiProcessorCount, dev));
    const int workers = std::max(1, ne->nsm * dag::dag_ctas_per_sm(NB) / nranks);
    int rc = dd::build_plan(M, N, NB, IB, nranks, workers, SC, &ne->plan);
    if (rc) return rc;
    const dd::Plan& p = *ne->plan;
    const size_t pkd = v2_pk_doubles(NB, IB);
    const size_t nsl = (size_t)p.nslots();
    if (cudaMalloc(&ne->slots, std::max<size_t>(1, nsl * pkd * nranks) * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&ne->ctr, (size_t)(257 + p.ntask * nranks) * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      set_error("tileqr_dist_emulate: workspace allocation failed");
      return TILEQR_ERR_ALLOC;
    }
    std::vector<dd::RankBufs> bufs(nranks);
    for (int r = 0; r < nranks; ++r)
      bufs[r] = {h_A_local[r], h_T_local[r], ne->slots + (size_t)r * nsl * pkd, ne->ctr + 257 + (size_t)r * p.ntask};
    std::vector<dag::Item> items;
    rc = dd::emit_items(p, -1, bufs, true, &items);
    if (rc) return rc;
    ne->nitems = (int)items.size();
    if (cudaMalloc(&ne->d_items, std::max<size_t>(1, items.size()) * sizeof(dag::Item)) != cudaSuccess) {
      cudaGetLastError();
      set_error("tileqr_dist_emulate: work list allocation failed");
      return TILEQR_ERR_ALLOC;
    }
    TQ_CUDA(cudaMemcpy(ne->d_items, items.data(), items.size() * sizeof(dag::Item), cudaMemcpyHostToDevice));
    g_emu = std::move(ne);
    e = g_emu.get();
  }
  const dd::Plan& p = *e->plan;
  if (d_info)
    for (int r = 0; r < nranks; ++r) {
      const int64_t nl = dd::local_cols(NT, nranks, r);
      if (nl > 0) {
        int rc = launch_nonfinite_check(h_A_local[r], nl * MT * NB * (int64_t)NB, d_info, s);
        if (rc) return rc;
      }
    }
  TQ_CUDA(cudaMemsetAsync(e->ctr, 0, (size_t)(257 + p.ntask * nranks) * sizeof(int), s));
  int grid = 0;
  return launch_dag(NB, IB, e->d_items, e->nitems, e->ctr, e->ctr + 257, e->nsm, nullptr, s, &grid, nullptr,
                    dag::kModeDist);
}

// Host-only export of one rank's work list (multi-rank dataflow plan), for
// CPU tests of the plan: per item, in the rank's claim order, 10 int64
// (kind, k, m, n, s, task, ndep, dep0, dep1, dep2); s = sub-task (panels),
// destination rank (COPY), slab (updates); ids are global task ids
// (ARRIVE(k, m, d) ids are the arrival of the copy of reflector tile (k, m)
// on the item's rank).
int tileqr_dist_plan_items(int64_t M, int64_t N, int NB, int IB, int nranks, int rank, int workers,
                           int sub_cols, int64_t* h_out, int64_t cap, int64_t* h_count) {
  if (M < 1) return -1;
  if (N < 1) return -2;
  if (!valid_nb_ib(NB, IB)) return -3;
  if (nranks < 1) return -5;
  if (rank < 0 || rank >= nranks) return -6;
  if (workers < 1) return -7;
  if (sub_cols < IB || NB % sub_cols || sub_cols % IB) return -8;
  if (!h_count) return -11;
  std::shared_ptr<dd::Plan> pl;
  int rc = dd::build_plan(M, N, NB, IB, nranks, workers, sub_cols, &pl);
  if (rc) return rc;
  const dd::Plan& p = *pl;
  int64_t cnt = 0;
  for (const sched::Slot& sl : p.order) {
    const sched::Task& t = p.tasks[sl.task];
    if (t.pool != rank) continue;
    if (h_out && (cnt + 1) * 10 <= cap) {
      int64_t* o = h_out + cnt * 10;
      o[0] = t.kind; o[1] = t.k; o[2] = t.m; o[3] = t.n;
      o[4] = (t.kind == dag::kLarfb || t.kind == dag::kSsrfb) ? sl.slab : t.s;
      o[5] = sl.task; o[6] = t.ndep;
      for (int d = 0; d < 3; ++d) o[7 + d] = d < t.ndep ? t.dep[d] : -1;
    }
    ++cnt;
  }
  *h_count = cnt;
  if (h_out && cnt * 10 > cap) return -10;
  return 0;
}

}  // extern "C"
