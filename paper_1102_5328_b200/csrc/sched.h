// sched.h -- host-side claim order of the dataflow DAG kernel (dag.cuh):
// topological order, bottom levels and a list-schedule simulation over the
// resident CTAs, shared by the single-GPU factorization (api.cu build_dag)
// and the multi-rank dataflow factorization (dist_dag.cu).
//
// PLASMA schedules its tile DAG statically over CPU cores;
// here the persistent kernel's CTAs claim work items in the order this
// simulation produces: P workers per pool (a pool = the resident CTAs of one
// GPU / rank), rough per-item durations, ready items started in
// bottom-level order, items sorted by simulated start time.  Start times
// respect every dependency, so the order is topological -- and, with several
// pools simulated together, one global order whose restriction to each rank
// is what that rank claims: the unfinished item with the smallest start time
// always has its inputs final, so claiming can never deadlock, across ranks
// included.
#pragma once

#include <algorithm>
#include <functional>
#include <vector>

namespace tileqr {
namespace sched {

struct Task {
  int kind;
  int k, m, n;
  int level;      // ASAP level (diagnostics, tie-break)
  int ndep;
  int dep[3];
  int s;          // sub-task (panels) or destination rank (copies)
  int pool = 0;   // rank whose CTAs run it
  bool worker = true;   // false: completes without a CTA (copy-engine arrival, remote signal)
  double fixed = -1.0;  // worker == false: completion time >= this (absolute)
};

struct Slot {
  double start;
  double bl;
  int task, slab;
};

struct Params {
  std::function<int(int)> parts;      // work items per task of a kind
  std::function<double(int)> weight;  // bottom-level weight per kind
  std::function<double(int)> dur;     // simulated duration of one item of a kind (worker tasks),
                                      // or the delay after the inputs are ready (non-worker tasks)
  std::vector<double> bl_override;    // per task (optional): priority set by the caller (>= 0 wins)
  int npools = 1;
  int workers = 1;                    // workers per pool
};

// Returns 0 and the items sorted by simulated start in *out (worker tasks
// only, parts(kind) items each); -1 if the graph has a cycle, -2 if the
// simulation did not schedule every item.
inline int simulate(const std::vector<Task>& tk, const Params& prm, std::vector<Slot>* out,
                    bool bl_order = false) {
  const int64_t ntask = (int64_t)tk.size();
  std::vector<int64_t> soff(ntask + 1, 0);
  for (int64_t i = 0; i < ntask; ++i)
    for (int d = 0; d < tk[i].ndep; ++d) ++soff[tk[i].dep[d] + 1];
  for (int64_t i = 0; i < ntask; ++i) soff[i + 1] += soff[i];
  std::vector<int> succ(soff[ntask]);
  {
    std::vector<int64_t> fill(soff.begin(), soff.end() - 1);
    for (int64_t i = 0; i < ntask; ++i)
      for (int d = 0; d < tk[i].ndep; ++d) succ[fill[tk[i].dep[d]]++] = (int)i;
  }
  std::vector<int> topo;
  topo.reserve(ntask);
  {
    std::vector<int> indeg(ntask);
    for (int64_t i = 0; i < ntask; ++i) {
      indeg[i] = tk[i].ndep;
      if (indeg[i] == 0) topo.push_back((int)i);
    }
    for (size_t q = 0; q < topo.size(); ++q)
      for (int64_t e = soff[topo[q]]; e < soff[topo[q] + 1]; ++e)
        if (--indeg[succ[e]] == 0) topo.push_back(succ[e]);
    if ((int64_t)topo.size() != ntask) return -1;
  }
  std::vector<double> bl(ntask, 0.0);
  for (int64_t q = ntask - 1; q >= 0; --q) {
    const int i = topo[q];
    double mx = 0.0;
    for (int64_t e = soff[i]; e < soff[i + 1]; ++e) mx = std::max(mx, bl[succ[e]]);
    bl[i] = prm.weight(tk[i].kind) + mx;
  }
  if (!prm.bl_override.empty())
    for (int64_t i = 0; i < ntask; ++i)
      if (prm.bl_override[i] >= 0.0) bl[i] = prm.bl_override[i];

  const int npools = std::max(1, prm.npools);
  std::vector<int> indeg(ntask), left(ntask);
  for (int64_t i = 0; i < ntask; ++i) {
    indeg[i] = tk[i].ndep;
    left[i] = tk[i].worker ? prm.parts(tk[i].kind) : 1;
  }
  struct Rd { double bl; int level, s, task, slab; };
  auto rd_less = [](const Rd& a, const Rd& b) {  // max-heap on priority
    if (a.bl != b.bl) return a.bl < b.bl;
    if (a.level != b.level) return a.level > b.level;
    if (a.s != b.s) return a.s > b.s;
    if (a.task != b.task) return a.task > b.task;
    return a.slab > b.slab;
  };
  std::vector<std::vector<Rd>> ready(npools);
  struct Ev { double t; int task; bool worker; };
  auto ev_greater = [](const Ev& a, const Ev& b) { return a.t > b.t; };
  std::vector<Ev> events;
  double now = 0.0;
  auto push_task = [&](int i) {
    if (!tk[i].worker) {  // completes without a CTA
      events.push_back({std::max(now + prm.dur(tk[i].kind), tk[i].fixed), i, false});
      std::push_heap(events.begin(), events.end(), ev_greater);
      return;
    }
    auto& rq = ready[tk[i].pool];
    for (int sl = 0; sl < prm.parts(tk[i].kind); ++sl) {
      rq.push_back({bl[i], tk[i].level, tk[i].s, i, sl});
      std::push_heap(rq.begin(), rq.end(), rd_less);
    }
  };
  for (int64_t i = 0; i < ntask; ++i)
    if (indeg[i] == 0) push_task((int)i);
  std::vector<Slot> sched;
  std::vector<int> freew(npools, std::max(1, prm.workers));
  auto any_ready = [&]() {
    for (auto& r : ready)
      if (!r.empty()) return true;
    return false;
  };
  while (any_ready() || !events.empty()) {
    for (int p = 0; p < npools; ++p) {
      auto& rq = ready[p];
      while (freew[p] > 0 && !rq.empty()) {
        std::pop_heap(rq.begin(), rq.end(), rd_less);
        const Rd r = rq.back();
        rq.pop_back();
        sched.push_back({now, r.bl, r.task, r.slab});
        events.push_back({now + prm.dur(tk[r.task].kind), r.task, true});
        std::push_heap(events.begin(), events.end(), ev_greater);
        --freew[p];
      }
    }
    if (events.empty()) break;
    std::pop_heap(events.begin(), events.end(), ev_greater);
    const Ev e = events.back();
    events.pop_back();
    now = e.t;
    if (e.worker) ++freew[tk[e.task].pool];
    if (--left[e.task] <= 0)
      for (int64_t q = soff[e.task]; q < soff[e.task + 1]; ++q)
        if (--indeg[succ[q]] == 0) push_task(succ[q]);
  }
  int64_t expect = 0;
  for (int64_t i = 0; i < ntask; ++i)
    if (tk[i].worker) expect += prm.parts(tk[i].kind);
  if ((int64_t)sched.size() != expect) return -2;
  if (bl_order)
    std::stable_sort(sched.begin(), sched.end(), [&](const Slot& a, const Slot& b) {
      if (a.bl != b.bl) return a.bl > b.bl;
      if (a.task != b.task) return a.task < b.task;
      return a.slab < b.slab;
    });
  else
    std::stable_sort(sched.begin(), sched.end(), [](const Slot& a, const Slot& b) { return a.start < b.start; });
  *out = std::move(sched);
  return 0;
}

}  // namespace sched
}  // namespace tileqr
