// dist_dag.h -- the multi-rank dataflow plan (dist_dag.cu): global task ids,
// the global claim order, and the per-rank work lists of the dataflow kernel.
#pragma once

#include <stdint.h>

#include <memory>
#include <vector>

#include "dag_item.h"
#include "sched.h"

namespace tileqr {
namespace dd {

struct Plan {
  int64_t M = 0, N = 0, MT = 0, NT = 0, KT = 0;
  int NB = 0, IB = 0, P = 1, SC = 0, NS = 1, cols = 0, nslab = 1;
  std::vector<int64_t> offL, offT, offS, cpo;
  std::vector<std::vector<int>> dests;  // per panel k: ranks receiving its reflector tiles
  int64_t nG = 0, nL = 0, nT = 0, nS = 0, base_cp = 0, base_ar = 0, ntask = 0;
  std::vector<sched::Task> tasks;       // global task graph (pool = rank)
  std::vector<sched::Slot> order;       // global claim order
  int owner(int64_t n) const { return (int)(n % P); }
  int64_t idG(int64_t k, int s) const { return k * NS + s; }
  int64_t idL(int64_t k, int64_t n) const { return nG + offL[k] + (n - k - 1); }
  int64_t idT(int64_t k, int64_t m, int s) const { return nG + nL + offT[k] + (m - k - 1) * NS + s; }
  int64_t idS(int64_t k, int64_t m, int64_t n) const {
    return nG + nL + nT + offS[k] + (m - k - 1) * (NT - k - 1) + (n - k - 1);
  }
  int64_t idCP(int64_t k, int64_t m, int di) const {
    return base_cp + cpo[k] + (m - k) * (int64_t)dests[k].size() + di;
  }
  int64_t idAR(int64_t k, int64_t m, int di) const {
    return base_ar + cpo[k] + (m - k) * (int64_t)dests[k].size() + di;
  }
  // slot of reflector tile (k, m), m >= k, in every rank's slot buffer
  int64_t slot(int64_t k, int64_t m) const;
  int64_t nslots() const;
};

// Device buffers of one rank (peer-mapped pointers for remote ranks):
// local tile columns, local T, the slot buffer of packed reflector tiles and
// the completion counters (ntask ints).
struct RankBufs {
  double* A;
  double* T;
  double* slots;
  int* done;
};

int64_t local_cols(int64_t NT, int P, int rank);
int build_plan(int64_t M, int64_t N, int NB, int IB, int P, int workers, int SC, std::shared_ptr<Plan>* out);
// rank >= 0: that rank's items (counter indices local to its array);
// rank < 0 with emul: every rank's items, counters of rank r at r * ntask.
int emit_items(const Plan& p, int rank, const std::vector<RankBufs>& bufs, bool emul,
               std::vector<dag::Item>* items);

}  // namespace dd
}  // namespace tileqr
