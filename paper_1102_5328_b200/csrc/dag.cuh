// dag.cuh -- dataflow execution of the whole tile-QR DAG in ONE persistent
// kernel (Fig. 1b, 163-164).
//
// PLASMA runs the DAG of GEQRT / TSQRT / LARFB / SSRFB tasks with a static
// schedule over CPU cores.  The GPU counterpart here is a
// persistent kernel of one 8-warp CTA per SM that claims work items from a
// host-built list in a fixed priority order (bottom level first, a
// topological order) with one atomicAdd, waits for the item's inputs on
// per-task completion counters (acquire loads), runs the task body (the same
// device code as the batched kernels: panel_fast.cuh / update_dmma.cuh), and
// publishes completion (fence + atomicAdd).  No level barriers: the panel
// chain advances as soon as the tiles it reads are final while the trailing
// updates of earlier steps fill the other SMs.  Deadlock-free because items
// are claimed in a topological order by CTAs that are all resident (every
// claimed item's dependencies were claimed earlier by running CTAs).
//
// Every tile sees exactly the same sequence of operations with the same
// arithmetic as in the level-synchronous launcher, so results are bitwise
// identical to it.
#pragma once

#include <algorithm>

#include "dag_item.h"
#include "panel_fast.cuh"
#include "update_dmma.cuh"

namespace tileqr {
namespace dag {

constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Update items of NB <= 128 run the barrier-free packed-reflector body
// (update_v2.cuh, the whole packed tile staged by TMA); larger NB the staged
// double-buffered body (update_dmma.cuh).
template <int NB>
constexpr bool dag_v2() { return NB <= 128; }

template <int NB, int KW>
struct DagSmem {
  static constexpr int MB = dag_mb(NB);
  using LS = upd::Layout<NB, MB, KW, false, false, kWarps>;
  static constexpr size_t old_bytes =
      (2 * (size_t)LS::STAGE + (size_t)kWarps * 8 * MB * (KW + 4)) * sizeof(double);
  static constexpr size_t v2_bytes = (NB % KW == 0) ? (size_t)v2::Pk<NB, (NB % KW == 0 ? KW : 8)>::TOTAL * sizeof(double) : 0;
  static constexpr size_t upd_bytes = dag_v2<NB>() ? v2_bytes : old_bytes;
  static constexpr size_t pan_bytes = sizeof(pf::FastSmem<NB, kWarps>);
  static constexpr size_t bytes = upd_bytes > pan_bytes ? upd_bytes : pan_bytes;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 16-byte async copy global -> shared (L2 only), for the item descriptors
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc)
               : "memory");
}

// prof (nullable, diagnostics): per item i, prof[3i .. 3i+2] = claim time,
// start time (inputs ready), end time in globaltimer ns.
//
// Claims overlap the tail of the running item: during the second-to-last
// inner panel of an update item thread 0 claims the next item (atomicAdd),
// during the last one its descriptor is copied into the other smem slot, so
// at the end only the dependency check remains.  A claimed item is held for
// about two inner panels.  Items are claimed in list order and a CTA's held
// item always follows its running one, so the smallest unfinished item is
// always running or about to (no deadlock).
template <int NB, int KW>
__global__ void __launch_bounds__(kThreads, 1)
dag_kernel(const Item* __restrict__ items, int nitems, int* next, int* done, int IB,
           unsigned long long* prof) {
  constexpr int MB = dag_mb(NB);
  static_assert(sizeof(Item) % 16 == 0, "Item is copied in 16-byte chunks");
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(16) Item s_desc[2];
  __shared__ int s_cur;
  __shared__ __align__(8) uint64_t bars[8];
  constexpr bool V2 = dag_v2<NB>();
  int nxt = -1;   // thread 0: item claimed ahead (-1: none)
  int slot = 0;   // descriptor slot of the running item (all threads)
  auto fetch_desc = [&](int i, int sl) {
    if (prof) prof[3 * (size_t)i] = globaltimer();
    for (int c = 0; c < (int)(sizeof(Item) / 16); ++c)
      cp_async16(reinterpret_cast<char*>(&s_desc[sl]) + 16 * c, reinterpret_cast<const char*>(items + i) + 16 * c);
    cp_async_commit();
  };
  for (;;) {
    if (threadIdx.x == 0) {
      int cur = nxt;
      if (cur < 0) {
        cur = atomicAdd(next, 1);
        if (cur < nitems) fetch_desc(cur, slot);
      }
      nxt = -1;
      s_cur = cur;
      if (cur < nitems) {
        cp_async_wait<0>();
        const Item& it = s_desc[slot];
        int need[3], got[3];
        const int nd = it.ndep;
#pragma unroll
        for (int d = 0; d < 3; ++d) {  // all flags in flight at once
          need[d] = d < nd ? it.need[d] : 0;
          got[d] = d < nd ? ld_acquire(done + it.dep[d]) : 0;
        }
#pragma unroll
        for (int d = 0; d < 3; ++d)
          while (got[d] < need[d]) {
            __nanosleep(64);
            got[d] = ld_acquire(done + it.dep[d]);
          }
        if (prof) prof[3 * (size_t)cur + 1] = globaltimer();
        if constexpr (V2) {
          if (it.kind == kLarfb || it.kind == kSsrfb) v2::issue_packed_loads<NB, KW>(it.pk, smem, bars);
        }
      }
    }
    __syncthreads();
    if (s_cur >= nitems) return;
    const int i = s_cur;
    const Item it = s_desc[slot];
    // claim-ahead hook of the update bodies (thread 0)
    constexpr int NPAN = NB / KW;
    auto hook = [&](int p) {
      if (threadIdx.x != 0) return;
      if (p == (NPAN >= 2 ? NPAN - 2 : 0)) nxt = atomicAdd(next, 1);
      if (p == NPAN - 1 && nxt < nitems) fetch_desc(nxt, slot ^ 1);
    };
    switch (it.kind) {
      case kGeqrt:  // inner panels [col0 & 0xffff, col0 >> 16)
        pf::panel_fast_body<false, NB, kWarps>(IB, it.p[0], nullptr, it.p[2],
                                               reinterpret_cast<unsigned char*>(smem), V2 ? it.pk : nullptr,
                                               it.col0 & 0xffff, it.col0 >> 16);
        break;
      case kTsqrt:
        pf::panel_fast_body<true, NB, kWarps>(IB, it.p[0], it.p[1], it.p[2],
                                              reinterpret_cast<unsigned char*>(smem), V2 ? it.pk : nullptr,
                                              it.col0 & 0xffff, it.col0 >> 16);
        break;
      case kLarfb:
        if constexpr (V2)
          v2::update_v2_body<NB, KW, MB, true, kWarps>(smem, bars, 0, nullptr, it.p[2], it.col0, hook);
        else upd::update_body<NB, MB, KW, true, true, false, kWarps>(IB, KW, NB, it.p[0], it.p[1], nullptr,
                                                                     it.p[2], 1, it.col0, smem);
        break;
      default:
        if constexpr (V2)
          v2::update_v2_body<NB, KW, MB, false, kWarps>(smem, bars, 0, it.p[2], it.p[3], it.col0, hook);
        else upd::update_body<NB, MB, KW, true, false, false, kWarps>(IB, KW, NB, it.p[0], it.p[1], it.p[2],
                                                                      it.p[3], 1, it.col0, smem);
        break;
    }
    __syncthreads();  // every write of the item issued; smem free for the next item
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(done + it.task, 1);
      if (prof) prof[3 * (size_t)i + 2] = globaltimer();
    }
    slot ^= 1;
  }
}

template <int NB, int KW>
int launch_dag_t(int IB, const Item* items, int nitems, int* next, int* done, int nsm,
                 unsigned long long* prof, cudaStream_t s) {
  auto kern = dag_kernel<NB, KW>;
  const size_t bytes = DagSmem<NB, KW>::bytes;
  static_assert(DagSmem<NB, KW>::bytes <= 227 * 1024, "DAG kernel shared memory");
  TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  int per_sm = 0;
  TQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, bytes));
  if (per_sm < 1) {
    set_error("DAG kernel does not fit on an SM");
    return TILEQR_ERR_CUDA;
  }
  const int grid = std::min(nitems, nsm * per_sm);
  kern<<<grid, kThreads, bytes, s>>>(items, nitems, next, done, IB, prof);
  TQ_LAUNCH_CHECK();
  return 0;
}

template <int NB>
int launch_dag_nb(int IB, const Item* items, int nitems, int* next, int* done, int nsm,
                  unsigned long long* prof, cudaStream_t s) {
  switch (IB) {
    case 8: return launch_dag_t<NB, 8>(IB, items, nitems, next, done, nsm, prof, s);
    case 16: return launch_dag_t<NB, 16>(IB, items, nitems, next, done, nsm, prof, s);
    case 24:
      if constexpr (NB % 24 == 0) return launch_dag_t<NB, 24>(IB, items, nitems, next, done, nsm, prof, s);
      set_error("DAG kernel: IB does not divide NB");
      return TILEQR_ERR_CUDA;
    case 32: return launch_dag_t<NB, 32>(IB, items, nitems, next, done, nsm, prof, s);
    default: set_error("DAG kernel: IB not in {8,16,24,32}"); return TILEQR_ERR_CUDA;
  }
}

}  // namespace dag
}  // namespace tileqr
