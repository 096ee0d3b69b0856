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

#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "dag_item.h"
#include "panel_fast.cuh"
#include "update_dmma.cuh"

namespace tileqr {
namespace dag {


__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// COPY item (multi-rank dataflow): push one packed reflector
// tile (V_p and T_p of every inner panel, update_v2.cuh layout) from this
// rank's slot to the same slot of a peer rank -- a peer-mapped (NVLink)
// pointer, or another buffer of the same GPU when the ranks are emulated.
// The source was just written by a panel item on another SM: L2 loads.
static __device__ __noinline__ void copy_body(const double* __restrict__ src, double* __restrict__ dst, int ndbl) {
  const int n2 = ndbl >> 1;
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (int e0 = threadIdx.x; e0 < n2; e0 += 4 * blockDim.x) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + u * (int)blockDim.x < n2) v[u] = __ldcg(s2 + e0 + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + u * (int)blockDim.x < n2) d2[e0 + u * blockDim.x] = v[u];
  }
  if ((ndbl & 1) && threadIdx.x == 0) dst[ndbl - 1] = __ldcg(src + ndbl - 1);
}

// Update items run the barrier-free packed-reflector body (update_v2.cuh,
// column groups of the packed tile streamed through a TMA ring) for every
// NB of the DAG kernel (TILEQR_DAG_STAGED: the staged double-buffered body of
// update_dmma.cuh for NB > 128, the previous design, for comparison).
template <int NB>
constexpr bool dag_v2() {
#ifdef TILEQR_DAG_STAGED
  return NB <= 128;
#else
  return NB <= 256;
#endif
}

// C2 prefetch (2 CTAs per SM, NB <= 128): during the last inner panel of an
// update item, thread 0 checks the next claimed item's dependencies without
// blocking and, if they hold and it is an update, copies that item's C2
// column slab (NB x W*8*MB doubles, contiguous in the tile) into a shared
// staging buffer with one TMA bulk copy; the next item then fills its
// accumulator registers from shared memory instead of from L2 at its start.
// Enabled where a ring of two stages plus the staging buffer fits the 2-CTA
// budget (110 KB) and the items are long enough (NB >= 96) for the check in
// the last panel to pay: same-box A/B at 10000^2, (128, 16) -1.4 %, while NB
// = 64 items (~5 us) lost 10-17 % to the extra latency on warp 0 and a
// one-stage budget (128, 32) halved the resident CTAs (+38 %).
template <int NB, int KW>
constexpr bool dag_c2pf() {
#ifdef TILEQR_NO_C2PF
  return false;
#else
  if constexpr (dag_v2<NB>() && dag_ctas_per_sm(NB) == 2 && NB >= 96 && NB % KW == 0) {
    using P = v2::Pk<NB, KW>;
    constexpr size_t stage = (size_t)(P::GDBL + P::PPG * P::TP) * sizeof(double);
    constexpr size_t c2 = (size_t)NB * dag_warps(NB) * 8 * dag_mb(NB) * sizeof(double);
    return 2 * stage + c2 <= 110 * 1024;
  } else {
    return false;
  }
#endif
}
template <int NB, int KW>
constexpr size_t dag_c2_bytes() {
  return dag_c2pf<NB, KW>() ? (size_t)NB * dag_warps(NB) * 8 * dag_mb(NB) * sizeof(double) : 0;
}

// Ring stages of the packed reflector tile per CTA: as many as fit in ~110 KB
// (2 CTAs per SM, NB <= 128; less the C2 staging buffer) or ~200 KB (1 CTA),
// at least 2, at most 8.
template <int NB, int KW>
constexpr int dag_stages() {
  if constexpr (dag_v2<NB>() && NB % KW == 0) {
    using P = v2::Pk<NB, KW>;
    constexpr size_t stage = (size_t)(P::GDBL + P::PPG * P::TP) * sizeof(double);
    constexpr size_t budget = (dag_ctas_per_sm(NB) == 2 ? 110 * 1024 : 200 * 1024) - dag_c2_bytes<NB, KW>();
#ifdef TILEQR_FULL_RING
    constexpr int s = P::NG;
#else
    constexpr int s = (int)(budget / stage);
#endif
    constexpr int s8 = s > 8 ? 8 : s;  // the kernel's mbarrier arrays hold 8
    return s8 < 2 ? 2 : (s8 > P::NG ? P::NG : s8);
  } else {
    return 1;
  }
}

template <int NB, int KW>
struct DagSmem {
  static constexpr int W = dag_warps(NB);
  static constexpr int MB = dag_mb(NB);
  using LS = upd::Layout<NB, MB, KW, false, false, W>;
  static constexpr size_t old_bytes =
      (2 * (size_t)LS::STAGE + (size_t)W * 8 * MB * (KW + 4)) * sizeof(double);
  static constexpr size_t v2_bytes =
      (NB % KW == 0) ? v2::Ring<NB, (NB % KW == 0 ? KW : 8), dag_stages<NB, KW>()>::bytes : 0;
  static constexpr size_t upd_bytes = dag_v2<NB>() ? v2_bytes + dag_c2_bytes<NB, KW>() : old_bytes;
  static constexpr size_t c2_off = v2_bytes;  // C2 staging buffer after the ring
  static constexpr size_t pan_bytes = sizeof(pf::FastSmem<NB, W>);
#ifdef TILEQR_ONE_CTA  // diagnostics: force one CTA per SM
  static constexpr size_t bytes0 = upd_bytes > pan_bytes ? upd_bytes : pan_bytes;
  static constexpr size_t bytes = bytes0 > 120 * 1024 ? bytes0 : 120 * 1024;
#else
  static constexpr size_t bytes = upd_bytes > pan_bytes ? upd_bytes : pan_bytes;
#endif
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// LOAD item: tiles (m, n), n in [n0, n1), m in [m0, m1), from the
// column-major staging buffer (padding of DESIGN.md R5: rows >= M are 0, a
// padded column j >= N is e_j when M <= j < MT*NB), flagging non-finite
// input.  Element pairs of a column (16-byte accesses on the tile side), 8
// pairs in flight per thread.
template <int NB>
__device__ __noinline__ void load_body(const DagIO* __restrict__ iop, int n0, int n1, int m0, int m1) {
  const DagIO io = *iop;
  const long long MT = io.MT;
  double* const tiles = io.tiles;
  constexpr int HP = NB / 2;  // row pairs per tile column segment
  int bad = 0;
  const int tm = m1 - m0;
  const long long per = (long long)(n1 - n0) * tm * NB * HP;  // pairs
  auto value = [&](long long i, long long j) {
    if (i < io.M && j < io.N) {
      const double v = __ldcg(io.in + i + j * io.ld);
      if (!isfinite(v)) bad = 1;
      return v;
    }
    return (j >= io.N && i == j && j >= io.M) ? 1.0 : 0.0;
  };
  for (long long e0 = threadIdx.x; e0 < per; e0 += 8LL * blockDim.x) {
    double2 v[8];
    long long dst[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      dst[u] = -1;
      if (e < per) {
        const long long t = e / ((long long)NB * HP), r = e - t * NB * HP;   // t: tile, r: pair in tile
        const long long n = n0 + t / tm, m = m0 + t % tm;
        const int jl = (int)(r / HP), il = 2 * (int)(r - (long long)jl * HP);
        const long long i = m * NB + il, j = n * NB + jl;
        v[u] = make_double2(value(i, j), value(i + 1, j));
        dst[u] = (m + n * MT) * NB * NB + il + (long long)jl * NB;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (dst[u] >= 0) *reinterpret_cast<double2*>(tiles + dst[u]) = v[u];
  }
  if (bad && io.info) *io.info = 1;  // benign race: every writer stores 1
}

// STORE item: tiles (m, n), m in [m0, m1) -> column-major output staging
// (16-byte loads from the tiles, 8 in flight per thread).
template <int NB>
__device__ __noinline__ void store_body(const DagIO* __restrict__ iop, int n, int m0, int m1) {
  const DagIO io = *iop;
  const long long MT = io.MT;
  const double* const tiles = io.tiles;
  constexpr int HP = NB / 2;
  const long long j0 = (long long)n * NB;
  const long long per = (long long)(m1 - m0) * NB * HP;
  for (long long e0 = threadIdx.x; e0 < per; e0 += 8LL * blockDim.x) {
    double2 v[8];
    long long i0[8], jj[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      i0[u] = -1;
      if (e < per) {
        const long long t = e / ((long long)NB * HP), r = e - t * NB * HP;
        const int jl = (int)(r / HP), il = 2 * (int)(r - (long long)jl * HP);
        const long long m = m0 + t;
        v[u] = __ldcg(reinterpret_cast<const double2*>(tiles + (m + (long long)n * MT) * NB * NB + il +
                                                       (long long)jl * NB));
        i0[u] = m * NB + il;
        jj[u] = j0 + jl;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0[u] < 0 || jj[u] >= io.N) continue;
      double* d = io.out + i0[u] + jj[u] * io.ld;
      if (i0[u] < io.M) d[0] = v[u].x;
      if (i0[u] + 1 < io.M) d[1] = v[u].y;
    }
  }
}

// 16-byte async copy global -> shared (L2 only), for the item descriptors
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc)
               : "memory");
}

// SSRFB slab of a tile row holding padding rows (~1/MT of the SSRFB items):
// only the first rbe row blocks of C2 (update_v2_body's RL form).  Out of
// line, so that its register allocation does not constrain the kernel's main
// update path; no claim-ahead hook in these items.
template <int NB, int KW, int MB, int W, int S>
__device__ __noinline__ void ssrfb_rows_body(const double* __restrict__ gpk, double* spk, uint64_t* full,
                                             uint64_t* empty, double* __restrict__ C1, double* __restrict__ C2,
                                             int col0, int cend, const double* c2s, uint64_t* c2bar,
                                             uint32_t c2par, uint64_t* c2free, int rbe) {
  v2::update_v2_body<NB, KW, MB, false, W, S, v2::NoHook, false, true>(gpk, spk, full, empty, C1, C2, col0,
                                                                       v2::NoHook(), cend, c2s, c2bar, c2par,
                                                                       c2free, rbe);
}

// prof (nullable, diagnostics): per item i, prof[3i .. 3i+2] = claim time,
// start time (inputs ready), end time in globaltimer ns.
//
// Claims overlap the tail of the running item: three inner panels before the
// end of an update item thread 0 claims the next item (atomicAdd), two before
// its descriptor is copied into the other smem slot, one before its operand
// tiles are prefetched into L2, so at the end only the dependency check
// remains.  A claimed item is held for about three inner panels.  Items are claimed in list order and a CTA's held
// item always follows its running one, so the smallest unfinished item is
// always running or about to (no deadlock).
//
// IO: the instantiation for tileqr_factor_host, with the LOAD / STORE items
// (their code in the kernel costs the device-only factorization ~1.8 %, same
// box A/B, so tileqr_factor runs an instantiation without them).
template <int NB, int KW, int MODE>
__global__ void __launch_bounds__(dag_warps(NB) * 32, dag_ctas_per_sm(NB))
dag_kernel(const Item* __restrict__ items, int nitems, int* next, int* done, int IB,
           unsigned long long* prof, const DagIO* io, int ca_lo, int ca_hi) {
  constexpr int W = dag_warps(NB);
  constexpr int MB = dag_mb(NB);
  constexpr int S = dag_stages<NB, KW>();
  static_assert(sizeof(Item) % 16 == 0, "Item is copied in 16-byte chunks");
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(16) Item s_desc[2];
  __shared__ int s_cur;
  __shared__ __align__(8) uint64_t full[8], empty[8];
  constexpr bool V2 = dag_v2<NB>();
  constexpr bool C2PF = dag_c2pf<NB, KW>();
  __shared__ __align__(8) uint64_t c2bar, c2free;  // C2 staging: data landed / every warp done reading
  __shared__ int s_c2item;                          // item whose C2 slab is staged (-1: none)
  // tail retirement (device-only factorization): the second CTA to arrive on
  // an SM stops claiming once it has started an item of the list's tail
  // (Item::aux[3] = 1), so the tail's items -- bound by the panel chain, not
  // by CTA slots -- have their SM to themselves. 0: keeps claiming, 1: retires
  // at the first tail item, 2: claims no more
  __shared__ int s_retire;
  constexpr bool RETIRE = MODE == kModePlainRetire;  // its own instantiation: the code costs the plain kernel 0.2-0.4 % at 10000^2
  uint32_t c2par = 0;   // all threads: phase of c2bar for the next staged slab
  uint32_t c2fpar = 0;  // thread 0: phase of c2free for the running update item
  if constexpr (C2PF) {
    if (threadIdx.x == 0) {
      v2::mbar_init(&c2bar, 1);
      v2::mbar_init(&c2free, W);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      s_c2item = -1;
    }
    __syncthreads();
  }
  if constexpr (RETIRE) {
    if (threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      s_retire = atomicAdd(next + 1 + (smid & 255u), 1) >= 1 ? 1 : 0;  // next[1..256]: reserved, zeroed per run
    }
  }
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
        if (RETIRE && s_retire == 2) cur = nitems;
        else cur = atomicAdd(next, 1);
        if (cur < nitems) fetch_desc(cur, slot);
      }
      nxt = -1;
      s_cur = cur;
      if (cur < nitems) {
        cp_async_wait<0>();
        const Item& it = s_desc[slot];
        if (RETIRE && it.aux[3] != 0 && s_retire == 1) s_retire = 2;
        int need[3], got[3];
        const int nd = it.ndep;
        if constexpr (MODE == kModeDist) {  // peer-written counters: system scope
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            need[d] = d < nd ? it.need[d] : 0;
            got[d] = d >= nd ? 0 : need[d] < 0 ? ld_acquire_sys(done + it.dep[d]) : ld_acquire(done + it.dep[d]);
          }
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const bool sys = need[d] < 0;
            const int want = sys ? -need[d] : need[d];
            while (got[d] < want) {
              __nanosleep(64);
              got[d] = sys ? ld_acquire_sys(done + it.dep[d]) : ld_acquire(done + it.dep[d]);
            }
          }
        } else {
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
        }
        if (prof) {  // start time; the claim time's low 10 bits carry SM id | C2 staged << 9
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          const unsigned long long tag = (smid & 0xffu) | ((C2PF && s_c2item == cur) ? 0x200u : 0u);
          prof[3 * (size_t)cur] = (prof[3 * (size_t)cur] & ~0x3ffull) | tag;
          prof[3 * (size_t)cur + 1] = globaltimer();
        }
        if constexpr (V2) {
          if (it.kind == kLarfb || it.kind == kSsrfb || (MODE == kModeTree && it.kind == kTtmqr)) {
            const int na = v2::active_warps<NB, MB, W>(it.col0, it.aux[0]);
            if (na > 0) v2::ring_start<NB, KW, S>(it.pk, smem, full, empty, na);
          }
        }
      }
    }
    __syncthreads();
    if (s_cur >= nitems) return;
    const int i = s_cur;
    const Item it = s_desc[slot];
    // claim-ahead hook of the update bodies (thread 0), one step per inner
    // panel near the end of the item: claim the next item, fetch its
    // descriptor, prefetch its operand tiles into L2 (bulk prefetch; data a
    // producer is still writing stays coherent in L2)
    constexpr int NPAN = NB / KW;
    constexpr int PC = NPAN >= 3 ? NPAN - 3 : 0, PD = NPAN >= 2 ? NPAN - 2 : 0, PF = NPAN - 1;
    auto hook = [&](int p) {
      if (threadIdx.x != 0) return;
      if (p == PC) {
        // diagnostics (TILEQR_DAG_CA_HEAD / _TAIL): no claim-ahead for the
        // items [0, ca_lo) and [ca_hi, nitems) of the list (same-box A/B at
        // 10000^2: within +-0.1 % for 300-2000 items at either end)
        if (i < ca_lo || i >= ca_hi) return;
        if (RETIRE && s_retire == 2) return;
        nxt = atomicAdd(next, 1);
        if constexpr (PC != PD) return;  // its result is first needed one panel later
      }
      if (nxt < 0 || nxt >= nitems) return;
      if (p == PD) fetch_desc(nxt, slot ^ 1);
#ifndef TILEQR_NO_HOOK_PREFETCH
      if (p == PF) {
        cp_async_wait<0>();
        const Item& n = s_desc[slot ^ 1];
        if (n.kind == kSsrfb || n.kind == kLarfb || (MODE == kModeTree && n.kind == kTtmqr)) {
          constexpr uint32_t tb = NB * NB * sizeof(double);
          const bool two = n.kind != kLarfb;
          bool staged = false;
          if constexpr (C2PF) {
            // the next item's inputs already final? (no spin: else it loads C2 from L2 itself)
            int got[3];
#pragma unroll
            for (int d = 0; d < 3; ++d)  // all three in flight at once
              got[d] = d >= n.ndep ? 0 : n.need[d] < 0 ? ld_acquire_sys(done + n.dep[d]) : ld_acquire(done + n.dep[d]);
            bool ready = n.aux[0] > n.col0;
#pragma unroll
            for (int d = 0; d < 3; ++d)
              ready = ready && (d >= n.ndep || got[d] >= (n.need[d] < 0 ? -n.need[d] : n.need[d]));
            if (ready) {
              // every warp of THIS item has read its slab from the staging buffer
              v2::mbar_wait(&c2free, c2fpar);
              const int ncol = min(dag_warps(NB) * 8 * dag_mb(NB), NB - n.col0);
              const uint32_t bytes = (uint32_t)(ncol * NB * sizeof(double));
              v2::fence_proxy_async();  // generic-proxy acquire before the async-proxy read
              v2::mbar_expect_tx(&c2bar, bytes);
              v2::bulk_g2s(smem + DagSmem<NB, KW>::c2_off / sizeof(double),
                           n.p[two ? 3 : 2] + (size_t)n.col0 * NB, bytes, &c2bar);
              staged = true;
            }
            s_c2item = staged ? nxt : -1;
          }
          if (!staged) prefetch_l2(n.p[two ? 3 : 2], tb);
          if (two) prefetch_l2(n.p[2], tb);
          if constexpr (V2) prefetch_l2(n.pk, (uint32_t)v2::Pk<NB, (NB % KW == 0 ? KW : 8)>::TOTAL * 8);
        }
      }
#endif
    };
    // C2 staging of this item (if the previous item's last panel staged it)
    const bool c2_here = C2PF && s_c2item == i;
    auto c2_src = [&]() -> const double* {
      return c2_here ? smem + DagSmem<NB, KW>::c2_off / sizeof(double) : nullptr;
    };
    auto c2_done = [&]() {  // after an update item: phases of the two staging barriers
      if constexpr (C2PF) {
        if (c2_here) c2par ^= 1u;
        if (threadIdx.x == 0) c2fpar ^= 1u;
      }
    };
    switch (it.kind) {
      case kGeqrt:  // inner panels [col0 & 0xffff, col0 >> 16)
        pf::panel_fast_body<false, NB, W, KW>(it.p[0], nullptr, it.p[2],
                                               reinterpret_cast<unsigned char*>(smem), V2 ? it.pk : nullptr,
                                               it.col0 & 0xffff, it.col0 >> 16);
        break;
      case kTsqrt:
        pf::panel_fast_body<true, NB, W, KW>(it.p[0], it.p[1], it.p[2],
                                              reinterpret_cast<unsigned char*>(smem), V2 ? it.pk : nullptr,
                                              it.col0 & 0xffff, it.col0 >> 16);
        break;
      case kLarfb:  // columns [col0, min(col0 + slab, aux[0])): the rest of the tile is padding
        if (it.aux[0] <= it.col0) break;
        if constexpr (V2) {
          v2::update_v2_body<NB, KW, MB, true, W, S>(it.pk, smem, full, empty, nullptr, it.p[2], it.col0, hook,
                                                     it.aux[0], c2_src(), &c2bar, c2par, C2PF ? &c2free : nullptr);
          c2_done();
        } else {
          upd::update_body<NB, MB, KW, true, true, false, W>(IB, KW, it.aux[0], it.p[0], it.p[1], nullptr,
                                                             it.p[2], 1, it.col0, smem);
        }
        break;
      case kLoad:
        if constexpr (MODE == kModeIO) load_body<NB>(io, it.aux[0], it.aux[1], it.aux[2], it.aux[3]);
        break;
      case kStore:
        if constexpr (MODE == kModeIO) store_body<NB>(io, it.aux[0], it.aux[2], it.aux[3]);
        break;
      case kCopy:
        if constexpr (MODE == kModeDist) copy_body(it.p[0], it.p[1], it.aux[0]);
        break;
      case kTtqrt:  // tree variant: merge R_b (upper triangle of tile p[1]) into R_a
        if constexpr (MODE == kModeTree)
          pf::panel_fast_body<true, NB, W, KW, true>(it.p[0], it.p[1], it.p[2],
                                                     reinterpret_cast<unsigned char*>(smem), V2 ? it.pk : nullptr,
                                                     it.col0 & 0xffff, it.col0 >> 16);
        break;
      case kTtmqr:  // tree variant: TTMQRT column slab
        if constexpr (MODE == kModeTree && V2) {
          if (it.aux[0] <= it.col0) break;
          v2::update_v2_body<NB, KW, MB, false, W, S, decltype(hook), true>(
              it.pk, smem, full, empty, it.p[2], it.p[3], it.col0, hook, it.aux[0], c2_src(), &c2bar, c2par,
              C2PF ? &c2free : nullptr);
          c2_done();
        }
        break;
      default:  // SSRFB: columns as LARFB; aux[1] > 0: rows of C2's tile above M (the rest padding)
        if (it.aux[0] <= it.col0) break;
        if constexpr (V2) {
          if (it.aux[1] > 0)
            ssrfb_rows_body<NB, KW, MB, W, S>(it.pk, smem, full, empty, it.p[2], it.p[3], it.col0, it.aux[0],
                                              c2_src(), &c2bar, c2par, C2PF ? &c2free : nullptr,
                                              (it.aux[1] + 7) / 8);
          else
            v2::update_v2_body<NB, KW, MB, false, W, S>(it.pk, smem, full, empty, it.p[2], it.p[3], it.col0,
                                                        hook, it.aux[0], c2_src(), &c2bar, c2par,
                                                        C2PF ? &c2free : nullptr);
          c2_done();
        } else {
          upd::update_body<NB, MB, KW, true, false, false, W>(IB, KW, it.aux[0], it.p[0], it.p[1], it.p[2],
                                                              it.p[3], 1, it.col0, smem);
        }
        break;
    }
    // every thread orders its generic-proxy shared-memory accesses of this
    // item before the async-proxy (TMA) writes of the next item into the same
    // shared memory (a CTA barrier alone does not order across proxies)
    v2::fence_proxy_async_smem();
    __syncthreads();  // every write of the item issued; smem free for the next item
    if (threadIdx.x == 0) {
      // STORE counters are read by the copy engine (cuStreamWaitValue32 on
      // the device-to-host stream), not by GPU threads: publish them at
      // system scope
      if (MODE == kModeIO && it.kind == kStore) {
        __threadfence_system();
      } else if (MODE == kModeDist && it.kind == kCopy) {
        // the pushed tile (NVLink stores of every thread, ordered before this
        // point by the CTA barrier) is released to the peer at system scope
        __threadfence_system();
        atomicAdd_system(reinterpret_cast<int*>(it.p[2]), 1);
      } else {
#ifdef TILEQR_FENCE_ATOMIC
        __threadfence();
#endif
      }
#ifdef TILEQR_FENCE_ATOMIC
      atomicAdd(done + it.task, 1);
#else
      if (MODE == kModeIO && it.kind == kStore) {
        atomicAdd(done + it.task, 1);
      } else {
        // release reduction: the item's writes (every thread's, ordered before
        // this point by the CTA barrier) become visible before the count does;
        // consumers acquire the counter (ld.acquire.gpu)
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(done + it.task) : "memory");
      }
#endif
      if (prof) prof[3 * (size_t)i + 2] = globaltimer();
    }
    slot ^= 1;
  }
}

template <int NB, int KW>
int launch_dag_t(int IB, const Item* items, int nitems, int* next, int* done, int nsm,
                 unsigned long long* prof, cudaStream_t s, int* grid_out, const DagIO* io, int mode) {
  auto kern = mode == kModeIO ? dag_kernel<NB, KW, kModeIO>
            : mode == kModeDist ? dag_kernel<NB, KW, kModeDist>
            : mode == kModeTree ? dag_kernel<NB, KW, kModeTree>
            : mode == kModePlainRetire ? dag_kernel<NB, KW, kModePlainRetire> : dag_kernel<NB, KW, kModePlain>;
  const size_t bytes = DagSmem<NB, KW>::bytes;
  static_assert(DagSmem<NB, KW>::bytes <= 227 * 1024, "DAG kernel shared memory");
  TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  int per_sm = 0;
  constexpr int kThreads = dag_warps(NB) * 32;
  TQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, bytes));
  if (per_sm < 1) {
    set_error("DAG kernel does not fit on an SM");
    return TILEQR_ERR_CUDA;
  }
  if (nitems <= 0) return 0;
  int grid = std::min(nitems, nsm * per_sm);
  if (const char* e = getenv("TILEQR_DAG_GRID")) {  // diagnostics: fewer resident CTAs
    const int g = atoi(e);
    if (g > 0 && g < grid) grid = g;
  }
  if (grid_out) *grid_out = grid;
  int ca_head = 0, ca_tail = 0;
  if (const char* e = getenv("TILEQR_DAG_CA_HEAD")) ca_head = atoi(e);
  if (const char* e = getenv("TILEQR_DAG_CA_TAIL")) ca_tail = atoi(e);
  kern<<<grid, kThreads, bytes, s>>>(items, nitems, next, done, IB, prof, io, ca_head, nitems - ca_tail);
  TQ_LAUNCH_CHECK();
  return 0;
}

template <int NB>
int launch_dag_nb(int IB, const Item* items, int nitems, int* next, int* done, int nsm,
                  unsigned long long* prof, cudaStream_t s, int* grid_out, const DagIO* io, int mode) {
  switch (IB) {
    case 8: return launch_dag_t<NB, 8>(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 16: return launch_dag_t<NB, 16>(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    case 24:
      if constexpr (NB % 24 == 0) return launch_dag_t<NB, 24>(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
      set_error("DAG kernel: IB does not divide NB");
      return TILEQR_ERR_CUDA;
    case 32: return launch_dag_t<NB, 32>(IB, items, nitems, next, done, nsm, prof, s, grid_out, io, mode);
    default: set_error("DAG kernel: IB not in {8,16,24,32}"); return TILEQR_ERR_CUDA;
  }
}

}  // namespace dag
}  // namespace tileqr
