// update_v2.cuh -- barrier-free DMMA trailing update (SSRFB / LARFB, Q^T
// form) of the tile QR,
// fed by a PACKED copy of the reflector tile that the panel kernels write.
//
// For every inner panel p of IB reflectors, ascending:
//   step A  W^T  = C1[p rows]^T + C2^T V_p          (LARFB: C^T V_p)
//   step B  W'^T = W^T T_p                           (W' = T_p^T W)
//   C1[p rows] -= W'                                 (SSRFB only)
//   step C  C2^T -= W'^T V_p^T                       (LARFB: C^T -= W'^T V_p^T)
//
// Design (B200, FP64 mma.sync.m8n8k4 = SASS DMMA.8x8x4; tcgen05 has no f64):
//  * Each warp owns 8*MB columns of C2 for ALL NB rows, in registers, as the
//    transposed accumulator C2^T, for the whole task (C2 crosses HBM once).
//  * The k index of every m8n8k4 step is permuted so that the A fragment of
//    a step is an accumulator register: step A feeds C2^T (k = rows
//    8rb+2t+j), step B feeds W^T (k = reflectors 8kb+2t+s) and step C feeds
//    W'^T (same).  W never leaves registers: no shared-memory round trip, no
//    __syncwarp, no CTA barrier anywhere in the task.
//  * V and T come from the packed tile (below), a smem image that TMA bulk
//    copies (cp.async.bulk + mbarrier complete_tx) land in one piece per
//    column group; each warp waits on the group's mbarrier and then runs all
//    its panels independently of the other warps.
//  * C1 rows of panel p+1 are prefetched into registers during step C of
//    panel p and serve both as W's initial value and for C1 -= W'.
//
// Packed reflector tile (written by the GEQRT/TSQRT kernels, panel_fast.cuh):
//   V: NG column groups of GW columns (GW = 16 for IB in {8,16}, 32 for IB in
//   {24,32}), each an NB x GW row-major block; element (r, c) of a group at
//   r*GW + (c ^ pk_f(r & 7)), pk_f(r) = (r&1) | (r&2)<<2 | (r&4).  Panel p
//   occupies group p / PPG, columns (p % PPG)*PW + [0, IB).  This XOR swizzle
//   makes both DMMA B-fragment patterns conflict free: step A reads
//   (row 8rb+2t+j, col 8nb+g), step C reads (row 8rb+g, col 8nb+2t+s).
//   GEQRT tiles store the unit lower trapezoid V (explicit 0 / 1).
//   T: after V, panel p at TOFF + p*IB*LDT2, T_p(l, i) at l*LDT2 + i
//   (LDT2 == 2 mod 16: conflict free for step B's (l = 8kb+2t+s, i = 8nb+g)).
#pragma once

#include <stdint.h>

#include "dmma.cuh"
#include "internal.h"

namespace tileqr {
namespace v2 {

// Wide panels (IB in {40, 48, 56, 64}): one panel per group of GW = IB rounded
// up to 16 columns (the XOR swizzle flips column bits 0-3 only, so it stays
// inside the group), T_p with ld 66 (== 2 mod 16), one warp column block
// (MB = 1) per warp; a one-stage ring where two stages do not fit.
template <int NB, int IB>
struct Pk {
  static constexpr int GW = IB <= 16 ? 16 : IB <= 32 ? 32 : (IB + 15) / 16 * 16;  // group width
  static constexpr int PW = IB == 8 ? 8 : GW;             // packed panel width
  static constexpr int PPG = GW / PW;                     // panels per group
  static constexpr int NP = NB / IB;                      // panels
  static constexpr int NG = (NP + PPG - 1) / PPG;         // groups
  static constexpr int LDT2 = IB <= 16 ? 18 : IB <= 32 ? 34 : 66;
  static constexpr int GDBL = NB * GW;                    // doubles per V group
  static constexpr int TOFF = NG * GDBL;
  static constexpr int TP = IB * LDT2;                    // doubles per T_p
  static constexpr int TOTAL = TOFF + NP * TP;            // doubles per packed tile
  static constexpr int NBK = IB / 8;
  static_assert(IB % 8 == 0 && IB <= 64 && NB % IB == 0, "packed tile geometry");
};

__host__ __device__ constexpr int pk_f(int r) { return (r & 1) | ((r & 2) << 2) | (r & 4); }

// packed-tile size in doubles for a runtime (NB, IB) (0 if unsupported)
inline size_t pk_doubles(int NB, int IB) {
  if (IB % 8 || IB > 64 || NB % IB) return 0;
  const int GW = IB <= 16 ? 16 : IB <= 32 ? 32 : (IB + 15) / 16 * 16, PW = IB == 8 ? 8 : GW, PPG = GW / PW;
  const int NP = NB / IB, NG = (NP + PPG - 1) / PPG, LDT2 = IB <= 16 ? 18 : IB <= 32 ? 34 : 66;
  return (size_t)NG * NB * GW + (size_t)NP * IB * LDT2;
}

// a wide-panel geometry is built only where two ring stages fit (<= 220 KB)
template <int NB, int IB>
constexpr bool pk_fits() {
  if constexpr (IB % 8 != 0 || IB > 64 || NB % IB != 0) {
    return false;
  } else {
    using P = Pk<NB, IB>;
    return IB <= 32 || (size_t)(P::GDBL + P::PPG * P::TP) * sizeof(double) <= 220 * 1024;
  }
}

// ---- mbarrier / bulk-copy helpers -------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TQ_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TQ_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// generic-proxy accesses before / async-proxy (TMA) accesses after
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Shared-memory ring of S stages for the column groups of a packed tile:
// stage s = [V block of a group (GDBL) | T_p of its panels (PPG * TP)].
// S >= NG stages hold the whole tile (no refill).
template <int NB, int IB, int S>
struct Ring {
  using P = Pk<NB, IB>;
  static constexpr int SD = P::GDBL + P::PPG * P::TP;  // doubles per stage
  static constexpr int NS = S < P::NG ? S : P::NG;     // stages in use
  static constexpr size_t bytes = (size_t)NS * SD * sizeof(double);
};

// Thread 0: copy group q of the packed tile gpk into its stage (barrier full[q % S]).
template <int NB, int IB, int S>
__device__ __forceinline__ void ring_issue(const double* __restrict__ gpk, double* spk, uint64_t* full, int q) {
  using P = Pk<NB, IB>;
  using RG = Ring<NB, IB, S>;
  const int st = q % RG::NS;
  const int p0 = q * P::PPG;
  const int np = (P::NP - p0) < P::PPG ? (P::NP - p0) : P::PPG;
  const uint32_t vb = P::GDBL * 8, tb = np * P::TP * 8;
  double* dst = spk + (size_t)st * RG::SD;
  mbar_expect_tx(&full[st], vb + tb);
  bulk_g2s(dst, gpk + q * P::GDBL, vb, &full[st]);
  bulk_g2s(dst + P::GDBL, gpk + P::TOFF + p0 * P::TP, tb, &full[st]);
}

// Thread 0, before the CTA barrier that starts an update item: (re)arm the
// ring barriers (full: 1 arrival + tx bytes; empty: one arrival per active
// warp) and issue the first stages.
template <int NB, int IB, int S>
__device__ __forceinline__ void ring_start(const double* __restrict__ gpk, double* spk, uint64_t* full,
                                           uint64_t* empty, int nact) {
  using RG = Ring<NB, IB, S>;
  fence_proxy_async();
  for (int s = 0; s < RG::NS; ++s) {
    mbar_init(&full[s], 1);
    mbar_init(&empty[s], nact);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int q = 0; q < RG::NS; ++q) ring_issue<NB, IB, S>(gpk, spk, full, q);
}

// All threads of a CTA (kThreads): write panel p of the packed tile from
// accessor callbacks v(r, i) (reflector matrix V_p, row r < NB, column i < IB,
// unit / zero entries included) and t(l, i) (T_p, upper triangle).
template <int NB, int IB, int kThreads, class VF, class TF>
__device__ __forceinline__ void pack_panel(double* __restrict__ gpk, int p, VF v, TF t) {
  using P = Pk<NB, IB>;
  const int q = p / P::PPG, cb = (p % P::PPG) * P::PW;
  double* gv = gpk + q * P::GDBL;
  // each packed row of the group holds PW (of GW) columns of this panel; for
  // PPG == 1 write the whole row (padding columns of IB = 24 as 0)
  constexpr int WC = P::PPG == 1 ? P::GW : P::PW;
  for (int e = threadIdx.x; e < NB * WC; e += kThreads) {
    const int r = e / WC, x = e - r * WC;
    int pos, i;
    if (P::PPG == 1) {
      pos = x;
      i = x ^ pk_f(r & 7);
    } else {
      i = x;
      pos = (cb + x) ^ pk_f(r & 7);
    }
    gv[r * P::GW + pos] = (i < IB) ? v(r, i) : 0.0;
  }
  double* gt = gpk + P::TOFF + p * P::TP;
  for (int e = threadIdx.x; e < IB * P::LDT2; e += kThreads) {
    const int l = e / P::LDT2, i = e - l * P::LDT2;
    gt[e] = (i < IB && l <= i) ? t(l, i) : 0.0;
  }
}

// ---- the update body ---------------------------------------------------------
// Columns [col0, col0 + W*8*MB) of one task; spk = the smem packed tile whose
// group barriers `bars` were armed by issue_packed_loads (parity `par`).
struct NoHook {
  __device__ void operator()(int) const {}
};

// hook(p) is called by every thread at the start of panel p (the DAG kernel
// claims its next work item there, overlapping the claim with the tail).
// Ring of S stages (ring_start issued by thread 0 before the CTA barrier);
// gpk = the packed tile in global memory (refills).
//
// TT: the TTMQRT of the tree variant: V2 of panel p is zero
// below row c0 + IB (the packed tile of a TTQRT holds those zeros), so steps A
// and C skip those row blocks -- half the flops of the SSRFB form.
//
// c2s (DAG kernel, nullable): the item's C2 column slab already staged in
// shared memory by a TMA bulk copy (column-major, ld NB, from column col0),
// complete when c2bar reaches phase c2par; c2free (nullable) gets one arrival
// per warp once the warp no longer reads the staging buffer.
//
// RL (runtime row limit, SSRFB of a tile row holding the padding rows >= M):
// only the first rbe row blocks of C2 are read, updated and written.  V2 is
// exactly zero in the rows past M (TSQRT of zero rows), so those rows add
// nothing to W in step A and step C leaves them as they are.
template <int NB, int IB, int MB, bool LARFB, int W, int S, class Hook = NoHook, bool TT = false, bool RL = false>
__device__ __forceinline__ void update_v2_body(const double* __restrict__ gpk, double* spk, uint64_t* full,
                                               uint64_t* empty, double* __restrict__ C1, double* __restrict__ C2,
                                               int col0, Hook hook = Hook(), int cend = NB,
                                               const double* c2s = nullptr, uint64_t* c2bar = nullptr,
                                               uint32_t c2par = 0, uint64_t* c2free = nullptr, int rbe = NB / 8) {
  using P = Pk<NB, IB>;
  using RG = Ring<NB, IB, S>;
  constexpr int RB = NB / 8;
  constexpr int NBK = P::NBK;
  constexpr bool SPLIT = NBK * MB < 4;  // two partial sums per step-A block when chains are few
  // C2 stored during the last panel's step C, one group of ES row blocks at a
  // time (NB >= 96; same-box A/B, r02as: 10000^2 (128, 16) -0.35 %, 4096^2
  // -1.0 %; NB = 64 +0.3 %, not used there)
#ifndef TILEQR_ES_GROUP
#define TILEQR_ES_GROUP 4
#endif
  constexpr int ES = TILEQR_ES_GROUP;
#ifdef TILEQR_NO_C2_EARLY_STORE
  constexpr bool ESTORE = false;
#else
  constexpr bool ESTORE = !TT && NB >= 96;
#endif
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane & 3, g = lane >> 2;
  const int wc0 = col0 + warp * 8 * MB;  // first column of this warp
  // idle warp (8*MB*W > NB, or every column from wc0 on is padding: cend,
  // the item's column limit): no CTA barrier follows
  if (wc0 >= cend) {
    if (c2free && lane == 0) mbar_arrive(c2free);
    for (int p = 0; p < P::NP; ++p) hook(p);
    return;
  }

  // ---- C2 slab -> registers: acc[mb][rb][j] = C2(8rb+2t+j, wc0+8mb+g) --------
  double acc[MB][RB][2];
  if (c2s) {  // staged by the previous item's last panel
    mbar_wait(c2bar, c2par);
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const double* src = c2s + 2 * t + (size_t)(wc0 - col0 + 8 * mb + g) * NB;
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        if (RL && rb >= rbe) {
          acc[mb][rb][0] = acc[mb][rb][1] = 0.0;
          continue;
        }
        const double2 v = *reinterpret_cast<const double2*>(src + 8 * rb);
        acc[mb][rb][0] = v.x;
        acc[mb][rb][1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const double* src = C2 + 2 * t + (size_t)(wc0 + 8 * mb + g) * NB;
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        if (RL && rb >= rbe) {
          acc[mb][rb][0] = acc[mb][rb][1] = 0.0;
          continue;
        }
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src + 8 * rb));  // streaming: L2 only
        acc[mb][rb][0] = v.x;
        acc[mb][rb][1] = v.y;
      }
    }
  }
  if (c2free) {  // done with the staging buffer: the next slab's TMA may overwrite it
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(c2free);
  }
  // C1 rows of panel 0 (SSRFB): c1n[mb][nb][j] = C1(c0 + 8nb+2t+j, col)
  double c1n[MB][NBK][2];
  if (!LARFB) {
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NBK; ++nb) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(C1 + 8 * nb + 2 * t + (size_t)(wc0 + 8 * mb + g) * NB));
        c1n[mb][nb][0] = v.x;
        c1n[mb][nb][1] = v.y;
      }
  }

#pragma unroll 1
  for (int p = 0; p < P::NP; ++p) {
    hook(p);
    const int c0 = p * IB;
    const int q = p / P::PPG, cb = (p % P::PPG) * P::PW;
    const int st = q % RG::NS;
    if (p % P::PPG == 0) mbar_wait(&full[st], (q / RG::NS) & 1);
    __syncwarp();  // reconverge (hook / refill / arrive are single-lane) before mma.sync.aligned
    const double* Vq = spk + (size_t)st * RG::SD;
    const double* Tp = Vq + P::GDBL + (p % P::PPG) * P::TP;

    // ---- step A: W^T = C1p^T + C2^T V_p ----------------------------------------
    double w[MB][NBK][2], w2[MB][NBK][2];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NBK; ++nb)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          w[mb][nb][j] = LARFB ? 0.0 : c1n[mb][nb][j];
          w2[mb][nb][j] = 0.0;
        }
    // B fragment (row 8rb+2t+j, col cb+8nb+g): per-thread base per (j, nb), the
    // row block rb is a compile-time offset
    const int rb0 = LARFB ? (c0 >> 3) : 0;  // V_p is zero above row c0
    const double* pa[2][NBK];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int nb = 0; nb < NBK; ++nb) pa[j][nb] = Vq + (2 * t + j) * P::GW + ((cb + 8 * nb + g) ^ pk_f(2 * t + j));
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      if (rb < rb0) continue;
      if (TT && 8 * rb >= c0 + IB) continue;
      if (RL && rb >= rbe) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) {
          const double bf = pa[j][nb][8 * rb * P::GW];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) {
            if (SPLIT && j == 1) dmma(w2[mb][nb][0], w2[mb][nb][1], acc[mb][rb][1], bf);
            else dmma(w[mb][nb][0], w[mb][nb][1], acc[mb][rb][j], bf);
          }
        }
    }
    if (SPLIT) {
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) {
          w[mb][nb][0] += w2[mb][nb][0];
          w[mb][nb][1] += w2[mb][nb][1];
        }
    }

    // ---- step B: W'^T(:, i) = sum_{l <= i} W^T(:, l) T_p(l, i), in place ---------
#pragma unroll
    for (int nb = NBK - 1; nb >= 0; --nb) {
      double o[MB][2];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) o[mb][0] = o[mb][1] = 0.0;
#pragma unroll
      for (int kb = 0; kb <= nb; ++kb)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const double bf = Tp[(8 * kb + 2 * t + s) * P::LDT2 + 8 * nb + g];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) dmma(o[mb][0], o[mb][1], w[mb][kb][s], bf);
        }
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        w[mb][nb][0] = o[mb][0];
        w[mb][nb][1] = o[mb][1];
      }
    }

    // ---- C1[p rows] -= W' (c1n still holds them), then prefetch panel p+1's --
    if (!LARFB) {
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) {
          double* dst = C1 + c0 + 8 * nb + 2 * t + (size_t)(wc0 + 8 * mb + g) * NB;
          *reinterpret_cast<double2*>(dst) =
              make_double2(c1n[mb][nb][0] - w[mb][nb][0], c1n[mb][nb][1] - w[mb][nb][1]);
        }
      if (p + 1 < P::NP) {  // in flight during step C
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
          for (int nb = 0; nb < NBK; ++nb) {
            const double2 v = __ldcg(reinterpret_cast<const double2*>(C1 + c0 + IB + 8 * nb + 2 * t +
                                                                     (size_t)(wc0 + 8 * mb + g) * NB));
            c1n[mb][nb][0] = v.x;
            c1n[mb][nb][1] = v.y;
          }
      }
    }

    // ---- step C: C2^T(:, r) -= sum_i W'^T(:, i) V_p(r, i) -----------------------
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NBK; ++nb) {
        w[mb][nb][0] = -w[mb][nb][0];
        w[mb][nb][1] = -w[mb][nb][1];
      }
    const int fg = pk_f(g);
    if (ESTORE && p == P::NP - 1) {
      // last panel: row blocks in groups of ES, each group's C2 rows stored
      // right after their last DMMA (the stores drain under the next groups'
      // DMMAs instead of after the loop); every accumulator sees the same
      // (nb, s) order as below, so the results are bitwise the same
#pragma unroll
      for (int r0 = 0; r0 < RB; r0 += ES) {
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb)
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const double* pc = Vq + g * P::GW + ((cb + 8 * nb + 2 * t + s) ^ fg);
#pragma unroll
            for (int rb = r0; rb < r0 + ES && rb < RB; ++rb) {
              if (rb < rb0) continue;
              if (RL && rb >= rbe) continue;
              const double bf = pc[8 * rb * P::GW];
#pragma unroll
              for (int mb = 0; mb < MB; ++mb) dmma(acc[mb][rb][0], acc[mb][rb][1], w[mb][nb][s], bf);
            }
          }
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          double* dst = C2 + 2 * t + (size_t)(wc0 + 8 * mb + g) * NB;
#pragma unroll
          for (int rb = r0; rb < r0 + ES && rb < RB; ++rb)
            if (!RL || rb < rbe)
              *reinterpret_cast<double2*>(dst + 8 * rb) = make_double2(acc[mb][rb][0], acc[mb][rb][1]);
        }
      }
    } else
#pragma unroll
    for (int nb = 0; nb < NBK; ++nb)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double* pc = Vq + g * P::GW + ((cb + 8 * nb + 2 * t + s) ^ fg);
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          if (rb < rb0) continue;
          if (TT && 8 * rb >= c0 + IB) continue;
          if (RL && rb >= rbe) continue;
          const double bf = pc[8 * rb * P::GW];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) dmma(acc[mb][rb][0], acc[mb][rb][1], w[mb][nb][s], bf);
        }
      }
    if (RG::NS < P::NG && (p % P::PPG == P::PPG - 1 || p == P::NP - 1)) {
      // group q done by this warp: release its stage; thread 0 refills it
      // with group q + NS once every active warp has released it.  The proxy
      // fence makes every lane's shared loads of the stage complete before the
      // release: the refill is an async-proxy (TMA) write, which neither the
      // arrive nor __syncwarp orders after generic loads still in flight
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (threadIdx.x == 0 && q + RG::NS < P::NG) {
        mbar_wait(&empty[st], (q / RG::NS) & 1);
        ring_issue<NB, IB, S>(gpk, spk, full, q + RG::NS);
      }
    }
  }

  // ---- registers -> C2 ----------------------------------------------------------
  if (ESTORE) return;  // stored during the last panel's step C
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    double* dst = C2 + 2 * t + (size_t)(wc0 + 8 * mb + g) * NB;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
      if (!RL || rb < rbe) *reinterpret_cast<double2*>(dst + 8 * rb) = make_double2(acc[mb][rb][0], acc[mb][rb][1]);
  }
}

// ---- batched kernels -----------------------------------------------------------
constexpr int kWarpsB = 8;  // warps per CTA of the batched v2 kernels (same geometry as the DAG kernel)

__host__ __device__ constexpr int v2_mb(int NB) { return (NB == 96 || NB == 128) ? 2 : 1; }
// batched kernel: wide panels keep one 8-column block per warp (registers)
__host__ __device__ constexpr int v2_mb(int NB, int IB) { return IB > 32 ? 1 : v2_mb(NB); }

// ring stages of the batched kernel: the whole packed tile when it fits
// (NB <= 128), else as many column groups as fit in ~200 KB (refilled by TMA
// as the panels advance, as in the DAG kernel)
template <int NB, int IB>
constexpr int v2_stages() {
  using P = Pk<NB, IB>;
  constexpr size_t stage = (size_t)(P::GDBL + P::PPG * P::TP) * sizeof(double);
  constexpr int s = (int)((200 * 1024) / stage);
  // wide panels whose group + T_p exceed 100 KB keep ONE stage (refilled when
  // every warp has released it: the TMA of the next group is then exposed)
  constexpr int lo = (IB > 32 && 2 * stage > 220 * 1024) ? 1 : 2;
  return s >= P::NG ? P::NG : (s < lo ? lo : s);
}

template <int NB, int IB>
constexpr size_t v2_smem_bytes() { return Ring<NB, IB, v2_stages<NB, IB>()>::bytes; }

// warps of a CTA (W warps of 8*MB columns from col0) that own columns < NB
template <int NB, int MB, int W>
__device__ __forceinline__ int active_warps(int col0, int cend = NB) {
  const int a = (cend - col0 + 8 * MB - 1) / (8 * MB);
  return a < 0 ? 0 : (a > W ? W : a);
}

// grid (slabs, batch): task b, columns [blockIdx.x * 64*MB, ...)
template <int NB, int IB, bool LARFB>
__global__ void __launch_bounds__(kWarpsB * 32, 1)
update_v2_kernel(const double* const* Pkp, double* const* C1p, double* const* C2p) {
  constexpr int MB = v2_mb(NB, IB);
  constexpr int S = v2_stages<NB, IB>();  // whole tile resident for NB <= 128
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int b = blockIdx.y;
  const int col0 = blockIdx.x * kWarpsB * 8 * MB;
  if (threadIdx.x == 0) ring_start<NB, IB, S>(Pkp[b], smem, full, empty, active_warps<NB, MB, kWarpsB>(col0));
  __syncthreads();
  update_v2_body<NB, IB, MB, LARFB, kWarpsB, S>(Pkp[b], smem, full, empty, LARFB ? nullptr : C1p[b], C2p[b],
                                                col0);
}

// grid (batch): standard V (NB x NB, GEQRT form if LARFB: unit lower
// trapezoid implied) and T (IB x NB) -> packed tile (the layout transform the
// panel kernels apply when they write the packed copy themselves)
template <int NB, int IB, bool LARFB>
__global__ void __launch_bounds__(256)
pack_kernel(const double* const* Vp, const double* const* Tp, double* const* Pkp) {
  const double* V = Vp[blockIdx.x];
  const double* T = Tp[blockIdx.x];
  double* pk = Pkp[blockIdx.x];
  for (int p = 0; p < NB / IB; ++p) {
    const int c0 = p * IB;
    pack_panel<NB, IB, 256>(
        pk, p,
        [&](int r, int i) {
          const int col = c0 + i;
          if (LARFB) return r > col ? V[r + (size_t)col * NB] : (r == col ? 1.0 : 0.0);
          return V[r + (size_t)col * NB];
        },
        [&](int l, int i) { return T[l + (size_t)(c0 + i) * IB]; });
  }
}

template <int NB, int IB, bool LARFB>
int launch_update_v2_t(int batch, const double* const* Pk_, double* const* C1, double* const* C2,
                       cudaStream_t s) {
  auto kern = update_v2_kernel<NB, IB, LARFB>;
  const size_t bytes = v2_smem_bytes<NB, IB>();
  static_assert(v2_smem_bytes<NB, IB>() <= 227 * 1024, "packed tile exceeds shared memory");
  TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  constexpr int cols = kWarpsB * 8 * v2_mb(NB, IB);
  dim3 grid((NB + cols - 1) / cols, batch);
  kern<<<grid, kWarpsB * 32, bytes, s>>>(Pk_, C1, C2);
  TQ_LAUNCH_CHECK();
  return 0;
}

template <int NB>
int launch_update_v2(bool larfb, int IB, int batch, const double* const* Pk_, double* const* C1,
                     double* const* C2, cudaStream_t s) {
  if (batch <= 0) return 0;
#define TQ_V2(ib)                                                                              \
  case ib:                                                                                     \
    return larfb ? launch_update_v2_t<NB, ib, true>(batch, Pk_, C1, C2, s)                     \
                 : launch_update_v2_t<NB, ib, false>(batch, Pk_, C1, C2, s);
#define TQ_V2W(ib)                                                                             \
  case ib:                                                                                     \
    if constexpr (pk_fits<NB, ib>())                                                           \
      return larfb ? launch_update_v2_t<NB, ib, true>(batch, Pk_, C1, C2, s)                   \
                   : launch_update_v2_t<NB, ib, false>(batch, Pk_, C1, C2, s);                 \
    break;
  switch (IB) {
    TQ_V2(8) TQ_V2(16) TQ_V2(32)
    TQ_V2W(24) TQ_V2W(40) TQ_V2W(48) TQ_V2W(56) TQ_V2W(64)
    default:
      break;
  }
  set_error("update_v2: unsupported IB");
  return TILEQR_ERR_CUDA;
#undef TQ_V2
#undef TQ_V2W
}

template <int NB>
int launch_pack(bool larfb, int IB, int batch, const double* const* V, const double* const* T,
                double* const* Pk_, cudaStream_t s) {
  if (batch <= 0) return 0;
#define TQ_PK(ib)                                                                             \
  case ib:                                                                                    \
    if (larfb) pack_kernel<NB, ib, true><<<batch, 256, 0, s>>>(V, T, Pk_);                    \
    else pack_kernel<NB, ib, false><<<batch, 256, 0, s>>>(V, T, Pk_);                         \
    break;
#define TQ_PKW(ib)                                                                            \
  case ib:                                                                                    \
    if constexpr (pk_fits<NB, ib>()) {                                                        \
      if (larfb) pack_kernel<NB, ib, true><<<batch, 256, 0, s>>>(V, T, Pk_);                  \
      else pack_kernel<NB, ib, false><<<batch, 256, 0, s>>>(V, T, Pk_);                       \
      break;                                                                                  \
    }                                                                                         \
    set_error("pack: unsupported IB");                                                        \
    return TILEQR_ERR_CUDA;
  switch (IB) {
    TQ_PK(8) TQ_PK(16) TQ_PK(32)
    TQ_PKW(24) TQ_PKW(40) TQ_PKW(48) TQ_PKW(56) TQ_PKW(64)
    default:
      set_error("pack: unsupported IB");
      return TILEQR_ERR_CUDA;
  }
#undef TQ_PK
#undef TQ_PKW
  TQ_LAUNCH_CHECK();
  return 0;
}

}  // namespace v2
}  // namespace tileqr
