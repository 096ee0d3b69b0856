// update_dmma.cuh -- DMMA (FP64 tensor core) trailing-update kernel of the
// tile QR: SSRFB (TSMQR) and LARFB (ORMQR).
//
// For every inner panel p of IB reflectors (ascending for Q^T, descending
// for Q):
//   step A  W^T  = C1[p rows]^T + C2^T V_p          (SSRFB; LARFB: C^T V_p)
//   step B  W'^T = W^T op(T_p)^T,  C1[p rows] -= W'
//   step C  C2^T -= W'^T V_p^T                       (LARFB: C^T -= W'^T V_p^T)
// A CTA of 4 warps owns a column slab of one task; each warp keeps 8*MB
// columns of C2 for ALL NB rows in registers as the transposed accumulator
// C2^T for the whole kernel (C2 read and written exactly once).  Step A
// feeds those accumulator registers straight back as DMMA A-fragments: the k
// index of each m8n8k4 step is permuted to rows {2t+j} of an 8-row block so
// that fragment == accumulator register j (no shuffles).
// Per panel, V_p (in chunks of KW <= 32 columns), T_p and the IB rows of C1
// are staged by cp.async into double buffers while the previous panel
// computes; V_p uses an XOR-swizzled row-major layout that is bank-conflict
// free both for the staging writes (4 rows x 8 columns per warp) and for the
// two fragment patterns.  Geometry (NB, MB, KW) is compile-time, so every
// shared address is an LDS/STS with a constant offset.
#pragma once

#include "dmma.cuh"
#include "internal.h"

namespace tileqr {
namespace upd {

constexpr int kWarps = 4;  // warps per CTA of the batched kernels (the DAG kernel uses 8)
constexpr int kThreads = kWarps * 32;

// Row-major V chunk, ld = LDV (a multiple of 16, no padding): element (r, i)
// lives at r*LDV + (i ^ usw(r)) with usw(r) = 4*((r>>1)&3) ^ 8*(r&1).  Every
// access pattern below touches 16 distinct 8-byte bank pairs per half warp:
// staging writes (4 rows x 8 columns), step A (row 8rb+2t+j, column 8nb+g)
// and step C (row 8rb+g, column k4+t).
__host__ __device__ constexpr int usw(int r) { return (((r >> 1) & 3) << 2) ^ ((r & 1) << 3); }

template <int KW>
struct Geo {
  static constexpr int LDV = (KW <= 16 ? 16 : 32);
  static constexpr int LDT = (KW <= 16 ? 16 : 32) + 4;  // == 4 mod 16
  static constexpr int LDC = (KW <= 16 ? 16 : 32) + 4;  // C1 rows per column, == 4 mod 16
};

// smem doubles of one stage buffer set and of the per-warp W^T
template <int NB, int MB, int KW, bool LARFB, bool MULTI, int W = kWarps>
struct Layout {
  static constexpr int CHUNK = NB * Geo<KW>::LDV;
  static constexpr int TBUF = MULTI ? 0 : KW * Geo<KW>::LDT;
  static constexpr int CBUF = LARFB ? 0 : W * 8 * MB * Geo<KW>::LDC;
  static constexpr int STAGE = CHUNK + TBUF + CBUF;
};

// MULTI: IBp > 32, processed as nch chunks of KW = 32 columns (last chunk
// zero-padded); V_p is staged twice per panel (for step A and for step C) and
// T_p is read from global memory.
// Body of one CTA (W warps): columns [col0, col0 + W*8*MB) of one task.
template <int NB, int MB, int KW, bool TRANS, bool LARFB, bool MULTI, int W>
__device__ __forceinline__ void update_body(int IB, int IBp, int ncols, const double* __restrict__ V,
                                            const double* __restrict__ T, double* __restrict__ C1,
                                            double* __restrict__ C2, int twobuf, int col0,
                                            double* __restrict__ smem) {
  constexpr int kThreads = W * 32;
  using L = Layout<NB, MB, KW, LARFB, MULTI, W>;
  constexpr int RB = NB / 8;
  constexpr int LDV = Geo<KW>::LDV;
  constexpr int LDT = Geo<KW>::LDT;
  constexpr int LDC = Geo<KW>::LDC;
  constexpr int NBK = KW / 8;  // 8-column blocks per chunk
  const int LDW = MULTI ? IBp + 4 : KW + 4;  // == 4 mod 16 (IBp % 32 == 0 when MULTI)
  // [stage 0: V | T | C1][stage 1: V | T | C1][W^T per warp] (one stage if !twobuf)
  const int nbuf = twobuf ? 2 : 1;
  double* const Wsw = smem + nbuf * L::STAGE + (threadIdx.x >> 5) * 8 * MB * LDW;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a = lane & 3, g = lane >> 2;
  constexpr int CPC = W * 8 * MB;  // columns per CTA
  const int wcl0 = warp * 8 * MB;  // first column of this warp (CTA-local)

  const int np = NB / IB;
  const int nch = MULTI ? (IBp + KW - 1) / KW : 1;
  const int nitems = MULTI ? np * 2 * nch : np;

  // item -> (panel p, chunk q, phase: 0 = A only, 1 = C only, 2 = both)
  auto item_p = [&](int idx) { int p = MULTI ? idx / (2 * nch) : idx; return TRANS ? p : np - 1 - p; };
  auto item_q = [&](int idx) { if (!MULTI) return 0; int r = idx % (2 * nch); return r < nch ? r : r - nch; };
  auto item_phase = [&](int idx) { if (!MULTI) return 2; return (idx % (2 * nch)) < nch ? 0 : 1; };

  // Per-thread constants of the fast V staging (SSRFB, one chunk per panel):
  // warp instruction `it` moves rows 4*((W*it % RG) + warp) + [0,4) of columns
  // 8*(W*it / RG) + [0,8); the swizzle of those rows is a per-thread constant.
  constexpr int RG = NB / 4;  // 4-row groups (NB % 32 == 0, so RG % W == 0)
  static_assert(RG % W == 0, "row groups per warp instruction");
  const int st_r = 4 * warp + (lane & 3), st_c = lane >> 2;
  const int st_sw = usw(st_r);
  auto stage = [&](int idx, int slot) {
    const int p = item_p(idx), q = item_q(idx), phase = item_phase(idx);
    const int c0 = p * IB;
    double* vb = smem + slot * L::STAGE;
    if (!LARFB && !MULTI) {
      const double* src = V + (size_t)c0 * NB + st_r + (size_t)st_c * NB;
      double* dst = vb + st_r * LDV + (st_c ^ st_sw);
#pragma unroll
      for (int it = 0; it < NB * KW / kThreads; ++it) {
        const int rg0 = (W * it) % RG, cg = (W * it) / RG;  // compile-time
        const int ii = 8 * cg + st_c;
        double* d = dst + 4 * rg0 * LDV + (((8 * cg) ^ (st_c ^ st_sw)) - (st_c ^ st_sw));
        if (ii < IB) cp_async8(d, src + 4 * rg0 + (size_t)(8 * cg) * NB);
        else *d = 0.0;
      }
    } else {
    // V chunk: each warp instruction moves a 4-row x 8-column block
#pragma unroll 4
    for (int e = threadIdx.x; e < NB * KW; e += kThreads) {
      const int blk = e >> 5, l = e & 31;
      const int r = 4 * (blk % RG) + (l & 3), ii = 8 * (blk / RG) + (l >> 2);
      const int i = q * KW + ii;  // column within the panel
      double* dst = vb + r * LDV + (ii ^ usw(r));
      if (i >= IB) {
        *dst = 0.0;
      } else if (LARFB) {
        const int col = c0 + i;
        if (r > col) cp_async8(dst, V + r + (size_t)col * NB);
        else *dst = (r == col) ? 1.0 : 0.0;
      } else {
        cp_async8(dst, V + r + (size_t)(c0 + i) * NB);
      }
    }
    }
    if (!MULTI) {
      double* tb = vb + L::CHUNK;
      for (int e = threadIdx.x; e < KW * KW; e += kThreads) {
        const int i = e / KW, l = e - i * KW;
        double* dst = tb + l + i * LDT;
        if (l < IB && i < IB) cp_async8(dst, T + (size_t)c0 * IB + l + (size_t)i * IB);
        else *dst = 0.0;
      }
    }
    if (!LARFB && phase != 1) {  // C1 rows c0 + q*KW + [0, KW) of the CTA's columns
      double* cb = vb + L::CHUNK + L::TBUF;
      for (int e = threadIdx.x; e < CPC * KW; e += kThreads) {
        const int cl = e / KW, ii = e - cl * KW;
        const int i = q * KW + ii, col = col0 + cl;
        double* dst = cb + cl * LDC + ii;
        if (i < IB && col < ncols) cp_async8(dst, C1 + c0 + i + (size_t)col * NB);
        else *dst = 0.0;
      }
    }
    cp_async_commit();
  };

  stage(0, 0);  // first panel's operands in flight while C2 is loaded

  // ---- C2 slab -> registers: acc[mb][rb][j] = C2(8rb+2a+j, col0+wcl0+8mb+g) ----
  double acc[MB][RB][2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int col = col0 + wcl0 + 8 * mb + g;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      double2 v = make_double2(0.0, 0.0);
      if (col < ncols) v = *reinterpret_cast<const double2*>(C2 + 8 * rb + 2 * a + (size_t)col * NB);
      acc[mb][rb][0] = v.x;
      acc[mb][rb][1] = v.y;
    }
  }

  for (int idx = 0; idx < nitems; ++idx) {
    const int slot = twobuf ? (idx & 1) : 0;
    const int p = item_p(idx), q = item_q(idx), phase = item_phase(idx);
    const int c0 = p * IB;
    const double* Vs = smem + slot * L::STAGE;
    const double* Ts = Vs + L::CHUNK;
    const double* C1s = Vs + L::CHUNK + L::TBUF;
    if (twobuf && idx + 1 < nitems) {
      stage(idx + 1, slot ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- step A --------------------------------------------------------------
    if (phase != 1) {
      // two partial sums per output block (k rows 2t and 2t+1 of each 8-row
      // block) so that every DMMA chain has 2*MB*NBK independent links
      double wacc[MB][NBK][2], wacc2[MB][NBK][2];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            wacc[mb][nb][j] = LARFB ? 0.0 : C1s[(wcl0 + 8 * mb + g) * LDC + 8 * nb + 2 * a + j];
            wacc2[mb][nb][j] = 0.0;
          }
      const int rb0 = LARFB ? (c0 >> 3) : 0;  // V_p is zero above row c0
      // B-fragment (row 8rb+2a+j, column 8nb+g): its swizzle usw = 4a ^ 8j for
      // every rb, so one per-thread base per (j, nb) and a compile-time offset per rb.
      const double* pa[2][NBK];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) pa[j][nb] = Vs + (2 * a + j) * LDV + ((8 * nb + g) ^ usw(2 * a + j));
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        if (rb < rb0) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int nb = 0; nb < NBK; ++nb) {
            const double bf = pa[j][nb][8 * rb * LDV];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
              if (j == 0) dmma(wacc[mb][nb][0], wacc[mb][nb][1], acc[mb][rb][0], bf);
              else dmma(wacc2[mb][nb][0], wacc2[mb][nb][1], acc[mb][rb][1], bf);
            }
          }
        }
      }
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) {
          wacc[mb][nb][0] += wacc2[mb][nb][0];
          wacc[mb][nb][1] += wacc2[mb][nb][1];
        }
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) {
          double* w = Wsw + (8 * mb + g) * LDW + q * KW + 8 * nb + 2 * a;
          w[0] = wacc[mb][nb][0];
          w[1] = wacc[mb][nb][1];
        }
    }

    // ---- step B (after the last A chunk of the panel) ------------------------
    const bool lastA = !MULTI || (phase == 0 && q == nch - 1);
    if (lastA && !MULTI) {
      __syncwarp();
      // all output blocks at once (independent DMMA chains), then write back.
      // TRANS: W'(:,i) = sum_{l<=i} W(:,l) T(l,i);  !TRANS: sum_{l>=i} W(:,l) T(i,l)
      double o[NBK][MB][2];
#pragma unroll
      for (int nb = 0; nb < NBK; ++nb)
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) o[nb][mb][0] = o[nb][mb][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < KW; k4 += 4) {
        double af[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) af[mb] = Wsw[(8 * mb + g) * LDW + k4 + a];
#pragma unroll
        for (int nb = 0; nb < NBK; ++nb) {
          if (TRANS ? (k4 >= 8 * nb + 8) : (k4 < 8 * nb)) continue;
          const double bf = TRANS ? Ts[(k4 + a) + (8 * nb + g) * LDT] : Ts[(8 * nb + g) + (k4 + a) * LDT];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) dmma(o[nb][mb][0], o[nb][mb][1], af[mb], bf);
        }
      }
      __syncwarp();
#pragma unroll
      for (int nb = 0; nb < NBK; ++nb)
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const int cl = wcl0 + 8 * mb + g, col = col0 + cl;
          double* w = Wsw + (8 * mb + g) * LDW + 8 * nb + 2 * a;
          w[0] = -o[nb][mb][0];
          w[1] = -o[nb][mb][1];
          if (!LARFB && col < ncols) {
            const int i = 8 * nb + 2 * a;
            if (i < IB) C1[c0 + i + (size_t)col * NB] = C1s[cl * LDC + i] - o[nb][mb][0];
            if (i + 1 < IB) C1[c0 + i + 1 + (size_t)col * NB] = C1s[cl * LDC + i + 1] - o[nb][mb][1];
          }
        }
      __syncwarp();
    }
    if (lastA && MULTI) {
      __syncwarp();
      const int nbt = IBp / 8;
      const double* Tgl = T + (size_t)c0 * IB;
      for (int s = 0; s < nbt; ++s) {
        const int nb = TRANS ? nbt - 1 - s : s;  // in place: descending for TRANS
        double o[MB][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) o[mb][0] = o[mb][1] = 0.0;
        const int kb = TRANS ? 0 : 8 * nb, ke = TRANS ? 8 * nb + 8 : IBp;
        for (int k4 = kb; k4 < ke; k4 += 4) {
          const int l = k4 + a, i = 8 * nb + g;
          double bf = 0.0;
          if (l < IB && i < IB) bf = TRANS ? __ldg(Tgl + l + (size_t)i * IB) : __ldg(Tgl + i + (size_t)l * IB);
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) dmma(o[mb][0], o[mb][1], Wsw[(8 * mb + g) * LDW + k4 + a], bf);
        }
        __syncwarp();
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const int col = col0 + wcl0 + 8 * mb + g;
          double* w = Wsw + (8 * mb + g) * LDW + 8 * nb + 2 * a;
          w[0] = -o[mb][0];
          w[1] = -o[mb][1];
          if (!LARFB && col < ncols) {
            const int i = 8 * nb + 2 * a;
            if (i < IB) C1[c0 + i + (size_t)col * NB] -= o[mb][0];
            if (i + 1 < IB) C1[c0 + i + 1 + (size_t)col * NB] -= o[mb][1];
          }
        }
        __syncwarp();
      }
    }

    // ---- step C --------------------------------------------------------------
    if (phase != 0) {
      const int rb0 = LARFB ? (c0 >> 3) : 0;
      // B-fragment (row 8rb+g, column k4+a): swizzle usw(g) for every rb
      const double* pc = Vs + g * LDV;
      const int sw = usw(g);
#pragma unroll
      for (int k4 = 0; k4 < KW; k4 += 4) {
        double af[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) af[mb] = Wsw[(8 * mb + g) * LDW + q * KW + k4 + a];
        const double* pck = pc + ((k4 + a) ^ sw);
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          if (rb < rb0) continue;
          const double bf = pck[8 * rb * LDV];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) dmma(acc[mb][rb][0], acc[mb][rb][1], af[mb], bf);
        }
      }
    }
    __syncthreads();  // stage buffer `slot` is restaged by the next iteration
    if (!twobuf && idx + 1 < nitems) stage(idx + 1, 0);
  }

  // ---- registers -> C2 -------------------------------------------------------
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int col = col0 + wcl0 + 8 * mb + g;
    if (col < ncols) {
#pragma unroll
      for (int rb = 0; rb < RB; ++rb)
        *reinterpret_cast<double2*>(C2 + 8 * rb + 2 * a + (size_t)col * NB) =
            make_double2(acc[mb][rb][0], acc[mb][rb][1]);
    }
  }
}

template <int NB, int MB, int KW, bool TRANS, bool LARFB, bool MULTI>
__global__ void __launch_bounds__(kThreads)
update_kernel(int IB, int IBp, int ncols, const double* const* Vp, const double* const* Tp,
              double* const* C1p, double* const* C2p, int twobuf) {
  extern __shared__ __align__(16) double smem[];
  const int b = blockIdx.y;
  update_body<NB, MB, KW, TRANS, LARFB, MULTI, kWarps>(IB, IBp, ncols, Vp[b], Tp[b], LARFB ? nullptr : C1p[b],
                                                       C2p[b], twobuf, blockIdx.x * kWarps * 8 * MB, smem);
}

inline int round_up8(int x) { return (x + 7) / 8 * 8; }

template <int NB, int MB, int KW, bool TRANS, bool LARFB, bool MULTI>
int launch_update_t(int IB, int batch, const double* const* V, const double* const* T,
                    double* const* C1, double* const* C2, int ncols, cudaStream_t s) {
  using L = Layout<NB, MB, KW, LARFB, MULTI>;
  const int IBp = MULTI ? (round_up8(IB) + 31) / 32 * 32 : KW;
  const int LDW = MULTI ? IBp + 4 : KW + 4;
  const size_t wd = (size_t)kWarps * 8 * MB * LDW;
  // double-buffer the staged operands when they fit in 227 KB, else single-buffer
  int twobuf = 1;
  size_t bytes = (2 * (size_t)L::STAGE + wd) * sizeof(double);
  if (bytes > 227 * 1024) {
    twobuf = 0;
    bytes = ((size_t)L::STAGE + wd) * sizeof(double);
  }
  auto kern = update_kernel<NB, MB, KW, TRANS, LARFB, MULTI>;
  TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  const int cols_per_cta = kWarps * 8 * MB;
  dim3 grid((ncols + cols_per_cta - 1) / cols_per_cta, batch);
  kern<<<grid, kThreads, bytes, s>>>(IB, IBp, ncols, V, T, C1, C2, twobuf);
  TQ_LAUNCH_CHECK();
  return 0;
}

template <int NB, bool TRANS, bool LARFB>
int launch_update_nb(int IB, int batch, const double* const* V, const double* const* T,
                     double* const* C1, double* const* C2, int ncols, cudaStream_t s) {
  constexpr int MB = NB <= 128 ? 2 : 1;
  const int ibp = round_up8(IB);
  switch (ibp) {
    case 8: return launch_update_t<NB, MB, 8, TRANS, LARFB, false>(IB, batch, V, T, C1, C2, ncols, s);
    case 16: return launch_update_t<NB, MB, 16, TRANS, LARFB, false>(IB, batch, V, T, C1, C2, ncols, s);
    case 24: return launch_update_t<NB, MB, 24, TRANS, LARFB, false>(IB, batch, V, T, C1, C2, ncols, s);
    case 32: return launch_update_t<NB, MB, 32, TRANS, LARFB, false>(IB, batch, V, T, C1, C2, ncols, s);
    default: return launch_update_t<NB, MB, 32, TRANS, LARFB, true>(IB, batch, V, T, C1, C2, ncols, s);
  }
}

// Entry of one NB (defined in update_nb<NB>.cu): LARFB selects the GEQRT form.
template <int NB>
int launch_update_dmma(bool trans, bool larfb, int IB, int batch, const double* const* V,
                       const double* const* T, double* const* C1, double* const* C2, int ncols,
                       cudaStream_t s) {
  if (larfb)
    return trans ? launch_update_nb<NB, true, true>(IB, batch, V, T, C1, C2, ncols, s)
                 : launch_update_nb<NB, false, true>(IB, batch, V, T, C1, C2, ncols, s);
  return trans ? launch_update_nb<NB, true, false>(IB, batch, V, T, C1, C2, ncols, s)
               : launch_update_nb<NB, false, false>(IB, batch, V, T, C1, C2, ncols, s);
}

}  // namespace upd
}  // namespace tileqr
