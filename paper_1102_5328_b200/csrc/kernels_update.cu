// kernels_update.cu -- the trailing-update kernels of the tile QR:
//   SSRFB (TSMQR): [C1; C2] <- op(Q) [C1; C2], Q from a TSQRT (PAPER.md:184-185,
//                  519-528: "calls to DSSRFB are predominant");
//   LARFB (ORMQR): C <- op(Q) C, Q from a GEQRT.
// For every inner panel p of IB reflectors (ascending for Q^T, descending for
// Q):
//   W = C1[p rows] + V2_p^T C2;  W = op(T_p) W;  C1[p rows] -= W;  C2 -= V2_p W
// (LARFB: W = V_p^T C, C -= V_p W with V_p unit lower trapezoidal).
//
// Two implementations:
//  * dmma_update_kernel -- the product path for NB % 32 == 0, 32 <= NB <= 256.
//    FP64 tensor-core MMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; sm_100a has
//    no tcgen05 kind::f64).  A CTA of 4 warps owns a column slab
//    of one tile pair; each warp keeps its 8*MB columns of C2 for ALL NB rows
//    in registers as the transposed accumulator C2^T for the whole kernel, so
//    C2 is read from and written to HBM exactly once.  Step A uses those
//    accumulator registers directly as DMMA A-fragments (the k index of each
//    m8n8k4 step is permuted to match the accumulator layout: chunk j of an
//    8-row block takes rows 2*(lane%4)+j), step B multiplies by T_p through a
//    per-warp shared-memory W^T, and step C accumulates -W'^T V2_p^T into the
//    registers.  V2_p is staged per panel (in 32-column chunks) by cp.async
//    into a double-buffered, XOR-swizzled row-major smem layout that keeps
//    both fragment access patterns bank-conflict free.
//  * simt_update_kernel -- any NB <= 512 (plain FMA, global operands); used
//    for NB not a multiple of 32 or > 256.
#include <stdio.h>
#include <stdlib.h>

#include "internal.h"

namespace tileqr {
namespace {

// ============================================================================
// Generic SIMT path
// ============================================================================
constexpr int kSimtThreads = 256;

__host__ __device__ inline int simt_cw(int IB) {
  int cw = 4096 / IB;
  if (cw > 64) cw = 64;
  if (cw < 1) cw = 1;
  return cw;
}

// LARFB = true: V is a GEQRT tile (unit lower), C1 unused, C2 = C.
template <bool LARFB>
__global__ void __launch_bounds__(kSimtThreads)
simt_update_kernel(bool trans, int NB, int IB, int ncols, const double* const* Vp,
                   const double* const* Tp, double* const* C1p, double* const* C2p) {
  extern __shared__ double W[];  // IB x CW
  const int CW = simt_cw(IB);
  const int b = blockIdx.y;
  const int cb = blockIdx.x * CW;
  const int nc = min(CW, ncols - cb);
  if (nc <= 0) return;
  const double* V = Vp[b];
  const double* T = Tp[b];
  double* C1 = LARFB ? nullptr : C1p[b];
  double* C2 = C2p[b];
  const int tid = threadIdx.x;
  const int np = NB / IB;
  for (int pp = 0; pp < np; ++pp) {
    const int p = trans ? pp : np - 1 - pp;
    const int c0 = p * IB;
    for (int idx = tid; idx < IB * nc; idx += kSimtThreads) {
      const int cc = idx / IB, i = idx - cc * IB;
      const int c = cb + cc;
      double acc;
      if (LARFB) {
        acc = C2[c0 + i + (size_t)c * NB];
        for (int r = c0 + i + 1; r < NB; ++r)
          acc = fma(V[r + (size_t)(c0 + i) * NB], C2[r + (size_t)c * NB], acc);
      } else {
        acc = C1[c0 + i + (size_t)c * NB];
        for (int r = 0; r < NB; ++r)
          acc = fma(V[r + (size_t)(c0 + i) * NB], C2[r + (size_t)c * NB], acc);
      }
      W[i + cc * IB] = acc;
    }
    __syncthreads();
    const double* Tb = T + (size_t)c0 * IB;  // T_p(l, i) = Tb[l + i*IB]
    for (int cc = tid; cc < nc; cc += kSimtThreads) {
      double* w = W + cc * IB;
      if (trans) {
        for (int i = IB - 1; i >= 0; --i) {
          double acc = 0.0;
          for (int l = 0; l <= i; ++l) acc = fma(Tb[l + i * IB], w[l], acc);
          w[i] = acc;
        }
      } else {
        for (int i = 0; i < IB; ++i) {
          double acc = 0.0;
          for (int l = i; l < IB; ++l) acc = fma(Tb[i + l * IB], w[l], acc);
          w[i] = acc;
        }
      }
    }
    __syncthreads();
    if (LARFB) {
      const int rows = NB - c0;
      for (int idx = tid; idx < rows * nc; idx += kSimtThreads) {
        const int cc = idx / rows, r = c0 + (idx - cc * rows);
        const int d = r - c0, iend = min(d, IB);
        double acc = 0.0;
        for (int i = 0; i < iend; ++i) acc = fma(V[r + (size_t)(c0 + i) * NB], W[i + cc * IB], acc);
        if (d < IB) acc += W[d + cc * IB];
        C2[r + (size_t)(cb + cc) * NB] -= acc;
      }
    } else {
      for (int idx = tid; idx < IB * nc; idx += kSimtThreads) {
        const int cc = idx / IB, i = idx - cc * IB;
        C1[c0 + i + (size_t)(cb + cc) * NB] -= W[i + cc * IB];
      }
      for (int idx = tid; idx < NB * nc; idx += kSimtThreads) {
        const int cc = idx / NB, r = idx - cc * NB;
        double acc = 0.0;
        for (int i = 0; i < IB; ++i) acc = fma(V[r + (size_t)(c0 + i) * NB], W[i + cc * IB], acc);
        C2[r + (size_t)(cb + cc) * NB] -= acc;
      }
    }
    __syncthreads();
  }
}

template <bool LARFB>
int launch_simt(bool trans, int NB, int IB, int batch, const double* const* V,
                const double* const* T, double* const* C1, double* const* C2, int ncols,
                cudaStream_t s) {
  const int CW = simt_cw(IB);
  dim3 grid((ncols + CW - 1) / CW, batch);
  const size_t bytes = (size_t)IB * CW * sizeof(double);
  auto kern = simt_update_kernel<LARFB>;
  if (bytes > 48 * 1024)
    TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  kern<<<grid, kSimtThreads, bytes, s>>>(trans, NB, IB, ncols, V, T, C1, C2);
  TQ_LAUNCH_CHECK();
  return 0;
}

// ============================================================================
// DMMA path
// ============================================================================
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int KC = 32;  // V2 columns per staged chunk

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct DmmaCfg {
  int IBp;    // IB rounded up to 8
  int nch;    // chunks per panel
  int LDV;    // staged chunk: row-major, ld LDV (== 8 mod 16), swizzled
  int LDW;    // per-warp W^T: [col][i], ld LDW (== 4 mod 16)
  int LDT;    // staged T_p: column-major, ld LDT (== 4 mod 16)
  bool stageT;
  int nbuf;   // chunk buffers (2 = double buffering)
  size_t smem_bytes;
};

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

inline DmmaCfg dmma_cfg(int NB, int IB, int MB) {
  DmmaCfg c;
  c.IBp = round_up(IB, 8);
  const int kc = c.IBp < KC ? c.IBp : KC;
  c.nch = (c.IBp + kc - 1) / kc;
  c.LDV = round_up(kc, 16) + 8;
  c.LDW = round_up(c.IBp, 16) + 4;
  c.LDT = round_up(c.IBp, 16) + 4;
  c.stageT = c.IBp <= 32;
  const size_t chunk = (size_t)NB * c.LDV;
  const size_t wbytes = (size_t)kWarps * 8 * MB * c.LDW;
  const size_t tbytes = c.stageT ? 2 * (size_t)c.IBp * c.LDT : 0;
  c.nbuf = 2;
  c.smem_bytes = (2 * chunk + wbytes + tbytes) * sizeof(double);
  if (c.smem_bytes > 220 * 1024) {
    c.nbuf = 1;
    c.smem_bytes = (chunk + wbytes + tbytes) * sizeof(double);
  }
  return c;
}

// swizzled offset of element (row r, column i) of a staged chunk
__device__ __forceinline__ int vsw(int r, int i, int LDV) { return r * LDV + (i ^ (((r >> 1) & 3) << 2)); }

// Stage chunk columns [q0, q0+kw) of panel p (V2 columns c0+q0..) into buf.
// LARFB: V_p(row, i) = 1 if row == c0+i, V(row, c0+i) if row > c0+i, else 0.
template <int NB, bool LARFB>
__device__ __forceinline__ void stage_chunk(double* buf, const double* __restrict__ V, int IB,
                                            int c0, int q0, int kw, int LDV) {
  for (int idx = threadIdx.x; idx < NB * kw; idx += kThreads) {
    const int ii = idx / NB, r = idx - ii * NB;  // r fastest: coalesced global reads
    const int i = q0 + ii;                       // column within the panel
    double* dst = buf + vsw(r, ii, LDV);
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

__device__ __forceinline__ void stage_t(double* Ts, const double* __restrict__ Tg, int IB, int IBp,
                                        int c0, int LDT) {
  for (int idx = threadIdx.x; idx < IBp * IBp; idx += kThreads) {
    const int i = idx / IBp, l = idx - i * IBp;
    double* dst = Ts + l + i * LDT;
    if (l < IB && i < IB) cp_async8(dst, Tg + (size_t)c0 * IB + l + (size_t)i * IB);
    else *dst = 0.0;
  }
}

// One work item of the chunk schedule: panel index p, chunk q, phase (0 = A, 1 = C, 2 = both).
struct Item {
  int p, q, phase;
};

__device__ __forceinline__ Item item_of(int idx, int nch, int np, bool trans) {
  Item it;
  if (nch == 1) {
    it.p = idx;
    it.q = 0;
    it.phase = 2;
  } else {
    it.p = idx / (2 * nch);
    const int r = idx - it.p * 2 * nch;
    it.phase = r < nch ? 0 : 1;
    it.q = r < nch ? r : r - nch;
  }
  if (!trans) it.p = np - 1 - it.p;
  return it;
}

template <int NB, int MB, bool TRANS, bool LARFB>
__global__ void __launch_bounds__(kThreads)
dmma_update_kernel(int IB, int ncols, const double* const* Vp, const double* const* Tp,
                   double* const* C1p, double* const* C2p, DmmaCfg cfg) {
  constexpr int RB = NB / 8;  // 8-row blocks of C2
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a = lane & 3, x = lane >> 2;  // fragment coordinates
  const int b = blockIdx.y;
  const int wcol0 = (blockIdx.x * kWarps + warp) * 8 * MB;  // first column of this warp
  const double* __restrict__ V = Vp[b];
  const double* __restrict__ T = Tp[b];
  double* __restrict__ C1 = LARFB ? nullptr : C1p[b];
  double* __restrict__ C2 = C2p[b];

  const int IBp = cfg.IBp, LDV = cfg.LDV, LDW = cfg.LDW, LDT = cfg.LDT, nch = cfg.nch;
  const int kc = IBp < KC ? IBp : KC;
  double* bufs[2];
  bufs[0] = smem;
  bufs[1] = smem + (cfg.nbuf == 2 ? (size_t)NB * LDV : 0);
  double* Ws = smem + (size_t)cfg.nbuf * NB * LDV + (size_t)warp * 8 * MB * LDW;
  double* Tsb = smem + (size_t)cfg.nbuf * NB * LDV + (size_t)kWarps * 8 * MB * LDW;

  // ---- C2 slab -> registers (transposed accumulator) ------------------------
  // acc[mb][rb][j] = C2(row 8rb + 2a + j, col wcol0 + 8mb + x)
  double acc[MB][RB][2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int col = wcol0 + 8 * mb + x;
    const bool ok = col < ncols;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      double2 v = make_double2(0.0, 0.0);
      if (ok) v = *reinterpret_cast<const double2*>(C2 + 8 * rb + 2 * a + (size_t)col * NB);
      acc[mb][rb][0] = v.x;
      acc[mb][rb][1] = v.y;
    }
  }

  const int np = NB / IB;
  const int nitems = nch == 1 ? np : np * 2 * nch;
  auto stage_item = [&](int idx, int slot) {
    const Item it = item_of(idx, nch, np, TRANS);
    const int c0 = it.p * IB;
    const int q0 = it.q * kc;
    const int kw = min(kc, IBp - q0);
    stage_chunk<NB, LARFB>(bufs[slot], V, IB, c0, q0, kw, LDV);
    if (cfg.stageT && it.phase != 1) stage_t(Tsb + (size_t)(slot & 1) * IBp * LDT, T, IB, IBp, c0, LDT);
    cp_async_commit();
  };

  stage_item(0, 0);
  for (int idx = 0; idx < nitems; ++idx) {
    const int slot = cfg.nbuf == 2 ? (idx & 1) : 0;
    const Item it = item_of(idx, nch, np, TRANS);
    const int c0 = it.p * IB;
    const int q0 = it.q * kc;
    const int kw = min(kc, IBp - q0);
    const double* Vs = bufs[slot];
    if (cfg.nbuf == 2 && idx + 1 < nitems) {
      stage_item(idx + 1, slot ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- step A: W^T(col, i) = C1(c0+i, col) + sum_r C2^T(col, r) V_p(r, i) ----
    if (it.phase != 1) {
      for (int ib0 = 0; ib0 < kw; ib0 += 32) {  // kw <= 32: one pass
        double wacc[MB][4][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const int col = wcol0 + 8 * mb + x;
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int i = q0 + ib0 + 8 * nb + 2 * a + j;  // panel column
              double v = 0.0;
              if (!LARFB && col < ncols && i < IB && 8 * nb < kw) v = C1[c0 + i + (size_t)col * NB];
              wacc[mb][nb][j] = v;
            }
        }
        const int nnb = kw / 8;
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          if (LARFB && 8 * rb + 7 < c0) continue;  // V_p is zero above row c0
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r = 8 * rb + 2 * a + j;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
              if (nb < nnb) {
                const double bf = Vs[vsw(r, ib0 + 8 * nb + x, LDV)];
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) dmma(wacc[mb][nb][0], wacc[mb][nb][1], acc[mb][rb][j], bf);
              }
            }
          }
        }
        // W^T -> per-warp smem: Ws[col_local * LDW + i]
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
            if (nb < nnb) {
              const int i = q0 + ib0 + 8 * nb + 2 * a;
              Ws[(8 * mb + x) * LDW + i] = wacc[mb][nb][0];
              Ws[(8 * mb + x) * LDW + i + 1] = wacc[mb][nb][1];
            }
      }
    }

    // ---- step B (after the last A chunk): W^T <- W^T op(T_p)^T; C1 -= W ----
    const bool lastA = (it.phase == 2) || (it.phase == 0 && it.q == nch - 1);
    if (lastA) {
      __syncwarp();
      const double* Tsrc;
      int ldt;
      if (cfg.stageT) {
        Tsrc = Tsb + (size_t)(slot & 1) * IBp * LDT;
        ldt = LDT;
      } else {
        Tsrc = T + (size_t)c0 * IB;
        ldt = IB;
      }
      const int nbt = IBp / 8;
      for (int s = 0; s < nbt; ++s) {
        // TRANS: W'(:,i) = sum_{l<=i} W(:,l) T(l,i): descending blocks (in place)
        // !TRANS: W'(:,i) = sum_{l>=i} W(:,l) T(i,l): ascending blocks
        const int nb = TRANS ? nbt - 1 - s : s;
        double o[MB][2];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) o[mb][0] = o[mb][1] = 0.0;
        const int kbeg = TRANS ? 0 : 8 * nb;
        const int kend = TRANS ? 8 * nb + 8 : IBp;
        for (int k4 = kbeg; k4 < kend; k4 += 4) {
          const int l = k4 + a, i = 8 * nb + x;
          double bf;
          if (cfg.stageT) {
            bf = TRANS ? Tsrc[l + i * ldt] : Tsrc[i + l * ldt];
          } else {
            bf = (l < IB && i < IB) ? (TRANS ? Tsrc[l + (size_t)i * ldt] : Tsrc[i + (size_t)l * ldt]) : 0.0;
          }
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) {
            const double af = Ws[(8 * mb + x) * LDW + k4 + a];
            dmma(o[mb][0], o[mb][1], af, bf);
          }
        }
        __syncwarp();
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const int col = wcol0 + 8 * mb + x;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i = 8 * nb + 2 * a + j;
            Ws[(8 * mb + x) * LDW + i] = -o[mb][j];  // -W' feeds step C
            if (!LARFB && col < ncols && i < IB) C1[c0 + i + (size_t)col * NB] -= o[mb][j];
          }
        }
        __syncwarp();
      }
    }

    // ---- step C: C2^T(col, r) += (-W'^T)(col, i) V_p(r, i) over this chunk ----
    if (it.phase != 0) {
      for (int k4 = 0; k4 < kw; k4 += 4) {
        double af[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) af[mb] = Ws[(8 * mb + x) * LDW + q0 + k4 + a];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          if (LARFB && 8 * rb + 7 < c0) continue;
          const double bf = Vs[vsw(8 * rb + x, k4 + a, LDV)];
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) dmma(acc[mb][rb][0], acc[mb][rb][1], af[mb], bf);
        }
      }
    }
    __syncthreads();  // chunk buffer `slot` may be restaged next
    if (cfg.nbuf == 1 && idx + 1 < nitems) stage_item(idx + 1, 0);
  }

  // ---- registers -> C2 ------------------------------------------------------
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int col = wcol0 + 8 * mb + x;
    if (col < ncols) {
#pragma unroll
      for (int rb = 0; rb < RB; ++rb)
        *reinterpret_cast<double2*>(C2 + 8 * rb + 2 * a + (size_t)col * NB) =
            make_double2(acc[mb][rb][0], acc[mb][rb][1]);
    }
  }
}

template <int NB, int MB, bool TRANS, bool LARFB>
int launch_dmma_t(int IB, int batch, const double* const* V, const double* const* T,
                  double* const* C1, double* const* C2, int ncols, cudaStream_t s) {
  const DmmaCfg cfg = dmma_cfg(NB, IB, MB);
  auto kern = dmma_update_kernel<NB, MB, TRANS, LARFB>;
  TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)cfg.smem_bytes));
  const int cols_per_cta = kWarps * 8 * MB;
  dim3 grid((ncols + cols_per_cta - 1) / cols_per_cta, batch);
  kern<<<grid, kThreads, cfg.smem_bytes, s>>>(IB, ncols, V, T, C1, C2, cfg);
  TQ_LAUNCH_CHECK();
  return 0;
}

template <int NB, bool LARFB>
int launch_dmma_nb(bool trans, int IB, int batch, const double* const* V, const double* const* T,
                   double* const* C1, double* const* C2, int ncols, cudaStream_t s) {
  constexpr int MB = NB <= 128 ? 2 : 1;
  return trans ? launch_dmma_t<NB, MB, true, LARFB>(IB, batch, V, T, C1, C2, ncols, s)
               : launch_dmma_t<NB, MB, false, LARFB>(IB, batch, V, T, C1, C2, ncols, s);
}

template <bool LARFB>
int launch_dmma(bool trans, int NB, int IB, int batch, const double* const* V,
                const double* const* T, double* const* C1, double* const* C2, int ncols,
                cudaStream_t s) {
  switch (NB) {
    case 32: return launch_dmma_nb<32, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 64: return launch_dmma_nb<64, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 96: return launch_dmma_nb<96, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 128: return launch_dmma_nb<128, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 160: return launch_dmma_nb<160, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 192: return launch_dmma_nb<192, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 224: return launch_dmma_nb<224, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    case 256: return launch_dmma_nb<256, LARFB>(trans, IB, batch, V, T, C1, C2, ncols, s);
    default: return -1;
  }
}

bool dmma_supported(int NB) { return NB % 32 == 0 && NB >= 32 && NB <= 256; }

bool force_simt() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TILEQR_FORCE_SIMT");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace

const char* ssrfb_impl_name(int NB, int IB) {
  (void)IB;
  return (dmma_supported(NB) && !force_simt()) ? "dmma" : "simt";
}

int launch_larfb(bool trans, int NB, int IB, int batch, const double* const* V,
                 const double* const* T, double* const* C, int ncols, cudaStream_t s) {
  if (batch <= 0) return 0;
  if (dmma_supported(NB) && !force_simt())
    return launch_dmma<true>(trans, NB, IB, batch, V, T, nullptr, C, ncols, s);
  return launch_simt<true>(trans, NB, IB, batch, V, T, nullptr, C, ncols, s);
}

int launch_ssrfb(bool trans, int NB, int IB, int batch, const double* const* V2,
                 const double* const* T, double* const* C1, double* const* C2, int ncols,
                 cudaStream_t s) {
  if (batch <= 0) return 0;
  if (dmma_supported(NB) && !force_simt())
    return launch_dmma<false>(trans, NB, IB, batch, V2, T, C1, C2, ncols, s);
  return launch_simt<false>(trans, NB, IB, batch, V2, T, C1, C2, ncols, s);
}

}  // namespace tileqr
