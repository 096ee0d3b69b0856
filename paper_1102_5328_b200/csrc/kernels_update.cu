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
//  * upd::update_kernel (update_dmma.cuh) -- the product path for NB % 32 == 0,
//    32 <= NB <= 256.
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
// DMMA path: update_dmma.cuh, instantiated per NB in update_nb<NB>.cu
// ============================================================================
}  // namespace
#define TQ_DECL_NB(nb)                                                                        \
  int launch_update_nb##nb(bool trans, bool larfb, int IB, int batch, const double* const* V, \
                           const double* const* T, double* const* C1, double* const* C2,      \
                           int ncols, cudaStream_t s);
TQ_DECL_NB(32) TQ_DECL_NB(64) TQ_DECL_NB(96) TQ_DECL_NB(128) TQ_DECL_NB(160) TQ_DECL_NB(192)
TQ_DECL_NB(224) TQ_DECL_NB(256)
namespace {

template <bool LARFB>
int launch_dmma(bool trans, int NB, int IB, int batch, const double* const* V,
                const double* const* T, double* const* C1, double* const* C2, int ncols,
                cudaStream_t s) {
  switch (NB) {
    case 32: return launch_update_nb32(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 64: return launch_update_nb64(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 96: return launch_update_nb96(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 128: return launch_update_nb128(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 160: return launch_update_nb160(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 192: return launch_update_nb192(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 224: return launch_update_nb224(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
    case 256: return launch_update_nb256(trans, LARFB, IB, batch, V, T, C1, C2, ncols, s);
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

// ---- packed-reflector (barrier-free) path: update_v2.cuh ----------------------
#define TQ_DECL_PK(nb)                                                                              \
  int launch_update_pk_nb##nb(bool larfb, int IB, int batch, const double* const* Pk, double* const* C1, \
                              double* const* C2, cudaStream_t s);                                   \
  int launch_pack_nb##nb(bool larfb, int IB, int batch, const double* const* V, const double* const* T, \
                         double* const* Pk, cudaStream_t s);
TQ_DECL_PK(32) TQ_DECL_PK(64) TQ_DECL_PK(96) TQ_DECL_PK(128) TQ_DECL_PK(160) TQ_DECL_PK(192) TQ_DECL_PK(224)
TQ_DECL_PK(256)
#undef TQ_DECL_PK

bool v2_supported(int NB, int IB) {
  if (force_simt()) return false;
  const char* e = getenv("TILEQR_NO_V2");
  if (e && e[0] == '1') return false;
  if (!(NB % 32 == 0 && NB >= 32 && NB <= 256 && IB % 8 == 0 && IB >= 8 && IB <= 64 && NB % IB == 0)) return false;
  if (IB <= 32) return true;
  // wide panels (update_v2.cuh pk_fits): one ring stage (a group + T_p) within 220 KB
  const size_t gw = (IB + 15) / 16 * 16;
  return ((size_t)NB * gw + (size_t)IB * 66) * sizeof(double) <= 220 * 1024;
}

size_t v2_pk_doubles(int NB, int IB) {
  if (IB % 8 || IB < 8 || IB > 64 || NB % IB) return 0;
  const int GW = IB <= 16 ? 16 : IB <= 32 ? 32 : (IB + 15) / 16 * 16, PW = IB == 8 ? 8 : GW, PPG = GW / PW;
  const int NP = NB / IB, NG = (NP + PPG - 1) / PPG, LDT2 = IB <= 16 ? 18 : IB <= 32 ? 34 : 66;
  return (size_t)NG * NB * GW + (size_t)NP * IB * LDT2;
}

int launch_update_pk(bool larfb, int NB, int IB, int batch, const double* const* Pk, double* const* C1,
                     double* const* C2, cudaStream_t s) {
  if (batch <= 0) return 0;
  switch (NB) {
    case 32: return launch_update_pk_nb32(larfb, IB, batch, Pk, C1, C2, s);
    case 64: return launch_update_pk_nb64(larfb, IB, batch, Pk, C1, C2, s);
    case 96: return launch_update_pk_nb96(larfb, IB, batch, Pk, C1, C2, s);
    case 128: return launch_update_pk_nb128(larfb, IB, batch, Pk, C1, C2, s);
    case 160: return launch_update_pk_nb160(larfb, IB, batch, Pk, C1, C2, s);
    case 192: return launch_update_pk_nb192(larfb, IB, batch, Pk, C1, C2, s);
    case 224: return launch_update_pk_nb224(larfb, IB, batch, Pk, C1, C2, s);
    case 256: return launch_update_pk_nb256(larfb, IB, batch, Pk, C1, C2, s);
    default: set_error("packed update: NB not in {32, 64, ..., 256}"); return TILEQR_ERR_CUDA;
  }
}

int launch_pack(bool larfb, int NB, int IB, int batch, const double* const* V, const double* const* T,
                double* const* Pk, cudaStream_t s) {
  if (batch <= 0) return 0;
  switch (NB) {
    case 32: return launch_pack_nb32(larfb, IB, batch, V, T, Pk, s);
    case 64: return launch_pack_nb64(larfb, IB, batch, V, T, Pk, s);
    case 96: return launch_pack_nb96(larfb, IB, batch, V, T, Pk, s);
    case 128: return launch_pack_nb128(larfb, IB, batch, V, T, Pk, s);
    case 160: return launch_pack_nb160(larfb, IB, batch, V, T, Pk, s);
    case 192: return launch_pack_nb192(larfb, IB, batch, V, T, Pk, s);
    case 224: return launch_pack_nb224(larfb, IB, batch, V, T, Pk, s);
    case 256: return launch_pack_nb256(larfb, IB, batch, V, T, Pk, s);
    default: set_error("pack: NB not in {32, 64, ..., 256}"); return TILEQR_ERR_CUDA;
  }
}

}  // namespace tileqr
