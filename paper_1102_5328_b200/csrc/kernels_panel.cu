// kernels_panel.cu -- the panel kernels of the tile QR: GEQRT (QR of a
// diagonal tile) and TSQRT (QR of a triangle stacked on a square tile)
// ("DGEQRT and DTSQRT serial kernels").
//
// One CTA per task (a batch of independent tasks per launch).  For each inner
// panel p of IB columns (inner blocking):
//   1. the panel columns are staged in shared memory (ld = NB+1, odd, so the
//      column-strided accesses of one warp hit distinct banks) when they fit,
//      else they are addressed in global memory (same code, generic pointer);
//   2. columns are factored one by one.  ONE reduction pass per column
//      computes sigma = ||x2||^2 and every dot d_c = x2 . P(:,c) of the
//      remaining panel columns at once (warp-shuffle trees), because
//      v2 = x2 / (alpha - beta) makes w_c = R(j,c) + d_c/(alpha - beta);
//      the rank-1 panel update follows: 2 CTA barriers per column;
//   3. T_p (IB x IB upper triangular, R3) is built by the
//      forward-columnwise recurrence T[0:i,i] = -tau_i T[0:i,0:i] (V^T v_i);
//   4. Q_p^T is applied to the trailing columns of the tile (pair).
// Reflector rule: DESIGN.md reading R1 (LAPACK larfg sign convention, no
// rescaling loop).  TSQRT never writes the strict lower part of R, which the
// LARFB of the same DAG level reads.
#include <math.h>
#include <stdlib.h>

#include "internal.h"

namespace tileqr {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr size_t kSmemBudget = 200 * 1024;

struct Mat {
  double* p;
  int ld;
  __device__ __forceinline__ double& operator()(int r, int c) const {
    return p[r + (size_t)c * ld];
  }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct PanelSmem {
  double* tau;  // [IB]
  double* dots; // [IB]
  double* rj;   // [IB]  row j of R restricted to the panel columns
  double* G;    // [IB*IB] Gram matrix of the panel's reflectors (IB <= 64) or [IB] column
  double* W;    // [IB*CW] trailing-update workspace
  double* P;    // [(NB+1)*IB] staged panel, or nullptr
};

__host__ __device__ inline int trailing_cw(int IB) {
  int cw = 4096 / IB;
  if (cw > 64) cw = 64;
  if (cw < 1) cw = 1;
  return cw;
}

inline size_t panel_smem_bytes(int NB, int IB, bool stage) {
  size_t g = (IB <= 64) ? (size_t)IB * IB : (size_t)IB;
  size_t n = 3 * (size_t)IB + g + (size_t)IB * trailing_cw(IB);
  if (stage) n += (size_t)(NB + 1) * IB;
  return n * sizeof(double);
}

inline bool panel_stage(int NB, int IB) { return panel_smem_bytes(NB, IB, true) <= kSmemBudget; }

// TS = true: TSQRT on (R = Rp[b] upper triangle, B = Bp[b]); false: GEQRT on A = Rp[b].
template <bool TS>
__global__ void __launch_bounds__(kThreads)
panel_kernel(int NB, int IB, double* const* Rp, double* const* Bp, double* const* Tp, int stage) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* const Rg = Rp[blockIdx.x];
  double* const Bg = TS ? Bp[blockIdx.x] : Rg;
  double* const Tg = Tp[blockIdx.x];
  const Mat R{Rg, NB};
  const Mat B{Bg, NB};
  const Mat Tm{Tg, IB};
  const int CW = trailing_cw(IB);
  const bool fullG = IB <= 64;

  PanelSmem s;
  s.tau = smem;
  s.dots = s.tau + IB;
  s.rj = s.dots + IB;
  s.G = s.rj + IB;
  s.W = s.G + (fullG ? IB * IB : IB);
  s.P = stage ? s.W + IB * CW : nullptr;

  for (int c0 = 0; c0 < NB; c0 += IB) {
    // P(r, c) = panel column c0 + c, rows 0..NB-1 (B for TSQRT, A for GEQRT)
    Mat P = stage ? Mat{s.P, NB + 1} : Mat{&B(0, c0), NB};
    if (stage) {
      for (int idx = tid; idx < NB * IB; idx += kThreads) {
        const int c = idx / NB, r = idx - c * NB;
        P(r, c) = B(r, c0 + c);
      }
      __syncthreads();
    }

    // ---- 2. factor the panel column by column --------------------------
    for (int jj = 0; jj < IB; ++jj) {
      const int j = c0 + jj;
      // rows of the reflector tail: TSQRT all NB rows of B; GEQRT rows j+1..NB-1
      const int r0 = TS ? 0 : j + 1;
      // (a) one pass: dots[c] = sum_r P(r,jj) P(r,c), c = jj..IB-1; rj[c] = R(j, c0+c)
      for (int c = jj + warp; c < IB; c += kWarps) {
        double acc = 0.0;
        for (int r = r0 + lane; r < NB; r += 32) acc = fma(P(r, jj), P(r, c), acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          s.dots[c] = acc;
          s.rj[c] = TS ? R(j, c0 + c) : P(j, c);
        }
      }
      __syncthreads();
      // (b) reflector (every thread computes the same scalars)
      const double sigma = s.dots[jj];
      const double alpha = s.rj[jj];
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (sigma != 0.0) {
        const double nrm = sqrt(alpha * alpha + sigma);
        beta = (alpha >= 0.0) ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      // (c) rank-1 update of the remaining panel columns, then scale v2
      if (sigma != 0.0) {
        for (int r = r0 + tid; r < NB; r += kThreads) {
          const double v = P(r, jj) * scal;
          for (int c = jj + 1; c < IB; ++c) {
            const double w = fma(scal, s.dots[c], s.rj[c]);
            P(r, c) = fma(-tau * v, w, P(r, c));
          }
          P(r, jj) = v;
        }
      }
      // row j of R (TSQRT: global R; GEQRT: row j of the staged panel)
      if (tid > jj && tid < IB && sigma != 0.0) {
        const double w = fma(scal, s.dots[tid], s.rj[tid]);
        if (TS) R(j, c0 + tid) = s.rj[tid] - tau * w;
        else P(j, tid) = s.rj[tid] - tau * w;
      }
      if (tid == 0) {
        if (TS) R(j, j) = beta;
        else P(j, jj) = beta;
        s.tau[jj] = tau;
      }
      __syncthreads();
    }

    // ---- write the factored panel back ------------------------------------
    if (stage) {
      for (int idx = tid; idx < NB * IB; idx += kThreads) {
        const int c = idx / NB, r = idx - c * NB;
        B(r, c0 + c) = P(r, c);
      }
    }

    // ---- 3. T_p -----------------------------------------------------------
    // z_l(i) = v_l . v_i.  TSQRT: the top parts e_j are distinct unit
    // vectors, so z = V2_l . V2_i.  GEQRT: v_l(c0+i) * 1 + sum_{r > c0+i}.
    auto vdot = [&](int l, int i) -> double {  // warp-cooperative, l < i
      double acc = 0.0;
      const int rs = TS ? 0 : c0 + i + 1;
      for (int r = rs + lane; r < NB; r += 32) acc = fma(P(r, l), P(r, i), acc);
      acc = warp_sum(acc);
      if (!TS) acc += P(c0 + i, l);
      return acc;
    };
    Mat Tp{&Tm(0, c0), IB};
    if (fullG) {
      for (int idx = warp; idx < IB * IB; idx += kWarps) {
        const int i = idx / IB, l = idx - i * IB;
        if (l < i) {
          const double z = vdot(l, i);
          if (lane == 0) s.G[l + i * IB] = z;
        }
      }
      __syncthreads();
      // thread r owns row r of T_p: T(r,i) = -tau_i sum_{l=r}^{i-1} T(r,l) z_l(i)
      if (tid < IB) {
        const int r = tid;
        for (int i = 0; i < IB; ++i) {
          double v;
          if (i < r) {
            v = 0.0;
          } else if (i == r) {
            v = s.tau[i];
          } else {
            double acc = 0.0;
            for (int l = r; l < i; ++l) acc = fma(Tp(r, l), s.G[l + i * IB], acc);
            v = -s.tau[i] * acc;
          }
          Tp(r, i) = v;
        }
      }
    } else {
      for (int i = 0; i < IB; ++i) {
        for (int l = warp; l < i; l += kWarps) {
          const double z = vdot(l, i);
          if (lane == 0) s.G[l] = z;
        }
        __syncthreads();
        for (int r = tid; r < IB; r += kThreads) {
          double v;
          if (i < r) {
            v = 0.0;
          } else if (i == r) {
            v = s.tau[i];
          } else {
            double acc = 0.0;
            for (int l = r; l < i; ++l) acc = fma(Tp(r, l), s.G[l], acc);
            v = -s.tau[i] * acc;
          }
          Tp(r, i) = v;
        }
        __syncthreads();
      }
    }
    __syncthreads();

    // ---- 4. trailing columns c >= c0+IB: W = V^T C; W = T^T W; C -= V W ---
    for (int cb = c0 + IB; cb < NB; cb += CW) {
      const int nc = min(CW, NB - cb);
      for (int idx = tid; idx < IB * nc; idx += kThreads) {
        const int cc = idx / IB, i = idx - cc * IB;
        const int c = cb + cc;
        double acc;
        if (TS) {
          acc = R(c0 + i, c);
          for (int r = 0; r < NB; ++r) acc = fma(P(r, i), B(r, c), acc);
        } else {
          acc = B(c0 + i, c);
          for (int r = c0 + i + 1; r < NB; ++r) acc = fma(P(r, i), B(r, c), acc);
        }
        s.W[i + cc * IB] = acc;
      }
      __syncthreads();
      for (int cc = tid; cc < nc; cc += kThreads) {  // W(:,cc) <- T_p^T W(:,cc), bottom-up
        double* w = s.W + cc * IB;
        for (int i = IB - 1; i >= 0; --i) {
          double acc = 0.0;
          for (int l = 0; l <= i; ++l) acc = fma(Tp(l, i), w[l], acc);
          w[i] = acc;
        }
      }
      __syncthreads();
      if (TS) {
        for (int idx = tid; idx < IB * nc; idx += kThreads) {
          const int cc = idx / IB, i = idx - cc * IB;
          R(c0 + i, cb + cc) -= s.W[i + cc * IB];
        }
        for (int idx = tid; idx < NB * nc; idx += kThreads) {
          const int cc = idx / NB, r = idx - cc * NB;
          double acc = 0.0;
          for (int i = 0; i < IB; ++i) acc = fma(P(r, i), s.W[i + cc * IB], acc);
          B(r, cb + cc) -= acc;
        }
      } else {
        for (int idx = tid; idx < (NB - c0) * nc; idx += kThreads) {
          const int cc = idx / (NB - c0), r = c0 + (idx - cc * (NB - c0));
          // V(r,i) = P(r,i) for r > c0+i, 1 for r == c0+i, 0 above
          const int d = r - c0, iend = min(d, IB);
          double acc = 0.0;
          for (int i = 0; i < iend; ++i) acc = fma(P(r, i), s.W[i + cc * IB], acc);
          if (d < IB) acc += s.W[d + cc * IB];
          B(r, cb + cc) -= acc;
        }
      }
      __syncthreads();
    }
  }
}

template <bool TS>
int launch_panel(int NB, int IB, int batch, double* const* R, double* const* B, double* const* T,
                 cudaStream_t s) {
  if (batch <= 0) return 0;
  const bool stage = panel_stage(NB, IB);
  const size_t bytes = panel_smem_bytes(NB, IB, stage);
  auto kern = panel_kernel<TS>;
  if (bytes > 48 * 1024) {
    TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  kern<<<batch, kThreads, bytes, s>>>(NB, IB, R, B, T, stage ? 1 : 0);
  TQ_LAUNCH_CHECK();
  return 0;
}

// ---- wide panels (IB > 32, IB % 8 == 0, IB <= 64): T assembly ------------------
// The GEQRT / TSQRT of a wide inner panel runs the register-resident panel
// kernel with inner blocking IBi (the largest of 32, 24, 16, 8 dividing IB):
// its reflectors, R and V are those of the IB-blocked algorithm (applying the
// IBi-blocks of a panel in order IS applying the panel's reflectors in order;
// DESIGN.md R22), only the compact-WY factor differs.  This kernel assembles
// T_p of every IB-panel from the reflectors (the
// oracle's recurrence): T[i,i] = tau_i (the diagonal of the IBi-blocked T),
// T[0:i, i] = -tau_i T[0:i, 0:i] z with z_l = v_l^T v_i -- GEQRT: v_i = e_i +
// strictly-lower column of the tile; TSQRT: v_i = [e_i; V2(:, i)].
constexpr int kWideIB = 64;

template <bool TS>
__global__ void __launch_bounds__(kThreads)
wide_t_kernel(int NB, int IB, int IBi, const double* const* Vp, const double* const* Tin, double* const* Tout) {
  extern __shared__ double sm[];
  double* Vs = sm;                        // NB x IB, column-major (ld NB + 1)
  double* G = Vs + (size_t)(NB + 1) * IB; // IB x IB
  double* Tp = G + (size_t)IB * IB;       // IB x IB
  const double* V = Vp[blockIdx.x];
  const double* Ti = Tin[blockIdx.x];
  double* To = Tout[blockIdx.x];
  const int tid = threadIdx.x, ldv = NB + 1;
  for (int c0 = 0; c0 < NB; c0 += IB) {
    for (int e = tid; e < NB * IB; e += kThreads) {
      const int c = e / NB, r = e - c * NB, j = c0 + c;
      double v = __ldcg(V + r + (size_t)j * NB);
      if (!TS) v = r == j ? 1.0 : (r > j ? v : 0.0);   // GEQRT: unit lower trapezoid
      Vs[r + c * ldv] = v;
    }
    __syncthreads();
    for (int e = tid; e < IB * IB; e += kThreads) {   // z: G[l, i] = v_l^T v_i, l < i
      const int i = e / IB, l = e - i * IB;
      double acc = 0.0;
      if (l < i)  // TSQRT: the top parts e_l, e_i are orthogonal, only V2 contributes
        for (int r = 0; r < NB; ++r) acc = fma(Vs[r + l * ldv], Vs[r + i * ldv], acc);
      G[l + i * IB] = acc;
      Tp[l + i * IB] = 0.0;
    }
    __syncthreads();
    for (int i = 0; i < IB; ++i) {                    // forward recurrence, one column at a time
      const int j = c0 + i;
      const double tau = __ldcg(Ti + (j % IBi) + (size_t)j * IBi);
      if (tid < i) {
        double acc = 0.0;
        for (int l = tid; l < i; ++l) acc = fma(Tp[tid + l * IB], G[l + i * IB], acc);
        Tp[tid + i * IB] = -tau * acc;
      } else if (tid == i) {
        Tp[i + i * IB] = tau;
      }
      __syncthreads();
    }
    for (int e = tid; e < IB * IB; e += kThreads) {
      const int i = e / IB, l = e - i * IB;
      To[l + (size_t)(c0 + i) * IB] = l <= i ? Tp[l + i * IB] : 0.0;
    }
    __syncthreads();
  }
}

}  // namespace

bool panel_fast_supported(int NB, int IB);
int launch_geqrt_fast(int NB, int IB, int batch, double* const* A, double* const* T, cudaStream_t s,
                      double* const* Pk);
int launch_tsqrt_fast(int NB, int IB, int batch, double* const* R, double* const* A2,
                      double* const* T, cudaStream_t s, double* const* Pk);

static int wide_inner(int IB) {
  for (int c : {32, 24, 16, 8})
    if (IB % c == 0) return c;
  return 0;
}

bool panel_wide_supported(int NB, int IB) {
  return NB % 32 == 0 && NB >= 32 && NB <= 256 && IB > 32 && IB <= kWideIB && IB % 8 == 0 && NB % IB == 0 &&
         panel_fast_supported(NB, wide_inner(IB));
}

// wide panel: the fast kernel at IBi into scratch T, T assembled at IB, then the packed copy
template <bool TS>
static int launch_wide(int NB, int IB, int batch, double* const* R, double* const* B, double* const* T,
                       cudaStream_t s, double* const* Pk) {
  const int IBi = wide_inner(IB);
  double* ti = nullptr;
  double** tp = nullptr;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&ti), (size_t)batch * IBi * NB * sizeof(double), s)) return rc_;
  if (int rc_ = stream_alloc(reinterpret_cast<void**>(&tp), (size_t)batch * sizeof(double*), s)) return rc_;
  int rc = launch_fill_ptrs(tp, ti, (size_t)IBi * NB, batch, s);
  if (!rc) rc = TS ? launch_tsqrt_fast(NB, IBi, batch, R, B, tp, s, nullptr) : launch_geqrt_fast(NB, IBi, batch, R, tp, s, nullptr);
  if (!rc) {
    const size_t bytes = ((size_t)(NB + 1) * IB + 2 * (size_t)IB * IB) * sizeof(double);
    auto kern = wide_t_kernel<TS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
      kern<<<batch, kThreads, bytes, s>>>(NB, IB, IBi, TS ? B : R, tp, T);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "wide_t_kernel", __FILE__, __LINE__);
  }
  if (!rc && Pk) rc = launch_pack(!TS, NB, IB, batch, TS ? B : R, T, Pk, s);
  cudaFreeAsync(ti, s);
  cudaFreeAsync(tp, s);
  return rc;
}

// T at inner blocking IBe (<= 64, a multiple of IB) from the reflectors V and
// tau = the diagonal of T at IB (R23): the batched update entry
// points run an IB that the packed update does not take at IBe.
int launch_t_assemble(bool ts, int NB, int IBe, int IB, int batch, const double* const* V,
                      const double* const* Tin, double* const* Tout, cudaStream_t s) {
  if (batch <= 0) return 0;
  if (IBe > kWideIB || IBe % IB || NB % IBe) {
    set_error("launch_t_assemble: IBe must be a multiple of IB dividing NB, at most 64");
    return TILEQR_ERR_CUDA;
  }
  const size_t bytes = ((size_t)(NB + 1) * IBe + 2 * (size_t)IBe * IBe) * sizeof(double);
  auto kern = ts ? wide_t_kernel<true> : wide_t_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) {
    kern<<<batch, kThreads, bytes, s>>>(NB, IBe, IB, V, Tin, Tout);
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? 0 : cuda_fail(e, "wide_t_kernel", __FILE__, __LINE__);
}

static bool generic_panel_forced() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TILEQR_GENERIC_PANEL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int launch_geqrt(int NB, int IB, int batch, double* const* A, double* const* T, cudaStream_t s,
                 double* const* Pk) {
  if (batch <= 0) return 0;
  if (panel_fast_supported(NB, IB) && !generic_panel_forced())
    return launch_geqrt_fast(NB, IB, batch, A, T, s, Pk);
  if (panel_wide_supported(NB, IB) && !generic_panel_forced())
    return launch_wide<false>(NB, IB, batch, A, nullptr, T, s, Pk);
  int rc = launch_panel<false>(NB, IB, batch, A, nullptr, T, s);
  if (!rc && Pk) rc = launch_pack(true, NB, IB, batch, A, T, Pk, s);
  return rc;
}

int launch_tsqrt(int NB, int IB, int batch, double* const* R, double* const* A2, double* const* T,
                 cudaStream_t s, double* const* Pk) {
  if (batch <= 0) return 0;
  if (panel_fast_supported(NB, IB) && !generic_panel_forced())
    return launch_tsqrt_fast(NB, IB, batch, R, A2, T, s, Pk);
  if (panel_wide_supported(NB, IB) && !generic_panel_forced())
    return launch_wide<true>(NB, IB, batch, R, A2, T, s, Pk);
  int rc = launch_panel<true>(NB, IB, batch, R, A2, T, s);
  if (!rc && Pk) rc = launch_pack(false, NB, IB, batch, A2, T, Pk, s);
  return rc;
}

}  // namespace tileqr
