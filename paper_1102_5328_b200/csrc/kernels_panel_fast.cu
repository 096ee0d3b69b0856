// kernels_panel_fast.cu -- batched launch of the low-latency GEQRT / TSQRT
// (body in panel_fast.cuh): one CTA of 8 warps per task.
#include <stdlib.h>

#include "dag_item.h"
#include "panel_fast.cuh"

namespace tileqr {

#ifndef TILEQR_PANEL_PROF
__device__ unsigned long long g_panel_prof[16];  // phase cycles; filled only with -DTILEQR_PANEL_PROF
#endif

namespace {
using pf::FastSmem;

template <bool TS, int NB, int kWarps, int IB, bool TT = false>
__global__ void __launch_bounds__(kWarps * 32, 1)
panel_fast_kernel(double* const* Rp, double* const* Bp, double* const* Tp, double* const* Pk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pf::panel_fast_body<TS, NB, kWarps, IB, TT>(Rp[blockIdx.x], TS ? Bp[blockIdx.x] : nullptr, Tp[blockIdx.x],
                                              smem_raw, Pk ? Pk[blockIdx.x] : nullptr);
}

template <bool TS, int NB, int NW, int IB, bool TT = false>
int launch_fast_i(int batch, double* const* R, double* const* B, double* const* T, cudaStream_t s,
                  double* const* Pk) {
  auto kern = panel_fast_kernel<TS, NB, NW, IB, TT>;
  const size_t bytes = sizeof(FastSmem<NB, NW>);
  TQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  kern<<<batch, NW * 32, bytes, s>>>(R, B, T, Pk);
  TQ_LAUNCH_CHECK();
  return 0;
}

template <bool TS, int NB, int NW, bool TT = false>
int launch_fast_w(int IB, int batch, double* const* R, double* const* B, double* const* T,
                  cudaStream_t s, double* const* Pk) {
  switch (IB) {
    case 8: return launch_fast_i<TS, NB, NW, 8, TT>(batch, R, B, T, s, Pk);
    case 16: return launch_fast_i<TS, NB, NW, 16, TT>(batch, R, B, T, s, Pk);
    case 24:
      if constexpr (NB % 24 == 0) return launch_fast_i<TS, NB, NW, 24, TT>(batch, R, B, T, s, Pk);
      return -1;
    case 32: return launch_fast_i<TS, NB, NW, 32, TT>(batch, R, B, T, s, Pk);
    default: return -1;
  }
}

// Warps per panel CTA: the DAG kernel's geometry for this NB (dag_item.h),
// so the batched and the dataflow schedules compute bitwise the same
// reductions; TILEQR_PANEL_WARPS=4|8 overrides (diagnostics).
int panel_warps(int NB) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TILEQR_PANEL_WARPS");
    v = e ? atoi(e) : 0;
    if (v != 4 && v != 8) v = 0;
  }
  return v ? v : dag::dag_warps(NB);
}

template <bool TS, int NB, bool TT = false>
int launch_fast_t(int IB, int batch, double* const* R, double* const* B, double* const* T,
                  cudaStream_t s, double* const* Pk) {
  return panel_warps(NB) == 8 ? launch_fast_w<TS, NB, 8, TT>(IB, batch, R, B, T, s, Pk)
                              : launch_fast_w<TS, NB, 4, TT>(IB, batch, R, B, T, s, Pk);
}

template <bool TS, bool TT = false>
int launch_fast(int NB, int IB, int batch, double* const* R, double* const* B, double* const* T,
                cudaStream_t s, double* const* Pk) {
  switch (NB) {
    case 32: return launch_fast_t<TS, 32, TT>(IB, batch, R, B, T, s, Pk);
    case 64: return launch_fast_t<TS, 64, TT>(IB, batch, R, B, T, s, Pk);
    case 96: return launch_fast_t<TS, 96, TT>(IB, batch, R, B, T, s, Pk);
    case 128: return launch_fast_t<TS, 128, TT>(IB, batch, R, B, T, s, Pk);
    case 160: return launch_fast_t<TS, 160, TT>(IB, batch, R, B, T, s, Pk);
    case 192: return launch_fast_t<TS, 192, TT>(IB, batch, R, B, T, s, Pk);
    case 224: return launch_fast_t<TS, 224, TT>(IB, batch, R, B, T, s, Pk);
    case 256: return launch_fast_t<TS, 256, TT>(IB, batch, R, B, T, s, Pk);
    default: return -1;
  }
}

}  // namespace

int panel_prof_read(unsigned long long* out, int reset) {
  TQ_CUDA(cudaMemcpyFromSymbol(out, g_panel_prof, sizeof(unsigned long long) * 16));
  if (reset) {
    unsigned long long z[16] = {};
    TQ_CUDA(cudaMemcpyToSymbol(g_panel_prof, z, sizeof z));
  }
  return 0;
}

bool panel_fast_supported(int NB, int IB) {
  return NB % 32 == 0 && NB >= 32 && NB <= 256 && IB % 8 == 0 && IB <= 32;
}

int launch_geqrt_fast(int NB, int IB, int batch, double* const* A, double* const* T, cudaStream_t s,
                      double* const* Pk) {
  return launch_fast<false>(NB, IB, batch, A, nullptr, T, s, Pk);
}

int launch_tsqrt_fast(int NB, int IB, int batch, double* const* R, double* const* A2,
                      double* const* T, cudaStream_t s, double* const* Pk) {
  return launch_fast<true>(NB, IB, batch, R, A2, T, s, Pk);
}

// TTQRT (tree variant, f3): the TS body with B upper triangular
int launch_ttqrt_fast(int NB, int IB, int batch, double* const* R, double* const* A2,
                      double* const* T, cudaStream_t s, double* const* Pk) {
  return launch_fast<true, true>(NB, IB, batch, R, A2, T, s, Pk);
}

}  // namespace tileqr
