// kernels_layout.cu -- HBM-bound data movement of the tile QR (SURVEY §8(a)
// rows a1/a7): LAPACK column-major <-> padded tile layout, the non-finite
// flag, and the device copy of the synthetic input generator.
//
// Tile layout ("split the initial matrix ... into NT x NT
// smaller square pieces of order NB, called tiles"): tile (m,n) is a
// contiguous NB x NB column-major block at offset (m + n*MT)*NB*NB.  A column
// segment of NB rows is contiguous in BOTH layouts, so each warp moves whole
// 256-B runs: one thread per element pair, grid-stride, 16-B accesses on the
// tile side when NB is even.
#include <math.h>

#include <algorithm>

#include "internal.h"

namespace tileqr {
namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work) {
  int64_t blocks = (work + kThreads - 1) / kThreads;
  // 148 SMs x 8 resident 256-thread CTAs; grid-stride beyond that.
  const int64_t cap = 148 * 8 * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

// Padded value of element (i, j) of the (MT*NB) x (NT*NB) matrix
// (reading R5: rows >= M are 0; a padded column j >= N is e_j when
// M <= j < MT*NB, else 0).
__device__ __forceinline__ double padded_value(int64_t i, int64_t j, int64_t M, int64_t N,
                                               const double* __restrict__ A, int64_t lda,
                                               int* bad) {
  if (i < M && j < N) {
    double v = __ldg(A + i + j * lda);
    if (!isfinite(v)) *bad = 1;
    return v;
  }
  return (j >= N && i == j && j >= M) ? 1.0 : 0.0;
}

// One CTA per tile (m, n) (grid MT x NT): the tile's NB column segments of NB
// rows are contiguous runs in both layouts, so an interior tile is a plain
// strided-to-contiguous block copy.  VEC (NB, lda even, A 16-byte aligned):
// 16-byte loads and stores, 8 in flight per thread; 32-bit index arithmetic
// inside the tile (the earlier element-pair kernels spent their time in 64-bit
// divisions: 57 % / 46 % of HBM, profiles/r02_ncu_layout_n10000_nb128.json).
// Edge tiles (rows >= M or columns >= N inside) take the per-element path with
// the padding of DESIGN.md R5.
constexpr int kUnroll = 8;

template <bool VEC>
__global__ void __launch_bounds__(kThreads)
layout_to_tiles_kernel(int64_t M, int64_t N, const double* __restrict__ A, int64_t lda, int NB,
                       int64_t MT, double* __restrict__ tiles, int* d_info) {
  const int64_t m = blockIdx.x, n = blockIdx.y;
  const int64_t i0 = m * NB, j0 = n * NB;
  double* __restrict__ dst = tiles + (m + n * MT) * (int64_t)NB * NB;
  const int tid = threadIdx.x;
  int bad = 0;
  if (VEC && i0 + NB <= M && j0 + NB <= N) {
    const int HP = NB >> 1, tot = NB * HP;
    const double* __restrict__ src = A + i0 + j0 * lda;
    for (int e0 = tid; e0 < tot; e0 += kUnroll * kThreads) {
      double2 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * kThreads;
        if (e < tot) {
          const int jl = e / HP, il = 2 * (e - jl * HP);
          v[u] = __ldcs(reinterpret_cast<const double2*>(src + il + jl * lda));
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * kThreads;
        if (e < tot) {
          if (!isfinite(v[u].x) || !isfinite(v[u].y)) bad = 1;
          reinterpret_cast<double2*>(dst)[e] = v[u];  // element 2e = (il, jl): il + jl*NB = 2e
        }
      }
    }
  } else {
    const int tot = NB * NB;
    for (int e = tid; e < tot; e += kThreads) {
      const int jl = e / NB, il = e - jl * NB;
      const int64_t i = i0 + il, j = j0 + jl;
      double v;
      if (i < M && j < N) {
        v = __ldcs(A + i + j * lda);
        if (!isfinite(v)) bad = 1;
      } else {
        v = (j >= N && i == j && j >= M) ? 1.0 : 0.0;
      }
      dst[e] = v;
    }
  }
  if (bad && d_info) *d_info = 1;  // benign race: every writer stores 1
}

template <bool VEC>
__global__ void __launch_bounds__(kThreads)
tiles_to_layout_kernel(int64_t M, int64_t N, double* __restrict__ A, int64_t lda, int NB, int64_t MT,
                       const double* __restrict__ tiles) {
  const int64_t m = blockIdx.x, n = blockIdx.y;
  const int64_t i0 = m * NB, j0 = n * NB;
  const double* __restrict__ src = tiles + (m + n * MT) * (int64_t)NB * NB;
  const int tid = threadIdx.x;
  if (VEC && i0 + NB <= M && j0 + NB <= N) {
    const int HP = NB >> 1, tot = NB * HP;
    double* __restrict__ d = A + i0 + j0 * lda;
    for (int e0 = tid; e0 < tot; e0 += kUnroll * kThreads) {
      double2 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * kThreads;
        if (e < tot) v[u] = __ldcs(reinterpret_cast<const double2*>(src) + e);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * kThreads;
        if (e < tot) {
          const int jl = e / HP, il = 2 * (e - jl * HP);
          __stcs(reinterpret_cast<double2*>(d + il + jl * lda), v[u]);
        }
      }
    }
  } else {
    const int tot = NB * NB;
    for (int e = tid; e < tot; e += kThreads) {
      const int jl = e / NB, il = e - jl * NB;
      const int64_t i = i0 + il, j = j0 + jl;
      if (i < M && j < N) A[i + j * lda] = src[e];
    }
  }
}

__global__ void __launch_bounds__(kThreads)
v_to_tiles_kernel(int64_t M, int64_t K, const double* __restrict__ A, int64_t lda, int NB,
                  int64_t MT, int64_t KT, double* __restrict__ tiles) {
  const int64_t rows = MT * NB, total = rows * KT * NB;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = w / rows, i = w - j * rows;
    const int64_t m = i / NB, il = i - m * NB, n = j / NB, jl = j - n * NB;
    tiles[(m + n * MT) * (int64_t)NB * NB + il + jl * NB] =
        (i < M && j < K) ? A[i + j * lda] : 0.0;
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void __launch_bounds__(kThreads)
rng_uniform_kernel(int64_t M, int64_t N, double* __restrict__ A, int64_t lda, uint64_t key,
                   uint64_t offset) {
  const int64_t total = M * N;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = w / M, i = w - j * M;
    const uint64_t bits = splitmix64(key + offset + (uint64_t)w) >> 11;
    A[i + j * lda] = (double)bits * 0x1.0p-53 - 0.5;
  }
}

__global__ void zero_int_kernel(int* p) { *p = 0; }

// Local tile columns of a 1D block-cyclic N x N matrix (dist path): local
// column j holds global tile column n = rank + j*P; element (il, jl) of tile
// (m, n) is the generator's value at global (i, c) = (m*NB+il, n*NB+jl),
// idx = i + c*N, with the same padding as layout_to_tiles.
__global__ void __launch_bounds__(kThreads)
dist_fill_kernel(int64_t M, int64_t N, int NB, int64_t MT, int P, int rank, int64_t nloc, double* __restrict__ A,
                 uint64_t key) {
  const int64_t tile = (int64_t)NB * NB;
  const int64_t total = nloc * MT * tile;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = w / tile, e = w - t * tile;
    const int64_t m = t % MT, j = t / MT;
    const int64_t jl = e / NB, il = e - jl * NB;
    const int64_t i = m * NB + il, c = (rank + j * P) * NB + jl;
    double v;
    if (i < M && c < N) {
      const uint64_t bits = splitmix64(key + (uint64_t)(i + c * M)) >> 11;
      v = (double)bits * 0x1.0p-53 - 0.5;
    } else {
      v = (c >= N && i == c && c >= M) ? 1.0 : 0.0;
    }
    A[w] = v;
  }
}

__global__ void __launch_bounds__(kThreads)
nonfinite_kernel(const double* __restrict__ A, int64_t n, int* d_info) {
  int bad = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n;
       w += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(A[w])) bad = 1;
  if (bad) *d_info = 1;
}

uint64_t host_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace

static bool layout_vec(const double* A, int64_t lda, int NB) {
  return (NB % 2 == 0) && (lda % 2 == 0) && ((uintptr_t)A % 16 == 0);
}

int launch_layout_to_tiles(int64_t M, int64_t N, const double* A, int64_t lda, int NB, int64_t MT,
                           int64_t NT, double* tiles, int* d_info, cudaStream_t s) {
  if (MT <= 0 || NT <= 0) return 0;
  if (NT > 65535) {
    set_error("layout_to_tiles: more than 65535 tile columns");
    return TILEQR_ERR_CUDA;
  }
  const dim3 grid((unsigned)MT, (unsigned)NT);
  if (layout_vec(A, lda, NB)) layout_to_tiles_kernel<true><<<grid, kThreads, 0, s>>>(M, N, A, lda, NB, MT, tiles, d_info);
  else layout_to_tiles_kernel<false><<<grid, kThreads, 0, s>>>(M, N, A, lda, NB, MT, tiles, d_info);
  TQ_LAUNCH_CHECK();
  return 0;
}

int launch_tiles_to_layout(int64_t M, int64_t N, double* A, int64_t lda, int NB, int64_t MT,
                           int64_t NT, const double* tiles, cudaStream_t s) {
  if (M <= 0 || N <= 0) return 0;
  const int64_t mt = (M + NB - 1) / NB, nt = (N + NB - 1) / NB;  // only tiles holding real entries
  (void)NT;
  if (nt > 65535) {
    set_error("tiles_to_layout: more than 65535 tile columns");
    return TILEQR_ERR_CUDA;
  }
  const dim3 grid((unsigned)mt, (unsigned)nt);
  if (layout_vec(A, lda, NB)) tiles_to_layout_kernel<true><<<grid, kThreads, 0, s>>>(M, N, A, lda, NB, MT, tiles);
  else tiles_to_layout_kernel<false><<<grid, kThreads, 0, s>>>(M, N, A, lda, NB, MT, tiles);
  TQ_LAUNCH_CHECK();
  return 0;
}

int launch_v_to_tiles(int64_t M, int64_t K, const double* A, int64_t lda, int NB, int64_t MT,
                      int64_t KT, double* tiles, cudaStream_t s) {
  v_to_tiles_kernel<<<grid_for(MT * NB * KT * NB), kThreads, 0, s>>>(M, K, A, lda, NB, MT, KT,
                                                                      tiles);
  TQ_LAUNCH_CHECK();
  return 0;
}

int launch_rng_uniform(int64_t M, int64_t N, double* A, int64_t lda, uint64_t seed,
                       uint64_t offset, cudaStream_t s) {
  if (M <= 0 || N <= 0) return 0;
  rng_uniform_kernel<<<grid_for(M * N), kThreads, 0, s>>>(M, N, A, lda, host_splitmix64(seed),
                                                          offset);
  TQ_LAUNCH_CHECK();
  return 0;
}

int launch_dist_fill(int64_t M, int64_t N, int NB, int64_t MT, int nranks, int rank, int64_t nloc, double* A,
                     uint64_t seed, cudaStream_t s) {
  dist_fill_kernel<<<grid_for(nloc * MT * NB * NB), kThreads, 0, s>>>(M, N, NB, MT, nranks, rank, nloc, A,
                                                                      host_splitmix64(seed));
  TQ_LAUNCH_CHECK();
  return 0;
}

int launch_nonfinite_check(const double* A, int64_t n, int* d_info, cudaStream_t s) {
  nonfinite_kernel<<<grid_for(n), kThreads, 0, s>>>(A, n, d_info);
  TQ_LAUNCH_CHECK();
  return 0;
}

__global__ void fill_ptrs_kernel(double** out, double* base, size_t stride, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = base + stride * i;
}

int launch_fill_ptrs(double** out, double* base, size_t stride, int n, cudaStream_t s) {
  if (n <= 0) return 0;
  fill_ptrs_kernel<<<(n + 255) / 256, 256, 0, s>>>(out, base, stride, n);
  TQ_LAUNCH_CHECK();
  return 0;
}

// T of inner blocking IB from the T of a factorization run at IBe (a multiple
// of IB): the diagonal IB x IB blocks of each IBe x IBe block (R23 --
// the compact-WY recurrence T[0:i, i] = -tau_i T[0:i, 0:i] V[:, 0:i]^T v_i
// restricted to the reflectors of one IB block involves only that block).
__global__ void t_extract_kernel(const double* __restrict__ Te, int IBe, double* __restrict__ T, int IB, int NB,
                                 long long total) {
  const long long per = (long long)IB * NB;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long tile = e / per;
    const int r = (int)(e - tile * per);
    const int j = r / IB, l = r - j * IB;
    const int jb = j % IB;               // column j within its IB block
    const int off = (j - jb) % IBe;      // first row of that IB block within the IBe block
    T[e] = l <= jb ? __ldg(Te + tile * (long long)IBe * NB + off + l + (long long)j * IBe) : 0.0;
  }
}

int launch_t_extract(const double* Te, int IBe, double* T, int IB, int NB, int64_t ntiles, cudaStream_t s) {
  const long long total = (long long)ntiles * IB * NB;
  if (total <= 0) return 0;
  t_extract_kernel<<<grid_for(total), kThreads, 0, s>>>(Te, IBe, T, IB, NB, total);
  TQ_LAUNCH_CHECK();
  return 0;
}

// Same for arrays of per-tile pointers (batched entry points): T at IBo, a
// divisor of IBi, from T at IBi -- the diagonal IBo-blocks.  One CTA per tile.
__global__ void t_extract_ptrs_kernel(const double* const* Tin, int IBi, double* const* Tout, int IBo, int NB) {
  const double* Ti = Tin[blockIdx.x];
  double* To = Tout[blockIdx.x];
  for (int e = threadIdx.x; e < IBo * NB; e += blockDim.x) {
    const int j = e / IBo, l = e - j * IBo;
    const int jb = j % IBo, off = (j - jb) % IBi;
    To[e] = l <= jb ? Ti[off + l + (size_t)j * IBi] : 0.0;
  }
}

int launch_t_extract_ptrs(const double* const* Tin, int IBi, double* const* Tout, int IBo, int NB, int batch,
                          cudaStream_t s) {
  if (batch <= 0) return 0;
  t_extract_ptrs_kernel<<<batch, kThreads, 0, s>>>(Tin, IBi, Tout, IBo, NB);
  TQ_LAUNCH_CHECK();
  return 0;
}

// T at IB (> 64) of a whole factorization run at IBs (a divisor of IB,
// DESIGN.md R23): for every tile (m, k), m >= k, k < KT, and every IB-panel,
// the compact-WY recurrence T[i, i] = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] z,
// z_l = v_l^T v_i, with V read from the factored tile
// (GEQRT form on the diagonal: unit lower trapezoid; TSQRT form below: the
// tops e_l, e_i are orthogonal, only V2 contributes) and tau_j the diagonal of
// T at IBs.  T must be zeroed by the caller (tiles m < k stay 0).  Multi-rank
// (P > 1): the tiles and T are rank r's local tile columns jl (global column
// r + jl*P).
__global__ void t_assemble_big_kernel(const double* __restrict__ tiles, const double* __restrict__ Ts,
                                      double* __restrict__ T, int NB, int IB, int IBs, long long MT,
                                      long long NTl, long long KT, int P, int r) {
  extern __shared__ double z[];  // IB
  for (long long t = blockIdx.x; t < MT * NTl; t += gridDim.x) {
    const long long jl = t / MT, m = t - jl * MT, k = r + jl * P;
    if (k >= KT || m < k) continue;
    const size_t tile = (size_t)t;
    const double* V = tiles + tile * NB * NB;
    const double* ts = Ts + tile * IBs * NB;
    double* To = T + tile * IB * NB;
    const bool ge = m == k;
    for (int c0 = 0; c0 < NB; c0 += IB) {
      for (int i = 0; i < IB; ++i) {
        const int j = c0 + i;
        for (int l = threadIdx.x; l < i; l += blockDim.x) {
          const int jl = c0 + l;
          const double* vl = V + (size_t)jl * NB;
          const double* vi = V + (size_t)j * NB;
          double acc = ge ? vl[j] : 0.0;  // GEQRT: v_l[j] * 1
          for (int r = ge ? j + 1 : 0; r < NB; ++r) acc = fma(vl[r], vi[r], acc);
          z[l] = acc;
        }
        __syncthreads();
        const double tau = ts[(j % IBs) + (size_t)j * IBs];
        for (int r = threadIdx.x; r < IB; r += blockDim.x) {
          double out = r == i ? tau : 0.0;
          if (r < i) {
            double acc = 0.0;
            for (int l = r; l < i; ++l) acc = fma(To[r + (size_t)(c0 + l) * IB], z[l], acc);
            out = -tau * acc;
          }
          To[r + (size_t)j * IB] = out;
        }
        __syncthreads();
      }
    }
  }
}

int launch_t_assemble_big(const double* tiles, const double* Ts, double* T, int NB, int IB, int IBs, int64_t MT,
                          int64_t NTl, int64_t KT, int P, int r, int nsm, cudaStream_t s) {
  const long long n = (long long)MT * NTl;
  if (n <= 0) return 0;
  const int grid = (int)std::min<long long>(n, (long long)std::max(1, nsm) * 4);
  t_assemble_big_kernel<<<grid, kThreads, (size_t)IB * sizeof(double), s>>>(tiles, Ts, T, NB, IB, IBs, MT, NTl,
                                                                            KT, P, r);
  TQ_LAUNCH_CHECK();
  return 0;
}

int launch_zero_int(int* p, cudaStream_t s) {
  zero_int_kernel<<<1, 1, 0, s>>>(p);
  TQ_LAUNCH_CHECK();
  return 0;
}

}  // namespace tileqr
