// dmma.cuh -- FP64 tensor-core and async-copy helpers shared by the sm_100a
// kernels of libtileqr.
//
// FP64 MMA on sm_100a is the warp-level mma.sync.m8n8k4.f64 (SASS
// DMMA.8x8x4); tcgen05 has no kind::f64.  Fragment layout
// (PTX ISA, m8n8k4 .f64), with g = lane>>2, t = lane&3:
//   A (8x4, row):  a = A[g][t]
//   B (4x8, col):  b = B[t][g]
//   C/D (8x8):     {c0, c1} = C[g][2t], C[g][2t+1]
#pragma once

#include <cuda_runtime.h>

namespace tileqr {

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

// Row-major staging of an NB x (<=32) column block of V with an XOR swizzle
// of column bits 2-3 by row bits 1-2 and ld == 8 (mod 16): both DMMA operand
// access patterns used on it, (row 8rb+2t+j, col 8nb+g) and (row 8rb+g,
// col 4kc+t), hit 16 distinct 8-byte bank pairs per half warp.
__device__ __forceinline__ int vsw(int r, int i, int LDV) {
  return r * LDV + (i ^ (((r >> 1) & 3) << 2));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace tileqr
