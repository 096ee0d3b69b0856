// DMMA (mma.sync.m8n8k4.f64) dependent-chain latency and per-warp throughput vs #chains.
#include <cstdio>
template <int C>
__global__ void k(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[C][2];
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0);
}
template <int C> void run(double* o, long long* c, int warps) {
  int iters = 200;
  k<C><<<1, 32 * warps>>>(o, c, iters); cudaDeviceSynchronize();
  k<C><<<1, 32 * warps>>>(o, c, iters); cudaDeviceSynchronize();
  printf("warps/CTA=%d chains/warp=%d: %.1f cycles per DMMA per warp (iter of %d dependent steps)\n", warps, C, (double)c[0] / (iters * C), iters);
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 4096); cudaMallocManaged(&c, 8 * 8);
  for (int w : {1, 4, 8, 16}) { run<1>(o, c, w); run<2>(o, c, w); run<4>(o, c, w); run<8>(o, c, w); run<16>(o, c, w); }
}
