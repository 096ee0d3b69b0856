// DMMA issue-rate microbenchmark: TFLOP/s of independent mma.sync.m8n8k4.f64
// chains vs warps per SMSP (1 CTA per SM of 128/256/512 threads) and chains
// per warp.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_occ tools/dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void loop(double* out, int iters, double seed) {
  const int lane = threadIdx.x & 31;
  double a = seed + lane * 1e-3, b = 1.0 - lane * 1e-4;
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}
template <int C>
void run(double* out, int sms, int threads) {
  const int iters = 8192 / C * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  loop<C><<<sms, threads>>>(out, iters, 0.5);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop<C><<<sms, threads>>>(out, iters, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flop = 512.0 * C * iters * (threads / 32) * (double)sms;
  printf("warps/SMSP %d chains %d: %.2f TFLOP/s\n", threads / 128, C, flop / (best * 1e-3) / 1e12);
}
int main() {
  double* out; cudaMalloc(&out, 4096 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {128, 256, 512}) { run<1>(out, sms, t); run<2>(out, sms, t); run<4>(out, sms, t); run<8>(out, sms, t); }
  return 0;
}
