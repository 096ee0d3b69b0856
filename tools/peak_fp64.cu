// FP64 peak microbenchmark for B200 (sm_100a).
//
// Measures the chip's FP64 throughput two ways, so that the roofline of the
// tile-QR update kernels has a measured denominator:
//   * DMMA: register-resident independent mma.sync.m8n8k4.f64 chains
//   * DFMA: register-resident independent fma.rn.f64 chains
// Each is run as a short burst (best of 10) and as a sustained loop (~4 s).
// Output: one JSON line.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peak_fp64 peak_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dmma_loop(double* out, int iters, double seed) {
  const int lane = threadIdx.x & 31;
  double a = seed + lane * 1e-3, b = 1.0 - lane * 1e-4;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[i][0]), "+d"(c[i][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-7;
  double c[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i];
  if (s == 123.456) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);

  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f", prop.name, sms, clk_khz / 1e3);
  for (int kind = 0; kind < 2; ++kind) {
    for (int threads : {128, 256, 512}) {
      const int blocks = sms * (kind == 0 ? 4 : 2);
      const int iters = 4096;
      const double flop_per_launch = kind == 0
          ? 2.0 * 256 * kChains * (double)iters * (threads / 32) * blocks
          : 2.0 * kChains * (double)iters * threads * blocks;
      auto launch = [&]() {
        if (kind == 0) dmma_loop<<<blocks, threads>>>(out, iters, 0.5);
        else dfma_loop<<<blocks, threads>>>(out, iters, 0.5);
      };
      launch();
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 10; ++r) {
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      // sustained: back to back for ~4 s
      int reps = (int)(4000.0 / best) + 1;
      CK(cudaEventRecord(e0));
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float tot;
      CK(cudaEventElapsedTime(&tot, e0, e1));
      printf(", \"%s_t%d_burst_tflops\": %.3f, \"%s_t%d_sustained_tflops\": %.3f",
             kind == 0 ? "dmma" : "dfma", threads, flop_per_launch / (best * 1e-3) / 1e12,
             kind == 0 ? "dmma" : "dfma", threads, flop_per_launch * reps / (tot * 1e-3) / 1e12);
      fflush(stdout);
    }
  }
  printf("}\n");
  return 0;
}
