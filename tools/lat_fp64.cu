// Dependent-chain latency of FP64 ops on sm_100a (clock64 around N dependent ops).
#include <cstdio>
__global__ void k(double* out, double x, long long* cyc) {
  double a = x, b = x * 0.5 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) a = fma(a, b, 0.25);
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) a = a + b;
  long long t2 = clock64();
  for (int i = 0; i < 100; ++i) a = sqrt(a + 2.0);
  long long t3 = clock64();
  for (int i = 0; i < 100; ++i) a = 1.0 / (a + 3.0);
  long long t4 = clock64();
  for (int i = 0; i < 100; ++i) a = __drcp_rn(a + 3.0);
  long long t5 = clock64();
  for (int i = 0; i < 100; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31) + 1.0;
  long long t6 = clock64();
  __shared__ double s[64];
  s[threadIdx.x & 63] = a;
  __syncthreads();
  long long t7 = clock64();
  for (int i = 0; i < 100; ++i) { __syncthreads(); }
  long long t8 = clock64();
  for (int i = 0; i < 100; ++i) a = s[((int)a) & 31] + a;
  long long t9 = clock64();
  for (int i = 0; i < 100; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a + 2.0)); a = r; }
  long long t10 = clock64();
  for (int i = 0; i < 100; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a + 2.0)); a = r; }
  long long t11 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 1000; cyc[1] = (t2 - t1) / 1000; cyc[2] = (t3 - t2) / 100; cyc[3] = (t4 - t3) / 100;
    cyc[4] = (t5 - t4) / 100; cyc[5] = (t6 - t5) / 100; cyc[6] = (t8 - t7) / 100; cyc[7] = (t9 - t8) / 100;
    cyc[8] = (t10 - t9) / 100; cyc[9] = (t11 - t10) / 100;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMallocManaged(&c, 8 * 10);
  for (int nt : {32, 128, 256}) {
    k<<<1, nt>>>(o, 1.1, c); cudaDeviceSynchronize();
    printf("threads=%d dfma=%lld dadd=%lld sqrt=%lld div=%lld drcp_rn=%lld shfl+dadd=%lld bar=%lld lds+dadd=%lld rsqrt_approx+dadd=%lld rcp_approx+dadd=%lld\n", nt, c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8], c[9]);
  }
}
