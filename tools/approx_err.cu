// Max relative error of rsqrt.approx.ftz.f64 and rcp.approx.ftz.f64 on sm_100a
// (log-uniform inputs over [2^-40, 2^40]), against 1/sqrt and 1/x in double.
#include <cstdio>
#include <cmath>
__global__ void k(double* err, int n) {
  double er = 0, ec = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double u = (i + 0.5) / n;               // uniform in (0,1)
    const double x = exp2(-40.0 + 80.0 * u) * (1.0 + 0.37 * sin(1e4 * u));
    double r, c;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(c) : "d"(x));
    er = fmax(er, fabs(r * sqrt(x) - 1.0));
    ec = fmax(ec, fabs(c * x - 1.0));
  }
  atomicMax((unsigned long long*)&err[0], __double_as_longlong(er));
  atomicMax((unsigned long long*)&err[1], __double_as_longlong(ec));
}
int main() {
  double* e; cudaMallocManaged(&e, 16); e[0] = e[1] = 0;
  k<<<1184, 256>>>(e, 1 << 26); cudaDeviceSynchronize();
  printf("rsqrt.approx.ftz.f64 max rel err %.3e (2^%.2f)\nrcp.approx.ftz.f64 max rel err %.3e (2^%.2f)\n", e[0], log2(e[0]), e[1], log2(e[1]));
}
