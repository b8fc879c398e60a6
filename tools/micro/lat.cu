// Dependent-chain latency of fp64 primitives on B200 (cycles per op).
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double rsqrt_fast(double x) {  // MUFU approx + 1 Newton step
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y * (1.5 - 0.5 * x * y * y);
}
template <int OP>
__global__ void k(double* out, long long* cyc, int n) {
  double x = 1.0 + threadIdx.x * 1e-9, acc = 0.0;
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = 1.0 + 1e-12 * threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, 0.9999999, 1e-7);
    if (OP == 1) x = sqrt(x) + 0.5;
    if (OP == 2) x = rsqrt(x) + 0.5;
    if (OP == 3) x = 1.0 / x + 0.5;
    if (OP == 4) { double s, c; sincos(x, &s, &c); x = s + c + 0.3; }
    if (OP == 5) x = rsqrt_fast(x) + 0.5;
    if (OP == 6) x = sm[((int)x) & 63] + 1e-9 * x;
    if (OP == 7) x = x / (x + 1.0) + 0.5;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + acc;
  if (threadIdx.x == 0) cyc[OP] = (t1 - t0) / n;
}
__global__ void acc_check(double* e) {
  double mx = 0, mx2 = 0;
  for (int i = 0; i < 100000; ++i) {
    double x = 1e-6 + i * 1.37e-3;
    double r = 1.0 / sqrt(x);
    double a = rsqrt_fast(x);
    double b = rsqrt(x);
    mx = fmax(mx, fabs(a - r) / r);
    mx2 = fmax(mx2, fabs(b - r) / r);
  }
  e[0] = mx; e[1] = mx2;
}
int main() {
  double* out; long long* cyc; double* e;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 16 * 8); cudaMallocManaged(&e, 16);
  const char* names[] = {"dfma", "sqrt", "rsqrt", "div(1/x)", "sincos", "rsqrt.approx+1NR", "lds(dep)", "x/(x+1)"};
  k<0><<<1, 32>>>(out, cyc, 4096); k<1><<<1, 32>>>(out, cyc, 4096); k<2><<<1, 32>>>(out, cyc, 4096);
  k<3><<<1, 32>>>(out, cyc, 4096); k<4><<<1, 32>>>(out, cyc, 1024); k<5><<<1, 32>>>(out, cyc, 4096);
  k<6><<<1, 32>>>(out, cyc, 4096); k<7><<<1, 32>>>(out, cyc, 4096);
  acc_check<<<1, 1>>>(e);
  cudaDeviceSynchronize();
  for (int i = 0; i < 8; ++i) printf("%-18s %lld cycles/op\n", names[i], cyc[i]);
  printf("rsqrt.approx+1NR max rel err %.3e ; rsqrt() %.3e\n", e[0], e[1]);
  return 0;
}
