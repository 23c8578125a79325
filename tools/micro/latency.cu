// Dependent-chain latencies on B200 (cycles per op): DFMA, SHFL (f64), rsqrt(f64),
// sqrt+div, rsqrt.approx.f64, LDS f64.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void lat(double* out, long long* cyc, double x0) {
  __shared__ double sm[64];
  double x = x0 + threadIdx.x * 1e-9;
  if (threadIdx.x < 64) sm[threadIdx.x] = 1.0 + threadIdx.x * 1e-3;
  __syncthreads();
  const int N = 1024;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    if (K == 0) x = fma(x, 0.999999, 1e-7);
    if (K == 1) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    if (K == 2) x = rsqrt(x) + 0.5;
    if (K == 3) x = 1.0 / sqrt(x) + 0.5;
    if (K == 4) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 0.5; }
    if (K == 5) x = sm[((int)x) & 63] + 0.5;
    if (K == 6) x = 1.0 / x + 0.5;
    if (K == 7) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 0.5; }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / N;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMallocManaged(&cyc, 8);
  const char* names[] = {"DFMA", "SHFL f64", "rsqrt(f64)", "1/sqrt(f64)", "rsqrt.approx.f64", "LDS f64 (dep addr)", "1/x f64", "rcp.approx.f64"};
#define RUN(K) lat<K><<<1, 32>>>(out, cyc, 1.7); cudaDeviceSynchronize(); lat<K><<<1, 32>>>(out, cyc, 1.7); cudaDeviceSynchronize(); printf("%-20s %lld cycles (+ add for the rsqrt/rcp/lds rows)\n", names[K], *cyc);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
  return 0;
}
