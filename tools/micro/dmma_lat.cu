// DMMA.8x8x4 dependent-chain latency and independent-chain throughput per warp (B200).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double acc[CH][2] = {};
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / 256;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMallocManaged(&cyc, 8);
#define RUN(CH) k<CH><<<1, 32>>>(out, cyc, 1.0, 1e-3); cudaDeviceSynchronize(); k<CH><<<1, 32>>>(out, cyc, 1.0, 1e-3); cudaDeviceSynchronize(); printf("%2d chains: %lld cycles per round (%.1f per DMMA)\n", CH, *cyc, (double)*cyc / CH);
  RUN(1) RUN(2) RUN(4) RUN(8) RUN(16)
  return 0;
}
