// Microbenchmark: latency of a 16x16 warp-shuffle Cholesky (executor.cu
// block_potrf panel factor) and variants, one warp, cycles per factor.
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned FULL = 0xffffffffu;

// v0: the executor's version (rsqrt, isfinite, badmask)
__device__ __forceinline__ unsigned f_v0(double (&r)[16], int i, double& my_il) {
  unsigned badmask = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double piv = __shfl_sync(FULL, r[k], k);
    const bool bad = !(piv > 0.0) || !isfinite(piv);
    badmask |= bad ? (1u << k) : 0u;
    const double il = bad ? 1.0 : rsqrt(piv);
    const double l = bad ? 1.0 : piv * il;
    my_il = (i == k) ? il : my_il;
    r[k] = (i == k) ? l : (i > k ? r[k] * il : r[k]);
#pragma unroll
    for (int j = 1; j < 16; ++j) {
      if (j > k) {
        const double v = __shfl_sync(FULL, r[k], j);
        r[j] = (i >= j) ? fma(-r[k], v, r[j]) : r[j];
      }
    }
  }
  return badmask;
}

// v1: fast reciprocal sqrt (MUFU.RSQ64H + 2 Newton steps), validity folded in
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // Newton: y = y * (1.5 - 0.5 x y^2), twice
  double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ unsigned f_v1(double (&r)[16], int i, double& my_il) {
  unsigned badmask = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double piv = __shfl_sync(FULL, r[k], k);
    const bool bad = !(piv > 0.0 && piv < 1.0e308);
    badmask |= bad ? (1u << k) : 0u;
    const double il = rsqrt_fast(bad ? 1.0 : piv);
    my_il = (i == k) ? il : my_il;
    r[k] = (i == k) ? (bad ? 1.0 : piv * il) : (i > k ? r[k] * il : r[k]);
#pragma unroll
    for (int j = 1; j < 16; ++j) {
      if (j > k) {
        const double v = __shfl_sync(FULL, r[k], j);
        r[j] = (i >= j) ? fma(-r[k], v, r[j]) : r[j];
      }
    }
  }
  return badmask;
}

// v2: lazy update (left-looking by column): column k of row i is finished
// right before it is needed; only the pivot chain is serial
__device__ __forceinline__ unsigned f_v2(double (&r)[16], int i, double& my_il) {
  unsigned badmask = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    // r[k] of every lane: subtract sum_{m<k} L[i][m] L[k][m]
    double acc0 = r[k], acc1 = 0.0;
#pragma unroll
    for (int m = 0; m < 15; ++m)
      if (m < k) {
        const double v = __shfl_sync(FULL, r[m], k);  // L[k][m]
        if (m & 1) acc1 = fma(-r[m], v, acc1); else acc0 = fma(-r[m], v, acc0);
      }
    const double a = acc0 + acc1;
    const double piv = __shfl_sync(FULL, a, k);
    const bool bad = !(piv > 0.0 && piv < 1.0e308);
    badmask |= bad ? (1u << k) : 0u;
    const double il = rsqrt_fast(bad ? 1.0 : piv);
    my_il = (i == k) ? il : my_il;
    r[k] = (i == k) ? (bad ? 1.0 : piv * il) : (i > k ? a * il : r[k]);
  }
  return badmask;
}

template <int V>
__global__ void bench(double* out, long long* cyc, int reps) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double r[16];
  for (int j = 0; j < 16; ++j) r[j] = (j == i) ? 20.0 : (j < i ? 1.0 / (1 + i + j) : 0.0);
  double il = 1.0;
  unsigned bm = 0;
  __syncwarp();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    double s[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s[j] = r[j] + rep * 1e-9;
    if (V == 0) bm |= f_v0(s, i, il);
    if (V == 1) bm |= f_v1(s, i, il);
    if (V == 2) bm |= f_v2(s, i, il);
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = 0.5 * r[j] + 0.5 * s[j] * 1e-3 + (j == i ? 10.0 : 0.0);
  }
  long long t1 = clock64();
  double acc = il + bm;
  for (int j = 0; j < 16; ++j) acc += r[j];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8);
  const int reps = 2000;
  bench<0><<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize();
  bench<0><<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize(); printf("v0 executor: %lld cycles per 16x16 factor\n", *cyc);
  bench<1><<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize(); printf("v1 fast rsqrt: %lld\n", *cyc);
  bench<2><<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize(); printf("v2 left-looking: %lld\n", *cyc);
  // 8 warps concurrently (one CTA), v0
  return 0;
}
