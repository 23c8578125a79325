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

// v3: two columns per step (2x2 pivot block, rank-2 update)
__device__ __forceinline__ unsigned f_v3(double (&r)[16], int i, double (&il_out)) {
  unsigned badmask = 0;
  double my_il = 1.0;
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const double a = __shfl_sync(FULL, r[k], k);          // A[k][k]
    const double bb = __shfl_sync(FULL, r[k], k + 1);     // A[k+1][k]
    const double c = __shfl_sync(FULL, r[k + 1], k + 1);  // A[k+1][k+1]
    const bool bad0 = !(a > 0.0) || !isfinite(a);
    const double il0 = bad0 ? 1.0 : rsqrt(a);
    const double l10 = bb * il0;
    const double d = fma(-l10, l10, c);
    const bool bad1 = !(d > 0.0) || !isfinite(d);
    const double il1 = bad1 ? 1.0 : rsqrt(d);
    badmask |= (bad0 ? (1u << k) : 0u) | (bad1 ? (2u << k) : 0u);
    // this row's entries of columns k, k+1
    const double lk = (i == k) ? (bad0 ? 1.0 : a * il0) : r[k] * il0;
    const double lk1 = (i == k + 1) ? (bad1 ? 1.0 : d * il1) : (r[k + 1] - lk * l10) * il1;
    if (i >= k) r[k] = lk;
    if (i >= k + 1) r[k + 1] = lk1;
    my_il = (i == k) ? il0 : ((i == k + 1) ? il1 : my_il);
#pragma unroll
    for (int j = 2; j < 16; ++j) {
      if (j > k + 1) {
        const double v0 = __shfl_sync(FULL, r[k], j);
        const double v1 = __shfl_sync(FULL, r[k + 1], j);
        if (i >= j) r[j] = fma(-r[k + 1], v1, fma(-r[k], v0, r[j]));
      }
    }
  }
  il_out = my_il;
  return badmask;
}

// v4: column broadcast through shared memory (1 STS + broadcast LDS per column)
__device__ __forceinline__ unsigned f_v4(double (&r)[16], int i, double& my_il, double* col) {
  const int lane = threadIdx.x & 31;
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
    if (lane < 16) col[i] = r[k];
    __syncwarp();
#pragma unroll
    for (int j = 1; j < 16; ++j) {
      if (j > k) {
        const double v = col[j];
        r[j] = (i >= j) ? fma(-r[k], v, r[j]) : r[j];
      }
    }
    __syncwarp();
  }
  return badmask;
}

template <int V>
__global__ void bench(double* out, long long* cyc, int reps) {
  __shared__ double colbuf[16];
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
    if (V == 3) bm |= f_v3(s, i, il);
    if (V == 4) bm |= f_v4(s, i, il, colbuf);
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = 0.5 * r[j] + 0.5 * s[j] * 1e-3 + (j == i ? 10.0 : 0.0);
  }
  long long t1 = clock64();
  double acc = il + bm;
  for (int j = 0; j < 16; ++j) acc += r[j];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
}

__global__ void check(double* out) {
  const int lane = threadIdx.x & 31, i = lane & 15;
  double r0[16], r3[16];
  for (int j = 0; j < 16; ++j) r0[j] = r3[j] = (j == i) ? 20.0 + i : (j < i ? 1.0 / (1 + i + j) : 0.0);
  double il0 = 0, il3 = 0;
  f_v0(r0, i, il0);
  f_v3(r3, i, il3);
  double e = fabs(il0 - il3);
  for (int j = 0; j <= i; ++j) e = fmax(e, fabs(r0[j] - r3[j]));
  for (int o = 16; o; o >>= 1) e = fmax(e, __shfl_xor_sync(FULL, e, o));
  if (lane == 0) out[0] = e;
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
  bench<3><<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize(); printf("v3 2-column steps: %lld\n", *cyc);
  bench<4><<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize(); printf("v4 smem column broadcast: %lld\n", *cyc);
  // correctness: v0 vs v3 on the same SPD 16x16
  check<<<1, 32>>>(out); cudaDeviceSynchronize();
  double h[64]; cudaMemcpy(h, out, 64 * 8, cudaMemcpyDeviceToHost); printf("max |v0 - v3| = %.3e\n", h[0]);
  // 8 warps concurrently (one CTA), v0
  return 0;
}
