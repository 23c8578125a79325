// Latency of one 8-wide Cholesky panel step pieces (B200): chol8_inv alone,
// and chol8_inv + one panel-row solve, per call (cycles), 128 threads.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int chol8_inv(const double* S, int ld, int p0, double (&l)[8][8], double (&x)[8][8]) {
  double il[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) l[i][j] = S[(p0 + i) * ld + p0 + j];
  int bad = -1;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double d = l[k][k];
    const bool b = !(d > 0.0) || !isfinite(d);
    bad = (b && bad < 0) ? k : bad;
    il[k] = b ? 1.0 : rsqrt(d);
    l[k][k] = b ? 1.0 : d * il[k];
#pragma unroll
    for (int i = k + 1; i < 8; ++i) l[i][k] *= il[k];
#pragma unroll
    for (int j = k + 1; j < 8; ++j)
#pragma unroll
      for (int i = j; i < 8; ++i) l[i][j] = fma(-l[i][k], l[j][k], l[i][j]);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c][c] = il[c];
#pragma unroll
    for (int i = c + 1; i < 8; ++i) {
      double t = 0.0;
#pragma unroll
      for (int k = c; k < i; ++k) t = fma(l[i][k], x[k][c], t);
      x[i][c] = -t * il[i];
    }
  }
  return bad;
}

// the executor's inv8: x[i][i] = 1 / l[i][i] (IEEE division), so an inverse
// formed from a stored factor is bitwise the one formed inside the factor
__device__ __forceinline__ void inv8_div(const double (&l)[8][8], double (&x)[8][8]) {
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = 1.0 / l[i][i];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c][c] = d[c];
#pragma unroll
    for (int i = c + 1; i < 8; ++i) {
      double t = 0.0;
#pragma unroll
      for (int k = c; k < i; ++k) t = fma(l[i][k], x[k][c], t);
      x[i][c] = -t * d[i];
    }
  }
}

template <int MODE>
__global__ void k(double* out, long long* cyc) {
  __shared__ double S[40 * 129];
  for (int e = threadIdx.x; e < 40 * 129; e += blockDim.x) S[e] = (e % 130 == 0) ? 4.0 : 0.01;
  __syncthreads();
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < 64; ++it) {
    double l[8][8], x[8][8];
    const int p0 = (it & 3) * 8;
    int bad = chol8_inv(S, 129, p0, l, x);
    if (MODE == 2) inv8_div(l, x);
    if (MODE == 1 || MODE == 2) {
      const int q = (p0 + 8 + threadIdx.x) % 40;
      double av[8], v[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) av[kk] = S[q * 129 + p0 + kk];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double t = 0.0;
#pragma unroll
        for (int kk = 0; kk <= c; ++kk) t = fma(av[kk], x[c][kk], t);
        v[c] = t;
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) S[q * 129 + p0 + kk] = v[kk] * 1e-30 + S[q * 129 + p0 + kk];
    }
    acc += x[7][0] + l[7][7] + bad;
    __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / 64;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 128 * 8); cudaMallocManaged(&cyc, 8);
  k<0><<<1, 128>>>(out, cyc); cudaDeviceSynchronize(); k<0><<<1, 128>>>(out, cyc); cudaDeviceSynchronize();
  printf("chol8_inv (+ barrier): %lld cycles\n", *cyc);
  k<1><<<1, 128>>>(out, cyc); cudaDeviceSynchronize(); k<1><<<1, 128>>>(out, cyc); cudaDeviceSynchronize();
  printf("chol8_inv + row solve (+ barrier): %lld cycles\n", *cyc);
  k<2><<<1, 128>>>(out, cyc); cudaDeviceSynchronize(); k<2><<<1, 128>>>(out, cyc); cudaDeviceSynchronize();
  printf("chol8_inv + inverse by division + row solve (+ barrier): %lld cycles\n", *cyc);
  return 0;
}
