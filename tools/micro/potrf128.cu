// Standalone timing of the executor's 128x128 block Cholesky (8-wide register
// panels + look-ahead DMMA updates), 256 threads, smem row stride 129.
// potrf128_body.inc = chol8_inv / upd8 / block_potrf cut from csrc/executor.cu.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int BLK = 128, SLD = 132;
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
#include "potrf128_body.inc"
__global__ void k(double* out, long long* cyc, int reps) {
  extern __shared__ double S[];
  __shared__ unsigned long long dbg[4];
  __shared__ int scan;
  if (threadIdx.x < 4) dbg[threadIdx.x] = 0;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < BLK * SLD; e += 256) {
      const int i = e / SLD, j = e % SLD;
      S[e] = (j > i || j >= BLK) ? 0.0 : (i == j ? 130.0 : 1.0 / (1 + i + j));
    }
    __syncthreads();
    long long t0 = clock64();
    int f = block_potrf(S, scan, dbg);
    long long t1 = clock64();
    tot += t1 - t0;
    if (threadIdx.x == 0) out[r] = S[127 * SLD + 127] + f;
    __syncthreads();
  }
  if (threadIdx.x == 0) { cyc[0] = tot / reps; cyc[1] = dbg[0] / reps; cyc[2] = dbg[1] / reps; cyc[3] = dbg[2] / reps; cyc[4] = dbg[3] / reps; }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 8 * 8);
  const int sm = (BLK * SLD + 64 + 1024) * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<1, 256, sm>>>(out, cyc, 4); cudaDeviceSynchronize();
  k<<<1, 256, sm>>>(out, cyc, 16); cudaError_t e = cudaDeviceSynchronize();
  printf("%s block_potrf 128: %lld cycles (phase A %lld, phase B %lld)\n", cudaGetErrorString(e), cyc[0], cyc[1], cyc[2]);
  return 0;
}
