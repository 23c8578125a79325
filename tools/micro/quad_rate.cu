// DMMA rate of the fused batched engine's block-product inner loop (k_bsmall's
// mma_quad, csrc/batched.cu) fed from swizzled shared memory, as a function of
// the CTAs resident per SM (1, 2, 3: one warp per SMSP each). Variants:
//   0  per-quad loop as in k_bsmall (16 LDS per 16 DMMA, runtime K bounds)
//   1  32x32 warp tile sharing fragments (8 LDS per 16 DMMA)
//   2  per-quad loop with the next k-step's fragments loaded before the DMMAs
// Prints DMMA per clock per SM against the peak 0.25 (one per 16 clocks per SMSP).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int BB = 64;
__device__ __forceinline__ int sw(int r, int c) { return r * BB + (c ^ ((r & 3) << 2)); }
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <bool TA, bool TB>
__device__ __forceinline__ void mma_quad(const double* SA, const double* SB, int qr, int qc, int k0, int k1,
                                         double (&acc)[2][2][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int r0 = 16 * qr, c0 = 16 * qc;
  for (int k = k0; k < k1; k += 16) {
    double a[4][2], b[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int kk = k + 4 * u + tg;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        a[u][t] = TA ? SA[sw(kk, r0 + 8 * t + g)] : SA[sw(r0 + 8 * t + g, kk)];
        b[u][t] = TB ? SB[sw(c0 + 8 * t + g, kk)] : SB[sw(kk, c0 + 8 * t + g)];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int tj = 0; tj < 2; ++tj) dmma(acc[ti][tj], a[u][ti], b[u][tj]);
  }
}
// software-pipelined per-quad loop: fragments of step k + 8 in flight during step k's DMMAs
template <bool TA, bool TB>
__device__ __forceinline__ void mma_quad_pipe(const double* SA, const double* SB, int qr, int qc, int k0, int k1,
                                              double (&acc)[2][2][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int r0 = 16 * qr, c0 = 16 * qc;
  double a[2][2][2], b[2][2][2];
  auto ld = [&](int k, double (&aa)[2][2], double (&bb)[2][2]) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int kk = k + 4 * u + tg;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        aa[u][t] = TA ? SA[sw(kk, r0 + 8 * t + g)] : SA[sw(r0 + 8 * t + g, kk)];
        bb[u][t] = TB ? SB[sw(c0 + 8 * t + g, kk)] : SB[sw(kk, c0 + 8 * t + g)];
      }
    }
  };
  ld(k0, a[0], b[0]);
  for (int k = k0; k < k1; k += 16) {
    ld(k + 8, a[1], b[1]);
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int tj = 0; tj < 2; ++tj) dmma(acc[ti][tj], a[0][u][ti], b[0][u][tj]);
    if (k + 16 < k1) ld(k + 16, a[0], b[0]);
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int tj = 0; tj < 2; ++tj) dmma(acc[ti][tj], a[1][u][ti], b[1][u][tj]);
  }
}
// 32x32 warp tile (rows 32 wr.., cols 32 wc..): 4 + 4 fragments per k4 step for 16 DMMAs
template <bool TA, bool TB>
__device__ __forceinline__ void mma_w32(const double* SA, const double* SB, int wr, int wc, int k0, int k1,
                                        double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int r0 = 32 * wr, c0 = 32 * wc;
  for (int k = k0; k < k1; k += 8) {
    double a[2][4], b[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int kk = k + 4 * u + tg;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[u][t] = TA ? SA[sw(kk, r0 + 8 * t + g)] : SA[sw(r0 + 8 * t + g, kk)];
        b[u][t] = TB ? SB[sw(c0 + 8 * t + g, kk)] : SB[sw(kk, c0 + 8 * t + g)];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int ti = 0; ti < 4; ++ti)
#pragma unroll
        for (int tj = 0; tj < 4; ++tj) dmma(acc[ti][tj], a[u][ti], b[u][tj]);
  }
}

template <int V>
__global__ void __launch_bounds__(128, 3) k(double* out, long long* cyc, int reps, int k0, int k1) {
  extern __shared__ __align__(128) double dsm[];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 2 * BB * BB; e += 128) dsm[e] = 1e-3 * (e % 17);
  __syncthreads();
  const double* SA = dsm;
  const double* SB = dsm + BB * BB;
  double acc[4][2][2][2] = {};
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (V == 0) {
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) mma_quad<false, true>(SA, SB, warp, sl, k0, k1, acc[sl]);
    } else if (V == 2) {
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) mma_quad_pipe<false, true>(SA, SB, warp, sl, k0, k1, acc[sl]);
    } else if (V == 3) {  // register operands only: 256 DMMAs per warp per rep
      const double a = 1.0 + tid * 1e-9, b = 1.0 - tid * 1e-9;
      for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int q = 0; q < 16; ++q)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"((&acc[0][0][0][0])[2 * q]), "+d"((&acc[0][0][0][0])[2 * q + 1]) : "d"(a), "d"(b));
    } else {
      mma_w32<false, true>(SA, SB, warp >> 1, warp & 1, k0, k1, *reinterpret_cast<double(*)[4][4][2]>(&acc));
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int q = 0; q < 32; ++q) s += (&acc[0][0][0][0])[q];
  out[blockIdx.x * 128 + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(int per_sm, int sms, double* out, long long* cyc) {
  const int reps = 2000;
  const int smem = per_sm == 1 ? 128 * 1024 : per_sm == 2 ? 96 * 1024 : 64 * 1024;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = sms * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(e0);
    k<V><<<grid, 128, smem>>>(out, cyc, reps, 0, 64);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("  kernel %.3f ms -> %.2f TFLOP/s by events\n", ms, 512.0 * 1024 * reps * grid / ms / 1e9);
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)cyc[i];
  mean /= grid;
  const double dm = 1024.0 * reps * per_sm;  // DMMAs per SM in `mean` cycles (64x64x64 product = 1024 DMMA)
  printf("variant %d, %d CTA/SM: %.0f cycles per 64x64x64 product per CTA, %.4f DMMA/clk/SM = %.1f %% of peak (%s)\n", V,
         per_sm, mean / reps, dm / mean, dm / mean / 0.25 * 100, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)p.multiProcessorCount * 3 * 128 * 8);
  cudaMallocManaged(&cyc, (size_t)p.multiProcessorCount * 3 * 8);
  for (int c = 1; c <= 3; ++c) run<0>(c, p.multiProcessorCount, out, cyc);
  for (int c = 1; c <= 3; ++c) run<2>(c, p.multiProcessorCount, out, cyc);
  for (int c = 1; c <= 3; ++c) run<1>(c, p.multiProcessorCount, out, cyc);
  for (int c = 1; c <= 3; ++c) run<3>(c, p.multiProcessorCount, out, cyc);
  return 0;
}
