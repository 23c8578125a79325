// FP64 peak probes for B200 (sm_100a): DMMA via mma.sync (m8n8k4, m16n8k16)
// and scalar DFMA. Register-only loops, many independent accumulators per
// warp, grid = multiple of the SM count. Prints TFLOP/s per probe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_peak(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, double flop_per_iter_per_warp,
                  double* out, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32.0;
  return warps * iters * flop_per_iter_per_warp / (best * 1e-3) / 1e12;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", p.name, sms, p.clockRate);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int threads = wpb * 32, blocks = sms * bps;
      double t1 = run(dmma_m8n8k4<8>, blocks, threads, iters, 8 * 2.0 * 8 * 8 * 4, out, 5);
      double t2 = run(dmma_m8n8k4<16>, blocks, threads, iters, 16 * 2.0 * 8 * 8 * 4, out, 5);
      double t3 = run(dmma_m16n8k16<4>, blocks, threads, iters / 4, 4 * 2.0 * 16 * 8 * 16, out, 5);
      double t4 = run(dfma_peak<16>, blocks, threads, iters, 16 * 2.0 * 32, out, 5);
      printf("warps/blk %2d blk/sm %d : dmma8x8x4(8acc) %.2f  dmma8x8x4(16acc) %.2f  "
             "dmma16x8x16(4acc) %.2f  dfma(16) %.2f TFLOP/s\n", wpb, bps, t1, t2, t3, t4);
    }
  }
  // sustained: ~3 s of dmma at the best config
  {
    int threads = 256, blocks = sms * 2;
    double best = 0;
    for (int r = 0; r < 6; ++r) {
      double t = run(dmma_m8n8k4<16>, blocks, threads, 200000, 16 * 2.0 * 8 * 8 * 4, out, 1);
      if (t > best) best = t;
      printf("sustained dmma rep %d: %.2f TFLOP/s\n", r, t);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
