// Standalone timing + check of the dataflow 128x128 block Cholesky
// (potrf_flow.inc) against the look-ahead version it replaces
// (potrf128_body.inc), 256 threads, smem row stride SLD.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int BLK = 128, SLD = 132;
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
#include "potrf128_body.inc"
#include "potrf_flow.inc"
template <int NEW>
__global__ void k(const double* A, double* out, long long* cyc, int reps) {
  extern __shared__ double S[];
  __shared__ unsigned long long dbg[8];
  __shared__ int scan;
  __shared__ PotrfFlags fl;
  __shared__ double lp[144];
  if (threadIdx.x < 8) dbg[threadIdx.x] = 0;
  long long tot = 0;
  int f = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < BLK * SLD; e += 256) {
      const int i = e / SLD, j = e % SLD;
      S[e] = (j > i || j >= BLK) ? 0.0 : A[i * BLK + j];
    }
    if (threadIdx.x == 0) { fl.fac = fl.rowdone = fl.ready = 0; scan = 1 << 30; }
    __syncthreads();
    long long t0 = clock64();
    if (NEW) f = block_potrf_flow(S, lp, fl, scan);
    else f = block_potrf(S, scan, dbg);
    long long t1 = clock64();
    tot += t1 - t0;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < BLK * BLK; e += 256) out[e] = S[(e / BLK) * SLD + e % BLK];
  if (threadIdx.x == 0) { cyc[0] = tot / reps; cyc[1] = f; }
}
int main() {
  const int n = BLK;
  double *hA = new double[n * n], *hL = new double[n * n], *hN = new double[n * n];
  // SPD: G G^T / n + I (G uniform)
  double* G = new double[n * n];
  unsigned s = 12345;
  for (int e = 0; e < n * n; ++e) { s = s * 1664525u + 1013904223u; G[e] = (s >> 8) / 16777216.0 - 0.5; }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double t = 0;
      for (int k2 = 0; k2 < n; ++k2) t += G[i * n + k2] * G[j * n + k2];
      hA[i * n + j] = t / n + (i == j ? 1.0 : 0.0);
    }
  double *A, *out; long long* cyc;
  cudaMalloc(&A, n * n * 8); cudaMalloc(&out, n * n * 8); cudaMallocManaged(&cyc, 8 * 8);
  cudaMemcpy(A, hA, n * n * 8, cudaMemcpyHostToDevice);
  const int sm = (BLK * SLD + 64 + 1024) * 8;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int v = 0; v < 2; ++v) {
    auto kk = v ? k<1> : k<0>;
    kk<<<1, 256, sm>>>(A, out, cyc, 4); cudaDeviceSynchronize();
    kk<<<1, 256, sm>>>(A, out, cyc, 16);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(v ? hN : hL, out, n * n * 8, cudaMemcpyDeviceToHost);
    printf("%s %s: %lld cycles, fail %lld\n", cudaGetErrorString(e), v ? "dataflow" : "look-ahead", cyc[0], cyc[1]);
  }
  // residual of L L^T - A (lower) for both, and their difference
  double md = 0, rL = 0, rN = 0, ma = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double tL = 0, tN = 0;
      for (int k2 = 0; k2 <= j; ++k2) { tL += hL[i * n + k2] * hL[j * n + k2]; tN += hN[i * n + k2] * hN[j * n + k2]; }
      rL = fmax(rL, fabs(tL - hA[i * n + j])); rN = fmax(rN, fabs(tN - hA[i * n + j]));
      md = fmax(md, fabs(hL[i * n + j] - hN[i * n + j])); ma = fmax(ma, fabs(hL[i * n + j]));
    }
#ifdef FLOW_PROBE
  long long pr[16];
  cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
  printf("warp 0 per panel (cycles, 20 runs): chol8 %.0f publish %.0f wait-ready %.0f row-solve %.0f diag-update %.0f\n",
         pr[0] / 320.0, pr[1] / 320.0, pr[2] / 300.0, pr[3] / 300.0, pr[4] / 300.0);
  printf("helper warp 1 per round: wait-fac %.0f solve %.0f wait-rowdone+bar %.0f first %.0f rest %.0f end-bar %.0f\n",
         pr[8] / 300.0, pr[9] / 300.0, pr[10] / 300.0, pr[11] / 280.0, pr[12] / 300.0, pr[13] / 300.0);
#endif
  printf("residual |LL^T - A|max: look-ahead %.3e dataflow %.3e; max |L_new - L_old| / max|L| = %.3e\n", rL, rN, md / ma);
  return 0;
}
