// Microbenchmark + check of the executor's 128x128 diagonal-block kernels
// (block_potrf / block_trtri from csrc/executor.cu) on one CTA of 256
// consumer threads: cycles per call, per-phase probes (ctl.dbg2), max error
// against a CPU Cholesky / triangular inverse.
#include "../../paper_1002_4057_b200/csrc/executor.cu"
#include <cmath>
#include <cstdio>
using namespace tinv;

__global__ void __launch_bounds__(256, 1) bench(const double* A, double* out, long long* cyc, unsigned long long* dbg,
                                                int reps, int which) {
  extern __shared__ __align__(16) char sm_[];
  __shared__ SmemCtl ctl;
  double* S = reinterpret_cast<double*>(sm_);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) ctl.dbg2[k] = 0;
    for (int k = 0; k < 4; ++k) ctl.dbg[k] = 0;
  }
  long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    load_block_lower(S, A, 128);
    cons_bar();
    const long long t0 = clock64();
    if (which == 0) {
      block_potrf(S, ctl);
    } else {
      block_trtri_dmma(S, ctl.dbg2);
    }
    cons_bar();
    tot += clock64() - t0;
  }
  store_block_lower(S, out, 128);
  if (threadIdx.x == 0) {
    *cyc = tot / reps;
    for (int k = 0; k < 8; ++k) dbg[k] = ctl.dbg2[k] / reps;
  }
}

int main() {
  const int n = 128;
  double *h = new double[n * n], *L = new double[n * n], *X = new double[n * n], *g = new double[n * n];
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) / 16777216.0) - 0.5; };
  double* G = new double[n * n];
  for (int k = 0; k < n * n; ++k) G[k] = rnd();
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double a = 0;
      for (int k = 0; k < n; ++k) a += G[i * n + k] * G[j * n + k];
      h[i * n + j] = a / n + (i == j ? 1.0 : 0.0);
    }
  // CPU Cholesky (lower) and inverse of L
  for (int k = 0; k < n * n; ++k) L[k] = 0;
  for (int j = 0; j < n; ++j) {
    double d = h[j * n + j];
    for (int k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
    L[j * n + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double v = h[i * n + j];
      for (int k = 0; k < j; ++k) v -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = v / L[j * n + j];
    }
  }
  for (int k = 0; k < n * n; ++k) X[k] = 0;
  for (int i = 0; i < n; ++i) {
    X[i * n + i] = 1.0 / L[i * n + i];
    for (int j = 0; j < i; ++j) {
      double v = 0;
      for (int k = j; k < i; ++k) v += L[i * n + k] * X[k * n + j];
      X[i * n + j] = -v / L[i * n + i];
    }
  }
  double *dA, *dL, *out;
  long long* cyc;
  unsigned long long* dbg;
  cudaMalloc(&dA, n * n * 8);
  cudaMalloc(&dL, n * n * 8);
  cudaMalloc(&out, n * n * 8);
  cudaMallocManaged(&cyc, 8);
  cudaMallocManaged(&dbg, 64);
  cudaMemcpy(dA, h, n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dL, L, n * n * 8, cudaMemcpyHostToDevice);
  const int smem = 128 * 129 * 8 + 64 * 65 * 8 * 2;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int which = 0; which < 2; ++which) {
    const double* in = which ? dL : dA;
    const double* ref = which ? X : L;
    bench<<<1, 256, smem>>>(in, out, cyc, dbg, 20, which);
    cudaDeviceSynchronize();
    bench<<<1, 256, smem>>>(in, out, cyc, dbg, 200, which);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(g, out, n * n * 8, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int k = 0; k < n * n; ++k) {
      err = std::fmax(err, std::fabs(g[k] - ref[k]));
      mx = std::fmax(mx, std::fabs(ref[k]));
    }
    printf("%s: %lld cycles per 128x128 call (%s), max rel err %.2e; probes:",
           which ? "block_trtri_dmma" : "block_potrf",
           *cyc, cudaGetErrorString(e), err / mx);
    for (int k = 0; k < 8; ++k) printf(" %llu", dbg[k]);
    printf("\n");
  }
  return 0;
}
