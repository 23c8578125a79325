// Helper-warp trailing updates of the dataflow block Cholesky in isolation:
// NW warps run the 15 rounds of rank-8 block updates (units of 4 blocks of a
// row, unit c -> warp c mod NW), no pivot chain. MODE 1: DFMA instead of DMMA;
// MODE 2: no shared loads (register operands).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int BLK = 128, SLD = 132;
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE, int NW>
__global__ void k(double* out, long long* cyc) {
  extern __shared__ double S[];
  for (int e = threadIdx.x; e < BLK * SLD; e += blockDim.x) S[e] = 1e-3 * ((e * 7) % 13);
  __syncthreads();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long t0 = clock64();
  const int hw = warp;
  constexpr int T8 = 16;
  long long units = 0;
  double acc4 = 0;
  for (int P = 0; P + 1 < T8; ++P) {
    const int p0 = 8 * P;
    const int g = lane >> 2, tg = lane & 3;
    int c = 0;
    for (int i = P + 3; i < T8; ++i) {
      const int r = 8 * i + g;
      for (int j0 = P + 1; j0 <= i; j0 += 4, ++c) {
        if (c % NW != hw) continue;
        ++units;
        double a0 = -S[r * SLD + p0 + tg], a1 = -S[r * SLD + p0 + 4 + tg];
        double x[4][2], b[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c0 = 8 * min(j0 + u, i);
          if (MODE == 2 || MODE == 3) {
            x[u][0] = c0; x[u][1] = r; b[u][0] = a0 * u; b[u][1] = a1 + u;
          } else {
            const double2 c2 = *reinterpret_cast<const double2*>(S + r * SLD + c0 + 2 * tg);
            x[u][0] = c2.x;
            x[u][1] = c2.y;
            b[u][0] = S[(c0 + g) * SLD + p0 + tg];
            b[u][1] = S[(c0 + g) * SLD + p0 + 4 + tg];
          }
        }
        if (MODE == 3) {  // skeleton: no math
#pragma unroll
          for (int u = 0; u < 4; ++u) { x[u][0] += 1.0; }
        } else if (MODE == 4) {  // loads, no DMMA / stores
          acc4 += x[0][0] + x[1][1] + x[2][0] + x[3][1] + b[0][0] + b[1][1] + b[2][0] + b[3][1] + a0 + a1;
          continue;
        } else if (MODE == 1) {
#pragma unroll
          for (int u = 0; u < 4; ++u) { x[u][0] = fma(a0, b[u][0], x[u][0]); x[u][1] = fma(a1, b[u][1], x[u][1]); }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(x[u], a0, b[u][0]);
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(x[u], a1, b[u][1]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u <= i)
            *reinterpret_cast<double2*>(S + r * SLD + 8 * (j0 + u) + 2 * tg) = make_double2(x[u][0] * 0.5, x[u][1] * 0.5);
      }
    }
    if (NW > 1) asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
  }
  long long t1 = clock64();
  out[tid] = S[tid] + acc4;
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = units; }
}
template <int MODE, int NW>
void run(const char* name) {
  double* out; long long* cyc;
  cudaMalloc(&out, 256 * 8); cudaMallocManaged(&cyc, 16);
  const int sm = BLK * SLD * 8;
  cudaFuncSetAttribute(k<MODE, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int r = 0; r < 2; ++r) { k<MODE, NW><<<1, 32 * NW, sm>>>(out, cyc); cudaDeviceSynchronize(); }
  printf("%-28s warps %d: %lld cycles, warp 0 ran %lld units (%.0f cycles per unit)\n", name, NW, cyc[0], cyc[1], (double)cyc[0] / cyc[1]);
}
int main() {
  run<0, 1>("DMMA, shared operands");
  run<0, 7>("DMMA, shared operands");
  run<1, 7>("DFMA, shared operands");
  run<2, 7>("DMMA, register operands");
  run<2, 1>("DMMA, register operands");
  run<3, 7>("skeleton");
  run<3, 1>("skeleton");
  run<4, 7>("loads only");
  run<4, 1>("loads only");
  return 0;
}
