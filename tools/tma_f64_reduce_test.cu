// Runtime check: TMA reduce-add (cp.reduce.async.bulk.tensor .add) on an FP64
// tensor map, 128B swizzle, box {16, 64}: global C += staged values.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int x0, int y0) {
  __shared__ __align__(1024) double s[64 * 16];
  for (int e = threadIdx.x; e < 64 * 16; e += blockDim.x) {
    int r = e / 16, c = e % 16;  // logical (row, col) -> swizzled position
    int chunk = (c >> 1) ^ (r & 7);
    s[r * 16 + chunk * 2 + (c & 1)] = 1000.0 * r + c + 0.25;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];"
                 :: "l"(reinterpret_cast<uint64_t>(&m)), "r"((uint32_t)__cvta_generic_to_shared(s)), "r"(x0), "r"(y0), "r"(1) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  const int bp = 128, slots = 3;
  std::vector<double> h((size_t)slots * bp * bp);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)(i % 7) * 0.5;
  double* d; cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {bp, bp, slots}, str[2] = {bp * 8, bp * bp * 8};
  cuuint32_t box[3] = {16, 64, 1}, es[3] = {1, 1, 1};
  CUresult r = ((EncFn)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(m, 32, 64);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<double> o(h.size());
  cudaMemcpy(o.data(), d, o.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0, checked = 0;
  for (int rr = 0; rr < bp; ++rr)
    for (int cc = 0; cc < bp; ++cc) {
      size_t i = (size_t)1 * bp * bp + rr * bp + cc;
      double exp = h[i];
      if (rr >= 64 && rr < 128 && cc >= 32 && cc < 48) exp += 1000.0 * (rr - 64) + (cc - 32) + 0.25;
      ++checked;
      if (o[i] != exp) { if (bad < 5) printf("mismatch r%d c%d got %f exp %f\n", rr, cc, o[i], exp); ++bad; }
    }
  printf("f64 TMA reduce-add: %s (%d/%d bad)\n", bad ? "FAIL" : "OK", bad, checked);
  return 0;
}
