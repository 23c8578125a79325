// Dense <-> tile layout conversion (tile_matrix.py:84-119 on the device).
//
// Device tile store: every lower tile (i >= j) of the matrix is a contiguous
// row-major bp x bp FP64 slot, bp = b rounded up to the 128 block. Padding is
// closed under every kernel of the inversion: off-diagonal tiles pad with 0,
// diagonal tiles pad with the identity.
//
// put: destination-driven copy of the real b x b part, pad filled.
// get: destination-driven gather into a dense row-major matrix; mode LOWER
// writes the lower tiles verbatim (to_dense on authoritative tiles), mode
// SYMMETRIZE writes the full matrix with the upper triangle mirrored from the
// lower one (symmetrize_lower(to_dense(tm)), tile_matrix.py:117-119), 64x64
// sub-blocks staged through shared memory (16-byte loads and stores).
// Both are HBM-bound: 8 bytes read + 8 written per element moved.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tinv_internal.h"

namespace tinv {

__device__ __forceinline__ void tri_decode(int64_t x, int& i, int& j) {
  int64_t r = (int64_t)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
  while (r * (r + 1) / 2 > x) --r;
  while ((r + 1) * (r + 2) / 2 <= x) ++r;
  i = (int)r;
  j = (int)(x - r * (r + 1) / 2);
}

// grid.x: lower tiles tri_lo .. tri_lo + gridDim.x - 1; grid.y: 8-row groups of bp
// src: dense rows starting at global row `row0`
// batched stores: tile x belongs to matrix x / T1 (matrices `mstride` doubles apart)
__global__ void __launch_bounds__(256) k_put(const double* __restrict__ src, int64_t lda, int64_t row0,
                                            double* __restrict__ pool, int64_t slot_elems,
                                            const int32_t* __restrict__ slot_of, int b, int bp, int64_t tri_lo,
                                            int64_t T1, int64_t mstride) {
  int i, j;
  const int64_t x = tri_lo + blockIdx.x;
  const int64_t m = x / T1;
  tri_decode(x - m * T1, i, j);
  if (slot_of[x] < 0) return;  // a partitioned store: another rank's tile
  double* dst = pool + (int64_t)slot_of[x] * slot_elems;
  const int rr = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (rr >= bp) return;
  const double* srow = src + m * mstride + ((int64_t)i * b + rr - row0) * lda + (int64_t)j * b;
  double* drow = dst + (int64_t)rr * bp;
  for (int cc = threadIdx.x & 31; cc < bp; cc += 32) {
    double v;
    if (rr < b && cc < b)
      v = __ldg(srow + cc);
    else
      v = (i == j && rr == cc) ? 1.0 : 0.0;
    drow[cc] = v;
  }
}

// One 64x64 destination sub-block per CTA (256 threads, 16 elements each):
// the source sub-block is read row-wise with 16-byte loads into shared memory
// and written row-wise with 16-byte stores, read back transposed for the
// mirrored (upper) part. grid.x: destination tiles; for panel gathers the tile
// row I is fixed (`panel_i` >= 0) and J = blockIdx.x; otherwise (I, J)
// enumerates the lower tiles (LOWER) or the full t x t grid (SYMMETRIZE).
// grid.y: sub-block index. `vec`: b, bp and ldd even (16-byte alignment).
template <int GSB, int NT>
__global__ void __launch_bounds__(NT) k_get(double* __restrict__ dst, int64_t ldd, int64_t row0,
                                            const double* __restrict__ pool, int64_t slot_elems,
                                            const int32_t* __restrict__ slot_of, int b, int bp, int t,
                                            int panel_i, int64_t tile_lo, int symmetrize, int64_t T1,
                                            int64_t mstride, int vec) {
  extern __shared__ double sm_raw[];
  double (*sm)[GSB + 1] = reinterpret_cast<double (*)[GSB + 1]>(sm_raw);
  constexpr int HP = GSB / 2;             // column pairs per row
  constexpr int NIT = GSB * HP / NT;      // pairs per thread
  int I, J;
  int64_t m = 0;
  if (panel_i >= 0) {
    I = panel_i;
    J = (int)(tile_lo + blockIdx.x);
  } else if (symmetrize == 1) {
    const int64_t x = tile_lo + blockIdx.x;
    m = x / ((int64_t)t * t);
    const int64_t loc = x - m * t * t;
    I = (int)(loc / t);
    J = (int)(loc % t);
  } else {  // LOWER, or MIRROR (2: lower tiles, each sub-block also written transposed into tile (J, I))
    const int64_t x = tile_lo + blockIdx.x;
    m = x / T1;
    tri_decode(x - m * T1, I, J);
  }
  dst += m * mstride;
  const int nsb = (b + GSB - 1) / GSB;
  const int sr = blockIdx.y / nsb, sc = blockIdx.y % nsb;
  const int tid = threadIdx.x;
  const bool mirror = symmetrize == 2;
  if (mirror && I == J && sr < sc) return;  // written as the mirror of sub-block (sc, sr)
  // source tile and whether the sub-block is read transposed
  bool transp;
  int si, sj;
  if (I > J) {
    transp = false;
    si = I;
    sj = J;
  } else if (I < J) {
    transp = true;
    si = J;
    sj = I;
  } else {
    si = sj = I;
    transp = symmetrize && (sr < sc);
  }
  const int32_t src_slot = slot_of[m * T1 + (int64_t)si * (si + 1) / 2 + sj];
  if (src_slot < 0) return;  // a partitioned store: another rank's tile (destination left as is)
  const double* tile = pool + (int64_t)src_slot * slot_elems;
  const int br = transp ? sc : sr, bc = transp ? sr : sc;  // source sub-block
  if (vec) {
#pragma unroll 8
    for (int u = 0; u < NIT; ++u) {
      const int idx = tid + NT * u, k = idx / HP, c2 = 2 * (idx % HP);
      const int r = br * GSB + k, c = bc * GSB + c2;
      double2 v = make_double2(0.0, 0.0);
      if (r < b && c < b) v = __ldcs(reinterpret_cast<const double2*>(tile + (int64_t)r * bp + c));
      sm[k][c2] = v.x;
      sm[k][c2 + 1] = v.y;
    }
  } else {
    for (int idx = tid; idx < GSB * GSB; idx += NT) {
      const int k = idx / GSB, cc = idx % GSB, r = br * GSB + k, c = bc * GSB + cc;
      sm[k][cc] = (r < b && c < b) ? tile[(int64_t)r * bp + c] : 0.0;
    }
  }
  __syncthreads();
  const bool diag_mix = symmetrize && I == J && sr == sc;
  if (mirror && !diag_mix) {  // the transposed copy into tile (J, I), sub-block (sc, sr)
    if (vec) {
      // a warp covers two destination rows (k) x 16 column pairs: its column
      // reads sm[c2][k], sm[c2 + 1][k] (row stride 65) then hit 16 distinct
      // 8-byte banks per half warp (32 pairs of one row: 2-way conflicts)
#pragma unroll 8
      for (int u = 0; u < NIT; ++u) {
        constexpr int WPR = HP / 16;  // warps per pair of destination rows
        const int idx = tid + NT * u, w = idx >> 5, l = idx & 31;
        const int k = 2 * (w / WPR) + (l & 1), c2 = 2 * ((l >> 1) + 16 * (w % WPR));
        const int r = sc * GSB + k, c = sr * GSB + c2;
        if (r >= b || c >= b) continue;
        *reinterpret_cast<double2*>(dst + ((int64_t)J * b + r - row0) * ldd + (int64_t)I * b + c) =
            make_double2(sm[c2][k], sm[c2 + 1][k]);
      }
    } else {
      for (int idx = tid; idx < GSB * GSB; idx += NT) {
        const int k = idx / GSB, cc = idx % GSB, r = sc * GSB + k, c = sr * GSB + cc;
        if (r >= b || c >= b) continue;
        dst[((int64_t)J * b + r - row0) * ldd + (int64_t)I * b + c] = sm[cc][k];
      }
    }
  }
  auto val = [&](int k, int cc) -> double {  // destination element (k, cc) of the sub-block
    if (diag_mix) return cc <= k ? sm[k][cc] : sm[cc][k];
    return transp ? sm[cc][k] : sm[k][cc];
  };
  if (vec) {
#pragma unroll 8
    for (int u = 0; u < NIT; ++u) {
      const int idx = tid + NT * u, k = idx / HP, c2 = 2 * (idx % HP);
      const int r = sr * GSB + k, c = sc * GSB + c2;  // destination element within tile (I, J)
      if (r >= b || c >= b) continue;
      *reinterpret_cast<double2*>(dst + ((int64_t)I * b + r - row0) * ldd + (int64_t)J * b + c) =
          make_double2(val(k, c2), val(k, c2 + 1));
    }
  } else {
    for (int idx = tid; idx < GSB * GSB; idx += NT) {
      const int k = idx / GSB, cc = idx % GSB, r = sr * GSB + k, c = sc * GSB + cc;
      if (r >= b || c >= b) continue;
      dst[((int64_t)I * b + r - row0) * ldd + (int64_t)J * b + c] = val(k, cc);
    }
  }
}

cudaError_t launch_put(const double* src, int64_t lda, int64_t row0, double* pool, int64_t slot_elems,
                       const int32_t* slot_of, int b, int bp, int64_t tri_lo, int64_t ntiles, cudaStream_t st,
                       int64_t T1, int64_t mstride) {
  if (ntiles <= 0) return cudaSuccess;
  dim3 grid((unsigned)ntiles, (unsigned)((bp + 7) / 8));
  k_put<<<grid, 256, 0, st>>>(src, lda, row0, pool, slot_elems, slot_of, b, bp, tri_lo, T1, mstride);
  return cudaGetLastError();
}

cudaError_t launch_get(double* dst, int64_t ldd, int64_t row0, const double* pool, int64_t slot_elems,
                       const int32_t* slot_of, int b, int bp, int t, int panel_i, int64_t tile_lo,
                       int64_t ntiles, int symmetrize, cudaStream_t st, int64_t T1, int64_t mstride) {
  if (ntiles <= 0) return cudaSuccess;
  const int vec = ((ldd | b | bp | row0) & 1) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
                  ((mstride & 1) == 0);
  // (128x128 sub-blocks -- 1 KB row segments, 132 KB of shared memory, one CTA per SM -- measured
  // 2.37 ms against 2.30 ms for 64x64 at C3)
  constexpr int G = 64, NT = 256;
  const int nsb = (b + G - 1) / G;
  dim3 grid((unsigned)ntiles, (unsigned)(nsb * nsb));
  k_get<G, NT><<<grid, NT, G * (G + 1) * 8, st>>>(dst, ldd, row0, pool, slot_elems, slot_of, b, bp, t, panel_i, tile_lo,
                                                  symmetrize, T1, mstride, vec);
  return cudaGetLastError();
}

// Padding only (streamed arrivals copy the b x b part): rows / columns >= b
// of every lower tile slot; identity on diagonal tiles, zero elsewhere.
__global__ void __launch_bounds__(256) k_pad(double* __restrict__ pool, int64_t slot_elems,
                                            const int32_t* __restrict__ slot_of, int b, int bp, int64_t T1) {
  int i, j;
  const int64_t x = blockIdx.x;
  tri_decode(x % T1, i, j);
  if (slot_of[x] < 0) return;
  double* dst = pool + (int64_t)slot_of[x] * slot_elems;
  const int rr = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (rr >= bp) return;
  double* drow = dst + (int64_t)rr * bp;
  for (int cc = (rr < b ? b : 0) + (threadIdx.x & 31); cc < bp; cc += 32)
    drow[cc] = (i == j && rr == cc) ? 1.0 : 0.0;
}

cudaError_t launch_pad(double* pool, int64_t slot_elems, const int32_t* slot_of, int b, int bp, int64_t ntiles,
                       int64_t T1, cudaStream_t st) {
  if (ntiles <= 0 || b == bp) return cudaSuccess;
  dim3 grid((unsigned)ntiles, (unsigned)((bp + 7) / 8));
  k_pad<<<grid, 256, 0, st>>>(pool, slot_elems, slot_of, b, bp, T1);
  return cudaGetLastError();
}

// D2D copy of whole slots (snapshot / restore for TINV_KEEP_ON_FAILURE)
__global__ void k_copy_slots(double* pool, int64_t slot_elems, const int32_t* from, const int32_t* to) {
  const double2* s = reinterpret_cast<const double2*>(pool + (int64_t)from[blockIdx.y] * slot_elems);
  double2* d = reinterpret_cast<double2*>(pool + (int64_t)to[blockIdx.y] * slot_elems);
  const int64_t n2 = slot_elems / 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x)
    d[e] = s[e];
}

cudaError_t launch_copy_slots(double* pool, int64_t slot_elems, const int32_t* from, const int32_t* to,
                              int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  for (int64_t off = 0; off < n; off += 65535) {
    const int64_t cnt = (n - off) < 65535 ? (n - off) : 65535;
    dim3 grid(8, (unsigned)cnt);
    k_copy_slots<<<grid, 256, 0, st>>>(pool, slot_elems, from + off, to + off);
  }
  return cudaGetLastError();
}

}  // namespace tinv
