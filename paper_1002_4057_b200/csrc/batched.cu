// Batched small SPD inversions (BASELINE config 4: 8192 independent n = 256
// matrices), one thread block per matrix.
//
// With nb = n the reference's stream is gen_inversion(1) = POTRF -> TRTRI ->
// LAUUM on a single tile (taskgen.py:178-223 at t = 1; kernels.py:59-76,
// 120-130, 148-151). Running that through the DAG executor spends most of the
// time in queue round trips and in 128x128 diagonal chains that hold a whole
// SM. Here the three steps of one matrix are fused into one CTA that walks a
// fixed program of 64x64 block operations:
//
//   step 1 (POTRF, right-looking over 64-wide panels p):
//     DIAG p      L_pp = chol(A_pp), Linv_pp = L_pp^-1     (smem, warp chains)
//     TRSM i>p    L_ip = A_ip Linv_pp^T                    (DMMA, triangular K)
//     UPD  i>=j>p A_ij -= L_ip L_jp^T                      (DMMA)
//   step 2 (TRTRI, column j, row i > j):
//     T = sum_{k=j}^{i-1} L_ik X_kj ;  X_ij = -X_ii T      (X_jj = Linv_jj from DIAG)
//   step 3 (LAUUM, row i, column j <= i):
//     W_ij = sum_{k>=i} X_ki^T X_kj, written with its mirror (full symmetric
//     output = symmetrize_lower(to_dense(...)), tile_matrix.py:102-119)
//
// The matrix itself is the working store (X's lower blocks, L2-resident while
// the CTA works on it). Operand blocks are staged with cp.async in two 32 KB
// shared-memory buffers that remember which block they hold (an operand the
// previous operation already loaded is not reloaded). Each CTA has 4 warps and
// ~66 KB of shared memory, so three matrices are resident per SM: one CTA's
// exposed loads and latency-bound diagonal chains overlap the others' DMMA
// work. Each warp owns four 16x16 output quads chosen (c_map) so that the
// triangular K ranges of TRSM / TRMM / SYRK-type products balance over warps.
//
// Products run on the FP64 tensor pipe (mma.sync m8n8k4 -> DMMA.8x8x4; there
// is no f64 tcgen05 kind on sm_100a). Smem blocks are 64x64 row-major with an
// XOR swizzle (column ^ 4 * (row & 3)) that makes every m8n8k4 fragment load
// -- row- or column-oriented -- hit 16 distinct 8-byte bank pairs per half warp.
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <string>

#include "tinv_internal.h"

namespace tinv {
int set_error(int code, const std::string& msg);

namespace bsm {

constexpr int BB = 64;            // block order
constexpr int NT = 128;           // 4 warps; 3 CTAs per SM
constexpr int NBMAX = 4;          // n <= 256
constexpr int MAXOPS = 56;        // program length for nbk = 4
constexpr int BUFD = BB * BB;     // doubles per smem block buffer
constexpr int SMEM_DYN = 2 * BUFD * 8;  // two block buffers

enum : int8_t { OP_DIAG = 1, OP_MMA = 2 };
// K range of a triangular operand per 16x16 output quad (qr, qc):
// LT_COL k < 16(qc+1), LT_ROW k < 16(qr+1), GE_COL k >= 16 qc, GE_ROW k >= 16 qr,
// GE_BOTH k >= 16 max(qr, qc)
enum : int8_t { KR_FULL, KR_LT_COL, KR_LT_ROW, KR_GE_COL, KR_GE_ROW, KR_GE_BOTH };
enum : int8_t { ST_NONE = 0, ST_FULL = 1, ST_LOWER = 2, ST_SYM = 3 };
enum : int8_t { F_ZERO = 1, F_NEGC = 2, F_SKIPU = 8, F_TA = 16, F_TB = 32 };

// One block operation; arrays: 0 = A (input), 1 = X (working store / output).
struct BOp {
  int8_t type, flags, kr, st;
  int8_t aa, ai, aj, ba;
  int8_t bi, bj, ca, ci;
  int8_t cj, oi, oj, sg;
  int8_t map, pad0, pad1, pad2;
};

// Output quads (16x16) of a warp; every operation of an accumulation chain
// uses the chain's map (see c_map).
enum : int8_t { MAP_COL = 0, MAP_ROW = 1, MAP_LOWER = 2 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ int sw(int r, int c) { return r * BB + (c ^ ((r & 3) << 2)); }
__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- program
__host__ __device__ int gen_program(BOp* ops, int nb) {
  int k = 0;
  auto mma = [&](int aa, int ai, int aj, int ba, int bi, int bj, int flags, int kr, int st, int oi, int oj, int sg,
                 int ca = 0, int ci = 0, int cj = 0) {
    BOp o;
    o.type = OP_MMA;
    o.flags = (int8_t)flags;
    o.kr = (int8_t)kr;
    o.st = (int8_t)st;
    o.aa = (int8_t)aa, o.ai = (int8_t)ai, o.aj = (int8_t)aj;
    o.ba = (int8_t)ba, o.bi = (int8_t)bi, o.bj = (int8_t)bj;
    o.ca = (int8_t)ca, o.ci = (int8_t)ci, o.cj = (int8_t)cj;
    o.oi = (int8_t)oi, o.oj = (int8_t)oj, o.sg = (int8_t)sg;
    o.map = (flags & F_SKIPU) ? MAP_LOWER : (kr == KR_LT_ROW || kr == KR_GE_ROW) ? MAP_ROW : MAP_COL;
    o.pad0 = o.pad1 = o.pad2 = 0;
    ops[k++] = o;
  };
  // step 1: Cholesky (POTRF), right-looking over 64-wide panels
  for (int p = 0; p < nb; ++p) {
    const int src = p ? 1 : 0;
    BOp d = {};
    d.type = OP_DIAG;
    d.aa = (int8_t)src, d.ai = (int8_t)p, d.aj = (int8_t)p, d.oi = (int8_t)p, d.oj = (int8_t)p;
    ops[k++] = d;
    for (int i = p + 1; i < nb; ++i)  // L_ip = A_ip Linv_pp^T
      mma(src, i, p, 1, p, p, F_ZERO | F_TB, KR_LT_COL, ST_FULL, i, p, 1);
    for (int i = p + 1; i < nb; ++i)  // A_ij -= L_ip L_jp^T
      for (int j = p + 1; j <= i; ++j)
        mma(1, i, p, 1, j, p, F_NEGC | F_TB | (i == j ? F_SKIPU : 0), KR_FULL, i == j ? ST_LOWER : ST_FULL, i, j,
            -1, src, i, j);
  }
  // step 2: X = L^-1 (TRTRI); X_jj = Linv_jj already in place
  for (int j = 0; j + 1 < nb; ++j)
    for (int i = j + 1; i < nb; ++i) {
      for (int q = j; q < i; ++q)  // T = sum_q L_iq X_qj (X_jj lower: K >= column)
        mma(1, i, q, 1, q, j, q == j ? F_ZERO : 0, q == j ? KR_GE_COL : KR_FULL, q == i - 1 ? ST_FULL : ST_NONE,
            i, j, 1);
      mma(1, i, i, 1, i, j, F_ZERO, KR_LT_ROW, ST_FULL, i, j, -1);  // X_ij = -X_ii T
    }
  // step 3: A^-1 = X^T X (LAUUM), lower blocks with their mirrors
  // (chains of one row i alternate the q direction: the first operand pair of
  // the next chain, X(q, i) with the q the previous chain ended on, is still
  // in shared memory)
  for (int i = 0; i < nb; ++i)
    for (int j = 0; j <= i; ++j)
      for (int s = 0; s < nb - i; ++s) {
        const int q = (j & 1) ? nb - 1 - s : i + s;
        mma(1, q, i, 1, q, j, F_TA | (s == 0 ? F_ZERO : 0) | (i == j ? F_SKIPU : 0),
            q == i ? (j == i ? KR_GE_BOTH : KR_GE_ROW) : KR_FULL, s == nb - i - 1 ? ST_SYM : ST_NONE, i, j, 1);
        if (i != j) ops[k - 1].map = MAP_ROW;  // the chain's map (its q == i operation is GE_ROW)
      }
  return k;
}

// the block programs for nb = 1..4, generated on the host once per device (a
// per-CTA gen_program put ~1100 instructions in front of every matrix)
__constant__ BOp c_prog[NBMAX][MAXOPS];
__constant__ int c_nops[NBMAX];

// ---------------------------------------------------------------- DMMA quad product
// acc (16x16 quad at rows 16 qr.., cols 16 qc..; 2x2 m8n8 tiles) +=
// sum_{k0 <= k < k1} A(r, k) B(k, c); A(r, k) = SA[r][k] (SA[k][r] if TA),
// B(k, c) = SB[k][c] (SB[c][k] if TB). k0, k1 multiples of 16.
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

// ---------------------------------------------------------------- diagonal block
// Cholesky of the lower 8x8 block at (p0, p0) of S in registers (right-looking;
// kernels.py:68-71 failure test: not d > 0, or d non-finite) and the inverse of
// the factor: x = L^-1 (lower; x[i][i] = 1 / L[i][i]). Returns the first
// failing pivot or -1.
__device__ __forceinline__ int chol8_inv(const double* S, int p0, double (&x)[8][8]) {
  double l[8][8], il[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) l[i][j] = S[sw(p0 + i, p0 + j)];
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

// One warp: 8x8 tile D(i, j) = sgn * sum_{k < K} A(i, k) B(k, j).
template <class FA, class FB, class FD>
__device__ __forceinline__ void tile8(FA A, FB B, FD D, int K, double sgn) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  double acc[2] = {0.0, 0.0};
  for (int k = 0; k < K; k += 4) dmma(acc, A(g, k + tg), B(k + tg, g));
  D(g, 2 * tg, sgn * acc[0]);
  D(g, 2 * tg + 1, sgn * acc[1]);
}

// ---------------------------------------------------------------- kernel pieces
__device__ __forceinline__ int tagof(int arr, int i, int j) { return 1 + ((arr << 8) | (i << 4) | j); }

// Three CTAs per SM, 4 warps each, two 32 KB block buffers (no scratch: the
// TRTRI products stage through the zero upper triangle of the inverse). Each
// warp owns four 16x16 output quads; with three matrices resident per SM one
// CTA's exposed loads and diagonal chains overlap the others' DMMA work.
// quads (qr << 2 | qc) of warp w: MAP_COL = quad row w, MAP_ROW = quad column
// w, MAP_LOWER = the 10 lower quads (K >= 16 qr work per warp 6,6,6,2 x16)
__constant__ int8_t c_map[3][4][4] = {
    {{0, 1, 2, 3}, {4, 5, 6, 7}, {8, 9, 10, 11}, {12, 13, 14, 15}},
    {{0, 4, 8, 12}, {1, 5, 9, 13}, {2, 6, 10, 14}, {3, 7, 11, 15}},
    {{0, 12, 13, -1}, {4, 5, -1, -1}, {8, 9, 10, -1}, {14, 15, -1, -1}},
};

__device__ __forceinline__ void load_blk(double* S, const double* G, int n, int bi, int bj) {
  const int r0 = bi * BB, c0 = bj * BB;
  if ((n & 1) == 0) {
#pragma unroll 4
    for (int u = 0; u < 16; ++u) {
      const int idx = threadIdx.x + NT * u, r = idx >> 5, c = (idx & 31) * 2;
      const bool ok = r0 + r < n && c0 + c < n;
      cp16(S + sw(r, c), ok ? G + (int64_t)(r0 + r) * n + c0 + c : G, ok ? 16 : 0);
    }
  } else {
    for (int e = threadIdx.x; e < BUFD; e += NT) {
      const int r = e >> 6, c = e & 63;
      S[sw(r, c)] = (r0 + r < n && c0 + c < n) ? G[(int64_t)(r0 + r) * n + c0 + c] : 0.0;
    }
  }
  cp_commit();
}

// Row block R of X = L^-1 by bordering (warp wl of nw, 8x8 tiles c < R):
// X_Rc = -X_RR (sum_{k=c}^{R-1} L_Rk X_kc). Needs L's row block R (final once
// panels < R are done), X's rows < R and X_RR. The partial sum is staged in
// X's strictly upper block (c, R) (zero in the result) and cleared after use.
__device__ __forceinline__ void border_row(const double* S, double* X, int R, int wl, int nw) {
  const int lane = threadIdx.x & 31;
  for (int c = wl; c < R; c += nw) {
    const int r0 = 8 * R, c0 = 8 * c;
    tile8([&](int i, int k) { return S[sw(r0 + i, c0 + k)]; }, [&](int k, int j) { return X[sw(c0 + k, c0 + j)]; },
          [&](int i, int j, double v) { X[sw(c0 + i, r0 + j)] = v; }, 8 * (R - c), 1.0);
    __syncwarp();
    tile8([&](int i, int k) { return X[sw(r0 + i, r0 + k)]; }, [&](int k, int j) { return X[sw(c0 + k, r0 + j)]; },
          [&](int i, int j, double v) { X[sw(r0 + i, c0 + j)] = v; }, 8, -1.0);
    __syncwarp();
    for (int e = lane; e < 64; e += 32) X[sw(c0 + (e >> 3), r0 + (e & 7))] = 0.0;
  }
}

// In-place Cholesky of the lower 64x64 block in S (8-wide panels, 4 warps)
// and X = L^-1: warps 0-1 factor the panel's 8x8 diagonal block in registers
// (its inverse -> X's diagonal) and solve the panel rows below it, while
// warps 2-3 border X with the previous row block; then all warps update the
// trailing lower 8x8 tiles on DMMA. X is zeroed here; S's strict upper part
// must be zero on entry (its 8x8 diagonal blocks are left unfactored: only
// the off-diagonal factor blocks and L^-1 are used).
__device__ void factor64(double* S, double* X, int* fail) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tg = lane & 3;
  for (int e = tid; e < BUFD; e += NT) X[e] = 0.0;
  __syncthreads();
  for (int P = 0; P < 8; ++P) {
    const int p0 = 8 * P;
    if (warp < 2) {
      double x[8][8];
      const int bad = chol8_inv(S, p0, x);
      if (tid == 0) {
        if (bad >= 0) atomicMin(fail, p0 + bad);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) X[sw(p0 + i, p0 + j)] = x[i][j];
      }
      const int q = p0 + 8 + tid;
      if (q < BB) {
        double a[8], v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = S[sw(q, p0 + k)];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k <= c; ++k) t = fma(a[k], x[c][k], t);
          v[c] = t;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) S[sw(q, p0 + k)] = v[k];
      }
    } else if (P >= 2) {
      border_row(S, X, P - 1, warp - 2, 2);  // row block P - 1 of the inverse
    }
    __syncthreads();
    if (P == 7) break;
    const int t0r = p0 + 8, nt8 = 7 - P, ntiles = nt8 * (nt8 + 1) / 2;
    for (int tt = warp; tt < ntiles; tt += NT / 32) {
      int ti = 0, rem = tt;
      while (rem > ti) {
        rem -= ti + 1;
        ++ti;
      }
      const int r0 = t0r + 8 * ti, c0 = t0r + 8 * rem;
      double acc[2] = {S[sw(r0 + g, c0 + 2 * tg)], S[sw(r0 + g, c0 + 2 * tg + 1)]};
#pragma unroll
      for (int k = 0; k < 8; k += 4) dmma(acc, -S[sw(r0 + g, p0 + k + tg)], S[sw(c0 + g, p0 + k + tg)]);
      S[sw(r0 + g, c0 + 2 * tg)] = acc[0];
      S[sw(r0 + g, c0 + 2 * tg + 1)] = acc[1];
    }
    __syncthreads();
  }
  border_row(S, X, 7, warp, NT / 32);  // the last row block
  __syncthreads();
}


template <bool PROF>
__global__ void __launch_bounds__(NT, 3)
    k_bsmall(const double* __restrict__ A, double* X, int n, int nb, int64_t mstride, unsigned long long* fail,
              int64_t id0, unsigned long long* prof) {
  extern __shared__ __align__(128) double dsm[];
  __shared__ int sfail;
  const BOp* ops = c_prog[nb - 1];
  const int64_t mat = blockIdx.x;
  const double* const a = A + mat * mstride;
  double* const x = X + mat * mstride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tg = lane & 3;
  if (tid == 0) sfail = 1 << 30;
  __syncthreads();
  const int nop = c_nops[nb - 1];
  auto buf = [&](int b) { return dsm + b * BUFD; };
  auto base = [&](int arr) -> const double* { return arr ? x : a; };
  int tag0 = 0, tag1 = 0;  // global block held by buffer 0 / 1 (0: none)
  double acc[4][2][2][2];
  long long pt = 0, pacc[8] = {};
  auto probe = [&](int c) {
    if constexpr (PROF) {
      const long long now = clock64();
      if (c >= 0) pacc[c] += now - pt;
      pt = now;
    }
  };
  probe(-1);
  for (int o = 0; o < nop; ++o) {
    const BOp op = ops[o];
    if (op.type == OP_DIAG) {
      __syncthreads();
      double* S = buf(0);
      double* Xs = buf(1);
      const int p = op.ai, gr = p * BB;
      load_blk(S, base(op.aa), n, p, p);
      cp_wait_all();
      __syncthreads();
      probe(0);
      for (int e = tid; e < BUFD; e += NT) {  // lower part only; identity on the padded diagonal
        const int r = e >> 6, c = e & 63;
        if (c > r) S[sw(r, c)] = 0.0;
        else if (c == r && gr + r >= n) S[sw(r, c)] = 1.0;
      }
      __syncthreads();
      factor64(S, Xs, &sfail);
      if (sfail < (1 << 30)) {
        if (tid == 0) atomicMin(fail, ((unsigned long long)(id0 + mat) << 32) | (unsigned)(gr + sfail));
        return;
      }
      if ((n & 1) == 0) {  // X_pp = Linv_pp -> global, 16-byte stores
        for (int e = tid; e < BUFD / 2; e += NT) {
          const int r = e >> 5, c = 2 * (e & 31);
          if (gr + r < n && gr + c < n)
            *reinterpret_cast<double2*>(x + (int64_t)(gr + r) * n + gr + c) =
                make_double2(Xs[sw(r, c)], Xs[sw(r, c + 1)]);
        }
      } else {
        for (int e = tid; e < BUFD; e += NT) {
          const int r = e >> 6, c = e & 63;
          if (gr + r < n && gr + c < n) x[(int64_t)(gr + r) * n + gr + c] = Xs[sw(r, c)];
        }
      }
      tag0 = 0;
      tag1 = tagof(1, p, p);
#pragma unroll
      for (int q = 0; q < 32; ++q) (&acc[0][0][0][0])[2 * q] = (&acc[0][0][0][0])[2 * q + 1] = 0.0;
      probe(1);
      continue;
    }
    const int ta = tagof(op.aa, op.ai, op.aj), tb = tagof(op.ba, op.bi, op.bj);
    int ba = tag0 == ta ? 0 : tag1 == ta ? 1 : -1;
    int bb = tb == ta ? ba : tag0 == tb ? 0 : tag1 == tb ? 1 : -1;
    if (ba < 0 || bb < 0) {
      __syncthreads();  // the previous operation's smem reads and global stores are done
      if (ba < 0) {
        ba = bb == 0 ? 1 : 0;
        load_blk(buf(ba), base(op.aa), n, op.ai, op.aj);
        if (ba) tag1 = ta; else tag0 = ta;
        if (tb == ta) bb = ba;
      }
      if (bb < 0) {
        bb = 1 - ba;
        load_blk(buf(bb), base(op.ba), n, op.bi, op.bj);
        if (bb) tag1 = tb; else tag0 = tb;
      }
      cp_wait_all();
      __syncthreads();
    }
    probe(0);
    const double* SA = buf(ba);
    const double* SB = buf(bb);
    int quad[4];
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) quad[sl] = c_map[op.map][warp][sl];
    if (op.flags & (F_ZERO | F_NEGC)) {
#pragma unroll
      for (int q = 0; q < 32; ++q) (&acc[0][0][0][0])[2 * q] = (&acc[0][0][0][0])[2 * q + 1] = 0.0;
    }
    const int fl = op.flags & (F_TA | F_TB);
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      if (quad[sl] < 0) continue;
      const int qr = quad[sl] >> 2, qc = quad[sl] & 3;
      int k0 = 0, k1 = BB;
      switch (op.kr) {
        case KR_LT_COL: k1 = 16 * (qc + 1); break;
        case KR_LT_ROW: k1 = 16 * (qr + 1); break;
        case KR_GE_COL: k0 = 16 * qc; break;
        case KR_GE_ROW: k0 = 16 * qr; break;
        case KR_GE_BOTH: k0 = 16 * max(qr, qc); break;
        default: break;
      }
      if (fl == F_TB)
        mma_quad<false, true>(SA, SB, qr, qc, k0, k1, acc[sl]);
      else if (fl == F_TA)
        mma_quad<true, false>(SA, SB, qr, qc, k0, k1, acc[sl]);
      else
        mma_quad<false, false>(SA, SB, qr, qc, k0, k1, acc[sl]);
      if (op.flags & F_NEGC) {
        const double* C = base(op.ca);
#pragma unroll
        for (int ti = 0; ti < 2; ++ti)
#pragma unroll
          for (int tj = 0; tj < 2; ++tj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = op.ci * BB + 16 * qr + 8 * ti + g, c = op.cj * BB + 16 * qc + 8 * tj + 2 * tg + e;
              if (r < n && c < n) acc[sl][ti][tj][e] -= C[(int64_t)r * n + c];
            }
      }
    }
    probe(2);
    if (op.st == ST_NONE) continue;
    const int to = tagof(1, op.oi, op.oj);
    if (tag0 == to) tag0 = 0;  // the cached copy is stale once the block is stored
    if (tag1 == to) tag1 = 0;
    const double sg = (double)op.sg;
    const int gr = op.oi * BB, gc = op.oj * BB;
    const bool diag = op.oi == op.oj;
    // the row's two accumulator columns (2 tg, 2 tg + 1) as one 16-byte store
    const bool pair = (n & 1) == 0 && (op.st == ST_FULL || op.st == ST_LOWER || (op.st == ST_SYM && !diag));
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      if (quad[sl] < 0) continue;
      if (pair) {
#pragma unroll
        for (int ti = 0; ti < 2; ++ti)
#pragma unroll
          for (int tj = 0; tj < 2; ++tj) {
            const int r = 16 * (quad[sl] >> 2) + 8 * ti + g, c = 16 * (quad[sl] & 3) + 8 * tj + 2 * tg;
            if (gr + r >= n || gc + c >= n) continue;
            const double v0 = sg * acc[sl][ti][tj][0], v1 = sg * acc[sl][ti][tj][1];
            if (op.st == ST_LOWER && c + 1 > r) {  // on / above the diagonal: lower entries only
              if (c <= r) x[(int64_t)(gr + r) * n + gc + c] = v0;
              continue;
            }
            *reinterpret_cast<double2*>(x + (int64_t)(gr + r) * n + gc + c) = make_double2(v0, v1);
            if (op.st == ST_SYM) {
              x[(int64_t)(gc + c) * n + gr + r] = v0;
              x[(int64_t)(gc + c + 1) * n + gr + r] = v1;
            }
          }
        continue;
      }
#pragma unroll
      for (int ti = 0; ti < 2; ++ti)
#pragma unroll
        for (int tj = 0; tj < 2; ++tj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 16 * (quad[sl] >> 2) + 8 * ti + g, c = 16 * (quad[sl] & 3) + 8 * tj + 2 * tg + e;
            if (gr + r >= n || gc + c >= n) continue;
            const double v = sg * acc[sl][ti][tj][e];
            if (op.st == ST_FULL) {
              x[(int64_t)(gr + r) * n + gc + c] = v;
            } else if (op.st == ST_LOWER) {
              if (c <= r) x[(int64_t)(gr + r) * n + gc + c] = v;
            } else {
              if (diag && c > r) continue;
              x[(int64_t)(gr + r) * n + gc + c] = v;
              if (!(diag && c == r)) x[(int64_t)(gc + c) * n + gr + r] = v;
            }
          }
    }
    probe(3);
  }
  if constexpr (PROF) {
    if (tid == 0)
      for (int c = 0; c < 4; ++c) atomicAdd(prof + c, (unsigned long long)pacc[c]);
  }
}

}  // namespace bsm

cudaError_t launch_bpipe(const double* dA, double* dX, int64_t batch, int64_t n, int64_t stride, cudaStream_t st,
                         unsigned long long* dfail, int64_t id0);

cudaError_t launch_bsmall(const double* dA, double* dX, int64_t batch, int64_t n, int64_t stride, cudaStream_t st,
                          unsigned long long* dfail, int64_t id0) {
  // TINV_BSMALL_ENGINE=pipe (even 64 <= n <= 256): the pipelined persistent
  // engine of csrc/batched_pipe.cu; default: the one-CTA-per-matrix program
  // below (measured 2-3 % faster at C4, profiles/r02/c4_engines.md)
  {
    const cudaError_t e = launch_bpipe(dA, dX, batch, n, stride, st, dfail, id0);
    if (e != cudaErrorNotSupported) return e;
  }
  // TINV_BSMALL_PROF=1: per-phase clock64 spans of thread 0, printed per launch
  // (process-wide state: like a context, this entry point is not thread-safe)
  static const int prof_mode = getenv("TINV_BSMALL_PROF") && atoi(getenv("TINV_BSMALL_PROF")) ? 1 : 0;
  // TINV_BSMALL_PAD_KB: extra dynamic shared memory per CTA (a profiling knob:
  // 32 -> 2 CTAs per SM, 64 -> 1, so the phase profile shows uncontended spans)
  static const int pad_smem = getenv("TINV_BSMALL_PAD_KB") ? atoi(getenv("TINV_BSMALL_PAD_KB")) * 1024 : 0;
  static unsigned long long* dprof[64] = {};
  static uint64_t attr_set = 0;  // devices whose kernel attributes are set
  int dev = 0;
  cudaError_t r = cudaGetDevice(&dev);
  if (r != cudaSuccess) return r;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!(attr_set >> dev & 1)) {
    {
      static bsm::BOp prog[bsm::NBMAX][bsm::MAXOPS];
      int nops[bsm::NBMAX];
      for (int nb = 1; nb <= bsm::NBMAX; ++nb) nops[nb - 1] = bsm::gen_program(prog[nb - 1], nb);
      r = cudaMemcpyToSymbol(bsm::c_prog, prog, sizeof prog);
      if (r == cudaSuccess) r = cudaMemcpyToSymbol(bsm::c_nops, nops, sizeof nops);
      if (r != cudaSuccess) return r;
    }
    r = cudaFuncSetAttribute(bsm::k_bsmall<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             bsm::SMEM_DYN + pad_smem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(bsm::k_bsmall<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               bsm::SMEM_DYN + pad_smem);
    if (r == cudaSuccess && prof_mode) r = cudaMalloc(&dprof[dev], 4 * sizeof(unsigned long long));
    if (r != cudaSuccess) return r;
    attr_set |= 1ull << dev;
  }
  const int nb = (int)((n + bsm::BB - 1) / bsm::BB);
  if (prof_mode) cudaMemsetAsync(dprof[dev], 0, 4 * sizeof(unsigned long long), st);
  for (int64_t b0 = 0; b0 < batch; b0 += 0x7fffffff) {
    const int64_t cnt = batch - b0 < 0x7fffffff ? batch - b0 : 0x7fffffff;
    if (prof_mode)
      bsm::k_bsmall<true><<<(unsigned)cnt, bsm::NT, bsm::SMEM_DYN + pad_smem, st>>>(dA + b0 * stride, dX + b0 * stride, (int)n,
                                                                         nb, stride, dfail, id0 + b0, dprof[dev]);
    else
      bsm::k_bsmall<false><<<(unsigned)cnt, bsm::NT, bsm::SMEM_DYN + pad_smem, st>>>(dA + b0 * stride, dX + b0 * stride, (int)n,
                                                                          nb, stride, dfail, id0 + b0, nullptr);
  }
  if (prof_mode) {
    unsigned long long h[4];
    cudaMemcpyAsync(h, dprof[dev], sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[tinv bsmall] cycles per matrix: wait %.0f diag %.0f mma %.0f store %.0f\n", (double)h[0] / batch,
            (double)h[1] / batch, (double)h[2] / batch, (double)h[3] / batch);
  }
  return cudaGetLastError();
}

}  // namespace tinv

using namespace tinv;

extern "C" {

int tinv_batch_small_launch(const double* dA, double* dX, int64_t batch, int64_t n, int64_t stride,
                            void* cuda_stream, unsigned long long* dfail) {
  if (!dA || !dX || !dfail) return set_error(TINV_ERR_BAD_ARG, "null pointer");
  if (batch < 0 || n < 1 || n > bsm::NBMAX * bsm::BB || stride < n * n)
    return set_error(TINV_ERR_BAD_ARG, "batched small inversion needs 1 <= n <= 256 and stride >= n*n");
  // even n: the engine moves matrix rows with 16-byte accesses (cp.async and
  // double2 stores at A/X + k*stride), so the bases must be 16-byte aligned and
  // the stride even -- a misaligned access would be a sticky context fault
  if ((n & 1) == 0 && (((uintptr_t)dA | (uintptr_t)dX) & 15 || (stride & 1)))
    return set_error(TINV_ERR_BAD_ARG, "batched small inversion with even n needs 16-byte aligned A/X and an even stride");
  if (batch == 0) return TINV_OK;
  const cudaError_t e = launch_bsmall(dA, dX, batch, n, stride, (cudaStream_t)cuda_stream, dfail, 0);
  if (e != cudaSuccess) return set_error(TINV_ERR_CUDA, std::string("k_bsmall: ") + cudaGetErrorString(e));
  return TINV_OK;
}

// Host-buffer pipeline state, kept between calls (one per process; not
// thread-safe, like a context).
namespace {
struct BsHost {
  int device = -1;
  size_t slot_bytes = 0;
  static constexpr int NS = 3;
  double* slot[NS] = {};
  unsigned long long* dfail = nullptr;
  cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
  cudaEvent_t h2d[NS] = {}, comp[NS] = {}, d2h[NS] = {};
};
BsHost g_bs;
}  // namespace

int tinv_batch_small_host(const double* hA, double* hX, int64_t batch, int64_t n, int device, int64_t* fail_matrix,
                          int64_t* fail_index, double* ms) {
  if (fail_matrix) *fail_matrix = -1;
  if (fail_index) *fail_index = -1;
  if (!hA || !hX) return set_error(TINV_ERR_BAD_ARG, "null pointer");
  if (batch < 0 || n < 1 || n > bsm::NBMAX * bsm::BB)
    return set_error(TINV_ERR_BAD_ARG, "batched small inversion needs 1 <= n <= 256");
  if (batch == 0) return TINV_OK;
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess || device < 0 || device >= nd) {
    cudaGetLastError();
    return set_error(TINV_ERR_NO_DEVICE, "no CUDA device");
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
    return set_error(TINV_ERR_NO_DEVICE, "device is not sm_100 (B200)");
#define BCK(call)                                                                               \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) return set_error(TINV_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
  BCK(cudaSetDevice(device));
  BsHost& H = g_bs;
  const int64_t mat_bytes = n * n * 8;
  // chunks of ~TINV_BSMALL_CHUNK_MB (default 64 MB, at least one wave of CTAs):
  // PCIe time per chunk dwarfs the kernel, three slots keep both copy
  // directions busy, and small chunks shorten the pipeline's fill and drain
  static const int64_t chunk_mb = getenv("TINV_BSMALL_CHUNK_MB") ? atoll(getenv("TINV_BSMALL_CHUNK_MB")) : 64;
  int64_t chunk = std::max<int64_t>(std::max<int64_t>(1, (chunk_mb << 20) / mat_bytes), 1);
  chunk = std::min<int64_t>(chunk, batch);
  const size_t need = (size_t)(chunk * mat_bytes);
  if (H.device != device) {
    if (H.device >= 0 && cudaSetDevice(H.device) == cudaSuccess) {  // release the previous device's state
      for (int s = 0; s < BsHost::NS; ++s) {
        if (H.slot[s]) cudaFree(H.slot[s]);
        if (H.h2d[s]) cudaEventDestroy(H.h2d[s]);
        if (H.comp[s]) cudaEventDestroy(H.comp[s]);
        if (H.d2h[s]) cudaEventDestroy(H.d2h[s]);
      }
      if (H.dfail) cudaFree(H.dfail);
      for (cudaStream_t q : {H.sh, H.sc, H.sd})
        if (q) cudaStreamDestroy(q);
      BCK(cudaSetDevice(device));
    }
    H = BsHost();
    H.device = device;
    BCK(cudaStreamCreateWithFlags(&H.sh, cudaStreamNonBlocking));
    BCK(cudaStreamCreateWithFlags(&H.sc, cudaStreamNonBlocking));
    BCK(cudaStreamCreateWithFlags(&H.sd, cudaStreamNonBlocking));
    for (int s = 0; s < BsHost::NS; ++s) {
      BCK(cudaEventCreateWithFlags(&H.h2d[s], cudaEventDisableTiming));
      BCK(cudaEventCreateWithFlags(&H.comp[s], cudaEventDisableTiming));
      BCK(cudaEventCreateWithFlags(&H.d2h[s], cudaEventDisableTiming));
    }
    BCK(cudaMalloc(&H.dfail, sizeof(unsigned long long)));
  }
  if (H.slot_bytes < need) {
    for (int s = 0; s < BsHost::NS; ++s) {
      if (H.slot[s]) cudaFree(H.slot[s]);
      H.slot[s] = nullptr;
    }
    H.slot_bytes = 0;
    for (int s = 0; s < BsHost::NS; ++s) BCK(cudaMalloc(&H.slot[s], need));
    H.slot_bytes = need;
  }
  const auto t0 = std::chrono::steady_clock::now();
  BCK(cudaMemsetAsync(H.dfail, 0xff, sizeof(unsigned long long), H.sc));
  const int64_t nchunks = (batch + chunk - 1) / chunk;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int s = (int)(c % BsHost::NS);
    const int64_t m0 = c * chunk, cnt = std::min(chunk, batch - m0);
    const size_t bytes = (size_t)(cnt * mat_bytes);
    if (c >= BsHost::NS) BCK(cudaStreamWaitEvent(H.sh, H.d2h[s], 0));
    // The engine reads only A's lower 64x64 blocks (diagonal blocks whole): for
    // nb >= 2 block rows copy block row i as one 3D transfer of its first
    // 64 (i + 1) columns (n = 256: 62.5 % of the bytes; the slot's other blocks
    // keep stale data the kernel never reads). TINV_BSMALL_H2D_FULL=1: whole matrices.
    static const bool h2d_full = getenv("TINV_BSMALL_H2D_FULL") && atoi(getenv("TINV_BSMALL_H2D_FULL"));
    const int nbr = (int)((n + bsm::BB - 1) / bsm::BB);
    if (h2d_full || nbr < 2) {
      BCK(cudaMemcpyAsync(H.slot[s], hA + m0 * n * n, bytes, cudaMemcpyHostToDevice, H.sh));
    } else {
      for (int i = 0; i < nbr; ++i) {
        cudaMemcpy3DParms cp = {};
        cp.srcPtr = make_cudaPitchedPtr((void*)(hA + m0 * n * n), (size_t)n * 8, (size_t)n, (size_t)n);
        cp.dstPtr = make_cudaPitchedPtr((void*)H.slot[s], (size_t)n * 8, (size_t)n, (size_t)n);
        cp.srcPos = make_cudaPos(0, (size_t)i * bsm::BB, 0);
        cp.dstPos = cp.srcPos;
        cp.extent = make_cudaExtent((size_t)std::min<int64_t>((int64_t)(i + 1) * bsm::BB, n) * 8,
                                    (size_t)std::min<int64_t>(bsm::BB, n - (int64_t)i * bsm::BB), (size_t)cnt);
        cp.kind = cudaMemcpyHostToDevice;
        BCK(cudaMemcpy3DAsync(&cp, H.sh));
      }
    }
    BCK(cudaEventRecord(H.h2d[s], H.sh));
    BCK(cudaStreamWaitEvent(H.sc, H.h2d[s], 0));
    BCK(launch_bsmall(H.slot[s], H.slot[s], cnt, n, n * n, H.sc, H.dfail, m0));  // failure ids absolute
    BCK(cudaEventRecord(H.comp[s], H.sc));
    BCK(cudaStreamWaitEvent(H.sd, H.comp[s], 0));
    BCK(cudaMemcpyAsync(hX + m0 * n * n, H.slot[s], bytes, cudaMemcpyDeviceToHost, H.sd));
    BCK(cudaEventRecord(H.d2h[s], H.sd));
  }
  BCK(cudaStreamSynchronize(H.sd));
  BCK(cudaStreamSynchronize(H.sc));
  unsigned long long f = ~0ull;
  BCK(cudaMemcpy(&f, H.dfail, sizeof f, cudaMemcpyDeviceToHost));
  if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
#undef BCK
  if (f != ~0ull) {
    if (fail_matrix) *fail_matrix = (int64_t)(f >> 32);
    if (fail_index) *fail_index = (int64_t)(f & 0xffffffffu);
    return set_error(TINV_ERR_NOT_SPD, "matrix is not positive definite");
  }
  return TINV_OK;
}

}  // extern "C"
