// Persistent on-device task executor for the SPD tile inversion
// (B200 / sm_100a). Replaces the reference's threaded dynamic scheduler
// (scheduler.py:261-351) and its numpy tile kernels (kernels.py:59-151).
//
// One CTA per SM, 384 threads:
//   warps 0-7  "consumers": FP64 DMMA (mma.sync m8n8k4 -> SASS DMMA.8x8x4)
//              on 128x128 output blocks, epilogues staged for the storer,
//              diagonal-block phases (128x128 factor / inverse in smem);
//   warp 8     "producer": claims ready work items from the device queues,
//              builds their jobs in the item's smem slot and streams operand
//              chunks into a 4-stage shared-memory ring with TMA
//              (cp.async.bulk.tensor, 128B swizzle) on mbarriers;
//   warp 9     "storer": TMA stores / FP64 TMA reduce-adds of the staged
//              epilogues, job completion, item completion (successor release);
//   warp 10    inbox poller: completes external tasks (RECV, ARRIVE).
// A task of kind K over tiles of order bp = R*128 is split into work items
// (128x128 output blocks) which run on any CTA; the last item to finish
// releases the task's successors in the hazard DAG (RAW/WAR/WAW edges built
// by the host planner from the stream exactly as scheduler.py:101-153).
// In-place kernels whose output block depends on other blocks of the same
// tile (TRMM*, LAUUM, TRSM) are array-renamed at the tile level: they read
// the current slot and write the alternate one, swapped at completion.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tinv_internal.h"

namespace tinv {

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load3(const CUtensorMap* map, void* dst, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch3(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
// global += smem (FP64 add performed by the TMA unit; verified exact on B200,
// tools/tma_f64_reduce_test.cu)
__device__ __forceinline__ void tma_reduce_add3(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int ld_relaxed_s32(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_sys_s32(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_sys_s32(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_release_sys_s32(int32_t* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_cta_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cta_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(const char* p) { return *reinterpret_cast<const double2*>(p); }
// permutation of the 8 rows of an MMA fragment so that 128-bit fragment
// loads from 128B-swizzled TMA tiles are bank-conflict free per quarter warp
__device__ __forceinline__ int rho(int x) { return (x >> 1) | ((x & 1) << 2); }

// ---------------------------------------------------------------- jobs
enum Variant : int8_t { V_NT = 0, V_NN = 1, V_TN = 2 };
enum JobType : int8_t { J_GEMM = 0, J_SPECIAL = 1 };
enum Special : int8_t { SP_BPOTRF = 0, SP_BTRTRI = 1, SP_COPY_ROWS = 2, SP_SEND = 3, SP_BCOPYINV = 4, SP_DEPART = 5 };

struct ItemInfo {
  int32_t task, item, phase, kind, step;  // phase: phase group index (queue entry)
  int32_t ph0, nph, grp;                  // first phase, fused single-item phases, phase group
  int32_t out_s, alt_s, in0_s, in1_s, scr_s;
  int32_t ref_id, nitems, njobs, flags;
  int32_t aux0, aux1;
};

struct Job {
  int8_t type, variant, special, mirror, dep, sign;
  int16_t d;  // special parameter (diagonal block)
  int32_t a_s, a_fix, a_k0, b_s, b_fix, b_k0;
  int32_t k0, k1, a_mask, b_mask;
  int32_t o_s, o_r, o_c, c_s;
  int32_t src_s;  // special: source slot
};

__device__ __forceinline__ void lower_pair(int i, int& r, int& c) {
  r = 0;
  while ((r + 1) * (r + 2) / 2 <= i) ++r;
  c = i - r * (r + 1) / 2;
}

// jobs of one item of phase p: two for the off-diagonal items of TRTRI / INV
// phases >= 1, one otherwise
__device__ __forceinline__ int phase_jobs(int kind, int p, int R) {
  return (((kind == TINV_TRTRI || kind == KIND_INV) && p > 0) || (kind == KIND_POTRF_INV && p >= 3 * R - 2)) ? 2 : 1;
}
__device__ __forceinline__ int job_count(const ItemInfo& it, int R) {
  int n = 0;
  for (int p = it.ph0; p < it.ph0 + it.nph; ++p) n += phase_jobs(it.kind, p, R);
  return n;
}

__device__ __forceinline__ void gemm_job(Job& j, int8_t v, int a_s, int a_fix, int a_k0, int b_s, int b_fix,
                                         int b_k0, int k0, int k1, int o_s, int o_r, int o_c, int c_s,
                                         int sign) {
  j.type = J_GEMM;
  j.variant = v;
  j.special = 0;
  j.mirror = 0;
  j.dep = 0;
  j.sign = (int8_t)sign;
  j.d = 0;
  j.a_s = a_s;
  j.a_fix = a_fix;
  j.a_k0 = a_k0;
  j.b_s = b_s;
  j.b_fix = b_fix;
  j.b_k0 = b_k0;
  j.k0 = k0;
  j.k1 = k1;
  j.a_mask = -1;
  j.b_mask = -1;
  j.o_s = o_s;
  j.o_r = o_r;
  j.o_c = o_c;
  j.c_s = c_s;
  j.src_s = -1;
}

__device__ __forceinline__ void special_job(Job& j, int8_t sp, int d, int src, int dst) {
  j.type = J_SPECIAL;
  j.special = sp;
  j.d = (int16_t)d;
  j.dep = 1;
  j.src_s = src;
  j.o_s = dst;
}

__device__ __forceinline__ void get_job_phase(const ItemInfo& it, int n, int R, Job& j) {
  const int o = it.out_s, a = it.alt_s, x = it.in0_s, y = it.in1_s;
  const int kind = it.kind;
  if (kind == KIND_POTRF_INV && it.phase >= 3 * R - 2) {  // X = L^-1 into aux x: X[r][r-s] (TRTRI phase s)
    const int s = it.phase - (3 * R - 2) + 1, r = s + it.item, d = r - s;
    if (n == 0) {  // X[r][d] <- sum_{k=d+1..r} X[r][k] L[k][d]
      gemm_job(j, V_NN, x, r, d + 1, o, d, d + 1, d + 1, r + 1, x, r, d, -1, 1);
      j.a_mask = r;
    } else {  // X[r][d] <- -X[r][d] X[d][d]
      gemm_job(j, V_NN, x, r, d, x, d, d, d, d + 1, x, r, d, -1, -1);
      j.b_mask = d;
      j.dep = 1;
    }
    return;
  }
  if (kind == TINV_POTRF || kind == KIND_POTRF_INV) {  // in place on o; inverse diagonal blocks -> aux x
    const int d = it.phase / 3;
    switch (it.phase % 3) {
      case 0:
        special_job(j, SP_BPOTRF, d, x, o);
        return;
      case 1: {  // A[r][d] <- A[r][d] inv(L_dd)^T
        const int r = d + 1 + it.item;
        gemm_job(j, V_NT, o, r, d, x, d, d, d, d + 1, o, r, d, -1, 1);
        j.b_mask = d;
        return;
      }
      default: {  // A[r][c] -= A[r][d] A[c][d]^T, r >= c > d
        int rr, cc;
        lower_pair(it.item, rr, cc);
        const int r = d + 1 + rr, c = d + 1 + cc;
        gemm_job(j, V_NT, o, r, d, o, c, d, d, d + 1, o, r, c, o, -1);
        return;
      }
    }
  }
  if (kind == TINV_TRTRI || kind == KIND_INV) {
    // X = L^-1: source L in `src`, result in `dst` (TRTRI: renamed cur -> alt)
    const int src = kind == KIND_INV ? x : o;
    const int dst = kind == KIND_INV ? o : a;
    if (it.phase == 0) {
      if (it.flags & TF_DIAG_FROM_AUX)  // inverse diagonal blocks already computed by POTRF
        special_job(j, SP_BCOPYINV, it.item, y, dst);
      else
        special_job(j, SP_BTRTRI, it.item, src, dst);
      return;
    }
    const int r = it.phase + it.item, d = r - it.phase;
    if (n == 0) {  // X[r][d] <- sum_{k=d+1..r} X[r][k] L[k][d]
      gemm_job(j, V_NN, dst, r, d + 1, src, d, d + 1, d + 1, r + 1, dst, r, d, -1, 1);
      j.a_mask = r;
    } else {  // X[r][d] <- -X[r][d] X[d][d]
      gemm_job(j, V_NN, dst, r, d, dst, d, d, d, d + 1, dst, r, d, -1, -1);
      j.b_mask = d;
      j.dep = 1;
    }
    return;
  }
  if (kind == TINV_COPY) {
    special_job(j, SP_COPY_ROWS, it.item, x, o);
    return;
  }
  if (kind == KIND_SEND) {  // block item of the tile version -> receiver's pool
    special_job(j, SP_SEND, it.item, x, -1);
    return;
  }
  if (kind == KIND_DEPART) {  // block (item / R, item % R) of the result tile -> host
    special_job(j, SP_DEPART, it.item, x, -1);
    return;
  }
  int r, c;
  if (kind == TINV_SYRK_SUB || kind == TINV_SYRK_ADD_T || kind == TINV_LAUUM) {
    lower_pair(it.item, r, c);
  } else if (kind == TINV_TRSM) {  // longest items (largest c) first
    c = R - 1 - it.item / R;
    r = it.item % R;
  } else {
    r = it.item / R;
    c = it.item % R;
  }
  // accumulate kernels write in place unless an operand aliases the output
  const int w = (it.flags & TF_RENAMED) ? a : o;
  switch (kind) {
    case TINV_GEMM:
      if (it.step == TINV_STEP_CHOLESKY)
        gemm_job(j, V_NT, x, r, 0, y, c, 0, 0, R, w, r, c, o, -1);
      else if (it.step == TINV_STEP_TRINV)
        gemm_job(j, V_NN, x, r, 0, y, c, 0, 0, R, w, r, c, o, 1);
      else
        gemm_job(j, V_TN, x, r, 0, y, c, 0, 0, R, w, r, c, o, 1);
      return;
    case TINV_SYRK_SUB:
      gemm_job(j, V_NT, x, r, 0, x, c, 0, 0, R, w, r, c, o, -1);
      j.mirror = (it.flags & TF_NO_MIRROR) ? 0 : 1;
      return;
    case TINV_SYRK_ADD_T:
      gemm_job(j, V_TN, x, r, 0, x, c, 0, 0, R, w, r, c, o, 1);
      j.mirror = 1;
      return;
    case TINV_TRMM_LEFT:  // tril(T) A : sum_{s<=r} T[r][s] A[s][c]
      gemm_job(j, V_NN, x, r, 0, o, c, 0, 0, r + 1, a, r, c, -1, 1);
      j.a_mask = r;
      return;
    case TINV_TRMM_RIGHT_NEG:  // -A tril(T) : -sum_{s>=c} A[r][s] T[s][c]
      gemm_job(j, V_NN, o, r, c, x, c, c, c, R, a, r, c, -1, -1);
      j.b_mask = c;
      return;
    case TINV_TRMM_LEFT_T:  // tril(T)^T A : sum_{s>=r} T[s][r]^T A[s][c]
      gemm_job(j, V_TN, x, r, r, o, c, r, r, R, a, r, c, -1, 1);
      j.a_mask = r;
      return;
    case TINV_LAUUM:  // tril(L)^T tril(L) : sum_{s>=r} L[s][r]^T L[s][c]
      gemm_job(j, V_TN, o, r, r, o, c, r, r, R, a, r, c, -1, 1);
      j.a_mask = r;
      j.b_mask = c;
      j.mirror = 1;
      return;
    case TINV_TRSM:  // X = A tril(L)^-T = sum_{s<=c} A[r][s] Linv[c][s]
      gemm_job(j, V_NT, o, r, 0, x, c, 0, 0, c + 1, a, r, c, -1, 1);
      j.b_mask = c;
      return;
    default:
      return;
  }
}

// job n of an item: walk the fused phases of its group; the first job of a
// fused phase after the first depends on everything before it
__device__ __forceinline__ void get_job(const ItemInfo& it, int n, int R, Job& j) {
  if (it.nph == 1) {
    get_job_phase(it, n, R, j);
    return;
  }
  ItemInfo sub = it;
  for (int p = it.ph0; p < it.ph0 + it.nph; ++p) {
    const int nj = phase_jobs(it.kind, p, R);
    if (n < nj) {
      sub.phase = p;
      sub.item = 0;
      get_job_phase(sub, n, R, j);
      if (n == 0 && p > it.ph0) j.dep = 1;
      return;
    }
    n -= nj;
  }
}

// ---------------------------------------------------------------- smem
// consumer -> storer hand-off records
enum RecType : int32_t { R_QUARTER = 0, R_JOB_END = 1, R_ITEM_END = 2, R_EXIT = 3 };
struct Rec {
  int32_t type, a, b, c, d, e, f, g;
};
constexpr int NREC = 16;
constexpr int MAXJ = 8;

struct PotrfFlags {
  int fac;      // panels whose L_PP (+ 1 / l_kk) is published
  int rowdone;  // panels whose row block P + 1 warp 0 has solved
  int ready;    // rounds P whose blocks (P + 2, P + 1) and (P + 2, P + 2) are updated by panel P
};
struct SmemCtl {
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  uint64_t item_full[2];
  uint64_t item_empty[2];
  uint64_t rec_full[NREC];
  uint64_t rec_empty[NREC];
  uint64_t stg_free[2];
  ItemInfo items[2];
  Job jobs[2][MAXJ + 2];  // per item slot: its first MAXJ jobs (producer-built); [MAXJ] consumers' and
                          // [MAXJ + 1] producer's scratch for later ones
  Rec recs[NREC];
  unsigned jobs_done;
  int fail_code;   // per item: 0 none
  int fail_index;
  int scan_min;
  unsigned long long dbg[4];
  unsigned long long dbg2[8];
  PotrfFlags pf;  // block_potrf's warp-0 / helper counters
};

constexpr unsigned FULL_MASK = 0xffffffffu;
// ---------------------------------------------------------------- consumers: DMMA chunk
// Warp w: rows [64*(w&1), +64), cols [32*(w>>1), +32) of the 128x128 block.
// A/B stage layouts: K-major = TMA box {16 k, 128 rows}; MN-major = 8 boxes
// {16 cols, 16 k-rows} at 2 KB each; both 128B-swizzled (16B chunk c of row r
// stored at c ^ (r & 7)).
template <int V, bool MA, bool MB>
__device__ __forceinline__ void chunk_mma(const char* sA, const char* sB, double (&acc)[8][4][2], int wm, int wn,
                                          int g, int tg, int kb16) {
  const int rg = rho(g);
  if constexpr (V == V_NT || V == V_NN) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 a[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int row = 64 * wm + 8 * p + rg;
        a[p] = lds128(sA + row * 128 + (((tg + 4 * h) ^ rg) << 4));
        if constexpr (MA) {  // keep A(m,k) iff k <= m
          const int k = kb16 + 2 * (tg + 4 * h);
          if (k > row) a[p].x = 0.0;
          if (k + 1 > row) a[p].y = 0.0;
        }
      }
      if constexpr (V == V_NT) {
        double2 b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int n = 32 * wn + 8 * q + rg;
          b[q] = lds128(sB + n * 128 + (((tg + 4 * h) ^ rg) << 4));
          if constexpr (MB) {  // keep B(k,n) iff k <= n  (stored [n][k] lower)
            const int k = kb16 + 2 * (tg + 4 * h);
            if (k > n) b[q].x = 0.0;
            if (k + 1 > n) b[q].y = 0.0;
          }
        }
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma(acc[p][q], a[p].x, b[q].x);
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma(acc[p][q], a[p].y, b[q].y);
      } else {  // NN: B stored [k][n], pairs of n per lane (sigma = identity)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 2 * tg + 8 * h + e;
          double2 b[2];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            b[v] = lds128(sB + (2 * wn + v) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
            if constexpr (MB) {  // keep B(k,n) iff n <= k (stored [k][n] lower)
              const int n0 = 32 * wn + 16 * v + 2 * g;
              if (n0 > kb16 + k) b[v].x = 0.0;
              if (n0 + 1 > kb16 + k) b[v].y = 0.0;
            }
          }
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const double av = e ? a[p].y : a[p].x;
            dmma(acc[p][0], av, b[0].x);
            dmma(acc[p][1], av, b[0].y);
            dmma(acc[p][2], av, b[1].x);
            dmma(acc[p][3], av, b[1].y);
          }
        }
      }
    }
  } else {  // TN: A stored [k][m], B stored [k][n], sigma = rho for both
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int k = 4 * s + tg;
      const int sw = (rg ^ (k & 7)) << 4;
      double2 a[4], b[2];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        a[w] = lds128(sA + (4 * wm + w) * 2048 + k * 128 + sw);
        if constexpr (MA) {  // keep A(m,k) iff m <= k (stored [k][m] lower)
          const int m0 = 64 * wm + 16 * w + 2 * rg;
          if (m0 > kb16 + k) a[w].x = 0.0;
          if (m0 + 1 > kb16 + k) a[w].y = 0.0;
        }
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        b[v] = lds128(sB + (2 * wn + v) * 2048 + k * 128 + sw);
        if constexpr (MB) {
          const int n0 = 32 * wn + 16 * v + 2 * rg;
          if (n0 > kb16 + k) b[v].x = 0.0;
          if (n0 + 1 > kb16 + k) b[v].y = 0.0;
        }
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const double av = (p & 1) ? a[p >> 1].y : a[p >> 1].x;
        dmma(acc[p][0], av, b[0].x);
        dmma(acc[p][1], av, b[0].y);
        dmma(acc[p][2], av, b[1].x);
        dmma(acc[p][3], av, b[1].y);
      }
    }
  }
}

template <int V>
__device__ __forceinline__ int out_row(int wm, int p, int g) {
  if constexpr (V == V_TN) return 64 * wm + 16 * (p >> 1) + 2 * rho(g) + (p & 1);
  return 64 * wm + 8 * p + rho(g);
}
template <int V>
__device__ __forceinline__ int out_col(int wn, int q, int j) {
  if constexpr (V == V_NT) return 32 * wn + 8 * q + rho(j);
  if constexpr (V == V_NN) return 32 * wn + 16 * (q >> 1) + 2 * j + (q & 1);
  return 32 * wn + 16 * (q >> 1) + 2 * rho(j) + (q & 1);
}

struct EpiState {
  unsigned rec;    // next hand-off record index (identical in every consumer thread)
  unsigned tjobs;  // TMA-epilogue jobs so far (staging buffer phases)
  unsigned jobs;   // jobs so far (published as jobs_done by the storer)
  int generic;     // this job / item wrote global memory with generic stores
};

__device__ __forceinline__ void push_rec(SmemCtl& ctl, unsigned idx, Rec r) {
  const int s = idx % NREC;
  mbar_wait(&ctl.rec_empty[s], ((idx / NREC) & 1) ^ 1);
  ctl.recs[s] = r;
  mbar_arrive(&ctl.rec_full[s]);
}

// Before a diagonal phase: every earlier job of this CTA has been retired by
// the storer (its TMA writes performed, its staged quarters read), so global
// reads see them and the staging area can serve as scratch.
__device__ __forceinline__ void drain_jobs(SmemCtl& ctl, const EpiState& es) {
  cons_bar();
  if (threadIdx.x == 0)
    while (ld_acquire_cta_u32(&ctl.jobs_done) < es.jobs) {
    }
  cons_bar();
  fence_proxy_async();
}

template <int V, typename Tick>
__device__ __forceinline__ void run_gemm(const Job& jb, const ExecParams& P, SmemCtl& ctl, char* ring, unsigned& ks,
                                         Tick& tick, EpiState& es) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp & 1, wn = warp >> 1, g = lane >> 2, tg = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q][0] = acc[p][q][1] = 0.0;

  for (int kb = jb.k0; kb < jb.k1; ++kb) {
    const bool ma = (kb == jb.a_mask), mb = (kb == jb.b_mask);
    // a tile order b that is not a multiple of 128 is padded to bp: K chunks
    // that lie wholly in the padding contribute zero (or, on a diagonal tile's
    // unit padding, only to the output's own padding): skip their DMMAs
    const int kreal = P.b - kb * BLK;
    for (int ch = 0; ch < BLK / KCH; ++ch, ++ks) {
      const int st = ks % NSTAGE;
      mbar_wait(&ctl.full[st], (ks / NSTAGE) & 1);
      const char* sA = ring + st * STAGE_BYTES;
      const char* sB = sA + STAGE_BYTES / 2;
      const int kb16 = ch * KCH;
      if (kb16 >= kreal) {
      } else if (!ma && !mb) {
        chunk_mma<V, false, false>(sA, sB, acc, wm, wn, g, tg, kb16);
      } else {
        // on a triangular operand's diagonal block, a chunk whose masked part
        // covers this warp's whole tile contributes nothing: skip its DMMAs
        const bool za = ma && ((V == V_TN) ? (64 * wm > kb16 + KCH - 1) : (kb16 > 64 * wm + 63));
        const bool zb = mb && ((V == V_NT) ? (kb16 > 32 * wn + 31) : (32 * wn > kb16 + KCH - 1));
        if (za || zb) {
        } else if (ma && !mb)
          chunk_mma<V, true, false>(sA, sB, acc, wm, wn, g, tg, kb16);
        else if (!ma && mb)
          chunk_mma<V, false, true>(sA, sB, acc, wm, wn, g, tg, kb16);
        else
          chunk_mma<V, true, true>(sA, sB, acc, wm, wn, g, tg, kb16);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.empty[st]);
    }
  }

  tick(1);
  const double sg = (double)jb.sign;
  if (!jb.mirror && (jb.c_s < 0 || jb.c_s == jb.o_s)) {
    // TMA epilogue: sign*acc staged 32 rows at a time (quarter k = rows
    // 32k..32k+31, written by the 4 warps owning them) into two alternating
    // 32 KB buffers of 128B-swizzled {16 cols x 32 rows} boxes; the storer
    // warp stores -- or for C += sign*acc reduce-adds -- each quarter with
    // cp.(reduce.)async.bulk.tensor while the consumers move on.
    char* stg = ring + NSTAGE * STAGE_BYTES;
    const int red = jb.c_s >= 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (wm == (k >> 1)) {
        const int buf = k & 1;
        const unsigned use = 2 * es.tjobs + (k >> 1);
        mbar_wait(&ctl.stg_free[buf], (use & 1) ^ 1);
        char* sb = stg + buf * 32768;
        // 16-byte stores, conflict-free per quarter warp (two rows g, g + 1 x
        // four lanes tg must hit eight distinct 16-byte chunks of the swizzled
        // 128-byte rows): NT exchanges one value with lane tg ^ 1 so each lane
        // holds two adjacent columns; NN / TN hold adjacent columns in
        // acc[p][2 qq][e], acc[p][2 qq + 1][e] and odd rows store e = 1 first.
        // (8-byte stores here were 2- to 4-way conflicts: 3.7e9 excess
        // wavefronts a C3 launch, profiles/r02/final/ncu_exec_c3_full_metrics.csv)
        auto st2 = [&](int r, int c, double v0, double v1) {
          *reinterpret_cast<double2*>(sb + (c >> 4) * 4096 + r * 128 + ((((c & 15) >> 1) ^ (r & 7)) << 4)) =
              make_double2(sg * v0, sg * v1);
        };
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          const int p = 4 * (k & 1) + pp;
          const int r = out_row<V>(wm, p, g) - 32 * k;
          if constexpr (V == V_NT) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // columns 32 wn + 8 q + tg (e = 0), + 4 (e = 1)
              const double mine0 = acc[p][q][0], mine1 = acc[p][q][1];
              const double got = __shfl_xor_sync(FULL_MASK, (tg & 1) ? mine0 : mine1, 1);
              const int c = 32 * wn + 8 * q + ((tg & 1) ? tg + 3 : tg);
              st2(r, c, (tg & 1) ? got : mine0, (tg & 1) ? mine1 : got);
            }
          } else {
#pragma unroll
            for (int qq = 0; qq < 2; ++qq)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const bool flip = g & 1;  // this lane's e for this instruction: e ^ (g & 1)
                const double v0 = flip ? acc[p][2 * qq][e ^ 1] : acc[p][2 * qq][e];
                const double v1 = flip ? acc[p][2 * qq + 1][e ^ 1] : acc[p][2 * qq + 1][e];
                const int el = e ^ (int)flip;
                const int c = out_col<V>(wn, 2 * qq, 2 * tg + el);
                st2(r, c, v0, v1);
              }
          }
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync %0, 128;" ::"r"(2 + wm) : "memory");
        if (warp == wm && lane == 0)
          push_rec(ctl, es.rec + k, Rec{R_QUARTER, buf, jb.o_c * BLK, jb.o_r * BLK + 32 * k, jb.o_s, red, 0, 0});
      }
    }
    es.rec += 4;
    es.tjobs += 1;
    return;
  }
  es.generic = 1;
  // general epilogue: out = [C +] sign * acc ; mirror -> also the transposed block
  const int64_t bp = P.bp;
  double* O = P.pool + (int64_t)jb.o_s * P.slot_elems + (int64_t)jb.o_r * BLK * bp + jb.o_c * BLK;
  double* OT = P.pool + (int64_t)jb.o_s * P.slot_elems + (int64_t)jb.o_c * BLK * bp + jb.o_r * BLK;
  const double* C =
      jb.c_s >= 0 ? P.pool + (int64_t)jb.c_s * P.slot_elems + (int64_t)jb.o_r * BLK * bp + jb.o_c * BLK : nullptr;
  const bool diag = jb.o_r == jb.o_c;
  // pass 1: v = [C +] sign * acc, all C loads independent of any store
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int r = out_row<V>(wm, p, g);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = out_col<V>(wn, q, 2 * tg + e);
        double v = sg * acc[p][q][e];
        if (C && !(jb.mirror && diag && c > r)) v += __ldcg(C + r * bp + c);
        acc[p][q][e] = v;
      }
  }
  // pass 2: stores (and the transposed copy for symmetric outputs)
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int r = out_row<V>(wm, p, g);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = out_col<V>(wn, q, 2 * tg + e);
        if (jb.mirror && diag && c > r) continue;
        O[r * bp + c] = acc[p][q][e];
        if (jb.mirror && !(diag && c == r)) OT[c * bp + r] = acc[p][q][e];
      }
  }
}

// ---------------------------------------------------------------- consumers: diagonal phases
// A 128x128 diagonal block in shared memory uses row stride SLD = 132 doubles.
constexpr int SLD = BLK + 4;  // = 4 mod 16 doubles: m8n8k4 fragment loads (rows g, cols tg) hit distinct banks
// after the 128x128 block (row stride SLD): [0, 16) block_potrf's 1 / l_kk of
// the last two panels, [XD_OFF, XD_OFF + 1024) the 8x8 diagonal inverses,
// then 8 x 64 doubles of level-8 products (all inside block_trtri_dmma's T area)
constexpr int XD_OFF = 64;
constexpr int XT_OFF = XD_OFF + 16 * 64;

// global -> global copy of n2 double2 by the 256 consumer threads, 8 loads in
// flight per thread (a dependent load->store loop is latency-bound)
__device__ __forceinline__ void copy_d2(double2* __restrict__ out, const double2* __restrict__ src, int64_t n2) {
  int64_t e = threadIdx.x;
  for (; e + 7 * 256 < n2; e += 8 * 256) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + e + u * 256);
#pragma unroll
    for (int u = 0; u < 8; ++u) out[e + u * 256] = v[u];
  }
  for (; e < n2; e += 256) out[e] = __ldcg(src + e);
}
// 128x128 block (row stride bp) -> S, lower part only, 8 row-pairs in flight per thread
__device__ __forceinline__ void load_block_lower(double* S, const double* blk, int64_t bp) {
  const int c2 = threadIdx.x & 63, r0 = threadIdx.x >> 6;  // each thread: columns 2*c2, 2*c2+1 of 32 rows
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(reinterpret_cast<const double2*>(blk + (r0 + 4 * (8 * g + u)) * bp) + c2);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = r0 + 4 * (8 * g + u), j = 2 * c2;
      S[i * SLD + j] = j <= i ? v[u].x : 0.0;
      S[i * SLD + j + 1] = j + 1 <= i ? v[u].y : 0.0;
    }
  }
}

__device__ void store_block_lower(const double* S, double* dst, int64_t bp) {
  const int c2 = threadIdx.x & 63;
  for (int i = threadIdx.x >> 6; i < BLK; i += 4) {
    const int j = 2 * c2;
    reinterpret_cast<double2*>(dst + i * bp)[c2] =
        make_double2(j <= i ? S[i * SLD + j] : 0.0, j + 1 <= i ? S[i * SLD + j + 1] : 0.0);
  }
}
// zero the blocks (d, c > d) of a tile (upper part of block row d)
__device__ void zero_upper_row(double* tile, int d, int R, int64_t bp) {
  const int w = (R - 1 - d) * BLK;  // doubles per row to clear
  if (w <= 0) return;
  double* base = tile + (int64_t)d * BLK * bp + (d + 1) * BLK;
  for (int e = threadIdx.x; e < BLK * w / 2; e += 256) {
    const int i = e / (w / 2), j = (e % (w / 2)) * 2;
    *reinterpret_cast<double2*>(base + i * bp + j) = make_double2(0.0, 0.0);
  }
}

// ---- 128x128 diagonal-block kernels on S (shared, row stride SLD): 8x8
// register factor / inverse blocks, DMMA for every product.
constexpr unsigned FULL = 0xffffffffu;

// ---- dataflow 128x128 block Cholesky (tools/micro/potrf_flow.cu times it and
// checks it against the look-ahead version it replaced: 66K -> 42K cycles).
//
// Warp 0 runs the pivot chain alone: per 8-wide panel P it factors the 8x8
// diagonal block in registers (chol8), publishes L_PP, solves row block P + 1
// of the panel (lanes 0-7, one row each, by substitution) and applies panel P
// to the diagonal block (P + 1, P + 1) itself -- the only work between two
// chol8's. Warps 1-7 (the helpers) solve the rest of the panel and apply it
// to the trailing blocks, the blocks warp 0 needs next first, synchronised
// with warp 0 through three shared counters (no CTA-wide barrier per panel).
// Every block (i, j) still receives panels 0, 1, ... in order, each as two
// m8n8k4 DMMAs (k 0-3, then 4-7).
__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void helper_bar() { asm volatile("bar.sync 4, 224;" ::: "memory"); }

// Cholesky of the lower 8x8 block at (p0, p0) of S in registers (kernels.py:68-71
// failure test: not d > 0, or d non-finite; the pivot is then taken as 1 so the
// chain completes): l = the factor, il[k] = 1 / l[k][k]. Returns the first
// failing pivot or -1.
__device__ __forceinline__ int chol8(const double* S, int p0, double (&l)[8][8], double (&il)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) l[i][j] = S[(p0 + i) * SLD + p0 + j];
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
  return bad;
}

// Row q of panel p0: v = a L_PP^-T by substitution, L_PP from S (broadcast
// reads), 1 / l_kk at il.
__device__ __forceinline__ void panel_row(double* S, int q, int p0, const double* il) {
  double v[8];
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const double2 t2 = *reinterpret_cast<const double2*>(S + q * SLD + p0 + c);
    v[c] = t2.x;
    v[c + 1] = t2.y;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double t = v[c];
#pragma unroll
    for (int k = 0; k < c; ++k) t = fma(-v[k], S[(p0 + c) * SLD + p0 + k], t);
    v[c] = t * il[c];
  }
#pragma unroll
  for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(S + q * SLD + p0 + c) = make_double2(v[c], v[c + 1]);
}

// One warp: 8x8 block (ti, tj) -= L_i L_j^T over panel p0 (two DMMAs).
__device__ __forceinline__ void upd_blk(double* S, int p0, int ti, int tj) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int r = 8 * ti + g, c0 = 8 * tj;
  double2* cp = reinterpret_cast<double2*>(S + r * SLD + c0 + 2 * tg);
  const double2 c2 = *cp;
  double x[2] = {c2.x, c2.y};
  const double a0 = -S[r * SLD + p0 + tg], a1 = -S[r * SLD + p0 + 4 + tg];
  const double b0 = S[(c0 + g) * SLD + p0 + tg], b1 = S[(c0 + g) * SLD + p0 + 4 + tg];
  dmma(x, a0, b0);
  dmma(x, a1, b1);
  *cp = make_double2(x[0], x[1]);
}

// Column c of x = l^-1 for the stored lower 8x8 block l at (p0, p0) of S, by
// one thread (eight threads form one block's inverse): x_cc = 1 / l_cc,
// x_ic = -(sum_{k<i} l_ik x_kc, fma in ascending k from 0.0) * x_ii with x_kc = 0
// for k < c. The one routine behind every 8x8 diagonal inverse (TRTRI, INV of a
// received tile, the inverse half of POTRF_INV), so they are bitwise equal.
// out: the full 8x8 (zero upper).
__device__ __forceinline__ void diag_inv8_col(const double* S, int p0, int c, double* out) {
  double l[8][8], d[8], x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) l[i][j] = S[(p0 + i) * SLD + p0 + j];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = 1.0 / l[i][i];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) t = fma(l[i][k], x[k], t);
    x[i] = i < c ? 0.0 : (i == c ? d[i] : -t * d[i]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) out[8 * i + c] = x[i];
}

// In-place Cholesky of the lower 128x128 block in S (all 256 consumer
// threads; lp: 16 doubles of shared scratch; fl zeroed and scan_min set by
// the caller before a barrier). Returns the first failing pivot or -1.
__device__ int block_potrf(double* S, double* lp, PotrfFlags& fl, int& scan_min) {
  constexpr int T8 = BLK / 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    for (int P = 0; P < T8; ++P) {
      const int p0 = 8 * P;
      double l[8][8], il[8];
      double* lpP = lp + 8 * (P & 1);  // double-buffered: helpers may still read panel P - 1's
      const int bad = chol8(S, p0, l, il);
      if (lane == 0 && bad >= 0) atomicMin(&scan_min, p0 + bad);
      if (lane < 8) {  // lane r publishes row r of L_PP to S and 1 / l_rr to lp (register selects)
        double row[8], ilr = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          row[j] = 0.0;
#pragma unroll
          for (int i = j; i < 8; ++i) row[j] = lane == i ? l[i][j] : row[j];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) ilr = lane == i ? il[i] : ilr;
#pragma unroll
        for (int j = 0; j < 8; j += 2)
          *reinterpret_cast<double2*>(S + (p0 + lane) * SLD + p0 + j) = make_double2(row[j], row[j + 1]);
        lpP[lane] = ilr;
      }
      __syncwarp();
      if (lane == 0) st_rel_cta(&fl.fac, P + 1);
      if (P + 1 == T8) break;
      // row block P + 1 needs panels < P applied to block (P + 1, P): helpers' round P - 1
      if (P >= 1)
        while (ld_acq_cta(&fl.ready) < P) {
        }
      __syncwarp();
      if (lane < 8) {  // row r of block (P + 1, P) by substitution with the factor in registers
        const int q = p0 + 8 + lane;
        double v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double t = S[q * SLD + p0 + c];
#pragma unroll
          for (int k = 0; k < c; ++k) t = fma(-v[k], l[c][k], t);
          v[c] = t * il[c];
        }
#pragma unroll
        for (int c = 0; c < 8; c += 2)
          *reinterpret_cast<double2*>(S + q * SLD + p0 + c) = make_double2(v[c], v[c + 1]);
      }
      __syncwarp();
      if (lane == 0) st_rel_cta(&fl.rowdone, P + 1);
      upd_blk(S, p0, P + 1, P + 1);  // block (P + 1, P + 1) had panels < P applied in round P - 1
      __syncwarp();
    }
  } else {
    const int hw = warp - 1;  // helper warp 0..6
    for (int P = 0; P + 1 < T8; ++P) {
      const int p0 = 8 * P;
      while (ld_acq_cta(&fl.fac) < P + 1) {
      }
      const int q = p0 + 16 + (tid - 32);  // rows of blocks P + 2 ..
      if (q < BLK) panel_row(S, q, p0, lp + 8 * (P & 1));
      while (ld_acq_cta(&fl.rowdone) < P + 1) {
      }
      helper_bar();  // every L_iP of the panel is in S
      // warp 0's next needs first: blocks (P + 2, P + 1), (P + 2, P + 2)
      if (P + 2 < T8 && hw == 0) {
        upd_blk(S, p0, P + 2, P + 1);
        upd_blk(S, p0, P + 2, P + 2);
        __syncwarp();
        if (lane == 0) st_rel_cta(&fl.ready, P + 1);
      }
      // the rest of the trailing blocks, rows P + 3 .. in units of four blocks of one row
      // (one A fragment pair per unit, every load before the first DMMA). Units run
      // chunk-major -- chunk q = block columns P + 1 + 4q .., rows max(P + 3, P + 1 + 4q) .. 15
      // -- and unit c goes to helper warp c mod 7 (decoded directly, no scan)
      {
        const int g = lane >> 2, tg = lane & 3;
        // warp 4 shares warp 0's SM sub-partition (FP64 pipe): it takes no update units
        const int uw = hw < 3 ? hw : hw - 1;  // updater index 0..5 (hw 3 = warp 4: none)
        for (int c = uw; hw != 3; c += 6) {
          int q = 0, rem = c, i = -1;
          for (; q < 4; ++q) {
            const int r0 = max(P + 3, P + 1 + 4 * q), n = T8 - r0;
            if (n <= 0) break;
            if (rem < n) {
              i = r0 + rem;
              break;
            }
            rem -= n;
          }
          if (i < 0) break;
          const int j0 = P + 1 + 4 * q, r = 8 * i + g;
          const double a0 = -S[r * SLD + p0 + tg], a1 = -S[r * SLD + p0 + 4 + tg];
          double x[4][2], b[4][2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c0 = 8 * min(j0 + u, i);
            const double2 c2 = *reinterpret_cast<const double2*>(S + r * SLD + c0 + 2 * tg);
            x[u][0] = c2.x;
            x[u][1] = c2.y;
            b[u][0] = S[(c0 + g) * SLD + p0 + tg];
            b[u][1] = S[(c0 + g) * SLD + p0 + 4 + tg];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(x[u], a0, b[u][0]);
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(x[u], a1, b[u][1]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u <= i)
              *reinterpret_cast<double2*>(S + r * SLD + 8 * (j0 + u) + 2 * tg) = make_double2(x[u][0], x[u][1]);
        }
      }
      helper_bar();  // round P done: column P + 1 (and every block) has panels <= P applied
    }
  }
  cons_bar();
  const int f = scan_min;
  return f < (1 << 30) ? f : -1;
}

// One warp: a 16x16 output group D[m0.., n0..] = sgn * sum_{k in [k0, k1)}
// Lf(m, k) Rt(k, n) on DMMA (m8n8k4, 2x2 tiles), operands in shared memory:
// Lf(m, k) = L[(lr + m) * lld + lc + k], Rt(k, n) = R[(rr + k) * rld + rc + n],
// k1 - k0 a multiple of 16. Result to D[(dr + m) * dld + dc + n].
__device__ __forceinline__ void dmma_group16(const double* L, int lld, int lr, int lc, const double* R, int rld, int rr,
                                             int rc, int k0, int k1, double* D, int dld, int dr, int dc, double sgn) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  double acc[2][2][2] = {};
  for (int k = k0; k < k1; k += 16) {  // 4 k-steps per round: 16 fragment loads in flight, then 16 MMAs
    double a[4][2], b[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[u][mi] = L[(lr + 8 * mi + g) * lld + lc + k + 4 * u + tg];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[u][ni] = R[(rr + k + 4 * u + tg) * rld + rc + 8 * ni + g];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[u][mi], b[u][ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) D[(dr + 8 * mi + g) * dld + dc + 8 * ni + 2 * tg + e] = sgn * acc[mi][ni][e];
}

// Same as dmma_group16 for a 16 x 32 output group (2 x 4 tiles: 8 accumulator
// chains, 6 fragment loads per 8 MMAs).
__device__ __forceinline__ void dmma_group16x32(const double* L, int lld, int lr, int lc, const double* R, int rld,
                                                int rr, int rc, int k0, int k1, double* D, int dld, int dr, int dc,
                                                double sgn) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  double acc[2][4][2] = {};
  for (int k = k0; k < k1; k += 8) {
    double a[2][2], b[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[u][mi] = L[(lr + 8 * mi + g) * lld + lc + k + 4 * u + tg];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[u][ni] = R[(rr + k + 4 * u + tg) * rld + rc + 8 * ni + g];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[u][mi], b[u][ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) D[(dr + 8 * mi + g) * dld + dc + 8 * ni + 2 * tg + e] = sgn * acc[mi][ni][e];
}

// In-place inverse of the lower-triangular 128x128 block in S by recursive
// doubling: the sixteen 8x8 diagonal inverses (diag_inv8_col), then for s = 8, 16, 32, 64 every pair [[A,0],[B,C]] ->
// [[A^-1,0],[-C^-1 B A^-1, C^-1]] with the products on DMMA. Strict upper
// part of S must be zero on entry. Per level s and pair c, T = B A^-1 (A^-1
// lower: k >= first output column) into scratch, then X21 = -C^-1 T (C^-1
// lower: k < last output row), 16x16 groups per warp.
__device__ void block_trtri_dmma(double* S, unsigned long long* ctl_dbg) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int TLD = 68;
  double* Tb = S + BLK * SLD;  // T of every pair of a level: pair c at Tb + c * s * TLD
  long long tq = clock64();
  int pk = 3;
  auto probe = [&]() {
    const long long now = clock64();
    if (tid == 0) ctl_dbg[pk] += now - tq;
    tq = now;
    ++pk;
  };
  if (tid < BLK) diag_inv8_col(S, 8 * (tid >> 3), tid & 7, S + BLK * SLD + XD_OFF + 64 * (tid >> 3));
  cons_bar();  // the 16 diagonal 8x8 inverses, one column per thread
  {
    // 16x16 diagonal inverses from the 8x8 ones (warp w = pair of 8x8 blocks
    // 2w, 2w + 1): X21 = -C^-1 (B A^-1), two 8x8 DMMA tiles
    const double* XD = S + BLK * SLD + XD_OFF;
    double* T = S + BLK * SLD + XT_OFF + 64 * warp;
    const int p0 = 16 * warp, g = lane >> 2, tg = lane & 3;
    const double* Ai = XD + 128 * warp;
    const double* Ci = Ai + 64;
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 8; k += 4) dmma(acc, S[(p0 + 8 + g) * SLD + p0 + k + tg], Ai[(k + tg) * 8 + g]);
    T[g * 8 + 2 * tg] = acc[0];
    T[g * 8 + 2 * tg + 1] = acc[1];
    __syncwarp();
    acc[0] = acc[1] = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k += 4) dmma(acc, Ci[g * 8 + k + tg], T[(k + tg) * 8 + g]);
    S[(p0 + 8 + g) * SLD + p0 + 2 * tg] = -acc[0];
    S[(p0 + 8 + g) * SLD + p0 + 2 * tg + 1] = -acc[1];
    for (int e = lane; e < 64; e += 32) {
      const int i = e >> 3, j = e & 7;
      S[(p0 + i) * SLD + p0 + j] = Ai[e];
      S[(p0 + 8 + i) * SLD + p0 + 8 + j] = Ci[e];
      S[(p0 + i) * SLD + p0 + 8 + j] = 0.0;
    }
  }
  cons_bar();
  probe();
  for (int s = 16; s < BLK; s *= 2) {
    if (s == 64) {  // 16 x 32 groups (more accumulator chains per warp; measured 13K -> 10K cycles)
      const int gm = s / 16, gn = s / 32, per = gm * gn, total = (BLK / (2 * s)) * per;
      for (int q = 0; q * NCONS_WARPS < total; ++q) {
        const int gi = (q & 1) ? (q + 1) * NCONS_WARPS - 1 - warp : q * NCONS_WARPS + warp;
        if (gi >= total) continue;
        const int c = gi / per, m0 = 16 * ((gi % per) / gn), n0 = 32 * (gi % gn);
        const int a0 = 2 * c * s, b0 = a0 + s;
        dmma_group16x32(S, SLD, b0 + m0, a0, S, SLD, a0, a0 + n0, n0, s, Tb + c * s * TLD, TLD, m0, n0, 1.0);
      }
      cons_bar();
      for (int q = 0; q * NCONS_WARPS < total; ++q) {
        const int gi = (q & 1) ? (q + 1) * NCONS_WARPS - 1 - warp : q * NCONS_WARPS + warp;
        if (gi >= total) continue;
        const int c = gi / per, m0 = 16 * ((gi % per) / gn), n0 = 32 * (gi % gn);
        const int a0 = 2 * c * s, b0 = a0 + s;
        dmma_group16x32(S, SLD, b0 + m0, b0, Tb + c * s * TLD, TLD, 0, n0, 0, m0 + 16, S, SLD, b0 + m0, a0 + n0, -1.0);
      }
      cons_bar();
      probe();
      continue;
    }
    const int gs = s / 16, per = gs * gs, total = (BLK / (2 * s)) * per;
    // snake assignment: a warp's groups have complementary triangular k-extents
    for (int q = 0; q * NCONS_WARPS < total; ++q) {  // T_c = B_c A_c^-1
      const int gi = (q & 1) ? (q + 1) * NCONS_WARPS - 1 - warp : q * NCONS_WARPS + warp;
      if (gi >= total) continue;
      const int c = gi / per, m0 = 16 * ((gi % per) / gs), n0 = 16 * (gi % gs);
      const int a0 = 2 * c * s, b0 = a0 + s;
      dmma_group16(S, SLD, b0 + m0, a0, S, SLD, a0, a0 + n0, n0, s, Tb + c * s * TLD, TLD, m0, n0, 1.0);
    }
    cons_bar();
    for (int q = 0; q * NCONS_WARPS < total; ++q) {  // X21_c = -C_c^-1 T_c
      const int gi = (q & 1) ? (q + 1) * NCONS_WARPS - 1 - warp : q * NCONS_WARPS + warp;
      if (gi >= total) continue;
      const int c = gi / per, m0 = 16 * ((gi % per) / gs), n0 = 16 * (gi % gs);
      const int a0 = 2 * c * s, b0 = a0 + s;
      dmma_group16(S, SLD, b0 + m0, b0, Tb + c * s * TLD, TLD, 0, n0, 0, m0 + 16, S, SLD, b0 + m0, a0 + n0, -1.0);
    }
    cons_bar();
    probe();
  }
}

// jb / it live in shared memory (the item slot)
__device__ __noinline__ void run_special(const Job& jb, const ItemInfo& it, const ExecParams& P, SmemCtl& ctl,
                                         double* S, int b) {
  const int special = jb.special, d = jb.d, src_s = jb.src_s, o_s = jb.o_s, aux0 = it.aux0, aux1 = it.aux1;
  const int64_t bp = P.bp;
  const int R = P.R;
  if (ctl.fail_code) return;  // item already failed: keep the job protocol, skip work
  double* dst = P.pool + (int64_t)o_s * P.slot_elems;
  switch (special) {
    case SP_BPOTRF: {  // factor block (d,d) of dst in place; inverse -> aux block (d,d)
      long long t0 = clock64();
      double* blk = dst + (int64_t)d * BLK * bp + d * BLK;
      if (threadIdx.x == 0) {
        ctl.scan_min = 1 << 30;
        ctl.pf.fac = ctl.pf.rowdone = ctl.pf.ready = 0;
      }
      load_block_lower(S, blk, bp);
      cons_bar();
      long long t1 = clock64();
      const int f = block_potrf(S, S + BLK * SLD, ctl.pf, ctl.scan_min);
      long long t2 = clock64();
      if (threadIdx.x == 0) {
        ctl.dbg[0] += t1 - t0;
        ctl.dbg[1] += t2 - t1;
      }
      if (f >= 0) {
        if (threadIdx.x == 0) {
          ctl.fail_code = TINV_ERR_NOT_SPD;
          ctl.fail_index = d * BLK + f;
        }
        cons_bar();
        return;
      }
      t0 = clock64();
      store_block_lower(S, blk, bp);
      zero_upper_row(dst, d, R, bp);
      cons_bar();
      t1 = clock64();
      block_trtri_dmma(S, ctl.dbg2);
      t2 = clock64();
      double* aux = P.pool + (int64_t)src_s * P.slot_elems;
      store_block_lower(S, aux + (int64_t)d * BLK * bp + d * BLK, bp);
      if (it.kind == KIND_POTRF_INV) zero_upper_row(aux, d, R, bp);  // aux becomes the full lower L^-1
      cons_bar();
      if (threadIdx.x == 0) {
        ctl.dbg[3] += t1 - t0 + clock64() - t2;
        ctl.dbg[2] += t2 - t1;
      }
      break;
    }
    case SP_BTRTRI: {  // dst block (d,d) <- inv(tril(src block (d,d))); zero dst blocks (d, c>d)
      const double* sb = P.pool + (int64_t)src_s * P.slot_elems + (int64_t)d * BLK * bp + d * BLK;
      if (threadIdx.x == 0) ctl.scan_min = 1 << 30;
      load_block_lower(S, sb, bp);
      cons_bar();
      if (threadIdx.x < BLK && d * BLK + threadIdx.x < b && S[threadIdx.x * SLD + threadIdx.x] == 0.0)
        atomicMin(&ctl.scan_min, threadIdx.x);  // kernels.py:125-127: zero diagonal
      cons_bar();
      if (ctl.scan_min < (1 << 30)) {
        if (threadIdx.x == 0) {
          ctl.fail_code = TINV_ERR_SINGULAR;
          ctl.fail_index = d * BLK + ctl.scan_min;
        }
        cons_bar();
        return;
      }
      long long t1 = clock64();
      block_trtri_dmma(S, ctl.dbg2);
      long long t2 = clock64();
      store_block_lower(S, dst + (int64_t)d * BLK * bp + d * BLK, bp);
      zero_upper_row(dst, d, R, bp);
      cons_bar();
      if (threadIdx.x == 0) {
        ctl.dbg[2] += t2 - t1;
        ctl.dbg[3] += clock64() - t2;
      }
      break;
    }
    case SP_SEND: {  // 128-block d of the tile version -> receiver's pool (peer memory); the inbox flag is
                     // set by the task's last item (complete_item) once every block is out
      const int64_t off = (int64_t)(d / R) * BLK * bp + (d % R) * BLK;
      const double* src = P.pool + (int64_t)src_s * P.slot_elems + off;
      double* out = P.peer_pool[aux0] + (int64_t)(P.peer_recv_base[aux0] + aux1) * P.slot_elems + off;
      const int c2 = threadIdx.x & 63;  // 64 double2 per block row, 4 rows per pass, 8 loads in flight
#pragma unroll 1
      for (int r0 = threadIdx.x >> 6; r0 < BLK; r0 += 32) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(reinterpret_cast<const double2*>(src + (int64_t)(r0 + 4 * u) * bp) + c2);
#pragma unroll
        for (int u = 0; u < 8; ++u) reinterpret_cast<double2*>(out + (int64_t)(r0 + 4 * u) * bp)[c2] = v[u];
      }
      __threadfence_system();
      break;
    }
    case SP_BCOPYINV: {  // dst block (d,d) <- aux block (d,d) (lower, zero upper); zero dst blocks (d, c>d)
      const double* sb = P.pool + (int64_t)src_s * P.slot_elems + (int64_t)d * BLK * bp + d * BLK;
      double* db = dst + (int64_t)d * BLK * bp + d * BLK;
      for (int i = threadIdx.x >> 6; i < BLK; i += 4)
        reinterpret_cast<double2*>(db + i * bp)[threadIdx.x & 63] =
            __ldcg(reinterpret_cast<const double2*>(sb + i * bp) + (threadIdx.x & 63));
      zero_upper_row(dst, d, R, bp);
      break;
    }
    case SP_DEPART: {
      // SYMMETRIZE output: the tile's staging slot receives the transposed
      // tile (off-diagonal; the copy engines move it to block (j, i) of the
      // host matrix) or the mirrored full tile (diagonal). LOWER: nothing to
      // do; the copy engines read the final slot itself once the task is done.
      if (P.depart_mode != TINV_DENSE_SYMMETRIZE) break;
      const int br = d / R, bc = d % R;
      const bool diag = (aux1 >> 16) == (aux1 & 0xffff);
      if (diag && br < bc) break;  // covered by the transposed copy of block (bc, br)
      constexpr int DLD = BLK + 1;  // odd stride: the transposed (column) reads below are conflict-free
      const double* src = P.pool + (int64_t)src_s * P.slot_elems + (int64_t)br * BLK * bp + bc * BLK;
      double* stg = P.pool + (int64_t)(P.stage_base + aux0) * P.slot_elems;
      for (int e = threadIdx.x; e < BLK * BLK / 2; e += 256) {
        const int y = e >> 6, x2 = (e & 63) * 2;
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src + (int64_t)y * bp + x2));
        S[y * DLD + x2] = v.x;
        S[y * DLD + x2 + 1] = v.y;
      }
      cons_bar();
      if (diag) {  // block (br, bc) of the mirrored tile: verbatim (diagonal block: mirrored inside)
        double* o = stg + (int64_t)br * BLK * bp + bc * BLK;
        for (int e = threadIdx.x; e < BLK * BLK; e += 256) {
          const int y = e >> 7, x = e & (BLK - 1);
          o[(int64_t)y * bp + x] = (br == bc && x > y) ? S[x * DLD + y] : S[y * DLD + x];
        }
      }
      if (!diag || br > bc) {  // transposed block -> (bc, br)
        double* o = stg + (int64_t)bc * BLK * bp + br * BLK;
        for (int e = threadIdx.x; e < BLK * BLK; e += 256) {
          const int x = e >> 7, y = e & (BLK - 1);
          o[(int64_t)x * bp + y] = S[y * DLD + x];
        }
      }
      cons_bar();
      break;
    }
    case SP_COPY_ROWS: {
      const double* src = P.pool + (int64_t)src_s * P.slot_elems + (int64_t)d * BLK * bp;
      double* out = dst + (int64_t)d * BLK * bp;
      copy_d2(reinterpret_cast<double2*>(out), reinterpret_cast<const double2*>(src), (int64_t)BLK * bp / 2);
      break;
    }
    default:
      break;
  }
}

// ---------------------------------------------------------------- scheduler (device side)
// Queue geometry: level `lev` of the queue set starting at qb (= rank * NLEV
// when ranks are emulated in one launch, else 0).
__device__ __forceinline__ int64_t qoff(const ExecParams& P, int qb, int lev) {
  return P.nranks > 1 ? __ldg(P.q_offs + qb + lev) : P.q_off[lev];
}
__device__ __forceinline__ int cta_qb(const ExecParams& P) {
  return P.nranks > 1 ? (int)(blockIdx.x % (unsigned)P.nranks) * NLEV : 0;
}

__device__ __forceinline__ void push_task(const ExecParams& P, int s, int phase) {
  const TaskDev& t = P.tasks[s];
  if (t.flags & TF_EXTERNAL) return;  // RECV: completed by the inbox poller
  const int lev = t.level;
  const int qb = P.nranks > 1 ? t.rank * NLEV : 0;  // the queue set of the task's rank
  const int n = group_items(t.kind, P.R, phase);
  const int pos = atomicAdd(&P.q_tail[qb + lev], n);
  unsigned long long* q = P.queue + qoff(P, qb, lev) + pos;
  for (int i = 0; i < n; ++i)
    st_release_u64(q + i, ((unsigned long long)(s + 1) << 32) | ((unsigned)phase << 16) | (unsigned)i);
}

constexpr unsigned long long POP_EXIT = ~0ull;

// Spin until a claimed queue position holds its entry; POP_EXIT if the run
// ends or aborts first (only an overshooting ticket can wait that long).
__device__ __noinline__ unsigned long long wait_entry(const ExecParams& P, const unsigned long long* slot) {
  for (unsigned spin = 0;; ++spin) {
    const unsigned long long v = ld_acquire_u64(slot);
    if (v) return v;
    if ((spin & 63) == 63) {
      if (ld_relaxed_s32(P.abort_flag) || ld_relaxed_s32(P.remaining) <= 0) return POP_EXIT;
      __nanosleep(128);
    }
  }
}

// A fetch-and-add ticket that overshot its level's tail: the position is
// this CTA's (the item pushed there later can only be claimed by it), but the
// producer does not block on it -- it keeps claiming elsewhere and takes the
// owned item on a later pop once it has been pushed. (A blocked producer
// idled its SM for the rest of a draining level: C2's step-3 tail.)
struct OwnedTicket {
  int lev = -1, pos = 0;
};

// Claim attempt over the priority levels (all 32 lanes; lane l holds the
// head / tail snapshot of level l): first the CTA's owned ticket position if
// its item has arrived, then the lowest non-empty level, by CAS on its head
// or -- deep levels, no ticket outstanding -- by a fetch-and-add ticket. The
// entry is read speculatively alongside the CAS (queue entries are written
// once per run), then ordered with an acquire fence. Returns 0 when nothing
// could be claimed.
__device__ __forceinline__ unsigned long long claim_item(const ExecParams& P, int qb, int h, int t, int minback,
                                                         bool tickets, OwnedTicket* own) {
  const int lane = threadIdx.x & 31;
  if (own && own->lev >= 0) {
    unsigned long long v = 0;
    if (lane == 0) v = ld_acquire_u64(P.queue + qoff(P, qb, own->lev) + own->pos);
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v) {
      own->lev = -1;
      return v;
    }
    tickets = false;  // one outstanding ticket per CTA
  }
  unsigned m = __ballot_sync(0xffffffffu, t - h >= minback);
  while (m) {
    const int lev = __ffs(m) - 1;
    unsigned long long v = 0;
    int got = 0, owned = -1;
    if (lane == lev) {
      if (tickets && t - h >= P.ticket_min) {
        // deep level: a fetch-and-add ticket always succeeds in one round trip
        // (148 producers CAS-ing one head convoy at about one claim per round
        // trip). A ticket past the current tail is kept as the CTA's owned
        // position (see OwnedTicket) unless no push can ever reach it.
        const int pos = atomicAdd(P.q_head + qb + lev, 1);
        const int64_t o0 = qoff(P, qb, lev);
        if (pos < qoff(P, qb, lev + 1) - o0) {
          if (pos < ld_relaxed_s32(P.q_tail + qb + lev) || !own) {  // pushed or reserved: the store is in flight
            v = wait_entry(P, P.queue + o0 + pos);
            got = 1;
          } else {
            owned = pos;
          }
        }
        h = t;  // drained by this claim round (or past the level's capacity)
      } else {
        const unsigned long long* slot = P.queue + qoff(P, qb, lev) + h;
        v = ld_relaxed_u64(slot);
        const int prev = atomicCAS(P.q_head + qb + lev, h, h + 1);
        if (prev == h) {
          if (v == 0ull) v = wait_entry(P, slot);  // pusher reserved the slot, store in flight
          fence_acq_rel_gpu();
          got = 1;
        } else {
          h = prev;  // lost the race: retry this level if still non-empty
        }
      }
    }
    const unsigned won = __ballot_sync(0xffffffffu, got);
    if (won) return __shfl_sync(0xffffffffu, v, __ffs(won) - 1);
    owned = __shfl_sync(0xffffffffu, owned, lev);
    if (owned >= 0) {
      own->lev = lev;
      own->pos = owned;
      tickets = false;
    }
    if (lane == lev && t - h < minback) m &= ~(1u << lev);
    m = __shfl_sync(0xffffffffu, m, lev);
  }
  return 0ull;
}

// Non-blocking pop (all 32 lanes): one snapshot of the levels, one claim pass
// over the levels holding at least P.prefetch_min ready items (a lone ready
// item is left to the CTAs that are idle right now).
__device__ __forceinline__ unsigned long long try_pop(const ExecParams& P) {
  static_assert(NLEV <= 32, "one lane per priority level");
  const int lane = threadIdx.x & 31;
  const int qb = cta_qb(P);
  int h = 0, t = 0;
  if (lane < NLEV) {
    h = ld_relaxed_s32(P.q_head + qb + lane);
    t = ld_relaxed_s32(P.q_tail + qb + lane);
  }
  // CAS only: an overshooting ticket could wait for a push behind this CTA's own item
  return claim_item(P, qb, h, t, P.prefetch_min, false, nullptr);
}

// Blocking pop (all 32 lanes): spins until an item is claimed, every task is
// complete, the run aborted, or the watchdog fires.
__device__ unsigned long long pop_item(const ExecParams& P, OwnedTicket& own) {
  const int lane = threadIdx.x & 31;
  const int qb = cta_qb(P);
  unsigned last_prog = ld_relaxed_u32(P.progress);
  unsigned long long t_last = globaltimer();
  const unsigned long long t_enter = t_last;
  unsigned spin = 0;
  while (true) {
    // one round trip: queue bounds of every level and the stop flags together
    int h = 0, t = 0, ab = 0, rem = 1;
    if (lane < NLEV) {
      h = ld_relaxed_s32(P.q_head + qb + lane);
      t = ld_relaxed_s32(P.q_tail + qb + lane);
    }
    if (lane == 0) {
      ab = ld_relaxed_s32(P.abort_flag);
      rem = ld_relaxed_s32(P.remaining);
    }
    if (__shfl_sync(0xffffffffu, ab || rem <= 0, 0)) {
      if (P.cta_idle && spin > 0 && lane == 0) P.cta_idle[blockIdx.x] += globaltimer() - t_enter;
      return POP_EXIT;
    }
    const unsigned long long v = claim_item(P, qb, h, t, 1, true, &own);
    if (v) {
      if (P.cta_idle && spin > 0 && lane == 0) P.cta_idle[blockIdx.x] += globaltimer() - t_enter;
      return v;
    }
    __nanosleep(spin < 64 ? 32 : 256);
    ++spin;
    if ((spin & 255) == 0) {  // watchdog: no item completed anywhere for 30 s
      int quit = 0;
      if (lane == 0) {
        const unsigned pr = ld_relaxed_u32(P.progress);
        const unsigned long long now = globaltimer();
        if (pr != last_prog) {
          last_prog = pr;
          t_last = now;
        } else if (now - t_last > 30ull * 1000000000ull) {
          atomicMin(P.err, ((unsigned long long)0x7fffffffu << 32) | ((unsigned long long)TINV_ERR_INTERNAL << 24));
          atomicExch(P.abort_flag, 1);
          quit = 1;
        }
      }
      if (__shfl_sync(0xffffffffu, quit, 0)) return POP_EXIT;
    }
  }
}

// Storer warp: completion of one work item (all its writes are performed and
// visible). Last item of a task: swap rename slots, release successors.
__device__ void complete_item(const ExecParams& P, const Rec& r) {
  const int task = r.a, ref_id = r.c, fail_code = r.d, fail_index = r.e, phase = r.f;
  const int lane = threadIdx.x & 31;
  int last = 0;
  if (lane == 0) {
    if (fail_code) {
      const unsigned long long key = ((unsigned long long)(unsigned)ref_id << 32) |
                                     ((unsigned long long)fail_code << 24) |
                                     (unsigned long long)(fail_index & 0xffffff);
      atomicMin(P.err, key);
      atomicExch(P.abort_flag, 1);
    } else {
      const TaskDev& t = P.tasks[task];
      const int old = atomicAdd(P.done + task, 1);
      if (old == group_items(t.kind, P.R, phase) - 1) {  // phase group complete
        if (phase + 1 < t.nphases) {
          P.done[task] = 0;  // every item of this phase has finished: no concurrent update
          __threadfence();
          push_task(P, task, phase + 1);
        } else {
          last = 1;
          if (t.flags & TF_RENAMED) {
            const int cs = __ldcg(P.cur_slot + t.out);
            P.cur_slot[t.out] = __ldcg(P.alt_slot + t.out);
            P.alt_slot[t.out] = cs;
          }
          if (P.trace_end) {
            atomicMax(P.trace_end + task, globaltimer() - P.t0);
            P.trace_sm[task] = (int)smid();
          }
          if (t.kind == KIND_SEND) {  // every block item fenced its copy (system scope): raise the flag
            __threadfence_system();
            st_release_sys_s32(P.peer_inbox[t.aux0] + t.aux1, 1);
          }
          if (t.kind == KIND_DEPART) {  // result tile final (and staged): release its copy-engine group
            P.depart_seq[atomicAdd(P.depart_seq_ctr, 1)] = t.aux0;
            __threadfence_system();
            atomicAdd_system(P.depart_count + P.depart_group[t.aux0], 1);
          }
          __threadfence();
        }
      }
    }
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) {
    __syncwarp();
    const TaskDev& t = P.tasks[task];
    for (int k = t.succ_begin + lane; k < t.succ_end; k += 32) {
      const int s = P.succ[k];
      if (atomicSub(P.indeg + s, 1) == 1) {
        if (P.trace_ready) P.trace_ready[s] = globaltimer() - P.t0;
        push_task(P, s, 0);
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicSub(P.remaining, 1);
    }
  }
  if (lane == 0) atomicAdd(P.progress, 1u);
}

// Producer warp (all 32 lanes; lane 0 does the stores, arrivals and TMA
// issues): publish one popped work item to the consumers and stream the
// operand chunks of its GEMM jobs through the TMA ring. When PREFETCH_AT
// chunks are left to issue (the ring is full, the consumers have about
// NSTAGE + PREFETCH_AT chunks of work left), the next item is claimed without
// blocking, hiding the queue round trips; returns it (0: none claimed).
constexpr int PREFETCH_AT = 4;
__device__ __forceinline__ unsigned long long produce_item(unsigned long long e, int slot, const ExecParams& P,
                                                           SmemCtl& ctl, char* ring, const CUtensorMap& tmK,
                                                           const CUtensorMap& tmM, int R, unsigned& ks,
                                                           unsigned& issued) {
  const int lane = threadIdx.x & 31;
  ItemInfo& it = ctl.items[slot];  // built in place
  if (e == POP_EXIT) {
    if (lane == 0) {
      it.task = -1;
      mbar_arrive(&ctl.item_full[slot]);
    }
    return 0ull;
  }
  if (lane == 0) {
    it.task = (int)(e >> 32) - 1;
    const int grp = (int)((e >> 16) & 0xffffu);
    it.item = (int)(e & 0xffffu);
    const TaskDev t = P.tasks[it.task];
    it.kind = t.kind;
    it.ph0 = group_first(t.kind, R, grp);
    it.nph = group_phases(t.kind, R, it.ph0);
    it.phase = it.ph0;  // phase of the first job; the group index travels in `grp`
    it.grp = grp;
    it.step = t.step;
    it.ref_id = t.ref_id;
    it.nitems = t.nitems;
    it.flags = t.flags;
    it.out_s = t.out >= 0 ? __ldcg(P.cur_slot + t.out) : -1;
    it.alt_s = (t.flags & TF_RENAMED) ? __ldcg(P.alt_slot + t.out) : -1;
    it.in0_s = t.in0 >= 0 ? __ldcg(P.cur_slot + t.in0) : -1;
    it.in1_s = t.in1 >= 0 ? __ldcg(P.cur_slot + t.in1) : -1;
    it.scr_s = P.scratch_base + blockIdx.x;
    it.aux0 = t.aux0;
    it.aux1 = t.aux1;
    it.njobs = job_count(it, R);
    for (int jn = 0; jn < it.njobs && jn < MAXJ; ++jn) get_job(it, jn, R, ctl.jobs[slot][jn]);
    fence_proxy_async();  // tiles written by other SMs (generic proxy) -> TMA reads
    mbar_arrive(&ctl.item_full[slot]);
  }
  __syncwarp();
  const int njobs = it.njobs;
  int left = 0;  // chunks left to issue (jobs past MAXJ are not counted: prefetch may come early)
  for (int jn = 0; jn < njobs && jn < MAXJ; ++jn) {
    const Job& j = ctl.jobs[slot][jn];
    if (j.type == J_GEMM) left += (j.k1 - j.k0) * (BLK / KCH);
  }
  unsigned long long next = 0ull;
  bool tried = false;
  for (int jn = 0; jn < njobs; ++jn, ++issued) {
    if (jn >= MAXJ) {
      if (lane == 0) get_job(it, jn, R, ctl.jobs[slot][MAXJ + 1]);
      __syncwarp();
    }
    const Job& jb = ctl.jobs[slot][jn < MAXJ ? jn : MAXJ + 1];
    if (jb.type == J_SPECIAL) {  // it uses the ring as scratch: no loads until it is done
      while (ld_acquire_cta_u32(&ctl.jobs_done) < issued + 1) {
        __nanosleep(200);  // a special job (diagonal chain) runs: leave the issue slots to it
      }
      fence_proxy_async();
      continue;
    }
    if (jb.dep) {
      while (ld_acquire_cta_u32(&ctl.jobs_done) < issued) {
      }
      fence_proxy_async();
    }
    if (lane == 0 && jb.c_s >= 0)  // warm L2 with the C block for the epilogue
      for (int x = 0; x < BLK; x += 16) tma_prefetch3(&tmK, jb.o_c * BLK + x, jb.o_r * BLK, jb.c_s);
    // job fields are re-read from smem (LDS) rather than held across the loop:
    // the producer runs on 56 registers
    for (int kb = jb.k0; kb < jb.k1; ++kb) {
      for (int ch = 0; ch < BLK / KCH; ++ch, ++ks, --left) {
        if (!tried && left <= PREFETCH_AT) {
          tried = true;
          if (P.prefetch_min > 0) next = try_pop(P);
        }
        const int st = ks % NSTAGE;
        mbar_wait(&ctl.empty[st], ((ks / NSTAGE) & 1) ^ 1);
        if (lane == 0) {
          const int ka = jb.a_k0 + (kb - jb.k0), kbb = jb.b_k0 + (kb - jb.k0);
          char* sA = ring + st * STAGE_BYTES;
          char* sB = sA + STAGE_BYTES / 2;
          mbar_arrive_tx(&ctl.full[st], STAGE_BYTES);
          if (jb.variant != V_TN) {  // A K-major
            tma_load3(&tmK, sA, &ctl.full[st], ka * BLK + ch * KCH, jb.a_fix * BLK, jb.a_s);
          } else {
            for (int q = 0; q < 8; ++q)
              tma_load3(&tmM, sA + q * 2048, &ctl.full[st], jb.a_fix * BLK + 16 * q, ka * BLK + ch * KCH, jb.a_s);
          }
          if (jb.variant == V_NT) {  // B K-major
            tma_load3(&tmK, sB, &ctl.full[st], kbb * BLK + ch * KCH, jb.b_fix * BLK, jb.b_s);
          } else {
            for (int q = 0; q < 8; ++q)
              tma_load3(&tmM, sB + q * 2048, &ctl.full[st], jb.b_fix * BLK + 16 * q, kbb * BLK + ch * KCH, jb.b_s);
          }
        }
        __syncwarp();
      }
    }
  }
  return next;
}

// ---------------------------------------------------------------- the kernel
template <bool PROF>
__global__ void __launch_bounds__(NTHREADS, 1)
    exec_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmM,
                const __grid_constant__ CUtensorMap tmE, const __grid_constant__ ExecParams P, int b) {
  extern __shared__ __align__(1024) char dsmem[];
  __shared__ SmemCtl ctl;
  // keep the pointer derived from the __shared__ array (arithmetic through an
  // integer would lose the address space and turn LDS into generic LD)
  char* ring = dsmem + ((1024u - (smem_u32(dsmem) & 1023u)) & 1023u);
  double* S = reinterpret_cast<double*>(ring);  // diagonal phases reuse the drained ring (+ extra)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int R = P.R;

  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&ctl.full[s], 1);
      mbar_init(&ctl.empty[s], NCONS_WARPS);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctl.item_full[s], 1);
      mbar_init(&ctl.item_empty[s], NCONS_WARPS);
      mbar_init(&ctl.stg_free[s], 1);
    }
    for (int s = 0; s < NREC; ++s) {
      mbar_init(&ctl.rec_full[s], 1);
      mbar_init(&ctl.rec_empty[s], 1);
    }
    ctl.jobs_done = 0;
    ctl.fail_code = 0;
    ctl.fail_index = -1;
    ctl.scan_min = -1;
    for (int k = 0; k < 4; ++k) ctl.dbg[k] = 0;
    for (int k = 0; k < 8; ++k) ctl.dbg2[k] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= NCONS_WARPS) {
    // ============================ producer / scheduler warp
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PROD_REGS));
    if (warp == NCONS_WARPS + 1) {
      // ============================ storer warp: epilogue TMA + completion
      unsigned long long sph[4] = {0, 0, 0, 0};  // PROF: quarter, job-end, item-end, idle cycles
      long long stc = clock64();
      for (unsigned idx = 0;; ++idx) {
        const int s = idx % NREC;
        mbar_wait(&ctl.rec_full[s], (idx / NREC) & 1);
        if constexpr (PROF) {
          const long long now = clock64();
          sph[3] += now - stc;
          stc = now;
        }
        const Rec r = ctl.recs[s];
        __syncwarp();
        if (r.type == R_EXIT) break;
        if (r.type == R_QUARTER) {
          if (lane == 0) {
            char* sb = ring + NSTAGE * STAGE_BYTES + r.a * 32768;
            for (int q = 0; q < 8; ++q) {
              if (r.e)
                tma_reduce_add3(&tmE, sb + q * 4096, r.b + 16 * q, r.c, r.d);
              else
                tma_store3(&tmE, sb + q * 4096, r.b + 16 * q, r.c, r.d);
            }
            bulk_commit();
            bulk_wait_read();
            mbar_arrive(&ctl.stg_free[r.a]);
          }
        } else if (r.type == R_JOB_END) {
          if (lane == 0) {
            bulk_wait_all();
            fence_proxy_async();
            st_release_cta_u32(&ctl.jobs_done, (unsigned)r.a);
          }
        } else {
          if (lane == 0) __threadfence();
          __syncwarp();
          complete_item(P, r);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl.rec_empty[s]);
        if constexpr (PROF) {
          const long long now = clock64();
          sph[r.type == R_QUARTER ? 0 : (r.type == R_JOB_END ? 1 : 2)] += now - stc;
          stc = now;
        }
      }
      if constexpr (PROF) {
        if (lane == 0 && P.phase)
          for (int k = 0; k < 4; ++k) P.phase[blockIdx.x * NPHASE + 24 + k] = sph[k];
      }
      return;
    }
    if (warp == NCONS_WARPS + 2) {
      // ============================ inbox pollers (warp 10 of every CTA): complete
      // external tasks (RECV, ARRIVE). CTA b owns inbox entries b, b + G, ...:
      // completions (successor pushes) proceed on all SMs in parallel.
      const int G = gridDim.x, bid = blockIdx.x;
      const int nloc = bid < P.nrecv ? (P.nrecv - bid + G - 1) / G : 0;
      if (nloc == 0) return;
      // Local entries below `lo` are all consumed. Flags mostly arrive in inbox
      // order (ARRIVE: copy order; RECV: send order), so each round scans a
      // window of PWIN local entries from `lo` with all loads in flight at
      // once, and every 64th idle round scans everything beyond it.
      constexpr int PW = 8, PWIN = PW * 32;
      int lo = 0;
      for (unsigned round = 0;; ++round) {
        if (ld_relaxed_s32(P.abort_flag) || ld_relaxed_s32(P.remaining) <= 0) break;
        bool any = false;
        const bool full = (round & 63) == 63;
        for (int base = lo; base < (full ? nloc : min(nloc, lo + PWIN)); base += PWIN) {
          int fl[PW], tk[PW];
#pragma unroll
          for (int k = 0; k < PW; ++k) {
            const int j = base + k * 32 + lane, i = bid + G * j;
            tk[k] = j < nloc ? __ldg(P.recv_task + i) : -1;
            fl[k] = (tk[k] >= 0) ? ld_relaxed_sys_s32(P.inbox + i) : 2;
            if (P.recv_gate && fl[k] == 0)  // gated entry: arrived when its copy run's flag is set
              fl[k] = ld_relaxed_sys_s32(P.gate_flag + __ldg(P.recv_gate + i));
          }
          bool lead = base == lo;  // consumed prefix of the window -> advance lo
#pragma unroll
          for (int k = 0; k < PW; ++k) {
            unsigned m = __ballot_sync(FULL, fl[k] == 1);
            if (m) fence_acq_rel_sys();
            while (m) {
              const int idx = bid + G * (base + k * 32 + __ffs(m) - 1);
              m &= m - 1;
              if (lane == 0) P.inbox[idx] = 2;
              __syncwarp();
              complete_item(P, Rec{R_ITEM_END, P.recv_task[idx], 1, -1, 0, 0, 0, 0});
              any = true;
            }
            const bool done = __all_sync(FULL, fl[k] != 0);
            if (lead && done)
              lo = base + (k + 1) * 32;
            else
              lead = false;
          }
        }
        if (!any) __nanosleep(256);
      }
      return;
    }
    if (warp != NCONS_WARPS) return;
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmM)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmE)) : "memory");
    }
    unsigned ks = 0, issued = 0;
    unsigned long long pph[4] = {0, 0, 0, 0};  // PROF: slot wait, pop, produce cycles, pops
    long long ptc = clock64();
    auto ptick = [&](int k) {
      if constexpr (PROF) {
        const long long now = clock64();
        pph[k] += now - ptc;
        ptc = now;
      }
    };
    unsigned long long next = 0ull;  // item claimed ahead while streaming the previous one
    OwnedTicket own;                 // overshot ticket position of this CTA
    for (unsigned itn = 0;; ++itn) {
      const int slot = itn & 1;
      mbar_wait(&ctl.item_empty[slot], ((itn >> 1) & 1) ^ 1);
      ptick(0);
      const unsigned long long e = next ? next : pop_item(P, own);  // all 32 lanes
      if (P.trace_ready && lane == 0 && e && e != POP_EXIT)  // TINV_READY_PROFILE: first claim of the task
        atomicMin(P.trace_ready + P.ntasks + (int)(e >> 32) - 1, globaltimer() - P.t0);
      ptick(1);
      next = produce_item(e, slot, P, ctl, ring, tmK, tmM, R, ks, issued);
      ptick(2);
      if constexpr (PROF) pph[3] += 1;
      if (e == POP_EXIT) break;
    }
    if constexpr (PROF) {
      if (lane == 0 && P.phase)
        for (int k = 0; k < 4; ++k) P.phase[blockIdx.x * NPHASE + 20 + k] = pph[k];
    }
    return;
  }

  // ============================ consumer warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONS_REGS));
  unsigned ks = 0;
  EpiState es = {0u, 0u, 0u, 0};
  unsigned long long ph[PHASE_BIN0] = {};
  const unsigned long long g_start = globaltimer();
  long long tc = clock64();
  auto tick = [&](int k) {
    if constexpr (PROF) {
      const long long now = clock64();
      ph[k] += (unsigned long long)(now - tc);
      tc = now;
    }
  };
  for (unsigned itn = 0;; ++itn) {
    const int slot = itn & 1;
    mbar_wait(&ctl.item_full[slot], (itn >> 1) & 1);
    if constexpr (PROF) {
      if (tid == 0 && P.phase) {  // item-wait by time bin
        const int bin = (int)min((globaltimer() - g_start) >> 20, (unsigned long long)(PHASE_NBIN - 1));
        P.phase[blockIdx.x * NPHASE + PHASE_BIN0 + bin] += (unsigned long long)(clock64() - tc);
      }
    }
    tick(0);
    const ItemInfo& it = ctl.items[slot];  // stays in smem: the slot is released at item end
    if (it.task < 0) {
      if (tid == 0) push_rec(ctl, es.rec, Rec{R_EXIT, 0, 0, 0, 0, 0, 0, 0});
      break;
    }
    if (tid == 0 && P.trace_start) atomicMin(P.trace_start + it.task, globaltimer() - P.t0);
    int item_generic = 0;
    for (int jn = 0; jn < it.njobs; ++jn) {
      if (jn >= MAXJ) {  // rare: long fused phase groups; build the job in the scratch entry
        cons_bar();
        if (tid == 0) get_job(it, jn, R, ctl.jobs[slot][MAXJ]);
        cons_bar();
      }
      const Job& jb = ctl.jobs[slot][jn < MAXJ ? jn : MAXJ];
      es.generic = 0;
      if (jb.type == J_SPECIAL) {
        drain_jobs(ctl, es);
        run_special(jb, it, P, ctl, S, b);
        es.generic = 1;
      } else if (jb.variant == V_NT) {
        run_gemm<V_NT>(jb, P, ctl, ring, ks, tick, es);
      } else if (jb.variant == V_NN) {
        run_gemm<V_NN>(jb, P, ctl, ring, ks, tick, es);
      } else {
        run_gemm<V_TN>(jb, P, ctl, ring, ks, tick, es);
      }
      tick(2);
      ++es.jobs;
      if (es.generic) {  // generic global writes: visible to the async proxy before the job is done
        fence_proxy_async();
        cons_bar();
        item_generic = 1;
      }
      if (tid == 0) push_rec(ctl, es.rec, Rec{R_JOB_END, (int)es.jobs, 0, 0, 0, 0, 0, 0});
      es.rec += 1;
      tick(3);
    }
    if (item_generic) {
      __threadfence();
      cons_bar();
    }
    tick(4);
    if (tid == 0) {
      push_rec(ctl, es.rec, Rec{R_ITEM_END, it.task, it.nitems, it.ref_id, ctl.fail_code, ctl.fail_index, it.grp, 0});
      ctl.fail_code = 0;
      ctl.fail_index = -1;
    }
    if constexpr (PROF) {
      ph[6] += 1;
      ph[7] += it.njobs;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl.item_empty[slot]);
    es.rec += 1;
    tick(5);
  }
  if constexpr (PROF) {
    if (tid == 0) {
      for (int k = 0; k < 4; ++k) ph[8 + k] = ctl.dbg[k];
      for (int k = 0; k < 8; ++k) ph[12 + k] = ctl.dbg2[k];
      if (P.phase)
        for (int k = 0; k < 20; ++k) P.phase[blockIdx.x * NPHASE + k] = ph[k];
    }
  }
}

// ---------------------------------------------------------------- host launch
int exec_smem_bytes() { return SMEM_BYTES; }

cudaError_t launch_exec(const CUtensorMap& tmK, const CUtensorMap& tmM, const CUtensorMap& tmE, const ExecParams& P,
                        int b, int grid, cudaStream_t stream) {
  auto kern = P.phase ? exec_kernel<true> : exec_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  kern<<<grid, NTHREADS, SMEM_BYTES, stream>>>(tmK, tmM, tmE, P, b);
  return cudaGetLastError();
}

}  // namespace tinv
