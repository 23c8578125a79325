// Batched small SPD inversions, pipelined engine (BASELINE config 4: 8192
// independent n = 256 matrices; even 64 <= n <= 256).
//
// The per-matrix computation is the reference's gen_inversion(1) stream --
// POTRF -> TRTRI -> LAUUM of one tile (taskgen.py:178-223 at t = 1;
// kernels.py:59-76, 120-130, 148-151) -- decomposed into a DAG of 64x64 block
// jobs (same block algorithm as csrc/batched.cu's program):
//
//   D(p)      L_pp = chol(A_pp), X_pp = L_pp^-1           (diagonal chain)
//   TRSM(i,p) X_ip = A_ip X_pp^T                          (1 DMMA op, K tri)
//   UPD(p,i,j) X_ij = A_ij - X_ip X_jp^T                  (1 op)
//   TT(i,j)   X_ij = sum_{q=j}^{i-1} X_iq X_qj            (i-j ops)
//   TX(i,j)   X_ij = -X_ii X_ij                           (1 op)
//   W(i,j)    X_ij = X_ji^T = sum_{q>=i} X_qi^T X_qj      (nb-i ops)
//
// The DAG's RAW / WAR / WAW edges come from a scoreboard over the blocks of X
// in program order, exactly as scheduler.py:101-153 builds the tile DAG.
//
// One persistent CTA per SM keeps several matrices in flight and schedules
// their jobs itself:
//   warps 0-3, 4-7   two DMMA groups: a 64x64 output block per job, 32x32
//                    warp tiles, mma.sync m8n8k4 f64 (SASS DMMA.8x8x4) fed
//                    from 128B-swizzled TMA tiles (16-wide K slices);
//   warps 8-11       diagonal group: D jobs (64x64 Cholesky on 8-wide register
//                    panels + bordered inverse, csrc/batched.cu's factor64);
//   warps 12, 13     loaders, one per DMMA group: claim the group's next ready
//                    job (oldest matrix first, then critical-path priority),
//                    stream its operand slices into the group's 4-stage
//                    mbarrier ring with cp.async.bulk.tensor.
// A job completes when its output block is in L2 (generic stores + proxy and
// gpu fences); the completing thread releases successors in shared memory and
// admits the CTA's next matrix (global atomic counter) into a finished slot.
// So one matrix's diagonal chain overlaps other matrices' block products, and
// only W matrices' working blocks compete for L2 per SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>

#include "tinv_internal.h"

namespace tinv {
namespace bpl {

constexpr int BB = 64;
constexpr int NSTG = 3;                    // ring stages per DMMA group
constexpr int SLICE_BYTES = 8192;          // one operand's 64 x 16 K slice
constexpr int STG_BYTES = 2 * SLICE_BYTES; // A + B
constexpr int NMG = 2;                     // DMMA groups
constexpr int NWARPS = 16;                 // four warpgroups (registers rebalanced by setmaxnreg)
constexpr int NTHR = NWARPS * 32;
constexpr int DWARP0 = 8;                  // diagonal group warps 8-11
constexpr int LWARP0 = 12;                 // loader warps 12, 13; storer warps 14, 15
constexpr int MMA_REGS = 160, DIAG_REGS = 152, LOAD_REGS = 40;  // per SMSP: 160 + 160 + 152 + 40 = 512 x 32
constexpr int MAXJ = 48;
constexpr int MAXW = 4;
constexpr int BUFD = BB * BB;
constexpr int RING_BYTES = NMG * NSTG * STG_BYTES;  // 96 KB
constexpr int STAGE_OFF = RING_BYTES;                // per DMMA group: 32 KB output staging (TMA store / C load)
constexpr int DBUF_OFF = STAGE_OFF + NMG * BUFD * 8; // diagonal sub-groups: one 64x64 block each (2 x 32 KB)
constexpr int SCHED_OFF = DBUF_OFF + 2 * BUFD * 8;   // 224 KB, then the scheduler state

enum : int8_t { JD = 0, JTRSM, JUPD, JTT, JTX, JW };
enum : int8_t { V_NT = 0, V_NN = 1, V_TN = 2 };
// warp-uniform zero-slice skips (operand triangular structure; the stored
// blocks carry exact zeros, so skipping is an optimisation, not a mask)
enum : int8_t { SK_NONE = 0, SK_KLEC = 1, SK_KGEC = 2, SK_KLER = 4, SK_KGER = 8, SK_UPPER = 16 };
enum : int8_t { ST_FULL = 0, ST_LOWER = 1, ST_SYM = 2 };
enum : uint8_t { MF_FIRST = 1, MF_LAST = 2, MF_EXIT = 4, MF_NEGC = 8 };

struct JobDef {
  int8_t type, i, j, p;  // p: panel (TRSM / UPD / D)
  int8_t nops, pad0, pad1, pad2;
  unsigned long long succ;  // successor jobs
  int32_t indeg;
  int32_t prio;  // bottom level: longest path to the end of the matrix's DAG (D = 16, a DMMA op = 1)
};

// slice hand-off record (written by the loader before it arms the stage)
struct Meta {
  uint8_t flags, variant, skip, st;
  int8_t oi, oj, sign, carr;  // output block, sign, C array of NEGC (0 A, 1 X)
  int32_t slot, job, mat, pad;
};

struct Sched {
  unsigned long long avail[MAXW];  // ready and unclaimed jobs per slot
  unsigned long long seq[MAXW];    // admission order (older first)
  int32_t indeg[MAXW][MAXJ];
  int32_t ndone[MAXW];
  int32_t mat[MAXW];
  int32_t active, finished, nj, nslots;
  unsigned long long mmask, dmask, init_avail, seqctr;
  int32_t dsel[2][2];  // diagonal sub-groups: claimed slot / job (-1: exit)
  int32_t fail[2];     // diagonal sub-groups: first failing pivot of the current D job
  JobDef jobs[MAXJ];
  Meta meta[NMG][NSTG];
  uint64_t full[NMG][NSTG], empty[NMG][NSTG];
  // output staging hand-off: the group stages a block and arrives `staged`; the
  // storer TMA-stores it, arrives `stgfree` once read, completes the job once
  // written. `cfull`: the loader's TMA load of an UPD job's C block into staging.
  uint64_t staged[NMG], stgfree[NMG], cfull[NMG];
  struct Req {
    int32_t mat, bi, bj, last, slot, job, final_;  // final_: a result block (W), stored evict-first
  } req[NMG];
};
constexpr int SMEM_DYN = SCHED_OFF + ((sizeof(Sched) + 127) / 128) * 128;
static_assert(SMEM_DYN <= 227 * 1024, "shared memory budget");

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
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// a wait that cannot complete (a scheduling bug) traps after 10 s instead of
// hanging the device: the launch fails with an error the host reports
constexpr unsigned long long WATCHDOG_NS = 10000000000ull;
__device__ __forceinline__ void watchdog_trap() { asm volatile("trap;"); }
// (no watchdog here: every wait inlines this loop, and the code must stay
// small -- the four warp roles share each SMSP's instruction cache)
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
// L2 evict-first policy: the input A is read once; the final result blocks are never re-read
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load3_ef(const CUtensorMap* map, void* dst, uint64_t* bar, int x, int y, int z,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store3_ef(const CUtensorMap* map, const void* src, int x, int y, int z,
                                              uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store3(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(const char* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ int rho(int x) { return (x >> 1) | ((x & 1) << 2); }
__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------- job DAG
// Program order (the sequential block program of csrc/batched.cu) and the
// blocks each job reads / writes; edges by a scoreboard over X's blocks.
__device__ void build_dag(Sched& S, int nb) {
  int nj = 0;
  auto add = [&](int8_t type, int i, int j, int p, int nops) {
    JobDef d = {};
    d.type = type, d.i = (int8_t)i, d.j = (int8_t)j, d.p = (int8_t)p, d.nops = (int8_t)nops;
    S.jobs[nj++] = d;
  };
  for (int p = 0; p < nb; ++p) {
    add(JD, p, p, p, 0);
    for (int i = p + 1; i < nb; ++i) add(JTRSM, i, p, p, 1);
    for (int i = p + 1; i < nb; ++i)
      for (int j = p + 1; j <= i; ++j) add(JUPD, i, j, p, 1);
  }
  for (int j = 0; j + 1 < nb; ++j)
    for (int i = j + 1; i < nb; ++i) {
      add(JTT, i, j, 0, i - j);
      add(JTX, i, j, 0, 1);
    }
  for (int i = 0; i < nb; ++i)
    for (int j = 0; j <= i; ++j) add(JW, i, j, 0, nb - i);
  S.nj = nj;
  // scoreboard: last writer and readers since it, per X block (i, j), i >= j
  int last_w[16];
  unsigned long long readers[16];
  for (int b = 0; b < 16; ++b) last_w[b] = -1, readers[b] = 0;
  unsigned long long pred[MAXJ];
  for (int k = 0; k < nj; ++k) pred[k] = 0;
  auto blk = [&](int i, int j) { return i * 4 + j; };
  for (int k = 0; k < nj; ++k) {
    const JobDef& d = S.jobs[k];
    int rd[12], nr = 0, wr = blk(d.i, d.j);
    switch (d.type) {
      case JD:
        if (d.p > 0) rd[nr++] = blk(d.p, d.p);
        break;
      case JTRSM:
        rd[nr++] = blk(d.p, d.p);
        if (d.p > 0) rd[nr++] = blk(d.i, d.p);
        break;
      case JUPD:
        rd[nr++] = blk(d.i, d.p);
        rd[nr++] = blk(d.j, d.p);
        if (d.p > 0) rd[nr++] = blk(d.i, d.j);
        break;
      case JTT:
        for (int q = d.j; q < d.i; ++q) rd[nr++] = blk(d.i, q), rd[nr++] = blk(q, d.j);
        break;
      case JTX:
        rd[nr++] = blk(d.i, d.i);
        rd[nr++] = blk(d.i, d.j);
        break;
      default:
        for (int q = d.i; q < nb; ++q) rd[nr++] = blk(q, d.i), rd[nr++] = blk(q, d.j);
        break;
    }
    for (int r = 0; r < nr; ++r) {
      if (last_w[rd[r]] >= 0 && last_w[rd[r]] != k) pred[k] |= 1ull << last_w[rd[r]];  // RAW
      readers[rd[r]] |= 1ull << k;
    }
    pred[k] |= readers[wr] & ~(1ull << k);                   // WAR
    if (last_w[wr] >= 0) pred[k] |= 1ull << last_w[wr];      // WAW
    last_w[wr] = k;
    readers[wr] = 0;
  }
  S.mmask = S.dmask = S.init_avail = 0;
  for (int k = 0; k < nj; ++k) {
    S.jobs[k].succ = 0;
    S.jobs[k].indeg = __popcll(pred[k]);
    if (S.jobs[k].type == JD) S.dmask |= 1ull << k;
    else S.mmask |= 1ull << k;
    if (!pred[k]) S.init_avail |= 1ull << k;
  }
  for (int k = 0; k < nj; ++k)
    for (int p = 0; p < nj; ++p)
      if (pred[k] >> p & 1) S.jobs[p].succ |= 1ull << k;
  for (int k = nj - 1; k >= 0; --k) {  // edges go from lower to higher ids (program order)
    int best = 0;
    for (int q = k + 1; q < nj; ++q)
      if (S.jobs[k].succ >> q & 1) best = max(best, S.jobs[q].prio);
    S.jobs[k].prio = best + (S.jobs[k].type == JD ? 16 : S.jobs[k].nops);
  }
}
// (job ids are in program order; among ready jobs of a slot the loaders take
// the lowest id, which is the sequential program's order -- the critical
// chain D(p) -> TRSM(p+1,p) -> UPD(p,p+1,p+1) -> D(p+1) comes first)

// ---------------------------------------------------------------- scheduler
// admit the CTA's next matrix into slot s (or retire the slot)
__device__ void admit(Sched& S, int s, int* mat_ctr, int64_t batch) {
  const int m = atomicAdd(mat_ctr, 1);
  if (m >= batch) {
    S.mat[s] = -1;
    if (atomicSub(&S.active, 1) == 1) atomicExch(&S.finished, 1);
    return;
  }
  S.mat[s] = m;
  S.ndone[s] = 0;
#pragma unroll 1
  for (int k = 0; k < S.nj; ++k) S.indeg[s][k] = S.jobs[k].indeg;
  S.seq[s] = atomicAdd(&S.seqctr, 1ull);
  __threadfence_block();
  atomicOr(&S.avail[s], S.init_avail);
}

// claim the best ready job among `mask` types: oldest matrix first, then the
// lowest job id. Returns false when none is ready.
__device__ bool claim(Sched& S, unsigned long long mask, int& slot, int& job) {
  // oldest matrix first, then the lowest job id (program order). (Taking the
  // longest bottom level over all slots instead was measured slower: it
  // spreads the work over more matrices' blocks in L2.)
  for (;;) {
    int best = -1;
    unsigned long long bseq = ~0ull;
#pragma unroll 1
    for (int s = 0; s < S.nslots; ++s) {
      const unsigned long long a = *reinterpret_cast<volatile unsigned long long*>(&S.avail[s]) & mask;
      if (a && S.seq[s] < bseq) best = s, bseq = S.seq[s];
    }
    if (best < 0) return false;
    const unsigned long long a = *reinterpret_cast<volatile unsigned long long*>(&S.avail[best]) & mask;
    if (!a) continue;
    const int j = __ffsll((long long)a) - 1;
    const unsigned long long old = atomicAnd(&S.avail[best], ~(1ull << j));
    if (old >> j & 1) {
      __threadfence_block();
      slot = best;
      job = j;
      return true;
    }
  }
}

// job (slot, j) done: its output block is written (caller fenced)
__device__ void complete(Sched& S, int s, int j, int* mat_ctr, int64_t batch) {
  __threadfence();
  unsigned long long succ = S.jobs[j].succ, newly = 0;
#pragma unroll 1
  while (succ) {
    const int k = __ffsll((long long)succ) - 1;
    succ &= succ - 1;
    if (atomicSub(&S.indeg[s][k], 1) == 1) newly |= 1ull << k;
  }
  if (newly) atomicOr(&S.avail[s], newly);
  if (atomicAdd(&S.ndone[s], 1) == S.nj - 1) admit(S, s, mat_ctr, batch);
}

// ---------------------------------------------------------------- DMMA slice (32x32 warp tile)
// Stage layouts (128B swizzle, 16B chunk c of row r at c ^ (r & 7)):
//  K-major (KM): one TMA box {16 k, 64 rows}: row m at m * 128 B;
//  MN-major (MNM): 4 boxes {16 mn, 16 k} of 2 KB: box v holds mn in [16v, 16v + 16).
// Fragment rows are permuted (rho) so that the 128-bit loads of a quarter warp
// hit 8 distinct 16-byte bank groups (same schemes as csrc/executor.cu's
// chunk_mma, on a 32x32 warp tile).
template <int V>
__device__ __forceinline__ void slice_mma(const char* sA, const char* sB, double (&acc)[4][4][2], int wm, int wn,
                                          int g, int tg) {
  const int rg = rho(g);
  if constexpr (V == V_NT || V == V_NN) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 a[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) a[p] = lds128(sA + (32 * wm + 8 * p + rg) * 128 + (((tg + 4 * h) ^ rg) << 4));
      if constexpr (V == V_NT) {
        double2 b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = lds128(sB + (32 * wn + 8 * q + rg) * 128 + (((tg + 4 * h) ^ rg) << 4));
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma(acc[p][q], a[p].x, b[q].x);
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma(acc[p][q], a[p].y, b[q].y);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 2 * tg + 8 * h + e;
          double2 b[2];
#pragma unroll
          for (int v = 0; v < 2; ++v) b[v] = lds128(sB + (2 * wn + v) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const double av = e ? a[p].y : a[p].x;
            dmma(acc[p][0], av, b[0].x);
            dmma(acc[p][1], av, b[0].y);
            dmma(acc[p][2], av, b[1].x);
            dmma(acc[p][3], av, b[1].y);
          }
        }
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int k = 4 * s + tg;
      const int swz = (rg ^ (k & 7)) << 4;
      double2 a[2], b[2];
#pragma unroll
      for (int w = 0; w < 2; ++w) a[w] = lds128(sA + (2 * wm + w) * 2048 + k * 128 + swz);
#pragma unroll
      for (int v = 0; v < 2; ++v) b[v] = lds128(sB + (2 * wn + v) * 2048 + k * 128 + swz);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
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
  if constexpr (V == V_TN) return 32 * wm + 16 * (p >> 1) + 2 * rho(g) + (p & 1);
  return 32 * wm + 8 * p + rho(g);
}
template <int V>
__device__ __forceinline__ int out_col(int wn, int q, int j) {
  if constexpr (V == V_NT) return 32 * wn + 8 * q + rho(j);
  if constexpr (V == V_NN) return 32 * wn + 16 * (q >> 1) + 2 * j + (q & 1);
  return 32 * wn + 16 * (q >> 1) + 2 * rho(j) + (q & 1);
}

// Epilogue into the staging block: v = sign * acc, or C - acc (C already in
// staging, loaded by the loader); lower / symmetric diagonal outputs skip the
// strictly upper warp tile (symmetric: written as the mirror of the lower
// entries); `tr`: the transposed block (second pass of a symmetric
// off-diagonal output). The staging block is 4 UNswizzled TMA boxes {16 cols,
// 64 rows}: element (r, c) at (c >> 4) * 8192 + r * 128 + (c & 15) * 8, so that
// every element of the warp tile (row r0 + dr[p], column c0 + dc[q] + de[e])
// sits at a row part + a column part from two small per-thread tables -- one
// add and one store per element. (The swizzled, per-variant unrolled version
// overflowed the instruction cache: ncu no_inst stalls, 30K cycles a job.)
__device__ __forceinline__ void stage_out(const Meta& m, const double (&acc)[4][4][2], char* stg, bool tr, int wm,
                                          int wn, int g, int tg) {
  if ((m.skip & SK_UPPER) && wm == 0 && wn == 1) return;
  const int V = m.variant;
  const int r0 = 32 * wm + (V == V_TN ? 2 * rho(g) : rho(g));
  const int c0 = 32 * wn + (V == V_NT ? tg : V == V_NN ? 4 * tg : 2 * tg);
  const int de1 = V == V_NT ? 4 : V == V_NN ? 2 : 8;
  int rr[4], cc[8], ra[4], ca[8];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    rr[p] = r0 + (V == V_TN ? 16 * (p >> 1) + (p & 1) : 8 * p);
    ra[p] = tr ? (rr[p] >> 4) * 8192 + (rr[p] & 15) * 8 : rr[p] * 128;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int q = k >> 1, e = k & 1;
    cc[k] = c0 + (V == V_NT ? 8 * q : 16 * (q >> 1) + (q & 1)) + e * de1;
    ca[k] = tr ? cc[k] * 128 : (cc[k] >> 4) * 8192 + (cc[k] & 15) * 8;
  }
  const bool negc = (m.flags & MF_NEGC) != 0;
  const double sg = (double)m.sign;
  if (V != V_NT && !tr) {  // NN / TN: tiles q = 2h, 2h + 1 hold adjacent columns -> 16-byte stores
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int k = 0; k < 8; k += 4)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          *reinterpret_cast<double2*>(stg + ra[p] + ca[k + e]) =
              make_double2(sg * acc[p][k >> 1][e], sg * acc[p][(k >> 1) + 1][e]);
    return;
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double* d = reinterpret_cast<double*>(stg + ra[p] + ca[k]);
      const double a = acc[p][k >> 1][k & 1];
      *d = negc ? *d - a : sg * a;
    }
}

// symmetric diagonal output: the strictly upper part of the staged block from
// its lower part (after stage_out wrote the lower warp tiles; group barrier first)
__device__ __forceinline__ void stage_mirror_upper(char* stg, int lt) {
#pragma unroll 1
  for (int e = lt; e < BB * BB; e += 128) {
    const int r = e >> 6, c = e & 63;
    if (c > r)
      *reinterpret_cast<double*>(stg + (c >> 4) * 8192 + r * 128 + (c & 15) * 8) =
          *reinterpret_cast<const double*>(stg + (r >> 4) * 8192 + c * 128 + (r & 15) * 8);
  }
}

// ---------------------------------------------------------------- diagonal group (4 warps)
__device__ __forceinline__ int sw(int r, int c) { return r * BB + (c ^ ((r & 3) << 2)); }

// 64x64 block (bi, bj) of an n x n matrix -> S (sw layout) by 64 threads, 16-byte cp.async (n even)
__device__ __forceinline__ void load_blk(double* S, const double* G, int n, int bi, int bj, int lt) {
  const int r0 = bi * BB, c0 = bj * BB;
#pragma unroll 4
  for (int u = 0; u < 32; ++u) {
    const int idx = lt + 64 * u, r = idx >> 5, c = (idx & 31) * 2;
    const bool ok = r0 + r < n && c0 + c < n;
    cp16(S + sw(r, c), ok ? G + (int64_t)(r0 + r) * n + c0 + c : G, ok ? 16 : 0);
  }
  cp_commit();
}

// 1/sqrt(d), d > 0 finite: the MUFU approximation and three Newton steps (full
// double precision; the library rsqrt inlines ~25 instructions of special-case
// handling per call, and the diagonal chain's code must stay small)
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
#pragma unroll
  for (int it = 0; it < 3; ++it) y = fma(y, fma(-h * y, y, 0.5), y);
  return y;
}

// 8x8 Cholesky (right-looking, kernels.py:68-71 failure test) and the inverse
// of the factor, x[i][i] = 1 / L[i][i]; returns the first failing pivot or -1
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
    il[k] = b ? 1.0 : rsqrt_nr(d);
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

// In-place Cholesky + inverse of the 64x64 diagonal block S (sw layout) by a
// two-warp sub-group (lt = 0..63), 8-wide panels. Layout as it proceeds:
// lower 8x8 tiles (i > j): the factor L_ij; diagonal tiles (P, P): X_PP =
// L_PP^-1 (lower); upper tiles (c, R), R > c: X_Rc^T, so the whole inverse
// lives in the block's 32 KB (two sub-groups run two D jobs at once).
// Per panel P: (A) both warps factor the 8x8 diagonal tile in registers
// (chol8_inv) and solve the panel rows below it; (B) X_PP into the diagonal
// tile; (C) trailing update by panel P (DMMA) and the bordered row block P of
// the inverse, X_Pc = -X_PP sum_{k=c}^{P-1} L_Pk X_kc, computed as T^T so that
// no lane transpose is needed.
__device__ void factor64_ip(double* S, int* fail, int lt, int bar, long long* ph) {
  const int warp = lt >> 5, lane = lt & 31, g = lane >> 2, tg = lane & 3;
  long long t0 = clock64();
#pragma unroll 1
  for (int P = 0; P < 8; ++P) {
    const int p0 = 8 * P;
    double x[8][8];
    const int bad = chol8_inv(S, p0, x);
    if (lt == 0 && bad >= 0) atomicMin(fail, p0 + bad);
    const int q = p0 + 8 + lt;
    if (q < BB) {  // panel row: v = a L^-T = a x^T
      double av[8], v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) av[k] = S[sw(q, p0 + k)];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k <= c; ++k) t = fma(av[k], x[c][k], t);
        v[c] = t;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) S[sw(q, p0 + k)] = v[k];
    }
    named_bar(bar, 64);
    {  // X_PP over the (dead) factor tile: thread lt writes element (lt / 8, lt % 8)
      const int i = lt >> 3, j = lt & 7;
      double v = 0.0;
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj <= ii; ++jj) v = (i == ii && j == jj) ? x[ii][jj] : v;
      S[sw(p0 + i, p0 + j)] = v;
    }
    long long t1 = clock64();
    named_bar(bar, 64);
    if (ph) {
      const long long t2 = clock64();
      ph[0] += t1 - t0, ph[1] += t2 - t1, t0 = t2;
    }
    // (C) trailing lower tiles by panel P, then row block P of the inverse
    const int t0r = p0 + 8, nt8 = 7 - P, ntiles = nt8 * (nt8 + 1) / 2;
#pragma unroll 1
    for (int tt = warp; tt < ntiles + P; tt += 2) {
      if (tt < ntiles) {
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
      } else {
        const int c = tt - ntiles, c0 = 8 * c;  // X_Pc, c < P
        // T^T[j][i] = sum_k sum_m X_kc[m][j] L_Pk[i][m]   (X_cc: diagonal tile; X_kc, k > c: tile (c, k) transposed)
        double tT[2] = {0.0, 0.0};
#pragma unroll 1
        for (int k = c; k < P; ++k) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = tg + 4 * h;
            const double a = k == c ? S[sw(c0 + m, c0 + g)] : S[sw(c0 + g, 8 * k + m)];
            dmma(tT, a, S[sw(p0 + g, 8 * k + m)]);
          }
        }
        // X_Pc = -X_PP T: k-steps {2 tg}, {2 tg + 1} so that T's entries are this thread's tT
        double o[2] = {0.0, 0.0};
        dmma(o, S[sw(p0 + g, p0 + 2 * tg)], tT[0]);
        dmma(o, S[sw(p0 + g, p0 + 2 * tg + 1)], tT[1]);
        S[sw(c0 + 2 * tg, p0 + g)] = -o[0];  // transposed into tile (c, P)
        S[sw(c0 + 2 * tg + 1, p0 + g)] = -o[1];
      }
    }
    t1 = clock64();
    named_bar(bar, 64);
    if (ph) {
      const long long t2 = clock64();
      ph[2] += t1 - t0, ph[3] += t2 - t1, t0 = t2;
    }
  }
}

// ---------------------------------------------------------------- kernel
struct Maps {
  CUtensorMap kA, mA, kX, mX;  // operand slices: K-major boxes {16, 64} and MN-major boxes {16, 16}, 128B swizzle
  CUtensorMap uA, uX;          // unswizzled boxes {16, 64}: staging (C loads from A / X, stores to X)
};

// PROF: clock64 spans per role (TINV_BPIPE_PROF=1), summed over CTAs into prof[]:
//  0-3 DMMA group leader: waiting for a stage, slices, epilogue, jobs
//  4-7 loader: no claimable job, waiting for a free stage, claims, waiting for free staging (C loads)
//  8-12 diagonal group leader: no claimable job, block load, factor, store + completion, jobs
//  13-15 storer: waiting for a staged block, store (read) + write completion, jobs
enum { NPROF = 24 };  // 20-23: factor64 phases
template <bool PROF>
__global__ void __launch_bounds__(NTHR, 1)
    k_bpipe(const __grid_constant__ Maps maps, const double* __restrict__ A, double* X, int n, int nb,
            int64_t mstride, int64_t batch, int nslots, int* mat_ctr, unsigned long long* fail, int64_t id0,
            unsigned long long* prof) {
  long long pt = 0, pacc[8] = {};
  auto tick = [&](int c) {
    if constexpr (PROF) {
      const long long now = clock64();
      if (c >= 0) pacc[c] += now - pt;
      pt = now;
    }
  };
  auto flush = [&](int base, int cnt) {
    if constexpr (PROF)
      for (int c = 0; c < cnt; ++c) atomicAdd(prof + base + c, (unsigned long long)pacc[c]);
  };
  extern __shared__ __align__(1024) char dsm[];
  Sched& S = *reinterpret_cast<Sched*>(dsm + SCHED_OFF);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (smem_u32(dsm) & 1023) watchdog_trap();  // 128B-swizzled TMA tiles need 1 KB alignment
    build_dag(S, nb);
    S.nslots = nslots;
    S.active = nslots;
    S.finished = 0;
    S.seqctr = 0;
    for (int s = 0; s < MAXW; ++s) S.avail[s] = 0, S.seq[s] = ~0ull, S.mat[s] = -1;
    for (int gq = 0; gq < NMG; ++gq) {
      for (int st = 0; st < NSTG; ++st) {
        mbar_init(&S.full[gq][st], 1);
        mbar_init(&S.empty[gq][st], 4);
      }
      mbar_init(&S.staged[gq], 4);
      mbar_init(&S.stgfree[gq], 1);
      mbar_init(&S.cfull[gq], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < nslots; ++s) admit(S, s, mat_ctr, batch);
  }
  __syncthreads();

  if (warp >= LWARP0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(LOAD_REGS));
    if (lane != 0) return;
    const int gq = (warp - LWARP0) & 1;
    char* stg = dsm + STAGE_OFF + gq * BUFD * 8;
    if (warp >= LWARP0 + NMG) {
      // ---------------------------------------------------------- storer of DMMA group gq
      unsigned use = 0;
      const uint64_t pol = policy_evict_first();
      tick(-1);
      for (;;) {
        mbar_wait(&S.staged[gq], use & 1);
        tick(0);
        const Sched::Req q = S.req[gq];
        if (q.mat < 0) break;
        if (q.final_) {
#pragma unroll 1
          for (int v = 0; v < 4; ++v) tma_store3_ef(&maps.uX, stg + v * 8192, q.bj * BB + 16 * v, q.bi * BB, q.mat, pol);
        } else {
#pragma unroll 1
          for (int v = 0; v < 4; ++v) tma_store3(&maps.uX, stg + v * 8192, q.bj * BB + 16 * v, q.bi * BB, q.mat);
        }
        bulk_commit();
        bulk_wait_read();
        mbar_arrive(&S.stgfree[gq]);
        if (q.last) {
          bulk_wait_all();
          complete(S, q.slot, q.job, mat_ctr, batch);
          if constexpr (PROF) pacc[2] += 1;
        }
        ++use;
        tick(1);
      }
      flush(13, 3);
      return;
    }
    // ------------------------------------------------------------ loader of DMMA group gq
    char* ring = dsm + gq * NSTG * STG_BYTES;
    const uint64_t pol = policy_evict_first();
    unsigned ks = 0, luse = 0;
    unsigned long long idle_t0 = 0;
    auto arm = [&](const Meta& m) -> char* {
      const int st = ks % NSTG;
      tick(-1);
      mbar_wait(&S.empty[gq][st], ((ks / NSTG) & 1) ^ 1);
      tick(1);
      S.meta[gq][st] = m;
      return ring + st * STG_BYTES;
    };
    tick(-1);
    for (;;) {
      int s, j;
      if (!claim(S, S.mmask, s, j)) {
        if (*reinterpret_cast<volatile int*>(&S.finished)) break;
        if (!idle_t0) idle_t0 = gtimer();
        else if (gtimer() - idle_t0 > WATCHDOG_NS) watchdog_trap();
        __nanosleep(64);
        continue;
      }
      tick(0);
      if constexpr (PROF) pacc[2] += 1;
      idle_t0 = 0;
      fence_proxy_async();
      const JobDef d = S.jobs[j];
      const int mat = S.mat[s];
      Meta m = {};
      m.slot = s, m.job = j, m.mat = mat, m.oi = d.i, m.oj = d.j, m.sign = 1, m.st = ST_FULL, m.carr = 1;
      for (int o = 0; o < d.nops; ++o) {
        // operands of op o: (array, block row, block col) and layout
        int aa = 1, ai = 0, aj = 0, ba = 1, bi = 0, bj = 0;
        m.skip = SK_NONE;
        switch (d.type) {
          case JTRSM:  // X_ip = src_ip X_pp^T
            m.variant = V_NT, aa = d.p ? 1 : 0, ai = d.i, aj = d.p, bi = d.p, bj = d.p, m.skip = SK_KLEC;
            break;
          case JUPD:  // X_ij = src_ij - X_ip X_jp^T
            m.variant = V_NT, ai = d.i, aj = d.p, bi = d.j, bj = d.p;
            m.carr = d.p ? 1 : 0;
            if (d.i == d.j) m.st = ST_LOWER, m.skip = SK_UPPER;
            break;
          case JTT: {  // T = sum_q X_iq X_qj
            const int q = d.j + o;
            m.variant = V_NN, ai = d.i, aj = q, bi = q, bj = d.j;
            if (q == d.j) m.skip = SK_KGEC;
            break;
          }
          case JTX:  // X_ij = -X_ii T
            m.variant = V_NN, ai = d.i, aj = d.i, bi = d.i, bj = d.j, m.skip = SK_KLER, m.sign = -1;
            break;
          default: {  // W: sum_q X_qi^T X_qj
            const int q = d.i + o;
            m.variant = V_TN, ai = q, aj = d.i, bi = q, bj = d.j, m.st = ST_SYM;
            if (q == d.i) m.skip |= SK_KGER | (d.i == d.j ? SK_KGEC : 0);
            if (d.i == d.j) m.skip |= SK_UPPER;
            break;
          }
        }
        const CUtensorMap* mapA = m.variant == V_TN ? (aa ? &maps.mX : &maps.mA) : (aa ? &maps.kX : &maps.kA);
        const CUtensorMap* mapB = m.variant == V_NT ? (ba ? &maps.kX : &maps.kA) : (ba ? &maps.mX : &maps.mA);
#pragma unroll 1
        for (int sl = 0; sl < 4; ++sl) {
          m.flags = (o == 0 && sl == 0 ? MF_FIRST : 0) | (o == d.nops - 1 && sl == 3 ? MF_LAST : 0) |
                    (d.type == JUPD ? MF_NEGC : 0);
          const int st = ks % NSTG;
          char* stage = arm(m);
          uint64_t* bar = &S.full[gq][st];
          mbar_arrive_tx(bar, STG_BYTES);
          if (m.variant == V_TN) {  // A(r, k) = M[k][r]: rows 16 sl.. of block (ai, aj), 4 boxes over its columns
#pragma unroll 1
            for (int v = 0; v < 4; ++v)
              tma_load3(mapA, stage + v * 2048, bar, aj * BB + 16 * v, ai * BB + 16 * sl, mat);
          } else if (aa) {  // A(r, k) = M[r][k]: columns 16 sl.. of the block
            tma_load3(mapA, stage, bar, aj * BB + 16 * sl, ai * BB, mat);
          } else {  // (the input A: read once)
            tma_load3_ef(mapA, stage, bar, aj * BB + 16 * sl, ai * BB, mat, pol);
          }
          if (m.variant == V_NT) {  // B(k, c) = M[c][k]
            tma_load3(mapB, stage + SLICE_BYTES, bar, bj * BB + 16 * sl, bi * BB, mat);
          } else {  // B(k, c) = M[k][c]
#pragma unroll 1
            for (int v = 0; v < 4; ++v)
              tma_load3(mapB, stage + SLICE_BYTES + v * 2048, bar, bj * BB + 16 * v, bi * BB + 16 * sl, mat);
          }
          ++ks;
        }
      }
      if (d.type == JUPD) {  // C block of src into the group's staging once its previous use is stored
        tick(-1);
        mbar_wait(&S.stgfree[gq], (luse & 1) ^ 1);
        tick(3);
        mbar_arrive_tx(&S.cfull[gq], BUFD * 8);
        const CUtensorMap* mapC = d.p ? &maps.uX : &maps.uA;
#pragma unroll 1
        for (int v = 0; v < 4; ++v) {
          if (d.p) tma_load3(mapC, stg + v * 8192, &S.cfull[gq], d.j * BB + 16 * v, d.i * BB, mat);
          else tma_load3_ef(mapC, stg + v * 8192, &S.cfull[gq], d.j * BB + 16 * v, d.i * BB, mat, pol);
        }
      }
      luse += (d.type == JW && d.i != d.j) ? 2 : 1;
    }
    tick(0);
    Meta m = {};
    m.flags = MF_EXIT;
    arm(m);
    mbar_arrive(&S.full[gq][ks % NSTG]);
    flush(4, 4);
    return;
  }

  if (warp >= DWARP0) {
    // ------------------------------------------------------------ diagonal group: two sub-groups of two warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(DIAG_REGS));
    const int sub = (warp - DWARP0) >> 1, lt = tid - (DWARP0 + 2 * sub) * 32, bar = 3 + sub;
    double* Sd = reinterpret_cast<double*>(dsm + DBUF_OFF + sub * BUFD * 8);
    long long dph[4] = {};
    tick(-1);
    for (;;) {
      if (lt == 0) {
        int s = -1, j = -1;
        const unsigned long long t0 = gtimer();
        while (!claim(S, S.dmask, s, j)) {
          if (*reinterpret_cast<volatile int*>(&S.finished)) {
            s = -1;
            break;
          }
          if (gtimer() - t0 > WATCHDOG_NS) watchdog_trap();
          __nanosleep(64);
        }
        S.dsel[sub][0] = s, S.dsel[sub][1] = j;
        S.fail[sub] = 1 << 30;
      }
      named_bar(bar, 64);
      tick(0);
      const int s = S.dsel[sub][0], j = S.dsel[sub][1];
      if (s < 0) break;
      fence_proxy_async();  // X_pp was written by TMA stores
      const int mat = S.mat[s], p = S.jobs[j].p, gr = p * BB;
      const int64_t mo = (int64_t)mat * mstride;
      load_blk(Sd, p ? X + mo : A + mo, n, p, p, lt);
      cp_wait_all();
      named_bar(bar, 64);
#pragma unroll 1
      for (int e = lt; e < BUFD; e += 64) {  // lower part only; identity on the padded diagonal
        const int r = e >> 6, c = e & 63;
        if (c > r) Sd[sw(r, c)] = 0.0;
        else if (c == r && gr + r >= n) Sd[sw(r, c)] = 1.0;
      }
      named_bar(bar, 64);
      tick(1);
      factor64_ip(Sd, &S.fail[sub], lt, bar, PROF && lt == 0 ? dph : nullptr);
      tick(2);
      if (lt == 0 && S.fail[sub] < (1 << 30))
        atomicMin(fail, ((unsigned long long)(id0 + mat) << 32) | (unsigned)(gr + S.fail[sub]));
      double* x = X + mo;
#pragma unroll 1
      for (int e = lt; e < BUFD / 2; e += 64) {  // X_pp = L_pp^-1 (in place: diagonal tiles + transposed upper tiles)
        const int r = e >> 5, c = 2 * (e & 31);
        if (gr + r < n && gr + c < n) {
          double v[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int cc = c + u;
            v[u] = cc > r ? 0.0 : (r >> 3) == (cc >> 3) ? Sd[sw(r, cc)] : Sd[sw(cc, r)];
          }
          *reinterpret_cast<double2*>(x + (int64_t)(gr + r) * n + gr + c) = make_double2(v[0], v[1]);
        }
      }
      fence_proxy_async();
      named_bar(bar, 64);
      if (lt == 0) complete(S, s, j, mat_ctr, batch);
      tick(3);
      if constexpr (PROF) pacc[4] += 1;
    }
    if (lt == 0) {
      flush(8, 5);
      if constexpr (PROF)
        for (int c = 0; c < 4; ++c) atomicAdd(prof + 20 + c, (unsigned long long)dph[c]);
    }
    return;
  }

  // -------------------------------------------------------------- DMMA group gq (warps 4 gq .. 4 gq + 3)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(MMA_REGS));
  const int gq = warp >> 2, wl = warp & 3, wm = wl & 1, wn = wl >> 1, g = lane >> 2, tg = lane & 3;
  const bool leader = wl == 0 && lane == 0;
  const char* ring = dsm + gq * NSTG * STG_BYTES;
  char* stg = dsm + STAGE_OFF + gq * BUFD * 8;
  double acc[4][4][2];
  unsigned ks = 0, use = 0, ccnt = 0;
  // each warp hands its part of the staged block over on its own (the storer's
  // `staged` barrier counts the 4 warps): no group barrier, so a warp whose
  // slices were skipped (triangular operands) moves on to the next job at once
  auto hand_off = [&](int bi, int bj, int mat, int last, int slot, int job, int final_) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (wl == 0) S.req[gq] = Sched::Req{mat, bi, bj, last, slot, job, final_};
      mbar_arrive(&S.staged[gq]);
    }
    ++use;
  };
  tick(-1);
  for (;;) {
    const int st = ks % NSTG;
    mbar_wait(&S.full[gq][st], (ks / NSTG) & 1);
    tick(0);
    const Meta m = S.meta[gq][st];
    if (m.flags & MF_EXIT) break;
    if (m.flags & MF_FIRST) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q][0] = acc[p][q][1] = 0.0;
    }
    const int sl = ks & 3;  // every op is 4 slices
    const int k0 = 16 * sl;
    bool skip = (m.skip & SK_UPPER) && wm == 0 && wn == 1;
    if ((m.skip & SK_KLEC) && k0 > 32 * wn + 31) skip = true;
    if ((m.skip & SK_KGEC) && k0 + 15 < 32 * wn) skip = true;
    if ((m.skip & SK_KLER) && k0 > 32 * wm + 31) skip = true;
    if ((m.skip & SK_KGER) && k0 + 15 < 32 * wm) skip = true;
    const char* sA = ring + st * STG_BYTES;
    if (!skip) {
      if (m.variant == V_NT) slice_mma<V_NT>(sA, sA + SLICE_BYTES, acc, wm, wn, g, tg);
      else if (m.variant == V_NN) slice_mma<V_NN>(sA, sA + SLICE_BYTES, acc, wm, wn, g, tg);
      else slice_mma<V_TN>(sA, sA + SLICE_BYTES, acc, wm, wn, g, tg);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[gq][st]);
    ++ks;
    tick(1);
    if (m.flags & MF_LAST) {
      if constexpr (PROF) {  // split the DMMA drain (results of the last slice) from the staging stores
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) asm volatile("" ::"d"(acc[p][q][0]), "d"(acc[p][q][1]));
        tick(7);
      }
      mbar_wait(&S.stgfree[gq], (use & 1) ^ 1);
      if (m.flags & MF_NEGC) mbar_wait(&S.cfull[gq], ccnt++ & 1);
      tick(4);
      const bool mirror = m.st == ST_SYM && m.oi != m.oj;
      for (int pass = 0; pass < 1 + mirror; ++pass) {  // pass 1: the transposed block (j, i)
        if (pass) mbar_wait(&S.stgfree[gq], (use & 1) ^ 1);
        tick(4);
        stage_out(m, acc, stg, pass == 1, wm, wn, g, tg);
        if (m.st == ST_SYM && m.oi == m.oj) {
          named_bar(1 + gq, 128);
          stage_mirror_upper(stg, tid & 127);
        }
        tick(5);
        const int fin = m.st == ST_SYM;
        if (pass) hand_off(m.oj, m.oi, m.mat, 1, m.slot, m.job, fin);
        else hand_off(m.oi, m.oj, m.mat, !mirror, m.slot, m.job, fin);
        tick(6);
      }
      tick(2);
      if constexpr (PROF) pacc[3] += 1;
    }
  }
  mbar_wait(&S.stgfree[gq], (use & 1) ^ 1);
  if (lane == 0) {
    if (wl == 0) S.req[gq].mat = -1;
    mbar_arrive(&S.staged[gq]);
  }
  if (leader) {
    flush(0, 4);
    if constexpr (PROF)
      for (int c = 4; c < 8; ++c) atomicAdd(prof + 16 + c - 4, (unsigned long long)pacc[c]);
  }
}

}  // namespace bpl

// engine selection (tinv_batch_small_engine; initial value from TINV_BSMALL_ENGINE)
static int g_bsmall_engine = -1;
static int bsmall_engine() {
  if (g_bsmall_engine < 0)
    g_bsmall_engine = getenv("TINV_BSMALL_ENGINE") && std::string(getenv("TINV_BSMALL_ENGINE")) == "pipe"
                          ? TINV_BSMALL_PIPE
                          : TINV_BSMALL_CTA;
  return g_bsmall_engine;
}

typedef CUresult (*EncodeTiledFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Pipelined engine for even 64 <= n <= 256 (TMA needs 16-byte row strides).
// Returns cudaErrorNotSupported when the shape is not covered (the caller runs
// the one-CTA-per-matrix engine).
cudaError_t launch_bpipe(const double* dA, double* dX, int64_t batch, int64_t n, int64_t stride, cudaStream_t st,
                         unsigned long long* dfail, int64_t id0) {
  if (bsmall_engine() != TINV_BSMALL_PIPE || (n & 1) || n < 64 || n > 256 || (stride & 1))
    return cudaErrorNotSupported;
  static EncodeTiledFn2 enc = nullptr;
  static int* dctr[64] = {};
  static int nsm[64] = {};
  static unsigned long long* dprof[64] = {};
  static const int prof_mode = getenv("TINV_BPIPE_PROF") && atoi(getenv("TINV_BPIPE_PROF")) ? 1 : 0;
  int dev = 0;
  cudaError_t r = cudaGetDevice(&dev);
  if (r != cudaSuccess) return r;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    r = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (r != cudaSuccess) return r;
    if (!p || q != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
    enc = (EncodeTiledFn2)p;
  }
  if (!dctr[dev]) {
    r = cudaFuncSetAttribute(bpl::k_bpipe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bpl::SMEM_DYN);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(bpl::k_bpipe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bpl::SMEM_DYN);
    if (r == cudaSuccess) r = cudaMalloc(&dprof[dev], bpl::NPROF * sizeof(unsigned long long));
    if (r == cudaSuccess) r = cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev);
    if (r == cudaSuccess) r = cudaMalloc(&dctr[dev], 64 * sizeof(int));
    if (r != cudaSuccess) return r;
  }
  static const int nslots_env = getenv("TINV_BPIPE_SLOTS") ? atoi(getenv("TINV_BPIPE_SLOTS")) : 4;
  const int nslots = nslots_env < 1 ? 1 : nslots_env > bpl::MAXW ? bpl::MAXW : nslots_env;
  const int nb = (int)((n + bpl::BB - 1) / bpl::BB);
  for (int64_t b0 = 0; b0 < batch; b0 += 0x7fffffff) {
    const int64_t cnt = batch - b0 < 0x7fffffff ? batch - b0 : 0x7fffffff;
    bpl::Maps maps;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)cnt};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)stride * 8};
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint32_t boxK[3] = {16, 64, 1}, boxM[3] = {16, 16, 1};
    CUtensorMap* outs[6] = {&maps.kA, &maps.mA, &maps.kX, &maps.mX, &maps.uA, &maps.uX};
    for (int k = 0; k < 6; ++k) {
      void* base = (void*)(((k == 0 || k == 1 || k == 4) ? (const double*)dA : (const double*)dX) + b0 * stride);
      const CUresult cr =
          enc(outs[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, k == 1 || k == 3 ? boxM : boxK, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, k >= 4 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    r = cudaMemsetAsync(dctr[dev], 0, sizeof(int), st);
    if (r != cudaSuccess) return r;
    const int grid = (int)(cnt < nsm[dev] ? cnt : nsm[dev]);
    if (prof_mode) {
      cudaMemsetAsync(dprof[dev], 0, bpl::NPROF * sizeof(unsigned long long), st);
      bpl::k_bpipe<true><<<grid, bpl::NTHR, bpl::SMEM_DYN, st>>>(maps, dA + b0 * stride, dX + b0 * stride, (int)n, nb,
                                                                 stride, cnt, nslots, dctr[dev], dfail, id0 + b0,
                                                                 dprof[dev]);
    } else {
      bpl::k_bpipe<false><<<grid, bpl::NTHR, bpl::SMEM_DYN, st>>>(maps, dA + b0 * stride, dX + b0 * stride, (int)n,
                                                                  nb, stride, cnt, nslots, dctr[dev], dfail, id0 + b0,
                                                                  nullptr);
    }
    r = cudaGetLastError();
    if (r != cudaSuccess) return r;
    if (prof_mode) {
      unsigned long long h[bpl::NPROF];
      cudaMemcpyAsync(h, dprof[dev], sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double per = (double)cnt;  // cycles per matrix (summed over CTAs / groups)
      fprintf(stderr,
              "[tinv bpipe] per matrix: DMMA groups wait %.0f slices %.0f epilogue %.0f (jobs %.1f) | loaders idle "
              "%.0f stage-wait %.0f (claims %.1f) C-wait %.0f | diag idle %.0f load %.0f factor %.0f store %.0f (jobs "
              "%.1f) | storers wait %.0f store %.0f (jobs %.1f)\n",
              h[0] / per, h[1] / per, h[2] / per, h[3] / per, h[4] / per, h[5] / per, h[6] / per, h[7] / per,
              h[8] / per, h[9] / per, h[10] / per, h[11] / per, h[12] / per, h[13] / per, h[14] / per, h[15] / per);
      fprintf(stderr, "[tinv bpipe] epilogue: staging-wait %.0f stage %.0f hand-off %.0f dmma-drain %.0f\n",
              h[16] / per, h[17] / per, h[18] / per, h[19] / per);
      fprintf(stderr, "[tinv bpipe] factor64_ip (both sub-groups): factor+solve+X_PP %.0f bar %.0f update+border %.0f bar %.0f\n",
              h[20] / per, h[21] / per, h[22] / per, h[23] / per);
    }
  }
  return cudaSuccess;
}

}  // namespace tinv

extern "C" int tinv_batch_small_engine(int engine) {
  const int prev = tinv::bsmall_engine();
  if (engine == TINV_BSMALL_CTA || engine == TINV_BSMALL_PIPE) tinv::g_bsmall_engine = engine;
  return prev;
}
