// Internal structures shared by the host planner (plan.cpp) and the device
// executor (executor.cu). Not part of the C-ABI.
#pragma once
#include <stdint.h>

#include "../../include/tileinv_b200.h"

namespace tinv {

// The sub-tile ("block") every device job works on: 128 x 128 FP64.
constexpr int BLK = 128;
// Work-item queue priority levels (0 = most critical).
constexpr int NLEV = 32;
// Executor CTA: two consumer warpgroups (8 DMMA warps) + one producer
// warpgroup (warp 8 = scheduler + TMA issue); registers are rebalanced with
// setmaxnreg (producer 56, consumers 224).
constexpr int NCONS_WARPS = 8;
constexpr int NTHREADS = (NCONS_WARPS + 4) * 32;
constexpr int PROD_REGS = 56;
constexpr int CONS_REGS = 224;
// TMA ring: stages of (A 128x16 + B 128x16) doubles.
constexpr int NSTAGE = 4;
constexpr int KCH = 16;                         // K per chunk
constexpr int STAGE_BYTES = 2 * BLK * KCH * 8;  // 32 KB
constexpr int EXTRA_SMEM = 64 * 1024;           // extra scratch for diagonal phases
constexpr int SMEM_BYTES = NSTAGE * STAGE_BYTES + EXTRA_SMEM + 2048;



// Hidden task kind inserted by the planner: INV(L) -> aux = tril(L)^-1,
// shared by every TRSM reading that version of L (TRSM then runs as a
// DMMA triangular multiply by the inverse).
constexpr int KIND_INV = 11;
// Multi-GPU transfer pseudo-tasks (csrc/api.cu tinv_plan_create_dist):
// SEND copies a tile version into the receiver's pool (peer memory; one item
// per 128-block) and, once every block is out, sets the receiver's inbox flag;
// RECV is completed by the receiver's inbox poller.
constexpr int KIND_SEND = 12;
constexpr int KIND_RECV = 13;
constexpr int MAX_RANKS = 8;
// Streamed host I/O pseudo-tasks (TINV_STREAM_IO plans): ARRIVE writes an
// input tile (the copy engine does; completed by the inbox poller when its
// arrival flag is set); DEPART reads a final result tile (SYMMETRIZE: writes
// its transposed / mirrored copy into a staging slot, one item per 128-block)
// and, when complete, counts it in its copy group, which the copy engines
// wait on before moving the tile to the host.
constexpr int KIND_ARRIVE = 14;
constexpr int KIND_DEPART = 15;
// POTRF whose aux tile receives the factor's full inverse (planner upgrade of
// a POTRF whose factor a TRSM reads: TRSM multiplies by the aux directly).
constexpr int KIND_POTRF_INV = 16;

enum TaskFlags : int32_t {
  TF_RENAMED = 1,   // output written to the alternate slot, slots swapped at completion
  TF_EXTERNAL = 2,  // never queued: completed by the inbox poller (RECV, ARRIVE)
  TF_DIAG_FROM_AUX = 4,  // TRTRI / INV: diagonal-block inverses copied from the POTRF aux tile (in1)
  TF_NO_MIRROR = 8,      // SYRK_SUB whose tile is next factored by POTRF (through SYRK_SUBs only): the
                         // strict upper part is dead, so the lower blocks reduce-add with no mirror
};

struct TaskDev {
  int8_t kind;
  int8_t step;
  int8_t flags;
  int8_t level;
  int16_t nphases;  // phase groups (queue round trips) of the task
  int8_t rank;      // ranks-in-one-launch plans: the rank (CTA group) that runs it; else 0
  int8_t pad;
  int32_t nitems;   // items over all phases
  int32_t out;     // logical tile ids
  int32_t in0;
  int32_t in1;
  int32_t ref_id;  // reference task id (errors / trace)
  int32_t succ_begin;
  int32_t succ_end;
  int32_t aux0;    // SEND: destination rank; DEPART: matrix tile id (staging slot / copy group)
  int32_t aux1;    // SEND / RECV / ARRIVE: inbox index (RECV: slot recv_base + seq); DEPART: i << 16 | j
};

struct ExecParams {
  double* pool;            // all tile slots, slot s at pool + s * slot_elems
  int64_t slot_elems;      // bp * bp
  int32_t bp;              // padded tile order (multiple of BLK)
  int32_t R;               // bp / BLK
  int32_t b;               // the tile order itself (rows / columns >= b of a slot are padding)
  int32_t ntasks;
  int32_t scratch_base;    // slot of CTA 0's scratch tile; CTA c uses scratch_base + c
  const TaskDev* tasks;
  const int32_t* succ;
  int32_t* indeg;
  int32_t* done;           // items finished per task
  int32_t* cur_slot;       // logical tile -> physical slot (mutable: renaming)
  int32_t* alt_slot;
  unsigned long long* queue;       // all levels back to back
  int64_t q_off[NLEV + 1];         // level l occupies queue[q_off[l] .. q_off[l+1])
  int32_t* q_head;                 // NLEV (x nranks)
  int32_t* q_tail;                 // NLEV (x nranks)
  // ranks emulated in one launch (nranks > 1): CTA b is rank b % nranks and
  // claims only from its rank's NLEV levels; level l of rank r occupies
  // queue[q_offs[r*NLEV + l] .. q_offs[r*NLEV + l + 1]) (q_off unused)
  int32_t nranks;
  const int64_t* q_offs;           // nranks * NLEV + 1
  unsigned long long* cta_idle;    // optional: per CTA, ns its producer waited for a claimable item
  int32_t* remaining;              // tasks not yet completed
  int32_t* abort_flag;
  unsigned long long* err;         // packed min failure (ref task << 32 | code << 24 | index)
  unsigned int* progress;          // completed items (watchdog)
  unsigned long long* trace_start; // per exec task, optional
  unsigned long long* trace_end;
  unsigned long long* trace_ready;  // optional (TRACE): time the task became ready (in-degree 0)
  int32_t* trace_sm;
  unsigned long long t0;           // globaltimer at launch (trace base)
  unsigned long long* phase;       // optional per-CTA phase cycle counters (NPHASE each)
  int prefetch_min;                // claim the next item ahead only from levels with this backlog (0: never)
  int ticket_min;                  // levels with at least this backlog are claimed by fetch-and-add
  // multi-GPU transfers
  double* peer_pool[MAX_RANKS];    // pools of the ranks (peer-mapped; the local pool for self)
  int32_t* peer_inbox[MAX_RANKS];  // inbox flag arrays of the ranks
  int32_t* inbox;                  // this rank's inbox flags (1 = arrived, 2 = consumed)
  const int32_t* recv_task;        // inbox index -> exec task id (-1: not received here)
  int32_t nrecv;                   // inbox length
  int32_t recv_base;               // slot of this store's receive sequence number 0
  int32_t peer_recv_base[MAX_RANKS];  // the same in each peer's store (SEND targets; differs when partitioned)
  const int32_t* recv_gate;        // streamed arrivals: entry -> copy run (null: the entry's own inbox flag)
  const int32_t* gate_flag;        // per copy run: 1 = arrived (stream write-value)
  // streamed host output (DEPART; the copy engines do the device -> host moves)
  int32_t depart_mode;             // TINV_DENSE_LOWER_TILES / TINV_DENSE_SYMMETRIZE
  int32_t stage_base;              // slot of the staging tile of matrix tile 0 (SYMMETRIZE)
  const int32_t* depart_group;     // matrix tile -> copy group
  int32_t* depart_count;           // per copy group: departed tiles (the copy streams wait on it)
  int32_t* depart_seq;             // observed departure order (matrix tile ids)
  int32_t* depart_seq_ctr;
};
constexpr int NPHASE = 60;  // item-wait, mainloop, epilogue, job-end, item-end, completion, items, jobs,
                            // special: load, factor, inverse, store; potrf/trtri sub-steps;
                            // producer: slot-wait, pop, produce, pops; storer: quarters, job-end, item-end, idle;
                            // 28..59: consumer item-wait cycles in 2^20 ns (~1 ms) bins from the CTA's start
constexpr int PHASE_BIN0 = 28, PHASE_NBIN = 32;

inline int64_t tri_index(int64_t i, int64_t j) { return i * (i + 1) / 2 + j; }

#ifdef __CUDACC__
#define TINV_HD __host__ __device__ __forceinline__
#else
#define TINV_HD inline
#endif

// Phases of a task over tiles of R x R blocks (128 x 128).
//  POTRF (3R-2 phases): d = p/3; p%3 == 0: factor + invert diagonal block d
//    (1 item; the inverse block goes to the aux tile); 1: block TRSMs A[r][d]
//    <- A[r][d] inv(L_dd)^T, r > d (R-1-d); 2: trailing block updates
//    A[r][c] -= A[r][d] A[c][d]^T, r >= c > d.
//  POTRF_INV (4R-3 phases): POTRF's, then s = p-(3R-2)+1 = 1..R-1: the
//    off-diagonal blocks X[r][r-s] of X = L^-1 in the aux tile (R-s items,
//    two block GEMMs each), so the aux holds the factor's full inverse (TRSM
//    multiplies by it, TRTRI of the factor copies it).
//  TRTRI / INV (R phases): 0: invert every diagonal block (R items);
//    s >= 1: X[r][r-s] for r = s..R-1 (R-s items, two block GEMMs each).
//  everything else: one phase.
TINV_HD int phases_of(int kind, int R) {
  if (kind == KIND_SEND || kind == KIND_RECV || kind == KIND_ARRIVE) return 1;
  if (kind == TINV_POTRF) return 3 * R - 2;
  if (kind == KIND_POTRF_INV) return 4 * R - 3;
  if (kind == TINV_TRTRI || kind == KIND_INV) return R;
  return 1;
}
TINV_HD int phase_items(int kind, int R, int p) {
  switch (kind) {
    case TINV_POTRF:
    case KIND_POTRF_INV: {
      if (p >= 3 * R - 2) return R - (p - (3 * R - 2) + 1);  // inverse phases (POTRF_INV)
      const int d = p / 3, m = R - 1 - d;
      return p % 3 == 0 ? 1 : (p % 3 == 1 ? m : m * (m + 1) / 2);
    }
    case TINV_TRTRI:
    case KIND_INV:
      return p == 0 ? R : R - p;
    case TINV_SYRK_SUB:
    case TINV_SYRK_ADD_T:
    case TINV_LAUUM:
      return R * (R + 1) / 2;
    case TINV_COPY:
      return R;
    case KIND_RECV:
    case KIND_ARRIVE:
      return 1;
    case KIND_SEND:  // one item per 128-block: the tile crosses NVLink from R^2 SMs at once
      return R * R;
    default:
      return R * R;
  }
}
// Phase groups: a run of consecutive single-item phases is fused into one
// work item (its jobs run back to back on one CTA, no queue round trip); a
// phase with several items is a group of its own.
// group_first(kind, R, g) -> first phase of group g; -1 past the end.
TINV_HD int group_first(int kind, int R, int g) {
  const int np = phases_of(kind, R);
  int p = 0;
  for (int k = 0; k < g && p < np; ++k) {
    if (phase_items(kind, R, p) > 1) {
      ++p;
    } else {
      while (p < np && phase_items(kind, R, p) == 1) ++p;
    }
  }
  return p < np ? p : -1;
}
TINV_HD int group_phases(int kind, int R, int first) {  // phases in the group starting at `first`
  if (phase_items(kind, R, first) > 1) return 1;
  int p = first;
  while (p < phases_of(kind, R) && phase_items(kind, R, p) == 1) ++p;
  return p - first;
}
TINV_HD int ngroups(int kind, int R) {
  int g = 0;
  while (group_first(kind, R, g) >= 0) ++g;
  return g;
}
TINV_HD int group_items(int kind, int R, int g) {
  const int f = group_first(kind, R, g);
  return f < 0 ? 0 : phase_items(kind, R, f);
}
TINV_HD int total_items(int kind, int R) {
  int n = 0;
  for (int g = 0; g < ngroups(kind, R); ++g) n += group_items(kind, R, g);
  return n;
}

}  // namespace tinv
