// Host-side context and compiled-plan structures shared by the C-ABI
// (api.cu) and the schedule model (model.cu). Not part of the C-ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "tinv_internal.h"

using namespace tinv;

struct tinv_ctx {
  int64_t n = 0, b = 0, t = 0, bp = 0, R = 0, T = 0;
  int64_t nmat = 1, T1 = 0;  // batched store: nmat matrices of T1 lower tiles each (T = nmat * T1)
  double* bstage = nullptr;  // batched host transfers: whole-batch device staging
  double* peer_pool[MAX_RANKS] = {};     // multi-GPU: peer-mapped pools (null: loopback)
  int32_t* peer_inbox[MAX_RANKS] = {};
  int32_t* inbox = nullptr;              // exported inbox (multi-process)
  int64_t inbox_len = 0;
  bool exported = false;                 // pool mapped by peers: must not move
  bool attached = false;                 // peers mapped by plain pointers (tinv_peer_attach), not IPC
  int rank = -1, world = 0;
  int device = 0, nsm = 0;
  cudaStream_t st = nullptr, st2 = nullptr, own = nullptr;
  cudaStream_t dst[8] = {};  // device -> host copy streams of streamed runs
  double* pool = nullptr;
  int64_t pool_slots = 0, slot_elems = 0;
  std::vector<int32_t> a_slot;  // current slot of each lower tile (its home slot or its shadow T+k)
  std::vector<int32_t> home;    // home slot of each lower tile: a permutation of [0, T) (identity, or
                                // column-major per matrix after a streamed run's reset); -1: a
                                // partitioned store's tile owned by another rank
  std::vector<int32_t> shadow;  // rename shadow slot of each lower tile (T + k; partitioned: compact)
  int64_t mslots = 0;           // slots of the matrix tiles and their shadows (2T; partitioned: 2 x owned)
  bool partitioned = false;     // tinv_create_owned: only this rank's tiles have slots
  int32_t peer_rbase[MAX_RANKS] = {};  // receive-slot base of each peer's store (SEND targets)
  int32_t* d_a_slot = nullptr;
  double* staging[2] = {nullptr, nullptr};
  size_t staging_bytes = 0;
  CUtensorMap tmK, tmM, tmE;
  std::string err;
};

struct tinv_plan {
  tinv_ctx* ctx = nullptr;
  uint32_t flags = 0;
  int64_t nref = 0, nexec = 0, items = 0, nedges = 0;
  std::vector<TaskDev> tasks;
  std::vector<int32_t> succ, indeg0, ref_kind, exec_ref;
  int64_t nlogical = 0;
  std::vector<int32_t> cur0, alt0;  // non-matrix logical tiles (matrix tiles filled at exec)
  int64_t dyn_slots = 0;
  int32_t nranks = 1;            // ranks emulated in one launch (CTA groups with their own queue sets)
  std::vector<int64_t> q_off;     // nranks * NLEV + 1
  int64_t* d_qoffs = nullptr;
  unsigned long long* d_idle = nullptr;  // per CTA: producer idle ns
  int64_t grid = 0;               // CTAs of the last launch
  std::vector<unsigned long long> h_idle;
  std::vector<unsigned long long> q_init;
  std::vector<int32_t> tail0;
  // device state
  TaskDev* d_tasks = nullptr;
  int32_t *d_succ = nullptr, *d_indeg = nullptr, *d_done = nullptr, *d_cur = nullptr, *d_alt = nullptr;
  unsigned long long* d_queue = nullptr;
  int32_t *d_head = nullptr, *d_tail = nullptr, *d_ctr = nullptr;  // ctr: remaining, abort
  unsigned long long* d_err = nullptr;
  unsigned* d_progress = nullptr;
  unsigned long long *d_ts = nullptr, *d_te = nullptr, *d_tr = nullptr;
  int32_t* d_tsm = nullptr;
  int32_t *d_snap_from = nullptr, *d_snap_to = nullptr;
  unsigned long long* d_phase = nullptr;
  int64_t nrecv = 0;
  std::vector<int32_t> recv_task_h;
  std::vector<int32_t> arrive_tile;  // TINV_STREAM_IO: logical tile of inbox index k (copy order)
  std::vector<int32_t> depart_tile;  // matrix tiles in expected completion order (last writer's bottom level)
  std::vector<uint8_t> rename_parity;  // per matrix tile: odd number of renaming writers (final slot = alt)
  int32_t *d_depart_group = nullptr, *d_depart_count = nullptr;
  int32_t *d_depart_seq = nullptr;  // observed completion order of the departures ([T] = counter)
  int32_t *d_recv_gate = nullptr, *d_gate_flag = nullptr;  // streamed arrivals: entry -> copy run, run flags
  int32_t *d_recv_task = nullptr, *d_inbox = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<unsigned long long> h_ts, h_te;
  std::vector<int32_t> h_tsm;
};

// Build a plan for `c` (csrc/api.cu). host_only: no device buffers (the
// schedule model's plans on a shape-only context).
int plan_build(tinv_ctx* c, const int32_t* table, int64_t n, int32_t stream_t, const int64_t* barriers,
               int64_t nbar, uint32_t flags, tinv_plan** out, tinv_err* err, const int32_t* aux, int64_t nrecv,
               const int32_t* rank_of, int32_t nranks, bool host_only);
