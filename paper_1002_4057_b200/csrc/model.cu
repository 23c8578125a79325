// Schedule model of the persistent executor (VERDICT r01
// item 3(d)): a discrete-event simulation of the compiled plan -- the same
// exec DAG, phase groups, work items and priority levels the device runs
// (plan_build, csrc/api.cu) -- on `nranks` GPUs of `sms_per_rank` SMs, each
// rank claiming its own tasks from its own level-FIFO queues as
// exec_kernel does (csrc/executor.cu pop_item / push_task). Item costs follow
// the job decomposition of executor.cu get_job_phase: block products of
// 128^3 (a masked diagonal block at a fraction), diagonal-block specials,
// copies. A SEND (one item on the sender) completes its RECV `link` us later.
//
// Host only: runs without a GPU (a shape-only context), so the multi-GPU
// prediction can be checked against the measured single-GPU runs on the box
// and reproduced in the CPU tests.
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <queue>
#include <string>
#include <vector>

#include "host_plan.h"

namespace tinv {
int set_error(int code, const std::string& msg);
}

namespace {

enum Cost {
  C_BLK = 0,      // one 128^3 block product (us)
  C_ITEM,         // per work item: claim, operand prologue, epilogue, completion (us)
  C_BPOTRF,       // 128-block Cholesky + inverse (special job)
  C_BTRTRI,       // 128-block triangular inverse (special job)
  C_BCOPY,        // copy of one 128-block (inverse blocks, COPY rows) (us per block)
  C_SEND,         // SEND: per 128-block of the tile moved by one SM to the peer
  C_LINK,         // SEND completion -> RECV completion on the receiver (us)
  C_MASK,         // cost of a masked (triangular) diagonal block product, in block products
  C_HOP,          // ready -> start latency of an item (queue push, claim, first operand loads) (us)
  NCOST
};

// Cost of one phase's job(s) for item `item` (executor.cu get_job_phase).
double phase_cost(int kind, int step, int flags, int p, int item, int R, const double* c) {
  const double blk = c[C_BLK], m = c[C_MASK];
  auto products = [&](double full, bool masked) { return blk * (full + (masked ? m : 0.0)); };
  (void)step;
  if (kind == KIND_POTRF_INV && p >= 3 * R - 2) {  // X[r][r-s]: (s - 1) full + 1 masked, then 1 masked
    const int s = p - (3 * R - 2) + 1;
    return products(s - 1, true) + products(0, true);
  }
  if (kind == TINV_POTRF || kind == KIND_POTRF_INV) {
    switch (p % 3) {
      case 0: return c[C_BPOTRF];
      case 1: return products(0, true);
      default: return products(1, false);
    }
  }
  if (kind == TINV_TRTRI || kind == KIND_INV) {
    if (p == 0) return (flags & TF_DIAG_FROM_AUX) ? c[C_BCOPY] : c[C_BTRTRI];
    return products(p - 1, true) + products(0, true);
  }
  if (kind == TINV_COPY) return c[C_BCOPY] * R;
  if (kind == KIND_SEND) return c[C_SEND];  // one 128-block per item
  int r, cc;
  if (kind == TINV_SYRK_SUB || kind == TINV_SYRK_ADD_T || kind == TINV_LAUUM) {
    r = 0;
    while ((r + 1) * (r + 2) / 2 <= item) ++r;
    cc = item - r * (r + 1) / 2;
  } else if (kind == TINV_TRSM) {
    cc = R - 1 - item / R;
    r = item % R;
  } else {
    r = item / R;
    cc = item % R;
  }
  switch (kind) {
    case TINV_GEMM:
    case TINV_SYRK_SUB:
    case TINV_SYRK_ADD_T: return products(R, false);
    case TINV_TRMM_LEFT: return products(r, true);
    case TINV_TRMM_RIGHT_NEG: return products(R - cc - 1, true);
    case TINV_TRMM_LEFT_T:
    case TINV_LAUUM: return products(R - r - 1, true);
    case TINV_TRSM: return products(cc, true);
    default: return 0.0;
  }
}

double item_cost(const TaskDev& t, int g, int item, int R, const double* c) {
  const int f = group_first(t.kind, R, g), np = group_phases(t.kind, R, f);
  double s = c[C_ITEM];
  for (int p = f; p < f + np; ++p) s += phase_cost(t.kind, t.step, t.flags, p, np > 1 ? 0 : item, R, c);
  return s;
}

struct Ev {
  double t;
  int64_t seq;
  int32_t task, group, rank;  // group -1: RECV completion
  bool operator>(const Ev& o) const { return t > o.t || (t == o.t && seq > o.seq); }
};

}  // namespace

extern "C" {

// Model run: see include/tileinv_b200.h (tinv_model_run).
int tinv_model_run(int64_t n, int64_t b, const int32_t* table, int64_t ntasks, int32_t stream_t,
                   const int64_t* barriers, int64_t nbar, const int32_t* aux, int64_t nrecv, const int32_t* rank_of,
                   int32_t nranks, int32_t sms_per_rank, uint32_t flags, const double* cost, double* out,
                   double* crit_kind) {
  if (n < 1 || b < 1 || n % b || !cost || !out || nranks < 1 || nranks > MAX_RANKS || sms_per_rank < 1)
    return tinv::set_error(TINV_ERR_BAD_ARG, "bad model arguments");
  tinv_ctx c;  // shape only: no device, no store
  c.n = n;
  c.b = b;
  c.t = n / b;
  c.bp = (b + BLK - 1) / BLK * BLK;
  c.R = c.bp / BLK;
  c.T1 = c.t * (c.t + 1) / 2;
  c.T = c.T1;
  c.nmat = 1;
  c.mslots = 2 * c.T;
  c.nsm = sms_per_rank * nranks;
  tinv_plan* p = nullptr;
  tinv_err err;
  if (flags & ~(uint32_t)TINV_SHARE_SLOTS) return tinv::set_error(TINV_ERR_BAD_ARG, "model: unsupported plan flags");
  int rc = plan_build(&c, table, ntasks, stream_t, barriers, nbar, flags, &p, &err, aux, nrecv,
                      nranks > 1 ? rank_of : nullptr, nranks, true);
  if (rc) return tinv::set_error(rc, "model: " + c.err);
  const int R = (int)c.R;
  const int64_t nx = p->nexec;
  std::vector<int32_t> indeg(p->indeg0), done(nx, 0);
  // ready items: per rank, (level, push order) -- the executor's per-level FIFOs
  struct Ready {
    int64_t key;
    double tready;
    int32_t task, group, item;
    bool operator>(const Ready& o) const { return key > o.key; }
  };
  std::vector<std::priority_queue<Ready, std::vector<Ready>, std::greater<Ready>>> ready(nranks);
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> ev;
  std::vector<int> free_sm(nranks, sms_per_rank);
  std::vector<double> busy(nranks, 0.0);
  int64_t seq = 0;
  double now = 0.0, makespan = 0.0;
  auto push_group = [&](int32_t u, int g) {
    const TaskDev& t = p->tasks[u];
    if (t.flags & TF_EXTERNAL) return;  // RECV: completed by its SEND's arrival
    const int ni = group_items(t.kind, R, g);
    for (int i = 0; i < ni; ++i)
      ready[t.rank].push({((int64_t)t.level << 40) | (seq++ & ((1ll << 40) - 1)), now, u, g, i});
  };
  for (int64_t u = 0; u < nx; ++u)
    if (indeg[u] == 0) push_group((int32_t)u, 0);
  // SEND -> RECV pairing: aux (dest, seq) of the source rows; RECV exec task by inbox sequence
  std::vector<int32_t> recv_of_seq(std::max<int64_t>(nrecv, 1), -1);
  for (int64_t u = 0; u < nx; ++u)
    if (p->tasks[u].kind == KIND_RECV) recv_of_seq[p->tasks[u].aux1] = (int32_t)u;
  int64_t remaining = nx;
  // critical chain: the predecessor whose completion released each task
  std::vector<int32_t> released_by(nx, -1);
  std::vector<double> t_rel(nx, 0.0), t_fin(nx, 0.0);
  auto complete_task = [&](int32_t u, double tt) {
    --remaining;
    makespan = std::max(makespan, tt);
    t_fin[u] = tt;
    const TaskDev& t = p->tasks[u];
    for (int32_t k = t.succ_begin; k < t.succ_end; ++k)
      if (--indeg[p->succ[k]] == 0) {
        released_by[p->succ[k]] = u;
        t_rel[p->succ[k]] = tt;
        push_group(p->succ[k], 0);
      }
    if (t.kind == KIND_SEND) {
      const int32_t rv = recv_of_seq[t.aux1];
      if (rv >= 0) {
        released_by[rv] = u;
        t_rel[rv] = tt;
        ev.push({tt + cost[C_LINK], seq++, rv, -1, -1});
      }
    }
  };
  // dispatch everything startable at `now`
  auto dispatch = [&]() {
    for (int r = 0; r < nranks; ++r)
      while (free_sm[r] > 0 && !ready[r].empty()) {
        const Ready x = ready[r].top();
        ready[r].pop();
        const double d = item_cost(p->tasks[x.task], x.group, x.item, R, cost);
        busy[r] += d;
        --free_sm[r];  // the SM's scheduler claimed it: it starts once its operands stream in
        ev.push({std::max(now, x.tready + cost[C_HOP]) + d, seq++, x.task, x.group, r});
      }
  };
  dispatch();
  while (!ev.empty()) {
    const Ev e = ev.top();
    ev.pop();
    now = e.t;
    if (e.group < 0) {  // RECV arrival
      complete_task(e.task, now);
    } else {
      ++free_sm[e.rank];
      const TaskDev& t = p->tasks[e.task];
      if (++done[e.task] == group_items(t.kind, R, e.group)) {
        done[e.task] = 0;
        if (e.group + 1 < t.nphases)
          push_group(e.task, e.group + 1);
        else
          complete_task(e.task, now);
      }
    }
    if (ev.empty() || ev.top().t > now) dispatch();
  }
  out[0] = makespan;
  for (int r = 0; r < nranks; ++r) out[1 + r] = busy[r];
  out[1 + nranks] = (double)remaining;  // 0 unless the plan deadlocks
  out[2 + nranks] = (double)(2 * c.T + p->dyn_slots + c.nsm);  // tile slots of the device store
  if (crit_kind) {  // time along the chain of releasing predecessors ending at the last task, per kind
    for (int k = 0; k < 17; ++k) crit_kind[k] = 0.0;
    int32_t u = -1;
    for (int64_t v = 0; v < nx; ++v)
      if (u < 0 || t_fin[v] > t_fin[u]) u = (int32_t)v;
    const bool dump = getenv("TINV_MODEL_CHAIN") != nullptr;
    while (u >= 0) {
      const int k = p->tasks[u].kind;
      if (k >= 0 && k < 17) crit_kind[k] += t_fin[u] - t_rel[u];
      if (dump)
        fprintf(stderr, "[chain] exec %d ref %d kind %d step %d out %d in0 %d in1 %d rel %.1f fin %.1f\n", u,
                p->tasks[u].ref_id, k, p->tasks[u].step, p->tasks[u].out, p->tasks[u].in0, p->tasks[u].in1, t_rel[u],
                t_fin[u]);
      u = released_by[u];
    }
  }
  tinv_plan_destroy(p);
  return TINV_OK;
}

}  // extern "C"
