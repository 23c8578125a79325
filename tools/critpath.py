"""Trace-based critical path of one inversion: walk back from the last task
through the predecessor that finished last; report time per kind and gaps."""
import sys
from collections import defaultdict
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

n, b = int(sys.argv[1]), int(sys.argv[2])
pl = sys.argv[3] if len(sys.argv) > 3 else "out"
t = n // b
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
ctx = _native.Context(n, b)
s = P.gen_inversion(t, P.VariantConfig(P.Placement(pl)))
table = s.table()
plan = _native.Plan(ctx, table, t, np.zeros(0, np.int64), _native.TRACE)
for _ in range(2):
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, ms = plan.run()
st, en, sm = plan.trace()
src, dst, kind = _native.dag_edges(table, np.zeros(0, np.int64))
pred = defaultdict(list)
for u, v in zip(src.tolist(), dst.tolist()):
    pred[v].append(u)
names = ["COPY", "POTRF", "TRSM", "SYRK_SUB", "SYRK_ADD_T", "GEMM", "TRTRI", "TRMM_L", "TRMM_RN", "TRMM_LT", "LAUUM"]
v = int(np.argmax(en))
path = []
while True:
    path.append(v)
    ps = pred[v]
    if not ps:
        break
    v = max(ps, key=lambda u: en[u])
path.reverse()
busy = defaultdict(float)
cnt = defaultdict(int)
gap = 0.0
prev_end = 0
for v in path:
    k = names[table[v, 0]]
    busy[k] += (en[v] - st[v]) / 1e3
    cnt[k] += 1
    gap += max(0, st[v] - prev_end) / 1e3
    prev_end = en[v]
print(f"n={n} b={b} {pl}: exec {ms:.2f} ms, critical path {len(path)} tasks, span {(en.max() - st.min()) / 1e6:.2f} ms")
print(f"  gaps (ready->start, dispatch) {gap / 1e3:.2f} ms")
for k in sorted(busy, key=lambda x: -busy[x]):
    print(f"  {k:10s} n={cnt[k]:5d} busy {busy[k] / 1e3:8.2f} ms  mean {busy[k] / cnt[k]:8.1f} us")

# gap per transition kind (predecessor kind -> task kind) along the critical path
trans = defaultdict(list)
for u, v in zip(path, path[1:]):
    trans[(names[table[u, 0]], names[table[v, 0]])].append((st[v] - en[u]) / 1e3)
print("  gaps by transition (count, mean us, max us):")
for k, g in sorted(trans.items(), key=lambda kv: -sum(kv[1])):
    print(f"    {k[0]:>10s} -> {k[1]:10s} {len(g):4d} {np.mean(g):8.1f} {np.max(g):8.1f}")

# for the slowest transitions: how many tasks were running when the successor became ready
order = np.argsort(st)
def running_at(t):
    return int(np.sum((st <= t) & (en > t)))
worst = sorted(zip(path, path[1:]), key=lambda uv: -(st[uv[1]] - en[uv[0]]))[:8]
print("  worst gaps: pred -> succ, gap us, tasks running at ready time, succ items' SM")
for u, v in worst:
    print(f"    {names[table[u, 0]]}({u}) -> {names[table[v, 0]]}({v}) gap {(st[v] - en[u]) / 1e3:7.1f} us,"
          f" running {running_at(en[u] + 1)}, sm {sm[v]}")
zero = defaultdict(int)
for v in range(len(en)):
    if en[v] <= st[v] or en[v] == 0:
        zero[names[table[v, 0]]] += 1
print("  tasks with an empty trace span:", dict(zero))
# the worst successor's direct predecessors (reference DAG) with their end times
u0, v0 = worst[0]
print(f"  preds of {names[table[v0, 0]]}({v0}) start {st[v0] / 1e3:.1f} us:",
      [(names[table[q, 0]], int(q), round(en[q] / 1e3, 1)) for q in pred[v0]])
# optional: the critical path's task ids and times, for joining with TINV_DUMP_LEVELS
if len(sys.argv) > 4:
    import json
    with open(sys.argv[4], "w") as fh:
        json.dump({"path": [int(v) for v in path], "st": [int(st[v]) for v in path], "en": [int(en[v]) for v in path],
                   "running_at_ready": [running_at(en[u] + 1) for u in path]}, fh)
# optional: what ran during the worst gaps (kind histogram of the tasks running at the successor's ready time)
if len(sys.argv) > 5:
    for u, v in worst[:4]:
        tr_ = en[u] + 1
        run_ = [q for q in range(len(en)) if st[q] <= tr_ < en[q]]
        started_ = [q for q in range(len(en)) if tr_ <= st[q] < st[v]]
        kinds = defaultdict(int)
        for q in started_:
            kinds[names[table[q, 0]]] += 1
        print(f"  gap before {names[table[v, 0]]}({v}): {len(run_)} running at ready, tasks started inside the gap "
              f"{len(started_)}: {dict(kinds)}; their ids {sorted(started_)[:12]}")
