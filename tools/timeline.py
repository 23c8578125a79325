"""Per-time-bin picture of one traced inversion: for each bin, the SM-time of
the tasks running in it by step (task span x items, capped at the SM count),
the flop share each step completed, and the critical-path task running.
usage: python tools/timeline.py n b [bin_us] [loops]"""
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from paper_1002_4057_b200 import _native  # noqa: E402

n, b = int(sys.argv[1]), int(sys.argv[2])
bin_us = float(sys.argv[3]) if len(sys.argv) > 3 else 500.0
loops = sys.argv[4] if len(sys.argv) > 4 else "UDU"
t = n // b
R = (b + 127) // 128
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
ctx = _native.Context(n, b)
s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE, loops, True))
table = s.table()
plan = _native.Plan(ctx, table, t, np.zeros(0, np.int64), _native.TRACE)
for _ in range(3):
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, ms = plan.run()
st, en, sm = plan.trace()
names = ["COPY", "POTRF", "TRSM", "SYRK_SUB", "SYRK_ADD_T", "GEMM", "TRTRI", "TRMM_L", "TRMM_RN", "TRMM_LT", "LAUUM"]
kind = table[:, 0]
step = table[:, 1]
# items per task (R x R blocks for block products; diagonal chains 1)
items = np.where(np.isin(kind, [1, 6, 10]), 1, R * R)
t0 = st.min()
st_us, en_us = (st - t0) / 1e3, (en - t0) / 1e3
span = en_us.max()
nb = int(np.ceil(span / bin_us))
busy = np.zeros((nb, 4))
for u in range(len(st)):
    if en[u] <= st[u]:
        continue
    lo, hi = st_us[u], en_us[u]
    for k in range(int(lo // bin_us), min(nb, int(hi // bin_us) + 1)):
        ov = min(hi, (k + 1) * bin_us) - max(lo, k * bin_us)
        if ov > 0:
            busy[k, step[u]] += ov * items[u]
busy /= bin_us * ctx.nsm if hasattr(ctx, "nsm") else bin_us * 148
# critical path
src, dst, _ = _native.dag_edges(table, np.zeros(0, np.int64))
pred = defaultdict(list)
for u, v in zip(src.tolist(), dst.tolist()):
    pred[v].append(u)
v = int(np.argmax(en))
path = []
while True:
    path.append(v)
    if not pred[v]:
        break
    v = max(pred[v], key=lambda q: en[q])
path.reverse()
print(f"n={n} b={b} {loops}: run {ms:.2f} ms, span {span / 1e3:.2f} ms, critical path {len(path)} tasks")
print("bin(ms)  load s0(copy) s1 s2 s3 (task-span x items / SMs; >1 = items queued behind)  critical-path tasks in bin")
for k in range(nb):
    on = [q for q in path if st_us[q] < (k + 1) * bin_us and en_us[q] > k * bin_us]
    desc = ",".join(f"{names[kind[q]]}{tuple(int(x) for x in table[q, 2:4])}" for q in on[:4])
    print(f"{k * bin_us / 1e3:6.2f}  {busy[k].sum():5.2f}  " + " ".join(f"{x:5.2f}" for x in busy[k]) + f"   {desc}")
