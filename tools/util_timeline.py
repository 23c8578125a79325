"""Items in flight over time for one full inversion (device trace of every
task: start = first item start, end = last item end; a task's items are
spread uniformly over its span): SM-occupancy timeline in 2 % buckets."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

n, b = int(sys.argv[1]), int(sys.argv[2])
loops = sys.argv[3] if len(sys.argv) > 3 else "UDU"
t = n // b
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
del g
ctx = _native.Context(n, b)
s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE, loops))
plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.TRACE)
for _ in range(2):
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, ms = plan.run()
st, en, sm = plan.trace()
R = (b + 127) // 128
items = {0: R, 1: 1, 2: R * R, 3: R * (R + 1) // 2, 4: R * (R + 1) // 2, 5: R * R, 6: R, 7: R * R, 8: R * R, 9: R * R,
         10: R * (R + 1) // 2}
kinds = s.table()[:, 0]
T = en.max()
nb_ = 50
edges = np.linspace(0, T, nb_ + 1)
busy = np.zeros(nb_)
for k in range(len(st)):
    if st[k] < 0:
        continue
    span = max(en[k] - st[k], 1)
    w = items[int(kinds[k])] * 70e3  # ~70 us per 128-block item at C3-like K (rough weight)
    lo, hi = st[k], en[k]
    for bi in range(nb_):
        ov = min(hi, edges[bi + 1]) - max(lo, edges[bi])
        if ov > 0:
            busy[bi] += w * ov / span
cap = 148 * (T / nb_)
print(f"n={n} b={b} {loops}: {ms:.1f} ms; estimated SM occupancy per 2% of the run:")
print(" ".join(f"{min(1.0, x / cap) * 100:3.0f}" for x in busy))
