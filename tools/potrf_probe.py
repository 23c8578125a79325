"""Latency of the step-1 chain tasks at nb=256 (C2's critical path): a t=2
step-1 stream (POTRF_INV(0) -> TRSM(1,0) -> SYRK_SUB(1,1) -> POTRF(1)) with
per-task device timestamps, plus TINV_PHASE_PROFILE counters when set."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from paper_1002_4057_b200 import _native  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = b * t
g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
a = g @ g.T / n
a.diagonal().add_(1.0)
ctx = _native.Context(n, b)
s = P.gen_step1(t)
plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.TRACE)
assert plan.rc == 0, plan.msg
best = None
for rep in range(5):
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, ms = plan.run()
    assert rc == 0, plan.msg
    st, en, sm = plan.trace()
    if best is None or ms < best[0]:
        best = (ms, st.copy(), en.copy())
ms, st, en = best
t0 = st.min()
print(f"b={b} t={t}: step-1 run {ms * 1e3:.1f} us")
for k, task in enumerate(s.tasks):
    kind = task.kind.value if task.kind else "COPY"
    print(f"  {kind:10s} {str(task.indices):12s} start {(st[k] - t0) / 1e3:8.1f} us  dur {(en[k] - st[k]) / 1e3:8.1f} us")
