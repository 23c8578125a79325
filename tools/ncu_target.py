"""One warm executor launch + one profiled launch (target for ncu -k exec_kernel -s 1 -c 1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
n, b = int(sys.argv[1]), int(sys.argv[2])
pl = sys.argv[3] if len(sys.argv) > 3 else "out"
t = n // b
g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
a = g @ g.T / n
a.diagonal().add_(1.0)
del g
ctx = _native.Context(n, b)
s = P.gen_inversion(t, P.VariantConfig(P.Placement(pl)))
plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
for _ in range(2):
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, ms = plan.run()
    assert rc == 0, plan.msg
print(f"n={n} b={b} {pl}: {ms:.2f} ms {n**3/ms/1e9:.2f} TF/s")
