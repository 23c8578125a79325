"""Phase profile of full inversions (set TINV_PHASE_PROFILE=1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

n, b = int(sys.argv[1]), int(sys.argv[2])
t = n // b
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
del g
ctx = _native.Context(n, b)
for pl in ("out", "in"):
    for pipe in (True, False):
        s = P.gen_inversion(t, P.VariantConfig(P.Placement(pl), "UDU", pipe))
        plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
        for _ in range(2):
            ctx.put_dense_device(a.data_ptr(), n)
            rc, err, ms = plan.run()
        print(f"n={n} b={b} {pl} {'pipelined' if pipe else 'barriered'}: {ms:.1f} ms = {n**3/ms/1e9:.2f} TF/s "
              f"({n**3/ms/1e9/37.07*100:.1f}%), cycles budget per SM {ms*1e-3*1.965e9:.3e}", flush=True)
        plan.close()
