"""Quick executor timing on device-resident input (not the bench contract)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

for n, b, pl in [(8192, 256, "in"), (8192, 256, "out"), (16384, 512, "out"), (32768, 512, "out")]:
    t = n // b
    g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    a = g @ g.T / n
    a.diagonal().add_(1.0)
    del g
    ctx = _native.Context(n, b)
    s = P.gen_inversion(t, P.VariantConfig(P.Placement(pl)))
    t0 = time.time()
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
    tp = time.time() - t0
    ms = []
    for r in range(3):
        ctx.put_dense_device(a.data_ptr(), n)
        rc, err, m = plan.run()
        assert rc == 0, (rc, plan.msg)
        ms.append(m)
    x = torch.empty_like(a)
    ctx.get_dense_device(x.data_ptr(), n)
    r = torch.eye(n, dtype=torch.float64, device="cuda") - a @ x
    res = (torch.linalg.matrix_norm(r, 1) / (n * torch.linalg.matrix_norm(a, 1) * torch.linalg.matrix_norm(x, 1) * 2.22e-16)).item()
    best = min(ms)
    print(f"n={n} b={b} {pl}: plan {tp:.2f}s exec ms {['%.1f' % v for v in ms]} -> {n**3/best/1e9:.0f} GF/s ({n**3/best/1e9/37070*100:.1f}% of 37.07 TF) residual {res:.2e} stats {plan.stats()}", flush=True)
    plan.close(); ctx.close(); del a, x, r
    torch.cuda.empty_cache()
