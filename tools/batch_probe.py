import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
rng = np.random.default_rng(0)
B, n = 40, 256
g = rng.standard_normal((B, n, n))
a = g @ g.transpose(0, 2, 1) / n + np.eye(n)
a = np.tril(a) + np.transpose(np.tril(a, -1), (0, 2, 1))
for nb in (256, 128):
    x = P.invert_batched(a, nb)
    ref = np.linalg.inv(a)
    err = max(np.abs(x[k] - ref[k]).max() / np.abs(ref[k]).max() for k in range(B))
    print(f"batched parity nb={nb}: max normwise {err:.2e}", flush=True)
# C4 timing, device-resident
B = 8192
gd = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
ad = gd @ gd.transpose(1, 2) / n
ad += torch.eye(n, dtype=torch.float64, device="cuda")
del gd
xd = torch.empty_like(ad)
for nb in (256, 128):
    t = n // nb
    ctx = _native.Context(n, nb, batch=B)
    s = P.gen_inversion(t, P.VariantConfig())
    t0 = time.time()
    plan = _native.Plan(ctx, s.table(), t, np.zeros(0, np.int64))
    tp = time.time() - t0
    for _ in range(3):
        ctx.put_dense_device(ad.data_ptr(), n)
        rc, err, ms = plan.run()
        assert rc == 0, plan.msg
    ctx.get_dense_device(xd.data_ptr(), n)
    res = (torch.eye(n, dtype=torch.float64, device="cuda") - ad @ xd).abs().max().item()
    print(f"C4 batch={B} n={n} nb={nb}: plan {tp:.2f}s exec {ms:.2f} ms -> {B*n**3/ms/1e9:.2f} TF/s "
          f"({B*n**3/ms/1e9/37.07*100:.1f}%) max|I-AX| {res:.2e} stats {plan.stats()}", flush=True)
    plan.close(); ctx.close()
