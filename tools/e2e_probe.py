"""Where end-to-end time goes: stream generation, host->device put (pinned),
plan build, executor run, device->host get (symmetrized)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

n, nb = int(sys.argv[1]), int(sys.argv[2])
t = n // nb
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
a = torch.tril(a) + torch.tril(a, -1).T
del g
ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True); ha.copy_(a)
hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
del a
torch.cuda.empty_cache()
ctx = _native.Context(n, nb)
cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE)
for rep in range(3):
    T = {}
    t0 = time.perf_counter(); s = P.gen_inversion(t, cfg); tab = s.table(); T["gen"] = time.perf_counter() - t0
    t0 = time.perf_counter(); ctx.put_dense(ha.numpy()); torch.cuda.synchronize(); T["put"] = time.perf_counter() - t0
    t0 = time.perf_counter(); pl = _native.Plan(ctx, tab, t, np.array(sorted(s.barriers), np.int64)); T["plan"] = time.perf_counter() - t0
    t0 = time.perf_counter(); rc, err, ms = pl.run(); T["run"] = time.perf_counter() - t0; T["kernel"] = ms / 1e3
    pl.close()
    t0 = time.perf_counter(); ctx.get_dense(hx.numpy(), _native.DENSE_SYMMETRIZE); T["get"] = time.perf_counter() - t0
    tot = T["gen"] + T["put"] + T["plan"] + T["run"] + T["get"]
    print(f"n={n} nb={nb} rep {rep}: " + " ".join(f"{k} {v*1e3:.1f}ms" for k, v in T.items()) +
          f" | total {tot*1e3:.1f} ms -> {n**3/tot/1e9:.0f} Gflop/s; H2D {n*n*8/T['put']/1e9:.1f} GB/s D2H {n*n*8/T['get']/1e9:.1f} GB/s", flush=True)
# streamed public path (plan cached after the first call)
for rep in range(4):
    t0 = time.perf_counter()
    P.invert_host(ha.numpy(), nb, cfg, out=hx.numpy())
    dt = time.perf_counter() - t0
    print(f"n={n} nb={nb} invert_host rep {rep}: {dt*1e3:.1f} ms -> {n**3/dt/1e9:.0f} Gflop/s", flush=True)
ref = torch.empty_like(hx)
ctx.put_dense(ha.numpy()); s = P.gen_inversion(t, cfg)
pl = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64)); pl.run(); pl.close()
ctx.get_dense(ref.numpy(), _native.DENSE_SYMMETRIZE)
print("bitwise equal to staged path:", bool(torch.equal(ref, hx)), flush=True)
