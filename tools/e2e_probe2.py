"""Streamed end to end: executor device time vs wall time, and the arrival
/ departure share (ARRIVE-only and DEPART-only timings by variants)."""
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
s = P.gen_inversion(t, cfg)
bars = np.array(sorted(s.barriers), np.int64)
sp = _native.Plan(ctx, s.table(), t, bars, _native.STREAM_IO)
for mode in (1, 0):
    for rep in range(3):
        t0 = time.perf_counter()
        rc, err, ms = sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, mode)
        wall = time.perf_counter() - t0
        print(f"run_host mode {mode} rep {rep}: rc {rc} exec {ms:.1f} ms wall {wall*1e3:.1f} ms", flush=True)
# phase profile of one streamed run
import os
os.environ["TINV_PHASE_PROFILE"] = "1"
rc, err, ms = sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, 1)
print(f"profiled streamed: {ms:.1f} ms", flush=True)
del os.environ["TINV_PHASE_PROFILE"]
sp.close()
# executor only with the same plan shape minus I/O
ctx.put_dense(ha.numpy())
pl = _native.Plan(ctx, s.table(), t, bars)
rc, err, ms = pl.run()
print(f"staged exec: {ms:.1f} ms", flush=True)
