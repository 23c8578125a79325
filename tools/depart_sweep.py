"""Streamed e2e wall time vs the departure weight (TINV_DEPART_WEIGHT)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
n, nb = int(sys.argv[1]), int(sys.argv[2])
loops = sys.argv[3] if len(sys.argv) > 3 else "UDU"
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
s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE, loops))
for w in sys.argv[4].split(",") if len(sys.argv) > 4 else ["0", "2", "8", "32", "128", "1000"]:
    os.environ["TINV_DEPART_WEIGHT"] = w
    os.environ["TINV_DEPART_PROFILE"] = "1"
    sp = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO | _native.TRACE)
    sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, 1)
    del os.environ["TINV_DEPART_PROFILE"]
    sp.close()
    sp = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO)
    walls, exs = [], []
    for rep in range(3):
        t0 = time.perf_counter()
        rc, err, ms = sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, 1)
        walls.append(time.perf_counter() - t0); exs.append(ms)
    print(f"{loops} weight {w}: exec {min(exs):.1f} ms wall {min(walls)*1e3:.1f} ms -> e2e {n**3/min(walls)/1e9:.0f} Gflop/s", flush=True)
    sp.close()
