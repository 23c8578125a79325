"""C4 streamed: executor time, departure profile, wall time."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
B, n, nb = 8192, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
a = torch.bmm(g, g.transpose(1, 2)) / n
a.diagonal(dim1=1, dim2=2).add_(1.0)
a = torch.tril(a) + torch.tril(a, -1).transpose(1, 2)
del g
ha = torch.empty(a.shape, dtype=torch.float64, pin_memory=True); ha.copy_(a)
hx = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
del a
torch.cuda.empty_cache()
t0 = time.perf_counter(); hx.copy_(ha); print(f"host memcpy 4.3 GB: {(time.perf_counter()-t0)*1e3:.1f} ms")
d = torch.empty(ha.shape, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(ha, non_blocking=True); torch.cuda.synchronize()
print(f"H2D 4.3 GB alone: {(time.perf_counter()-t0)*1e3:.1f} ms")
t0 = time.perf_counter(); hx.copy_(d, non_blocking=True); torch.cuda.synchronize()
print(f"D2H 4.3 GB alone: {(time.perf_counter()-t0)*1e3:.1f} ms")
s2 = torch.cuda.Stream()
d2 = torch.empty_like(d)
torch.cuda.synchronize(); t0 = time.perf_counter()
d2.copy_(ha, non_blocking=True)
with torch.cuda.stream(s2):
    hx.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D + D2H concurrently: {(time.perf_counter()-t0)*1e3:.1f} ms")
del d, d2
torch.cuda.empty_cache()
t = n // nb
ctx = _native.Context(n, nb, batch=B)
s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE))
os.environ["TINV_DEPART_PROFILE"] = "1"
sp = _native.Plan(ctx, s.table(), t, np.zeros(0, np.int64), _native.STREAM_IO | _native.TRACE)
for rep in range(3):
    t0 = time.perf_counter()
    rc, err, ms = sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, 1)
    print(f"streamed: rc {rc} exec {ms:.1f} ms wall {(time.perf_counter()-t0)*1e3:.1f} ms", flush=True)
