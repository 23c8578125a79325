"""When do result tiles become final in a streamed run? (TRACE + TINV_DEPART_PROFILE)"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
os.environ["TINV_DEPART_PROFILE"] = "1"
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
for pl, loops in (("out", "UDU"), ("in", "UDU"), ("out", "UDD"), ("out", "UUU"), ("out", "DDU")):
    s = P.gen_inversion(t, P.VariantConfig(P.Placement(pl), loops))
    sp = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO | _native.TRACE)
    for rep in range(2):
        rc, err, ms = sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, 1)
    print(f"{pl} {loops}: exec {ms:.1f} ms", flush=True)
    sp.close()
