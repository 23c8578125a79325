"""C3 streamed end to end (bench config: out-of-place DDU pipelined): executor
device time vs wall time per call, and when result tiles become final
(TINV_DEPART_PROFILE=1 prints quantiles)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from paper_1002_4057_b200 import _native  # noqa: E402

n, nb = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (32768, 512)
t = n // nb
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
a = torch.tril(a) + torch.tril(a, -1).T
del g
ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
ha.copy_(a)
hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
del a
torch.cuda.empty_cache()
ctx = _native.Context(n, nb)
s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE, "DDU", True))
sp = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO)
for rep in range(3):
    if rep == 2:
        os.environ["TINV_DEPART_PROFILE"] = "1"
    t0 = time.perf_counter()
    rc, err, ms = sp.run_host(ha.data_ptr(), n, hx.data_ptr(), n, _native.DENSE_SYMMETRIZE)
    print(f"rep {rep}: rc {rc} exec {ms:.1f} ms wall {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
