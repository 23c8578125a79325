"""Phase profile of diagonal tasks only (TINV_PHASE_PROFILE=1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1002_4057_b200 import _native
n, b = int(sys.argv[1]), int(sys.argv[2])
t = n // b
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
ctx = _native.Context(n, b)
def row(kind, step, out):
    r = [-1] * 16
    r[0], r[1] = kind, step
    r[5:9] = [0, out[0], out[1], 1]
    r[9] = 0
    return r
for kind, name in ((1, "POTRF"), (6, "TRTRI")):
    for serial in (False, True):
        tab = np.array([row(kind, 1, (i, i)) for i in range(t if not serial else 4)], np.int32)
        plan = _native.Plan(ctx, tab, t, np.zeros(0, np.int64), _native.SERIAL if serial else 0)
        ctx.put_dense_device(a.data_ptr(), n)
        rc, err, ms = plan.run()
        print(f"{name} x{len(tab)} {'serial' if serial else 'parallel'}: {ms:.3f} ms", flush=True)
        plan.close()
