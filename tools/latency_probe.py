"""Per-task dispatch latency: serial chains of tiny tasks on an idle GPU."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1002_4057_b200 import _native
n, b = 2048, 128
t = n // b
ctx = _native.Context(n, b)
a = torch.eye(n, dtype=torch.float64, device="cuda") * 4
def row(kind, step, out, reads, mode=1):
    r = [-1] * 16
    r[0], r[1] = kind, step
    r[5:9] = [out[0], out[1], out[2], mode]
    r[9] = len(reads)
    for x, rd in enumerate(reads):
        r[10 + 3 * x:13 + 3 * x] = list(rd)
    return r
for name, rows in (("COPY (A->B, 1 block row)", [row(0, 0, (1, 1, 0), [(0, 1, 0)], 2) for _ in range(200)]),
                   ("GEMM K=128 (1 item)", [row(5, 1, (0, 2, 1), [(0, 2, 0), (0, 1, 0)]) for _ in range(200)]),
                   ("POTRF 128 (1 special)", [row(1, 1, (0, 3, 3), []) for _ in range(50)])):
    for serial in (True,):
        plan = _native.Plan(ctx, np.array(rows, np.int32), t, np.zeros(0, np.int64), _native.SERIAL)
        ctx.put_dense_device(a.data_ptr(), n)
        plan.run()
        ctx.put_dense_device(a.data_ptr(), n)
        rc, err, ms = plan.run()
        print(f"{name:28s}: {len(rows)} serial tasks {ms:.3f} ms -> {ms / len(rows) * 1e3:.1f} us per task (rc={rc})", flush=True)
        plan.close()
