"""C4 fused batched engine: device-resident timing (CUDA events), residual spot check."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1002_4057_b200 import _native  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
torch.manual_seed(0)
g = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
a = torch.bmm(g, g.transpose(1, 2)) / n
a.diagonal(dim1=1, dim2=2).add_(1.0)
del g
x = torch.empty_like(a)
fail = torch.full((1,), -1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _native.batch_small_launch(a.data_ptr(), x.data_ptr(), B, n, n * n, st, fail.data_ptr())
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.batch_small_launch(a.data_ptr(), x.data_ptr(), B, n, n * n, st, fail.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
ti = []
for _ in range(10):  # in place: x <- a (untimed), then x <- x^-1
    x.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.batch_small_launch(x.data_ptr(), x.data_ptr(), B, n, n * n, st, fail.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ti.append(e0.elapsed_time(e1))
ti.sort()
print(f"in place: median {ti[len(ti) // 2]:.3f} ms -> {B * n**3 / ti[len(ti) // 2] / 1e9:.2f} TF/s")
print(f"B={B} n={n}: median {ms:.3f} ms  min {ts[0]:.3f}  -> {B * n**3 / ms / 1e9:.2f} TF/s "
      f"({B * n**3 / ms / 1e9 / 37.07 * 100:.1f} % of 37.07)  fail={int(fail.item())}")
k = torch.arange(0, B, max(1, B // 16), device="cuda")
r = torch.bmm(a[k], x[k]) - torch.eye(n, dtype=torch.float64, device="cuda")
res = r.abs().sum(1).amax(1) / (n * a[k].abs().sum(1).amax(1) * x[k].abs().sum(1).amax(1) * 2.0 ** -52)
print("residual max", float(res.max()), "sym", float((x - x.transpose(1, 2)).abs().max()))
