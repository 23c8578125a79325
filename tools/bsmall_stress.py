"""Determinism stress of the fused batched engine (races show up as
run-to-run differences): 20 runs of C4, bitwise equal checksums; in-place
equals out-of-place; odd n too."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1002_4057_b200 import _native  # noqa: E402

for B, n in ((8192, 256), (2000, 255), (3000, 100)):
    g = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
    a = torch.bmm(g, g.transpose(1, 2)) / n
    a.diagonal(dim1=1, dim2=2).add_(1.0)
    a = torch.tril(a) + torch.tril(a, -1).transpose(1, 2)
    del g
    x = torch.empty_like(a)
    fail = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ref = None
    bad = 0
    for r in range(20):
        _native.batch_small_launch(a.data_ptr(), x.data_ptr(), B, n, n * n, st, fail.data_ptr())
        torch.cuda.synchronize()
        if ref is None:
            ref = x.clone()
        elif not torch.equal(x, ref):
            bad += 1
    y = a.clone()
    _native.batch_small_launch(y.data_ptr(), y.data_ptr(), B, n, n * n, st, fail.data_ptr())
    torch.cuda.synchronize()
    print(f"B={B} n={n}: {bad} of 19 reruns differ; in place equal: {torch.equal(y, ref)}; fail {int(fail.item())}",
          flush=True)
