"""Timing of the layout kernels at C3 size (k_put dense->tiles, k_get tiles->dense symmetrize)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1002_4057_b200 import _native  # noqa: E402

n, nb = 32768, 512
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
x = torch.empty_like(a)
ctx = _native.Context(n, nb)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
for name, fn, by in (("put", lambda: ctx.put_dense_device(a.data_ptr(), n), 16 * (n * (n + nb) // 2)),
                     ("get symmetrize", lambda: ctx.get_dense_device(x.data_ptr(), n, _native.DENSE_SYMMETRIZE),
                      8 * (n * (n + nb) // 2) + 8 * n * n)):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    print(f"{name}: {ms:.3f} ms = {by / ms / 1e6:.0f} GB/s (algorithmic bytes {by / 1e9:.2f} GB)", flush=True)
ctx.set_stream(0)
