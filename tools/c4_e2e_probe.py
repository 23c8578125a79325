"""C4 end to end through the fused engine: PCIe rates alone vs invert_batched_host."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402

B, n = 8192, 256
g = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
a = torch.bmm(g, g.transpose(1, 2)) / n
a.diagonal(dim1=1, dim2=2).add_(1.0)
del g
ha = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
ha.copy_(a)
hx = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
d = torch.empty_like(a)
for name, fn in [("H2D", lambda: d.copy_(ha, non_blocking=True)), ("D2H", lambda: hx.copy_(a, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name} 4.3 GB: {dt * 1e3:.1f} ms = {ha.numel() * 8 / dt / 1e9:.1f} GB/s", flush=True)
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
d.copy_(ha, non_blocking=True)
with torch.cuda.stream(s2):
    hx.copy_(a, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D + D2H concurrently: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
del a, d
torch.cuda.empty_cache()
for _ in range(4):
    t0 = time.perf_counter()
    P.invert_batched_host(ha.numpy(), out=hx.numpy())
    print(f"invert_batched_host: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
