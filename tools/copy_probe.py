"""Copy-engine H2D throughput with flag writes interleaved (the streamed
arrival pattern), with and without concurrent D2H."""
import time
import torch
from cuda.bindings import driver as d

MB = 1 << 20
nrun, run_bytes = 128, 32 * MB
src = torch.empty(nrun * run_bytes // 8, dtype=torch.float64, pin_memory=True)
dst = torch.empty_like(src, device="cuda")
back = torch.empty_like(src, pin_memory=True)
dsrc = torch.empty_like(src, device="cuda")
flags = torch.zeros(nrun * 64, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def h2d(nflags, with_d2h):
    flags.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(nrun):
        o = r * run_bytes // 8
        with torch.cuda.stream(s1):
            dst[o:o + run_bytes // 8].copy_(src[o:o + run_bytes // 8], non_blocking=True)
        for f in range(nflags):
            d.cuStreamWriteValue32(s1.cuda_stream, flags.data_ptr() + 4 * (r * 64 + f), 1, 0)
        if with_d2h:
            with torch.cuda.stream(s2):
                back[o:o + run_bytes // 8].copy_(dsrc[o:o + run_bytes // 8], non_blocking=True)
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"flags/run {nflags:3d} d2h {with_d2h}: {dt*1e3:7.1f} ms ({nrun*run_bytes/dt/1e9:5.1f} GB/s per direction), enqueue {t_enq*1e3:.1f} ms", flush=True)

for nf in (0, 1, 64):
    for dd in (False, True):
        h2d(nf, dd)
        h2d(nf, dd)
