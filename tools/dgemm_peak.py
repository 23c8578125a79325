"""cuBLAS DGEMM comparator (torch.matmul float64) for the FP64 roofline.

Only a comparator for the measured FP64 peak; never on the product path.
"""
import json
import time

import torch


def main():
    dev = torch.device("cuda:0")
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_burst_tflops"] = 2 * n**3 / (best * 1e-3) / 1e12
        # sustained: back to back for ~4 s
        t0 = time.time()
        k = 0
        e0.record()
        while time.time() - t0 < 4.0:
            torch.matmul(a, b)
            k += 1
            if k % 8 == 0:
                torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        out[f"dgemm_{n}_sustained_tflops"] = k * 2 * n**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
