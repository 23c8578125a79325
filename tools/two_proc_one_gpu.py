"""Functional check of the multi-PROCESS data path on one B200: two ranks, each
its own process and CUDA context on cuda:0, exchange tile versions through
CUDA-IPC mapped stores and inbox flags (the path `bench.py --gpus N` takes
under torchrun; there one GPU per rank and NCCL for the control plane, here
gloo because NCCL refuses two ranks on one device). The two persistent
executors are time-sliced by the driver, so this says nothing about speed:
it checks the IPC export/open, receive bases, system-scope flag hand-off and
the owned-tile gather against a single-process run, bitwise.

  python tools/two_proc_one_gpu.py [n] [nb] [rows] [cols]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, n, nb, grid, port, out):
    import paper_1002_4057_b200 as P
    from paper_1002_4057_b200 import distributed as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    g = rng.standard_normal((n, n))
    a = g @ g.T / n + np.eye(n)
    cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True)
    tm = P.from_dense(a, nb)
    stream = P.gen_inversion(tm.t, cfg)
    D.execute_multi_gpu(stream, tm, grid=grid, partition=True)
    x = np.tril(P.to_dense(tm))
    if rank == 0:
        ref = P.from_dense(a, nb)
        P.execute(stream, ref)
        xr = np.tril(P.to_dense(ref))
        out.put((bool(np.array_equal(x, xr)), float(np.max(np.abs(x - xr)))))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    grid = (int(sys.argv[3]) if len(sys.argv) > 3 else 1, int(sys.argv[4]) if len(sys.argv) > 4 else 2)
    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import socket
    with socket.socket() as sk:  # a free rendezvous port
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ps = [ctx.Process(target=worker, args=(r, world, n, nb, grid, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(240)
    alive = [p for p in ps if p.is_alive()]
    for p in alive:
        p.kill()
    if alive or any(p.exitcode != 0 for p in ps):
        print("FAILED: exit codes", [p.exitcode for p in ps])
        sys.exit(1)
    same, diff = q.get(timeout=5)
    print(f"two processes on one GPU, n={n} nb={nb} grid={grid}: bitwise equal to one process: {same} (max diff {diff:.3e})")
    sys.exit(0 if same else 1)
