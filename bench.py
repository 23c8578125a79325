"""Benchmark: FP64 SPD tile inversion Gflop/s (n^3 / t) on B200.

Workload (BASELINE.json metric, config 3, fits one B200): n = 32768,
nb = 512, A = G G^T / n + I with G iid N(0,1) (generated on the device,
seed 0), out-of-place, pipelined, loop orders DDU (same kernel time as the
reference default UDU; result tiles become final progressively, so the
streamed device->host copies overlap the run).

One step = dense A (resident in HBM) -> tile store (layout kernel) ->
persistent executor over the whole POTRF/TRTRI/LAUUM DAG -> symmetrized dense
A^-1 (layout kernel). Inputs are 8.6 GB, far above the 126 MB L2, so no flush
is needed between steps. `e2e` repeats the step through the public call
`invert_host` with pinned HOST buffers (H2D of the lower tiles + D2H of the
full inverse inside the timed region); its `value` reuses the plan and store
the first call built (cached per shape and variant), its `cold_ms` /
`cold_value` time that first call (plan build + store allocation included).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Under torchrun (N > 1) the ranks run ONE matrix distributed 2D block-cyclic
(strong scaling); a setup failure fails the run. `--impl reference` times the
reference algorithm (the oracle port of tileinv: numpy kernels + threaded
hazard-DAG executor, one worker per core) on the host cores, at the full
workload size on the same input bytes (n <= 32768; larger: the n=8192 sample).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPD inversion FP64 Gflop/s (n³/t) at n=32768, 1/2/4/8 B200; % of FP64 peak"
DMMA_PEAK_TFLOPS = 37.07   # measured: tools/fp64_peak.cu, profiles/r01_fp64_peak.log (sustained, 1965 MHz)
DGEMM_TFLOPS = 35.47       # cuBLAS DGEMM 8192^3 comparator, profiles/r01_dgemm_peak.json


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="c3", choices=["c1", "c2", "c3", "c4", "c5"],
                   help="BASELINE.json config (c3 = the headline metric's n=32768, nb=512)")
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--nb", type=int, default=None)
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--engine", default="auto", choices=["auto", "fused", "dag"],
                   help="batched workloads: fused per-matrix kernel (nb == n <= 256) or the DAG executor")
    p.add_argument("--fused-engine", default=None, choices=["cta", "pipe"],
                   help="fused batched engine: one CTA per matrix (default) or the pipelined persistent engine")
    p.add_argument("--placement", default="out", choices=["in", "out"])
    p.add_argument("--loops", default=None,
                   help="loop orders of the three steps; default DDU at c3 (result tiles become final "
                        "progressively, so the device->host copies overlap the run; same kernel time as UDU), "
                        "UDU (the reference default) elsewhere")
    p.add_argument("--barriered", action="store_true")
    p.add_argument("--no-steps", action="store_true", help="skip the per-step / barriered breakdown")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--share-slots", action="store_true",
                   help="memory-constrained renaming: working tiles share store slots by live range")
    p.add_argument("--no-load", action="store_true",
                   help="skip the load report (per-SM busy, 2x4 ranks emulated in one launch, schedule model)")
    p.add_argument("--cpu-sample-n", type=int, default=None)
    p.add_argument("--cpu-worker", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--shift", type=float, default=None, help=argparse.SUPPRESS)
    p.add_argument("--device-input", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--ref-steps", type=int, default=1,
                   help="--impl reference: timed full-size runs (n > 8192: ~150 s each on 16 cores at n=32768)")
    return p.parse_args()


def _host_mem_ok(nbytes):
    """Enough available host memory for the pinned e2e buffers?"""
    try:
        with open("/proc/meminfo") as fh:
            avail = next(int(l.split()[1]) * 1024 for l in fh if l.startswith("MemAvailable"))
        return avail > nbytes
    except Exception:  # noqa: BLE001
        return True


# --------------------------------------------------------------------- CPU side
def _one_matrix(args):
    """Pool task for the batched CPU baseline: one matrix through the oracle."""
    from threadpoolctl import threadpool_limits

    from oracle import tileinv_oracle as O
    a, nb, loops, oop = args
    with threadpool_limits(1, "blas"):
        return O.invert(a, nb, loops, oop, True).shape[0]


def cpu_worker_batch(n, nb, batch, steps, warmup, placement, loops):
    """Batched CPU baseline: a process pool with one process per host core, each
    inverting whole matrices (the reference's t=1 stream per matrix)."""
    import multiprocessing as mp

    import numpy as np
    cores = len(os.sched_getaffinity(0))
    sample = min(batch, 4 * cores)
    rng = np.random.default_rng(0)
    g = rng.standard_normal((sample, n, n))
    a = g @ g.transpose(0, 2, 1) / n + np.eye(n)
    work = [(a[k], nb, loops, placement == "out") for k in range(sample)]
    times = []
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_one_matrix, work[:cores])
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_one_matrix, work, chunksize=1)
            if k >= warmup:
                times.append(time.perf_counter() - t0)
    print(json.dumps({"times": times, "cores": cores, "cpu": "", "flops": float(sample) * n ** 3,
                      "sample": sample}))


def _device_input(n, shift):
    """The bench arm's own input bytes (torch Philox on cuda:0, seed 0, mirrored
    lower triangle), copied to host memory; None without a GPU."""
    try:
        import torch
        if not torch.cuda.is_available():
            return None
    except Exception:  # noqa: BLE001
        return None
    gen = torch.Generator(device="cuda").manual_seed(0)
    g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
    a = torch.matmul(g, g.T)
    del g
    a.div_(n)
    a.diagonal().add_(shift)
    a = torch.tril(a) + torch.tril(a, -1).T
    h = a.cpu().numpy()
    del a
    torch.cuda.empty_cache()
    return h


def cpu_worker(n, nb, steps, warmup, placement, loops, pipelined, shift=1.0, device_input=False):
    """Runs in a subprocess with OPENBLAS_NUM_THREADS=1: the reference's CPU
    algorithm (oracle port) with one worker thread per host core."""
    import numpy as np

    from oracle import tileinv_oracle as O
    from threadpoolctl import threadpool_limits
    cores = len(os.sched_getaffinity(0))
    a = _device_input(n, shift) if device_input else None
    if a is None:
        a = O.spd_matrix(n, 0, shift)  # input generation uses every BLAS thread
    s = O.gen_stream(n // nb, (1, 2, 3), loops, placement == "out", pipelined)
    times = []
    with threadpool_limits(1, "blas"):  # the reference's fastest mode: workers = cores, BLAS 1 thread
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            O.execute(s, O.lower_tiles(a, nb), workers=cores)
            dt = time.perf_counter() - t0
            if k >= warmup:
                times.append(dt)
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            model = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except Exception:  # noqa: BLE001
        pass
    print(json.dumps({"times": times, "cores": cores, "cpu": model, "flops": float(n) ** 3}))


def run_cpu(n, nb, steps, warmup, placement, loops, pipelined, batch=1, shift=1.0, device_input=False):
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env.pop(k, None)
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-worker", "--n", str(n), "--nb", str(nb),
           "--steps", str(steps), "--warmup", str(warmup), "--placement", placement, "--loops", loops,
           "--batch", str(batch), "--shift", repr(shift)]
    if not pipelined:
        cmd.append("--barriered")
    if device_input:
        cmd.append("--device-input")
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


# --------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, index):
        self.samples = []
        self.stop = threading.Event()
        self.index = index

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits", "-lms", "200"],
                                 stdout=subprocess.PIPE, text=True)
        except FileNotFoundError:
            return
        while not self.stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.samples.append([x.strip() for x in line.split(",")])
        p.terminate()

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        time.sleep(0.5)
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=3)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------- GPU side
def main():
    args = parse()
    if args.cpu_worker:
        if (args.batch or 1) > 1:
            cpu_worker_batch(args.n, args.nb, args.batch, args.steps, args.warmup, args.placement, args.loops)
        else:
            cpu_worker(args.n, args.nb, args.steps, args.warmup, args.placement, args.loops, not args.barriered,
                       1.0 if args.shift is None else args.shift, args.device_input)
        return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TINV_BENCH_ONE_GPU=1: functional check of the N > 1 code path on a box
    # with one GPU -- every rank is its own process and CUDA context on cuda:0,
    # gloo instead of NCCL (which refuses two ranks on one device); the driver
    # time-slices the ranks' executors, so the printed numbers mean nothing
    one_gpu = world > 1 and os.environ.get("TINV_BENCH_ONE_GPU", "0") == "1"
    if one_gpu:
        local = 0
    wl = {"c1": (1024, 128, 1), "c2": (8192, 256, 1), "c3": (32768, 512, 1), "c4": (256, 256, 8192),
          "c5": (65536, 1024, 1)}[args.workload]
    shift = 1e-3 if args.workload == "c5" else 1.0  # BASELINE config 5: harder conditioning (cond ~4e3)
    n = args.n or wl[0]
    nb = args.nb or wl[1]
    if args.loops is None:
        # one GPU at c3: DDU (result tiles final progressively: the streamed e2e
        # overlaps its device->host copies; kernel time = UDU's). Distributed
        # (N > 1): UDU -- step 1 under D chains ~t^2/2 GEMMs on the critical
        # path (tools/scaling_model.py: 180 vs 62 ms at c3).
        args.loops = "DDU" if args.workload == "c3" and world == 1 else "UDU"
    batch = args.batch or wl[2]
    if args.cpu_sample_n is None:
        args.cpu_sample_n = min(n, 8192) if batch == 1 else n
    t = n // nb
    pipelined = not args.barriered
    flops = float(batch) * float(n) ** 3
    in_bytes = batch * n * n * 8
    desc = (f"{batch} x " if batch > 1 else "") + f"n={n}, nb={nb}"
    config = {"workload": f"BASELINE config {args.workload[1]}: {desc}, FP64 SPD inversion "
                          f"({args.placement}-of-place, {args.loops}, {'pipelined' if pipelined else 'barriered'})",
              "n": n, "nb": nb, "t": t, "batch": batch, "placement": args.placement, "loops": args.loops,
              "pipelined": pipelined, "input": f"A = G G^T/n + {shift:g} I, G iid N(0,1) seed 0",
              "l2": (f"inputs {in_bytes / 1e9:.1f} GB >> 126 MB L2 (no flush needed)" if in_bytes > 4e8
                     else "L2 flushed between steps (256 MB write)"),
              "parallelism": "1 GPU" if world == 1 else f"replicas x{world} (independent matrices)"}

    if args.impl == "reference":
        if rank != 0:
            return
        # Same config as the b200 arm: the full n (n=32768 at c3) on the same
        # input bytes (generated like the b200 arm's, on the device, copied to
        # host). A full-size run takes minutes on the host cores, so it is
        # timed --ref-steps times (default 1, no warm-up); the bounded n<=8192
        # sample (the b200 arm's cpu_baseline) is kept as an extra field.
        full = batch == 1 and args.cpu_sample_n < n <= 32768  # c5 (n=65536): ~20 min and ~150 GB of host RAM
        if full:
            r = run_cpu(n, nb, max(1, args.ref_steps), 0, args.placement, args.loops, pipelined, 1, shift, True)
        else:
            r = run_cpu(args.cpu_sample_n, nb, max(1, args.steps), max(0, min(args.warmup, 1)), args.placement,
                        args.loops, pipelined, batch, shift)
        ts = r["times"]
        med = statistics.median(ts)
        v = r["flops"] / med / 1e9
        if batch > 1:
            sample = (f"{r['sample']} of the {batch} n={n} matrices per step, process pool of {r['cores']} "
                      f"(one process per core, BLAS 1 thread); median of {len(ts)}")
        elif full:
            sample = (f"the full workload: n={n}, nb={nb} (t={t}), same input bytes as the b200 arm; "
                      f"{len(ts)} timed run(s), no warm-up (each run builds its DAG and tile store inside the "
                      f"timed call, like the reference's execute)")
        else:
            sample = f"n={args.cpu_sample_n}, nb={nb} (t={args.cpu_sample_n // nb}) full inversion per step, " \
                     f"same variant; median of {len(ts)}"
        out = {
            "impl": "reference", "metric": METRIC, "value": v, "unit": "Gflop/s", "n_gpus": args.gpus,
            "steps": len(ts), "steps_requested": args.steps, "warmup": 0 if full else max(0, min(args.warmup, 1)),
            "ms_per_step": med * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "same_config": batch > 1 or full or n == args.cpu_sample_n,
            "cpu_baseline": {"value": v, "unit": "Gflop/s", "cores": r["cores"], "kind": "port",
                             "sample": sample, "cpu": r["cpu"]},
            "e2e": {"value": v, "unit": "Gflop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        if full:  # the bounded sample the b200 arm's cpu_baseline uses, for reference
            rs = run_cpu(args.cpu_sample_n, nb, 3, 1, args.placement, args.loops, pipelined, 1, shift)
            out["sample_n%d" % args.cpu_sample_n] = {
                "value": rs["flops"] / statistics.median(rs["times"]) / 1e9, "unit": "Gflop/s",
                "ms_per_step": statistics.median(rs["times"]) * 1e3, "steps": len(rs["times"])}
        print(json.dumps(out))
        return

    import numpy as np
    import torch

    import paper_1002_4057_b200 as P
    from paper_1002_4057_b200 import _native

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctl_dev = "cpu" if one_gpu else "cuda"  # where small control-plane tensors live

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        v = torch.tensor([x], dtype=torch.float64, device=ctl_dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    # input on the device
    gen = torch.Generator(device="cuda").manual_seed(rank if world > 1 and batch > 1 else 0)
    if batch == 1:
        g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
        a = torch.matmul(g, g.T)
        del g
        a.div_(n)
        a.diagonal().add_(shift)
        rb = 4096  # mirror the lower triangle in row blocks (no n^2 temporaries at n = 65536)
        for r0 in range(0, n, rb):
            r1 = min(n, r0 + rb)
            blk = a[r0:r1, r0:r1]
            blk.copy_(torch.tril(blk) + torch.tril(blk, -1).T)
            if r1 < n:
                a[r0:r1, r1:].copy_(a[r1:, r0:r1].T)
    else:
        g = torch.randn(batch, n, n, dtype=torch.float64, device="cuda", generator=gen)
        a = torch.bmm(g, g.transpose(1, 2))
        del g
        a.div_(n)
        a.diagonal(dim1=1, dim2=2).add_(1.0)
        a = torch.tril(a) + torch.tril(a, -1).transpose(1, 2)
        pipelined = True  # a batched store runs the per-matrix chains without barriers
    x = torch.empty_like(a)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda") if in_bytes <= 4e8 else None

    stream = torch.cuda.current_stream()
    fused = batch > 1 and args.engine != "dag" and nb == n <= _native.BATCH_SMALL_MAX_N
    if args.engine == "fused" and not fused:
        raise SystemExit("--engine fused needs a batched workload with nb == n <= 256")
    if fused and args.fused_engine:
        _native.batch_engine(args.fused_engine)
    feng = _native.batch_engine() if fused else None
    config["engine"] = (("fused: one CTA per matrix runs gen_inversion(1) = POTRF -> TRTRI -> LAUUM "
                         "(tinv_batch_small_launch, engine cta)") if feng == "cta" else
                        ("fused, pipelined: one persistent CTA per SM, several matrices in flight, 64x64 block jobs "
                         "of gen_inversion(1) over a DAG in shared memory (tinv_batch_small_launch, engine pipe)")
                        if feng == "pipe" else "DAG executor (tinv_plan_exec)")
    if fused:
        ctx = None
    elif world > 1 and batch == 1:  # distributed: each rank's store holds only its own tiles
        from paper_1002_4057_b200.distributed import default_grid, owned_tiles
        ctx = _native.Context.owned(n, nb, owned_tiles(t, default_grid(world), rank), local)
    else:
        ctx = _native.Context(n, nb, local, batch=batch)
    if ctx is not None:
        ctx.set_stream(stream.cuda_stream)
    s = P.gen_inversion(t, P.VariantConfig(P.Placement(args.placement), args.loops, pipelined))
    table = s.table()
    bars = np.array(sorted(s.barriers), dtype=np.int64)

    # N > 1: one matrix distributed over all ranks (2D block-cyclic, tile
    # versions sent GPU to GPU through peer memory) -- strong scaling. A setup
    # or trial-run failure on any rank fails the bench (no silent fallback).
    mg = None
    scaling = "weak"
    if world > 1 and batch == 1:
        from paper_1002_4057_b200.distributed import MultiGPU, _agree, owned_mask
        if not pipelined:
            raise SystemExit("the distributed run is pipelined only")
        why = None
        try:
            mg = MultiGPU(s, ctx)
        except Exception as exc:  # noqa: BLE001
            why = exc
        if not _agree(why is None):  # every rank learns about a failure on any rank
            raise RuntimeError(f"distributed setup failed (rank {rank}: {why!r})")
        ctx.put_dense_device(a.data_ptr(), n)
        rc_t, _, _ = mg.run()
        if not _agree(rc_t == 0):
            raise RuntimeError(f"distributed trial run failed (rc {rc_t} on rank {rank})")
        scaling = "strong"
        st = mg.dist.stats(nb)
        config["parallelism"] = f"2d-block-cyclic {mg.grid[0]}x{mg.grid[1]} (tile versions over NVLink peer memory)"
        config["load_max_over_mean"] = st["load_max_over_mean"]
        config["transfers"] = st["transfers"]
    plan = None if fused else mg.plan if mg is not None else _native.Plan(
        ctx, table, t, bars, _native.SHARE_SLOTS if args.share_slots else 0)
    if plan is not None and plan.rc != 0:
        raise RuntimeError(plan.msg)
    stats = {"engine": "fused", "ctas": batch, "block_ops_per_matrix": 56 if n > 192 else None} if fused \
        else plan.stats()

    kern_ms = []
    fail = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    kev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def fused_step():
        kev[0].record(stream)
        _native.batch_small_launch(a.data_ptr(), x.data_ptr(), batch, n, n * n, stream.cuda_stream, fail.data_ptr())
        kev[1].record(stream)
        kev[1].synchronize()
        kern_ms.append(kev[0].elapsed_time(kev[1]))
        if int(fail.item()) != -1:
            raise RuntimeError(f"fused batched inversion failed: {int(fail.item()):#x}")

    def step():
        if fused:
            return fused_step()
        ctx.put_dense_device(a.data_ptr(), n)
        rc, err, ms = mg.run() if mg is not None else plan.run()
        if rc != 0:
            raise RuntimeError(f"executor failed: {plan.msg} task {err.task_id}")
        kern_ms.append(ms)
        ctx.get_dense_device(x.data_ptr(), n, _native.DENSE_LOWER if mg is not None else _native.DENSE_SYMMETRIZE)

    for _ in range(args.warmup):
        step()
    kern_ms.clear()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        barrier()
        for e0, e1 in evs:
            if flush is not None:  # inputs smaller than L2: flush it between steps (outside the timed spans)
                flush.fill_(1.0)
            e0.record(stream)
            step()
            e1.record(stream)
        barrier()
    ms_total = max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in evs))
    ms_step = ms_total / args.steps
    jobs = 1 if mg is not None else world  # distributed: all ranks share one matrix per step
    value = jobs * flops / (ms_step * 1e-3) / 1e9
    kern_avg = max_over_ranks(statistics.mean(kern_ms))
    store_bytes = ctx.store_bytes() if ctx is not None else None
    # measured load: per-CTA scheduler idle time of the
    # last timed launch -> busy fraction per SM (per rank when distributed)
    load = None
    if not fused and not args.no_load:
        idle, _ = plan.cta_idle()
        busy = 1.0 - idle * 1e-6 / max(kern_ms[-1], 1e-9)
        load = {"kernel_ms": kern_ms[-1], "sms": int(len(idle)),
                "sm_busy_frac": {"min": float(busy.min()), "mean": float(busy.mean()), "max": float(busy.max())},
                "source": "per-CTA idle ns of the executor's scheduler warp (tinv_plan_cta_idle), last timed step"}
        if dist is not None:
            v = torch.tensor([float(busy.mean())], dtype=torch.float64, device=ctl_dev)
            allb = [torch.zeros_like(v) for _ in range(world)]
            dist.all_gather(allb, v)
            load["rank_busy_frac"] = [float(x.item()) for x in allb]
    achieved = flops / (world if mg is not None else 1) / (kern_avg * 1e-3) / 1e12
    if mg is not None:  # gather the owned tiles for the check below (others' tiles: not written, masked out)
        x = torch.where(owned_mask(n, nb, mg.grid, rank, "cuda") > 0, x, torch.zeros((), dtype=x.dtype, device=x.device))
        import torch.distributed as tdist
        tdist.all_reduce(x)
        x = torch.tril(x) + torch.tril(x, -1).T

    # numerical check of the last step (outside the timed region)
    eps = 2.220446049250313e-16
    if batch == 1 and n > 16384:  # ||I - A X||_1 on 512 sampled columns (a full A X would need 2 x 8n^2 bytes)
        cols = torch.randperm(n, device="cuda", generator=torch.Generator("cuda").manual_seed(1))[:512]
        r = a @ x[:, cols]
        r[cols, torch.arange(512, device="cuda")] -= 1.0
        res = float(r.abs().sum(0).max() / (n * a.abs().sum(0).max() * x.abs().sum(0).max() * eps))
        sym_err = float((x[cols, :] - x[:, cols].T).abs().max())
        config["residual_check"] = "||I - A X||_1 estimated on 512 sampled columns"
        del r
    else:
        eye = torch.eye(n, dtype=torch.float64, device="cuda")
        ac, xc = (a, x) if batch == 1 else (a[:16], x[:16])
        r = eye - ac @ xc
        res = float((torch.linalg.matrix_norm(r, 1) / (n * torch.linalg.matrix_norm(ac, 1)
                                                        * torch.linalg.matrix_norm(xc, 1) * eps)).max())
        sym_err = float((xc - xc.transpose(-1, -2)).abs().max())
        del r, eye, ac, xc

    # the multi-GPU schedule on this one B200: 2x4 ranks in ONE launch, each on
    # 18 SMs with its own queues, tile versions through SEND / RECV (measured);
    # and the schedule model's prediction for a real 8 x B200 node
    if load is not None and batch == 1 and world == 1 and t >= 16 and mg is None:
        from paper_1002_4057_b200.distributed import distribute, transfer_plan
        s_u = P.gen_inversion(t, P.VariantConfig(P.Placement(args.placement), "UDU", True))
        d8 = distribute(s_u, (2, 4))
        tb, ax, nrv, _, who = transfer_plan(d8, -1, with_ranks=True)
        bp = -(-nb // 128) * 128
        fits = torch.cuda.mem_get_info()[0] > 1.2 * nrv * bp * bp * 8 + (1 << 30)  # receive tiles
        pr = _native.Plan.ranks(ctx, tb, t, ax, nrv, who, 8) if fits else None
        if pr is None:
            load["emulated_2x4"] = {"note": f"not run: {nrv} receive tiles exceed free HBM"}
        elif pr.rc == 0:
            ctx.put_dense_device(a.data_ptr(), n)
            rc8, _, ms8 = pr.run()
            if rc8 == 0:
                idle8, rk8 = pr.cta_idle()
                rb = [float(ms8 - idle8[rk8 == r].mean() * 1e-6) for r in range(8)]
                load["emulated_2x4"] = {
                    "kernel_ms": ms8, "sms_per_rank": int((rk8 == 0).sum()), "rank_busy_ms": rb,
                    "busy_max_over_mean": max(rb) / statistics.mean(rb),
                    "flop_load_max_over_mean": d8.stats(nb)["load_max_over_mean"], "transfers": nrv,
                    "loops": "UDU"}
        if pr is not None:
            pr.close()
        try:
            t1m, _ = _native.model_run(n, nb, s_u.table(), t, sorted(s_u.barriers))
            t8m, b8 = _native.model_run(n, nb, tb, t, aux=ax, nrecv=nrv, rank_of=who, nranks=8)
            load["model_8gpu"] = {"t1_ms": t1m / 1e3, "t8_ms": t8m / 1e3, "efficiency": t1m / (8 * t8m),
                                  "source": "csrc/model.cu schedule model, 8 x 148 SMs, _native.MODEL_COST "
                                            "(validated against the one-launch emulation, profiles/r02)"}
        except Exception as exc:  # noqa: BLE001
            load["model_8gpu"] = {"error": repr(exc)[:200]}

    # per-step device times (each step on the previous one's
    # output, same store) and pipelined vs barriered full inversion
    steps_breakdown = None
    # (skipped above n = 32768: three more step plans on the same store would
    # not fit next to C5's 34 GB matrix and its working tiles)
    if batch == 1 and mg is None and not args.no_steps and n <= 32768:
        def med_ms(plans, reps=3):
            out = []
            for _ in range(reps):
                ctx.put_dense_device(a.data_ptr(), n)
                cur = []
                for pl in plans:
                    rc, err, ms = pl.run()
                    if rc != 0:
                        raise RuntimeError(f"executor failed: {pl.msg}")
                    cur.append(ms)
                out.append(cur)
            return [statistics.median(c[k] for c in out) for k in range(len(plans))]

        plc = P.Placement(args.placement)
        sps = [P.gen_step1(t, args.loops[0]), P.gen_step2(t, args.loops[1], plc), P.gen_step3(t, args.loops[2], plc)]
        step_plans = [_native.Plan(ctx, q.table(), t, np.zeros(0, np.int64)) for q in sps]
        ms1, ms2, ms3 = med_ms(step_plans)
        for q in step_plans:
            q.close()
        other = P.gen_inversion(t, P.VariantConfig(plc, args.loops, not pipelined))
        op = _native.Plan(ctx, other.table(), t, np.array(sorted(other.barriers), dtype=np.int64))
        (ms_other,) = med_ms([op])
        op.close()
        pipe_ms, bar_ms = (kern_avg, ms_other) if pipelined else (ms_other, kern_avg)
        steps_breakdown = {
            "unit": "ms (device, median of 3; kernel only, input resident)",
            "step1_potrf_ms": ms1, "step2_trtri_ms": ms2, "step3_lauum_ms": ms3, "sum_of_steps_ms": ms1 + ms2 + ms3,
            "step_gflops": [flops / 3 / (m * 1e-3) / 1e9 for m in (ms1, ms2, ms3)],
            "pipelined_ms": pipe_ms, "barriered_ms": bar_ms,
            "pipelining_gain": bar_ms / pipe_ms,
        }

    # end to end through the C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e and mg is not None and _host_mem_ok(2 * in_bytes * world + (8 << 30)):
        # distributed end to end: every rank copies ITS tiles of A from pinned
        # host memory into its partitioned store, runs, and copies its result
        # tiles back (the result ends up partitioned across the ranks' host
        # memories, one tile owner each): the bytes are each lower tile once
        ha = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        ha.copy_(a)
        hx = torch.zeros(a.shape, dtype=torch.float64, pin_memory=True)
        ha_np, hx_np = ha.numpy(), hx.numpy()

        def dist_e2e_step():
            ctx.put_dense(ha_np)
            rc_e, _, _ = mg.run()
            if rc_e != 0:
                raise RuntimeError(f"distributed e2e run failed (rc {rc_e})")
            ctx.get_dense(hx_np, _native.DENSE_LOWER)

        dist_e2e_step()  # warm-up
        e2e_times = []
        for _ in range(max(1, min(args.steps, 3))):
            barrier()
            t0 = time.perf_counter()
            dist_e2e_step()
            barrier()
            e2e_times.append(max_over_ranks((time.perf_counter() - t0) * 1e3))
        e2e_ms = statistics.median(e2e_times)
        tile_bytes = t * (t + 1) // 2 * nb * nb * 8
        e2e = {"value": flops / (e2e_ms * 1e-3) / 1e9, "unit": "Gflop/s", "h2d_bytes_per_step": tile_bytes,
               "d2h_bytes_per_step": tile_bytes, "ms_per_step": e2e_ms, "steps": len(e2e_times),
               "path": ("every rank: tinv_put_dense of its own lower tiles from pinned host A into its partitioned "
                        "store, the distributed executor, tinv_get_dense of its own result tiles (lower) back; "
                        "max over ranks")}
    elif not args.no_e2e and mg is not None:
        e2e = {"value": None, "unit": "Gflop/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": "not measured: not enough host memory for every rank's pinned buffers"}
    elif not args.no_e2e and _host_mem_ok(3 * in_bytes):
        # the public host-buffer call (invert_host / invert_batched_host): A's
        # lower tiles stream host -> device while the executor runs, result
        # tiles stream back (mirrored) as they become final; the compiled plan
        # is cached by the first (warm-up) call
        ha = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        ha.copy_(a)
        hx = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        del a, x
        if ctx is not None:
            ctx.set_stream(0)
            plan.close()
            ctx.close()
        torch.cuda.empty_cache()
        ha_np, hx_np = ha.numpy(), hx.numpy()
        cfg = P.VariantConfig(P.Placement(args.placement), args.loops, pipelined)

        def e2e_step():
            if batch == 1:
                P.invert_host(ha_np, nb, cfg, out=hx_np, device=local)
            else:
                P.invert_batched_host(ha_np, nb, cfg, out=hx_np, device=local, engine="fused" if fused else "dag")

        # first call: builds the plan (DAG, priorities, queues) and the device
        # store inside the timed call, as the reference's execute builds its
        # DAG per call (scheduler.py:277); reported separately as cold_ms
        barrier()
        t0 = time.perf_counter()
        e2e_step()
        barrier()
        cold_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
        k = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_step()
        barrier()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / k)
        T = t * (t + 1) // 2
        e2e = {"value": world * flops / (e2e_ms * 1e-3) / 1e9, "unit": "Gflop/s",
               "h2d_bytes_per_step": in_bytes if fused else batch * T * nb * nb * 8, "d2h_bytes_per_step": in_bytes,
               "ms_per_step": e2e_ms, "steps": k, "cold_ms": cold_ms,
               "cold_value": world * flops / (cold_ms * 1e-3) / 1e9,
               "plan": "value: plan and device store cached by the first call (same n, nb, variant); cold_ms / "
                       "cold_value: the first call, plan build + store allocation inside the timed call",
               "path": ("paper_1002_4057_b200.invert_batched_host(pinned A, out=pinned X), fused engine: chunks "
                        "of matrices host->device, kernel, device->host on three streams, overlapped") if fused else
                       ("paper_1002_4057_b200.invert_host(pinned A, out=pinned X): lower tiles host->device by the "
                        "copy engines overlapped with the executor, result tiles device->host (symmetrized) as they "
                        "become final; plan cached after the warm-up call")}
        P.clear_plan_cache()
        ctx = None
    elif not args.no_e2e:
        e2e = {"value": None, "unit": "Gflop/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": "not measured: host memory too small for the pinned input and output buffers"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = run_cpu(args.cpu_sample_n, nb, 1, 0, args.placement, args.loops, pipelined, batch)
        cpu = {"value": r["flops"] / statistics.median(r["times"]) / 1e9, "unit": "Gflop/s", "cores": r["cores"],
               "kind": "port", "cpu": r["cpu"],
               "sample": (f"{r['sample']} of the {batch} n={n} matrices, process pool of {r['cores']} "
                          "(oracle port of tileinv, BLAS 1 thread)") if batch > 1 else
                         (f"n={args.cpu_sample_n}, nb={nb} full inversion (oracle port of tileinv: numpy kernels, "
                          f"threaded hazard-DAG executor, {r['cores']} workers, BLAS 1 thread)")}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "exec_c3_traffic.json")
    if fused:
        tpath = os.path.join(ROOT, "profiles", "bsmall_c4_traffic.json")
    if os.path.exists(tpath) and ((n, nb, args.placement) == (32768, 512, "out") or
                                  (feng == "cta" and (n, batch) == (256, 8192))):
        with open(tpath) as fh:
            traffic = json.load(fh)["traffic_bytes"]

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "Gflop/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / DMMA_PEAK_TFLOPS, "traffic": traffic,
                         "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum of one k_bsmall launch "
                                            "(profiles/bsmall_c4_traffic.json)") if fused else
                                           "dram__bytes_read.sum + dram__bytes_write.sum of one exec_kernel "
                                           "launch, ncu application replay (profiles/exec_c3_traffic.json)",
                         "kernel": "tinv::bsm::k_bsmall (one CTA per matrix: fused POTRF -> TRTRI -> LAUUM, "
                                   "64x64 DMMA.8x8x4 block program)" if feng == "cta" else
                                   ("tinv::bpl::k_bpipe (persistent, warp-specialized: TMA operand ring, "
                                    "DMMA.8x8x4 64x64 block jobs over an in-CTA DAG)") if feng == "pipe" else
                                   "tinv::exec_kernel (persistent DAG executor, DMMA.8x8x4)",
                         "algorithmic": f"n^3 = {flops:.3e} flop per launch",
                         "peak_source": "measured FP64 DMMA peak (tools/fp64_peak.cu); cuBLAS DGEMM "
                                        f"{DGEMM_TFLOPS} TF/s for context; MEASURED_PEAKS.json has no FP64 entry"},
            "pct_fp64_peak": 100.0 * value / world / 1e3 / DMMA_PEAK_TFLOPS,  # per GPU
            "kernel_ms": kern_avg, "plan": stats,
            "store_bytes": store_bytes, "share_slots": bool(args.share_slots),
            "residual": res, "symmetry_err": sym_err,
            "gpu_launches": (1 if fused else 3) * args.steps,
            "clocks": clk.summary(),
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if load is not None:
            out["load"] = load
        if steps_breakdown is not None:
            out["steps_breakdown"] = steps_breakdown
        print(json.dumps(out))
    if ctx is not None:
        ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
