"""Multi-GPU distribution of the tile inversion.

2D block-cyclic owner-computes over a P x Q grid of B200s: tile (i, j) of
every array lives on rank (i mod P) * Q + (j mod Q) and each task runs on the
owner of its output tile. `tinv_dist_stream` (csrc/api.cu) turns a stream into
the distributed stream: remote reads are redirected to receive tiles, and each
tile version a rank consumes from another owner becomes one explicit transfer
(a write-only COPY into a fresh receive tile, so receivers never carry
anti-dependences on in-flight data) placed right after its producer.

* `execute_distributed(stream, a, grid)` runs the distributed stream with a
  loopback transport on one B200: every rank's tasks and transfers in one
  executor launch. Results are bitwise identical to `execute` (transfers are
  exact copies, every tile sees the same kernel sequence), which pins the
  transform on the hardware we have.
* `transfer_plan(dist, rank)` turns transfers into device SEND / RECV
  pseudo-tasks: a CTA copies the version into the receiver's pool (peer
  memory over NVLink) and sets its inbox flag with a system-scope release; the
  receiver's inbox poller completes the RECV. `execute_distributed(...,
  transport="device")` runs every rank's plan in one launch with the local
  pool standing in for the peers -- the exact device protocol, on one GPU.
* `rank_slice(dist, r)` is the stream a rank executes in a multi-process run
  (its tasks, its outgoing transfers, its incoming receive points); the
  message schedule is exercised with real processes and gloo in
  tests/test_distributed.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .taskgen import TaskStream

# flop weights in b^3 units per kind code (COPY, POTRF, TRSM, SYRK_SUB, SYRK_ADD_T,
# GEMM, TRTRI, TRMM_LEFT, TRMM_RIGHT_NEG, TRMM_LEFT_T, LAUUM)
_W = np.array([0.0, 1 / 3, 1.0, 1.0, 1.0, 2.0, 1 / 3, 1.0, 1.0, 1.0, 1 / 3])


@dataclass
class DistStream:
    table: np.ndarray   # (m, 16) int32 distributed stream
    owner: np.ndarray   # rank executing each task (transfers: sender)
    dest: np.ndarray    # receiving rank of a transfer, -1 otherwise
    ref: np.ndarray     # source task id, -1 for transfers
    grid: tuple
    t: int

    @property
    def world(self):
        return self.grid[0] * self.grid[1]

    def stats(self, b=1):
        """Per-rank load (flops in b^3 units), tasks, transfers in/out, bytes in."""
        kinds = self.table[:, 0]
        is_x = self.dest >= 0
        out = []
        for r in range(self.world):
            mine = (self.owner == r) & ~is_x
            out.append({"rank": r, "tasks": int(mine.sum()), "flops_b3": float(_W[kinds[mine]].sum()),
                        "sends": int(((self.owner == r) & is_x).sum()), "recvs": int((self.dest == r).sum()),
                        "bytes_in": int((self.dest == r).sum()) * b * b * 8})
        loads = np.array([o["flops_b3"] for o in out])
        return {"ranks": out, "load_max_over_mean": float(loads.max() / loads.mean()) if loads.mean() else 1.0,
                "transfers": int(is_x.sum())}


def distribute(stream: TaskStream, grid=(1, 2), matrix_label: str = "A") -> DistStream:
    P, Q = grid
    table, owner, dest, ref = _native.dist_stream(stream.table(matrix_label), stream.t, P, Q)
    return DistStream(table, owner, dest, ref, (P, Q), stream.t)


def rank_slice(d: DistStream, r: int):
    """Positions of the distributed stream rank r takes part in, with its role:
    'run' (its task), 'send' (transfer it sends), 'recv' (transfer it receives)."""
    pos = []
    for k in range(len(d.table)):
        if d.dest[k] >= 0:
            if d.owner[k] == r:
                pos.append((k, "send"))
            elif d.dest[k] == r:
                pos.append((k, "recv"))
        elif d.owner[k] == r:
            pos.append((k, "run"))
    return pos


def transfer_plan(d: DistStream, rank: int = -1, with_ranks: bool = False):
    """Table + aux (dest, seq) + inbox length with SEND / RECV pseudo-tasks.

    rank -1: every rank's tasks (one-GPU execution, sequence = transfer index);
    rank r: the tasks of rank r, sequence numbers counted per receiver.
    with_ranks: also the rank that runs each row (task owner, SEND: sender,
    RECV: receiver), for plans that emulate the ranks in one launch."""
    rows, aux, src, who = [], [], [], []
    per_dest = {}
    nrecv = 0
    for k in range(len(d.table)):
        f = d.table[k]
        if d.dest[k] < 0:
            if rank < 0 or d.owner[k] == rank:
                rows.append(f)
                aux.append((-1, -1))
                src.append(int(d.ref[k]))
                who.append(int(d.owner[k]))
            continue
        dst, snd = int(d.dest[k]), int(d.owner[k])
        if rank < 0:
            seq = nrecv
        else:
            seq = per_dest.get(dst, 0)
            per_dest[dst] = seq + 1
        send = np.full(16, -1, np.int32)
        send[0], send[1], send[8], send[9] = 12, 0, 0, 1
        send[10:13] = f[10:13]
        recv = np.full(16, -1, np.int32)
        recv[0], recv[1], recv[8], recv[9] = 13, 0, 2, 0
        recv[5:8] = f[5:8]
        if rank < 0 or snd == rank:
            rows.append(send)
            aux.append((dst, seq))
            src.append(-1)
            who.append(snd)
        if rank < 0 or dst == rank:
            rows.append(recv)
            aux.append((dst, seq))
            src.append(-1)
            who.append(dst)
        if rank < 0 or dst == rank:
            nrecv = max(nrecv, seq + 1)
    out = (np.array(rows, np.int32), np.array(aux, np.int32), nrecv, np.array(src, np.int64))
    return out + (np.array(who, np.int32),) if with_ranks else out


def execute_distributed(stream: TaskStream, a, grid=(1, 2), transport="loopback"):
    """Run `stream` as distributed over `grid` on one B200: transport
    "loopback" (transfers as device copies), "device" (the SEND / RECV
    protocol with the local pool standing in for peers, any SM runs any
    rank's task) or "ranks" (the same protocol with every rank on its own
    group of nsm / P*Q SMs and its own priority queues: the multi-GPU
    schedule emulated in one launch; the returned DistStream's `last_run`
    holds the kernel time and per-CTA idle times). Same results and errors
    as `execute` (task ids refer to `stream`)."""
    from .scheduler import ExecutionError, InvalidStreamError, _cause, _run
    from .tile_matrix import _DEVICE
    if a.t != stream.t:
        raise InvalidStreamError(f"stream generated for t={stream.t} cannot run on a t={a.t} matrix")
    d = distribute(stream, grid, a.label)
    if transport in ("device", "ranks"):
        table, aux, nrecv, src, who = transfer_plan(d, -1, with_ranks=True)
        ctx = a._device()
        if transport == "ranks":
            plan = _native.Plan.ranks(ctx, table, stream.t, aux, nrecv, who, d.world)
        else:
            plan = _native.Plan.xfer(ctx, table, stream.t, aux, nrecv)
        rc, err, ms = plan.run()
        msg = plan.msg
        if rc == _native.OK and transport == "ranks":
            idle, rk = plan.cta_idle()
            d.last_run = {"kernel_ms": ms, "cta_idle_ns": idle, "cta_rank": rk}
        plan.close()
        if rc != _native.OK:
            if err.task_id < 0 or src[err.task_id] < 0:
                raise _native.NativeError(rc, msg)
            cause = _cause(err, msg)
            raise ExecutionError(stream.tasks[int(src[err.task_id])], cause) from cause
        a._state = _DEVICE
        return d
    ref = np.where(d.ref >= 0, d.ref, 0)
    bars = np.array(sorted(stream.barriers), dtype=np.int64)
    if len(bars):  # barrier positions refer to source tasks: move them to distributed positions
        first = {}
        for k, v in enumerate(d.ref):
            if v >= 0 and v not in first:
                first[int(v)] = k
        bars = np.array([first.get(int(p), len(d.table)) for p in bars], dtype=np.int64)
    _run(stream, a, d.table, bars, 0, ref_ids=ref, trace_path=None)
    return d


def execute_ranks_local(stream: TaskStream, a, grid=(1, 2), sms_per_rank=None, partition=False):
    """The multi-process runtime with every rank in THIS process on one B200:
    one tile store (tinv_ctx) and one transfer plan per rank (exactly what
    `MultiGPU` builds per process), each rank's persistent executor on its own
    share of the SMs (`tinv_set_sms`) so the ranks run concurrently, peers
    mapped by device pointer (`tinv_peer_attach`, the in-process form of the
    CUDA-IPC mapping), SEND work items writing into the receivers' stores and
    inboxes. `partition`: each rank's store holds only the tiles it owns
    (tinv_create_owned). Gathers every rank's owned tiles into `a`.
    -> (DistStream, per-rank device ms, per-rank store bytes)."""
    import threading

    import torch

    from .scheduler import ExecutionError, InvalidStreamError, _cause
    from .tile_matrix import _NONE
    if a.t != stream.t:
        raise InvalidStreamError(f"stream generated for t={stream.t} cannot run on a t={a.t} matrix")
    d = distribute(stream, grid, a.label)
    W = d.world
    nsm = sms_per_rank or torch.cuda.get_device_properties(0).multi_processor_count // W
    P, Q = grid
    a._pull()
    host = a._host
    ctxs, plans, srcs = [], [], []
    try:
        for r in range(W):
            if partition:
                ctx = _native.Context.owned(a.n, a.b, owned_tiles(a.t, grid, r))
            else:
                ctx = _native.Context(a.n, a.b)
            ctx.set_sms(nsm)
            ctx.put_dense(host)
            table, aux, nrecv, src = transfer_plan(d, r)
            plan = _native.Plan.xfer(ctx, table, stream.t, aux, nrecv)
            if plan.rc != _native.OK:
                raise _native.NativeError(plan.rc, plan.msg)
            plan.ipc_export()
            ctxs.append(ctx)
            plans.append(plan)
            srcs.append(src)
        for r, ctx in enumerate(ctxs):
            ctx.peer_attach(r, ctxs)
            ctx.ipc_reset()
        res = [None] * W
        start = threading.Barrier(W)

        def run(r):
            start.wait()
            res[r] = plans[r].run()

        th = [threading.Thread(target=run, args=(r,)) for r in range(W)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        fails = []
        for r, (rc, err, ms) in enumerate(res):
            if rc != _native.OK:
                sid = int(srcs[r][err.task_id]) if 0 <= err.task_id < len(srcs[r]) else -1
                fails.append((sid if sid >= 0 else 2 ** 62, r, rc, err.code, err.index, plans[r].msg))
        if fails:
            a._state = _NONE
            sid, r, rc, code, index, msg = min(fails)
            if sid >= 2 ** 62:
                raise _native.NativeError(rc, msg or f"rank {r} failed")
            e = _native.TinvErr(int(sid), -1, int(code), int(index))
            cause = _cause(e, msg)
            raise ExecutionError(stream.tasks[int(sid)], cause) from cause
        b = a.b
        for r, ctx in enumerate(ctxs):
            out = np.zeros((a.n, a.n))
            ctx.get_dense(out, _native.DENSE_LOWER)
            for i in range(a.t):
                for j in range(i + 1):
                    if (i % P) * Q + (j % Q) == r:
                        a._host[i * b:(i + 1) * b, j * b:(j + 1) * b] = out[i * b:(i + 1) * b, j * b:(j + 1) * b]
        a._state = _NONE
        return d, [x[2] for x in res], [c.store_bytes() for c in ctxs]
    finally:
        for pl in plans:
            pl.close()
        for c in ctxs:
            c.close()


def default_grid(world: int):
    """P x Q with P <= Q, as square as possible (1x2, 2x2, 2x4, ...)."""
    p = int(np.sqrt(world))
    while world % p:
        p -= 1
    return (p, world // p)


def owned_tiles(t, grid, rank):
    """(t, t) int32 mask of the lower tiles `rank` owns (2D block-cyclic) --
    the ownership argument of a partitioned store (`_native.Context.owned`)."""
    P, Q = grid
    return np.array([[1 if j <= i and (i % P) * Q + (j % Q) == rank else 0 for j in range(t)] for i in range(t)],
                    np.int32)


def owned_mask(n, b, grid, rank, device):
    """(n, n) float mask of the lower tiles rank owns (2D block-cyclic)."""
    import torch
    t = n // b
    P, Q = grid
    m = torch.zeros((t, t), dtype=torch.float64, device=device)
    for i in range(t):
        for j in range(i + 1):
            if (i % P) * Q + (j % Q) == rank:
                m[i, j] = 1.0
    return m.repeat_interleave(b, 0).repeat_interleave(b, 1)


class MultiGPU:
    """One rank of a multi-process run (torch.distributed, one B200 per rank).

    Builds the rank's transfer plan from the distributed stream, exports its
    tile store and inbox (CUDA IPC) and maps every peer's, so SEND work items
    write tile versions straight into the receivers' pools over NVLink."""

    def __init__(self, stream: TaskStream, ctx, grid=None, matrix_label="A"):
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.grid = grid or default_grid(self.world)
        if self.grid[0] * self.grid[1] != self.world:
            raise ValueError(f"grid {self.grid} does not match world size {self.world}")
        self.stream, self.ctx = stream, ctx
        self.dist = distribute(stream, self.grid, matrix_label)
        table, aux, nrecv, self.src = transfer_plan(self.dist, self.rank)
        self.plan = _native.Plan.xfer(ctx, table, stream.t, aux, nrecv)
        ok = _agree(self.plan.rc == _native.OK)
        if not ok:
            raise _native.NativeError(self.plan.rc, self.plan.msg or "plan failed on a peer rank")
        hp, hi = self.plan.ipc_export()
        hs = [None] * self.world
        dist.all_gather_object(hs, (hp, hi, ctx.recv_base()))
        ctx.ipc_open(self.rank, self.world, [h[0] for h in hs], [h[1] for h in hs])
        ctx.ipc_recv_bases([h[2] for h in hs])  # partitioned stores: each peer's receive slots start elsewhere

    def run(self):
        """Every rank: reset inbox, barrier, execute. -> (rc, err, device ms)."""
        import torch.distributed as dist
        self.ctx.ipc_reset()
        dist.barrier()
        return self.plan.run()


def _agree(flag: bool) -> bool:
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    v = torch.tensor([0 if flag else 1], device=dev)
    dist.all_reduce(v)
    return int(v.item()) == 0


def execute_multi_gpu(stream: TaskStream, a, grid=None, partition=True):
    """`execute` over all ranks of the default process group (one B200 each):
    every rank passes the same stream and matrix; on return every rank's `a`
    holds the full result (owned tiles all-reduced over NCCL). partition: each
    rank's store holds only its own tiles (tinv_create_owned)."""
    import torch
    import torch.distributed as dist

    from .scheduler import ExecutionError, InvalidStreamError, _cause
    from .tile_matrix import _NONE
    if a.t != stream.t:
        raise InvalidStreamError(f"stream generated for t={stream.t} cannot run on a t={a.t} matrix")
    dev = torch.cuda.current_device()
    grid = grid or default_grid(dist.get_world_size())
    if partition:
        a._pull()
        ctx = _native.Context.owned(a.n, a.b, owned_tiles(a.t, grid, dist.get_rank()), dev)
        ctx.put_dense(a._host)
    else:
        ctx = a._device(dev)
    mg = MultiGPU(stream, ctx, grid, a.label)
    rc, err, _ = mg.run()
    src_id = int(mg.src[err.task_id]) if rc != _native.OK and 0 <= err.task_id < len(mg.src) else -1
    # control-plane tensors live where the backend can gather them (gloo: host)
    info = torch.tensor([src_id if src_id >= 0 else 2 ** 62, err.code, err.index, rc], dtype=torch.int64,
                        device="cuda" if dist.get_backend() == "nccl" else "cpu")
    allinfo = [torch.zeros_like(info) for _ in range(mg.world)]
    dist.all_gather(allinfo, info)
    fails = [x.tolist() for x in allinfo if x[3] != 0]
    if fails:
        a._state = _NONE
        tid, code, index, r = min(fails)
        if tid >= 2 ** 62:
            raise _native.NativeError(r, "multi-GPU execution failed")
        e = _native.TinvErr(int(tid), -1, int(code), int(index))
        cause = _cause(e, "")
        raise ExecutionError(stream.tasks[int(tid)], cause) from cause
    x = torch.zeros((a.n, a.n), dtype=torch.float64, device="cuda")
    # the zero fill runs on torch's stream, the gather on the context's own
    # (non-blocking) stream: order them (get_dense_device syncs its stream on return)
    torch.cuda.current_stream().synchronize()
    ctx.get_dense_device(x.data_ptr(), a.n, _native.DENSE_LOWER)  # (a partitioned store leaves others' tiles 0)
    x *= owned_mask(a.n, a.b, mg.grid, mg.rank, "cuda")
    if partition:
        ctx.close()
    dist.all_reduce(x)
    full = x.cpu().numpy()
    b = a.b
    for i in range(a.t):  # lower tiles only: the strictly-upper tiles keep the stale input (tile_matrix.py:30-33)
        a._host[i * b:(i + 1) * b, :(i + 1) * b] = full[i * b:(i + 1) * b, :(i + 1) * b]
    a._state = _NONE
    return a
