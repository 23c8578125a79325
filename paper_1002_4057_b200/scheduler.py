"""Hazard DAG and the on-device dynamic executor -- same API as the
reference `tileinv.scheduler` (scheduler.py:1-358).

`build_dag` runs the reference's per-tile scoreboard natively
(csrc/api.cu `scoreboard`, scheduler.py:101-153). `execute` compiles the
stream into a device plan (hazard DAG incl. barrier edges, tile-level array
renaming of in-place multi-block kernels, flop-weighted bottom-level
priorities) and runs it with the persistent B200 executor
(csrc/executor.cu). Results are bitwise deterministic for any schedule:
every task computes with a fixed summation order, no atomics touch data.
"""

from __future__ import annotations

import enum
from collections import Counter
from dataclasses import dataclass

import numpy as np

from . import _native
from .kernels import NotPositiveDefiniteError, SingularTileError
from .taskgen import Step, Task, TaskStream
from .tile_matrix import _DEVICE, _NONE, TileId, TileMatrix


class HazardKind(enum.Enum):
    RAW = "RAW"
    WAR = "WAR"
    WAW = "WAW"


INTRA_STEP = "intra_step"
CROSS_STEP = "cross_step"
COPY_RELATED = "copy_related"


@dataclass(frozen=True)
class DagEdge:
    src: int
    dst: int
    kind: HazardKind | None  # None for barrier-induced edges
    tile: TileId | None
    barrier: bool = False


class TaskDag:
    """Tasks plus hazard / barrier edges (scheduler.py:55-83)."""

    def __init__(self, tasks, edges, stream, edge_stats=None):
        self.tasks = tasks
        self.edges = edges
        self.stream = stream
        self.succ = [[] for _ in tasks]
        self.pred = [[] for _ in tasks]
        seen = set()
        for e in edges:
            if (e.src, e.dst) not in seen:
                seen.add((e.src, e.dst))
                self.succ[e.src].append(e.dst)
                self.pred[e.dst].append(e.src)
        for adj in self.succ:
            adj.sort()
        for adj in self.pred:
            adj.sort()
        self.edge_stats = edge_stats if edge_stats is not None else _census(tasks, edges)

    def __len__(self):
        return len(self.tasks)


def _census(tasks, edges):
    """scheduler.py:86-98: hazard counts by category."""
    stats = {k: Counter() for k in HazardKind}
    for e in edges:
        if e.kind is None:
            continue
        if tasks[e.src].is_copy or tasks[e.dst].is_copy:
            cat = COPY_RELATED
        elif tasks[e.src].step is tasks[e.dst].step:
            cat = INTRA_STEP
        else:
            cat = CROSS_STEP
        stats[e.kind][cat] += 1
    return stats


_EDGE_KIND = (HazardKind.RAW, HazardKind.WAR, HazardKind.WAW, None)


def build_dag(stream: TaskStream) -> TaskDag:
    """Hazard DAG of a stream (scheduler.py:101-140) with barrier edges
    linking prefix sinks to suffix sources (scheduler.py:143-153)."""
    tasks = stream.tasks
    table = stream.table(_matrix_label(stream))
    src, dst, kind = _native.dag_edges(table, sorted(stream.barriers))
    edges = []
    for u, v, k in zip(src.tolist(), dst.tolist(), kind.tolist()):
        hk = _EDGE_KIND[k]
        if hk is None:
            edges.append(DagEdge(u, v, None, None, barrier=True))
        elif hk is HazardKind.WAR:
            edges.append(DagEdge(u, v, hk, tasks[v].output.tile))
        else:
            edges.append(DagEdge(u, v, hk, tasks[u].output.tile))
    hazard = [e for e in edges if not e.barrier]
    return TaskDag(tasks, edges, stream, _census(tasks, hazard))


def _matrix_label(stream):
    if stream._table is not None and stream._labels:
        return stream._labels[0]
    for task in stream.tasks:
        return task.output.tile.label
    return "A"


def prune(dag: TaskDag) -> TaskDag:
    """Drop transitively redundant edges (scheduler.py:156-172)."""
    n = len(dag)
    reach = [0] * n
    for u in range(n - 1, -1, -1):
        r = 0
        for v in dag.succ[u]:
            r |= (1 << v) | reach[v]
        reach[u] = r
    kept = [e for e in dag.edges
            if not any(w != e.dst and (reach[w] >> e.dst) & 1 for w in dag.succ[e.src])]
    kept.sort(key=lambda e: (e.src, e.dst))
    return TaskDag(dag.tasks, kept, dag.stream, dag.edge_stats)


def ready_set(dag: TaskDag, completed: set) -> set:
    """scheduler.py:175-182."""
    return {t.id for t in dag.tasks
            if t.id not in completed and all(p in completed for p in dag.pred[t.id])}


class ExecutionError(RuntimeError):
    """The stream-order-first task failure (scheduler.py:185-190)."""

    def __init__(self, task: Task, cause: BaseException):
        self.task = task
        self.cause = cause
        super().__init__(f"task {task.id} {task} failed: {cause}")


class InvalidStreamError(ValueError):
    """Stream and matrix disagree on tiling (scheduler.py:193-194)."""


def _cause(err, msg):
    if err.code == _native.ERR_NOT_SPD:
        return NotPositiveDefiniteError(err.index)
    if err.code == _native.ERR_SINGULAR:
        return SingularTileError(err.index)
    if err.code == _native.ERR_STREAM:
        return KeyError(msg)
    return RuntimeError(msg)


def _run(stream: TaskStream, a: TileMatrix, table, barriers, flags, ref_ids=None, trace_path=None):
    ctx = a._device()
    keep = a._state == _DEVICE
    if keep:
        flags |= _native.KEEP_ON_FAILURE
    if trace_path is not None:
        flags |= _native.TRACE
    plan = _native.Plan(ctx, table, stream.t, barriers, flags)
    rc, err, _ = plan.run()
    if rc != _native.OK:
        msg = plan.msg
        plan.close()
        if err.task_id < 0:
            raise _native.NativeError(rc, msg)
        if not keep:
            a._state = _NONE  # device copy is stale; the host copy is the pre-run state
        tid = err.task_id if ref_ids is None else int(ref_ids[err.task_id])
        task = stream.tasks[tid]
        cause = _cause(err, msg)
        raise ExecutionError(task, cause) from cause
    a._state = _DEVICE
    if trace_path is not None:
        _write_trace(trace_path, stream, plan.trace(), ref_ids)
    plan.close()
    return a


def execute(stream: TaskStream, a: TileMatrix, workers: int = 1, trace_path=None, *,
            share_slots: bool = False) -> TileMatrix:
    """Run the stream's DAG on the B200 (scheduler.py:261-351), updating `a`.

    `workers` is validated as in the reference; the device executor always
    uses every SM. On failure the smallest failing task id is raised as
    ExecutionError and `a` keeps its pre-call content. With trace_path set,
    writes `task_id,kind,indices,worker,start_ns,end_ns` per task from device
    timestamps (worker = SM id). share_slots (off by default): memory-
    constrained renaming -- working tiles (B / C copies, aux tiles) share
    device slots by live range (TINV_SHARE_SLOTS; out-of-place 4T -> 3T tiles)."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if a.t != stream.t:
        raise InvalidStreamError(f"stream generated for t={stream.t} cannot run on a t={a.t} matrix")
    table = stream.table(a.label)
    flags = _native.SHARE_SLOTS if share_slots else 0
    return _run(stream, a, table, np.array(sorted(stream.barriers), dtype=np.int64), flags, trace_path=trace_path)


def run_in_order(stream: TaskStream, a: TileMatrix, order=None) -> TileMatrix:
    """Sequential execution in stream order or a given order (scheduler.py:248-258):
    the tasks run one after another on the device (each one still split
    over all SMs)."""
    if a.t != stream.t:
        raise InvalidStreamError(f"stream generated for t={stream.t} cannot run on a t={a.t} matrix")
    table = stream.table(a.label)
    ref_ids = None
    if order is not None:
        ref_ids = np.asarray(list(order), dtype=np.int64)
        table = table[ref_ids]
    return _run(stream, a, table, np.zeros(0, np.int64), _native.SERIAL, ref_ids=ref_ids)


def _write_trace(path, stream, trace, ref_ids):
    start, end, sm = trace
    rows = []
    for n in range(len(start)):
        tid = n if ref_ids is None else int(ref_ids[n])
        task = stream.tasks[tid]
        rows.append((tid, task.kind_name, ";".join(str(i) for i in task.indices), int(sm[n]),
                     int(start[n]), int(end[n])))
    with open(path, "w") as fh:
        fh.write("task_id,kind,indices,worker,start_ns,end_ns\n")
        for row in sorted(rows):
            fh.write(",".join(str(x) for x in row) + "\n")


def _step_of(task):
    return task.step if isinstance(task.step, Step) else Step(task.step)
