"""CPU oracle for the SPD tile inversion path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference package
`tileinv` (arxiv/paper_1002_4057, `/root/reference/pkg/src/tileinv`). It is
the checker for the CUDA product path, never the product: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it. The product package (`paper_1002_4057_b200`) must not
import anything from here.

Parity pin: every kernel, the stream generators, the hazard scoreboard and the
executor below are checked against golden vectors produced by the live
reference (`tests/golden/make_golden.py`, run in the build container where
`/root/reference` exists) and against the SPEC.md known-answer examples
(`tests/test_oracle.py`).

Each function cites the reference `file:line` it restates.
"""

from __future__ import annotations

import heapq
import math
import queue
import threading
from dataclasses import dataclass, field

import numpy as np

# Kernel kind codes shared with the C-ABI task table (include/tileinv_b200.h).
COPY, POTRF, TRSM, SYRK_SUB, SYRK_ADD_T, GEMM, TRTRI, TRMM_LEFT, TRMM_RIGHT_NEG, TRMM_LEFT_T, LAUUM = range(11)
KIND_NAMES = ["COPY", "POTRF", "TRSM", "SYRK_SUB", "SYRK_ADD_T", "GEMM", "TRTRI",
              "TRMM_LEFT", "TRMM_RIGHT_NEG", "TRMM_LEFT_T", "LAUUM"]
# Step codes: CHOLESKY, TRINV, PRODUCT, COPY  (taskgen.py:37-41)
S1, S2, S3, SCOPY = 1, 2, 3, 0
STEP_NAMES = {S1: "1", S2: "2", S3: "3", SCOPY: "copy"}


class NotPositiveDefinite(ArithmeticError):
    """kernels.py:38-43: non-positive (or non-finite) pivot at tile-local index."""

    def __init__(self, index):
        self.index = index
        super().__init__(f"non-positive pivot at step {index}")


class SingularTile(ArithmeticError):
    """kernels.py:46-51: zero diagonal entry at tile-local index."""

    def __init__(self, index):
        self.index = index
        super().__init__(f"zero diagonal entry at index {index}")


class TaskFailed(RuntimeError):
    """scheduler.py:185-190: the stream-order-first task failure."""

    def __init__(self, task_id, cause):
        self.task_id = task_id
        self.cause = cause
        super().__init__(f"task {task_id} failed: {cause}")


# --------------------------------------------------------------------------
# Tile kernels (kernels.py:54-151). All pure: return a fresh tile.
# --------------------------------------------------------------------------

def sym_lower(c):
    """kernels.py:54-56: mirror the lower triangle of c onto its upper one."""
    return np.tril(c) + np.tril(c, -1).T


def potrf(a):
    """kernels.py:59-76: left-looking column Cholesky of tril(a)."""
    b = a.shape[0]
    lo = np.tril(a)
    l = np.zeros_like(lo)
    for k in range(b):
        d = lo[k, k] - l[k, :k] @ l[k, :k]
        if not (d > 0.0) or not math.isfinite(d):
            raise NotPositiveDefinite(k)
        r = math.sqrt(d)
        l[k, k] = r
        if k + 1 < b:
            l[k + 1:, k] = (lo[k + 1:, k] - l[k + 1:, :k] @ l[k, :k]) / r
    return l


def trsm_right_lt(a, l):
    """kernels.py:79-88: X with X @ tril(l).T == a, column by column."""
    b = l.shape[0]
    lo = np.tril(l)
    x = np.empty_like(a)
    for j in range(b):
        if lo[j, j] == 0.0:
            raise SingularTile(j)
        x[:, j] = (a[:, j] - x[:, :j] @ lo[j, :j]) / lo[j, j]
    return x


def syrk_sub(c, a):
    """kernels.py:91-93."""
    return sym_lower(c) - a @ a.T


def syrk_add_t(c, a):
    """kernels.py:96-98."""
    return sym_lower(c) + a.T @ a


def gemm(c, a, b, trans_a=False, sign=1):
    """kernels.py:101-117: the three shapes (NT-, NN+, TN+)."""
    if not trans_a and sign == -1:
        return c - a @ b.T
    if not trans_a and sign == 1:
        return c + a @ b
    if trans_a and sign == 1:
        return c + a.T @ b
    raise ValueError(f"unsupported gemm shape: trans_a={trans_a}, sign={sign}")


def trtri(l):
    """kernels.py:120-130: row-wise forward substitution for tril(l)^-1."""
    b = l.shape[0]
    lo = np.tril(l)
    x = np.zeros_like(lo)
    for i in range(b):
        if lo[i, i] == 0.0:
            raise SingularTile(i)
        x[i, :i] = -(lo[i, :i] @ x[:i, :i]) / lo[i, i]
        x[i, i] = 1.0 / lo[i, i]
    return x


def trmm_left(a, tri):
    """kernels.py:133-135."""
    return np.tril(tri) @ a


def trmm_right_neg(a, tri):
    """kernels.py:138-140."""
    return -(a @ np.tril(tri))


def trmm_left_t(a, tri):
    """kernels.py:143-145."""
    return np.tril(tri).T @ a


def lauum(l):
    """kernels.py:148-151."""
    lo = np.tril(l)
    return lo.T @ lo


def gemm_shape(step):
    """scheduler.py:198-203: GEMM shape chosen by the task's step."""
    if step == S1:
        return False, -1
    if step == S2:
        return False, 1
    return True, 1


def apply_kernel(kind, step, out, ops):
    """scheduler.py:206-235 (`run_task`): dispatch one task's kernel."""
    if kind == COPY:
        return ops[0].copy()
    if kind == POTRF:
        return potrf(out)
    if kind == TRSM:
        return trsm_right_lt(out, ops[0])
    if kind == SYRK_SUB:
        return syrk_sub(out, ops[0])
    if kind == SYRK_ADD_T:
        return syrk_add_t(out, ops[0])
    if kind == GEMM:
        ta, sg = gemm_shape(step)
        return gemm(out, ops[0], ops[1], ta, sg)
    if kind == TRTRI:
        return trtri(out)
    if kind == TRMM_LEFT:
        return trmm_left(out, ops[0])
    if kind == TRMM_RIGHT_NEG:
        return trmm_right_neg(out, ops[0])
    if kind == TRMM_LEFT_T:
        return trmm_left_t(out, ops[0])
    if kind == LAUUM:
        return lauum(out)
    raise ValueError(kind)


# --------------------------------------------------------------------------
# Task streams (taskgen.py:149-269). A task is a tuple
#   (kind, step, indices, reads, out, out_mode)
# with tiles as (label, row, col) and out_mode "RW" or "W" (copies only).
# --------------------------------------------------------------------------

@dataclass
class Stream:
    tasks: list
    barriers: set = field(default_factory=set)
    t: int = 0


def krange(lo, hi, direction):
    """taskgen.py:149-153: U ascends, D descends over [lo, hi)."""
    return range(lo, hi) if direction == "U" else range(hi - 1, lo - 1, -1)


def _copies(tasks, t, src, dst):
    """taskgen.py:164-170: one write-only COPY per lower tile, row-major."""
    for r in range(t):
        for c in range(r + 1):
            tasks.append((COPY, SCOPY, (r, c), [(src, r, c)], (dst, r, c), "W"))


def step1(tasks, t, d):
    """taskgen.py:178-189 (tile Cholesky)."""
    for j in range(t):
        for k in range(j):
            tasks.append((SYRK_SUB, S1, (j, k), [("A", j, k)], ("A", j, j), "RW"))
        tasks.append((POTRF, S1, (j,), [], ("A", j, j), "RW"))
        for i in range(j + 1, t):
            for k in krange(0, j, d):
                tasks.append((GEMM, S1, (i, j, k), [("A", i, k), ("A", j, k)], ("A", i, j), "RW"))
        for i in range(j + 1, t):
            tasks.append((TRSM, S1, (i, j), [("A", j, j)], ("A", i, j), "RW"))


def step2(tasks, t, d, out_of_place):
    """taskgen.py:192-205 (tile triangular inversion)."""
    if out_of_place and t > 1:
        _copies(tasks, t, "A", "B")
    col = "B" if out_of_place else "A"
    for j in range(t - 1, -1, -1):
        tasks.append((TRTRI, S2, (j,), [], ("A", j, j), "RW"))
        for i in range(t - 1, j, -1):
            tasks.append((TRMM_LEFT, S2, (i, j), [("A", i, i)], ("A", i, j), "RW"))
            for k in krange(j + 1, i, d):
                tasks.append((GEMM, S2, (i, j, k), [("A", i, k), (col, k, j)], ("A", i, j), "RW"))
            tasks.append((TRMM_RIGHT_NEG, S2, (i, j), [("A", j, j)], ("A", i, j), "RW"))


def step3(tasks, t, d, out_of_place):
    """taskgen.py:208-223 (product L^-T L^-1)."""
    if out_of_place and t > 1:
        _copies(tasks, t, "A", "C")
    src = "C" if out_of_place else "A"
    for i in range(t):
        for j in range(i):
            tasks.append((TRMM_LEFT_T, S3, (i, j), [(src, i, i)], ("A", i, j), "RW"))
        tasks.append((LAUUM, S3, (i,), [], ("A", i, i), "RW"))
        for j in range(i):
            for k in krange(i + 1, t, d):
                tasks.append((GEMM, S3, (i, j, k), [(src, k, i), (src, k, j)], ("A", i, j), "RW"))
        for k in range(i + 1, t):
            tasks.append((SYRK_ADD_T, S3, (i, k), [(src, k, i)], ("A", i, i), "RW"))


def gen_stream(t, steps=(1, 2, 3), loops="UDU", out_of_place=False, pipelined=True):
    """taskgen.py:230-269: per-step or full stream; barriers between steps
    when not pipelined. For a single step, loops[0] is its direction."""
    if t < 1:
        raise ValueError("tile count must be >= 1")
    tasks, barriers = [], set()
    for n, s in enumerate(steps):
        d = loops[n] if len(steps) > 1 else loops[0]
        if n > 0 and not pipelined:
            barriers.add(len(tasks))
        if s == 1:
            step1(tasks, t, d)
        elif s == 2:
            step2(tasks, t, d, out_of_place)
        else:
            step3(tasks, t, d, out_of_place)
    return Stream(tasks, barriers, t)


def format_task(tid, task, barriers=()):
    """taskgen.py:272-282: `<id> <step> <kind>(<indices>) R:<tiles> RW:<tile>`."""
    kind, step, idx, reads, out, _ = task
    tiles = ",".join(f"{l}[{r},{c}]" for l, r, c in reads) or "-"
    s = f"{tid} {STEP_NAMES[step]} {KIND_NAMES[kind]}({','.join(map(str, idx))}) R:{tiles} RW:{out[0]}[{out[1]},{out[2]}]"
    return ("BARRIER\n" if tid in barriers else "") + s


# --------------------------------------------------------------------------
# Hazard scoreboard (scheduler.py:101-153)
# --------------------------------------------------------------------------

def build_edges(stream):
    """scheduler.py:101-140 + :143-153. Returns (edges, kinds) with kinds in
    {"RAW","WAR","WAW","BAR"}; an RW->RW pair on one tile is a single RAW."""
    last_writer, readers = {}, {}
    edges = []
    for tid, (kind, step, idx, reads, out, mode) in enumerate(stream.tasks):
        acc = [(r, "R") for r in reads] + [(out, mode)]
        raw = set()
        for tile, m in acc:
            if m in ("R", "RW") and tile in last_writer:
                edges.append((last_writer[tile], tid, "RAW"))
                raw.add((last_writer[tile], tile))
        for tile, m in acc:
            if m in ("RW", "W"):
                for r in readers.get(tile, ()):
                    edges.append((r, tid, "WAR"))
                u = last_writer.get(tile)
                if u is not None and (u, tile) not in raw:
                    edges.append((u, tid, "WAW"))
        for tile, m in acc:
            if m in ("R", "RW"):
                readers.setdefault(tile, []).append(tid)
        for tile, m in acc:
            if m in ("RW", "W"):
                last_writer[tile] = tid
                readers[tile] = []
    n = len(stream.tasks)
    for pos in sorted(stream.barriers):
        has_out = [False] * n
        has_in = [False] * n
        for u, v, _ in edges:
            if u < pos and v < pos:
                has_out[u] = True
            if u >= pos and v >= pos:
                has_in[v] = True
        sinks = [u for u in range(pos) if not has_out[u]]
        sources = [v for v in range(pos, n) if not has_in[v]]
        edges.extend((u, v, "BAR") for u in sinks for v in sources)
    return edges


def critical_path(stream, edges=None, count_copies=False):
    """dag_analysis.py:46-83: longest chain counted in (non-COPY) tasks."""
    edges = build_edges(stream) if edges is None else edges
    n = len(stream.tasks)
    pred = [[] for _ in range(n)]
    for u, v, _ in edges:
        pred[v].append(u)
    best = [0] * n
    for v in range(n):
        w = 1 if (count_copies or stream.tasks[v][0] != COPY) else 0
        best[v] = w + max((best[u] for u in pred[v]), default=0)
    return max(best, default=0)


# --------------------------------------------------------------------------
# Executors (scheduler.py:238-351)
# --------------------------------------------------------------------------

def lower_tiles(dense, b):
    """tile_matrix.py:84-99 + scheduler.py:238-239: the store of A's lower tiles."""
    t = dense.shape[0] // b
    return {("A", i, j): np.ascontiguousarray(dense[i * b:(i + 1) * b, j * b:(j + 1) * b])
            for i in range(t) for j in range(i + 1)}


def run_in_order(stream, store, order=None):
    """scheduler.py:248-258: sequential execution; returns the updated store."""
    store = dict(store)
    ids = range(len(stream.tasks)) if order is None else order
    for tid in ids:
        kind, step, idx, reads, out, mode = stream.tasks[tid]
        try:
            store[out] = apply_kernel(kind, step, store.get(out), [store[r] for r in reads])
        except Exception as exc:  # noqa: BLE001 - mirrors the reference's catch-all
            raise TaskFailed(tid, exc) from exc
    return store


def execute(stream, store, workers=1):
    """scheduler.py:261-351: heap-ordered ready set (ascending id) on a pool of
    `workers` threads; stops dispatch on failure and raises the minimum id."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    n = len(stream.tasks)
    succ = [[] for _ in range(n)]
    seen = set()
    indeg = [0] * n
    for u, v, _ in build_edges(stream):
        if (u, v) not in seen:
            seen.add((u, v))
            succ[u].append(v)
            indeg[v] += 1
    store = dict(store)
    lock = threading.Lock()
    work_q, done_q = queue.Queue(), queue.Queue()

    def worker():
        while True:
            tid = work_q.get()
            if tid is None:
                return
            kind, step, idx, reads, out, mode = stream.tasks[tid]
            try:
                res = apply_kernel(kind, step, store.get(out), [store[r] for r in reads])
            except Exception as exc:  # noqa: BLE001
                done_q.put((tid, exc))
                continue
            with lock:
                store[out] = res
            done_q.put((tid, None))

    threads = [threading.Thread(target=worker, daemon=True) for _ in range(workers)]
    for th in threads:
        th.start()
    ready = [i for i in range(n) if indeg[i] == 0]
    heapq.heapify(ready)
    inflight, failures = 0, []
    try:
        while True:
            while ready and inflight < workers and not failures:
                work_q.put(heapq.heappop(ready))
                inflight += 1
            if inflight == 0:
                break
            tid, exc = done_q.get()
            inflight -= 1
            if exc is not None:
                failures.append((tid, exc))
                continue
            for s in succ[tid]:
                indeg[s] -= 1
                if indeg[s] == 0:
                    heapq.heappush(ready, s)
    finally:
        for _ in threads:
            work_q.put(None)
        for th in threads:
            th.join()
    if failures:
        tid, exc = min(failures, key=lambda f: f[0])
        raise TaskFailed(tid, exc) from exc
    return store


def assemble_lower(store, n, b, label="A"):
    """np.tril of to_dense(...) restricted to the authoritative lower tiles."""
    t = n // b
    out = np.zeros((n, n))
    for i in range(t):
        for j in range(i + 1):
            out[i * b:(i + 1) * b, j * b:(j + 1) * b] = store[(label, i, j)]
    return out


def invert(dense, b, loops="UDU", out_of_place=False, pipelined=True, workers=1):
    """Full inversion: symmetrize_lower(to_dense(execute(gen_inversion(...))))."""
    n = dense.shape[0]
    s = gen_stream(n // b, (1, 2, 3), loops, out_of_place, pipelined)
    st = execute(s, lower_tiles(dense, b), workers) if workers > 1 else run_in_order(s, lower_tiles(dense, b))
    lo = np.tril(assemble_lower(st, n, b))
    return lo + np.tril(lo, -1).T


# --------------------------------------------------------------------------
# Inputs and metrics (BASELINE.json configs)
# --------------------------------------------------------------------------

def spd_matrix(n, seed=0, shift=1.0):
    """A = G G^T / n + shift I with G iid N(0,1) (PCG64, seed), mirrored so A is
    bitwise symmetric. Large n is built in row blocks."""
    g = np.random.default_rng(seed).standard_normal((n, n))
    a = np.empty((n, n))
    blk = 4096
    for r in range(0, n, blk):
        a[r:r + blk] = g[r:r + blk] @ g.T
    a /= n
    a[np.diag_indices(n)] += shift
    lo = np.tril(a)
    return lo + np.tril(lo, -1).T


def normwise_diff(x, r):
    """max|X-R| / max|R| (SURVEY.md §8(d) parity metric)."""
    return float(np.max(np.abs(x - r)) / np.max(np.abs(r)))


def residual(a, x):
    """||I - A X||_1 / (n ||A||_1 ||X||_1 eps)."""
    n = a.shape[0]
    e = np.eye(n) - a @ x
    return float(np.linalg.norm(e, 1) / (n * np.linalg.norm(a, 1) * np.linalg.norm(x, 1) * np.finfo(float).eps))
