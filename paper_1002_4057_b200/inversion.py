"""Whole-matrix entry points composed from the reference API:
from_dense -> gen_* -> execute -> to_dense, all on the B200."""

from __future__ import annotations

import numpy as np

from .scheduler import execute
from .taskgen import Placement, VariantConfig, gen_inversion, gen_step1, gen_step2, gen_step3
from .tile_matrix import from_dense, to_dense, to_dense_symmetric


def invert(a: np.ndarray, nb: int, config: VariantConfig = VariantConfig(), *,
           share_slots: bool = False) -> np.ndarray:
    """A^-1 of an SPD matrix: symmetrize_lower(to_dense(execute(gen_inversion(...))))."""
    tm = from_dense(a, nb)
    execute(gen_inversion(tm.t, config), tm, share_slots=share_slots)
    return to_dense_symmetric(tm)


def plan_under_memory(n: int, nb: int, budget_bytes: float, loops=None, sms: int = 148):
    """Performance under a memory constraint (PAPER.md's closing open problem):
    among the placements (out-of-place = the reference's array renaming into
    B / C, in-place = none), the loop orders, and slot sharing (memory-
    constrained renaming, TINV_SHARE_SLOTS), the variant the schedule model
    (csrc/model.cu, calibrated on the B200) predicts fastest whose device store
    fits `budget_bytes`. Host only. -> dict(config, share_slots, store_bytes,
    model_ms) or None when nothing fits."""
    from . import _native

    t = n // nb
    bp = -(-nb // 128) * 128
    best = None
    for pl in (Placement.OUT_OF_PLACE, Placement.IN_PLACE):
        for lo in ([loops] if loops else ("UDU", "DDU", "UDD")):
            cfg = VariantConfig(pl, lo, True)
            s = gen_inversion(t, cfg)
            for share in (False, True):
                mk, _ = _native.model_run(n, nb, s.table(), t, sorted(s.barriers), sms_per_rank=sms,
                                          flags=_native.SHARE_SLOTS if share else 0)
                store = _native.model_run.last_slots * bp * bp * 8
                if store <= budget_bytes and (best is None or mk < best["model_ms"] * 1e3 * 0.999):
                    best = {"config": cfg, "share_slots": share, "store_bytes": store, "model_ms": mk / 1e3}
    return best


def step_potrf(a: np.ndarray, nb: int, direction: str = "U") -> np.ndarray:
    """Step 1 alone: lower tiles hold L (to_dense verbatim, upper tiles stale)."""
    tm = from_dense(a, nb)
    execute(gen_step1(tm.t, direction), tm)
    return to_dense(tm)


def step_trtri(l: np.ndarray, nb: int, direction: str = "D", placement: Placement = Placement.IN_PLACE):
    """Step 2 alone on a lower factor: lower tiles hold L^-1."""
    tm = from_dense(l, nb)
    execute(gen_step2(tm.t, direction, placement), tm)
    return to_dense(tm)


def step_lauum(linv: np.ndarray, nb: int, direction: str = "U", placement: Placement = Placement.IN_PLACE):
    """Step 3 alone on L^-1: lower tiles hold the lower part of A^-1."""
    tm = from_dense(linv, nb)
    execute(gen_step3(tm.t, direction, placement), tm)
    return to_dense(tm)


def _fused_ok(n: int, nb: int, engine: str) -> bool:
    from . import _native

    if engine not in ("auto", "fused", "dag"):
        raise ValueError(f"engine must be 'auto', 'fused' or 'dag', got {engine!r}")
    ok = nb == n and n <= _native.BATCH_SMALL_MAX_N
    if engine == "fused" and not ok:
        raise ValueError(f"the fused batched engine needs nb == n <= {_native.BATCH_SMALL_MAX_N}")
    return ok and engine != "dag"


def _fused_host(a: np.ndarray, out: np.ndarray, config: VariantConfig, device: int) -> np.ndarray:
    """tinv_batch_small_host on C-contiguous (batch, n, n) float64 buffers."""
    from . import _native
    from .kernels import NotPositiveDefiniteError
    from .scheduler import ExecutionError

    batch, n = a.shape[0], a.shape[-1]
    rc, fm, fi, _ = _native.batch_small_host(a.ctypes.data, out.ctypes.data, batch, n, device)
    if rc != _native.OK:
        s = gen_inversion(1, VariantConfig(config.placement, config.loops, True, config.workers))
        potrf = next(t for t in s.tasks if t.kind.name == "POTRF")
        cause = NotPositiveDefiniteError(fi)
        exc = ExecutionError(potrf, cause)
        exc.matrix = fm
        raise exc from cause
    return out


def invert_batched(a: np.ndarray, nb: int | None = None, config: VariantConfig = VariantConfig(),
                   device: int = 0, engine: str = "auto") -> np.ndarray:
    """Inverses of a batch of SPD matrices a[k] (BASELINE config 4: 8192 x n=256).

    engine "fused" (the default when nb == n <= 256): the per-matrix stream
    gen_inversion(1) = POTRF -> TRTRI -> LAUUM runs fused in one thread block
    per matrix (csrc/batched.cu), the batch streamed through the device in
    chunks. engine "dag": one device store holds the whole batch; the
    per-matrix stream (gen_inversion(n/nb, config), pipelined) is replicated
    into one merged DAG of independent chains and run by the persistent
    executor. Failures raise ExecutionError for the failing task of the lowest
    failing matrix; the exception carries `.matrix`.
    """
    from . import _native
    from .scheduler import ExecutionError, _cause
    from .tile_matrix import InvalidSizeError

    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise InvalidSizeError(f"expected a (batch, n, n) array, got shape {a.shape}")
    batch, n = a.shape[0], a.shape[1]
    nb = n if nb is None else nb
    if n < 1 or nb < 1 or n % nb:
        raise InvalidSizeError(f"matrix order {n} not divisible by tile order {nb}")
    if not np.isfinite(a).all():
        raise ValueError("matrix contains non-finite values")
    if _fused_ok(n, nb, engine):
        return _fused_host(a, np.empty_like(a), config, device)
    t = n // nb
    cfg = VariantConfig(config.placement, config.loops, True, config.workers)
    s = gen_inversion(t, cfg)
    ctx = _native.Context(n, nb, device, batch=batch)
    try:
        ctx.put_dense(a.reshape(batch * n, n))
        plan = _native.Plan(ctx, s.table(), t, np.zeros(0, np.int64))
        rc, err, _ = plan.run()
        msg = plan.msg
        plan.close()
        if rc != _native.OK:
            if err.task_id < 0:
                raise _native.NativeError(rc, msg)
            m, tid = divmod(err.task_id, len(s))
            cause = _cause(err, msg)
            exc = ExecutionError(s.tasks[tid], cause)
            exc.matrix = m
            raise exc from cause
        out = np.empty_like(a)
        ctx.get_dense(out.reshape(batch * n, n), _native.DENSE_SYMMETRIZE)
        return out
    finally:
        ctx.close()


# ---------------------------------------------------------------- host-buffer fast path
# (n, nb, batch, device, placement, loops, pipelined) -> (Context, Plan, TaskStream)
_HOST_PLANS: dict = {}


def clear_plan_cache() -> None:
    """Release the device stores and plans kept by invert_host / invert_batched_host."""
    for ctx, plan, _ in _HOST_PLANS.values():
        plan.close()
        ctx.close()
    _HOST_PLANS.clear()


def _host_buffer(x, name):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            if x.device.type != "cpu":
                raise ValueError(f"{name} must be a host array")
            x = x.numpy()
    except ImportError:  # pragma: no cover
        pass
    return x


def _run_host(a: np.ndarray, out, nb: int, batch: int, config: VariantConfig, device: int,
              engine: str = "dag") -> np.ndarray:
    from . import _native
    from .scheduler import ExecutionError, _cause
    from .tile_matrix import InvalidSizeError

    a = _host_buffer(a, "a")
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[-1]
    if a.shape[-2] != n or n < 1 or nb < 1 or n % nb:
        raise InvalidSizeError(f"matrix order {n} not divisible by tile order {nb}" if a.shape[-2] == n
                               else f"expected square matrices, got shape {a.shape}")
    out = np.empty_like(a) if out is None else _host_buffer(out, "out")
    if out.shape != a.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array shaped like a")
    if np.shares_memory(a, out):  # result tiles stream out while input tiles still stream in
        raise ValueError("out must not overlap a")
    if a.ndim == 3 and _fused_ok(n, nb, engine):
        return _fused_host(a, out, config, device)
    t = n // nb
    pipelined = True if batch > 1 else config.pipelined
    key = (n, nb, batch, device, config.placement, config.loops, pipelined)
    hit = _HOST_PLANS.get(key)
    if hit is None:
        s = gen_inversion(t, VariantConfig(config.placement, config.loops, pipelined, config.workers))
        ctx = _native.Context(n, nb, device, batch=batch)
        plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), dtype=np.int64), _native.STREAM_IO)
        if plan.rc != _native.OK:
            msg = plan.msg
            plan.close()
            ctx.close()
            raise _native.NativeError(plan.rc, msg)
        hit = _HOST_PLANS[key] = (ctx, plan, s)
    ctx, plan, s = hit
    rx = a.reshape(-1, n)
    xo = out.reshape(-1, n)
    rc, err, _ = plan.run_host(rx.ctypes.data, n, xo.ctypes.data, n, _native.DENSE_SYMMETRIZE)
    if rc == _native.ERR_BAD_ARG and "page-locked" in plan.msg:
        # output not page-locked: the staged path (put -> execute -> get) on the same store
        ctx.put_dense(rx)
        p2 = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), dtype=np.int64))
        rc, err, _ = p2.run()
        plan.msg = p2.msg
        p2.close()
        if rc == _native.OK:
            ctx.get_dense(xo, _native.DENSE_SYMMETRIZE)
    if rc != _native.OK:
        msg = plan.msg
        if err.task_id < 0:
            raise _native.NativeError(rc, msg)
        m, tid = divmod(err.task_id, len(s))
        cause = _cause(err, msg)
        exc = ExecutionError(s.tasks[tid], cause)
        if batch > 1:
            exc.matrix = m
        raise exc from cause
    return out


def invert_host(a, nb: int, config: VariantConfig = VariantConfig(), out=None, device: int = 0) -> np.ndarray:
    """A^-1 of an SPD matrix held in host memory, end to end on the B200 with
    the transfers overlapped with the computation: symmetrize_lower(to_dense(
    execute(gen_inversion(...), from_dense(a, nb)))) as one call.

    A's lower tiles stream host -> device (copy engines, column order) while
    the executor already factors the first panels, and each result tile is
    written into `out` (mirrored) as soon as it is final. Pass page-locked
    buffers (e.g. ``torch.empty(..., pin_memory=True).numpy()``) for the
    overlap; other buffers take the staged path. The compiled plan and the
    device store are cached per (n, nb, config, device) -- see
    clear_plan_cache(). `a` is not pre-scanned for non-finite values (the
    reference's from_dense check); such values surface as
    NotPositiveDefiniteError from the factorization."""
    a = _host_buffer(a, "a")
    if np.ndim(a) != 2:
        from .tile_matrix import InvalidSizeError

        raise InvalidSizeError(f"expected a square matrix, got shape {np.shape(a)}")
    return _run_host(a, out, nb, 1, config, device)


def invert_batched_host(a, nb: int | None = None, config: VariantConfig = VariantConfig(), out=None,
                        device: int = 0, engine: str = "auto") -> np.ndarray:
    """invert_batched with streamed transfers (BASELINE config 4 end to end):
    a is (batch, n, n) in host memory, out likewise. The fused engine moves
    the batch in chunks (host -> device, kernel, device -> host overlapped on
    three streams); the DAG engine uses invert_host's tile arrivals /
    departures."""
    a = _host_buffer(a, "a")
    if np.ndim(a) != 3 or a.shape[1] != a.shape[2]:
        from .tile_matrix import InvalidSizeError

        raise InvalidSizeError(f"expected a (batch, n, n) array, got shape {np.shape(a)}")
    return _run_host(a, out, a.shape[1] if nb is None else nb, a.shape[0], config, device, engine)
