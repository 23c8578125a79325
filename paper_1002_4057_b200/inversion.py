"""Whole-matrix entry points composed from the reference API:
from_dense -> gen_* -> execute -> to_dense, all on the B200."""

from __future__ import annotations

import numpy as np

from .scheduler import execute
from .taskgen import Placement, VariantConfig, gen_inversion, gen_step1, gen_step2, gen_step3
from .tile_matrix import from_dense, to_dense, to_dense_symmetric


def invert(a: np.ndarray, nb: int, config: VariantConfig = VariantConfig()) -> np.ndarray:
    """A^-1 of an SPD matrix: symmetrize_lower(to_dense(execute(gen_inversion(...))))."""
    tm = from_dense(a, nb)
    execute(gen_inversion(tm.t, config), tm)
    return to_dense_symmetric(tm)


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


def invert_batched(a: np.ndarray, nb: int | None = None, config: VariantConfig = VariantConfig(),
                   device: int = 0) -> np.ndarray:
    """Inverses of a batch of SPD matrices a[k] (BASELINE config 4: 8192 x n=256).

    One device store holds the whole batch; the per-matrix stream
    (gen_inversion(n/nb, config), pipelined) is replicated into one merged DAG
    of independent chains and run by the persistent executor. Failures raise
    ExecutionError for the failing task of the lowest failing matrix; the
    exception carries `.matrix`.
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
