"""Tile kernels -- same names and signatures as the reference
`tileinv.kernels` (kernels.py:23-151), executed on the B200.

Each per-tile call (the reference's operator plugin point, dispatched by
`run_task`, scheduler.py:206-235) places its operands in a small device tile
store and runs a one-task stream through the same persistent DMMA executor
that runs whole inversions. Triangular operands are read below the diagonal
only; outputs follow the reference (strict upper zeroed for POTRF/TRTRI,
full symmetric tiles for SYRK/LAUUM).
"""

from __future__ import annotations

import enum
import threading

import numpy as np


class KernelKind(enum.Enum):
    """kernels.py:23-35."""

    POTRF = "POTRF"
    TRSM = "TRSM"
    SYRK_SUB = "SYRK_SUB"
    SYRK_ADD_T = "SYRK_ADD_T"
    GEMM = "GEMM"
    TRTRI = "TRTRI"
    TRMM_LEFT = "TRMM_LEFT"
    TRMM_RIGHT_NEG = "TRMM_RIGHT_NEG"
    TRMM_LEFT_T = "TRMM_LEFT_T"
    LAUUM = "LAUUM"


class NotPositiveDefiniteError(ArithmeticError):
    """Non-positive pivot; index mirrors LAPACK info (kernels.py:38-43)."""

    def __init__(self, index: int, detail: str = ""):
        self.index = index
        super().__init__(detail or f"non-positive pivot at step {index}")


class SingularTileError(ArithmeticError):
    """Zero diagonal entry in a triangular operand (kernels.py:46-51)."""

    def __init__(self, index: int):
        self.index = index
        super().__init__(f"zero diagonal entry at index {index}")


# --------------------------------------------------------------------------
# per-tile device execution
# --------------------------------------------------------------------------
# Operand placement on a t=3 store: diagonal slots carry identity padding,
# off-diagonal slots zero padding, so triangular operands go on the diagonal.
_D0, _D1, _O10, _O20, _O21 = (0, 0), (1, 1), (1, 0), (2, 0), (2, 1)
_bench = threading.local()


def _store(b):
    from . import _native
    cache = getattr(_bench, "ctx", None)
    if cache is None or cache.b != b:
        cache = _native.Context(3 * b, b)
        _bench.ctx = cache
    return cache


def _run_one(kind, step, out, reads, tiles):
    """Put `tiles` {(i,j): array}, run one task, return the output tile."""
    from . import _native
    b = next(iter(tiles.values())).shape[0]
    ctx = _store(b)
    for (i, j), a in tiles.items():
        ctx.put_tile(i, j, np.asarray(a, dtype=np.float64))
    row = np.full((1, _native.TASK_FIELDS), -1, dtype=np.int32)
    row[0, :2] = (kind, step)
    row[0, 5:9] = (0, out[0], out[1], 1)
    row[0, 9] = len(reads)
    for x, (i, j) in enumerate(reads):
        row[0, 10 + 3 * x:13 + 3 * x] = (0, i, j)
    plan = _native.Plan(ctx, row, 3, np.zeros(0, np.int64))
    rc, err, _ = plan.run()
    plan.close()
    if rc == _native.ERR_NOT_SPD:
        raise NotPositiveDefiniteError(err.index)
    if rc == _native.ERR_SINGULAR:
        raise SingularTileError(err.index)
    if rc != _native.OK:
        raise _native.NativeError(rc, plan.msg)
    return ctx.get_tile(*out)


def _sq(*arrays):
    b = arrays[0].shape[0]
    for a in arrays:
        if a.shape != (b, b):
            raise ValueError("tile kernels take square tiles of one order")
    return b


def potrf(a: np.ndarray) -> np.ndarray:
    """Cholesky factor of tril(a); strict upper of the result zero (kernels.py:59-76)."""
    _sq(a)
    return _run_one(1, 1, _D0, [], {_D0: a})


def trsm_right_lt(a: np.ndarray, l: np.ndarray) -> np.ndarray:
    """X with X tril(l)^T = a (kernels.py:79-88)."""
    _sq(a, l)
    return _run_one(2, 1, _O10, [_D0], {_D0: l, _O10: a})


def syrk_sub(c: np.ndarray, a: np.ndarray) -> np.ndarray:
    """sym(c) - a a^T (kernels.py:91-93)."""
    _sq(c, a)
    return _run_one(3, 1, _D1, [_O10], {_D1: c, _O10: a})


def syrk_add_t(c: np.ndarray, a: np.ndarray) -> np.ndarray:
    """sym(c) + a^T a (kernels.py:96-98)."""
    _sq(c, a)
    return _run_one(4, 3, _D1, [_O10], {_D1: c, _O10: a})


def gemm(c: np.ndarray, a: np.ndarray, b: np.ndarray, trans_a: bool = False, sign: int = 1) -> np.ndarray:
    """c - a b^T | c + a b | c + a^T b (kernels.py:101-117)."""
    _sq(c, a, b)
    if not trans_a and sign == -1:
        step = 1
    elif not trans_a and sign == 1:
        step = 2
    elif trans_a and sign == 1:
        step = 3
    else:
        raise ValueError(f"unsupported gemm shape: trans_a={trans_a}, sign={sign}")
    return _run_one(5, step, _O21, [_O20, _O10], {_O21: c, _O20: a, _O10: b})


def trtri(l: np.ndarray) -> np.ndarray:
    """tril(l)^-1 (kernels.py:120-130)."""
    _sq(l)
    return _run_one(6, 2, _D0, [], {_D0: l})


def trmm_left(a: np.ndarray, tri: np.ndarray) -> np.ndarray:
    """tril(tri) a (kernels.py:133-135)."""
    _sq(a, tri)
    return _run_one(7, 2, _O10, [_D1], {_D1: tri, _O10: a})


def trmm_right_neg(a: np.ndarray, tri: np.ndarray) -> np.ndarray:
    """-a tril(tri) (kernels.py:138-140)."""
    _sq(a, tri)
    return _run_one(8, 2, _O10, [_D0], {_D0: tri, _O10: a})


def trmm_left_t(a: np.ndarray, tri: np.ndarray) -> np.ndarray:
    """tril(tri)^T a (kernels.py:143-145)."""
    _sq(a, tri)
    return _run_one(9, 3, _O10, [_D1], {_D1: tri, _O10: a})


def lauum(l: np.ndarray) -> np.ndarray:
    """tril(l)^T tril(l), full symmetric (kernels.py:148-151)."""
    _sq(l)
    return _run_one(10, 3, _D0, [], {_D0: l})
