"""Tiled SPD storage with a B200-resident tile store -- same API as the
reference `tileinv.tile_matrix` (tile_matrix.py:1-155).

A TileMatrix keeps a host dense copy (the reference's tiles, incl. the stale
strictly-upper tiles that no task reads, tile_matrix.py:30-33) and, once it
is executed on, a device tile store (`_native.Context`) holding the
authoritative lower tiles in padded slots. Dense <-> tile conversion runs on
the device (csrc/layout.cu); only lower tiles cross PCIe.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from . import _native


class InvalidSizeError(ValueError):
    """Unusable matrix/tile geometry (tile_matrix.py:16-17)."""


class ShapeMismatchError(ValueError):
    """Two dense matrices were expected to share a shape (tile_matrix.py:20-21)."""


class TileId(NamedTuple):
    """Matrix tag plus grid coordinates (tile_matrix.py:24-32)."""

    label: str
    row: int
    col: int

    def __str__(self) -> str:
        return f"{self.label}[{self.row},{self.col}]"


# device-store states
_NONE, _SYNCED, _DEVICE = 0, 1, 2


class TileMatrix:
    """Order-n matrix as a t x t grid of b x b float64 tiles (tile_matrix.py:35-66)."""

    def __init__(self, n: int, b: int, tiles, label: str = "A"):
        if n < 1 or b < 1:
            raise InvalidSizeError(f"matrix order {n} and tile order {b} must be >= 1")
        if n % b:
            raise InvalidSizeError(f"matrix order {n} not divisible by tile order {b}")
        self.n = n
        self.b = b
        self.t = n // b
        self.label = label
        self._ctx = None
        self._state = _NONE
        if isinstance(tiles, np.ndarray) and tiles.shape == (n, n):
            self._host = tiles
        else:
            self._host = np.empty((n, n))
            for i in range(self.t):
                for j in range(self.t):
                    self._host[i * b:(i + 1) * b, j * b:(j + 1) * b] = tiles[i][j]

    # ---- host view (reference attribute `tiles`)
    def _pull(self):
        """Bring device results to the host copy (lower tiles only)."""
        if self._state == _DEVICE:
            self._ctx.get_dense(self._host, _native.DENSE_LOWER)
            self._state = _SYNCED

    @property
    def tiles(self):
        self._pull()
        self._state = _NONE  # caller may write through the views
        b = self.b
        return [[self._host[i * b:(i + 1) * b, j * b:(j + 1) * b] for j in range(self.t)] for i in range(self.t)]

    @tiles.setter
    def tiles(self, value):
        self._pull()
        b = self.b
        for i in range(self.t):
            for j in range(self.t):
                self._host[i * b:(i + 1) * b, j * b:(j + 1) * b] = value[i][j]
        self._state = _NONE

    def tile(self, i: int, j: int) -> np.ndarray:
        self._pull()
        self._state = _NONE  # the view is writable
        b = self.b
        return self._host[i * b:(i + 1) * b, j * b:(j + 1) * b]

    def set_tile(self, i: int, j: int, data: np.ndarray) -> None:
        self._pull()
        b = self.b
        self._host[i * b:(i + 1) * b, j * b:(j + 1) * b] = data
        self._state = _NONE

    def tile_id(self, i: int, j: int) -> TileId:
        return TileId(self.label, i, j)

    def lower_ids(self) -> list:
        """Authoritative tiles (row >= col), row-major (tile_matrix.py:62-66)."""
        return [TileId(self.label, i, j) for i in range(self.t) for j in range(i + 1)]

    # ---- device store
    def _device(self, device: int = 0):
        """The device tile store, uploaded from the host copy if stale."""
        if self._ctx is None:
            self._ctx = _native.Context(self.n, self.b, device)
        if self._state == _NONE:
            self._ctx.put_dense(self._host)
            self._state = _SYNCED
        return self._ctx

    def _dense(self, symmetrize: bool) -> np.ndarray:
        if symmetrize and self._state == _DEVICE:
            out = np.empty((self.n, self.n))
            self._ctx.get_dense(out, _native.DENSE_SYMMETRIZE)
            return out
        self._pull()
        out = self._host.copy()
        return symmetrize_lower(out) if symmetrize else out


def generate_spd(n: int, seed: int) -> np.ndarray:
    """M M^T + n I, M uniform [0,1) from PCG64(seed), mirrored (tile_matrix.py:69-81).
    Test-input helper, not on the inversion path."""
    if n < 1:
        raise InvalidSizeError(f"matrix order must be >= 1, got {n}")
    m = np.random.default_rng(seed).random((n, n))
    a = m @ m.T + n * np.eye(n)
    return np.tril(a) + np.tril(a, -1).T


def from_dense(m: np.ndarray, b: int, label: str = "A") -> TileMatrix:
    """Tile a dense square matrix (tile_matrix.py:84-99): same validation,
    the input is copied."""
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise InvalidSizeError(f"expected a square matrix, got shape {m.shape}")
    n = m.shape[0]
    if n < 1 or b < 1 or n % b:
        raise InvalidSizeError(f"matrix order {n} not divisible by tile order {b}")
    if not np.isfinite(m).all():
        raise ValueError("matrix contains non-finite values")
    return TileMatrix(n, b, np.array(m, dtype=np.float64, order="C", copy=True), label)


def to_dense(tm: TileMatrix) -> np.ndarray:
    """Reassemble the dense matrix, tiles verbatim (tile_matrix.py:102-114)."""
    return tm._dense(False)


def symmetrize_lower(m: np.ndarray) -> np.ndarray:
    """Mirror the lower triangle onto the upper one (tile_matrix.py:117-119)."""
    return np.tril(m) + np.tril(m, -1).T


def to_dense_symmetric(tm: TileMatrix) -> np.ndarray:
    """symmetrize_lower(to_dense(tm)) fused on the device (one gather kernel)."""
    return tm._dense(True)


def copy_lower(src: TileMatrix, dst_label: str) -> TileMatrix:
    """Deep copy of the lower tiles, zero upper tiles (tile_matrix.py:122-135)."""
    src._pull()
    b, t = src.b, src.t
    out = np.zeros((src.n, src.n))
    for i in range(t):
        for j in range(i + 1):
            out[i * b:(i + 1) * b, j * b:(j + 1) * b] = src._host[i * b:(i + 1) * b, j * b:(j + 1) * b]
    return TileMatrix(src.n, src.b, out, dst_label)


def max_abs_diff(a: np.ndarray, b: np.ndarray) -> float:
    """tile_matrix.py:138-144."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise ShapeMismatchError(f"shape mismatch: {a.shape} vs {b.shape}")
    return float(np.max(np.abs(a - b)))


def save_dense_csv(m: np.ndarray, path) -> None:
    """tile_matrix.py:147-149."""
    np.savetxt(path, np.asarray(m, dtype=np.float64), delimiter=",", fmt="%.17g")


def load_dense_csv(path) -> np.ndarray:
    """tile_matrix.py:152-155."""
    return np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
