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
