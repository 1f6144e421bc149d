"""Diffusion test problems: the reference's coefficient fields and assembly.

Drop-in for the reference ``ntdprecon.problem_gen``
(/root/reference/pkg/src/ntdprecon/problem_gen.py).  Setup-time input
generation (host, numpy; see problems.py for the restated kernels) -- not on
the solve path.  ``make_rhs`` uses the GPU spmv.
"""

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import problems
from .banded_core import BandedMatrix, spmv


class CoefficientField(IntEnum):
    SKYSCRAPER = 1
    RING = 2
    POISSON = 3


@dataclass(frozen=True)
class GridSpec:
    nx: int
    ny: int
    nz: int

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1 or self.nz < 1:
            raise ValueError("grid dimensions must be positive")

    @property
    def h(self):
        return 1.0 / (self.nx + 1)

    @property
    def n_rows(self):
        return self.nx * self.ny * self.nz


def kappa_eval(field, point):
    """Coefficient at a point strictly inside the unit cube (problem_gen.py:65-71)."""
    kind = int(CoefficientField(field))
    x, y, z = (float(c) for c in point)
    if not (0.0 < x < 1.0 and 0.0 < y < 1.0 and 0.0 < z < 1.0):
        raise ValueError(f"point {point!r} is not inside the open unit cube")
    if kind == 1:
        ix, iy, iz = int(np.floor(10.0 * x)), int(np.floor(10.0 * y)), int(np.floor(10.0 * z))
        if ix % 2 == 0 and iy % 2 == 0 and iz % 2 == 0:
            return 1.0e3 * (iy + 1.0)
        return 1.0
    if kind == 2:
        dx, dy, dz = x - 0.5, y - 0.5, z - 0.5
        r = np.sqrt(dx * dx + dy * dy + dz * dz)
        return 1.0e3 if 1.0 / (2.0 * np.sqrt(2.0)) <= r <= 0.5 else 1.0
    return 1.0


def assemble(grid, field, workers=1):
    """7-point finite-volume operator for `field` on `grid` (problem_gen.py:136-151)."""
    kind = int(CoefficientField(field))
    kap = problems.reference_kappa(kind, grid.nx, grid.ny, grid.nz)
    data = problems.assemble_kappa(kap, grid.nx, grid.ny, grid.nz)
    return BandedMatrix(grid.nx, grid.ny, grid.nz, data)


def make_rhs(a, mode="ones", workers=1):
    """problem_gen.py:154-165"""
    ones = np.ones(a.n_rows)
    if mode == "ones":
        return ones
    if mode == "manufactured":
        return spmv(a, ones)
    raise ValueError(f"unknown rhs mode {mode!r}")
