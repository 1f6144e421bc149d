"""Building the nested twisted preconditioner on the GPU.

Drop-in for the reference ``ntdprecon.ntd_factor``
(/root/reference/pkg/src/ntdprecon/ntd_factor.py).  ``factor_level3`` runs
the whole three-level twisted filtered factorisation -- filtered plane
corrections with the sandwich diagonal shift (:378-404), filtered line
corrections (:113-144) and exact twisted line pivots (:80-110) -- in one
kernel launch (libntdgpu ``ntd_factor``); the factor stays on the device.
"""

import numpy as np
import torch

from . import device as D
from .banded_core import BandedMatrix, FactorizationError, as_device

_DUMP_ORDER = ("l1", "u1", "l2", "u2", "l3", "u3", "m_recip")


def twist_index(num_blocks):
    """1-indexed block where the two elimination sweeps meet (ntd_factor.py:23-27)."""
    if num_blocks < 1:
        raise ValueError("need at least one block")
    return (num_blocks - 1) // 2 + 1


class LineBands:
    """Tridiagonal bands of one grid line (ntd_factor.py:30-36)."""

    def __init__(self, diag, lower, upper):
        self.diag, self.lower, self.upper = diag, lower, upper


class PlaneBands:
    """Pentadiagonal bands of one grid plane (ntd_factor.py:39-48)."""

    def __init__(self, diag, lower1, upper1, lower2, upper2):
        self.diag, self.lower1, self.upper1 = diag, lower1, upper1
        self.lower2, self.upper2 = lower2, upper2


class PreconBands:
    """Factored preconditioner (ntd_factor.py:51-77): l1,u1,l2,u2,l3,u3,m_recip.

    The seven bands live in one (7, N) fp64 CUDA tensor ``bands``; the
    reference's array attributes are materialised on the host lazily."""

    def __init__(self, nx, ny, nz, l1=None, u1=None, l2=None, u2=None, l3=None, u3=None, m_recip=None,
                 twist1=None, twist2=None, twist3=None, bands=None):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        n = self.nx * self.ny * self.nz
        if bands is None:
            arrs = [l1, u1, l2, u2, l3, u3, m_recip]
            if any(a is None for a in arrs):
                raise ValueError("PreconBands needs all seven bands")
            bands = torch.stack([as_device(a).reshape(-1) for a in arrs])
        if tuple(bands.shape) != (7, n):
            raise ValueError(f"bands must have shape (7, {n})")
        self.bands = bands
        self.twist1 = twist_index(self.nx) if twist1 is None else twist1
        self.twist2 = twist_index(self.ny) if twist2 is None else twist2
        self.twist3 = twist_index(self.nz) if twist3 is None else twist3
        self._host = None
        self._solve = None

    @property
    def n_rows(self):
        return self.nx * self.ny * self.nz

    @property
    def solve(self):
        """Apply-side solve arrays on the device (derived from the bands, cached)."""
        if self._solve is None:
            self._solve = D.solve_bands(self.bands, self.nx, self.ny, self.nz, 1)
        return self._solve

    def host(self):
        if self._host is None:
            self._host = self.bands.cpu().numpy()
        return self._host

    l1 = property(lambda s: s.host()[0])
    u1 = property(lambda s: s.host()[1])
    l2 = property(lambda s: s.host()[2])
    u2 = property(lambda s: s.host()[3])
    l3 = property(lambda s: s.host()[4])
    u3 = property(lambda s: s.host()[5])
    m_recip = property(lambda s: s.host()[6])


def factor_level3(a, lanes=4, workers=1):
    """Factor the full three-level preconditioner (ntd_factor.py:351-458).

    ``lanes`` / ``workers`` are accepted for compatibility; the GPU result
    does not depend on them.  Raises FactorizationError with the reference's
    messages."""
    ad = a.device_data()
    pre, status = D.ntd_factor(ad, a.nx, a.ny, a.nz, 1)
    code, plane, row = (int(v) for v in status[0])
    if code:
        raise FactorizationError(D.ntd_factor_message(code, plane, row))
    return PreconBands(a.nx, a.ny, a.nz, bands=pre[0])


def factor_level1(line, twist=None):
    """Exact twisted factorisation of one line (ntd_factor.py:277-300)."""
    td = np.asarray(line.diag, dtype=np.float64)
    tl = np.asarray(line.lower, dtype=np.float64)
    tu = np.asarray(line.upper, dtype=np.float64)
    n = td.shape[0]
    if tl.shape[0] != n or tu.shape[0] != n:
        raise ValueError("line bands must have equal length")
    if n < 1:
        raise ValueError("empty line")
    if twist is not None and twist != twist_index(n):
        raise ValueError("twist must be the midpoint block used by the solver")
    data = np.zeros((7, n))
    data[3], data[2], data[4] = td, tl, tu
    data[2, 0] = 0.0
    data[4, n - 1] = 0.0
    try:
        pre = factor_level3(BandedMatrix(n, 1, 1, data))
    except FactorizationError as exc:
        row = str(exc).split("row ")[1].split(" ")[0]
        raise FactorizationError(f"zero or non-finite pivot at row {row}") from None
    return pre.m_recip.copy()


def factor_level2(plane, grid, lanes=4):
    """Twisted factorisation of one plane (ntd_factor.py:303-333);
    returns (l1, u1, m_recip)."""
    nx, ny = grid.nx, grid.ny
    nxy = nx * ny
    bands = []
    for arr in (plane.diag, plane.lower1, plane.upper1, plane.lower2, plane.upper2):
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        if arr.shape != (nxy,):
            raise ValueError(f"plane bands must have length {nxy}")
        bands.append(arr)
    data = np.zeros((7, nxy))
    data[3], data[2], data[4], data[1], data[5] = bands
    try:
        pre = factor_level3(BandedMatrix(nx, ny, 1, data))
    except FactorizationError as exc:
        msg = str(exc).replace(" (plane 0)", "")
        raise FactorizationError(msg) from None
    return pre.l1.copy(), pre.u1.copy(), pre.m_recip.copy()


def compute_beta(apply_inv, u_seg):
    """Filter weights beta = apply_inv(u) / u, zero where u is zero
    (ntd_factor.py:242-263)."""
    u = as_device(u_seg)
    w = as_device(apply_inv(u_seg))
    if w.shape != u.shape:
        raise ValueError("apply_inv changed the segment length")
    beta = torch.where(u != 0.0, w / torch.where(u != 0.0, u, torch.ones_like(u)), torch.zeros_like(u))
    if not bool(torch.isfinite(beta).all()):
        raise FactorizationError("non-finite filter weights")
    return beta.cpu().numpy() if not isinstance(u_seg, torch.Tensor) else beta


def dump_precon_bands(pre, path):
    """Binary dump (ntd_factor.py:464-471): int64 LE header (N,nx,ny,nz) then
    the seven float64 LE bands."""
    h = pre.host()
    with open(path, "wb") as fh:
        np.array([pre.n_rows, pre.nx, pre.ny, pre.nz], dtype="<i8").tofile(fh)
        for i in range(7):
            h[i].astype("<f8").tofile(fh)


def load_precon_bands(path):
    """Inverse of dump_precon_bands (ntd_factor.py:474-491)."""
    with open(path, "rb") as fh:
        hdr = np.fromfile(fh, dtype="<i8", count=4)
        if hdr.shape[0] != 4:
            raise ValueError("truncated header")
        n, nx, ny, nz = (int(v) for v in hdr)
        if nx < 1 or ny < 1 or nz < 1 or n != nx * ny * nz:
            raise ValueError("inconsistent header")
        arrays = {}
        for name in _DUMP_ORDER:
            arr = np.fromfile(fh, dtype="<f8", count=n)
            if arr.shape[0] != n:
                raise ValueError(f"truncated band data ({name})")
            arrays[name] = arr.astype(np.float64)
    return PreconBands(nx, ny, nz, **arrays)
