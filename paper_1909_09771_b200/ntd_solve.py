"""Applying the inverse of the nested twisted preconditioner on the GPU.

Drop-in for the reference ``ntdprecon.ntd_solve``
(/root/reference/pkg/src/ntdprecon/ntd_solve.py).  ``ntd_apply`` is one
launch of libntdgpu ``ntd_apply``: twisted plane sweeps (one warp pair per
level-3 half), twisted line sweeps (one warp per level-2 half) and
warp-shuffle affine scans for the innermost bidiagonal chains.  ``lanes``
(the reference's K-lane chain composition, :17) and ``workers`` are accepted
and ignored; results match the reference to rounding (<= 1e-10 relative is
the parity bar, typically ~1e-15).
"""

import numpy as np
import torch

from . import _lib
from . import device as D
from .banded_core import as_device, like_input, shape_of

CHAIN_LANES = 4


class SolveWorkspace:
    """Scratch reused across applications (ntd_solve.py:256-269): one device
    vector for the level-3 upper sweep's plane solves."""

    def __init__(self, n):
        self.n = int(n)
        self.scratch = None  # sized on first use (depends on the grid shape)

    def work(self, nx, ny, nz):
        need = _lib.load().ntd_apply_work_doubles(nx, ny, nz, 1)
        if self.scratch is None or self.scratch.numel() < need:
            self.scratch = torch.empty(need, dtype=torch.float64, device=torch.device("cuda"))
        return self.scratch


def chain_bidiagonal_solve(diag_recip, offdiag, b, direction="forward", lanes=CHAIN_LANES):
    """Public bidiagonal chain helper (ntd_solve.py:272-300).  Reference
    utility, not on the solve path: evaluated as the plain sequential
    recurrence (the reference's lanes == 1 form)."""
    dr = np.ascontiguousarray(diag_recip, dtype=np.float64)
    off = np.ascontiguousarray(offdiag, dtype=np.float64)
    rhs = np.ascontiguousarray(b, dtype=np.float64)
    n = dr.shape[0]
    if off.shape[0] != n or rhs.shape[0] != n:
        raise ValueError("chain solve operands must have equal length")
    if lanes < 1:
        raise ValueError("lanes must be >= 1")
    if direction not in ("forward", "backward"):
        raise ValueError(f"unknown direction {direction!r}")
    x = np.empty(n)
    order = range(n) if direction == "forward" else range(n - 1, -1, -1)
    xp = 0.0
    for p in order:
        xp = (rhs[p] - off[p] * xp) * dr[p]
        x[p] = xp
    return x


def ntd_apply(pre, b, workers=1, lanes=CHAIN_LANES, workspace=None):
    """x = B^{-1} b (ntd_solve.py:303-322).  b is not modified."""
    n = pre.n_rows
    if shape_of(b) != (n,):
        raise ValueError(f"rhs length {shape_of(b)} does not match {n} rows")
    bd = as_device(b)
    work = workspace.work(pre.nx, pre.ny, pre.nz) if workspace is not None else None
    x = D.ntd_apply(pre.bands, bd, pre.nx, pre.ny, pre.nz, 1, work=work, solve=pre.solve)
    return like_input(x, b)
