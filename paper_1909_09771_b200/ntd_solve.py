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
    """Bidiagonal chain x[i] = (b[i] - offdiag[i]*x[i_prev]) * diag_recip[i]
    (ntd_solve.py:272-300), on the GPU (libntdgpu ``ntd_chain_solve``) with
    the reference's lane composition: ``lanes`` equal chunks composed as
    affine maps, carries stitched in order, remainder walked sequentially,
    the plain recurrence when lanes == 1 or the chain is shorter than
    2*lanes (_chain_scaled, ntd_solve.py:20-64).  Bitwise the reference's
    result for every ``lanes``."""
    dr = as_device(diag_recip).reshape(-1)
    off = as_device(offdiag).reshape(-1)
    rhs = as_device(b).reshape(-1)
    n = dr.numel()
    if off.numel() != n or rhs.numel() != n:
        raise ValueError("chain solve operands must have equal length")
    if lanes < 1:
        raise ValueError("lanes must be >= 1")
    x = torch.empty_like(rhs)
    if n == 0:
        return like_input(x, b)
    if direction not in ("forward", "backward"):
        raise ValueError(f"unknown direction {direction!r}")
    work = torch.empty(_lib.load().ntd_chain_work_doubles(n, 1), dtype=torch.float64, device=rhs.device)
    _lib.call("ntd_chain_solve", _lib.ptr(dr), _lib.ptr(off), _lib.ptr(rhs), _lib.ptr(x), _lib.ptr(work), n, 1,
              0 if direction == "forward" else 1, int(lanes), _lib.stream())
    return like_input(x, b)


def ntd_apply(pre, b, workers=1, lanes=CHAIN_LANES, workspace=None):
    """x = B^{-1} b (ntd_solve.py:303-322).  b is not modified."""
    n = pre.n_rows
    if shape_of(b) != (n,):
        raise ValueError(f"rhs length {shape_of(b)} does not match {n} rows")
    bd = as_device(b)
    work = workspace.work(pre.nx, pre.ny, pre.nz) if workspace is not None else None
    x = D.ntd_apply(pre.bands, bd, pre.nx, pre.ny, pre.nz, 1, work=work, solve=pre.solve)
    return like_input(x, b)
