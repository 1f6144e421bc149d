"""Zero-fill ILU of the two decoupled halves of a banded matrix, on the GPU.

Drop-in for the reference ``ntdprecon.ilu0``
(/root/reference/pkg/src/ntdprecon/ilu0.py).  Factor and triangular solves
run in libntdgpu (``ntd_ilu0_factor`` / ``ntd_ilu0_apply``) as skewed
wavefronts that reproduce the reference's natural-order row loops bit for
bit.
"""


from . import device as D
from .banded_core import FactorizationError, as_device, like_input, shape_of


class ILU0Factors:
    """Factored bands in the 7-diagonal layout (ilu0.py:17-31); ``data`` is
    materialised on the host lazily, ``device_data`` stays on the GPU."""

    def __init__(self, nx, ny, nz, split, data):
        self.nx, self.ny, self.nz, self.split = int(nx), int(ny), int(nz), int(split)
        self.device_data = as_device(data)
        self._host = None
        self._skew = False  # lazily built skewed coefficient records (fast apply path)

    def skew(self):
        if self._skew is False:
            self._skew = D.ilu0_skew_build(self.device_data, self.split, self.nx, self.ny, self.nz, 1)
        return self._skew

    @property
    def n_rows(self):
        return self.nx * self.ny * self.nz

    @property
    def data(self):
        if self._host is None:
            self._host = self.device_data.cpu().numpy()
        return self._host


def build_block_ilu0(a, workers=1, split=None):
    """ILU0 of blkdiag(A[:M,:M], A[M:,M:]), M = floor(N/2) (ilu0.py:134-156)."""
    n = a.n_rows
    if n < 2:
        raise ValueError("need at least two rows to split")
    if split is None:
        split = n // 2
    if not 1 <= split <= n:
        raise ValueError("split out of range")
    ad = a.device_data()
    if not D.check_grid_pattern(ad, a.nx, a.ny, a.nz):
        raise ValueError("band entries coupling across a grid line/plane boundary must be zero "
                         "(BandedMatrix invariant)")
    f, status = D.ilu0_factor(ad, a.nx, a.ny, a.nz, 1, split)
    if int(status[0, 0]):
        raise FactorizationError(f"zero or non-finite pivot at row {int(status[0, 2])}")
    return ILU0Factors(a.nx, a.ny, a.nz, split, f[0])


def ilu0_apply(factors, r, workers=1):
    """z = (L U)^{-1} r, both halves independent (ilu0.py:159-169)."""
    n = factors.n_rows
    if shape_of(r) != (n,):
        raise ValueError(f"operand length {shape_of(r)} does not match {n} rows")
    rd = as_device(r)
    z = D.ilu0_apply(factors.device_data, factors.split, rd, factors.nx, factors.ny, factors.nz, 1,
                     skew=factors.skew())
    return like_input(z, r)


__all__ = ["ILU0Factors", "build_block_ilu0", "ilu0_apply"]
