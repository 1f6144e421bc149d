"""Batched solves of independent systems and the preconditioner factory.

``BatchSolver`` factors and solves B independent systems of one grid shape
in single kernel launches (one CTA per system / system-half), the B200-native
form of BASELINE config 4 (64 independent 96^3 systems).  The reference has
no batch API: it runs one process per system.  ``build_precond`` mirrors the
reference CLI's string-keyed factory (bench_cli.py:113-142).
"""

from dataclasses import dataclass
from time import perf_counter

import torch

from . import _lib
from . import device as D
from .banded_core import FactorizationError, as_device
from .ilu0 import build_block_ilu0
from .ntd_factor import factor_level3
from .ntd_solve import SolveWorkspace
from .precond_pcg import CombinedPrecond

PRECOND_KINDS = ("ntd+ilu0", "ntd", "ilu0", "none")


class _NtdPrecond:
    """'ntd': the nested twisted preconditioner alone (bench_cli.py:113-121)."""

    def __init__(self, a):
        self.pre = factor_level3(a)
        self.workspace = SolveWorkspace(a.n_rows)
        self.a = a

    def device_apply(self, r_dev, z_dev, active=None):
        return D.ntd_apply(self.pre.bands, r_dev, self.a.nx, self.a.ny, self.a.nz, 1, x=z_dev,
                           work=self.workspace.work(self.a.nx, self.a.ny, self.a.nz), active=active,
                           solve=self.pre.solve)

    def __call__(self, r):
        from .ntd_solve import ntd_apply
        return ntd_apply(self.pre, r, workspace=self.workspace)


class _IluPrecond:
    """'ilu0': block ILU0 alone (bench_cli.py:124-130)."""

    def __init__(self, a):
        self.f = build_block_ilu0(a)
        self.a = a

    def device_apply(self, r_dev, z_dev, active=None):
        return D.ilu0_apply(self.f.device_data, self.f.split, r_dev, self.a.nx, self.a.ny, self.a.nz, 1,
                            z=z_dev, active=active, skew=self.f.skew())

    def __call__(self, r):
        from .ilu0 import ilu0_apply
        return ilu0_apply(self.f, r)


def build_precond(a, kind):
    """bench_cli.py:133-142: 'ntd+ilu0' | 'ntd' | 'ilu0' | 'none'."""
    if kind == "ntd+ilu0":
        return CombinedPrecond(a)
    if kind == "ntd":
        return _NtdPrecond(a)
    if kind == "ilu0":
        return _IluPrecond(a)
    if kind == "none":
        return None
    raise ValueError(f"unknown preconditioner {kind!r}")


@dataclass
class BatchResult:
    x: torch.Tensor            # (B, N) device
    iterations: list           # per system
    converged: list
    final_relres: list
    status: list               # ntdgpu NTD_PCG_* codes
    history: torch.Tensor      # (B, max_iters) device
    setup_seconds: float
    solve_seconds: float


class BatchSolver:
    """B independent systems (B, 7, N) on one grid shape, ntd+ilu0 PCG."""

    def __init__(self, a_dev, nx, ny, nz, kind="ntd+ilu0", max_iters=200):
        if kind not in ("ntd+ilu0", "none"):
            raise ValueError("BatchSolver supports 'ntd+ilu0' and 'none'")
        self.a = as_device(a_dev)
        self.batch = self.a.shape[0]
        self.nx, self.ny, self.nz = nx, ny, nz
        self.n = nx * ny * nz
        if tuple(self.a.shape) != (self.batch, 7, self.n):
            raise ValueError("a_dev must have shape (B, 7, nx*ny*nz)")
        self.kind = kind
        self.max_iters = max_iters
        self.precond = None
        self.setup_seconds = 0.0
        self.pcg = D.PcgDevice(self.a, nx, ny, nz, self.batch, max_iters)

    def setup(self):
        """Both factorisations for all systems (CombinedPrecond.__init__,
        precond_pcg.py:45-51)."""
        if self.kind == "none":
            return self
        torch.cuda.synchronize()
        t0 = perf_counter()
        g = (self.nx, self.ny, self.nz, self.batch)
        pre, st = D.ntd_factor(self.a, *g)
        bad = [(s, *map(int, st[s])) for s in range(self.batch) if int(st[s, 0])]
        if bad:
            s, code, plane, row = bad[0]
            raise FactorizationError(f"system {s}: " + D.ntd_factor_message(code, plane, row))
        if not D.check_grid_pattern(self.a, self.nx, self.ny, self.nz):
            raise ValueError("band entries coupling across a grid line/plane boundary must be zero")
        split = self.n // 2
        f, st2 = D.ilu0_factor(self.a, *g, split)
        bad = [s for s in range(self.batch) if int(st2[s, 0])]
        if bad:
            raise FactorizationError(f"system {bad[0]}: zero or non-finite pivot at row {int(st2[bad[0], 2])}")
        self.precond = D.CombinedDevice(self.a, *g, pre=pre, ilu=f, split=split)
        torch.cuda.synchronize()
        self.setup_seconds = perf_counter() - t0
        return self

    def solve(self, b_dev, tol=1e-8):
        b = as_device(b_dev).reshape(self.batch, self.n)
        torch.cuda.synchronize()
        t0 = perf_counter()
        papply = None if self.precond is None else self.precond.apply
        self.pcg.solve(b, tol, papply, None)
        fl, st = self.pcg.read_flags()
        dt = perf_counter() - t0
        fl = fl.clone()
        st = st.clone()
        return BatchResult(
            x=self.pcg.x, iterations=[int(v) for v in fl[:, _lib.NTD_FL["ITERS"]]],
            converged=[int(v) == _lib.PCG_CONVERGED for v in fl[:, _lib.NTD_FL["STATUS"]]],
            final_relres=[float(v) for v in st[:, _lib.NTD_ST["RELRES"]]],
            status=[int(v) for v in fl[:, _lib.NTD_FL["STATUS"]]],
            history=self.pcg.history, setup_seconds=self.setup_seconds, solve_seconds=dt)
