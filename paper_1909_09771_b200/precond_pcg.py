"""Combination preconditioning and the conjugate gradient driver, on the GPU.

Drop-in for the reference ``ntdprecon.precond_pcg``
(/root/reference/pkg/src/ntdprecon/precond_pcg.py).  The PCG loop keeps all
vectors and per-iteration scalars on the device (device.PcgDevice); the host
reads back only the convergence flags and the relative residual each
iteration.  ``pcg`` accepts any callable ``r -> z`` as preconditioner (the
reference's plugin point, :71-74); the package's own preconditioners are
applied without leaving the device.
"""

from dataclasses import dataclass, field
from time import perf_counter

import torch

from . import _lib
from . import device as D
from .banded_core import as_device, like_input, shape_of
from .ilu0 import build_block_ilu0
from .ntd_factor import factor_level3
from .ntd_solve import CHAIN_LANES, SolveWorkspace


class DivergenceError(RuntimeError):
    """Raised when the iteration produces a non-finite or breakdown value
    (precond_pcg.py:14-15)."""


@dataclass
class SolveStats:
    """precond_pcg.py:18-25"""

    iterations: int
    converged: bool
    relres_history: list = field(default_factory=list)
    final_relres: float = 0.0
    solve_seconds: float = 0.0
    setup_seconds: float = 0.0


class CombinedPrecond:
    """Block ILU0 smoothing wrapped symmetrically around the nested twisted
    solve (precond_pcg.py:28-54):  w = B_ilu^-1 r;  z = w + B_ntd^-1 (r - A w);
    z += B_ilu^-1 (r - A z).  Construction performs both factorisations on the
    GPU."""

    def __init__(self, a, workers=1, lanes=CHAIN_LANES):
        t0 = perf_counter()
        self.a = a
        self.workers = workers
        self.lanes = lanes
        self.ntd = factor_level3(a, lanes=lanes, workers=workers)
        self.ilu = build_block_ilu0(a, workers=workers)
        self.workspace = SolveWorkspace(a.n_rows)
        self._ad = a.device_data()
        self._dev = D.CombinedDevice(self._ad, a.nx, a.ny, a.nz, 1, pre=self.ntd.bands,
                                     ilu=self.ilu.device_data, split=self.ilu.split,
                                     solve=self.ntd.solve, skew=self.ilu.skew())
        torch.cuda.current_stream().synchronize()
        self.setup_seconds = perf_counter() - t0

    def device_apply(self, r_dev, z_dev, active=None):
        """z = M^-1 r on device (B=1) tensors."""
        return self._dev.apply(r_dev, z_dev, active)

    def __call__(self, r):
        return combined_apply(self, r)


def combined_apply(precond, r):
    """precond_pcg.py:57-65"""
    rd = as_device(r).reshape(1, -1)
    z = torch.empty_like(rd)
    precond.device_apply(rd, z)
    return like_input(z.reshape(-1), r)


def pcg(a, b, precond=None, tol=1e-7, max_iters=200, workers=1, callback=None):
    """Preconditioned CG from x0 = 0 with true-residual stopping
    ||b - A x|| / ||b|| < tol (precond_pcg.py:68-122).  Returns (x, SolveStats);
    x follows the type of b (numpy in, numpy out; CUDA tensor in, tensor out)."""
    n = a.n_rows
    if shape_of(b) != (n,):
        raise ValueError(f"rhs length {shape_of(b)} does not match {n} rows")
    if tol <= 0.0:
        raise ValueError("tol must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    t0 = perf_counter()
    ad = a.device_data()
    bd = as_device(b).reshape(1, n)

    if precond is None:
        papply = None
    elif hasattr(precond, "device_apply"):
        papply = precond.device_apply
    else:
        def papply(r_dev, z_dev, active):
            # generic plugin: hand the callable a vector in the caller's flavour
            rv = like_input(r_dev.reshape(-1), b)
            zv = precond(rv)
            z_dev.copy_(as_device(zv).reshape(z_dev.shape))
            return z_dev

    if callback is None and (precond is None or hasattr(precond, "device_apply")):
        # device-only iteration: replayed as a CUDA graph, no per-iteration
        # host round trip (PcgDevice.solve_graph)
        solver = _graphed_solver(precond, ad, a, max_iters)
        solver.solve_graph(bd, tol, papply, graph_key=id(precond))
        fl, st = solver.read_flags()
        iters = int(fl[0, _lib.NTD_FL["ITERS"]])
        status = int(fl[0, _lib.NTD_FL["STATUS"]])
        history = solver.history[0, :iters].cpu().tolist()
        if status == _lib.PCG_BREAKDOWN:
            pap = float(st[0, _lib.NTD_ST["PAP"]])
            raise DivergenceError(f"breakdown at iteration {iters + 1}: p.A.p = {pap}")
        if status == _lib.PCG_NONFINITE:
            raise DivergenceError(f"non-finite residual at iteration {iters}")
        x = like_input(solver.x.reshape(-1).clone(), b)
        final = history[-1] if history else 0.0
        return x, SolveStats(iters, status == _lib.PCG_CONVERGED, history, final, perf_counter() - t0)

    solver = D.PcgDevice(ad, a.nx, a.ny, a.nz, 1, max_iters)
    history = []
    err = []

    def on_iter(it, fl, st):
        status = int(fl[0, _lib.NTD_FL["STATUS"]])
        if status == _lib.PCG_BREAKDOWN:
            pap = float(st[0, _lib.NTD_ST["PAP"]])
            err.append(DivergenceError(f"breakdown at iteration {it}: p.A.p = {pap}"))
            raise err[-1]
        relres = float(st[0, _lib.NTD_ST["RELRES"]])
        history.append(relres)
        if status == _lib.PCG_NONFINITE:
            raise DivergenceError(f"non-finite residual at iteration {it}")
        if callback is not None:
            callback(it, like_input(solver.x.reshape(-1).clone(), b), relres)

    it = solver.solve(bd, tol, papply, on_iter)
    fl, _ = solver.read_flags()
    converged = int(fl[0, _lib.NTD_FL["STATUS"]]) == _lib.PCG_CONVERGED
    x = like_input(solver.x.reshape(-1), b)
    final = history[-1] if history else 0.0
    return x, SolveStats(it, converged, history, final, perf_counter() - t0)


def _graphed_solver(precond, ad, a, max_iters):
    """The PcgDevice (with its captured iteration) for this operator and
    preconditioner, cached on the preconditioner object so repeated solves
    reuse the graph."""
    key = (ad.data_ptr(), a.nx, a.ny, a.nz, max_iters)
    cache = getattr(precond, "_pcg_devices", None) if precond is not None else None
    if cache is not None and key in cache:
        return cache[key]
    solver = D.PcgDevice(ad, a.nx, a.ny, a.nz, 1, max_iters)
    if precond is not None:
        try:
            precond._pcg_devices = {key: solver}  # one operator at a time
        except AttributeError:
            pass
    return solver


__all__ = ["CombinedPrecond", "DivergenceError", "SolveStats", "combined_apply", "pcg"]
