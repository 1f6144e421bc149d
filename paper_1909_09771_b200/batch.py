"""Batched solves of independent systems and the preconditioner factory.

``BatchSolver`` factors and solves B independent systems of one grid shape
in single kernel launches (one CTA per system / system-half), the B200-native
form of BASELINE config 4 (64 independent 96^3 systems).  The reference has
no batch API: it runs one process per system.  ``build_precond`` mirrors the
reference CLI's string-keyed factory (bench_cli.py:113-142).
"""

import os
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


def default_groups(batch):
    """Stream groups for a batch: the NTD apply and the ILU0 sweeps are
    latency-bound (one CTA per system / half), so while one group sweeps, the
    bandwidth-bound stencil/CG kernels of the other run on the idle SMs."""
    # CUDA multiplexes streams over CUDA_DEVICE_MAX_CONNECTIONS hardware queues
    # (default 8; the package raises the default to 32 before CUDA starts):
    # more groups than queues serialise (16 groups on 8 queues: 1.5x slower).
    # Measured on the 64-system batch with 32 queues: 8 groups 4756, 16 groups
    # 4988, 32 groups 5008 Munk-iter/s; 16 keeps the host's launch work low.
    queues = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
    return max(1, min(16 if queues >= 16 else 8, batch))


class _Group:
    """One slice [lo, hi) of the batch: its own factors, PCG state and stream."""

    def __init__(self, a, lo, hi, nx, ny, nz, max_iters, x_view, stream):
        self.lo, self.hi = lo, hi
        self.a = a[lo:hi]
        self.stream = stream
        self.pcg = D.PcgDevice(self.a, nx, ny, nz, hi - lo, max_iters, x=x_view, a4=None)
        self.precond = None
        self.flags_host = [torch.zeros((hi - lo, _lib.NTD_FL["N"]), dtype=torch.int32).pin_memory()
                           for _ in range(2)]
        self.events = [torch.cuda.Event() for _ in range(2)]


class BatchSolver:
    """B independent systems (B, 7, N) on one grid shape, ntd+ilu0 PCG.

    The batch is split into `groups` slices, each enqueued on its own CUDA
    stream, so the latency-bound sweeps of one slice overlap the
    bandwidth-bound kernels of another.  The host never blocks inside the
    iteration loop: convergence flags are copied asynchronously and checked
    one iteration late (converged systems are masked on the device, so the
    extra enqueued iteration does no work for them)."""

    def __init__(self, a_dev, nx, ny, nz, kind="ntd+ilu0", max_iters=200, groups=None, sweep_priority="hi",
                 dynamic_ctas=True):
        if kind not in ("ntd+ilu0", "ntd", "none"):
            raise ValueError("BatchSolver supports 'ntd+ilu0', 'ntd' and 'none'")
        self.a = as_device(a_dev)
        self.batch = self.a.shape[0]
        self.nx, self.ny, self.nz = nx, ny, nz
        self.n = nx * ny * nz
        if tuple(self.a.shape) != (self.batch, 7, self.n):
            raise ValueError("a_dev must have shape (B, 7, nx*ny*nz)")
        if sweep_priority not in ("hi", "lo", "off"):
            raise ValueError("sweep_priority must be 'hi', 'lo' or 'off'")
        self.kind = kind
        self.max_iters = max_iters
        # sweep_priority: stream priority of the latency-bound sweeps (see
        # setup); dynamic_ctas: re-map the ILU0 CTAs to the systems still
        # iterating (bitwise neutral).  Both exist for measurements.
        self.sweep_priority = sweep_priority
        self.dynamic_ctas = dynamic_ctas
        self.setup_seconds = 0.0
        G = default_groups(self.batch) if groups is None else max(1, min(int(groups), self.batch))
        self.x = torch.empty((self.batch, self.n), dtype=torch.float64, device=self.a.device)
        self.history = torch.zeros((self.batch, max(1, max_iters)), dtype=torch.float64, device=self.a.device)
        bounds = [self.batch * g // G for g in range(G + 1)]
        self.groups = []
        for g in range(G):
            lo, hi = bounds[g], bounds[g + 1]
            st = torch.cuda.current_stream() if G == 1 else torch.cuda.Stream()
            self.groups.append(_Group(self.a, lo, hi, nx, ny, nz, max_iters, self.x[lo:hi], st))

    @property
    def precond(self):
        """The first group's preconditioner (all of it when groups == 1)."""
        return self.groups[0].precond

    def setup(self):
        """Both factorisations for all systems (CombinedPrecond.__init__,
        precond_pcg.py:45-51)."""
        if self.kind == "none":
            return self
        torch.cuda.synchronize()
        t0 = perf_counter()
        if not D.check_grid_pattern(self.a, self.nx, self.ny, self.nz):
            raise ValueError("band entries coupling across a grid line/plane boundary must be zero")
        # both factorisations and the symmetric pack for the whole batch, one
        # launch each (the setup kernels are latency-bound per system, so one
        # launch of B CTAs costs what one group would); the stream groups
        # then work on views of these tensors
        g = (self.nx, self.ny, self.nz, self.batch)
        pre, st = D.ntd_factor(self.a, *g)
        bad = [(s, *map(int, st[s])) for s in range(self.batch) if int(st[s, 0])]
        if bad:
            s, code, plane, row = bad[0]
            raise FactorizationError(f"system {s}: " + D.ntd_factor_message(code, plane, row))
        split = self.n // 2
        if self.kind == "ntd+ilu0":
            f, st2 = D.ilu0_factor(self.a, *g, split)
            bad = [s for s in range(self.batch) if int(st2[s, 0])]
            if bad:
                raise FactorizationError(f"system {bad[0]}: zero or non-finite pivot at row {int(st2[bad[0], 2])}")
        a4 = D.sym_pack(self.a, *g)  # symmetric 4-band operator for the stencil kernels
        # The latency-bound sweeps (ILU0, NTD) of every group run on a
        # high-priority stream of their own, so an SM freed by a short stencil
        # kernel goes to a waiting sweep CTA first: +1.8% on the 64-system
        # batch (8 alternating runs).  Two streams per group: only while they
        # all get a hardware queue of their own (32 groups -> 64 streams on 32
        # queues: 20% slower).
        prio = self.sweep_priority
        if 2 * len(self.groups) > int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")):
            prio = "off"
        for grp in self.groups:
            lo, hi = grp.lo, grp.hi
            grp.pcg.a4 = None if a4 is None else a4[lo:hi]
            if self.kind == "ntd":
                grp.precond = D.NtdDevice(pre[lo:hi], self.nx, self.ny, self.nz, hi - lo,
                                          ntd_ctas_=D.ntd_ctas(self.batch))
            else:
                grp.precond = D.CombinedDevice(grp.a, self.nx, self.ny, self.nz, hi - lo, pre=pre[lo:hi],
                                               ilu=f[lo:hi], split=split, a4=grp.pcg.a4,
                                               ilu_ctas=D.ilu0_ctas(self.batch), ntd_ctas_=D.ntd_ctas(self.batch),
                                               ilu_hp=D.ilu0_hp_config(self.nx, self.ny, self.nz, split, self.batch))
            if prio in ("hi", "lo") and len(self.groups) > 1:
                lo_p, hi_p = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
                    else (0, -1)
                grp.precond.sweep_stream = torch.cuda.Stream(priority=hi_p if prio == "hi" else lo_p)
                if prio == "lo":
                    grp.stream = torch.cuda.Stream(priority=hi_p)
        torch.cuda.synchronize()
        self.setup_seconds = perf_counter() - t0
        return self

    def solve(self, b_dev, tol=1e-8, x_out=None):
        """Solve all systems.  x_out: optional device (B, N) tensor that
        receives the solutions (default: the solver's own buffer), so a caller
        can copy one solve's x to the host while the next solve runs."""
        return self._solve(as_device(b_dev).reshape(self.batch, self.n), tol, x_out)

    def solve_host(self, b_host, x_host, tol=1e-8):
        """Solve from and to host memory: b_host, x_host (B, N) fp64 CPU
        tensors (pinned for asynchronous copies).  Each stream group uploads
        its slice of b on its own stream just before its PCG starts and
        downloads its slice of x as soon as the host sees that all its systems
        have stopped, so the transfers overlap the other groups' sweeps.
        x_host holds the solutions when this returns."""
        if tuple(b_host.shape) != (self.batch, self.n) or tuple(x_host.shape) != (self.batch, self.n):
            raise ValueError(f"b_host and x_host must have shape ({self.batch}, {self.n})")
        if b_host.is_cuda or x_host.is_cuda:
            raise ValueError("solve_host takes host tensors; use solve() for device tensors")
        if getattr(self, "_b_dev", None) is None:
            self._b_dev = torch.empty((self.batch, self.n), dtype=torch.float64, device=self.a.device)
        b = self._b_dev

        def upload(grp):
            b[grp.lo:grp.hi].copy_(b_host[grp.lo:grp.hi], non_blocking=True)

        def download(grp):
            x_host[grp.lo:grp.hi].copy_(self.x[grp.lo:grp.hi], non_blocking=True)

        return self._solve(b, tol, None, on_start=upload, on_done=download)

    def solve_many(self, bs, tol=1e-8, x_outs=None):
        """Solve K right-hand-side batches bs[k] (B, N) one after another,
        pipelined per stream group: a group starts its slice of solve k+1 as
        soon as its own systems have stopped in solve k, so the converged
        groups' SMs go to the next solve instead of idling through the
        stragglers' last iterations.  Results (one BatchResult per solve) are
        bitwise those of K solve() calls.  x_outs: optional K device (B, N)
        tensors (default: one fresh tensor per solve)."""
        bs = [as_device(b).reshape(self.batch, self.n) for b in bs]
        if x_outs is None:
            x_outs = [torch.empty((self.batch, self.n), dtype=torch.float64, device=self.a.device) for _ in bs]
        xs = [x.reshape(self.batch, self.n) for x in x_outs]
        return self._solve_pipelined(bs, xs, tol)

    def solve_host_many(self, b_hosts, x_hosts, tol=1e-8):
        """solve_many from and to host memory (pinned (B, N) CPU tensors):
        each group uploads its slice of b_hosts[k] when it starts solve k and
        downloads its slice of x as soon as it has finished it."""
        if len(b_hosts) != len(x_hosts):
            raise ValueError("b_hosts and x_hosts must have the same length")
        for b_host, x_host in zip(b_hosts, x_hosts):
            if tuple(b_host.shape) != (self.batch, self.n) or tuple(x_host.shape) != (self.batch, self.n):
                raise ValueError(f"b_hosts and x_hosts must have shape ({self.batch}, {self.n})")
            if b_host.is_cuda or x_host.is_cuda:
                raise ValueError("solve_host_many takes host tensors; use solve_many() for device tensors")
        if getattr(self, "_b_dev", None) is None:
            self._b_dev = torch.empty((self.batch, self.n), dtype=torch.float64, device=self.a.device)
        b = self._b_dev  # each group reads and writes only its own slice

        def upload(grp, k):
            b[grp.lo:grp.hi].copy_(b_hosts[k][grp.lo:grp.hi], non_blocking=True)

        def download(grp, k):
            x_hosts[k][grp.lo:grp.hi].copy_(self.x[grp.lo:grp.hi], non_blocking=True)

        K = len(b_hosts)
        return self._solve_pipelined([b] * K, [self.x] * K, tol, upload, download)

    def reserve(self, solves):
        """Preallocate the per-solve result buffers of solve_many for up to
        `solves` right-hand sides (pinned host memory is slow to allocate).
        The buffers are reused by later calls."""
        bufs = getattr(self, "_pipe_bufs", None) or ([], [], [])
        while len(bufs[0]) < solves:
            bufs[0].append(torch.empty_like(self.history))
            bufs[1].append(torch.zeros((self.batch, _lib.NTD_FL["N"]), dtype=torch.int32))
            bufs[2].append(torch.zeros((self.batch, _lib.NTD_ST["N"]), dtype=torch.float64).pin_memory())
        self._pipe_bufs = bufs

    def _solve_pipelined(self, bs, xs, tol, on_start=None, on_done=None):
        K = len(bs)
        if K == 0:
            return []
        groups = self.groups
        cur = torch.cuda.current_stream()
        t0 = perf_counter()
        for grp in groups:
            grp.stream.wait_stream(cur)
        self.reserve(K)
        hist, flags_out, state_out = (v[:K] for v in self._pipe_bufs)
        self._dynamic_ctas = self.dynamic_ctas
        self._map_ctas(self.batch)

        def begin(grp, it):
            grp.k_begin = it
            grp.its = 0
            with torch.cuda.stream(grp.stream):
                grp.pcg.x = xs[grp.k][grp.lo:grp.hi]
                if on_start is not None:
                    on_start(grp, grp.k)
                grp.pcg.init(bs[grp.k][grp.lo:grp.hi], tol)
                z = grp.pcg.r if grp.precond is None else grp.precond.apply(grp.pcg.r, grp.pcg.z, grp.pcg.active)
                grp.pcg.start(z)

        def finish(grp, slot):
            k, lo, hi = grp.k, grp.lo, grp.hi
            flags_out[k][lo:hi] = grp.flags_host[slot]
            with torch.cuda.stream(grp.stream):
                state_out[k][lo:hi].copy_(grp.pcg.state, non_blocking=True)
                hist[k][lo:hi].copy_(grp.pcg.history)
                if on_done is not None:
                    on_done(grp, k)

        for grp in groups:
            grp.k = 0
            grp.finished = False
            grp.its_slot = [0, 0]
            begin(grp, 0)
        it = 0
        while not all(grp.finished for grp in groups):
            it += 1
            if it > K * (self.max_iters + 3):
                raise RuntimeError("pipelined solve did not terminate")  # protocol error
            for grp in groups:
                if not grp.finished and grp.its < self.max_iters:
                    with torch.cuda.stream(grp.stream):
                        grp.pcg.step_update()
                    grp.its += 1
            for grp in groups:
                grp.its_slot[it % 2] = grp.its
            self._flags_async(it % 2)
            slot = (it - 1) % 2
            n_act = 0
            restarted = set()
            act = _lib.NTD_FL["ACTIVE"]
            for grp in groups:
                if grp.finished:
                    continue
                if it < grp.k_begin + 2:  # no flags of this solve yet
                    n_act += grp.hi - grp.lo
                    continue
                grp.events[slot].synchronize()
                g_act = int(grp.flags_host[slot][:, act].sum())
                if g_act and grp.its_slot[slot] < self.max_iters:
                    n_act += g_act
                    continue
                finish(grp, slot)
                restarted.add(grp)
                grp.k += 1
                if grp.k < K:
                    begin(grp, it)
                    n_act += grp.hi - grp.lo
                else:
                    grp.finished = True
            self._map_ctas(n_act)
            for grp in groups:
                if grp.finished or grp in restarted or grp.its >= self.max_iters:
                    continue
                with torch.cuda.stream(grp.stream):
                    z = grp.pcg.r if grp.precond is None else grp.precond.apply(grp.pcg.r, grp.pcg.z,
                                                                                  grp.pcg.active)
                    grp.pcg.direction(z)
        for grp in groups:
            cur.wait_stream(grp.stream)
        torch.cuda.current_stream().synchronize()
        dt = perf_counter() - t0
        out = []
        for k in range(K):
            fl, st = flags_out[k], state_out[k]
            out.append(BatchResult(
                x=xs[k], iterations=[int(v) for v in fl[:, _lib.NTD_FL["ITERS"]]],
                converged=[int(v) == _lib.PCG_CONVERGED for v in fl[:, _lib.NTD_FL["STATUS"]]],
                final_relres=[float(v) for v in st[:, _lib.NTD_ST["RELRES"]]],
                status=[int(v) for v in fl[:, _lib.NTD_FL["STATUS"]]],
                history=hist[k], setup_seconds=self.setup_seconds, solve_seconds=dt))
        return out

    def _solve(self, b, tol, x_out, on_start=None, on_done=None):
        x = self.x if x_out is None else x_out.reshape(self.batch, self.n)
        for grp in self.groups:
            grp.pcg.x = x[grp.lo:grp.hi]
        cur = torch.cuda.current_stream()
        t0 = perf_counter()
        for grp in self.groups:
            grp.stream.wait_stream(cur)  # b may have been produced on the caller's stream
        self._run(b, tol, on_start, on_done)
        for grp in self.groups:
            cur.wait_stream(grp.stream)
        fl = torch.cat([grp.pcg.flags for grp in self.groups]).cpu()
        st = torch.cat([grp.pcg.state for grp in self.groups]).cpu()
        for grp in self.groups:
            self.history[grp.lo:grp.hi] = grp.pcg.history
        dt = perf_counter() - t0
        return BatchResult(
            x=x, iterations=[int(v) for v in fl[:, _lib.NTD_FL["ITERS"]]],
            converged=[int(v) == _lib.PCG_CONVERGED for v in fl[:, _lib.NTD_FL["STATUS"]]],
            final_relres=[float(v) for v in st[:, _lib.NTD_ST["RELRES"]]],
            status=[int(v) for v in fl[:, _lib.NTD_FL["STATUS"]]],
            history=self.history, setup_seconds=self.setup_seconds, solve_seconds=dt)

    def _flags_async(self, slot):
        for grp in self.groups:
            with torch.cuda.stream(grp.stream):
                grp.flags_host[slot].copy_(grp.pcg.flags, non_blocking=True)
                grp.events[slot].record(grp.stream)

    def _any_active(self, slot, on_done=None, done=None):
        """Whether any system is still iterating (flags of the copy in
        `slot`).  on_done(grp) is enqueued on a group's stream the first time
        all its systems have stopped (their later kernels are masked no-ops)."""
        act = _lib.NTD_FL["ACTIVE"]
        alive = False
        n_act = 0
        for grp in self.groups:
            grp.events[slot].synchronize()
            g_act = int(grp.flags_host[slot][:, act].sum())
            n_act += g_act
            alive = alive or g_act > 0
            if g_act == 0 and on_done is not None and grp not in done:
                done.add(grp)
                with torch.cuda.stream(grp.stream):
                    on_done(grp)
        self._map_ctas(n_act)
        return alive

    def _map_ctas(self, systems):
        """Skewed-ILU0 CTA mapping for the systems still iterating (masked
        systems' CTAs exit at once): as the batch converges, the stragglers'
        sweeps spread over the SMs the finished systems freed.  (The choice
        of the hyperplane kernel stays fixed for the batch: switching to it
        for the tail was 3% slower at 64 systems.)  Bitwise the same results
        for every mapping."""
        if not self._dynamic_ctas:
            return
        ctas = D.ilu0_ctas(max(1, systems))
        for grp in self.groups:
            if isinstance(grp.precond, D.CombinedDevice):
                grp.precond.ilu_ctas = ctas

    def _run(self, b, tol, on_start=None, on_done=None):
        """PCG (precond_pcg.py:84-119) on every group, enqueued round-robin.
        Iteration it's update is enqueued before the host looks at the flags
        of iteration it-1, so the GPU always has queued work."""
        groups = self.groups
        done = set()
        try:
            self._run_groups(b, tol, on_start, on_done, done)
        finally:
            if on_done is not None:
                for grp in groups:
                    if grp not in done:
                        done.add(grp)
                        with torch.cuda.stream(grp.stream):
                            on_done(grp)

    def _run_groups(self, b, tol, on_start, on_done, done):
        groups = self.groups
        self._dynamic_ctas = self.dynamic_ctas
        self._map_ctas(self.batch)
        for grp in groups:
            with torch.cuda.stream(grp.stream):
                if on_start is not None:
                    on_start(grp)
                grp.pcg.init(b[grp.lo:grp.hi], tol)
        self._flags_async(0)
        for grp in groups:
            with torch.cuda.stream(grp.stream):
                z = grp.pcg.r if grp.precond is None else grp.precond.apply(grp.pcg.r, grp.pcg.z, grp.pcg.active)
                grp.pcg.start(z)
        if not self._any_active(0, on_done, done):
            return
        for it in range(1, self.max_iters + 1):
            for grp in groups:
                with torch.cuda.stream(grp.stream):
                    grp.pcg.step_update()
            self._flags_async(it % 2)
            if it >= 2 and not self._any_active((it - 1) % 2, on_done, done):
                break  # everything had converged at it-1; iteration it was fully masked
            if it == self.max_iters:
                break
            for grp in groups:
                with torch.cuda.stream(grp.stream):
                    z = grp.pcg.r if grp.precond is None else grp.precond.apply(grp.pcg.r, grp.pcg.z,
                                                                                  grp.pcg.active)
                    grp.pcg.direction(z)
