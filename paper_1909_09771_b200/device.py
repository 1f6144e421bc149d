"""Batched device-side building blocks (B independent systems per launch).

Everything here works on CUDA tensors laid out batch-major -- operators and
factors (B, 7, N), vectors (B, N) -- and calls libntdgpu.so through the C ABI
(include/ntdgpu.h).  The reference-compatible single-system API
(banded_core / ntd_factor / ntd_solve / ilu0 / precond_pcg) and the batched
solver both sit on top of these functions.
"""

import contextlib

import torch

from . import _lib

FACTOR_MESSAGES = {1: "zero or non-finite pivot", 2: "non-finite filter weight",
                   3: "non-finite sandwich adjustment"}


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def ntd_factor_message(code, plane, row):
    """Reference FactorizationError texts (ntd_factor.py:383-386,397-399,414-419)."""
    if code == 1:
        return f"zero or non-finite pivot at row {row} (plane {plane})"
    if code == 2 and row >= 0:
        return f"non-finite filter weight at row {row} (plane {plane})"
    if code == 2:
        return f"plane {plane}: non-finite filter weights"
    return f"plane {plane}: non-finite sandwich adjustment"


def assemble(kappa_dev, nx, ny, nz, dirichlet=(True,) * 6):
    """7-band operators (B,7,N) from cellwise kappa (B, nz, ny, nx) or (B, N)
    on the device (problem_gen.py:87-133, bitwise); dirichlet: six face flags
    x-, x+, y-, y+, z-, z+ (False = Neumann)."""
    k = kappa_dev.reshape(-1, nx * ny * nz).contiguous()
    batch = k.shape[0]
    mask = sum(1 << f for f, on in enumerate(dirichlet) if on)
    a = torch.empty((batch, 7, nx * ny * nz), dtype=torch.float64, device=k.device)
    _lib.call("ntd_assemble", _lib.ptr(k), _lib.ptr(a), nx, ny, nz, mask, batch, _lib.stream())
    return a


def ntd_factor(a_dev, nx, ny, nz, batch):
    """factor_level3 on B systems.  Returns (pre (B,7,N), status (B,3) host)."""
    lib = _lib.load()
    n = nx * ny * nz
    pre = torch.empty((batch, 7, n), dtype=torch.float64, device=_dev())
    work = torch.empty(lib.ntd_factor_work_doubles(nx, ny, nz, batch), dtype=torch.float64, device=_dev())
    status = torch.zeros((batch, 3), dtype=torch.int64, device=_dev())
    _lib.call("ntd_factor", _lib.ptr(a_dev), _lib.ptr(pre), _lib.ptr(work), _lib.ptr(status), nx, ny, nz,
              batch, _lib.stream())
    return pre, status.cpu()


def solve_bands(pre_dev, nx, ny, nz, batch):
    """Apply-side solve arrays of a factor (slot layout, chain coefficients
    precomputed); None when the grid uses the direct apply path."""
    size = _lib.load().ntd_solve_doubles(nx, ny, nz, batch)
    if size == 0:
        return None
    sv = torch.empty(size, dtype=torch.float64, device=_dev())
    _lib.call("ntd_solve_bands", _lib.ptr(pre_dev), _lib.ptr(sv), nx, ny, nz, batch, _lib.stream())
    return sv


def ntd_apply(pre_dev, b_dev, nx, ny, nz, batch, x=None, work=None, active=None, solve=None, ctas=None):
    """x = M_NTD^{-1} b on B systems; ctas: CTAs per system (default
    ntd_ctas(batch)); results are bitwise independent of it."""
    lib = _lib.load()
    if x is None:
        x = torch.empty_like(b_dev)
    if work is None or work.numel() < lib.ntd_apply_work_doubles(nx, ny, nz, batch):
        work = torch.empty(lib.ntd_apply_work_doubles(nx, ny, nz, batch), dtype=torch.float64, device=_dev())
    _lib.call("ntd_apply_ex", _lib.ptr(pre_dev), _lib.ptr(solve), _lib.ptr(b_dev), _lib.ptr(x), _lib.ptr(work), nx,
              ny, nz, batch, _lib.ptr(active), ntd_ctas(batch) if ctas is None else ctas, _lib.stream())
    return x


def ntd_apply_direct(pre_dev, b_dev, nx, ny, nz, batch, x=None, work=None, active=None):
    """x = M_NTD^{-1} b by the direct-load kernel on the reference band layout
    (the path of grids without slot-layout records, e.g. nx > 352)."""
    lib = _lib.load()
    if x is None:
        x = torch.empty_like(b_dev)
    if work is None or work.numel() < lib.ntd_apply_work_doubles(nx, ny, nz, batch):
        work = torch.empty(lib.ntd_apply_work_doubles(nx, ny, nz, batch), dtype=torch.float64, device=_dev())
    _lib.call("ntd_apply_direct", _lib.ptr(pre_dev), _lib.ptr(b_dev), _lib.ptr(x), _lib.ptr(work), nx, ny, nz, batch,
              _lib.ptr(active), _lib.stream())
    return x


def check_grid_pattern(a_dev, nx, ny, nz):
    """True when no band couples across a line or plane boundary
    (BandedMatrix invariant, banded_core.py:39-42); required by the ILU0
    wavefront kernels."""
    d = a_dev.reshape(-1, 7, nz, ny, nx)
    bad = (d[:, 2, :, :, 0] != 0).any() | (d[:, 4, :, :, nx - 1] != 0).any()
    bad = bad | (d[:, 1, :, 0, :] != 0).any() | (d[:, 5, :, ny - 1, :] != 0).any()
    return not bool(bad.item())


def ilu0_factor(a_dev, nx, ny, nz, batch, split):
    n = nx * ny * nz
    f = torch.empty((batch, 7, n), dtype=torch.float64, device=_dev())
    status = torch.zeros((batch, 3), dtype=torch.int64, device=_dev())
    _lib.call("ntd_ilu0_factor", _lib.ptr(a_dev), _lib.ptr(f), split, _lib.ptr(status), nx, ny, nz, batch,
              _lib.stream())
    return f, status.cpu()


def ilu0_skew_build(f_dev, split, nx, ny, nz, batch):
    """Skewed-layout coefficient records of an ILU0 factor, or None when the
    split is not a plane boundary (then the reference-layout kernel is used)."""
    size = _lib.load().ntd_ilu0_skew_doubles(nx, ny, nz, batch, split)
    if size == 0:
        return None
    coef = torch.empty(size, dtype=torch.float64, device=_dev())
    _lib.call("ntd_ilu0_skew_build", _lib.ptr(f_dev), _lib.ptr(coef), split, nx, ny, nz, batch, _lib.stream())
    return coef


SMS = 148


ILU0_WARPS = 24  # warps per CTA of the one-CTA-per-half sweep (skew::WARPS)


def ilu0_ctas(systems_on_gpu):
    """(CTAs per system half, warps per CTA) for the skewed ILU0 sweep: a
    cluster of up to 8 CTAs on separate SMs when the GPU's whole load (all
    systems, every stream group) leaves SMs idle, else one 24-warp CTA per
    half."""
    # measured (tools/ilu0_ctas_scan.py, 96^3, ms per apply at 1 / 8 / 16
    # systems): 1x24 1.25/1.27/1.28, 2x24 1.10/1.12/1.15, 4x12 0.95/0.99/1.03;
    # 8x6 0.84 at 1 system.  Whole solves (bench.py): 8x6 instead of 4x12 is
    # 1-2.5% faster for configs 1-3 and 8 systems, 10% slower at 16 systems
    c = max(1, min(8, SMS // max(1, 2 * systems_on_gpu)))
    if c >= 8:
        return 8, 6
    if c >= 4:
        return 4, 12
    return (2, ILU0_WARPS) if c >= 2 else (1, ILU0_WARPS)


def _hp_warps(umax):
    """(warps per CTA, units per warp) for a CTA share of umax units, within
    the kernels' register budgets (1 unit per warp: <= 24 warps; 2-8: <= 16)."""
    if umax <= 24:
        return max(1, umax), 1
    if umax <= 128:
        return 16, -(-umax // 16)
    return None


def ilu0_hp_config(nx, ny, nz, split, systems_on_gpu):
    """(CTAs per half, warps per CTA[, link mode]) of the hyperplane ILU0 kernel
    (ntd_ilu0_hp_apply_ex) for this grid, or None when the batch leaves it no
    room (then the skewed progress-word kernel, which needs one SM per half,
    is used: at 64 systems per GPU it is 1.8x faster alone and the whole
    batched solve runs 3-25% faster with it; at 8 systems the hyperplane
    kernel on 16-CTA clusters gives +14%).  One CTA per half when
    it holds the half at one unit per warp (the CTA barrier is cheaper than
    the cluster barrier: 32^3 0.079 ms vs 0.13-0.15 ms on 2-16 CTAs), else
    the largest cluster the batch leaves room for (148 / systems SMs per
    half, at most 16; the halves of a batch do not all sweep at once): the step time grows with the units per CTA (64^3:
    0.27 ms on 16 CTAs, 0.41 ms on one; 128^3 0.83 ms on 16)."""
    units = _lib.load(require_device=False).ntd_ilu0_hp_units(nx, ny, nz, split)
    if units <= 0 or systems_on_gpu > 16:
        return None
    g = (ny + 31) // 32
    nk = units // g
    budget = max(1, SMS // max(1, systems_on_gpu))
    if units <= 24:
        return 1, max(1, units)
    nc = min(16, budget, nk)
    if systems_on_gpu <= 8:
        # up to 8 systems per GPU: CTAs linked through global-memory rings
        # (third element 2 = that link mode) beat a cluster with its barrier
        # per step, and with the halo requested one step ahead fewer, fuller
        # CTAs beat many thin ones (every CTA of the chain adds a step of lag):
        # about 12 units = warps per CTA; at most 74 CTAs per half for a lone
        # system (cooperative launch), 16 otherwise (a cluster launch keeps the
        # CTAs of a half co-resident).  Measured per apply, one system: 64^3
        # 0.22 ms (cluster 0.27), 96^3 0.41 ms on 12-24 CTAs (0.45 on 48,
        # cluster 0.53), 128^3 0.62 ms, 350^3 2.5 ms on 74 CTAs x 16 warps;
        # whole solves at 2 / 4 / 8 systems: 604 / 1082 / 2058 Munk-iter/s
        # against 563 / 1004 / 1921 with clusters (at 16 systems 2857 against
        # 2940, so the cluster mapping below stays there).
        cap = 74 if systems_on_gpu == 1 else 16
        ncg = min(cap, nk, -(-nk // max(1, 12 // g)))
        wu = _hp_warps(-(-nk // ncg) * g)
        if ncg > 1 and wu is not None:
            return ncg, wu[0], 2
    while nc >= 2:
        wu = _hp_warps(-(-nk // nc) * g)
        if wu is not None:
            return nc, wu[0]
        nc -= 1
    return None


def ntd_ctas(systems_on_gpu):
    """CTAs per system for the NTD apply sweep: 2 (one level-3 half per SM,
    a cluster of two) while the GPU's systems fit one CTA per SM, else 1.
    Measured on the config-4 batch: 2 is faster at every size up to 64
    systems per GPU (4327 -> 4747 Munk-iter/s at 64, 1795 -> 1947 at 16)."""
    return 2 if 2 * systems_on_gpu <= SMS else 1


def ilu0_apply(f_dev, split, r_dev, nx, ny, nz, batch, z=None, acc=None, active=None, skew=None, work=None,
               ctas=None, hp="auto"):
    """z = (LU)^-1 r (and/or acc += z).  skew: coefficient records from
    ilu0_skew_build (fast paths); work: scratch for them; hp: (CTAs per half,
    warps per CTA) of the hyperplane kernel, None for the skewed kernel, or
    "auto" (ilu0_hp_config for this batch alone); ctas: (CTAs per system
    half, warps per CTA) of the skewed kernel (default ilu0_ctas).  Every
    path gives bitwise the same result."""
    if z is None and acc is None:
        z = torch.empty_like(r_dev)
    if skew is not None:
        need = _lib.load().ntd_ilu0_skew_work_doubles(nx, ny, nz, batch)
        if work is None or work.numel() < need:
            work = torch.empty(need, dtype=torch.float64, device=_dev())
        if isinstance(hp, str):
            hp = ilu0_hp_config(nx, ny, nz, split, batch)
        if hp is not None:
            _lib.call("ntd_ilu0_hp_apply_ex", _lib.ptr(skew), split, _lib.ptr(r_dev), _lib.ptr(z), _lib.ptr(acc),
                      _lib.ptr(work), nx, ny, nz, batch, _lib.ptr(active), hp[0], hp[1],
                      hp[2] if len(hp) > 2 else 0, _lib.stream())
            return z
        nc, nw = ilu0_ctas(batch) if ctas is None else ctas
        _lib.call("ntd_ilu0_skew_apply_ex", _lib.ptr(skew), split, _lib.ptr(r_dev), _lib.ptr(z), _lib.ptr(acc),
                  _lib.ptr(work), nx, ny, nz, batch, _lib.ptr(active), nc, nw, _lib.stream())
        return z
    if z is None:
        z = torch.empty_like(r_dev)
    _lib.call("ntd_ilu0_apply", _lib.ptr(f_dev), split, _lib.ptr(r_dev), _lib.ptr(z), _lib.ptr(acc), nx, ny,
              nz, batch, _lib.ptr(active), _lib.stream())
    return z


def sym_pack(a_dev, nx, ny, nz, batch):
    """(B,4,N) symmetric packed operator (bands 0,+1,+nx,+nxy) when every
    system's A is bitwise symmetric, else None (the 7-band kernels are used).
    One pass over A plus one small device->host read (setup time)."""
    n = nx * ny * nz
    a4 = torch.empty((batch, 4, n), dtype=torch.float64, device=a_dev.device)
    ok = torch.ones(batch, dtype=torch.int32, device=a_dev.device)
    _lib.call("ntd_sym_pack", _lib.ptr(a_dev), _lib.ptr(a4), _lib.ptr(ok), nx, ny, nz, batch, _lib.stream())
    return a4 if bool(ok.all().item()) else None


def residual(a_dev, r_dev, w_dev, nx, ny, nz, batch, t=None, v=None, z_out=None, active=None, a4=None):
    """t = r - A w, or (v given) z_out = v + w and t = r - A z_out.  With a4
    (sym_pack) the symmetric 4-band kernel is used (bitwise the same)."""
    if t is None:
        t = torch.empty_like(r_dev)
    name, op = ("ntd_residual", a_dev) if a4 is None else ("ntd_residual_sym", a4)
    _lib.call(name, _lib.ptr(op), _lib.ptr(r_dev), _lib.ptr(w_dev), _lib.ptr(v), _lib.ptr(z_out),
              _lib.ptr(t), nx, ny, nz, batch, _lib.ptr(active), _lib.stream())
    return t


class CombinedDevice:
    """Symmetric ILU0 -> NTD -> ILU0 preconditioner on B systems
    (precond_pcg.py:28-65), all buffers preallocated on the device."""

    def __init__(self, a_dev, nx, ny, nz, batch, pre=None, ilu=None, split=None, solve=None, skew=None,
                 a4="auto", ilu_ctas=None, ntd_ctas_=None, ilu_hp="auto"):
        self.a, self.nx, self.ny, self.nz, self.batch = a_dev, nx, ny, nz, batch
        self.ilu_ctas = ilu0_ctas(batch) if ilu_ctas is None else ilu_ctas
        self.split = (nx * ny * nz) // 2 if split is None else split
        self.ilu_hp = ilu0_hp_config(nx, ny, nz, self.split, batch) if isinstance(ilu_hp, str) else ilu_hp
        self.ntd_ctas = ntd_ctas(batch) if ntd_ctas_ is None else ntd_ctas_
        self.a4 = sym_pack(a_dev, nx, ny, nz, batch) if isinstance(a4, str) else a4
        n = nx * ny * nz
        self.n = n
        self.pre = pre
        self.solve = solve if solve is not None else solve_bands(pre, nx, ny, nz, batch)
        self.ilu = ilu
        self.skew = skew if skew is not None else ilu0_skew_build(ilu, self.split, nx, ny, nz, batch)
        self.skew_work = None
        shape = (batch, n)
        self.w = torch.empty(shape, dtype=torch.float64, device=_dev())
        self.t = torch.empty(shape, dtype=torch.float64, device=_dev())
        self.xn = torch.empty(shape, dtype=torch.float64, device=_dev())
        # zero-filled: the slot-layout padding of the NTD input is never written
        self.work = torch.zeros(_lib.load().ntd_apply_work_doubles(nx, ny, nz, batch), dtype=torch.float64,
                                device=_dev())
        # fused residual <-> NTD apply stages on the slot layout when available
        self.fused = self.solve is not None and n < 2 ** 31
        self.ntd_events = None  # list: (start, end) CUDA events around every NTD apply (bench timing)
        # optional stream (e.g. of another priority) for the ILU0 / NTD sweeps;
        # the stencil kernels stay on the caller's stream
        self.sweep_stream = None

    @contextlib.contextmanager
    def _sweep(self):
        s = self.sweep_stream
        if s is None:
            yield
            return
        cur = torch.cuda.current_stream()
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            yield
        cur.wait_stream(s)

    def apply(self, r, z, active=None):
        """z = M^{-1} r:  w = ilu(r); t = r - A w; z = ntd(t) + w;
        t = r - A z; z += ilu(t)   (precond_pcg.py:57-65)."""
        g = (self.nx, self.ny, self.nz, self.batch)
        if self.skew is not None and self.skew_work is None:
            self.skew_work = torch.empty(_lib.load().ntd_ilu0_skew_work_doubles(*g), dtype=torch.float64,
                                         device=_dev())
        with self._sweep():
            ilu0_apply(self.ilu, self.split, r, *g, z=self.w, active=active, skew=self.skew, work=self.skew_work,
                       ctas=self.ilu_ctas, hp=self.ilu_hp)
        op, nb = (self.a, 7) if self.a4 is None else (self.a4, 4)
        if self.fused:
            _lib.call("ntd_residual_to_slot", _lib.ptr(op), nb, _lib.ptr(self.solve), _lib.ptr(r), _lib.ptr(self.w),
                      _lib.ptr(self.work), *g, _lib.ptr(active), _lib.stream())
        else:
            residual(self.a, r, self.w, *g, t=self.t, active=active, a4=self.a4)
        with self._sweep():
            if self.ntd_events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            if self.fused:
                _lib.call("ntd_apply_slot_ex", _lib.ptr(self.solve), _lib.ptr(self.work), *g, _lib.ptr(active),
                          self.ntd_ctas, _lib.stream())
            else:
                ntd_apply(self.pre, self.t, *g, x=self.xn, work=self.work, active=active, solve=self.solve)
            if self.ntd_events is not None:
                ev[1].record()
                self.ntd_events.append(ev)
        if self.fused:
            _lib.call("ntd_residual_from_slot", _lib.ptr(op), nb, _lib.ptr(self.work), _lib.ptr(r),
                      _lib.ptr(self.w), _lib.ptr(z), _lib.ptr(self.t), *g, _lib.ptr(active), _lib.stream())
        else:
            residual(self.a, r, self.w, *g, t=self.t, v=self.xn, z_out=z, active=active, a4=self.a4)
        with self._sweep():
            if self.skew is not None:
                ilu0_apply(self.ilu, self.split, self.t, *g, z=None, acc=z, active=active, skew=self.skew,
                           work=self.skew_work, ctas=self.ilu_ctas, hp=self.ilu_hp)
            else:
                ilu0_apply(self.ilu, self.split, self.t, *g, z=self.xn, acc=z, active=active)
        return z


class NtdDevice:
    """NTD-only preconditioner z = M_NTD^{-1} r on B systems (the reference
    CLI's 'ntd' kind: factor_level3 + ntd_apply, bench_cli.py:113-142)."""

    def __init__(self, pre, nx, ny, nz, batch, ntd_ctas_=None):
        self.pre, self.nx, self.ny, self.nz, self.batch = pre, nx, ny, nz, batch
        self.ntd_ctas = ntd_ctas(batch) if ntd_ctas_ is None else ntd_ctas_
        self.solve = solve_bands(pre, nx, ny, nz, batch)
        self.work = torch.zeros(_lib.load().ntd_apply_work_doubles(nx, ny, nz, batch), dtype=torch.float64,
                                device=_dev())
        self.ntd_events = None
        self.sweep_stream = None

    _sweep = CombinedDevice._sweep

    def apply(self, r, z, active=None):
        with self._sweep():
            if self.ntd_events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            ntd_apply(self.pre, r, self.nx, self.ny, self.nz, self.batch, x=z, work=self.work, active=active,
                      solve=self.solve, ctas=self.ntd_ctas)
            if self.ntd_events is not None:
                ev[1].record()
                self.ntd_events.append(ev)
        return z


class PcgDevice:
    """Device-resident PCG over B systems (precond_pcg.py:68-122).

    Per-system scalars (rz, alpha, beta, relres, convergence) live on the
    device; one small device->host read of the flags per iteration decides
    whether to continue.  Converged systems are masked out of every kernel."""

    def __init__(self, a_dev, nx, ny, nz, batch, max_iters, x=None, a4="auto"):
        lib = _lib.load()
        self.a, self.nx, self.ny, self.nz, self.batch = a_dev, nx, ny, nz, batch
        self.a4 = sym_pack(a_dev, nx, ny, nz, batch) if isinstance(a4, str) else a4
        n = nx * ny * nz
        self.n = n
        self.max_iters = max_iters
        dev = _dev()
        shape = (batch, n)
        self.x = torch.empty(shape, dtype=torch.float64, device=dev) if x is None else x
        self.r = torch.empty(shape, dtype=torch.float64, device=dev)
        self.z = torch.empty(shape, dtype=torch.float64, device=dev)
        self.p = torch.empty(shape, dtype=torch.float64, device=dev)
        self.ap = torch.empty(shape, dtype=torch.float64, device=dev)
        self.state = torch.zeros((batch, _lib.NTD_ST["N"]), dtype=torch.float64, device=dev)
        self.flags = torch.zeros((batch, _lib.NTD_FL["N"]), dtype=torch.int32, device=dev)
        self.active = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.history = torch.zeros((batch, max(1, max_iters)), dtype=torch.float64, device=dev)
        self.work = torch.empty(lib.ntd_dot_work_doubles(batch), dtype=torch.float64, device=dev)
        self.host_flags = torch.zeros((batch, _lib.NTD_FL["N"]), dtype=torch.int32).pin_memory()
        self.host_state = torch.zeros((batch, _lib.NTD_ST["N"]), dtype=torch.float64).pin_memory()

    def _g(self):
        return self.nx, self.ny, self.nz, self.batch

    def init(self, b, tol):
        self.b = b
        _lib.call("ntd_pcg_init", _lib.ptr(b), _lib.ptr(self.x), _lib.ptr(self.r), _lib.ptr(self.state),
                  _lib.ptr(self.flags), _lib.ptr(self.active), float(tol), self.n, self.batch,
                  _lib.ptr(self.work), _lib.stream())

    def start(self, z):
        _lib.call("ntd_pcg_start", _lib.ptr(self.r), _lib.ptr(z), _lib.ptr(self.p), _lib.ptr(self.state),
                  _lib.ptr(self.active), self.n, self.batch, _lib.ptr(self.work), _lib.stream())

    def step_update(self):
        """ap = A p; alpha; x, r update; true residual; convergence flags."""
        sym = self.a4 is not None
        op = self.a4 if sym else self.a
        _lib.call("ntd_pcg_spmv_alpha_sym" if sym else "ntd_pcg_spmv_alpha", _lib.ptr(op), _lib.ptr(self.p),
                  _lib.ptr(self.ap),
                  _lib.ptr(self.state), _lib.ptr(self.flags), _lib.ptr(self.active), *self._g(),
                  _lib.ptr(self.work), _lib.stream())
        _lib.call("ntd_pcg_update_residual_sym" if sym else "ntd_pcg_update_residual", _lib.ptr(op),
                  _lib.ptr(self.b), _lib.ptr(self.x),
                  _lib.ptr(self.r), _lib.ptr(self.p), _lib.ptr(self.ap), _lib.ptr(self.state),
                  _lib.ptr(self.flags), _lib.ptr(self.active), _lib.ptr(self.history), self.max_iters,
                  *self._g(), _lib.ptr(self.work), _lib.stream())

    def direction(self, z):
        _lib.call("ntd_pcg_direction", _lib.ptr(self.r), _lib.ptr(z), _lib.ptr(self.p), _lib.ptr(self.state),
                  _lib.ptr(self.active), self.n, self.batch, _lib.ptr(self.work), _lib.stream())

    def read_flags(self):
        """Synchronising D2H copy of flags and scalars (pinned)."""
        self.host_flags.copy_(self.flags, non_blocking=True)
        self.host_state.copy_(self.state, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.host_flags, self.host_state

    def solve(self, b, tol, precond_apply=None, callback=None):
        """Run PCG to completion.  precond_apply(r, z, active) -> z (device),
        or None for plain CG.  callback(it, x_dev, relres_host_array)."""
        self.init(b, tol)
        fl, _ = self.read_flags()
        if not bool(fl[:, _lib.NTD_FL["ACTIVE"]].any()):
            return 0
        z = self.r if precond_apply is None else precond_apply(self.r, self.z, self.active)
        self.start(z)
        it = 0
        for it in range(1, self.max_iters + 1):
            self.step_update()
            fl, st = self.read_flags()
            if callback is not None:
                callback(it, fl, st)
            if not bool(fl[:, _lib.NTD_FL["ACTIVE"]].any()):
                break
            if precond_apply is not None:
                z = precond_apply(self.r, self.z, self.active)
            self.direction(z)
        return it

    # ------------------------------------------------------------ graphed loop
    def _iteration(self, precond_apply):
        """One PCG iteration: update (ap, alpha, x, r, true residual, flags),
        preconditioner, new direction -- every kernel masked by `active`."""
        self.step_update()
        z = self.r if precond_apply is None else precond_apply(self.r, self.z, self.active)
        self.direction(z)

    def solve_graph(self, b, tol, precond_apply=None, graph_key=None):
        """PCG to completion with one iteration replayed as a CUDA graph.

        The host neither launches the ~15 kernels of an iteration nor waits
        for each one: it replays the captured iteration and reads the
        convergence flags of iteration i-1 while iteration i runs (converged
        systems are masked on the device, so the one extra replay does no
        work).  Captured once per (PcgDevice, graph_key); precond_apply must
        only enqueue device work on the current stream.  Returns the number
        of host-side iterations (the per-system count is in the flags)."""
        if getattr(self, "_b_buf", None) is None:
            self._b_buf = torch.empty((self.batch, self.n), dtype=torch.float64, device=self.r.device)
            self._flag_slots = [torch.zeros((self.batch, _lib.NTD_FL["N"]), dtype=torch.int32).pin_memory()
                                for _ in range(2)]
            self._flag_events = [torch.cuda.Event() for _ in range(2)]
        self._b_buf.copy_(b.reshape(self.batch, self.n))
        self.init(self._b_buf, tol)
        z = self.r if precond_apply is None else precond_apply(self.r, self.z, self.active)
        self.start(z)
        if getattr(self, "_graph", None) is None or self._graph_key != graph_key:
            # one eager iteration first: it allocates every lazily sized
            # buffer, so the capture below allocates nothing
            self._iteration(precond_apply)
            done = 1
            self._flag_slots[1].copy_(self.flags, non_blocking=True)
            self._flag_events[1].record()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    self._iteration(precond_apply)
            torch.cuda.current_stream().wait_stream(side)
            self._graph, self._graph_key = g, graph_key
        else:
            done = 0
        act = _lib.NTD_FL["ACTIVE"]
        it = done
        while it < self.max_iters:
            self._graph.replay()
            it += 1
            slot = it & 1
            self._flag_slots[slot].copy_(self.flags, non_blocking=True)
            self._flag_events[slot].record()
            if it >= 2:
                prev = 1 - slot
                self._flag_events[prev].synchronize()
                if not bool(self._flag_slots[prev][:, act].any()):
                    break
        return it
