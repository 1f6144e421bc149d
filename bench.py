"""NTD-PCG benchmark (driver contract: one JSON line from rank 0).

Workload: BASELINE.json config 4 -- a batch of 64 independent 96^3 diffusion
systems (seeded cellwise log-normal kappa on 4^3 blocks, Dirichlet faces,
b = A x_true), ntd+ilu0 PCG to relative residual 1e-8 from x0 = 0.  One
"step" = one full batched PCG solve (all systems to convergence).  The 64
systems are sharded across ranks (rank r solves systems [64r/N, 64(r+1)/N)),
each rank builds its systems from their seeds; no data-path collective, one
NCCL all_gather of per-system statistics at the end.

Metric: PCG Munknowns/s = sum over systems of N * iterations / solve time
(the reference's "M unknown-iter/s").  `value` is device-timed
with inputs resident; `e2e` adds the host->device copy of b and the
device->host copy of x every step (public BatchSolver API).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ntd|reference]

`--gpus N` with N > 1 outside torchrun re-launches itself under
`torch.distributed.run` with N ranks (one per GPU, NCCL); under torchrun the
world size must equal N.  At N = 1 the line also carries `configs`: the
single-system BASELINE configs 1, 2, 3 and 5 (PCG, NTD and combined apply
rates, % of HBM, iterations against the reference's, apply error against the
CPU oracle, and a CPU-port baseline for configs 1-3).
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

# stream groups need hardware queues (before any CUDA context; see batch.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# reference iteration counts for config 4, systems 0..63 (reference package
# run on the same seeded inputs)
CFG4_REF_ITERS = [21, 21, 24, 21, 22, 22, 20, 20, 20, 24, 22, 23, 20, 21, 19, 21, 23, 20, 23, 20, 19, 23, 20, 25,
                  22, 22, 22, 23, 21, 23, 21, 20, 21, 25, 21, 24, 21, 22, 21, 21, 19, 20, 23, 20, 25, 21, 25, 21,
                  20, 22, 23, 21, 20, 21, 21, 21, 20, 21, 21, 21, 23, 20, 23, 22]

# Costs measured on this pool's B200s (tools/micro_lat2.cu, micro_tput2.cu,
# micro_line_ts.cu; profiles/r02g_micro_*.txt): a dependent DFMA/DADD/DMUL 8.2
# cycles, a dependent 64-bit shuffle 24.3 (two SHFL.32); one warp issues a
# SHFL.32 every 4.5 cycles, an LDS.64 every 2.25 and an STS.64 every ~6.4.  A
# line step of the NTD apply (ntd_apply_ts.cuh) is one warp: 24 shuffles,
# (5.5 K + 8) 8-byte shared loads per lane on average over the lower- and
# upper-sweep steps, 1.5 K stores; the two-sided line solve alone (its
# dependent chain: 5 shuffle rounds + 2 K + 8 fp64 operations) measures
# 214 + 16 K cycles.  An apply is (nz + 1)(ny + 1) dependent line steps, so
# its roofline is the longer of the two per step.
SHFL32_ISSUE = 4.5
LDS64_ISSUE = 2.25
ST64_ISSUE = 6.4


def ntd_latency_roofline(nx, ny, nz, apply_s, sm_mhz):
    K = next(k for k in (1, 2, 3, 4, 5, 6, 8, 11, 12, 16) if 32 * k >= nx)
    mio = 24 * SHFL32_ISSUE + (5.5 * K + 8) * LDS64_ISSUE + 1.5 * K * ST64_ISSUE
    chain = 214.0 + 16.0 * K
    bound = max(mio, chain)
    steps = (nz + 1) * (ny + 1)
    measured = apply_s * sm_mhz * 1e6 / steps
    return {"bound": "latency: the dependent chain of a line step (5 shuffle rounds + fp64 chain of the two-sided "
                     "line solve), or one warp's shuffle / shared-memory issue per step if longer",
            "line_steps_per_apply": steps, "mio_cycles_per_step": round(mio, 1),
            "chain_cycles_per_step": round(chain, 1), "measured_cycles_per_step": round(measured, 1),
            "sm_mhz": sm_mhz, "frac": round(bound / measured, 3),
            "source": "tools/micro_tput2.cu, micro_lat2.cu, micro_line_ts.cu; profiles/r02g_micro_*.txt"}


METRIC = "pcg_munknowns_per_s"
UNIT = "Munknown-iterations/s"
NTD_APPLY_BYTES_PER_UNKNOWN = 48  # canonical algorithmic bytes


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ntd", choices=["ntd", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--systems", type=int, default=None, help="batch size (config 4: 64)")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--precond", default="ntd+ilu0", choices=["ntd+ilu0", "ntd"],
                    help="preconditioner (SURVEY.md 8(d) also reports ntd-only for configs 1 and 3)")
    ap.add_argument("--cpu-systems", type=int, default=None, help="CPU baseline sample size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the single-system configs 1, 2, 3, 5")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shard(total, world, rank):
    from paper_1909_09771_b200.dist import shard as _shard
    return _shard(total, world, rank)


def system_inputs(cfg, s):
    from paper_1909_09771_b200 import problems
    data, x_true, grid = problems.baseline_config(cfg, s)
    return data, x_true, grid


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU leg
def cpu_solve_systems(cfg, systems, threads, tol, kind="ntd+ilu0"):
    """Oracle (C restatement of the reference) PCG on `systems`, `threads`
    systems at a time.  Returns (unknown-iterations, solve seconds wall,
    setup seconds wall, iterations list)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    def setup(s):
        data, x_true, (nx, ny, nz) = system_inputs(cfg, s)
        b = oracle.spmv(data, x_true, nx, ny, nz)
        pre = oracle.factor_level3(data, nx, ny, nz)
        ilu = oracle.build_block_ilu0(data, nx, ny, nz) if kind == "ntd+ilu0" else None
        return data, b, (nx, ny, nz), pre, ilu

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        built = list(ex.map(setup, systems))
    t_setup = time.perf_counter() - t0

    def solve(item):
        data, b, (nx, ny, nz), pre, ilu = item
        _, it, conv, _ = oracle.pcg(data, b, nx, ny, nz, kind=kind, tol=tol, pre=pre, ilu=ilu)
        return nx * ny * nz * it, it

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(solve, built))
    t_solve = time.perf_counter() - t0
    return sum(r[0] for r in res), t_solve, t_setup, [r[1] for r in res]


def host_cores():
    """(cores of the host, cores this process may run on)."""
    total = os.cpu_count() or 1
    try:
        usable = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        usable = total
    return total, usable


def cpu_threads():
    """P = min(64, cores) systems at once, one
    per thread (the reference has no batch API: one solve per core)."""
    return max(1, min(64, host_cores()[1]))


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    sample = args.cpu_systems or cpu_threads()
    cfg = args.config
    n_sys = args.systems or (64 if cfg == 4 else 1)
    systems = list(range(min(sample, n_sys)))
    for _ in range(args.warmup):
        cpu_solve_systems(cfg, systems[:1], 1, args.tol, args.precond)
    vals, ts = [], []
    for _ in range(args.steps):
        work, t, _, iters = cpu_solve_systems(cfg, systems, sample, args.tol, args.precond)
        vals.append(work / t / 1e6)
        ts.append(t)
    v = float(np.median(vals))
    total, usable = host_cores()
    desc = (f"{len(systems)} of the {n_sys} config-{cfg} systems per step, each a full {args.precond} PCG solve "
            f"to {args.tol:g} by the C oracle (restatement of the reference kernels), one system per thread, "
            f"{len(systems)} threads on a host with {total} cores ({usable} usable)")
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(ts)), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": f"cfg{cfg}", "systems": n_sys, "grid": "96^3" if cfg == 4 else None,
                      "precond": args.precond, "tol": args.tol, "parallelism": "cpu-threads"},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": len(systems), "threads": len(systems),
                            "host_cores": total, "usable_cores": usable, "kind": "port", "sample": desc},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- GPU leg
def run_ntd(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    # NTD_BENCH_ONE_GPU=1 (validation only): every rank on cuda:0 with gloo
    # statistics exchange, to exercise the multi-rank path on a 1-GPU box (the
    # ranks share nothing on the data path, so none waits on another)
    one_gpu = os.environ.get("NTD_BENCH_ONE_GPU") == "1"
    gpu = 0 if one_gpu else local
    torch.cuda.set_device(gpu)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1909_09771_b200 import _lib
    from paper_1909_09771_b200 import device as D
    from paper_1909_09771_b200.batch import BatchSolver

    cfg = args.config
    n_total = args.systems or (64 if cfg == 4 else 1)
    mine = shard(n_total, world, rank)
    # seeded kappa fields on the host, assembled on the
    # device (ntd_assemble, bitwise the reference's _assemble_kernel)
    from paper_1909_09771_b200 import problems
    nx, ny, nz = problems.CONFIGS[cfg]["grid"]
    n = nx * ny * nz
    B = len(mine)
    kaps, xts, bc = [], [], None
    for s in mine:
        kap, bc, rng = problems.baseline_kappa(cfg, s)
        kaps.append(kap)
        xts.append(rng.uniform(-1.0, 1.0, n))
    a_dev = D.assemble(torch.from_numpy(np.stack(kaps)).cuda(), nx, ny, nz, bc)
    xt_dev = torch.from_numpy(np.stack(xts)).cuda()
    del kaps, xts
    b_dev = torch.empty_like(xt_dev)
    _lib.call("ntd_spmv", _lib.ptr(a_dev), _lib.ptr(xt_dev), _lib.ptr(b_dev), nx, ny, nz, B, None, _lib.stream())
    b_host = b_dev.cpu().pin_memory()
    x_host = torch.empty_like(b_host).pin_memory()

    solver = BatchSolver(a_dev, nx, ny, nz, args.precond, max_iters=200 if args.precond == "ntd+ilu0" else 400)
    solver.setup()
    setup_s = solver.setup_seconds

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (the same pipelined call the timed region makes)
    solver.reserve(max(args.steps, args.warmup))
    # (at least one solve: it also yields the iteration stats checked below)
    nw = max(1, args.warmup)
    res = solver.solve_many([b_dev] * nw, args.tol, x_outs=[solver.x] * nw)[-1]
    solver.solve_host_many([b_host], [x_host], args.tol)
    barrier()
    # ---- device-timed steps (inputs resident)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    _lib.reset_launch_count()
    for grp in solver.groups:
        grp.precond.ntd_events = []
    with ClockSampler(gpu) as clk:
        barrier()
        ev[0].record()
        work_local = 0
        # K solves of the batch, pipelined per stream group (solve_many:
        # a group starts the next solve as soon as its own systems stop)
        for res in solver.solve_many([b_dev] * args.steps, args.tol, x_outs=[solver.x] * args.steps):
            work_local += n * sum(res.iterations)
        ev[1].record()
        barrier()
    launches = _lib.launch_count()
    for grp in solver.groups:
        evs_keep = grp.precond.ntd_events
        grp.precond.ntd_events = None
        grp.precond.ntd_events_timed = evs_keep
    t_dev = ev[0].elapsed_time(ev[1]) / 1e3
    # ---- e2e through the public API with host buffers: every step uploads
    # its b from pinned host memory and downloads its x (BatchSolver.solve_host_many:
    # each stream group moves its own slice on its own stream, so the copies
    # overlap the other groups' sweeps), all inside the timed region
    ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    barrier()
    ev2[0].record()
    work_e2e = 0
    for r2 in solver.solve_host_many([b_host] * args.steps, [x_host] * args.steps, args.tol):
        work_e2e += n * sum(r2.iterations)
    ev2[1].record()
    barrier()
    t_e2e = ev2[0].elapsed_time(ev2[1]) / 1e3
    # ---- dominant kernel: the NTD apply launches of the timed region
    # (CUDA events recorded on each group's stream around every apply)
    evs = [e for grp in solver.groups for e in grp.precond.ntd_events_timed]
    torch.cuda.synchronize()
    t_apply_sum = float(np.sum([a.elapsed_time(b) for a, b in evs])) / 1e3
    t_apply = t_apply_sum / max(1, len(evs))
    # algorithmic bytes of the timed applies: each system is preconditioned
    # once per PCG iteration it takes (masked systems do no work)
    apply_gbs = NTD_APPLY_BYTES_PER_UNKNOWN * work_local / t_apply_sum / 1e9
    g0 = solver.groups[0]
    Bg = g0.hi - g0.lo  # systems per NTD launch
    # standalone context timings for one group's launch (ILU0 apply, spmv)
    P = g0.precond
    v = torch.rand((Bg, n), dtype=torch.float64, device="cuda")
    xa = torch.empty_like(v)
    R = 5
    has_ilu = args.precond == "ntd+ilu0"
    for _ in range(2 if has_ilu else 0):
        D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, Bg, z=xa, skew=P.skew, work=P.skew_work, ctas=P.ilu_ctas,
                     hp=P.ilu_hp)
    e4 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e4[0].record()
    for _ in range(R if has_ilu else 0):
        D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, Bg, z=xa, skew=P.skew, work=P.skew_work, ctas=P.ilu_ctas,
                     hp=P.ilu_hp)
    e4[1].record()
    e5 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e5[0].record()
    for _ in range(R):
        _lib.call("ntd_spmv", _lib.ptr(g0.a), _lib.ptr(v), _lib.ptr(xa), nx, ny, nz, Bg, None, _lib.stream())
    e5[1].record()
    torch.cuda.synchronize()
    t_ilu = e4[0].elapsed_time(e4[1]) / 1e3 / R
    t_spmv = e5[0].elapsed_time(e5[1]) / 1e3 / R
    stencil = stencil_roofline(solver.a, B, n, nx, ny, nz)

    # ---- reductions over ranks (NCCL: max of timings, sum of work, one all_gather of stats)
    from paper_1909_09771_b200 import dist as pdist
    dev = torch.device("cpu") if one_gpu else torch.device("cuda", local)
    times = pdist.reduce_max([t_dev, t_e2e, t_apply, t_ilu, t_spmv, setup_s, -apply_gbs], dev)
    work = pdist.reduce_sum([work_local, work_e2e, launches], dev)
    stats = pdist.gather_stats([[s, it, int(cv), rr] for s, it, cv, rr in
                                zip(mine, res.iterations, res.converged, res.final_relres)], n_total, dev)
    stats = stats.cpu().numpy()
    if rank == 0:
        t_dev, t_e2e, t_apply, t_ilu, t_spmv, setup_s, apply_gbs = times
        apply_gbs = -apply_gbs  # min over ranks
        value = work[0] / t_dev / 1e6
        e2e = work[1] / t_e2e / 1e6
        iters = [int(v) for v in stats[:, 1]]
        sys_ids = [int(v) for v in stats[:, 0]]
        ref_match = None
        if cfg == 4 and args.precond == "ntd+ilu0":
            ref_match = sum(abs(it - CFG4_REF_ITERS[s]) <= 1 for s, it in zip(sys_ids, iters))
        achieved = apply_gbs
        peak = _measured_peak()
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config recipe, SURVEY.md 8(d))",
            "config": {"workload": f"cfg{cfg}", "systems": n_total, "grid": f"{nx}x{ny}x{nz}",
                       "precond": args.precond, "tol": args.tol, "parallelism": f"batch-shard x{world}",
                       "stream_groups": len(solver.groups), "systems_per_ntd_launch": Bg,
                       "l2": "inputs larger than L2 (each batch vector %.0f MB)" % (8 * n * B / 1e6)},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n * B * world,
                    "d2h_bytes_per_step": 8 * n * B * world},
            "roofline": {"kernel": "NTD apply sweep ts::k_apply (ntd_apply_slot), timed-region launches, rank 0",
                         "bound": "hbm",
                         "achieved": achieved, "peak": peak[0], "unit": "GB/s", "frac": achieved / peak[0],
                         "peak_source": peak[1], "traffic": _traffic(cfg, Bg),
                         "traffic_unit": "bytes per launch (ncu dram read+write)",
                         "bytes_per_unknown": NTD_APPLY_BYTES_PER_UNKNOWN, "apply_ms": 1e3 * t_apply,
                         "apply_munknowns_per_s": n * Bg / t_apply / 1e6,
                         "concurrent_launches": len(solver.groups),
                         "aggregate_gbs": NTD_APPLY_BYTES_PER_UNKNOWN * work[0] / t_dev / 1e9,
                         "launches_timed": len(evs)},
            "latency_roofline": ntd_latency_roofline(nx, ny, nz, t_apply, clk.summary()["sm_mhz"] or 1965.0),
            "kernels_ms": {"ntd_apply": 1e3 * t_apply, "ilu0_apply": 1e3 * t_ilu if has_ilu else None,
                           "spmv": 1e3 * t_spmv},
            "stencil_roofline": stencil,
            "step_hbm": _step_hbm(cfg, Bg, n, work[0] / t_dev, stencil, peak[0]) if has_ilu else None,
            "setup_seconds": setup_s,
            "iterations": {"min": min(iters), "max": max(iters), "mean": float(np.mean(iters)),
                           "within_1_of_reference": ref_match, "systems": len(iters)},
            "max_final_relres": float(stats[:, 3].max()),
            "all_converged": bool(stats[:, 2].all()),
            "gpu_launches": int(work[2]),
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        if world == 1 and cfg == 4 and not args.no_configs:
            out["configs"] = single_configs(peak[0], cpu=not args.no_cpu_baseline,
                                            sm_mhz=out["clocks"]["sm_mhz"] or 1965.0)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def stencil_roofline(a_dev, B, n, nx, ny, nz):
    """The bandwidth-bound stencil / CG kernels on B systems (a_dev (B,7,N))
    in one launch each (CUDA events, median of 5): algorithmic bytes per
    unknown (SURVEY.md 8(d), A as its 4 symmetric bands) / time, against
    the HBM peak.  north_star asks >= 70% for these."""
    import torch
    from paper_1909_09771_b200 import _lib
    from paper_1909_09771_b200 import device as D

    class _S:
        a = a_dev
    solver = _S()
    a4 = D.sym_pack(solver.a, nx, ny, nz, B)
    if a4 is None:
        return None
    gen = torch.Generator(device="cuda").manual_seed(11)
    r, w, v = (torch.rand((B, n), dtype=torch.float64, device="cuda", generator=gen) for _ in range(3))
    t, z = torch.empty_like(r), torch.empty_like(r)
    cg = D.PcgDevice(solver.a, nx, ny, nz, B, 2, a4=a4)
    cg.init(r, 1e-30)
    cg.p.copy_(w)
    cg.state[:, _lib.NTD_ST["RZ"]] = 1.0
    peak = _measured_peak()[0]

    def timed(fn):
        fn()
        ts = []
        for _ in range(5):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            fn()
            e[1].record()
            torch.cuda.synchronize()
            ts.append(e[0].elapsed_time(e[1]) / 1e3)
        return float(np.median(ts))

    cases = {
        # t = r - A w: A (32) + r, w (16) + t (8)
        "residual": (56, lambda: D.residual(solver.a, r, w, nx, ny, nz, B, t=t, a4=a4)),
        # z = v + w, t = r - A z: A (32) + r, v, w (24) + z, t (16)
        "residual_sum": (72, lambda: D.residual(solver.a, r, w, nx, ny, nz, B, t=t, v=v, z_out=z, a4=a4)),
        # ap = A p, p.ap: A (32) + p (8) + ap (8)
        "spmv_dot": (48, lambda: _lib.call("ntd_pcg_spmv_alpha_sym", _lib.ptr(a4), _lib.ptr(cg.p), _lib.ptr(cg.ap),
                                           _lib.ptr(cg.state), _lib.ptr(cg.flags), _lib.ptr(cg.active), nx, ny, nz,
                                           B, _lib.ptr(cg.work), _lib.stream())),
        # x, r axpys (x, r, p, ap read, x, r written: 48) + true residual (A 32 + b, x: 48)
        "update_true_residual": (96, lambda: _lib.call(
            "ntd_pcg_update_residual_sym", _lib.ptr(a4), _lib.ptr(r), _lib.ptr(cg.x), _lib.ptr(cg.r), _lib.ptr(cg.p),
            _lib.ptr(cg.ap), _lib.ptr(cg.state), _lib.ptr(cg.flags), _lib.ptr(cg.active), _lib.ptr(cg.history), 2,
            nx, ny, nz, B, _lib.ptr(cg.work), _lib.stream())),
        # r.z (16) + p = beta p + z (p, z read, p written: 24)
        "direction": (40, lambda: _lib.call("ntd_pcg_direction", _lib.ptr(cg.r), _lib.ptr(w), _lib.ptr(cg.p),
                                            _lib.ptr(cg.state), _lib.ptr(cg.active), n, B, _lib.ptr(cg.work),
                                            _lib.stream())),
    }
    out = {}
    for name, (bpu, fn) in cases.items():
        dt = timed(fn)
        gbs = bpu * n * B / dt / 1e9
        out[name] = {"bytes_per_unknown": bpu, "ms": 1e3 * dt, "achieved_gbs": gbs, "frac": gbs / peak}
    return out


# reference iteration counts of the single-system configs (reference package
# on the seeded inputs)
SINGLE_REF_ITERS = {1: 9, 2: 26, 3: 10, 5: 71}
COMBINED_APPLY_BYTES_PER_UNKNOWN = 304
PCG_ITER_BYTES = 488


def single_configs(peak, cfgs=(1, 2, 3, 5), cpu=True, sm_mhz=1965.0):
    """BASELINE configs 1, 2, 3, 5 (one system each) through the public API on
    device-resident inputs: PCG (ntd+ilu0, tol 1e-8) solve rate and
    iterations against the reference's, the NTD and combined applies alone
    (CUDA events, median), each against the HBM roofline at the canonical
    bytes (48 / 304 / 488 B per unknown), apply errors
    against the CPU oracle (the C restatement of the reference) on a seeded
    vector, and for configs 1-3 the oracle's own single-thread PCG solve as
    the CPU baseline."""
    import torch
    import paper_1909_09771_b200 as ntd
    from paper_1909_09771_b200 import _lib, problems
    from paper_1909_09771_b200 import device as D
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    out = {}
    for cfg in cfgs:
        nx, ny, nz = problems.CONFIGS[cfg]["grid"]
        n = nx * ny * nz
        kap, bc, rng = problems.baseline_kappa(cfg, 0)
        x_true = rng.uniform(-1.0, 1.0, n)
        a_dev = D.assemble(torch.from_numpy(kap).cuda(), nx, ny, nz, bc)[0]
        a = ntd.BandedMatrix(nx, ny, nz, a_dev)
        b = ntd.spmv(a, torch.from_numpy(x_true).cuda())
        del kap
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cp = ntd.CombinedPrecond(a)
        setup_s = time.perf_counter() - t0
        reps = {1: 5, 2: 3, 3: 3, 5: 1}[cfg]
        solves = []
        for r in range(reps + 1):
            x, st = ntd.pcg(a, b, cp, tol=1e-8)
            if r:
                solves.append(st.solve_seconds)
        solve_s = float(np.median(solves))
        rate = n * st.iterations / solve_s / 1e6
        # applies alone: CUDA events around R calls on the device-level objects
        dv = cp._dev
        v = torch.from_numpy(np.random.default_rng(100 + cfg).uniform(-1.0, 1.0, n)).cuda().reshape(1, n)
        z = torch.empty_like(v)
        pre = cp.ntd

        def timed(fn, R):
            fn()
            ts = []
            for _ in range(R):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                e[0].record()
                fn()
                e[1].record()
                torch.cuda.synchronize()
                ts.append(e[0].elapsed_time(e[1]) / 1e3)
            return float(np.median(ts))
        R = {1: 20, 2: 10, 3: 5, 5: 3}[cfg]
        t_ntd = timed(lambda: D.ntd_apply(pre.bands.reshape(1, 7, n), v, nx, ny, nz, 1, x=z,
                                          work=cp.workspace.work(nx, ny, nz), solve=pre.solve), R)
        t_comb = timed(lambda: dv.apply(v, z), R)
        t_ilu = timed(lambda: D.ilu0_apply(dv.ilu, dv.split, v, nx, ny, nz, 1, z=z, skew=dv.skew,
                                           work=dv.skew_work, ctas=dv.ilu_ctas, hp=dv.ilu_hp), R)
        # parity against the oracle on the same vector (the GPU factor is
        # bitwise the reference's: tests/test_gpu_api.py)
        vh = v[0].cpu().numpy()
        pre_h = pre.host()
        x_gpu = ntd.ntd_apply(pre, vh)
        x_orc = oracle.ntd_apply(pre_h, vh, nx, ny, nz, nthreads=2)
        err = float(np.abs(x_gpu - x_orc).max() / np.abs(x_orc).max())
        rec = {"workload": f"cfg{cfg}", "grid": f"{nx}x{ny}x{nz}", "unknowns": n,
               "pcg": {"iterations": st.iterations, "reference_iterations": SINGLE_REF_ITERS[cfg],
                       "converged": st.converged, "final_relres": st.final_relres, "setup_ms": 1e3 * setup_s,
                       "solve_ms": 1e3 * solve_s, "value": rate, "unit": UNIT,
                       "hbm_frac_canonical": PCG_ITER_BYTES * rate * 1e6 / 1e9 / peak},
               "ntd_apply": {"ms": 1e3 * t_ntd, "munknowns_per_s": n / t_ntd / 1e6,
                             "hbm_frac": NTD_APPLY_BYTES_PER_UNKNOWN * n / t_ntd / 1e9 / peak,
                             "latency_roofline": ntd_latency_roofline(nx, ny, nz, t_ntd, sm_mhz)},
               "combined_apply": {"ms": 1e3 * t_comb, "munknowns_per_s": n / t_comb / 1e6,
                                  "hbm_frac": COMBINED_APPLY_BYTES_PER_UNKNOWN * n / t_comb / 1e9 / peak},
               "ilu0_apply_ms": 1e3 * t_ilu,
               "ntd_apply_rel_err_vs_oracle": err}
        if cfg in (3, 5):  # the stencil / CG kernels on one system (north_star: >= 70% of HBM)
            rec["stencil_roofline"] = {k: {"frac": round(v["frac"], 3), "ms": round(v["ms"], 3)}
                                       for k, v in stencil_roofline(a_dev.reshape(1, 7, n), 1, n, nx, ny, nz).items()}
        if cfg != 5:
            data = a.host_data()
            fo, split = oracle.build_block_ilu0(data, nx, ny, nz)
            zc = oracle.combined_apply(data, pre_h, fo, split, vh, nx, ny, nz)
            zg = ntd.combined_apply(cp, vh)
            rec["combined_apply_rel_err_vs_oracle"] = float(np.abs(zg - zc).max() / np.abs(zc).max())
            if cpu:
                bh = b.cpu().numpy()
                t0 = time.perf_counter()
                _, it_o, conv_o, _ = oracle.pcg(data, bh, nx, ny, nz, tol=1e-8, pre=pre_h, ilu=(fo, split))
                t_o = time.perf_counter() - t0
                rec["cpu_baseline"] = {"value": n * it_o / t_o / 1e6, "unit": UNIT, "cores": 1, "threads": 1,
                                       "kind": "port", "iterations": it_o,
                                       "sample": f"one full ntd+ilu0 PCG solve of config {cfg} by the C oracle "
                                                 f"(single thread, factorisations excluded), {t_o:.2f} s"}
                rec["gpu_over_cpu"] = rate / rec["cpu_baseline"]["value"]
        out[f"cfg{cfg}"] = rec
        del cp, a, a_dev, b, x, pre_h
        torch.cuda.empty_cache()
    return out


def _traffic(cfg, systems):
    """ncu-measured DRAM bytes per launch of the dominant kernel (profiles/)."""
    try:
        with open(os.path.join(REPO, "profiles", "roofline_traffic.json")) as fh:
            rec = json.load(fh).get(f"cfg{cfg}-{systems}")
        return None if rec is None else float(rec["bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


PCG_ITER_BYTES_PER_UNKNOWN = 488


def _step_hbm(cfg, systems, n, unknown_iters_per_s, stencil, peak):
    """The whole PCG iteration against HBM: DRAM bytes per unknown-iteration
    (NTD and 2 ILU0 sweeps measured by ncu, profiles/roofline_traffic.json;
    stencil/CG kernels at their algorithmic bytes) x the measured rate."""
    try:
        with open(os.path.join(REPO, "profiles", "roofline_traffic.json")) as fh:
            rec = json.load(fh)
        ntd = rec[f"cfg{cfg}-{systems}"]["bytes_per_launch"] / (systems * n)
        ilu = rec[f"ilu0-cfg{cfg}-{systems}"]["bytes_per_launch"] / (systems * n)
    except (OSError, ValueError, KeyError):
        return None
    sten = sum(v["bytes_per_unknown"] for v in stencil.values()) if stencil else 0
    bpu = ntd + 2 * ilu + sten
    gbs = bpu * unknown_iters_per_s / 1e9
    # canonical algorithmic bytes of one ntd+ilu0 PCG
    # iteration (each distinct input read once, A as 4 symmetric bands)
    canon = PCG_ITER_BYTES_PER_UNKNOWN * unknown_iters_per_s / 1e9
    return {"bytes_per_unknown_iter": round(bpu, 1), "ntd": round(ntd, 1), "ilu0_x2": round(2 * ilu, 1),
            "stencil_cg": sten, "achieved_gbs": gbs, "frac": gbs / peak,
            "canonical_bytes_per_unknown_iter": PCG_ITER_BYTES_PER_UNKNOWN, "canonical_gbs": canon,
            "canonical_frac": canon / peak, "canonical_frac_of_8tbs": canon / 8000.0}


def _measured_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_baseline(args):
    sample = args.cpu_systems or cpu_threads()
    systems = list(range(sample))
    work, t, _, iters = cpu_solve_systems(args.config, systems, sample, args.tol, args.precond)
    total, usable = host_cores()
    return {"value": work / t / 1e6, "unit": UNIT, "cores": sample, "threads": sample, "host_cores": total,
            "usable_cores": usable, "kind": "port",
            "sample": f"{sample} config-{args.config} systems, full {args.precond} PCG solve each (C oracle), "
                      f"one system per host thread ({sample} threads, host {total} cores, {usable} usable); "
                      f"solve wall {t:.1f} s, iterations {iters}"}


def relaunch(args):
    """`--gpus N` outside torchrun: run this script as N ranks under
    torch.distributed.run (one process per GPU, NCCL on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator log shows every rank
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        sys.exit(relaunch(args))
    if world > 1 and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ntd(args)


if __name__ == "__main__":
    main()
