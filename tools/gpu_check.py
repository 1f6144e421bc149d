"""Staged GPU sanity check (debug aid): runs each kernel family on growing
inputs and prints parity numbers, so a crash or hang is localised."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import torch
import oracle
import paper_1909_09771_b200 as ntd
from paper_1909_09771_b200 import problems

def rel(a, b):
    d = np.abs(b).max()
    return float(np.abs(a - b).max() / (d if d else 1))

z = np.load("tests/golden/small_cases.npz")
stage = sys.argv[1] if len(sys.argv) > 1 else "all"
for name in [str(n) for n in z["names"]]:
    nx, ny, nz = (int(t) for t in name.split("_")[0][1:].split("x"))
    A = z[name + "/A"]; v = z[name + "/v"]
    a = ntd.BandedMatrix(nx, ny, nz, A)
    out = [name]
    y = ntd.spmv(a, v); out.append("spmv=%s" % np.array_equal(y, z[name + "/spmv"]))
    pre = ntd.PreconBands(nx, ny, nz, *z[name + "/pre"])
    x = ntd.ntd_apply(pre, v); out.append("apply=%.1e" % rel(x, z[name + "/ntd"]))
    torch.cuda.synchronize()
    p2 = ntd.factor_level3(a); out.append("factor=%.1e" % rel(p2.host(), z[name + "/pre"]))
    if name + "/ilu" in z:
        f = ntd.build_block_ilu0(a); out.append("ilu=%s" % np.array_equal(f.data, z[name + "/ilu"]))
        zz = ntd.ilu0_apply(f, v); out.append("iluap=%s" % np.array_equal(zz, z[name + "/ilu_apply"]))
        cp = ntd.CombinedPrecond(a)
        out.append("comb=%.1e" % rel(ntd.combined_apply(cp, v), z[name + "/combined"]))
        xs, st = ntd.pcg(a, z[name + "/spmv"], cp, tol=1e-8, max_iters=100)
        out.append("pcg=%d/%d %.1e" % (st.iterations, z[name + "/pcg_iters"][0], st.final_relres))
    print(" ".join(out), flush=True)

for cfg in (1, 2, 3):
    data, xt, (nx, ny, nz) = problems.baseline_config(cfg)
    a = ntd.BandedMatrix(nx, ny, nz, data)
    b = ntd.spmv(a, xt)
    t = time.perf_counter(); cp = ntd.CombinedPrecond(a); ts = time.perf_counter() - t
    t = time.perf_counter(); x, st = ntd.pcg(a, b, cp, tol=1e-8); tsol = time.perf_counter() - t
    pre_o = oracle.factor_level3(data, nx, ny, nz)
    vv = np.random.default_rng(1).uniform(-1, 1, a.n_rows)
    ea = rel(ntd.ntd_apply(cp.ntd, vv), oracle.ntd_apply(pre_o, vv, nx, ny, nz))
    ef = rel(cp.ntd.host(), pre_o)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bd = torch.from_numpy(vv).cuda()
    ntd.device.ntd_apply(cp.ntd.bands, bd, nx, ny, nz, 1, solve=cp.ntd.solve)
    ev0.record()
    for _ in range(5):
        ntd.device.ntd_apply(cp.ntd.bands, bd, nx, ny, nz, 1, solve=cp.ntd.solve)
    ev1.record(); torch.cuda.synchronize()
    print(f"cfg{cfg}: iters {st.iterations} relres {st.final_relres:.3e} setup {ts:.3f}s solve {tsol:.3f}s "
          f"factor_err {ef:.1e} apply_err {ea:.1e} apply_ms {ev0.elapsed_time(ev1)/5:.3f}", flush=True)
