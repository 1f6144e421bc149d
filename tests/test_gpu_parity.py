"""GPU parity of the product path (C ABI via the drop-in API) against the
reference's own outputs (tests/golden, generated from /root/reference by
tests/golden/gen_golden.py) and against the CPU oracle.

Bars: spmv and ILU0 bitwise; NTD factor bands and NTD / combined applies
<= 1e-10 relative (BASELINE.json north_star); PCG iteration counts within
+-1 and final relres < tol.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, grid_of

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-10  # north_star: preconditioner apply relative error <= 1e-10 (fp64)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def ntd():
    import paper_1909_09771_b200 as m
    return m


def names(golden):
    return [str(n) for n in golden["names"]]


def test_spmv_bitwise(ntd, golden):
    for name in names(golden):
        nx, ny, nz = grid_of(name)
        a = ntd.BandedMatrix(nx, ny, nz, golden[name + "/A"])
        y = ntd.spmv(a, golden[name + "/v"])
        assert np.array_equal(y, golden[name + "/spmv"]), name


def test_factor_bands_match_reference(ntd, golden):
    for name in names(golden):
        nx, ny, nz = grid_of(name)
        a = ntd.BandedMatrix(nx, ny, nz, golden[name + "/A"])
        pre = ntd.factor_level3(a)
        want = golden[name + "/pre"]
        got = pre.host()
        # the setup's nested solves follow the reference's chain order
        # (CHAIN_LANES = 4): every band is bitwise the reference's
        for i in range(7):
            assert np.array_equal(got[i], want[i]), (name, i, rel(got[i], want[i]))


def test_ntd_apply_matches_reference(ntd, golden):
    for name in names(golden):
        nx, ny, nz = grid_of(name)
        want = golden[name + "/ntd"]
        pre = ntd.PreconBands(nx, ny, nz, *golden[name + "/pre"])
        x = ntd.ntd_apply(pre, golden[name + "/v"])
        assert rel(x, want) <= APPLY_TOL, (name, rel(x, want))
        # and with the GPU's own factor
        a = ntd.BandedMatrix(nx, ny, nz, golden[name + "/A"])
        x2 = ntd.ntd_apply(ntd.factor_level3(a), golden[name + "/v"])
        assert rel(x2, want) <= APPLY_TOL, (name, rel(x2, want))


def test_ilu0_bitwise(ntd, golden):
    for name in names(golden):
        if name + "/ilu" not in golden:
            continue
        nx, ny, nz = grid_of(name)
        a = ntd.BandedMatrix(nx, ny, nz, golden[name + "/A"])
        f = ntd.build_block_ilu0(a)
        assert f.split == int(golden[name + "/ilu_split"][0])
        assert np.array_equal(f.data, golden[name + "/ilu"]), name
        z = ntd.ilu0_apply(f, golden[name + "/v"])
        assert np.array_equal(z, golden[name + "/ilu_apply"]), name


def test_combined_apply_and_pcg(ntd, golden):
    for name in names(golden):
        if name + "/combined" not in golden:
            continue
        nx, ny, nz = grid_of(name)
        a = ntd.BandedMatrix(nx, ny, nz, golden[name + "/A"])
        cp = ntd.CombinedPrecond(a)
        z = ntd.combined_apply(cp, golden[name + "/v"])
        assert rel(z, golden[name + "/combined"]) <= APPLY_TOL, name
        b = golden[name + "/spmv"]
        x, st = ntd.pcg(a, b, cp, tol=1e-8, max_iters=100)
        it_ref, conv_ref = (int(v) for v in golden[name + "/pcg_iters"])
        assert st.converged == bool(conv_ref), name
        assert abs(st.iterations - it_ref) <= 1, (name, st.iterations, it_ref)
        assert st.final_relres < 1e-8


def test_baseline_configs_1_2(ntd):
    from paper_1909_09771_b200 import problems
    with open(os.path.join(GOLDEN, "configs.json")) as fh:
        cfgs = json.load(fh)
    for key, rec in cfgs.items():
        cfg = int(key)
        data, x_true, (nx, ny, nz) = problems.baseline_config(cfg)
        a = ntd.BandedMatrix(nx, ny, nz, data)
        idx = rec["sample_idx"]
        b = ntd.spmv(a, x_true)
        assert [float(b[i]) for i in idx] == rec["b"]["sample"]
        pre = ntd.factor_level3(a)
        for nm in ("l1", "u1", "l2", "u2", "m_recip"):
            got = np.array([getattr(pre, nm)[i] for i in idx])
            want = np.array(rec["pre_" + nm]["sample"])
            assert rel(got, want) <= APPLY_TOL, (cfg, nm)
        v = np.random.default_rng(rec["apply_v_seed"]).uniform(-1.0, 1.0, a.n_rows)
        x = ntd.ntd_apply(pre, v)
        assert rel(x[idx], rec["ntd_apply"]["sample"]) <= APPLY_TOL
        f = ntd.build_block_ilu0(a)
        z = ntd.ilu0_apply(f, v)
        assert [float(z[i]) for i in idx] == rec["ilu_apply"]["sample"]
        cp = ntd.CombinedPrecond(a)
        assert rel(ntd.combined_apply(cp, v)[idx], rec["combined"]["sample"]) <= APPLY_TOL
        xs, st = ntd.pcg(a, b, cp, tol=1e-8, max_iters=200)
        assert st.converged and st.final_relres < 1e-8
        assert abs(st.iterations - rec["pcg_iters"]) <= 1, (cfg, st.iterations, rec["pcg_iters"])


def test_symmetric_packed_stencil_bitwise(ntd, golden):
    """The 4-band symmetric operator (ntd_sym_pack) gives bitwise the same
    residuals and CG iterates as the reference-order 7-band kernels; a
    non-symmetric operator is refused (stays on the 7-band path)."""
    import torch
    from paper_1909_09771_b200 import device as D
    for name in names(golden):
        nx, ny, nz = grid_of(name)
        n = nx * ny * nz
        A = torch.from_numpy(np.ascontiguousarray(golden[name + "/A"])).cuda().reshape(1, 7, n)
        a4 = D.sym_pack(A, nx, ny, nz, 1)
        assert a4 is not None, name
        gen = torch.Generator().manual_seed(7)
        r, w, v = ((torch.rand((1, n), generator=gen, dtype=torch.float64) * 2 - 1).cuda() for _ in range(3))
        assert torch.equal(D.residual(A, r, w, nx, ny, nz, 1), D.residual(A, r, w, nx, ny, nz, 1, a4=a4)), name
        z7, z4 = torch.empty_like(r), torch.empty_like(r)
        t7 = D.residual(A, r, w, nx, ny, nz, 1, v=v, z_out=z7)
        t4 = D.residual(A, r, w, nx, ny, nz, 1, v=v, z_out=z4, a4=a4)
        assert torch.equal(t7, t4) and torch.equal(z7, z4), name
        xs = []
        for op in (None, a4):
            cg = D.PcgDevice(A, nx, ny, nz, 1, 30, a4=op)
            it = cg.solve(r, 1e-10)
            xs.append((it, cg.x.clone()))
        assert xs[0][0] == xs[1][0] and torch.equal(xs[0][1], xs[1][1]), name
    B = A.clone()
    B[0, 2, 1] += 1e-3  # A[1][0] != A[0][1]
    assert D.sym_pack(B, nx, ny, nz, 1) is None


def test_fused_slot_stages_bitwise(ntd, golden):
    """The combined apply with the residuals fused into the NTD apply's slot
    layout (ntd_residual_to_slot / ntd_apply_slot / ntd_residual_from_slot)
    is bitwise the unfused sequence (natural-layout residuals + ntd_apply),
    with the 7-band and the symmetric 4-band operator."""
    import torch
    from paper_1909_09771_b200 import device as D
    for name in names(golden):
        nx, ny, nz = grid_of(name)
        n = nx * ny * nz
        a = ntd.BandedMatrix(nx, ny, nz, golden[name + "/A"])
        A = a.device_data().reshape(1, 7, n)
        if n < 2:
            continue
        pre = ntd.factor_level3(a).bands.reshape(1, 7, n)
        g = ntd.build_block_ilu0(a)
        f = g.device_data.reshape(1, 7, n)
        r = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (1, n))).cuda()
        for a4 in ("auto", None):
            cd = D.CombinedDevice(A, nx, ny, nz, 1, pre=pre, ilu=f, split=g.split, a4=a4)
            if not cd.fused:
                continue
            z1 = cd.apply(r, torch.empty_like(r)).clone()
            cd.fused = False
            z2 = cd.apply(r, torch.empty_like(r)).clone()
            assert torch.equal(z1, z2), (name, a4)


def test_device_assembly_bitwise(ntd):
    """ntd_assemble (problem_gen.py:87-133 on the device) is
    bitwise the host restatement (itself pinned bitwise to the reference by
    test_problems.py) on the reference's fields, degenerate grids, and the
    BASELINE fields including config 2's Neumann faces."""
    import torch
    from paper_1909_09771_b200 import device as D
    from paper_1909_09771_b200 import problems
    cases = []
    for field in (1, 2, 3):
        for grid in ((7, 5, 6), (1, 3, 2), (2, 1, 1), (1, 1, 1), (12, 12, 12)):
            cases.append((problems.reference_kappa(field, *grid), grid, problems.ALL_DIRICHLET))
    for cfg, s in ((1, 0), (2, 0), (3, 0), (4, 0), (4, 63)):
        kap, bc, _ = problems.baseline_kappa(cfg, s)
        cases.append((kap, problems.CONFIGS[cfg]["grid"], bc))
    rng = np.random.default_rng(5)
    cases.append((np.exp(rng.normal(0, 3, (9, 4, 11))), (11, 4, 9), (True, False, False, True, True, False)))
    for kap, (nx, ny, nz), bc in cases:
        want = problems.assemble_kappa(kap, nx, ny, nz, bc)
        got = D.assemble(torch.from_numpy(np.ascontiguousarray(kap)).cuda(), nx, ny, nz, bc)
        assert np.array_equal(got[0].cpu().numpy(), want), ((nx, ny, nz), bc)


def test_sm_mappings_bitwise(ntd):
    """The ILU0 sweep with one CTA per system half or a cluster of CTAs per
    half, and the NTD sweep with one or two CTAs per system, give bitwise the
    same results (config 2 plus a small odd grid, two systems per launch)."""
    import torch
    from paper_1909_09771_b200 import _lib, problems
    from paper_1909_09771_b200 import device as D
    from paper_1909_09771_b200.batch import BatchSolver
    grids = [problems.baseline_config(2)]
    rng = np.random.default_rng(9)
    kap = np.exp(rng.normal(0, 2, (10, 37, 21)))
    grids.append((problems.assemble_kappa(kap, 21, 37, 10), None, (21, 37, 10)))
    for data, _, (nx, ny, nz) in grids:
        n = nx * ny * nz
        A = torch.from_numpy(np.stack([data, data])).cuda()
        s = BatchSolver(A, nx, ny, nz, groups=1).setup()
        P = s.precond
        v = torch.from_numpy(rng.uniform(-1, 1, (2, n))).cuda()
        # reference-layout ILU0 kernel (ilu0.cu) as the anchor
        z_ref = torch.empty_like(v)
        D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, 2, z=z_ref)
        outs = []
        need = _lib.load().ntd_ilu0_skew_work_doubles(nx, ny, nz, 2)
        for ctas in ((1, 24), (2, 24), (4, 12), (8, 6)):
            z = torch.empty_like(v)
            # the sweep never reads the empty (padding) slots of its skewed
            # work arrays: NaN there must not reach the result
            work = torch.full((need,), float("nan"), dtype=torch.float64, device=v.device)
            D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, 2, z=z, skew=P.skew, work=work, ctas=ctas, hp=None)
            outs.append(z)
        # the hyperplane kernel: one CTA or a cluster of CTAs per half, 1..8
        # units per warp, z and / or acc outputs
        g = (ny + 31) // 32
        nk = max(P.split // (nx * ny), nz - P.split // (nx * ny))
        for nc in (1, 2, 4, 8, 16, 24, 32):  # > 16: CTAs linked through global memory
            if nc > nk or 2 * 2 * nc > 148:
                continue
            umax = -(-nk // nc) * g
            for w in sorted({max(1, -(-umax // 8)), min(16, umax), min(24, umax)}):
                if -(-umax // w) > 8 or (w > 16 and -(-umax // w) > 1) or umax > 380:
                    continue
                z = torch.empty_like(v)
                acc = torch.full_like(v, 0.5)
                work = torch.full((need,), float("nan"), dtype=torch.float64, device=v.device)
                D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, 2, z=z, acc=acc, skew=P.skew, work=work, hp=(nc, w))
                assert torch.equal(z, z_ref), (nx, ny, nz, nc, w)
                assert torch.equal(acc, z_ref + 0.5), (nx, ny, nz, nc, w)
                if 1 < nc <= 16:  # the same mapping with global-memory rings inside a cluster launch
                    z3 = torch.empty_like(v)
                    D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, 2, z=z3, skew=P.skew, work=work, hp=(nc, w, 2))
                    assert torch.equal(z3, z_ref), (nx, ny, nz, nc, w, "global links")
                z2 = torch.empty_like(v)
                D.ilu0_apply(P.ilu, P.split, v, nx, ny, nz, 2, z=z2, skew=P.skew, work=work, hp=(nc, w))
                assert torch.equal(z2, z_ref), (nx, ny, nz, nc, w)
        assert all(torch.equal(z_ref, o) for o in outs), (nx, ny, nz)
        if P.fused:
            xs = []
            for c in (1, 2):
                P.work.zero_()
                _lib.call("ntd_residual_to_slot", _lib.ptr(P.a4), 4, _lib.ptr(P.solve), _lib.ptr(v), _lib.ptr(outs[0]),
                          _lib.ptr(P.work), nx, ny, nz, 2, None, _lib.stream())
                _lib.call("ntd_apply_slot_ex", _lib.ptr(P.solve), _lib.ptr(P.work), nx, ny, nz, 2, None, c,
                          _lib.stream())
                # the apply's result x in the slot layout: work[s:2s]
                kk = next(k for k in (1, 2, 3, 4, 5, 6, 8, 11, 12, 16) if 32 * k >= nx)
                s_ = ny * nz * (32 * kk) * 2
                xs.append(P.work[s_:2 * s_].clone())
            assert torch.equal(xs[0], xs[1]), (nx, ny, nz)


def test_reduction_tree_depends_on_n_only(ntd):
    """The stencil / CG reductions partition rows over red_vblocks(n) virtual
    blocks (a function of n alone), so a system's PCG iterates are bitwise
    the same solved alone or inside a batch, and for any stream grouping."""
    import torch
    from paper_1909_09771_b200 import problems
    from paper_1909_09771_b200.batch import BatchSolver
    data, x_true, (nx, ny, nz) = problems.baseline_config(2, 0)
    a = ntd.BandedMatrix(nx, ny, nz, data)
    b = ntd.spmv(a, x_true)
    x1, st = ntd.pcg(a, b, ntd.CombinedPrecond(a), tol=1e-8)
    assert st.iterations == 26  # config 2: the reference's 26 iterations
    A = torch.from_numpy(np.stack([data] * 3)).cuda()
    B = torch.from_numpy(np.stack([b] * 3)).cuda()
    for groups in (1, 3):
        res = BatchSolver(A, nx, ny, nz, groups=groups).setup().solve(B, 1e-8)
        assert res.iterations == [26] * 3
        for k in range(3):
            assert np.array_equal(res.x[k].cpu().numpy(), x1), (groups, k)
