"""Pin the CPU oracle (oracle/ntd_oracle.c) against the reference's own
outputs (tests/golden/small_cases.npz, generated from /root/reference by
tests/golden/gen_golden.py).  The oracle restates the reference arithmetic in
the same order, so everything except the PCG dot products is bitwise."""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, grid_of


def names(golden):
    return [str(n) for n in golden["names"]]


def test_spmv_factor_apply_bitwise(golden):
    for name in names(golden):
        nx, ny, nz = grid_of(name)
        A, v = golden[name + "/A"], golden[name + "/v"]
        assert np.array_equal(oracle.spmv(A, v, nx, ny, nz), golden[name + "/spmv"]), name
        pre = oracle.factor_level3(A, nx, ny, nz)
        assert np.array_equal(pre, golden[name + "/pre"]), name
        assert np.array_equal(oracle.ntd_apply(pre, v, nx, ny, nz), golden[name + "/ntd"]), name
        assert np.array_equal(oracle.ntd_apply(pre, v, nx, ny, nz, lanes=1), golden[name + "/ntd_lanes1"]), name


def test_ilu0_combined_bitwise_and_pcg_iterations(golden):
    for name in names(golden):
        if name + "/ilu" not in golden:
            continue
        nx, ny, nz = grid_of(name)
        A, v = golden[name + "/A"], golden[name + "/v"]
        f, split = oracle.build_block_ilu0(A, nx, ny, nz)
        assert split == int(golden[name + "/ilu_split"][0])
        assert np.array_equal(f, golden[name + "/ilu"]), name
        assert np.array_equal(oracle.ilu0_apply(f, split, v, nx, ny, nz), golden[name + "/ilu_apply"])
        pre = oracle.factor_level3(A, nx, ny, nz)
        z = oracle.combined_apply(A, pre, f, split, v, nx, ny, nz)
        assert np.array_equal(z, golden[name + "/combined"]), name
        x, it, conv, hist = oracle.pcg(A, golden[name + "/spmv"], nx, ny, nz, tol=1e-8, max_iters=100)
        it_ref, conv_ref = (int(t) for t in golden[name + "/pcg_iters"])
        assert (it, conv) == (it_ref, bool(conv_ref)), name
        np.testing.assert_allclose(hist, golden[name + "/pcg_hist"], rtol=1e-6, atol=0)


def test_chain_known_answers(golden):
    for n in (1, 2, 7, 8, 9, 33):
        dr, off, bb = golden[f"chain/{n}/in"]
        for direction in ("forward", "backward"):
            for lanes in (1, 4):
                got = oracle.chain_bidiagonal_solve(dr, off, bb, direction, lanes)
                assert np.array_equal(got, golden[f"chain/{n}/{direction}/{lanes}"])


def test_oracle_on_baseline_configs_1_2():
    from paper_1909_09771_b200 import problems
    with open(os.path.join(GOLDEN, "configs.json")) as fh:
        cfgs = json.load(fh)
    for key, rec in cfgs.items():
        data, x_true, (nx, ny, nz) = problems.baseline_config(int(key))
        idx = rec["sample_idx"]
        b = oracle.spmv(data, x_true, nx, ny, nz)
        assert [float(b[i]) for i in idx] == rec["b"]["sample"]
        pre = oracle.factor_level3(data, nx, ny, nz)
        for i, nm in enumerate(("l1", "u1", "l2", "u2")):
            assert [float(pre[i][j]) for j in idx] == rec["pre_" + nm]["sample"]
        assert [float(pre[6][j]) for j in idx] == rec["pre_m_recip"]["sample"]
        v = np.random.default_rng(rec["apply_v_seed"]).uniform(-1.0, 1.0, nx * ny * nz)
        assert [float(t) for t in oracle.ntd_apply(pre, v, nx, ny, nz)[idx]] == rec["ntd_apply"]["sample"]
        x, it, conv, hist = oracle.pcg(data, b, nx, ny, nz, tol=1e-8, max_iters=200)
        assert conv and it == rec["pcg_iters"]


def test_oracle_factorization_errors():
    a = np.zeros((7, 8))
    a[3] = 1.0
    a[3, 5] = 0.0
    with pytest.raises(oracle.OracleFactorizationError, match="row 5"):
        oracle.factor_level3(a, 8, 1, 1)
    with pytest.raises(oracle.OracleFactorizationError, match="row 5"):
        oracle.build_block_ilu0(a, 8, 1, 1)
