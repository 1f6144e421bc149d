"""The product package never imports or links the oracle, and its hot-path
entry points fail loudly without the native library / a device."""

import os
import re

import numpy as np
import pytest
import torch

from conftest import REPO

PKG = os.path.join(REPO, "paper_1909_09771_b200")


def test_no_oracle_reference_in_product_sources():
    for root, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"\bimport\s+oracle|from\s+oracle|ntd_oracle|libntd_oracle", src), f


def test_reference_name_surface():
    import paper_1909_09771_b200 as ntd
    ref_names = ["BandedMatrix", "FactorizationError", "axpy", "clamp_workers", "dot", "norm2", "spmv",
                 "to_matrix_market", "CoefficientField", "GridSpec", "assemble", "kappa_eval", "make_rhs",
                 "CHAIN_LANES", "SolveWorkspace", "chain_bidiagonal_solve", "ntd_apply", "LineBands", "PlaneBands",
                 "PreconBands", "compute_beta", "dump_precon_bands", "factor_level1", "factor_level2",
                 "factor_level3", "load_precon_bands", "twist_index", "ILU0Factors", "build_block_ilu0",
                 "ilu0_apply", "CombinedPrecond", "DivergenceError", "SolveStats", "combined_apply", "pcg",
                 "BenchConfig", "BenchReport", "run_benchmark", "speedup_probe"]
    for n in ref_names:
        assert hasattr(ntd, n), n
        assert n in ntd.__all__, n


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_hot_path_fails_loudly_without_device():
    import paper_1909_09771_b200 as ntd
    from paper_1909_09771_b200._lib import NativeUnavailable
    a = ntd.assemble(ntd.GridSpec(4, 4, 4), 3)
    for call in (lambda: ntd.spmv(a, np.ones(64)), lambda: ntd.factor_level3(a),
                 lambda: ntd.build_block_ilu0(a), lambda: ntd.pcg(a, np.ones(64))):
        with pytest.raises(NativeUnavailable):
            call()


def test_argument_validation_matches_reference():
    import paper_1909_09771_b200 as ntd
    a = ntd.BandedMatrix(4, 1, 1)
    with pytest.raises(ValueError):
        ntd.spmv(a, np.ones(3))
    with pytest.raises(ValueError):
        ntd.pcg(a, np.ones(3))
    with pytest.raises(ValueError):
        ntd.pcg(a, np.ones(4), tol=0.0)
    with pytest.raises(ValueError):
        ntd.pcg(a, np.ones(4), max_iters=0)
    with pytest.raises(ValueError):
        ntd.BandedMatrix(0, 1, 1)
    with pytest.raises(ValueError):
        ntd.BandedMatrix(2, 2, 2, np.zeros((7, 7)))
    with pytest.raises(ValueError):
        ntd.twist_index(0)
    assert [ntd.twist_index(n) for n in (1, 2, 3, 7)] == [1, 1, 2, 4]
    with pytest.raises(ValueError):
        ntd.build_block_ilu0(ntd.BandedMatrix(1, 1, 1))
    with pytest.raises(ValueError):
        ntd.clamp_workers(0)
