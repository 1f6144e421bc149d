"""CPU oracle for the NTD-PCG hot path -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``ntd_oracle.c``, a plain-C restatement of the reference
``ntdprecon`` kernels (/root/reference/pkg/src/ntdprecon, file:line cited per
function in the C source).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg may import this module,
and only as the checker or the timed CPU baseline.  The product package
``paper_1909_09771_b200`` never imports it (tests/test_product_boundary.py
checks that).

Parity pin: tests/test_oracle_golden.py checks every function here against
fixtures generated from the real reference by tests/golden/gen_golden.py
(bitwise for spmv / factor / apply / ILU0; PCG iteration counts exact).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libntd_oracle.so")
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_pi64 = ctypes.POINTER(ctypes.c_int64)


class OracleFactorizationError(RuntimeError):
    pass


class OracleDivergenceError(RuntimeError):
    pass


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_spmv.argtypes = [_d, _d, _d, _i64, _i64, _i64, ctypes.c_int]
        L.orc_chain_solve.argtypes = [_d, _d, _d, _d, _i64, ctypes.c_int, ctypes.c_int]
        L.orc_ntd_apply.argtypes = [_d, _d, _d, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]
        L.orc_factor_level3.argtypes = [_d, _d, _i64, _i64, _i64, ctypes.c_int,
                                        ctypes.c_int, _pi64]
        L.orc_build_ilu0.argtypes = [_d, _d, _i64, _i64, _i64, _i64, ctypes.c_int]
        L.orc_build_ilu0.restype = _i64
        L.orc_ilu0_apply.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, ctypes.c_int]
        L.orc_combined_apply.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64,
                                         ctypes.c_int, ctypes.c_int, _d, _d]
        L.orc_pcg.argtypes = [_d, _d, _d, _i64, _i64, _i64, _i64, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, _d, _d, ctypes.c_double,
                              _i64, _d, ctypes.POINTER(ctypes.c_int)]
        L.orc_pcg.restype = _i64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_d)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def spmv(data, x, nx, ny, nz, nthreads=1):
    """banded_core.py:95-130"""
    data = _f64(data)
    x = _f64(x)
    n = nx * ny * nz
    y = np.empty(n)
    lib().orc_spmv(_p(data), _p(x), _p(y), n, nx, nx * ny, nthreads)
    return y


def chain_bidiagonal_solve(dr, off, b, direction="forward", lanes=4):
    """ntd_solve.py:272-300"""
    dr, off, b = _f64(dr), _f64(off), _f64(b)
    n = dr.shape[0]
    x = np.empty(n)
    lib().orc_chain_solve(_p(dr), _p(off), _p(b), _p(x), n,
                          0 if direction == "forward" else 1, lanes)
    return x


_FACTOR_MSG = {1: "zero or non-finite pivot", 2: "non-finite filter weight",
               3: "non-finite sandwich adjustment"}


def factor_level3(data, nx, ny, nz, lanes=4, nthreads=1):
    """ntd_factor.py:351-458.  Returns the (7, N) array l1,u1,l2,u2,l3,u3,m_recip."""
    data = _f64(data)
    n = nx * ny * nz
    pre = np.empty((7, n))
    st = np.zeros(3, dtype=np.int64)
    lib().orc_factor_level3(_p(data), _p(pre), nx, ny, nz, lanes, nthreads,
                            st.ctypes.data_as(_pi64))
    if st[0]:
        raise OracleFactorizationError(
            f"{_FACTOR_MSG[int(st[0])]} at row {int(st[2])} (plane {int(st[1])})")
    return pre


def ntd_apply(pre, b, nx, ny, nz, lanes=4, nthreads=1):
    """ntd_solve.py:303-322"""
    pre, b = _f64(pre), _f64(b)
    x = np.empty(nx * ny * nz)
    lib().orc_ntd_apply(_p(pre), _p(b), _p(x), nx, ny, nz, lanes, nthreads)
    return x


def build_block_ilu0(data, nx, ny, nz, split=None, nthreads=1):
    """ilu0.py:134-156.  Returns (f (7,N), split)."""
    data = _f64(data)
    n = nx * ny * nz
    if split is None:
        split = n // 2
    f = np.empty((7, n))
    bad = lib().orc_build_ilu0(_p(data), _p(f), nx, ny, nz, split, nthreads)
    if bad >= 0:
        raise OracleFactorizationError(f"zero or non-finite pivot at row {bad}")
    return f, split


def ilu0_apply(f, split, r, nx, ny, nz, nthreads=1):
    """ilu0.py:159-169"""
    f, r = _f64(f), _f64(r)
    z = np.empty(nx * ny * nz)
    lib().orc_ilu0_apply(_p(f), _p(r), _p(z), nx, ny, nz, split, nthreads)
    return z


def combined_apply(data, pre, f, split, r, nx, ny, nz, lanes=4, nthreads=1):
    """precond_pcg.py:57-65"""
    data, pre, f, r = _f64(data), _f64(pre), _f64(f), _f64(r)
    z = np.empty(nx * ny * nz)
    lib().orc_combined_apply(_p(data), _p(pre), _p(f), nx, ny, nz, split, lanes,
                             nthreads, _p(r), _p(z))
    return z


def pcg(data, b, nx, ny, nz, kind="ntd+ilu0", tol=1e-7, max_iters=200,
        lanes=4, nthreads=1, pre=None, ilu=None):
    """precond_pcg.py:68-122 with the combined (ntd+ilu0), the ntd-only
    (bench_cli.py:113-121) or no preconditioner.
    Returns (x, iterations, converged, history).  Factorizations are built
    here unless passed in (pre, (f, split))."""
    data, b = _f64(data), _f64(b)
    n = nx * ny * nz
    if kind == "ntd+ilu0":
        if pre is None:
            pre = factor_level3(data, nx, ny, nz, lanes, nthreads)
        if ilu is None:
            ilu = build_block_ilu0(data, nx, ny, nz, nthreads=nthreads)
        f, split = ilu
        k = 1
    elif kind == "ntd":
        if pre is None:
            pre = factor_level3(data, nx, ny, nz, lanes, nthreads)
        f, split = np.zeros(1), 0
        k = 2
    elif kind == "none":
        pre = np.zeros(1)
        f, split = np.zeros(1), 0
        k = 0
    else:
        raise ValueError(kind)
    x = np.empty(n)
    hist = np.zeros(max_iters)
    conv = ctypes.c_int(0)
    it = lib().orc_pcg(_p(data), _p(_f64(pre)), _p(_f64(f)), nx, ny, nz, split,
                       lanes, nthreads, k, _p(b), _p(x), tol, max_iters, _p(hist),
                       ctypes.byref(conv))
    if it < 0:
        raise OracleDivergenceError("breakdown")
    return x, int(it), bool(conv.value), hist[:it].tolist()
