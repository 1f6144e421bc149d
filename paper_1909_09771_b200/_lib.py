"""ctypes binding of libntdgpu.so (include/ntdgpu.h).

There is no fallback: if the library is missing or no CUDA device is present,
every hot-path call raises ``NativeUnavailable``.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libntdgpu.so")

NTD_ST = dict(RZ=0, PAP=1, ALPHA=2, BETA=3, BNORM=4, RELRES=5, TOL=6, N=8)
NTD_FL = dict(ACTIVE=0, STATUS=1, ITERS=2, N=4)
PCG_RUNNING, PCG_CONVERGED, PCG_BREAKDOWN, PCG_NONFINITE = 0, 1, 2, 3

_P = ctypes.c_void_p
_I = ctypes.c_int64
_INT = ctypes.c_int

# name -> (restype, argtypes); mirrors include/ntdgpu.h
_SIGS = {
    "ntd_version": (ctypes.c_char_p, []),
    "ntd_last_error": (ctypes.c_char_p, []),
    "ntd_max_nx": (_I, []),
    "ntd_assemble": (_INT, [_P, _P, _I, _I, _I, _I, _I, _P]),
    "ntd_spmv": (_INT, [_P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_residual": (_INT, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_sym_pack": (_INT, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "ntd_residual_sym": (_INT, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_dot_work_doubles": (_I, [_I]),
    "ntd_dot": (_INT, [_P, _P, _P, _INT, _I, _I, _P, _P, _P]),
    "ntd_axpy": (_INT, [ctypes.c_double, _P, _P, _P, _I, _P]),
    "ntd_chain_work_doubles": (_I, [_I, _I]),
    "ntd_chain_solve": (_INT, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P]),
    "ntd_pcg_init": (_INT, [_P, _P, _P, _P, _P, _P, ctypes.c_double, _I, _I, _P, _P]),
    "ntd_pcg_start": (_INT, [_P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "ntd_pcg_spmv_alpha": (_INT, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_pcg_update_residual": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I,
                                       _I, _P, _P]),
    "ntd_pcg_spmv_alpha_sym": (_INT, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_pcg_update_residual_sym": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I,
                                           _I, _P, _P]),
    "ntd_pcg_direction": (_INT, [_P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "ntd_factor_work_doubles": (_I, [_I, _I, _I, _I]),
    "ntd_factor": (_INT, [_P, _P, _P, _P, _I, _I, _I, _I, _P]),
    "ntd_apply_work_doubles": (_I, [_I, _I, _I, _I]),
    "ntd_solve_doubles": (_I, [_I, _I, _I, _I]),
    "ntd_solve_bands": (_INT, [_P, _P, _I, _I, _I, _I, _P]),
    "ntd_apply": (_INT, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_apply_ex": (_INT, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _P]),
    "ntd_apply_direct": (_INT, [_P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_residual_to_slot": (_INT, [_P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_apply_slot": (_INT, [_P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_apply_slot_ex": (_INT, [_P, _P, _I, _I, _I, _I, _P, _I, _P]),
    "ntd_residual_from_slot": (_INT, [_P, _I, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_ilu0_factor": (_INT, [_P, _P, _I, _P, _I, _I, _I, _I, _P]),
    "ntd_ilu0_apply": (_INT, [_P, _I, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_ilu0_skew_doubles": (_I, [_I, _I, _I, _I, _I]),
    "ntd_ilu0_skew_build": (_INT, [_P, _P, _I, _I, _I, _I, _I, _P]),
    "ntd_ilu0_skew_work_doubles": (_I, [_I, _I, _I, _I]),
    "ntd_ilu0_skew_apply": (_INT, [_P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P]),
    "ntd_ilu0_skew_apply_ex": (_INT, [_P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _I, _P]),
    "ntd_ilu0_hp_units": (_I, [_I, _I, _I, _I]),
    "ntd_ilu0_hp_apply": (_INT, [_P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _I, _P]),
    "ntd_ilu0_hp_apply_ex": (_INT, [_P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _I, _I, _P]),
}

EXPORTED = tuple(_SIGS)

# kernels launched by one successful call of each entry point (counted for
# bench.py's gpu_launches; see the launch sites in csrc/)
KERNELS_PER_CALL = {
    "ntd_assemble": 1, "ntd_spmv": 1, "ntd_residual": 1, "ntd_axpy": 1, "ntd_chain_solve": 1, "ntd_dot": 2, "ntd_pcg_init": 3, "ntd_pcg_start": 3,
    "ntd_pcg_spmv_alpha": 2, "ntd_pcg_update_residual": 3, "ntd_pcg_direction": 3, "ntd_factor": 1,
    "ntd_apply": 3, "ntd_apply_ex": 3, "ntd_apply_direct": 1, "ntd_solve_bands": 1, "ntd_ilu0_factor": 2, "ntd_ilu0_apply": 1, "ntd_ilu0_skew_build": 1,
    "ntd_ilu0_skew_apply": 1, "ntd_ilu0_skew_apply_ex": 1, "ntd_sym_pack": 1, "ntd_residual_sym": 1, "ntd_pcg_spmv_alpha_sym": 2,
    "ntd_pcg_update_residual_sym": 3, "ntd_residual_to_slot": 1, "ntd_apply_slot": 1, "ntd_apply_slot_ex": 1,
    "ntd_residual_from_slot": 1, "ntd_ilu0_hp_apply": 2, "ntd_ilu0_hp_apply_ex": 2,
}
_launches = [0]


def reset_launch_count():
    _launches[0] = 0


def launch_count():
    return _launches[0]


class NativeUnavailable(RuntimeError):
    """libntdgpu.so is missing or no CUDA device is available."""


class NativeError(RuntimeError):
    """A libntdgpu call returned an error code."""


_lib = None


def load(require_device=True):
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} not built; run `python -m paper_1909_09771_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device and not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the NTD-PCG path runs only on the GPU")
    return _lib


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def call(name, *args):
    fn = getattr(load(), name)
    rc = fn(*args)
    _launches[0] += KERNELS_PER_CALL.get(name, 0)
    if rc != 0:
        msg = (_lib.ntd_last_error() or b"").decode()
        if rc == -1:
            raise ValueError(f"{name}: invalid arguments")
        if rc == -2:
            raise ValueError(f"{name}: grid not supported (nx <= {_lib.ntd_max_nx()})")
        raise NativeError(f"{name} failed ({rc}): {msg}")
    return rc
