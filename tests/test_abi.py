"""The C-ABI library loads and exports every symbol include/ntdgpu.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "ntdgpu.h")
LIB = os.path.join(REPO, "paper_1909_09771_b200", "libntdgpu.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ntd_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_1909_09771_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_python_binding_covers_header():
    from paper_1909_09771_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared()


def test_host_only_entry_points(lib):
    lib.ntd_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.ntd_version()
    lib.ntd_max_nx.restype = ctypes.c_int64
    assert lib.ntd_max_nx() >= 512
    for fn, args in (("ntd_apply_work_doubles", (96, 96, 96, 64)), ("ntd_factor_work_doubles", (8, 8, 8, 2)),
                     ("ntd_dot_work_doubles", (3,))):
        f = getattr(lib, fn)
        f.restype = ctypes.c_int64
        f.argtypes = [ctypes.c_int64] * len(args)
        assert f(*args) > 0


def test_invalid_arguments_rejected_without_device(lib):
    # argument validation happens before any CUDA call
    lib.ntd_spmv.restype = ctypes.c_int
    rc = lib.ntd_spmv(None, None, None, ctypes.c_int64(1), ctypes.c_int64(1), ctypes.c_int64(1),
                      ctypes.c_int64(1), None, None)
    assert rc == -1


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
