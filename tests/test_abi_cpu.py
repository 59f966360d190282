"""CPU-side checks of the boundary: the C-ABI library builds/loads and exports every
symbol include/seaice.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2204_10822_b200 import build as B
from paper_2204_10822_b200 import seaice


def test_library_builds_and_exports_header_symbols():
    path = B.build()
    assert os.path.exists(path)
    L = ctypes.CDLL(path)
    names = seaice.header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    # the binding declares a signature for every header function
    bound = seaice.lib()
    for name in names:
        assert getattr(bound, name).argtypes is not None or name == "seaice_launch_count", name


def test_library_has_no_torch_dependency_and_targets_sm100a():
    path = B.build()
    out = subprocess.run(["ldd", path], capture_output=True, text=True).stdout
    assert "libtorch" not in out and "libc10" not in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_default_params_and_struct_layout():
    L = seaice.lib()
    p = seaice.Params()
    L.seaice_default_params(ctypes.byref(p), 64)
    assert p.n == 64 and p.L == 512e3 and p.P_star == 27500.0 and p.f_c == 1.46e-4
    assert p.newton_rtol == 1e-8 and p.newton_maxit == 200 and p.restart == 60 and p.krylov_maxit == 300
    assert p.ls_max_halvings == 20 and p.e == 2.0 and p.delta_min == 2e-9


def test_create_rejects_bad_params_without_gpu_work():
    """Parameter validation happens before any device call."""
    L = seaice.lib()
    p = seaice.Params()
    L.seaice_default_params(ctypes.byref(p), 1)  # n < 2
    h = ctypes.c_void_p()
    assert L.seaice_create(ctypes.byref(p), None, ctypes.byref(h)) == seaice.EINVAL
    L.seaice_default_params(ctypes.byref(p), 50000)  # int32 index overflow
    assert L.seaice_create(ctypes.byref(p), None, ctypes.byref(h)) == seaice.EINVAL
    assert L.seaice_destroy(None) == 0
