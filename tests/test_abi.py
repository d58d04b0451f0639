"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads, exports every
symbol include/earl_dispatch.h declares, and fails loudly (never falls back) without a GPU."""
import os
import re
import subprocess

import pytest

from paper_2510_05943_b200 import build, earl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "earl_dispatch.h")).read()
    return sorted(set(re.findall(r"EARL_API\s+[\w\s\*]+?\b(earl_\w+)\s*\(", text)))


def test_library_builds_for_sm100a():
    lib = build.build()
    assert os.path.exists(lib)
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_exported():
    build.build()
    decl = declared_symbols()
    assert len(decl) >= 20
    assert sorted(earl.EXPORTED) == decl
    nm = subprocess.run(["nm", "-D", "--defined-only", earl.LIB_PATH], capture_output=True,
                        text=True).stdout
    exported = set(re.findall(r" T (earl_\w+)", nm))
    assert set(decl) <= exported
    L = earl.lib()
    for name in decl:
        getattr(L, name)
    assert L.earl_abi_version() == 1
    assert L.earl_status_string(2) == b"EARL_ERR_LAYOUT"


def test_no_internal_symbols_leak():
    nm = subprocess.run(["nm", "-D", "--defined-only", earl.LIB_PATH], capture_output=True,
                        text=True).stdout
    exported = re.findall(r" T (\S+)", nm)
    assert all(s.startswith("earl_") for s in exported), exported


def test_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(earl.EarlError) as e:
        earl.Comm(earl.EARL_ALL_RANKS, 2, 0, 0)
    assert e.value.status in (1, 4)  # INVALID_ARGUMENT (no device) or CUDA


def test_argument_validation_needs_no_gpu():
    import ctypes as C
    L = earl.lib()
    assert L.earl_comm_create(0, 9, 0, 0, C.byref(C.c_void_p())) == 8  # UNSUPPORTED
    assert b"world 9" in L.earl_last_error()
    assert L.earl_comm_create(3, 2, 0, 0, C.byref(C.c_void_p())) == 1
