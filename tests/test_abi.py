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
    assert L.earl_abi_version() == 3
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


def _build_c_smoke(tmp_path):
    build.build()
    exe = str(tmp_path / "abi_smoke")
    libdir = os.path.dirname(earl.LIB_PATH)
    cmd = ["gcc", "-O1", "-o", exe, os.path.join(ROOT, "tests", "c", "abi_smoke.c"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-L", libdir, "-learl_dispatch", "-Wl,-rpath," + libdir,
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_links_and_validates_without_gpu(tmp_path):
    """A plain C program compiles against include/earl_dispatch.h, links libearl_dispatch.so
    and gets the documented status codes for invalid arguments (no GPU involved)."""
    exe = _build_c_smoke(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "no-GPU checks passed" in r.stdout


@pytest.mark.gpu
def test_c_program_dispatches_on_gpu(tmp_path):
    """The same C program plans and executes BASELINE configs[0] through the C ABI alone and
    checks bytes, cu_seqlens, stats and the exported plan against tests/golden/c1_tiny.json."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = _build_c_smoke(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GPU dispatch checks passed" in r.stdout


def test_ptr_array_marshals_once():
    """earl.PtrArray: the pointer array is built once and passed through unchanged; None and 0
    entries become NULL, ints pass as addresses, tensors as their data pointers."""
    import torch
    t = torch.zeros(4, dtype=torch.uint8)
    pa = earl.PtrArray([t, None, 0x1000, 0])
    assert len(pa) == 4
    arr = earl._ptr_array(pa)
    assert arr is pa.arr and earl._ptr_array(pa) is arr
    assert [arr[k] for k in range(4)] == [t.data_ptr(), None, 0x1000, None]
    fresh = earl._ptr_array([t, None, 0x1000, 0])
    assert [fresh[k] for k in range(4)] == [arr[k] for k in range(4)]
