"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/pbicgstab.h declares, rejects bad arguments before touching the
device, and reports a missing device instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "pbicgstab.h")).read()
    return sorted(set(re.findall(r"\b(pbicgstab_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    from paper_1809_01948_b200 import binding
    return binding.lib()


def test_library_exports_every_header_symbol(L):
    from paper_1809_01948_b200 import _build
    syms = header_symbols()
    assert len(syms) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\b(pbicgstab_\w+)\b", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(L, s)


def test_binding_declares_every_symbol():
    from paper_1809_01948_b200 import binding
    assert sorted(binding.SYMBOLS) == header_symbols()


def test_sm100a_code_present():
    from paper_1809_01948_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_rejected_without_device(L):
    from paper_1809_01948_b200 import binding
    h = ctypes.c_void_p()
    st = binding._Stencil(4, 10, 10, 10, (ctypes.c_double * 7)(4, -1, -1, -1, -1, 0, 0))
    assert L.pbicgstab_create_stencil(ctypes.byref(st), 1, None, None, ctypes.byref(h)) == 1
    assert b"dim" in L.pbicgstab_last_error(None)
    st = binding._Stencil(2, 10, 10, 1, (ctypes.c_double * 7)(0, -1, -1, -1, -1, 0, 0))
    assert L.pbicgstab_create_stencil(ctypes.byref(st), 1, None, None, ctypes.byref(h)) == 1
    assert L.pbicgstab_create_stencil(None, 1, None, None, ctypes.byref(h)) == 1
    assert L.pbicgstab_solve(None, None, None, 0.0, 1, 0, None, None, None, None, None) == 1
    L.pbicgstab_destroy(None)  # no-op


def test_no_cpu_fallback_without_device(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_1809_01948_b200 import binding
    h = ctypes.c_void_p()
    st = binding._Stencil(2, 10, 10, 1, (ctypes.c_double * 7)(4, -1, -1, -1, -1, 0, 0))
    assert L.pbicgstab_create_stencil(ctypes.byref(st), 1, None, None, ctypes.byref(h)) == 2
    assert not h.value


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1809_01948_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*|\"\"\"[\s\S]*?\"\"\"", "", txt), f
