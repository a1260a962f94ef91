"""CPU-side checks of the C ABI boundary (no compute calls, no GPU needed):
liblms.so builds for sm_100a, loads, and exports every symbol include/lms.h
declares; the binding wraps exactly that set; the product path never imports
the oracle."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lms.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lms_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    syms = declared_symbols()
    for name in ["lms_build_csr", "lms_order", "lms_permute", "lms_smooth"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_1606_00803_b200 import _lms, build_lib
    path = build_lib.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", path]).decode()
    exported = set(re.findall(r"\bT (lms_[a-z0-9_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert sorted(_lms.EXPORTS) == declared_symbols()
    lib = _lms.load_library()                      # dlopen works without a GPU
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a():
    from paper_1606_00803_b200 import build_lib
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build_lib.build()]).decode()
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1606_00803_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "oracle.c" not in txt and "liboracle" not in txt, f


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_1606_00803_b200 as lms
    with pytest.raises(Exception):
        lms.Mesh.build_csr([torch.zeros(3, dtype=torch.float64)] * 2, torch.zeros((1, 3), dtype=torch.int32))


def test_set_allocator_arguments():
    """lms_set_allocator: exactly one hook NULL is LMS_E_ARG; (NULL, NULL)
    restores the default allocator (no device work, so it runs on CPU)."""
    import ctypes as ct
    import paper_1606_00803_b200 as lms
    L = lms.lib()
    cb = ct.CFUNCTYPE(ct.c_void_p, ct.c_size_t, ct.c_void_p, ct.c_void_p)(lambda n, s, c: None)
    assert L.lms_set_allocator(ct.cast(cb, ct.c_void_p), None, None) == -1  # LMS_E_ARG
    assert L.lms_set_allocator(None, None, None) == 0
