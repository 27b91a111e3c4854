"""CPU-side checks of the drop-in boundary: the C-ABI library loads (no GPU
needed to dlopen it) and exports every entry point include/hood_b200.h
declares; the C++ header compiles as the reference's callers would use it;
the product path never touches oracle/ and fails loudly without its library."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hood_b200.h")
PKG = os.path.join(ROOT, "paper_1203_5004_b200")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(hood_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1203_5004_b200 import build as B
    B.build()
    return ctypes.CDLL(B.SO)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["hood_create", "hood_destroy", "hood_build_f32", "hood_build_f64", "hood_build_host_f32",
              "hood_build_host_f64", "hood_merge_segments_f64", "hood_last_error"]:
        assert s in syms, s


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_lists_every_export():
    from paper_1203_5004_b200 import hood as H
    assert sorted(H.EXPORTS) == declared_symbols()


def test_cpu_safe_entry_points(lib):
    lib.hood_abi_version.restype = ctypes.c_int
    assert lib.hood_abi_version() == 1
    lib.hood_status_string.restype = ctypes.c_char_p
    assert b"increasing" in lib.hood_status_string(2).lower()


def test_create_without_gpu_reports_cuda_error(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = ctypes.c_void_p()
    rc = lib.hood_create(ctypes.byref(ctx), 0)
    assert rc == 5  # HOOD_ERR_CUDA: no silent CPU path


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cpp_header_compiles(tmp_path):
    for src in [os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")]:
        subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        "-I", os.path.join(ROOT, "include"), src], check=True)
    c = tmp_path / "c_abi.c"
    c.write_text('#include "hood_b200.h"\nint main(void) { return hood_abi_version() == 1 ? 0 : 1; }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                    str(c)], check=True)


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), f
                assert "hood_oracle" not in txt and "libhoodref" not in txt, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_1203_5004_b200 import hood as H
    monkeypatch.setattr(H, "SO", str(tmp_path / "absent.so"))
    monkeypatch.setattr(H, "_lib", None)
    with pytest.raises(ImportError):
        H.library()
