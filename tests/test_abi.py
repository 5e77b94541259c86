"""CPU checks of the C-ABI boundary: the in-tree library loads and exports
every entry point include/ttdvm_cuda.h declares (no compute without a GPU),
and the product package never imports the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ttdvm_cuda.h")).read()
    return sorted(set(re.findall(r"\b(ttdvm_cuda_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_1912_04582_b200.cuda import EXPORTS
    assert header_symbols() == sorted(EXPORTS)


def test_library_exports_every_symbol():
    from paper_1912_04582_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1912_04582_b200.cuda import Context
    with pytest.raises(RuntimeError):
        Context(0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1912_04582_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
