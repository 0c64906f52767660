"""The drop-in boundary on CPU: the C-ABI library loads, exports every symbol
include/rcscm_gpu.h declares (and the ctypes table matches the header), fails
loudly without a GPU, and the product package never touches the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rcscm_gpu.h")


def declared_symbols(path):
    text = open(path).read()
    return sorted(set(re.findall(r"\b(rcscm_gpu_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1908_01964_b200 import _capi

    lib = _capi.load()
    syms = declared_symbols(HEADER)
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.SIGNATURES), "ctypes table out of sync with include/rcscm_gpu.h"


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1908_01964_b200", "librcscm_gpu.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    """Without a GPU the context cannot be created: an error, never a CPU fallback."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1908_01964_b200 import CudaError, GpuContext

    with pytest.raises(CudaError):
        GpuContext(0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1908_01964_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|librcscm_oracle|oracle_\w+\(", src, re.M), f


def test_oracle_exports_every_declared_symbol(O):
    lib = ctypes.CDLL(O.build())
    text = open(os.path.join(ROOT, "oracle", "rcscm_oracle.h")).read()
    for s in sorted(set(re.findall(r"\b(oracle_\w+)\s*\(", text))):
        assert hasattr(lib, s), s


def test_cpp_front_end_compiles():
    """include/rcscm_gpu.hpp compiles and links against the C ABI."""
    out = os.path.join(ROOT, "build", "shim_check_cpu")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-o", out,
                        os.path.join(ROOT, "tests", "cpp", "shim_check.cpp"),
                        "-L" + os.path.join(ROOT, "paper_1908_01964_b200"), "-lrcscm_gpu"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
