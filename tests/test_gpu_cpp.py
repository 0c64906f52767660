"""The C++ front end (include/rcscm_gpu.hpp) run on the GPU: the compiled
reference-style call site tests/cpp/shim_check.cpp must exit 0."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_shim_runs():
    exe = os.path.join(ROOT, "build", "shim_check")
    if not os.path.exists(exe):
        subprocess.run(["g++", "-std=c++17", "-O1", "-o", exe, os.path.join(ROOT, "tests", "cpp", "shim_check.cpp"),
                        "-L" + os.path.join(ROOT, "paper_1908_01964_b200"), "-lrcscm_gpu",
                        "-Wl,-rpath," + os.path.join(ROOT, "paper_1908_01964_b200")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim_check" in r.stdout
