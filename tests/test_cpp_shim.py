"""The C++ drop-in header (include/qmsort_gpu.hpp): compiles against the
library (CPU) and sorts like qmsort::sort on a B200 (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "build", "shim_demo")


def test_shim_header_compiles_and_links():
    src = os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp")
    out = "/tmp/qmsort_shim_compile_check"
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src,
                        "-L", os.path.join(ROOT, "paper_1804_10062_b200"), "-l:libqmsort_gpu.so", "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_shim_demo_runs_on_gpu():
    assert os.path.exists(DEMO), "build() compiles build/shim_demo"
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "shim ok" in r.stdout, r.stdout + r.stderr
