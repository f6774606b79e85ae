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


BAD_REC_CMP = r"""
#include <algorithm>
#include <vector>
#include "qmsort_gpu.hpp"
struct Rec { std::uint64_t w[4]; };
namespace qmsort::gpu { template <> struct is_rec32<Rec> : std::true_type {}; }
struct ByLastWord { bool operator()(const Rec& a, const Rec& b) const { return a.w[3] < b.w[3]; } };
int main() {
    std::vector<Rec> r(10);
    qmsort::gpu::sort(r.begin(), r.end(), qmsort::gpu::qms(), ByLastWord{});
}
"""


def test_shim_rejects_an_undeclared_record_comparator(tmp_path):
    """A record comparator the GPU cannot run is a compile error, never a silent
    substitution of the lexicographic order."""
    src = tmp_path / "bad.cpp"
    src.write_text(BAD_REC_CMP)
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode != 0 and "rec32_order" in r.stderr


def test_shim_cpp17_compiles():
    """The header also builds as C++17 (contiguity from pointer / std::vector iterators)."""
    src = os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp")
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
