"""CPU suite: the C-ABI library loads, exports every symbol include/qmsort_gpu.h
declares, mirrors the reference presets, and fails loudly (status codes, no
CPU fallback) -- no compute call needs a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1804_10062_b200 as q
from paper_1804_10062_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qmsort_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(qmsort_gpu_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), f"{n} declared in qmsort_gpu.h but not exported"
    assert set(_lib.EXPORTED) <= set(names)


def test_struct_layouts_match_header():
    # GpuConfig / GpuMetrics mirror the C structs compiled into the library
    lib = ctypes.CDLL(_lib.LIB_PATH)
    cb, mb = ctypes.c_size_t(), ctypes.c_size_t()
    lib.qmsort_gpu_abi_sizes(ctypes.byref(cb), ctypes.byref(mb))
    assert ctypes.sizeof(_lib.GpuConfig) == cb.value
    assert ctypes.sizeof(_lib.GpuMetrics) == mb.value


def test_presets_mirror_sortconfig():
    """qms/qmqs/momqms/hqms (sort.hpp:37-66) and SortConfig defaults (25-34)."""
    lib = _lib.load()
    for variant, pivot, kind, thr, lv in [(0, 0, 1, 10, 0), (1, 0, 2, 16, 1), (2, 2, 1, 10, 0), (3, 3, 1, 10, 0)]:
        c = _lib.GpuConfig()
        lib.qmsort_gpu_config_init(ctypes.byref(c), variant)
        assert (c.variant, c.pivot, c.base_case_kind, c.base_case_size_threshold,
                c.base_case_use_levels) == (variant, pivot, kind, thr, lv)
        assert c.beta == 0.5 and c.delta == 1.0 / 16.0 and c.block == 128 and c.side == 1
    # the Python mirror builds the same C struct
    for py, variant in [(q.qms, 0), (q.qmqs, 1), (q.momqms, 2), (q.hqms, 3)]:
        c = py().to_c()
        ref = _lib.GpuConfig()
        lib.qmsort_gpu_config_init(ctypes.byref(ref), variant)
        for f, _ in _lib.GpuConfig._fields_:
            if f not in ("seed", "max_levels", "profile", "algorithm"):
                assert getattr(c, f) == getattr(ref, f), f


def test_dtype_helpers_and_workspace():
    lib = _lib.load()
    assert [lib.qmsort_gpu_dtype_size(d) for d in range(6)] == [4, 4, 8, 8, 32, 8]
    assert lib.qmsort_gpu_dtype_size(9) == 0
    assert [lib.qmsort_gpu_core_dtype(d) for d in range(6)] == [1, 1, 2, 2, 4, 2]
    # f3 / f4 workspaces: records + Rec32 samplesort + gathered elements; select
    we = lib.qmsort_gpu_elements_workspace_bytes(1 << 20, 24)
    assert we >= (1 << 20) * (32 + 32 + 24)
    assert lib.qmsort_gpu_select_workspace_bytes(5, 1 << 20) > lib.qmsort_gpu_workspace_bytes(5, 1 << 20, None)
    w1 = lib.qmsort_gpu_workspace_bytes(1, 1 << 20, None)
    w2 = lib.qmsort_gpu_workspace_bytes(1, 1 << 24, None)
    assert (1 << 20) * 4 <= w1 < w2
    assert lib.qmsort_gpu_workspace_bytes(4, 1 << 20, None) >= (1 << 20) * 32
    assert b"sm_100a" in lib.qmsort_gpu_version()


def test_invalid_arguments_are_rejected_before_any_cuda_call():
    lib = _lib.load()
    buf = (ctypes.c_uint32 * 4)()
    c = _lib.GpuConfig()
    lib.qmsort_gpu_config_init(ctypes.byref(c), 0)
    assert lib.qmsort_gpu_sort(7, 0, ctypes.addressof(buf), 4, ctypes.byref(c), None, 0, None, None) == _lib.QMSORT_EINVAL
    assert b"dtype" in lib.qmsort_gpu_last_error()
    assert lib.qmsort_gpu_sort(1, 5, ctypes.addressof(buf), 4, ctypes.byref(c), None, 0, None, None) == _lib.QMSORT_EINVAL
    assert lib.qmsort_gpu_sort(1, 0, None, 4, ctypes.byref(c), None, 0, None, None) == _lib.QMSORT_EINVAL
    assert lib.qmsort_gpu_sort(1, 0, ctypes.addressof(buf), 1 << 32, ctypes.byref(c), None, 0, None, None) == _lib.QMSORT_EINVAL
    assert lib.qmsort_gpu_partition(0, ctypes.addressof(buf), 4, None, 5, None, None, None, 0, None) == _lib.QMSORT_EINVAL
    assert lib.qmsort_gpu_generate(99, ctypes.addressof(buf), 4, 0, 0, 0, None) == _lib.QMSORT_EINVAL
    # elements: bad element size / misaligned key / record keys; select: k out of range
    sz = ctypes.c_size_t(0)
    for args in [(5, 2, 24, 0), (5, 0, 22, 0), (5, 0, 24, 4), (4, 0, 64, 0), (5, 0, 8, 4)]:
        kd, cm, eb, ko = args
        assert lib.qmsort_gpu_sort_elements_host(kd, cm, ctypes.addressof(buf), 2, eb, ko, None, None) == _lib.QMSORT_EINVAL, args
    for k in (0, 5):
        assert lib.qmsort_gpu_select_nth_host(1, 0, ctypes.addressof(buf), 4, k, ctypes.byref(sz), None, None) == _lib.QMSORT_EINVAL
        assert lib.qmsort_gpu_select_nth(1, 0, ctypes.addressof(buf), 4, k, ctypes.byref(sz), None, None, 0, None, None) == _lib.QMSORT_EINVAL
    assert b"1-based" in lib.qmsort_gpu_last_error()
    assert lib.qmsort_gpu_sort_host_batch(1, 0, None, None, 2, None, None) == _lib.QMSORT_EINVAL
    assert lib.qmsort_gpu_sort_host_batch(1, 0, None, None, 0, None, None) == _lib.QMSORT_OK
    with pytest.raises(ValueError):
        q.sort(np.zeros(4, np.int16))
    with pytest.raises(ValueError):
        q.sort(np.zeros(4, np.uint32), less="unknown")


def test_empty_and_singleton_are_noops_without_device():
    """n <= 1 costs nothing (test_sort.cpp:47-57) -- no device touched."""
    a = np.array([], dtype=np.uint32)
    m = q.sort(a)
    assert m.elapsed_ns == 0
    b = np.array([42], dtype=np.uint32)
    q.sort(b)
    assert b.tolist() == [42]


def test_no_cpu_fallback_without_gpu():
    """On a GPU-less host the product path must fail loudly, never sort on the CPU."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    a = np.arange(100, 0, -1).astype(np.uint32)
    with pytest.raises(q.QmsortError) as e:
        q.sort(a)
    assert e.value.code == _lib.QMSORT_ECUDA
    assert a[0] == 100  # untouched


def test_product_package_does_not_reference_the_oracle():
    """Only tests/, smoke() and bench.py's CPU legs may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_1804_10062_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "liboracle" not in text and "qmso_" not in text and "qmsref" not in text, f
