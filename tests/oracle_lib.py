"""ctypes wrapper of the CPU parity checker (oracle/liboracle.so and, when
built, the reference itself in oracle/_ref/libqmsref.so).  TEST
INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and bench.py's
CPU baseline / reference legs."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libqmsref.so")

DT_I32, DT_U32, DT_U64, DT_F64, DT_REC32, DT_I64 = 0, 1, 2, 3, 4, 5
NP_DTYPE = {DT_I32: np.int32, DT_U32: np.uint32, DT_U64: np.uint64, DT_F64: np.float64,
            DT_I64: np.int64}
# Element<16> (element.hpp:13-20): int64 key + 16 opaque payload bytes, 24 bytes
ELEM16 = np.dtype([("key", "<i8"), ("payload", "V16")])


def _vp(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
        self.lib = ctypes.CDLL(ORACLE_SO)
        L = self.lib
        L.qmso_sort.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
        L.qmso_sm.restype = ctypes.c_uint64
        L.qmso_sm.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.qmso_is_sorted.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
        for name in ("qmso_gen_u32_uniform", "qmso_gen_u64_uniform", "qmso_gen_rec32"):
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64]
        L.qmso_gen_f64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int]
        L.qmso_gen_perm_i64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64]
        L.qmso_gen_randomdup_i64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64]
        L.qmso_swap_merge_i64.argtypes = [ctypes.c_void_p] + [ctypes.c_size_t] * 4
        self.ref = None
        if os.path.exists(REF_SO):
            self.ref = ctypes.CDLL(REF_SO)
            self.ref.qmsref_sort.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_size_t,
                                                                  ctypes.c_void_p]
            self.ref.qmsref_generate.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t,
                                                 ctypes.c_uint64, ctypes.c_void_p]
            self.ref.qmsref_swap_merge_i64.argtypes = [ctypes.c_void_p] + [ctypes.c_size_t] * 4
            self.ref.qmsref_sort_elem16.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
            self.ref.qmsref_select_nth_i64.argtypes = [ctypes.c_void_p, ctypes.c_size_t,
                                                       ctypes.c_size_t, ctypes.c_int]
            self.ref.qmsref_select_nth_i64.restype = ctypes.c_size_t

    # --- sorting -------------------------------------------------------
    def sort(self, dt: int, a: np.ndarray, greater: bool = False, pivot: int = 0) -> np.ndarray:
        """Restated QuickMergesort (qms preset) on a copy of a."""
        b = np.ascontiguousarray(a).copy()
        n = b.shape[0]
        rc = self.lib.qmso_sort(dt, int(greater), pivot, _vp(b), n)
        assert rc == 0
        return b

    def ref_sort(self, dt: int, a: np.ndarray, greater: bool = False, variant: int = 0,
                 use_std: bool = False) -> np.ndarray:
        """The reference qmsort::sort itself (oracle/_ref), when built."""
        assert self.ref is not None
        b = np.ascontiguousarray(a).copy()
        m = (ctypes.c_uint64 * 4)()
        rc = self.ref.qmsref_sort(dt, int(greater), variant, 0, int(use_std), _vp(b), b.shape[0], m)
        assert rc == 0
        return b

    def ref_sort_elem16(self, a: np.ndarray, greater: bool = False) -> np.ndarray:
        """The reference qmsort::sort over Element<16> (qms preset)."""
        assert self.ref is not None and a.dtype == ELEM16
        b = np.ascontiguousarray(a).copy()
        assert self.ref.qmsref_sort_elem16(_vp(b), b.shape[0], int(greater)) == 0
        return b

    def ref_select_nth_i64(self, a: np.ndarray, k: int, greater: bool = False) -> tuple[int, np.ndarray]:
        """The reference select_nth (selection.hpp:207-212): (position, rearranged copy)."""
        assert self.ref is not None
        b = np.ascontiguousarray(a, dtype=np.int64).copy()
        p = int(self.ref.qmsref_select_nth_i64(_vp(b), b.shape[0], k, int(greater)))
        return p, b

    def is_sorted(self, dt: int, a: np.ndarray, greater: bool = False) -> bool:
        return self.lib.qmso_is_sorted(dt, int(greater), _vp(np.ascontiguousarray(a)), a.shape[0]) == 1

    # --- generators ----------------------------------
    def sm(self, seed: int, j: int) -> int:
        return int(self.lib.qmso_sm(seed, j))

    def gen(self, cfg: str, n: int, seed: int = 42, start: int = 0) -> np.ndarray:
        L = self.lib
        if cfg == "u32":
            a = np.empty(n, np.uint32); L.qmso_gen_u32_uniform(_vp(a), n, seed, start); return a
        if cfg == "u64":
            a = np.empty(n, np.uint64); L.qmso_gen_u64_uniform(_vp(a), n, seed, start); return a
        if cfg == "i64":  # full-range signed keys: the u64 recipe reinterpreted
            a = np.empty(n, np.uint64); L.qmso_gen_u64_uniform(_vp(a), n, seed, start)
            return a.view(np.int64)
        if cfg == "rec32":
            a = np.empty((n, 4), np.uint64); L.qmso_gen_rec32(_vp(a), n, seed, start); return a
        if cfg.startswith("f64"):
            kind = {"f64_sorted": 0, "f64_reverse": 1, "f64_distinct16": 2, "f64_gauss": 3,
                    "f64_organ": 4}[cfg]
            a = np.empty(n, np.float64); L.qmso_gen_f64(_vp(a), n, seed, kind); return a
        if cfg == "i32_perm":
            v = np.empty(n, np.int64); L.qmso_gen_perm_i64(_vp(v), n, seed)
            return (v - 1).astype(np.int32)
        raise ValueError(cfg)

    def gen_elem16(self, n: int, seed: int, key_range: int = 64) -> np.ndarray:
        """Element<16> inputs: keys in [-key_range/2, key_range/2) (many
        duplicates, like test_sort.cpp:330-334), 16 seeded payload bytes."""
        out = np.empty(n, ELEM16)
        j = np.arange(n, dtype=np.uint64)
        k = np.array([self.sm(seed, 3 * int(i)) for i in j], dtype=np.uint64)
        out["key"] = (k % np.uint64(key_range)).astype(np.int64) - key_range // 2
        pay = np.empty((n, 2), np.uint64)
        pay[:, 0] = [self.sm(seed, 3 * int(i) + 1) for i in j]
        pay[:, 1] = [self.sm(seed, 3 * int(i) + 2) for i in j]
        out["payload"] = pay.view("V16").reshape(n)
        return out

    def gen_randomdup_i64(self, n: int, seed: int, m: int) -> np.ndarray:
        v = np.empty(n, np.int64)
        self.lib.qmso_gen_randomdup_i64(_vp(v), n, seed, m)
        return v
