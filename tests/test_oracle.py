"""CPU suite: pin the oracle (C restatement of the reference hot path) against
the reference's own golden vectors and against the reference itself.

Golden data: tests/golden/golden.json, produced by tests/golden/make_golden.py
from the reference compiled unmodified out of /root/reference.  Where the
reference library itself is present (oracle/_ref, this container) the oracle
is also fuzzed against it directly, like test_sort.cpp:59-77.
"""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

from oracle_lib import DT_F64, DT_I32, DT_I64, DT_REC32, DT_U32, DT_U64, ELEM16

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_fig1_worked_example(oracle):
    """Fig. 1 array sorts to 0..11 (test_sort.cpp:24,37-45); the golden file
    holds the reference's output for every preset."""
    a = np.array(GOLDEN["fig1"]["input"], dtype=np.int32)
    for name, expect in GOLDEN["fig1"]["outputs"].items():
        assert expect == list(range(12)), name
    np.testing.assert_array_equal(oracle.sort(DT_I32, a), np.arange(12, dtype=np.int32))
    np.testing.assert_array_equal(oracle.sort(DT_I32, a, pivot=1), np.arange(12, dtype=np.int32))


@pytest.mark.parametrize("case", range(3))
def test_swap_merge_golden(oracle, case):
    """swap_merge restatement reproduces the reference's array byte for byte
    (test_merge.cpp:48-85), including where the displaced dummies land."""
    g = GOLDEN["swap_merge"][case]
    a = np.array(g["input"], dtype=np.int64)
    oracle.lib.qmso_swap_merge_i64(a.ctypes.data_as(ctypes.c_void_p), *g["args"])
    assert a.tolist() == g["output"]


def test_generator_patterns(oracle):
    """SplitMix64 counter form and dataset recipes (rng.hpp:10-38,
    dataset.hpp:62-99; test_dataset.cpp:18-38)."""
    for g in GOLDEN["generators"]:
        if g["kind"] == 3:  # organ-pipe, also the f64 C4e recipe
            x = oracle.gen("f64_organ", g["n"])
            assert x.astype(np.int64).tolist() == g["output"]
    perm = np.empty(1000, np.int64)
    oracle.lib.qmso_gen_perm_i64(perm.ctypes.data_as(ctypes.c_void_p), 1000, 41)
    assert sha(perm) == GOLDEN["random_perm_1000_seed41_sha256"]
    dup = oracle.gen_randomdup_i64(1 << 16, 42, 16)
    assert sha(dup) == GOLDEN["randomdup16_65536_seed42_sha256"]
    # bounded(rng,16) == sm >> 60 (no rejection for powers of two)
    sm = np.array([oracle.sm(42, j) for j in range(1 << 16)], dtype=np.uint64)
    np.testing.assert_array_equal(dup, (sm >> np.uint64(60)).astype(np.int64) + 1)


@pytest.mark.parametrize("key", sorted(GOLDEN["configs"]))
def test_config_shapes_against_reference(oracle, key):
    """Every config shape x seed: our input recipe matches the frozen digest
    and the oracle's sorted output equals the reference qms() / std::sort."""
    g = GOLDEN["configs"][key]
    name, _ = key.split("/")
    a = oracle.gen(name, g["n"], seed=g["seed"])
    assert sha(a) == g["input_sha256"]
    assert g["qms_sha256"] == g["std_sort_sha256"] == g["hqms_sha256"]  # unique sorted order
    assert sha(oracle.sort(g["dtype"], a)) == g["qms_sha256"]
    assert sha(oracle.sort(g["dtype"], a, greater=True)) == g["qms_greater_sha256"]


def test_c1_known_answer(oracle):
    """C1: the sorted permutation of [0,n) is 0..n-1 (closed form)."""
    a = oracle.gen("i32_perm", 1 << 20, seed=42)
    np.testing.assert_array_equal(oracle.sort(DT_I32, a), np.arange(1 << 20, dtype=np.int32))


needs_ref = pytest.mark.skipif(not os.path.exists(os.path.join(
    os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "libqmsref.so")),
    reason="reference library not built (no /root/reference)")


@needs_ref
def test_fuzz_oracle_vs_reference(oracle):
    """Random n < 3000 over the six reference distributions (test_sort.cpp:59-77)."""
    rng = np.random.default_rng(1001)
    for trial in range(120):
        n = int(rng.integers(0, 3000))
        kind = trial % 6
        v = np.empty(max(n, 1), np.int64)
        param = {4: 7, 5: 13}.get(kind, 0)
        oracle.ref.qmsref_generate(kind, param, n, int(rng.integers(0, 2**62)),
                                   v.ctypes.data_as(ctypes.c_void_p))
        v = v[:n]
        for dt, conv in [(DT_I32, np.int32), (DT_U32, np.uint32), (DT_U64, np.uint64), (DT_F64, np.float64),
                         (DT_I64, np.int64)]:
            a = v.astype(conv)
            for greater in (False, True):
                np.testing.assert_array_equal(oracle.sort(dt, a, greater),
                                              oracle.ref_sort(dt, a, greater))


@needs_ref
def test_rec32_oracle_vs_reference(oracle):
    a = oracle.gen("rec32", 50000, seed=9)
    np.testing.assert_array_equal(oracle.sort(DT_REC32, a), oracle.ref_sort(DT_REC32, a))


def test_is_sorted_helper(oracle):
    a = np.array([1, 2, 2, 5], dtype=np.uint32)
    assert oracle.is_sorted(DT_U32, a)
    assert not oracle.is_sorted(DT_U32, a[::-1].copy())
    assert oracle.is_sorted(DT_U32, a[::-1].copy(), greater=True)


def canon_elems(a):
    """Element multiset in canonical (byte-sorted) form."""
    n = a.shape[0]
    return np.sort(np.ascontiguousarray(a).view(np.uint8).reshape(n, 24).view("V24").reshape(n))


@pytest.mark.parametrize("case", range(4))
def test_elements16_golden(oracle, case):
    """Element<16> (element.hpp:13-20): the oracle's qms over the keys gives the
    reference's key sequence; the input recipe and multiset match the frozen
    digests (test_sort.cpp:328-339)."""
    g = GOLDEN["elements16"][case]
    a = oracle.gen_elem16(g["n"], g["seed"])
    assert a.dtype == ELEM16
    assert sha(a) == g["input_sha256"]
    keys = oracle.sort(DT_I64, np.ascontiguousarray(a["key"]), greater=bool(g["greater"]))
    assert sha(keys) == g["keys_sha256"]
    assert sha(canon_elems(a)) == g["multiset_sha256"]


@pytest.mark.parametrize("case", range(8))
def test_select_nth_golden(oracle, case):
    """select_nth (selection.hpp:207-212): the oracle's sorted order puts the
    reference's k-th element at k-1 (test_selection.cpp:101-160)."""
    g = GOLDEN["select_nth"][case]
    a = oracle.gen("i64", g["n"], seed=g["seed"])
    s = oracle.sort(DT_I64, a, greater=bool(g["greater"]))
    assert g["pos"] == g["k"] - 1
    assert int(s[g["k"] - 1]) == g["value"]


@needs_ref
def test_reference_select_partitions(oracle):
    """The reference's select_nth leaves the range partitioned around k-1
    (selection.hpp:124-126) -- the contract the GPU select keeps."""
    rng = np.random.default_rng(5)
    for n in (1, 7, 100, 5000):
        a = rng.integers(-50, 50, n).astype(np.int64)
        for k in (1, (n + 1) // 2, n):
            p, b = oracle.ref_select_nth_i64(a, k)
            assert p == k - 1
            assert (b[:p] <= b[p]).all() and (b[p + 1:] >= b[p]).all()
            np.testing.assert_array_equal(np.sort(b), np.sort(a))
