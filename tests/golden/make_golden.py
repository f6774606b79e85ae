"""Regenerate tests/golden/golden.json from the REFERENCE itself.

Runs the unmodified reference QuickMergesort (compiled from /root/reference by
oracle/Makefile into oracle/_ref/libqmsref.so) on the reference's own worked
examples and on seeded inputs of every BASELINE.json config shape, and
freezes the results (small arrays verbatim, large ones as SHA-256 digests).
The GPU box has no /root/reference; the committed JSON travels instead.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import DT_F64, DT_I32, DT_I64, DT_REC32, DT_U32, DT_U64, Oracle  # noqa: E402

N_CFG = 1 << 16
SEEDS = [42, 1, 2]
CONFIGS = {
    "i32_perm": DT_I32, "u32": DT_U32, "u64": DT_U64, "f64_sorted": DT_F64, "f64_reverse": DT_F64,
    "f64_distinct16": DT_F64, "f64_gauss": DT_F64, "f64_organ": DT_F64, "rec32": DT_REC32,
    "i64": DT_I64,
}
# select_nth cases (selection.hpp:207-212; test_selection.cpp:101-160): n, k, seed, greater
SELECT_CASES = [(6, 1, 0, 0), (101, 51, 1, 0), (1000, 1, 2, 0), (1000, 1000, 3, 0),
                (4096, 2048, 4, 0), (4096, 17, 5, 1), (65536, 30000, 6, 0), (65536, 65536, 7, 1)]
VARIANTS = {"qms": 0, "qmqs": 1, "momqms": 2, "hqms": 3}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    o = Oracle()
    if o.ref is None:
        raise SystemExit("oracle/_ref/libqmsref.so is not built (needs /root/reference)")
    ref = o.ref
    out: dict = {"generated_by": "tests/golden/make_golden.py (reference qmsort compiled from "
                                 "/root/reference/proj/core/include)"}

    # Fig. 1 worked example under every preset (reference test_sort.cpp:24,37-45)
    fig = np.array([7, 11, 4, 5, 6, 10, 9, 2, 3, 1, 0, 8], dtype=np.int64)
    out["fig1"] = {"input": fig.tolist(), "outputs": {}}
    for name, var in VARIANTS.items():
        b = fig.copy()
        ref.qmsref_sort(5, 0, var, 0, 0, b.ctypes.data_as(ctypes.c_void_p), b.shape[0], None)
        out["fig1"]["outputs"][name] = b.tolist()

    # swap_merge examples (reference test_merge.cpp:48-85)
    cases = [([3, 5, 100, 101, 2, 4], (0, 2, 2, 6)), ([7, 1, 2, 3], (1, 1, 1, 4)),
             ([9, 10, 8, 11, 2, 3, 4, 7, 0, 1, 5, 6], (8, 12, 0, 7))]
    out["swap_merge"] = []
    for arr, (b1, e1, t, te) in cases:
        a = np.array(arr, dtype=np.int64)
        ref.qmsref_swap_merge_i64(a.ctypes.data_as(ctypes.c_void_p), b1, e1, t, te)
        out["swap_merge"].append({"input": arr, "args": [b1, e1, t, te], "output": a.tolist()})

    # generator patterns and replay (reference test_dataset.cpp:18-38)
    gens = []
    for kind, param, n, seed in [(1, 0, 4, 0), (2, 0, 4, 0), (3, 0, 6, 0), (3, 0, 5, 0), (4, 3, 7, 0)]:
        v = np.empty(n, np.int64)
        ref.qmsref_generate(kind, param, n, seed, v.ctypes.data_as(ctypes.c_void_p))
        gens.append({"kind": kind, "param": param, "n": n, "seed": seed, "output": v.tolist()})
    out["generators"] = gens
    perm = np.empty(1000, np.int64)
    ref.qmsref_generate(0, 0, 1000, 41, perm.ctypes.data_as(ctypes.c_void_p))
    dup = np.empty(N_CFG, np.int64)
    ref.qmsref_generate(5, 16, N_CFG, 42, dup.ctypes.data_as(ctypes.c_void_p))
    out["random_perm_1000_seed41_sha256"] = sha(perm)
    out["randomdup16_65536_seed42_sha256"] = sha(dup)

    # seeded config shapes: input digest (our recipe) and the
    # reference qms() / std::sort output digests, ascending and descending
    cfgs = {}
    for name, dt in CONFIGS.items():
        for seed in SEEDS:
            a = o.gen(name, N_CFG, seed=seed)
            rec = {"n": N_CFG, "seed": seed, "dtype": dt, "input_sha256": sha(a)}
            rec["qms_sha256"] = sha(o.ref_sort(dt, a))
            rec["std_sort_sha256"] = sha(o.ref_sort(dt, a, use_std=True))
            rec["hqms_sha256"] = sha(o.ref_sort(dt, a, variant=3))
            rec["qms_greater_sha256"] = sha(o.ref_sort(dt, a, greater=True))
            cfgs[f"{name}/{seed}"] = rec
    out["configs"] = cfgs

    # Element<16> (element.hpp:13-20; test_sort.cpp:328-339): the reference's key
    # sequence and element multiset (its arrangement of equal keys is its own)
    elems = []
    for n, seed, greater in [(100, 8, 0), (2000, 9, 0), (2000, 10, 1), (1 << 14, 11, 0)]:
        a = o.gen_elem16(n, seed)
        r = o.ref_sort_elem16(a, greater=bool(greater))
        canon = np.sort(r.view(np.uint8).reshape(n, 24).view("V24").reshape(n))
        elems.append({"n": n, "seed": seed, "greater": greater, "input_sha256": sha(a),
                      "keys_sha256": sha(np.ascontiguousarray(r["key"])),
                      "multiset_sha256": sha(canon)})
    out["elements16"] = elems

    sel = []
    for n, k, seed, greater in SELECT_CASES:
        a = o.gen("i64", n, seed=seed)
        p, b = o.ref_select_nth_i64(a, k, greater=bool(greater))
        sel.append({"n": n, "k": k, "seed": seed, "greater": greater, "pos": p,
                    "value": int(b[p])})
    out["select_nth"] = sel

    # CLI harness: kCsvHeader / to_csv (trial.hpp:62-77)
    # and the per-trial input streams of `bench` (qmsort.cpp:51-53, 112-113)
    ref.qmsref_mix_seed.restype = ctypes.c_uint64
    ref.qmsref_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    ref.qmsref_csv.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t,
                               ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int]
    buf = ctypes.create_string_buffer(512)
    ref.qmsref_csv(buf, 512, b"", 0, b"", 0, 0, 0, 0, 0, 0, 0.0, 0.0, 1)
    cli = {"header": buf.value.decode(), "lines": [], "trial_inputs": []}
    for fields in [("gpu", 65536, "random", 1, 0, 0, 0, 1234567, 2, -16.0, 0.0),
                   ("gpu-hqms", 1000, "fewdistinct:8", 7, 3, 0, 0, 99, 1, -9.965784284662087, 0.0),
                   ("qms", 2, "randomdup:64", 18446744073709551615, 9, 1, 0, 5, 0, 0.0, 0.5)]:
        a, n, d, sd, t, c, mv, tm, dep, lin, rat = fields
        ref.qmsref_csv(buf, 512, a.encode(), n, d.encode(), sd, t, c, mv, tm, dep, lin, rat, 0)
        cli["lines"].append({"fields": list(fields), "csv": buf.value.decode()})
    for dist, kind, param, n, seed, t in [("random", 0, 0, 1000, 1, 0), ("random", 0, 0, 65536, 1, 2),
                                          ("randomdup:64", 5, 64, 5000, 3, 1),
                                          ("fewdistinct:8", 4, 8, 777, 1, 0),
                                          ("organpipe", 3, 0, 1001, 1, 0)]:
        ts = int(ref.qmsref_mix_seed(seed, n * 1000003 + t))
        v = np.empty(n, np.int64)
        ref.qmsref_generate(kind, param, n, ts, v.ctypes.data_as(ctypes.c_void_p))
        cli["trial_inputs"].append({"dist": dist, "n": n, "seed": seed, "trial": t,
                                    "trial_seed": ts, "sha256": sha(v)})
    out["cli"] = cli
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {len(cfgs)} config records")


if __name__ == "__main__":
    main()
