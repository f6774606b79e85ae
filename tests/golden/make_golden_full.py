"""Full-size golden digests: SHA-256 of the REFERENCE's sorted output for every
BASELINE.json config at its full size (seed 42), computed once here with the
reference compiled from /root/reference (oracle/_ref).  The GPU tests hash the
device output and compare -- bit-exact parity at full size without running the
CPU sort on the GPU box.

    python tests/golden/make_golden_full.py <config> ...   (one process per config)
    python tests/golden/make_golden_full.py --merge        (collect into golden_full.json)
"""
import glob
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import DT_F64, DT_I32, DT_REC32, DT_U32, DT_U64, Oracle  # noqa: E402

FULL = {  # name: (n, dtype, reference routine)
    "i32_perm": (1 << 20, DT_I32, "qms"), "u32": (1 << 28, DT_U32, "qms"),
    "u64": (1 << 30, DT_U64, "std"), "f64_sorted": (1 << 27, DT_F64, "qms"),
    "f64_reverse": (1 << 27, DT_F64, "qms"), "f64_distinct16": (1 << 27, DT_F64, "qms"),
    "f64_gauss": (1 << 27, DT_F64, "qms"), "f64_organ": (1 << 27, DT_F64, "qms"),
    "rec32": (1 << 26, DT_REC32, "qms"),
}


def sha(a):
    h = hashlib.sha256()
    mv = memoryview(np.ascontiguousarray(a)).cast("B")
    for i in range(0, len(mv), 1 << 28):
        h.update(mv[i:i + (1 << 28)])
    return h.hexdigest()


# more seeds at full size (BASELINE.md parity seeds {42, 1, 2}) and C3 through
# the reference's own qms() (the "u64" entry uses std::sort; the sorted order
# is unique, so the digests must agree)
EXTRA = {"u32@1": ("u32", 1, None), "u32@2": ("u32", 2, None), "rec32@1": ("rec32", 1, None),
         "rec32@2": ("rec32", 2, None), "u64@qms": ("u64", 42, "qms")}


def one(key):
    name, seed, how_over = EXTRA.get(key, (key, 42, None))
    n, dt, how = FULL[name]
    how = how_over or how
    o = Oracle()
    a = o.gen(name, n, seed=seed)
    rec = {"n": n, "dtype": dt, "seed": seed, "config": name, "input_sha256": sha(a), "routine": how}
    t = time.time()
    b = o.ref_sort(dt, a, use_std=(how == "std"))
    rec["cpu_seconds"] = time.time() - t
    rec["sorted_sha256"] = sha(b)
    os.makedirs("/tmp/fullgold", exist_ok=True)
    json.dump(rec, open(f"/tmp/fullgold/{key}.json", "w"))
    print(key, rec["cpu_seconds"])


if __name__ == "__main__":
    if sys.argv[1:] == ["--merge"]:
        old = json.load(open(os.path.join(HERE, "golden_full.json")))
        out = dict(old)
        out.update({os.path.basename(p)[:-5]: json.load(open(p)) for p in glob.glob("/tmp/fullgold/*.json")})
        json.dump(out, open(os.path.join(HERE, "golden_full.json"), "w"), indent=1)
        print(sorted(out))
    else:
        for name in sys.argv[1:]:
            one(name)
