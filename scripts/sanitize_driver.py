"""Small-size workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every dtype and comparator through every kernel path -- the
samplesort levels, the packed 16-bit and record-prefix block sorts, equal-key
buckets and fills, the merge fallback and mergesort passes, key + payload
elements, select_nth, the three-way partition and the sharded exchange --
each result checked against numpy.  Run by scripts/sanitize.sh on the GPU box."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_10062_b200 as q  # noqa: E402
from paper_1804_10062_b200 import sharded  # noqa: E402

SIZES = [int(x) for x in os.environ.get("SAN_SIZES", "1000,40000,150007").split(",")]
rng = np.random.default_rng(7)
fails = 0


def check(name, got, want):
    global fails
    if not np.array_equal(got, want):
        fails += 1
        print("FAIL", name, flush=True)


def gen(dt, n, kind):
    if dt == "rec32":
        a = rng.integers(0, 2**63, (n, 4), dtype=np.uint64)
        a[:, 0] >>= np.uint64(52 if kind == "uniform" else 62)
        return a
    if kind == "narrow":
        base = rng.integers(0, 2**20)
        a = base + rng.integers(0, 3000, n)
    elif kind == "dup":
        a = rng.integers(0, 16, n)
    else:
        a = rng.integers(0, 2**62, n)
    return {"i32": lambda x: (x % 2**32 - 2**31).astype(np.int32),
            "u32": lambda x: (x % 2**32).astype(np.uint32),
            "u64": lambda x: x.astype(np.uint64) * np.uint64(3),
            "i64": lambda x: x.astype(np.int64) - 2**61,
            "f64": lambda x: (x.astype(np.float64) - 2**61) / 7.0}[dt](a)


def ref(a, greater):
    if a.ndim == 2:
        o = a[np.lexsort(a.T[::-1])]
    else:
        o = np.sort(a, kind="stable")
    return o[::-1].copy() if greater else o


for n in SIZES:
    for dt in ("i32", "u32", "u64", "i64", "f64", "rec32"):
        for kind in ("uniform", "narrow", "dup"):
            if dt == "rec32" and kind == "narrow":
                continue
            a = gen(dt, n, kind)
            for greater in (False, True):
                for cfgname in ("qms", "hqms", "sqrt", "merge"):
                    cfg = {"qms": q.qms(), "hqms": q.hqms(), "sqrt": q.qms(), "merge": q.qms()}[cfgname]
                    if cfgname == "sqrt":
                        cfg.pivot = q.PivotStrategy.median_of_sqrt_n
                    if cfgname == "merge":
                        cfg.algorithm = q.Algorithm.mergesort
                    x = torch.from_numpy(a.copy()).cuda()
                    q.sort(x, cfg, "greater" if greater else "less")
                    check(f"sort {dt} {kind} n={n} greater={greater} {cfgname}", x.cpu().numpy(), ref(a, greater))
            # max_levels = 1: the merge fallback of oversized buckets
            cfg = q.qms()
            cfg.max_levels = 1
            x = torch.from_numpy(a.copy()).cuda()
            q.sort(x, cfg)
            check(f"fallback {dt} {kind} n={n}", x.cpu().numpy(), ref(a, False))
            if dt != "rec32" and n > 1:
                k = n // 3 + 1
                x = torch.from_numpy(a.copy()).cuda()
                p = q.select_nth(x, k)
                check(f"select {dt} {kind} n={n}", x.cpu().numpy()[p:p + 1], ref(a, False)[k - 1:k])
                pv = a[n // 2]
                x = torch.from_numpy(a.copy()).cuda()
                pr = q.partition(x, pv)
                got = x.cpu().numpy()
                check(f"partition {dt} {kind} n={n}", np.array([pr.lt_end, pr.gt_begin]),
                      np.array([(a < pv).sum(), (a <= pv).sum()]))
                check(f"partition-multiset {dt} {kind} n={n}", np.sort(got), np.sort(a))
            # the sharded exchange (P ranks on this GPU): Python path and the C entry
            for P in (3,):
                shards = [torch.from_numpy(s.copy()).cuda() for s in np.array_split(a, P)]
                out = sharded.sort_sharded_emulated_fused(shards, "less")
                check(f"sharded {dt} {kind} n={n}", np.concatenate([o.cpu().numpy() for o in out]), ref(a, False))
                out, _ = sharded.sort_sharded_devices(shards, [0] * P, "less")
                check(f"sharded-c {dt} {kind} n={n}", np.concatenate([o.cpu().numpy() for o in out]), ref(a, False))
    # key + payload elements
    el = np.zeros(n, dtype=[("key", "<i8"), ("payload", "V16")])
    el["key"] = rng.integers(-50, 50, n)
    e = el.copy()
    q.sort_elements(e)
    check(f"elements n={n}", e["key"], np.sort(el["key"], kind="stable"))
torch.cuda.synchronize()
print("sanitize driver done, failures:", fails, flush=True)
sys.exit(1 if fails else 0)
