"""Debug helper: skewed inputs (frac of keys in a window of `width` values,
the rest spread over [0, 2^bits)) -- one sort per process invocation."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1804_10062_b200 as q
dt, n, frac, width, bits, seed = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
rng = np.random.default_rng(seed)
raw = rng.integers(0, 2**bits, size=n, dtype=np.uint64)
m = rng.random(n) < frac
raw[m] = rng.integers(1000, 1000 + width, size=int(m.sum()), dtype=np.uint64)
a = raw.astype(np.uint32) if dt == "u32" else raw
t = torch.from_numpy(a.copy()).cuda()
try:
    mm = q.sort(t, q.qms()); torch.cuda.synchronize()
    ok = np.array_equal(t.cpu().numpy(), np.sort(a))
    print(dt, n, frac, width, bits, "ok" if ok else "WRONG", "levels", mm.levels)
except Exception as e:
    print(dt, n, frac, width, bits, "ERROR", str(e)[:80])
