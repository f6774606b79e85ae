"""Randomised GPU stress (seeded, reproducible): dtype x comparator x preset x
size x value distribution drawn at random, each sort checked byte-for-byte
against the CPU oracle -- the reference's own fuzz (test_sort.cpp:59-77,
acceptance.cpp:86-114) at sizes that exercise one and two partition levels,
the packed 16-bit and record-prefix block sorts, the fused transform and the
few-bin scatter."""
import os

import numpy as np
import pytest

import paper_1804_10062_b200 as q
from oracle_lib import DT_F64, DT_I32, DT_I64, DT_REC32, DT_U32, DT_U64
from test_gpu_parity import gpu_sort

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PRESETS = [q.qms, q.qmqs, q.momqms, q.hqms]


def _draw(rng, dt, n):
    kind = rng.integers(0, 6)
    w = (n, 4) if dt == DT_REC32 else (n,)
    if kind == 0:  # full range
        raw = rng.integers(0, 2**63, size=w, dtype=np.uint64) * 2 + rng.integers(0, 2, size=w, dtype=np.uint64)
    elif kind == 1:  # narrow range (packed block sort territory)
        raw = rng.integers(0, int(rng.integers(2, 1 << 20)), size=w, dtype=np.uint64) + np.uint64(rng.integers(0, 1 << 40))
    elif kind == 2:  # few distinct
        vals = rng.integers(0, 2**63, size=int(rng.integers(1, 40)), dtype=np.uint64)
        raw = vals[rng.integers(0, len(vals), size=w)]
    elif kind == 3:  # sorted runs
        raw = np.sort(rng.integers(0, 2**40, size=w, dtype=np.uint64), axis=0)
        if rng.integers(0, 2):
            raw = raw[::-1].copy()
    elif kind == 4:  # skew: most keys in a small window
        raw = rng.integers(0, 2**62, size=w, dtype=np.uint64)
        m = rng.random(w) < 0.9
        raw[m] = rng.integers(1000, 1100, size=int(m.sum()), dtype=np.uint64)
    else:  # organ pipe
        i = np.arange(n, dtype=np.uint64)
        raw = np.minimum(i + 1, np.uint64(n) - i)
        if dt == DT_REC32:
            raw = np.repeat(raw[:, None], 4, axis=1)
    if dt == DT_I32:
        return (raw & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    if dt == DT_U32:
        return (raw & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    if dt == DT_U64:
        return raw.astype(np.uint64)
    if dt == DT_I64:
        return raw.astype(np.uint64).view(np.int64)
    if dt == DT_F64:
        x = ((raw >> np.uint64(11)).astype(np.int64) - (1 << 51)).astype(np.float64) * 3.0e-5
        x[x == 0] = 0.0
        return x
    r = raw.astype(np.uint64).copy()
    if kind == 0:
        r[:, 0] >>= np.uint64(52)
    return r


# QMSORT_STRESS_CASES / QMSORT_STRESS_SEED widen the sweep for one-off runs
_CASES = int(os.environ.get("QMSORT_STRESS_CASES", "120"))
_SEED = int(os.environ.get("QMSORT_STRESS_SEED", "1000"))


@pytest.mark.parametrize("case", range(_CASES))
def test_random_sorts(oracle, case):
    rng = np.random.default_rng(_SEED + case)
    dt = [DT_I32, DT_U32, DT_U64, DT_F64, DT_REC32, DT_I64][int(rng.integers(0, 6))]
    cap = 1 << 21 if dt == DT_REC32 else 1 << 23
    n = int(min(cap, 2 ** rng.uniform(0, 23)))
    a = _draw(rng, dt, n)
    greater = bool(rng.integers(0, 2))
    preset = PRESETS[int(rng.integers(0, 4))]()
    got, _ = gpu_sort(a, preset, "greater" if greater else "less")
    np.testing.assert_array_equal(got, oracle.sort(dt, a, greater=greater))


@pytest.mark.parametrize("case", range(max(1, _CASES // 3)))
def test_random_elements(oracle, case):
    """Key + payload elements (f3): random element size, key type/offset,
    distribution and comparator; keys must equal the oracle's key sequence and
    the arrangement the stable one."""
    rng = np.random.default_rng(_SEED + 7919 + case)
    key_dt = [DT_I32, DT_U32, DT_U64, DT_F64, DT_I64][int(rng.integers(0, 5))]
    kw = 4 if key_dt in (DT_I32, DT_U32) else 8
    eb = int(rng.choice([kw, 8, 16, 24, 32, 48, 64]))
    eb = max(eb, kw)
    key_off = int(rng.integers(0, (eb - kw) // kw + 1)) * kw
    n = int(min(1 << 20, 2 ** rng.uniform(0, 20)))
    k = _draw(rng, key_dt, n)
    raw = rng.integers(0, 256, size=(n, eb), dtype=np.uint8)
    raw[:, key_off:key_off + kw] = np.ascontiguousarray(k).view(np.uint8).reshape(n, kw)
    less = "greater" if rng.integers(0, 2) else "less"
    t = torch.from_numpy(raw.copy()).cuda()
    q.sort_elements(t, key_dt, q.qms(), less, key_offset=key_off)
    got = t.cpu().numpy()
    np_dt = {DT_I32: np.int32, DT_U32: np.uint32, DT_U64: np.uint64, DT_F64: np.float64, DT_I64: np.int64}[key_dt]
    keys = got[:, key_off:key_off + kw].copy().view(np_dt).reshape(-1)
    np.testing.assert_array_equal(keys, oracle.sort(key_dt, k, greater=(less == "greater")))
    if less == "greater":
        _, inv = np.unique(k, return_inverse=True)
        order = np.argsort(-inv, kind="stable")
    else:
        order = np.argsort(k, kind="stable")
    np.testing.assert_array_equal(got, raw[order])


@pytest.mark.parametrize("case", range(max(1, _CASES // 3)))
def test_random_select_nth(oracle, case):
    """select_nth (f4): random dtype, size, distribution, rank and comparator;
    the k-th element equals the oracle's sorted[k-1] and the range is
    partitioned around it."""
    rng = np.random.default_rng(_SEED + 104729 + case)
    dt = [DT_I32, DT_U32, DT_U64, DT_F64, DT_I64][int(rng.integers(0, 5))]
    n = int(min(1 << 21, 2 ** rng.uniform(0, 21))) or 1
    a = _draw(rng, dt, n)
    greater = bool(rng.integers(0, 2))
    k = int(rng.integers(1, n + 1))
    t = torch.from_numpy(a.copy()).cuda()
    p = q.select_nth(t, k, "greater" if greater else "less")
    b = t.cpu().numpy()
    s = oracle.sort(dt, a, greater=greater)
    assert p == k - 1
    np.testing.assert_array_equal(b[p:p + 1].view(np.uint8), s[k - 1:k].view(np.uint8))
    np.testing.assert_array_equal(np.sort(b.view(np.uint8).reshape(n, -1).view(f"V{b.itemsize}").reshape(n)),
                                  np.sort(a.view(np.uint8).reshape(n, -1).view(f"V{a.itemsize}").reshape(n)))
    left, right = b[:p], b[p + 1:]
    if greater:
        assert (left.size == 0 or not (left < b[p]).any()) and (right.size == 0 or not (right > b[p]).any())
    else:
        assert (left.size == 0 or not (left > b[p]).any()) and (right.size == 0 or not (right < b[p]).any())


@pytest.mark.parametrize("case", range(max(1, _CASES // 6)))
def test_random_sharded_fused(oracle, case):
    """The distributed samplesort with the exchange fused into the scatter
    (peer stores), P ranks emulated on one GPU: random P, dtype, ragged shard
    sizes, distribution and comparator; the concatenated slices equal the
    oracle's sort of the whole array."""
    from paper_1804_10062_b200 import sharded
    rng = np.random.default_rng(_SEED + 15485863 + case)
    dt = [DT_I32, DT_U32, DT_U64, DT_F64, DT_REC32, DT_I64][int(rng.integers(0, 6))]
    P = int(rng.integers(1, 9))
    n = int(min(1 << 21, 2 ** rng.uniform(4, 21)))
    a = _draw(rng, dt, n)
    cuts = np.sort(rng.integers(0, n + 1, size=P - 1))
    bounds = [0, *cuts.tolist(), n]
    shards = [torch.from_numpy(np.ascontiguousarray(a[bounds[i]:bounds[i + 1]])).cuda() for i in range(P)]
    greater = bool(rng.integers(0, 2))
    out = sharded.sort_sharded_emulated_fused(shards, "greater" if greater else "less", dtype=dt)
    torch.cuda.synchronize()
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, oracle.sort(dt, a, greater=greater))
