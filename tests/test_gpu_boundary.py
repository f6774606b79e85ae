"""GPU: the boundary rows of SURVEY.md 8(a) beyond qmsort::sort itself --
PartitionResult (partition_result.hpp:12-17) as a three-way partition around a
pivot value, the Median-of-sqrt(n) sample size of median_of_sqrt_pivot
(partition.hpp:235-251), beta as the block-sort takeover size
(base_case_levels, sort.hpp:91-96), and sort_range_counted (sort.hpp:207-211)."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1804_10062_b200 as q
from oracle_lib import DT_F64, DT_I32, DT_REC32, DT_U32, DT_U64

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_full.json")))


def rec_key(a):
    return [tuple(r) for r in a.tolist()]


@pytest.mark.parametrize("cfg,dt", [("u32", DT_U32), ("u64", DT_U64), ("f64_gauss", DT_F64),
                                    ("f64_distinct16", DT_F64), ("rec32", DT_REC32)])
@pytest.mark.parametrize("less", ["less", "greater"])
@pytest.mark.parametrize("where", ["device", "host"])
def test_partition_three_way(oracle, cfg, dt, less, where):
    n = 300007
    a = oracle.gen(cfg, n, seed=5)
    pivot = a[n // 3].copy()
    x = torch.from_numpy(a.copy()).cuda() if where == "device" else a.copy()
    pr = q.partition(x, pivot, less, dtype=dt)
    got = x.cpu().numpy() if where == "device" else x
    if dt == DT_REC32:
        keys, pv = rec_key(got), tuple(pivot.tolist())
        lt = [k < pv for k in keys] if less == "less" else [k > pv for k in keys]
        eq = [k == pv for k in keys]
    else:
        lt = (got < pivot) if less == "less" else (got > pivot)
        eq = got == pivot
    lt, eq = np.asarray(lt), np.asarray(eq)
    assert pr.lt_end == int(lt.sum()) and pr.gt_begin - pr.lt_end == int(eq.sum())
    assert pr.left_size == pr.lt_end and pr.right_size == n - pr.gt_begin
    assert lt[:pr.lt_end].all() and eq[pr.lt_end:pr.gt_begin].all()
    assert not (lt[pr.gt_begin:] | eq[pr.gt_begin:]).any()
    srt = oracle.sort(dt, a)
    np.testing.assert_array_equal(oracle.sort(dt, got), srt)  # a permutation of the input


def test_partition_edge_cases():
    for a, p in ((np.zeros(0, np.int32), 1), (np.array([5], np.int32), 5), (np.full(1000, 7, np.int32), 7),
                 (np.arange(1000, dtype=np.int32), -1), (np.arange(1000, dtype=np.int32), 5000)):
        b = a.copy()
        pr = q.partition(b, p)
        assert pr.lt_end == int((a < p).sum()) and pr.gt_begin == int((a <= p).sum())
        assert sorted(b.tolist()) == sorted(a.tolist())


def _sha(t) -> str:
    h = hashlib.sha256()
    mv = memoryview(np.ascontiguousarray(t.cpu().numpy())).cast("B")
    for i in range(0, len(mv), 1 << 28):
        h.update(mv[i:i + (1 << 28)])
    return h.hexdigest()


@pytest.mark.slow
def test_median_of_sqrt_n_draws_the_reference_sample_size():
    """C2 at 2^28: median_of_3 draws 32 K keys per segment; median_of_sqrt_n
    draws the reference's s = 2 floor(sqrt(n)/2) + 1 = 16385 strided keys at
    level 0 (sorted by the host path: more than one block sort) and
    2 floor(sqrt(len)/2) + 1 per later segment -- different samples, the same
    bit-exact output (the reference digest)."""
    g = GOLD["u32"]
    n = g["n"]
    x = torch.empty(n, dtype=torch.uint32, device="cuda")
    q.generate(q.GEN_U32, x, seed=g["seed"])
    y = x.clone()
    m3 = q.sort(x, q.qms())
    assert _sha(x) == g["sorted_sha256"]
    cfg = q.qms()
    cfg.pivot = q.PivotStrategy.median_of_sqrt_n
    ms = q.sort(y, cfg)
    assert _sha(y) == g["sorted_sha256"]
    assert m3.sample_keys != ms.sample_keys
    assert ms.sample_keys >= 16385  # level 0 alone
    # level 0 of median_of_3 draws min(8192, 32 * 256) keys
    assert m3.sample_keys % 8192 == 0 or m3.sample_keys > 8192


@pytest.mark.parametrize("dt,cfgname", [(DT_U32, "u32"), (DT_U64, "u64"), (DT_REC32, "rec32"),
                                        (DT_F64, "f64_organ")])
def test_median_of_sqrt_n_bit_exact(oracle, dt, cfgname):
    for n in (10000, 1 << 20, (1 << 22) + 3):
        a = oracle.gen(cfgname, n, seed=9)
        x = torch.from_numpy(a.copy()).cuda()
        cfg = q.qms()
        cfg.pivot = q.PivotStrategy.median_of_sqrt_n
        m = q.sort(x, cfg)
        np.testing.assert_array_equal(x.cpu().numpy(), oracle.sort(dt, a))
        if n > 16384:
            assert m.sample_keys > 0


def test_beta_is_the_block_sort_takeover_size(oracle):
    """qmqs (base_case.use_levels): buckets of about n^beta go to the block
    sorter; a smaller beta means more partition levels, same output."""
    n = 1 << 22
    a = oracle.gen("u32", n, seed=3)
    ref = oracle.sort(DT_U32, a)
    levels = []
    for beta in (0.75, 0.5):  # n^beta = 2^16.5 -> the 16384-key cap; 2^11 = 2048
        cfg = q.qmqs()
        cfg.beta = beta
        x = torch.from_numpy(a.copy()).cuda()
        m = q.sort(x, cfg)
        np.testing.assert_array_equal(x.cpu().numpy(), ref)
        levels.append(m.levels)
    assert levels[1] > levels[0], levels
    # beta is ignored without use_levels (the qms preset): same plan as default
    cfg = q.qms()
    cfg.beta = 0.5
    x = torch.from_numpy(a.copy()).cuda()
    assert q.sort(x, cfg).levels == q.sort(torch.from_numpy(a.copy()).cuda(), q.qms()).levels


def test_sort_range_counted_accumulates(oracle):
    a = np.random.default_rng(1).integers(-2**31, 2**31, 1 << 20).astype(np.int32)
    x = torch.from_numpy(a.copy()).cuda()
    m = q.Metrics()
    q.sort_range_counted(x, q.qms(), m)
    t1 = m.elapsed_ns
    x2 = torch.from_numpy(a.copy()).cuda()
    q.sort_range_counted(x2, q.qms(), m)
    assert t1 > 0 and m.elapsed_ns > t1 and m.comparisons == 0
    np.testing.assert_array_equal(x.cpu().numpy(), np.sort(a))
    assert q.dtype_of(x) == DT_I32
