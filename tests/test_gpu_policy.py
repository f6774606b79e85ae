"""GPU: the worst-case policies of SURVEY.md 8(f) row f1 and the K8 fallback.

Reference: momqms always takes the median of the floor(n/3) triple medians
(sort.hpp:52-57, selection.hpp:219-229); hqms switches to it for one step after
a pivot outside [delta n, (1-delta) n] (pivot_outside_band, sort.hpp:114-118,
160-172).  On the GPU the pivot choice is a splitter sample: mom_of_thirds
samples strided triple medians (no seed) at every level, hybrid re-samples a bucket
that came out larger than (parent / buckets) / delta, and after max_levels
partition levels the remaining buckets are merge-sorted (guaranteed
O(n log n) work).  Every policy must return the oracle's bytes.
"""
import numpy as np
import pytest

import paper_1804_10062_b200 as q
from oracle_lib import DT_F64, DT_I64, DT_REC32, DT_U32, DT_U64
from test_gpu_parity import gpu_sort, rand_input

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [DT_U32, DT_U64, DT_F64, DT_REC32, DT_I64])
@pytest.mark.parametrize("dist", ["uniform", "fewdistinct", "organpipe", "sorted"])
def test_momqms_triple_median_sampling(oracle, dt, dist):
    """mom_of_thirds takes no random positions; the first level's split (of the
    caller's arrangement) is therefore identical under any seed.  Deeper levels
    sample buckets whose internal order depends on scatter timing, so only the
    result is compared there."""
    a = rand_input(dt, 600000, seed=11, dist=dist)
    firsts = []
    for seed in (1, 2):
        cfg = q.momqms()
        cfg.seed = seed
        got, m = gpu_sort(a, cfg)
        np.testing.assert_array_equal(got, oracle.sort(dt, a))
        cfg.max_levels = 1  # stop after level 1; the rest is merge-sorted
        cfg.profile = True
        got, m1 = gpu_sort(a, cfg)
        np.testing.assert_array_equal(got, oracle.sort(dt, a))
        firsts.append((m1.phase_bytes[5], m1.phase_bytes[6], m1.phase_bytes[7]))
    assert firsts[0] == firsts[1]  # same buckets: same block-sort / merge / fill volume


@pytest.mark.parametrize("dt", [DT_U32, DT_U64, DT_REC32])
def test_hybrid_resplits_buckets_outside_the_band(oracle, dt):
    n = (1 << 24) if dt == DT_U32 else (1 << 22)  # two partition levels: children exist
    a = rand_input(dt, n, seed=5)
    got, m = gpu_sort(a, q.hqms())
    np.testing.assert_array_equal(got, oracle.sort(dt, a))
    assert m.resplits == 0  # delta = 1/16: random samples never leave the band
    cfg = q.hqms()
    cfg.delta = 1.0  # band = the expected bucket size: about half the buckets leave it
    got, m = gpu_sort(a, cfg)
    np.testing.assert_array_equal(got, oracle.sort(dt, a))
    assert m.resplits > 0
    cfg = q.qms()
    cfg.delta = 1.0  # median_of_3 never re-splits
    _, m = gpu_sort(a, cfg)
    assert m.resplits == 0


@pytest.mark.parametrize("pivot", list(q.PivotStrategy))
@pytest.mark.parametrize("dt", [DT_U32, DT_F64, DT_REC32])
def test_every_pivot_strategy(oracle, pivot, dt):
    for dist in ("uniform", "reverse", "allequal"):
        a = rand_input(dt, 250000, seed=int(pivot), dist=dist)
        cfg = q.qms()
        cfg.pivot = pivot
        got, _ = gpu_sort(a, cfg)
        np.testing.assert_array_equal(got, oracle.sort(dt, a))


@pytest.mark.parametrize("dt", [DT_U32, DT_U64, DT_REC32])
@pytest.mark.parametrize("max_levels", [1, 2])
def test_merge_fallback_after_max_levels(oracle, dt, max_levels):
    """K8: buckets still too large after max_levels are merge-sorted."""
    # needs two partition levels (even splitters leave 512 buckets of exactly
    # n / 512 keys on this uniform input: beyond 512 block-sort tiles)
    n = {DT_U32: 12 << 20, DT_U64: 6 << 20}.get(dt, 3 << 20)
    a = rand_input(dt, n, seed=max_levels)
    cfg = q.qms()
    cfg.max_levels = max_levels
    got, m = gpu_sort(a, cfg)
    np.testing.assert_array_equal(got, oracle.sort(dt, a))
    if max_levels == 1:
        assert m.merge_passes >= 1 and m.levels == 1
