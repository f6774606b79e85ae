"""Distributed samplesort: exchange logic on CPU.

* world_size 2 and 3 over torch.distributed gloo (127.0.0.1), with the CPU
  doubles of the device ops (tests/sharded_doubles.py);
* P = 1..8 in-process emulation.
Concatenating the per-rank slices in rank order must equal the sorted input.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_10062_b200 import _lib, sharded
from sharded_doubles import NumpyOps


def make(dt, n, seed):
    rng = np.random.default_rng(seed)
    if dt == _lib.DT_I32:
        return rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    if dt == _lib.DT_U32:
        return rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    if dt == _lib.DT_U64:
        return rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2)
    if dt == _lib.DT_F64:
        x = rng.normal(size=n)
        x[x == 0] = 0.0
        return x
    a = rng.integers(0, 2**63, (n, 4), dtype=np.uint64)
    a[:, 0] >>= np.uint64(52)
    return a


def reference_sort(dt, a, greater):
    if dt == _lib.DT_REC32:
        o = a[np.lexsort(a.T[::-1])]
        return o[::-1].copy() if greater else o
    o = np.sort(a, kind="stable")
    return o[::-1].copy() if greater else o


def _wire_dtype(dt):
    return {_lib.DT_I32: torch.int32, _lib.DT_U32: torch.int32}.get(dt, torch.int64)


def _worker(rank, world, port, dt, greater, sizes, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = make(dt, sum(sizes), seed=11)
        off = sum(sizes[:rank])
        shard = torch.from_numpy(full[off:off + sizes[rank]].copy())
        out = sharded.sort_sharded(shard, "greater" if greater else "less", dtype=dt,
                                   exchange=sharded.TorchExchange(), ops=NumpyOps(), oversample=16)
        parts = [None] * world
        dist.all_gather_object(parts, out.numpy())
        if rank == 0:
            got = np.concatenate(parts)
            q.put(bool(np.array_equal(got, reference_sort(dt, full, greater))))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("dt", [_lib.DT_I32, _lib.DT_U32, _lib.DT_U64, _lib.DT_F64, _lib.DT_REC32])
@pytest.mark.parametrize("world,greater", [(2, False), (3, True)])
def test_gloo_world(dt, world, greater):
    sizes = [5000, 3100, 0][:world] if world == 3 else [4000, 2500]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dt, greater, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dt", [_lib.DT_U32, _lib.DT_F64, _lib.DT_REC32])
def test_emulated_ranks(P, dt):
    rng = np.random.default_rng(P)
    sizes = [int(x) for x in rng.integers(0, 3000, P)]
    full = make(dt, sum(sizes), seed=P + 100)
    shards, off = [], 0
    for s in sizes:
        shards.append(torch.from_numpy(full[off:off + s].copy()))
        off += s
    out = sharded.sort_sharded_emulated(shards, "less", dtype=dt, ops=NumpyOps(), oversample=8)
    got = np.concatenate([o.numpy() for o in out])
    np.testing.assert_array_equal(got, reference_sort(dt, full, False))


def test_duplicate_heavy_keys_emulated():
    """16 distinct values (config 4c shape): equal keys all go to one rank."""
    full = (np.random.default_rng(3).integers(0, 16, 20000) + 1).astype(np.float64)
    shards = [torch.from_numpy(x.copy()) for x in np.array_split(full, 4)]
    out = sharded.sort_sharded_emulated(shards, "less", dtype=_lib.DT_F64, ops=NumpyOps())
    np.testing.assert_array_equal(np.concatenate([o.numpy() for o in out]), np.sort(full))


def test_duplicate_heavy_keys_balanced():
    """A value that fills several splitter slots is spread over the ranks it
    spans (fills), so no rank receives every copy of a frequent key."""
    full = np.where(np.random.default_rng(4).random(40000) < 0.7, 5.0,
                    np.random.default_rng(5).normal(size=40000))
    full[full == 0] = 0.0
    shards = [torch.from_numpy(x.copy()) for x in np.array_split(full, 8)]
    out = sharded.sort_sharded_emulated(shards, "less", dtype=_lib.DT_F64, ops=NumpyOps(), oversample=16)
    np.testing.assert_array_equal(np.concatenate([o.numpy() for o in out]), np.sort(full))
    sizes = [o.shape[0] for o in out]
    assert max(sizes) < 0.3 * full.shape[0], sizes


def _plan_random(P, m, rng):
    mult = [1] * m
    for _ in range(P - 1 - m):
        mult[int(rng.integers(0, m))] += 1
    C = rng.integers(0, 50, (P, 2 * m + 1))
    return mult, C


@pytest.mark.parametrize("P", [1, 2, 5, 8])
def test_plan_tiles_every_receive_buffer(P):
    """qmsort_gpu_shard_plan: sender s's bin b occupies [bin_off[s][b],
    bin_off[s][b] + C[s][b]) of rank bin_rank[b]'s buffer; the pieces tile
    [0, recv_n[r]) in sender order, and each rank's slice (fills + received)
    covers the global order exactly once."""
    rng = np.random.default_rng(P)
    for trial in range(20):
        m = int(rng.integers(0 if P == 1 else 1, P)) if P > 1 else 0
        mult, C = _plan_random(P, m, rng)
        pl = sharded.plan(P, mult, C)
        br, bo = pl["bin_rank"], pl["bin_off"]
        for r in range(P):
            pos = 0
            for s_ in range(P):
                for b in range(2 * m + 1):
                    if br[b] == r:
                        assert bo[s_][b] == pos
                        pos += C[s_][b]
            assert pos == pl["recv_n"][r]
        # global order: bin b's keys (all senders) precede bin b+1's
        total = int(C.sum())
        assert int((pl["recv_n"] + pl["lo_fill"] + pl["hi_fill"]).sum()) == total
        for j in range(m):
            e = int(C[:, 2 * j + 1].sum())
            if mult[j] >= 2:
                assert br[2 * j + 1] == -1
                shares = [int(pl["hi_fill"][r]) for r in range(P) if pl["hi_val"][r] == j] + \
                         [int(pl["lo_fill"][r]) for r in range(P) if pl["lo_val"][r] == j]
                assert sum(shares) == e and max(shares) - min(shares) <= 1
            else:
                assert br[2 * j + 1] == br[2 * j]
        assert list(br[::2]) == sorted(br[::2])


def test_splitters_merge_duplicates():
    smp = np.array([1, 1, 1, 1, 1, 1, 7, 9], dtype=np.uint32)  # quantiles at 1,2,...,7 of 8 for P=8
    uniq, mult = sharded.splitters(_lib.DT_U32, smp, 8)
    assert uniq.view(np.uint32).tolist() == [1, 7, 9] and mult == [5, 1, 1]
    uniq, mult = sharded.splitters(_lib.DT_U32, smp, 1)
    assert uniq.size == 0 and mult == []


def _folded_random(P, rng):
    K0 = sharded.subbuckets(_lib.DT_U64, P, 1 << 30)
    S = P * K0 - 1
    m = int(rng.integers(1, S + 1))
    mult = [1] * m
    for _ in range(S - m):
        mult[int(rng.integers(0, m))] += 1
    C = rng.integers(0, 40, (P, 2 * m + 1))
    return K0, mult, C


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_folded_plan_is_every_ranks_level_zero(P):
    """qmsort_gpu_shard_plan_folded: every key lands exactly once -- open bins
    sent to one rank at disjoint offsets inside that rank's own bin list,
    equal-key bins never sent but filled in even shares -- and each rank's
    local bins alternate open / equal with counts summing to its slice."""
    rng = np.random.default_rng(P + 7)
    for _ in range(30):
        K0, mult, C = _folded_random(P, rng)
        m = len(mult)
        pl = sharded.plan_folded(P, K0, mult, C)
        br, bo, out_n = pl["bin_rank"], pl["bin_off"], pl["out_n"]
        assert int(out_n.sum()) == int(C.sum())
        assert all(br[2 * j + 1] == -1 for j in range(m))
        assert list(br[::2]) == sorted(br[::2])
        for r in range(P):
            lm = int(pl["loc_m"][r])
            cnt = pl["loc_cnt"][r][:2 * lm + 1].astype(np.int64)
            assert int(cnt.sum()) == int(out_n[r])
            starts = np.concatenate([[0], np.cumsum(cnt)])
            # the open bins routed here tile their local bins, senders in order
            covered = np.zeros(int(out_n[r]), dtype=np.int64)
            for j in range(m + 1):
                if br[2 * j] != r:
                    continue
                for s_ in range(P):
                    a = int(bo[s_][2 * j])
                    covered[a:a + int(C[s_][2 * j])] += 1
            eq_slots = sum(int(cnt[2 * k + 1]) for k in range(lm))
            assert int(covered.sum()) + eq_slots == int(out_n[r])
            assert covered.max(initial=0) <= 1
            # local values are increasing global indices
            lu = pl["loc_uniq"][r][:lm]
            assert list(lu) == sorted(lu) and len(set(lu)) == lm
        # equal keys: every global value's total is split, never lost
        for j in range(m):
            tot = int(C[:, 2 * j + 1].sum())
            got = sum(int(pl["loc_cnt"][r][2 * k + 1]) for r in range(P)
                      for k in range(int(pl["loc_m"][r])) if pl["loc_uniq"][r][k] == j)
            assert got == tot
