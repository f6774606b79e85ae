"""GPU: the sharded samplesort building blocks with the real sm_100a kernels.

P ranks are emulated in one process on one GPU (the exchange is done with
tensor slicing; no kernel waits on another), so the device ops -- transform,
seeded sample, partition by splitters, local sort -- run exactly as on each
rank of a multi-GPU job.  Parity: the concatenated slices equal the CPU oracle.
"""
import numpy as np
import pytest

import paper_1804_10062_b200 as q
from paper_1804_10062_b200 import _lib, sharded
from oracle_lib import DT_F64, DT_REC32, DT_U32, DT_U64

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def shards_of(a, P):
    return [torch.from_numpy(x.copy()).cuda() for x in np.array_split(a, P)]


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("cfg,dt", [("u32", DT_U32), ("u64", DT_U64), ("rec32", DT_REC32),
                                    ("f64_gauss", DT_F64), ("f64_distinct16", DT_F64)])
def test_emulated_sharded_matches_oracle(oracle, P, cfg, dt):
    n = 1 << 20
    a = oracle.gen(cfg, n, seed=42)
    out = sharded.sort_sharded_emulated(shards_of(a, P), "less", dtype=dt)
    torch.cuda.synchronize()
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, oracle.sort(dt, a))


@pytest.mark.parametrize("P", [3, 8])
def test_emulated_sharded_descending(oracle, P):
    a = oracle.gen("u64", 300000, seed=5)
    out = sharded.sort_sharded_emulated(shards_of(a, P), "greater", dtype=DT_U64)
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, oracle.sort(DT_U64, a, greater=True))


def test_c3_shard_generation_is_rank_independent(oracle):
    """C3 recipe: shard r of P generates global indices [r n/P, (r+1) n/P)."""
    n, P = 1 << 18, 4
    full = oracle.gen("u64", n, seed=42)
    parts = []
    for r in range(P):
        t = torch.empty(n // P, dtype=torch.uint64, device="cuda")
        q.generate(q.GEN_U64, t, seed=42, start=r * (n // P), total=n)
        parts.append(t.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(parts), full)


@pytest.mark.parametrize("nsplit", [1, 7, 255])
def test_partition_by_splitters(nsplit):
    rng = np.random.default_rng(nsplit)
    a = rng.integers(0, 2**32, 200000, dtype=np.uint64).astype(np.uint32)
    spl = np.sort(rng.integers(0, 2**32, nsplit, dtype=np.uint64).astype(np.uint32))
    t = torch.from_numpy(a).cuda()
    s = torch.from_numpy(spl).cuda()
    out, counts = sharded.GpuOps().partition(t.view(torch.int32), _lib.DT_U32, s.view(torch.int32))
    torch.cuda.synchronize()
    b = np.searchsorted(spl, a, side="left")
    np.testing.assert_array_equal(counts.cpu().numpy(), np.bincount(b, minlength=nsplit + 1))
    got = out.cpu().numpy().view(np.uint32)
    off = 0
    for j, c in enumerate(counts.cpu().numpy()):
        np.testing.assert_array_equal(np.sort(got[off:off + c]), np.sort(a[b == j]))
        off += c


# ---- the exchange fused into the partition's scatter (peer stores) ----------
@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg,dt", [("u32", DT_U32), ("u64", DT_U64), ("rec32", DT_REC32),
                                    ("f64_distinct16", DT_F64)])
def test_emulated_fused_exchange_matches_oracle(oracle, P, cfg, dt):
    """Every rank's scatter kernel stores its bucket j straight into rank j's
    receive buffer (qmsort_gpu_partition_scatter_peers); no exchange copy."""
    n = (1 << 20) + 12345
    a = oracle.gen(cfg, n, seed=7)
    out = sharded.sort_sharded_emulated_fused(shards_of(a, P), "less", dtype=dt)
    torch.cuda.synchronize()
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, oracle.sort(dt, a))


def test_emulated_fused_exchange_descending_and_ragged(oracle):
    a = oracle.gen("u64", 200001, seed=3)
    shards = [torch.from_numpy(x.copy()).cuda() for x in (a[:5], a[5:150000], a[150000:150000], a[150000:])]
    out = sharded.sort_sharded_emulated_fused(shards, "greater", dtype=DT_U64)
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, oracle.sort(DT_U64, a, greater=True))


def _peer_worker(rank, world, port, n, seed, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = np.random.default_rng(seed).integers(0, 2**63, 3 * n * world, dtype=np.uint64)
        ex = sharded.PeerExchange()
        ops = sharded.GpuOps()
        res = []
        # call 2 reuses the opened peer buffers; call 3 has 3x the keys, so every
        # rank grows its receive buffer and the handles are swapped again
        for rep, m in enumerate((n, n, 3 * n)):
            shard = torch.from_numpy(full[rank * m:(rank + 1) * m].copy()).cuda()
            out = sharded.sort_sharded(shard, "less", dtype=DT_U64, exchange=ex, ops=ops,
                                       force_exchange=True)
            res.append(out.cpu().numpy().copy())
            ex.barrier()
        parts = [None] * world
        dist.all_gather_object(parts, res)
        if rank == 0:
            q.put((full, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_peer_exchange_processes(world):
    """One process per rank (here all on GPU 0): receive buffers exported with
    qmsort_gpu_ipc_handle, opened by the peers, written by the peers' scatter
    kernels.  Host collectives over gloo; no kernel waits on another."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, 300000, 9, qq)) for r in range(world)]
    for p in procs:
        p.start()
    full, parts = qq.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    n = 300000
    for rep, m in enumerate((n, n, 3 * n)):
        got = np.concatenate([parts[r][rep] for r in range(world)])
        np.testing.assert_array_equal(got, np.sort(full[:m * world]))
