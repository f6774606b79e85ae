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
    out = torch.empty_like(t)
    counts = torch.zeros(nsplit + 1, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    rc = lib.qmsort_gpu_partition(_lib.DT_U32, t.data_ptr(), t.shape[0], s.data_ptr(), nsplit, out.data_ptr(),
                                  counts.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "qmsort_gpu_partition")
    torch.cuda.synchronize()
    b = np.searchsorted(spl, a, side="left")
    np.testing.assert_array_equal(counts.cpu().numpy(), np.bincount(b, minlength=nsplit + 1))
    got = out.cpu().numpy()
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


def test_emulated_fused_exchange_leaves_input_untouched(oracle):
    a = oracle.gen("f64_gauss", 100000, seed=1)
    shards = shards_of(a, 4)
    before = [t.clone() for t in shards]
    out = sharded.sort_sharded_emulated_fused(shards, "less", dtype=DT_F64)
    assert all(torch.equal(x, y) for x, y in zip(shards, before))
    np.testing.assert_array_equal(np.concatenate([o.cpu().numpy() for o in out]), np.sort(a))


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
            out = sharded.sort_sharded(shard, "less", dtype=DT_U64, exchange=ex, ops=ops)
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
    full, parts = qq.get(timeout=240)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    n = 300000
    for rep, m in enumerate((n, n, 3 * n)):
        got = np.concatenate([parts[r][rep] for r in range(world)])
        np.testing.assert_array_equal(got, np.sort(full[:m * world]))


# ---- the single-process C entry over several (here: repeated) devices ------
@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg,dt", [("u32", DT_U32), ("u64", DT_U64), ("rec32", DT_REC32),
                                    ("f64_gauss", DT_F64), ("f64_distinct16", DT_F64), ("i32", 0)])
def test_c_sort_sharded_matches_oracle(oracle, P, cfg, dt):
    """qmsort_gpu_sort_sharded with devices [0] * P: the same kernels and the
    same peer-store exchange as P GPUs, driven by one host thread per rank."""
    n = (1 << 19) + 777
    if cfg == "i32":
        a = np.random.default_rng(3).integers(-2**31, 2**31, n).astype(np.int32)
    else:
        a = oracle.gen(cfg, n, seed=11)
    shards = shards_of(a, P)
    before = [t.clone() for t in shards]
    out, m = sharded.sort_sharded_devices(shards, [0] * P, "less", dtype=dt)
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, np.sort(a) if cfg == "i32" else oracle.sort(dt, a))
    assert all(torch.equal(x, y) for x, y in zip(shards, before)), "input shards must be read only"
    assert m.kernel_launches > 0 and m.elapsed_ns > 0


@pytest.mark.parametrize("P", [2, 5, 8])
def test_c_sort_sharded_descending_ragged_empty(oracle, P):
    a = oracle.gen("u64", 300001, seed=4)
    cuts = sorted(np.random.default_rng(P).integers(0, a.shape[0], P - 1).tolist())
    parts = np.split(a, cuts)
    if P > 2:
        parts[1] = parts[1][:0]  # an empty shard
    a = np.concatenate(parts)
    shards = [torch.from_numpy(x.copy()).cuda() for x in parts]
    out, _ = sharded.sort_sharded_devices(shards, [0] * P, "greater", dtype=DT_U64)
    got = np.concatenate([o.cpu().numpy() for o in out])
    np.testing.assert_array_equal(got, oracle.sort(DT_U64, a, greater=True))


@pytest.mark.parametrize("path", ["c", "emulated_fused", "emulated_staged"])
def test_sharded_duplicate_heavy_is_balanced(oracle, path):
    """C4c-shaped input (16 distinct values) and a 70 % hot key: the ranks a
    repeated splitter spans share its keys as fills -- no rank takes them all."""
    for a in (oracle.gen("f64_distinct16", 1 << 20, seed=2),
              np.where(np.random.default_rng(1).random(1 << 20) < 0.7, 3.0,
                       np.random.default_rng(2).normal(size=1 << 20))):
        a = a.copy()
        a[a == 0] = 0.0
        P = 8
        shards = shards_of(a, P)
        if path == "c":
            out, _ = sharded.sort_sharded_devices(shards, [0] * P, "less", dtype=DT_F64)
        elif path == "emulated_fused":
            out = sharded.sort_sharded_emulated_fused(shards, "less", dtype=DT_F64)
        else:
            out = sharded.sort_sharded_emulated(shards, "less", dtype=DT_F64)
        got = np.concatenate([o.cpu().numpy() for o in out])
        np.testing.assert_array_equal(got, np.sort(a))
        sizes = [o.shape[0] for o in out]
        assert max(sizes) <= 0.2 * a.shape[0], sizes


def test_c_sort_sharded_errors():
    import ctypes
    lib = _lib.load()
    x = torch.arange(1000, dtype=torch.int64, device="cuda").view(torch.uint64)
    din = (ctypes.c_void_p * 2)(x.data_ptr(), x.data_ptr())
    nin = (ctypes.c_size_t * 2)(1000, 1000)
    dev = (ctypes.c_int * 2)(0, 0)
    small = torch.empty(10, dtype=torch.uint64, device="cuda")
    dout = (ctypes.c_void_p * 2)(small.data_ptr(), small.data_ptr())
    cap = (ctypes.c_size_t * 2)(10, 10)
    on = (ctypes.c_size_t * 2)()
    rc = lib.qmsort_gpu_sort_sharded(DT_U64, 0, 2, dev, din, nin, dout, cap, on, None, None)
    assert rc == _lib.QMSORT_ENOWS and on[0] + on[1] == 2000
    rc = lib.qmsort_gpu_sort_sharded(DT_U64, 0, 9, dev, din, nin, dout, cap, on, None, None)
    assert rc == _lib.QMSORT_EINVAL
    bad = (ctypes.c_int * 2)(0, 99)
    rc = lib.qmsort_gpu_sort_sharded(DT_U64, 0, 2, bad, din, nin, dout, cap, on, None, None)
    assert rc == _lib.QMSORT_EINVAL


@pytest.mark.parametrize("P,cfg", [(2, "c2"), (3, "c5")])
def test_bench_multi_rank_path(tmp_path, P, cfg):
    """bench.py --gpus P: re-launched under torch.distributed.run, P ranks
    (here all on GPU 0, QMSORT_BENCH_ONE_GPU=1, gloo host collectives), the
    folded peer exchange through real IPC handles; rank 0 prints one line with
    n_gpus = P and the cross-rank verification."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QMSORT_BENCH_ONE_GPU="1")
    env.pop("WORLD_SIZE", None)
    args = [sys.executable, os.path.join(root, "bench.py"), "--gpus", str(P), "--steps", "2", "--warmup", "1",
            "--config", cfg]
    if cfg == "c2":
        args += ["--n", str(1 << 22)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == P
    assert line["verify"] == {"order_violations_within_slices": 0, "slices_ordered_across_ranks": True,
                              "multiset_preserved": True}
    assert 7.9 < line["roofline"]["ledger_bytes_over_nw"] < 8.5
