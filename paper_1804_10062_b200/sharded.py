"""Distributed samplesort across the GPUs of one node.

The array is sharded: rank r holds n_r keys.  One sort call
  1. draws ``oversample * P`` seeded sample keys per rank, mapped into the
     unsigned core key domain (``qmsort_gpu_shard_sample``),
  2. all-gathers the samples; every rank sorts the same P*s keys and picks the
     same P-1 global splitters, merged into distinct values with
     multiplicities (``qmsort_gpu_shard_splitters``, host),
  3. classifies and counts its keys three-way against them on the GPU
     (``qmsort_gpu_shard_count``: bin 2j = keys between splitters j-1 and j,
     2j+1 = keys equal to splitter j),
  4. all-gathers the P x (2m+1) count matrix and computes the exchange plan
     (``qmsort_gpu_shard_plan``, host, identical on every rank): each bin's
     rank and offset in that rank's receive buffer; keys equal to a splitter
     value that repeats are not sent -- the ranks that value spans fill their
     even share of it (duplicate-heavy input stays balanced),
  5. exchanges the keys: by default the exchange IS the partition's scatter
     (``qmsort_gpu_shard_scatter`` stores every bin straight into its rank's
     receive buffer, peer memory mapped through CUDA IPC, over NVLink); the
     baseline alternative scatters into a local staging buffer grouped by rank
     and runs one NCCL all-to-all,
  6. sorts the received keys into a fresh output between its fills
     (``qmsort_gpu_shard_finish``).
Rank r's result is the r-th slice of the global order; concatenating the
slices in rank order gives the sorted array.  The input shards are only read.

The same C functions drive the single-process entry over several devices
(``qmsort_gpu_sort_sharded``, :func:`sort_sharded_devices`).  The exchange is
expressed against a small interface so the same code runs over
``torch.distributed`` (NCCL or IPC between GPUs, gloo for the CPU tests) and
over an in-process emulation of P ranks on one GPU.  The per-rank compute ops
(``GpuOps``) are the C-ABI kernels; tests substitute CPU doubles
(tests/sharded_doubles.py) to exercise the exchange logic without a GPU.
"""
from __future__ import annotations

import ctypes
from typing import Any, Sequence

import numpy as np

from . import _lib

CORE = {_lib.DT_I32: _lib.DT_U32, _lib.DT_U32: _lib.DT_U32, _lib.DT_U64: _lib.DT_U64,
        _lib.DT_F64: _lib.DT_U64, _lib.DT_REC32: _lib.DT_REC32, _lib.DT_I64: _lib.DT_U64}
KEY_BYTES = {_lib.DT_I32: 4, _lib.DT_U32: 4, _lib.DT_U64: 8, _lib.DT_F64: 8, _lib.DT_I64: 8,
             _lib.DT_REC32: 32}
MAX_RANKS = 8


def rank_seed(seed: int, r: int) -> int:
    """Sample seed of rank r (shard.cuh shard_seed)."""
    return (seed ^ (0x9E3779B97F4A7C15 * (r + 1))) & 0xFFFFFFFFFFFFFFFF


def wire(t, dt: int):
    """Keys as int32 / int64 words for the collectives (records: (n, 4) int64)."""
    import torch
    return t.view(torch.int32) if KEY_BYTES[dt] == 4 else t.view(torch.int64)


# ---------------------------------------------------------------------------
# host-only plan (C, no device work): identical on every rank
# ---------------------------------------------------------------------------
MAX_BINS = 1024  # three-way bins of one exchange (kMaxPeerBins)


def subbuckets(dt: int, P: int, n_total: int) -> int:
    """K0: sub-buckets per rank of the folded exchange (qmsort_gpu_shard_subbuckets)."""
    return int(_lib.load().qmsort_gpu_shard_subbuckets(dt, P, n_total))


def splitters(core: int, sorted_sample: np.ndarray, nbuckets: int) -> tuple[np.ndarray, list]:
    """nbuckets - 1 quantile splitters of the sorted core-key sample, merged
    into distinct values: (unique splitters as uint8 rows, multiplicities)."""
    lib = _lib.load()
    w = KEY_BYTES[core]
    smp = np.ascontiguousarray(sorted_sample).view(np.uint8).reshape(-1)
    m = smp.shape[0] // w
    uniq = np.zeros(MAX_BINS // 2 * w, dtype=np.uint8)
    mult = (ctypes.c_uint32 * (MAX_BINS // 2))()
    nu = ctypes.c_uint32(0)
    _lib.check(lib.qmsort_gpu_shard_splitters(core, smp.ctypes.data, m, nbuckets, uniq.ctypes.data, mult,
                                              ctypes.byref(nu)), "qmsort_gpu_shard_splitters")
    k = int(nu.value)
    return uniq[:k * w].copy(), [int(mult[i]) for i in range(k)]


def plan(P: int, mult: Sequence[int], C: np.ndarray) -> dict:
    """Exchange plan from the P x (2m+1) count matrix (row = sender)."""
    lib = _lib.load()
    m = len(mult)
    nb = 2 * m + 1
    C = np.ascontiguousarray(np.asarray(C, dtype=np.uint64).reshape(P, nb))
    u64p = ctypes.POINTER(ctypes.c_uint64)
    i32p = ctypes.POINTER(ctypes.c_int32)
    bin_rank = np.zeros(nb, dtype=np.int32)
    bin_off = np.zeros((P, nb), dtype=np.uint64)
    recv_n, lo_fill, hi_fill = (np.zeros(P, dtype=np.uint64) for _ in range(3))
    lo_val, hi_val = np.zeros(P, dtype=np.int32), np.zeros(P, dtype=np.int32)
    mu = (ctypes.c_uint32 * max(1, m))(*mult)
    _lib.check(lib.qmsort_gpu_shard_plan(P, m, mu, C.ctypes.data_as(u64p), bin_rank.ctypes.data_as(i32p),
                                         bin_off.ctypes.data_as(u64p), recv_n.ctypes.data_as(u64p),
                                         lo_fill.ctypes.data_as(u64p), hi_fill.ctypes.data_as(u64p),
                                         lo_val.ctypes.data_as(i32p), hi_val.ctypes.data_as(i32p)),
               "qmsort_gpu_shard_plan")
    return {"bin_rank": bin_rank, "bin_off": bin_off, "recv_n": recv_n.astype(np.int64),
            "lo_fill": lo_fill.astype(np.int64), "hi_fill": hi_fill.astype(np.int64),
            "lo_val": lo_val, "hi_val": hi_val, "C": C.astype(np.int64)}


def plan_folded(P: int, K0: int, mult: Sequence[int], C: np.ndarray) -> dict:
    """The folded plan (qmsort_gpu_shard_plan_folded): every rank's slice as
    the three-way bin list of its local sort's level 0."""
    lib = _lib.load()
    m = len(mult)
    nb = 2 * m + 1
    LM = K0 + 1
    C = np.ascontiguousarray(np.asarray(C, dtype=np.uint64).reshape(P, nb))
    u64p, i32p, u32p = (ctypes.POINTER(t) for t in (ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32))
    bin_rank = np.zeros(nb, dtype=np.int32)
    bin_off = np.zeros((P, nb), dtype=np.uint64)
    out_n = np.zeros(P, dtype=np.uint64)
    loc_m = np.zeros(P, dtype=np.uint32)
    loc_uniq = np.zeros((P, LM), dtype=np.int32)
    loc_cnt = np.zeros((P, 2 * LM + 1), dtype=np.uint64)
    mu = (ctypes.c_uint32 * max(1, m))(*mult)
    _lib.check(lib.qmsort_gpu_shard_plan_folded(P, K0, m, mu, C.ctypes.data_as(u64p), bin_rank.ctypes.data_as(i32p),
                                                bin_off.ctypes.data_as(u64p), out_n.ctypes.data_as(u64p),
                                                loc_m.ctypes.data_as(u32p), loc_uniq.ctypes.data_as(i32p),
                                                loc_cnt.ctypes.data_as(u64p)), "qmsort_gpu_shard_plan_folded")
    return {"bin_rank": bin_rank, "bin_off": bin_off, "out_n": out_n.astype(np.int64), "loc_m": loc_m,
            "loc_uniq": loc_uniq, "loc_cnt": loc_cnt, "C": C.astype(np.int64)}


def local_splitters(uniq_h: np.ndarray, w: int, pl: dict, r: int) -> np.ndarray:
    """Rank r's local distinct splitters (uint8 rows) for its presplit sort."""
    rows = uniq_h.reshape(-1, w)
    k = int(pl["loc_m"][r])
    return np.ascontiguousarray(rows[pl["loc_uniq"][r][:k]]).reshape(-1) if k else np.zeros(0, np.uint8)


def staging_offsets(pl: dict, r: int) -> tuple[np.ndarray, list]:
    """Non-fused exchange: sender r's bins grouped by destination rank in a
    local staging buffer -- each bin's offset there and the per-rank sizes."""
    C, br = pl["C"], pl["bin_rank"]
    P = C.shape[0]
    send = [int(sum(C[r][b] for b in range(len(br)) if br[b] == t)) for t in range(P)]
    base = np.concatenate([[0], np.cumsum(send)]).astype(np.int64)
    off = np.zeros(len(br), dtype=np.uint64)
    acc = list(base[:P])
    for b, t in enumerate(br):
        if t >= 0:
            off[b] = acc[t]
            acc[t] += int(C[r][b])
    return off, send


def recv_counts(pl: dict, r: int) -> list:
    """What each sender ships to rank r (non-fused exchange)."""
    C, br = pl["C"], pl["bin_rank"]
    return [int(sum(C[s][b] for b in range(len(br)) if br[b] == r)) for s in range(C.shape[0])]


# ---------------------------------------------------------------------------
# per-rank compute ops (GPU: the C-ABI kernels)
# ---------------------------------------------------------------------------
class GpuOps:
    """Device ops of one rank, all through include/qmsort_gpu.h."""

    def __init__(self, stream: Any = None):
        import torch
        self.torch = torch
        self.lib = _lib.load()
        self.stream = stream
        self.launches = 0  # kernels of the local sorts (bench.py gpu_launches)
        self.alg_bytes = 0
        self.wsbuf = None

    def _s(self):
        return self.torch.cuda.current_stream().cuda_stream if self.stream is None else self.stream

    def synchronize(self) -> None:
        if self.stream is None:
            self.torch.cuda.current_stream().synchronize()
        else:
            self.torch.cuda.synchronize()

    def _ws(self, nbytes: int, device):
        """Grow-only device workspace shared by the partition and the local sort."""
        if self.wsbuf is None or self.wsbuf.numel() < nbytes or self.wsbuf.device != device:
            self.wsbuf = None
            self.wsbuf = self.torch.empty(int(nbytes * 1.25) + 4096, dtype=self.torch.uint8, device=device)
        return self.wsbuf

    def sample(self, t, dt: int, cmp: int, s: int, seed: int):
        """s seeded keys of t in the core domain (wire words)."""
        core = CORE[dt]
        out = self.torch.empty((s,) + tuple(t.shape[1:]), dtype=wire(t, dt).dtype, device=t.device)
        if t.shape[0] == 0:
            return out[:0]
        _lib.check(self.lib.qmsort_gpu_shard_sample(dt, cmp, t.data_ptr(), t.shape[0], s, seed,
                                                    out.data_ptr(), self._s()), "qmsort_gpu_shard_sample")
        assert KEY_BYTES[core] == KEY_BYTES[dt]
        return out

    def sort_core(self, t, core: int) -> None:
        from . import SortConfig, sort
        if t.shape[0] > 1:
            ws = self._ws(self.lib.qmsort_gpu_workspace_bytes(core, t.shape[0], None), t.device)
            m = sort(t, SortConfig(), "less", dtype=core, stream=self._s(), workspace=ws)
            self.launches += m.kernel_launches

    def put(self, host_bytes: np.ndarray, like):
        """Unique splitters (uint8 rows) onto this rank's device."""
        t = self.torch.from_numpy(np.ascontiguousarray(host_bytes)).to(like.device)
        return t

    def count(self, t, dt: int, cmp: int, uniq, m: int, three_way: bool = True):
        """Bin counts as three-way bins (2m + 1).  three_way = False (distinct
        splitters): two-way classification, counted into the open bins 2j."""
        torch = self.torch
        nc = 2 * m + 1 if three_way else m + 1
        counts = torch.zeros(nc, dtype=torch.int64, device=t.device)
        n = t.shape[0]
        ws = self._ws(self.lib.qmsort_gpu_shard_workspace_bytes(dt, n), t.device)
        _lib.check(self.lib.qmsort_gpu_shard_count(dt, cmp, t.data_ptr(), n, uniq.data_ptr() if m else None, m,
                                                   int(three_way), counts.data_ptr(), ws.data_ptr(), ws.numel(),
                                                   self._s()), "qmsort_gpu_shard_count")
        self.alg_bytes += n * KEY_BYTES[dt]
        if three_way:
            return counts
        full = torch.zeros(2 * m + 1, dtype=torch.int64, device=t.device)
        full[0::2] = counts
        return full

    def scatter(self, t, dt: int, cmp: int, m: int, bin_rank, bin_off, dests: Sequence[Any],
                recv_n: Sequence[int], raw: bool = True, three_way: bool = True) -> None:
        """Bin b of t (planned by count) -> dests[bin_rank[b]] + bin_off[b] keys;
        rank r's buffer holds recv_n[r] keys.  dests: device pointers (ints,
        e.g. IPC-mapped peers) or tensors.  raw: ship the caller's keys (else
        core keys)."""
        n = t.shape[0]
        if not n:
            return
        P = len(dests)
        nb = 2 * m + 1
        br = (ctypes.c_int32 * nb)(*[int(x) for x in bin_rank])
        bo = (ctypes.c_uint64 * nb)(*[int(x) for x in bin_off])
        rn = (ctypes.c_uint64 * P)(*[int(x) for x in recv_n])
        # an empty receive buffer may report a null pointer; no key goes there
        d = (ctypes.c_void_p * P)(*[int(x) if isinstance(x, int) else (x.data_ptr() or t.data_ptr())
                                    for x in dests])
        ws = self.wsbuf
        _lib.check(self.lib.qmsort_gpu_shard_scatter(dt, cmp, t.data_ptr(), n, m, int(three_way), br, bo, d, rn, P,
                                                     int(raw),
                                                     ws.data_ptr(), ws.numel(), self._s()),
                   "qmsort_gpu_shard_scatter")
        self.alg_bytes += 2 * n * KEY_BYTES[dt]

    def recv_workspace(self, n: int, dt: int, device):
        """A receive buffer for the folded exchange: the workspace of the local
        sort of n keys (its B half, offset 0, receives the keys)."""
        nbytes = int(self.lib.qmsort_gpu_workspace_bytes(dt, max(2, n), None))
        return self.torch.empty(nbytes, dtype=self.torch.uint8, device=device)

    def finish_presplit(self, ws, n: int, dt: int, cmp: int, luniq, lm: int, lcnt, like, out=None):
        """The local sort of a folded exchange: ws's B half holds the n core
        keys at their level-0 offsets; returns the sorted slice (caller dtype)
        -- in `out` (wire dtype, >= n rows) when given, else a fresh tensor."""
        torch = self.torch
        if out is None or out.shape[0] < n:
            out = torch.empty((max(1, n),) + tuple(like.shape[1:]), dtype=like.dtype, device=like.device)
        out = out[:n]
        if n == 0:
            return out
        from . import SortConfig
        c = SortConfig().to_c()
        mt = _lib.GpuMetrics()
        cnt = np.ascontiguousarray(np.asarray(lcnt[:2 * lm + 1], dtype=np.uint64))
        _lib.check(self.lib.qmsort_gpu_shard_finish_presplit(
            dt, cmp, out.data_ptr(), n, luniq.data_ptr() if lm else None, lm,
            cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(c), ws.data_ptr(), ws.numel(),
            ctypes.byref(mt), self._s()), "qmsort_gpu_shard_finish_presplit")
        self.launches += mt.kernel_launches
        self.alg_bytes += mt.alg_bytes
        return out

    def alloc(self, n: int, like):
        # never a null pointer, even for 0 keys (a peer's scatter is handed every buffer)
        t = self.torch.empty((max(1, n),) + tuple(like.shape[1:]), dtype=like.dtype, device=like.device)
        return t[:n]

    def finish(self, recv, n_recv: int, dt: int, cmp: int, uniq, lo_val: int, lo_fill: int, hi_val: int,
               hi_fill: int, like):
        """[lo fill | received keys sorted | hi fill] as a fresh tensor."""
        torch = self.torch
        n_out = n_recv + lo_fill + hi_fill
        out = torch.empty((n_out,) + tuple(like.shape[1:]), dtype=like.dtype, device=like.device)
        if n_out == 0:
            return out
        ws = self._ws(self.lib.qmsort_gpu_workspace_bytes(dt, max(2, n_recv), None), like.device)
        from . import SortConfig
        c = SortConfig().to_c()
        mt = _lib.GpuMetrics()
        _lib.check(self.lib.qmsort_gpu_shard_finish(dt, cmp, recv.data_ptr() if n_recv else None, n_recv,
                                                    uniq.data_ptr() if uniq is not None and uniq.numel() else None,
                                                    lo_val, lo_fill, hi_val, hi_fill, out.data_ptr(),
                                                    ctypes.byref(c), ws.data_ptr(), ws.numel(), ctypes.byref(mt),
                                                    self._s()), "qmsort_gpu_shard_finish")
        self.launches += mt.kernel_launches
        self.alg_bytes += mt.alg_bytes
        return out


# ---------------------------------------------------------------------------
# exchanges
# ---------------------------------------------------------------------------
class TorchExchange:
    """torch.distributed process group (NCCL on GPUs, gloo on CPUs): the
    non-fused baseline -- one all-to-all of a staging buffer."""

    fused = False

    def __init__(self, group: Any = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather_object(self, obj) -> list:
        out = [None] * self.P
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def _cpu_group(self) -> bool:
        return self.dist.get_backend(self.group) == "gloo"

    def all_gather(self, t):
        import torch
        if self._cpu_group() and t.is_cuda:
            t = t.cpu()
        parts = [torch.empty_like(t) for _ in range(self.P)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts)

    def all_to_all_v(self, t, send: Sequence[int], recv: Sequence[int]):
        import torch
        out = torch.empty((int(sum(recv)),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        self.dist.all_to_all_single(out, t, output_split_sizes=list(recv), input_split_sizes=list(send),
                                    group=self.group)
        return out


class PeerExchange(TorchExchange):
    """The data exchange fused into the partition (one process per GPU): every
    rank exports a receive buffer through CUDA IPC once; senders' scatter
    kernels then store their bins for rank j straight into rank j's buffer
    over NVLink (qmsort_gpu_shard_scatter).  torch.distributed only carries
    the samples, the count matrix, the handles and two barriers -- no
    collective touches the keys.  The receive buffer is reused across calls;
    every call returns a fresh output tensor (the local sort reads the
    receive buffer out of place)."""

    fused = True  # the folded exchange: the receive buffer is the local sort's workspace

    def __init__(self, group: Any = None):
        super().__init__(group)
        self.lib = _lib.load()
        self.recv = None       # this rank's receive buffer (uint8 device tensor)
        self.cap = 0           # its capacity in bytes
        self.ptrs: list = []   # device pointers of every rank's buffer, opened here
        self.opened: list = []  # mapping bases to close

    def ensure_capacity(self, nbytes: int, device) -> None:
        """Collective: (re)allocate every rank's buffer to >= nbytes and swap handles."""
        import torch
        need = [None] * self.P
        self.dist.all_gather_object(need, int(self.recv is None or self.cap < nbytes), group=self.group)
        if not any(need):
            return
        for p in self.opened:
            _lib.check(self.lib.qmsort_gpu_ipc_close(ctypes.c_void_p(p)), "qmsort_gpu_ipc_close")
        self.opened = []
        self.cap = max(int(nbytes * 1.25) + 4096, self.cap, 1 << 20)
        self.recv = torch.empty(self.cap, dtype=torch.uint8, device=device)
        h = (ctypes.c_uint8 * _IPC_BYTES)()
        off = ctypes.c_uint64()
        _lib.check(self.lib.qmsort_gpu_ipc_handle(ctypes.c_void_p(self.recv.data_ptr()), h,
                                                  ctypes.byref(off)), "qmsort_gpu_ipc_handle")
        handles: list = [None] * self.P
        self.dist.all_gather_object(handles, (bytes(h), int(off.value)), group=self.group)
        self.ptrs = []
        for j, (hb, ho) in enumerate(handles):
            if j == self.rank:
                self.ptrs.append(self.recv.data_ptr())
                continue
            buf = (ctypes.c_uint8 * _IPC_BYTES).from_buffer_copy(hb)
            p, base = ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(self.lib.qmsort_gpu_ipc_open(buf, ho, ctypes.byref(p), ctypes.byref(base)),
                       "qmsort_gpu_ipc_open")
            self.ptrs.append(int(p.value))
            self.opened.append(int(base.value))

    def barrier(self, ops: Any = None) -> None:
        """Every stream the rank's ops ran on has drained, then a host barrier."""
        import torch
        if ops is not None and hasattr(ops, "synchronize"):
            ops.synchronize()
        else:
            torch.cuda.synchronize()
        self.dist.barrier(group=self.group)


_IPC_BYTES = 64  # QMSORT_IPC_HANDLE_BYTES


def _pad_sample(smp, s: int, like):
    """An empty (or short) shard contributes maximum keys (never a splitter below them)."""
    import torch
    if smp.shape[0] >= s:
        return smp
    pad = torch.full((s - smp.shape[0],) + tuple(smp.shape[1:]), -1, dtype=smp.dtype, device=smp.device)
    return torch.cat([smp, pad])


def _np_rows(t) -> np.ndarray:
    return t.detach().cpu().contiguous().numpy()


def sort_sharded(local, less: Any = "less", *, dtype: int | None = None, exchange: Any = None,
                 ops: Any = None, oversample: int = 64, seed: int = 42, out: Any = None):
    """Globally sort the keys held by all ranks; returns this rank's slice
    (of the caller's dtype): a view of ``out`` when that has room for it
    (e.g. a buffer reused across calls), else a fresh tensor.  ``local`` is
    only read."""
    from . import _cmp_code, dtype_of
    dt = dtype_of(local) if dtype is None else dtype
    core = CORE[dt]
    cmp = _cmp_code(less)
    ex = exchange or TorchExchange()
    ops = ops or GpuOps()
    P, r = ex.P, ex.rank
    if P > MAX_RANKS:
        raise ValueError(f"at most {MAX_RANKS} ranks")
    w = KEY_BYTES[dt]
    wl = wire(local, dt)
    folded = getattr(ex, "fused", False)
    n_total = int(local.shape[0])
    if folded and P > 1:  # every rank's size (one small all-gather of a tensor)
        import torch
        sz = torch.tensor([int(local.shape[0])], dtype=torch.int64,
                          device=local.device if local.is_cuda else "cpu")
        n_total = int(ex.all_gather(sz).sum().item())
    K0 = subbuckets(dt, P, n_total) if folded else 1
    s = max(oversample * P, 32 * K0)
    smp = _pad_sample(ops.sample(local, dt, cmp, s, rank_seed(seed, r)), s, local)
    all_smp = ex.all_gather(smp).contiguous()
    if all_smp.device != local.device:
        all_smp = all_smp.to(local.device)
    ops.sort_core(all_smp, core)
    uniq_h, mult = splitters(core, _np_rows(all_smp), P * K0)
    m = len(mult)
    uniq = ops.put(uniq_h, local)
    tw = any(c > 1 for c in mult)  # a repeated splitter value: its equal keys become fills
    counts = ops.count(local, dt, cmp, uniq, m, tw)
    C = _np_rows(ex.all_gather(counts)).reshape(P, 2 * m + 1)
    if folded:
        # the exchange scatter is level 0 of every rank's local sort: core keys
        # straight into the B half of the receivers' sort workspaces
        pl = plan_folded(P, K0, mult, C)
        n_out = int(pl["out_n"][r])
        need = int(ops.lib.qmsort_gpu_workspace_bytes(dt, max(2, n_out), None))
        ex.ensure_capacity(need, local.device)
        ex.barrier(ops)  # every receiver is done with its buffer and holds the handles
        ops.scatter(local, dt, cmp, m, pl["bin_rank"], pl["bin_off"][r], ex.ptrs, pl["out_n"], raw=False,
                    three_way=tw)
        ex.barrier(ops)  # every sender's stores into this rank's buffer have landed
        luniq = ops.put(local_splitters(uniq_h, w, pl, r), local)
        res = ops.finish_presplit(ex.recv, n_out, dt, cmp, luniq, int(pl["loc_m"][r]), pl["loc_cnt"][r], wl,
                                  out=None if out is None else wire(out, dt))
        return res.view(local.dtype)
    # plain exchange (the NCCL baseline): local staging grouped by rank, one
    # all-to-all, then the out-of-place local sort between the fills
    pl = plan(P, mult, C)
    n_recv = int(pl["recv_n"][r])
    off, send = staging_offsets(pl, r)
    staging = ops.alloc(local.shape[0], wl)
    ops.scatter(local, dt, cmp, m, pl["bin_rank"], off, [staging] * P, [local.shape[0]] * P, raw=True,
                three_way=tw)
    recv = ex.all_to_all_v(staging, send, recv_counts(pl, r)).contiguous()
    out = ops.finish(recv, n_recv, dt, cmp, uniq, int(pl["lo_val"][r]), int(pl["lo_fill"][r]),
                     int(pl["hi_val"][r]), int(pl["hi_fill"][r]), wl)
    return out.view(local.dtype)


def sort_sharded_emulated_fused(shards: list, less: Any = "less", *, dtype: int | None = None,
                                oversample: int = 64, seed: int = 42) -> list:
    """The fused exchange with P ranks emulated in one process on one GPU: each
    rank's scatter stores its bins straight into the other ranks' receive
    buffers (plain device pointers instead of IPC-mapped peers)."""
    return _emulated(shards, less, dtype, [GpuOps() for _ in shards], oversample, seed, fused=True)


def sort_sharded_emulated(shards: list, less: Any = "less", *, dtype: int | None = None,
                          ops: Any = None, oversample: int = 64, seed: int = 42) -> list:
    """Same algorithm as sort_sharded with the (non-fused) exchange done in-process."""
    opss = [ops] * len(shards) if ops is not None else [GpuOps() for _ in shards]
    return _emulated(shards, less, dtype, opss, oversample, seed, fused=False)


def _emulated(shards, less, dtype, opss, oversample, seed, fused):
    import torch
    from . import _cmp_code, dtype_of
    dt = dtype_of(shards[0]) if dtype is None else dtype
    core = CORE[dt]
    cmp = _cmp_code(less)
    P = len(shards)
    w = KEY_BYTES[dt]
    wl = [wire(t, dt) for t in shards]
    K0 = subbuckets(dt, P, sum(int(t.shape[0]) for t in shards)) if fused else 1
    s = max(oversample * P, 32 * K0)
    smps = [_pad_sample(opss[r].sample(t, dt, cmp, s, rank_seed(seed, r)), s, t) for r, t in enumerate(shards)]
    all_smp = torch.cat(smps).contiguous()
    opss[0].sort_core(all_smp, core)
    uniq_h, mult = splitters(core, _np_rows(all_smp), P * K0)
    m = len(mult)
    uniqs = [opss[r].put(uniq_h, t) for r, t in enumerate(shards)]
    tw = any(c > 1 for c in mult)
    C = np.stack([_np_rows(opss[r].count(t, dt, cmp, uniqs[r], m, tw)) for r, t in enumerate(shards)])
    out = []
    if fused:  # folded: the receive buffers are the local sorts' workspaces
        pl = plan_folded(P, K0, mult, C)
        wss = [opss[j].recv_workspace(int(pl["out_n"][j]), dt, shards[j].device) for j in range(P)]
        for r, t in enumerate(shards):  # ops[r] still holds rank r's plan in its workspace
            opss[r].scatter(t, dt, cmp, m, pl["bin_rank"], pl["bin_off"][r], wss, pl["out_n"], raw=False,
                            three_way=tw)
        for j in range(P):
            luniq = opss[j].put(local_splitters(uniq_h, w, pl, j), shards[j])
            o = opss[j].finish_presplit(wss[j], int(pl["out_n"][j]), dt, cmp, luniq, int(pl["loc_m"][j]),
                                        pl["loc_cnt"][j], wl[j])
            out.append(o.view(shards[j].dtype))
        return out
    pl = plan(P, mult, C)
    stagings, sends = [], []
    for r, t in enumerate(shards):
        off, send = staging_offsets(pl, r)
        st = opss[r].alloc(t.shape[0], wl[r])
        opss[r].scatter(t, dt, cmp, m, pl["bin_rank"], off, [st] * P, [t.shape[0]] * P, raw=True, three_way=tw)
        stagings.append(st)
        sends.append(np.concatenate([[0], np.cumsum(send)]).astype(np.int64))
    for j in range(P):  # rank j receives, in sender order, what each sender grouped for it
        pieces = [stagings[r][int(sends[r][j]):int(sends[r][j + 1])] for r in range(P)]
        recv = torch.cat(pieces).contiguous() if pieces else opss[j].alloc(0, wl[j])
        o = opss[j].finish(recv, int(pl["recv_n"][j]), dt, cmp, uniqs[j], int(pl["lo_val"][j]),
                           int(pl["lo_fill"][j]), int(pl["hi_val"][j]), int(pl["hi_fill"][j]), wl[j])
        out.append(o.view(shards[j].dtype))
    return out


def sort_sharded_devices(shards: list, devices: Sequence[int] | None = None, less: Any = "less", *,
                         dtype: int | None = None, cfg: Any = None):
    """The single-process C entry (qmsort_gpu_sort_sharded): shard r lives on
    devices[r] (a device may repeat); returns (slices, Metrics)."""
    import torch
    from . import Metrics, SortConfig, _cmp_code, dtype_of
    lib = _lib.load()
    dt = dtype_of(shards[0]) if dtype is None else dtype
    P = len(shards)
    devs = list(devices) if devices is not None else [t.device.index or 0 for t in shards]
    total = sum(int(t.shape[0]) for t in shards)
    ia = (ctypes.c_int * P)(*devs)
    din = (ctypes.c_void_p * P)(*[t.data_ptr() for t in shards])
    nin = (ctypes.c_size_t * P)(*[int(t.shape[0]) for t in shards])
    on = (ctypes.c_size_t * P)()
    c = (cfg or SortConfig()).to_c()
    mt = _lib.GpuMetrics()
    # a balanced split needs about total / P per rank; on QMSORT_ENOWS the call
    # reports the exact sizes and is repeated once with them
    caps = [min(total, (3 * total) // (2 * P) + 65536)] * P
    for attempt in range(2):
        outs = [torch.empty((max(1, cp),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                for cp, t in zip(caps, shards)]
        dout = (ctypes.c_void_p * P)(*[o.data_ptr() for o in outs])
        cap = (ctypes.c_size_t * P)(*caps)
        rc = lib.qmsort_gpu_sort_sharded(dt, _cmp_code(less), P, ia, din, nin, dout, cap, on, ctypes.byref(c),
                                         ctypes.byref(mt))
        if rc == _lib.QMSORT_ENOWS and attempt == 0:
            caps = [int(on[r]) for r in range(P)]
            del outs
            continue
        _lib.check(rc, "qmsort_gpu_sort_sharded")
        break
    return [outs[r][: int(on[r])] for r in range(P)], Metrics.from_c(mt)


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun) and --sharded: the north-star sharded configs
# ---------------------------------------------------------------------------
# config -> (dtype attr, torch dtype, row shape, generator, keys, key bytes,
#            scaling, description)
SHARDED_CONFIGS = {
    "c2": ("DT_U32", "uint32", (), "GEN_U32", 1 << 28, 4, "weak",
           "C2 recipe, 2^28 uint32 keys per GPU"),
    "c3": ("DT_U64", "uint64", (), "GEN_U64", 1 << 30, 8, "strong",
           "C3: 2^30 uint64 keys in total, shard r = global indices [r n/P, (r+1) n/P)"),
    "c5": ("DT_REC32", "uint64", (4,), "GEN_REC32", 1 << 26, 32, "strong",
           "C5: 2^26 32-byte records in total, shard r = global records [r n/P, (r+1) n/P)"),
}


def bench_main(args: Any, metric: str, unit: str) -> None:
    import json
    import os
    import statistics
    import time

    import torch
    import torch.distributed as dist

    import paper_1804_10062_b200 as q

    for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531")):
        os.environ.setdefault(k, v)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # QMSORT_BENCH_ONE_GPU=1 (a test aid): every rank on GPU 0 with gloo for the
    # host collectives -- the IPC peer exchange and this driver's multi-rank
    # logic on a one-GPU box (NCCL refuses two ranks on one device)
    one_gpu = os.environ.get("QMSORT_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    rank, P = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if one_gpu else dev  # where the bench's own collectives run
    cfgname = args.config if args.config in SHARDED_CONFIGS else "c2"
    dt_name, tdt, tail, gen, n_cfg, kb, scaling, desc = SHARDED_CONFIGS[cfgname]
    dt = getattr(q, dt_name)
    if scaling == "weak":
        n_total = args.n * P
        n_loc = args.n
        start = rank * n_loc
    else:
        n_total = n_cfg
        start = rank * n_total // P
        n_loc = (rank + 1) * n_total // P - start
    pristine = torch.empty((n_loc,) + tail, dtype=getattr(torch, tdt), device=dev)
    q.generate(getattr(q, gen), pristine, seed=42, start=start, total=n_total)
    exchange = getattr(args, "exchange", "peer")
    ex = PeerExchange() if exchange == "peer" else TorchExchange()
    ops = GpuOps()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # two output buffers, alternated: a slice stays valid for one more step,
    # and no step allocates
    outs = [torch.empty((n_loc * 3 // 2 + 65536,) + tail, dtype=pristine.dtype, device=dev) for _ in range(2)]
    cnt = [0]

    def step():
        torch.cuda.synchronize()
        dist.barrier()
        cnt[0] += 1
        e0.record()
        out = sort_sharded(pristine, "less", dtype=dt, exchange=ex, ops=ops, out=outs[cnt[0] & 1])
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    for _ in range(max(1, args.warmup)):
        step()
    ops.launches = ops.alg_bytes = 0
    times, out = [], None
    for _ in range(args.steps):
        t, out = step()
        times.append(t)
    launches, alg_rank = ops.launches, ops.alg_bytes // max(1, args.steps)
    # verification (untimed): every slice sorted, slices ordered across ranks,
    # multiset of all keys preserved
    viol, s_out, _ = q.check(out)
    _, s_in, _ = q.check(pristine, order=False)
    mask = (1 << 62) - 1
    lens = torch.tensor([out.shape[0]], dtype=torch.int64, device=cdev)
    all_lens = [torch.empty_like(lens) for _ in range(P)]
    dist.all_gather(all_lens, lens)
    wout = wire(out, dt)  # NCCL has no unsigned types: int32 / int64 words
    ends_rows = torch.zeros((2,) + tail, dtype=wout.dtype, device=dev)
    if out.shape[0]:
        ends_rows[0], ends_rows[1] = wout[0], wout[-1]
    ends_rows = ends_rows.to(cdev)
    all_ends = [torch.empty_like(ends_rows) for _ in range(P)]
    dist.all_gather(all_ends, ends_rows)
    stats = torch.tensor([viol, s_out & mask, s_in & mask], dtype=torch.int64, device=cdev)
    dist.all_reduce(stats)
    alg_t = torch.tensor([alg_rank], dtype=torch.float64, device=cdev)
    dist.all_reduce(alg_t, op=dist.ReduceOp.MAX)
    ms = statistics.mean(times)
    # end to end: pinned host shard -> H2D -> distributed sort -> D2H of the slice
    host_in = pristine.cpu().pin_memory()
    host_out = torch.empty((n_loc * 3 // 2 + 1024,) + tail, dtype=pristine.dtype, pin_memory=True)
    xd = torch.empty_like(pristine)
    e2e_t, d2h = [], 0
    for i in range(1 + min(args.steps, 3)):
        dist.barrier()
        t0 = time.perf_counter()
        xd.copy_(host_in, non_blocking=True)
        res = sort_sharded(xd, "less", dtype=dt, exchange=ex, ops=ops)
        if res.shape[0] <= host_out.shape[0]:
            host_out[:res.shape[0]].copy_(res)
        else:
            res = res.cpu()
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], device=cdev)
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        if i:
            e2e_t.append(float(el.item()))
            d2h = res.shape[0]
    d2h_t = torch.tensor([d2h], dtype=torch.int64, device=cdev)
    dist.all_reduce(d2h_t)
    if rank == 0:
        def key_of(row):
            v = row.view(-1).tolist() if tail else [row.item()]
            return [x & ((1 << (8 * min(kb, 8))) - 1) for x in v]
        pairs = [(int(all_lens[r].item()), all_ends[r]) for r in range(P)]
        nonempty = [e for ln, e in pairs if ln > 0]
        seam_ok = all(key_of(nonempty[i][1]) <= key_of(nonempty[i + 1][0]) for i in range(len(nonempty) - 1))
        e2e_ms = statistics.mean(e2e_t) * 1e3
        peak = 6555.2
        try:
            peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)),
                                                     "MEASURED_PEAKS.json")))["hbm_gbs"])
        except OSError:
            pass
        n_max = max(int(x.item()) for x in all_lens)
        # per-rank pass ledger from the device counters: count 1 + scatter
        # (= the exchange) 2 + the local sort's own ledger (8 for uniform keys)
        alg = float(alg_t.item())
        nvl_bytes = (P - 1) * n_loc * kb / P  # bytes each rank ships over NVLink
        t_hbm = alg / peak / 1e6           # ms at the HBM roofline
        t_nvl = nvl_bytes / 900.0 / 1e6    # ms at 900 GB/s per direction
        line = {"metric": metric if cfgname == "c2" else f"sorted Gkeys/s, {desc} (sharded)",
                "value": n_total / (ms / 1e3) / 1e9, "unit": unit, "n_gpus": P,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
                "dtype": {"DT_U32": "u32", "DT_U64": "u64", "DT_REC32": "4xu64"}[dt_name],
                "data": f"synthetic (seeded SplitMix64, SURVEY.md 8(d) {cfgname.upper()} recipe, seed 42)",
                "config": {"workload": f"distributed samplesort, {desc}, {P} rank(s) (" +
                                       ("exchange fused into the scatter: IPC peer stores over NVLink"
                                        if exchange == "peer" else "one NCCL all-to-all") + ")",
                           "n_total": n_total, "n_per_gpu": n_loc, "largest_slice": n_max,
                           "key_bytes": kb, "parallelism": f"sharded samplesort x{P}",
                           "l2": "input > L2 on every rank"},
                "step_ms": [round(t, 4) for t in times],
                "gpu_launches": launches,
                "roofline": {"bound": "hbm", "kernel": "whole per-GPU pipeline (max over ranks)",
                             "achieved": alg / (ms * 1e6), "peak": peak, "unit": "GB/s",
                             "frac": alg / (ms * 1e6) / peak, "traffic": None,
                             "alg_bytes_per_rank": alg, "ledger_bytes_over_nw": alg / (n_loc * kb),
                             "hbm_frac": t_hbm / ms,
                             "nvlink": {"bytes_per_rank": nvl_bytes, "peak_GBps": 900.0,
                                        "achieved_GBps": nvl_bytes / (ms * 1e6), "frac": t_nvl / ms},
                             "t_roof_ms": t_hbm + t_nvl, "frac_of_serial_roofline": (t_hbm + t_nvl) / ms},
                "e2e": {"value": n_total / (e2e_ms / 1e3) / 1e9, "unit": unit, "ms_per_step": e2e_ms,
                        "h2d_bytes_per_step": n_total * kb, "d2h_bytes_per_step": int(d2h_t.item()) * kb,
                        "api": "sharded.sort_sharded on pinned host shards (H2D + sort + D2H per rank)"},
                "verify": {"order_violations_within_slices": int(stats[0].item()),
                           "slices_ordered_across_ranks": seam_ok,
                           # the per-rank fingerprint sums are taken mod 2^62 before the
                           # all-reduce: compare the totals mod 2^62 too
                           "multiset_preserved": (int(stats[1].item()) - int(stats[2].item())) & mask == 0}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
