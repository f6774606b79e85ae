"""CPU test doubles of the per-rank device ops used by sharded.py, so the
exchange logic of the distributed samplesort can run under gloo on CPU.
They restate, in numpy, what the C-ABI kernels compute: the order-preserving
transform into the unsigned core domain, the seeded sample, the three-way
count against distinct splitters, the scatter of bins to (bin_rank, bin_off),
and the finishing sort between the equal-key fills.  The host-only plan
(qmsort_gpu_shard_splitters / qmsort_gpu_shard_plan) is the real C code."""
from __future__ import annotations

import bisect

import numpy as np
import torch

from paper_1804_10062_b200 import _lib
from paper_1804_10062_b200.sharded import CORE, KEY_BYTES

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def sm_mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def to_core(a: np.ndarray, dt: int, cmp: int) -> np.ndarray:
    """Caller keys -> unsigned core keys (uint32 / uint64 / (n,4) uint64)."""
    if dt == _lib.DT_I32:
        return a.view(np.uint32) ^ np.uint32(0x7FFFFFFF if cmp else 0x80000000)
    if dt == _lib.DT_I64:
        return a.view(np.uint64) ^ np.uint64(0x7FFFFFFFFFFFFFFF if cmp else 1 << 63)
    if dt == _lib.DT_F64:
        u = a.view(np.uint64)
        top = np.uint64(1 << 63)
        c = np.where((u >> np.uint64(63)) == 1, ~u, u | top)
        return ~c if cmp else c
    u = a.view(np.uint32 if dt == _lib.DT_U32 else np.uint64)
    return ~u if cmp else u.copy()


def from_core(c: np.ndarray, dt: int, cmp: int) -> np.ndarray:
    if dt == _lib.DT_I32:
        return (c ^ np.uint32(0x7FFFFFFF if cmp else 0x80000000)).view(np.int32)
    if dt == _lib.DT_I64:
        return (c ^ np.uint64(0x7FFFFFFFFFFFFFFF if cmp else 1 << 63)).view(np.int64)
    if dt == _lib.DT_F64:
        u = ~c if cmp else c
        top = np.uint64(1 << 63)
        return np.where((u >> np.uint64(63)) == 1, u & ~top, ~u).view(np.float64)
    return ~c if cmp else c.copy()


def _keys(c: np.ndarray, core: int) -> list:
    return [tuple(r) for r in c.tolist()] if core == _lib.DT_REC32 else c.tolist()


def _sorted_core(c: np.ndarray, core: int) -> np.ndarray:
    if core == _lib.DT_REC32:
        return c[np.lexsort(c.T[::-1])] if c.shape[0] else c
    return np.sort(c, kind="stable")


class NumpyOps:
    def _np(self, t, dt):
        """The caller keys of t (caller or wire dtype) as a numpy view."""
        return t.contiguous().numpy().view(
            {_lib.DT_I32: np.int32, _lib.DT_U32: np.uint32, _lib.DT_U64: np.uint64, _lib.DT_F64: np.float64,
             _lib.DT_I64: np.int64, _lib.DT_REC32: np.uint64}[dt])

    def sample(self, t, dt, cmp, s, seed):
        n = t.shape[0]
        wt = torch.int32 if KEY_BYTES[dt] == 4 else torch.int64
        if n == 0:
            return torch.empty((0,) + tuple(t.shape[1:]), dtype=wt)
        idx = [((sm_mix((seed + (i + 1) * GAMMA) & MASK64)) * n) >> 64 for i in range(s)]
        c = to_core(self._np(t, dt), dt, cmp)[idx]
        return torch.from_numpy(np.ascontiguousarray(c)).view(wt)

    def sort_core(self, t, core):
        a = t.numpy().view(np.uint32 if core == _lib.DT_U32 else np.uint64)
        a[...] = _sorted_core(a.copy(), core)

    def put(self, host_bytes, like):
        return torch.from_numpy(np.ascontiguousarray(host_bytes))

    def _uniq(self, uniq, core, m):
        u = uniq.numpy().view(np.uint32 if core == _lib.DT_U32 else np.uint64)
        return _keys(u.reshape(m, 4) if core == _lib.DT_REC32 else u[:m], core)

    def _bins(self, t, dt, cmp, uniq, m, three_way=True):
        core = CORE[dt]
        keys = _keys(to_core(self._np(t, dt), dt, cmp), core)
        us = self._uniq(uniq, core, m) if m else []
        out = []
        for k in keys:
            j = bisect.bisect_left(us, k)
            out.append(2 * j + (1 if three_way and j < m and us[j] == k else 0))
        return np.array(out, dtype=np.int64)

    def count(self, t, dt, cmp, uniq, m, three_way=True):
        # the plan stays with the rank's data (one double may serve every emulated rank)
        if not hasattr(self, "_plans"):
            self._plans = {}
        b = self._bins(t, dt, cmp, uniq, m, three_way)
        self._plans[t.data_ptr()] = b
        return torch.from_numpy(np.bincount(b, minlength=2 * m + 1).astype(np.int64))

    def scatter(self, t, dt, cmp, m, bin_rank, bin_off, dests, recv_n=None, raw=True, three_way=True):
        b = self._plans[t.data_ptr()]
        src = t.numpy()
        pos = {bb: int(bin_off[bb]) for bb in range(2 * m + 1)}
        for i, bb in enumerate(b.tolist()):
            r = int(bin_rank[bb])
            if r < 0:
                continue
            dests[r].numpy().view(src.dtype)[pos[bb]] = src[i]
            pos[bb] += 1

    def alloc(self, n, like):
        return torch.empty((n,) + tuple(like.shape[1:]), dtype=like.dtype)

    def finish(self, recv, n_recv, dt, cmp, uniq, lo_val, lo_fill, hi_val, hi_fill, like):
        core = CORE[dt]
        c = to_core(self._np(recv[:n_recv], dt), dt, cmp)
        c = _sorted_core(c, core)
        u = uniq.numpy().view(np.uint32 if core == _lib.DT_U32 else np.uint64)
        if core == _lib.DT_REC32:
            u = u.reshape(-1, 4)
        parts = []
        if lo_fill:
            parts.append(np.repeat(u[lo_val:lo_val + 1], lo_fill, axis=0))
        parts.append(c)
        if hi_fill:
            parts.append(np.repeat(u[hi_val:hi_val + 1], hi_fill, axis=0))
        allc = np.concatenate(parts) if parts else c
        x = from_core(allc, dt, cmp)
        return torch.from_numpy(np.ascontiguousarray(x)).view(like.dtype)
