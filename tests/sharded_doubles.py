"""CPU test doubles of the per-rank device ops used by sharded.py, so the
exchange logic of the distributed samplesort can run under gloo on CPU.
They restate, in numpy, what the C-ABI kernels compute (transform into the
unsigned core domain, seeded sample, local sort, partition by splitters)."""
from __future__ import annotations

import numpy as np
import torch

from paper_1804_10062_b200 import _lib

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def sm_mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def _np(t):
    return t.numpy()


class NumpyOps:
    def to_core(self, t, dt, cmp, inverse=False):
        a = _np(t)
        if dt == _lib.DT_I32:
            u = a.view(np.uint32)
            u ^= np.uint32(0x7FFFFFFF if cmp else 0x80000000)
        elif dt == _lib.DT_U32:
            if cmp:
                a[...] = ~a
        elif dt in (_lib.DT_U64, _lib.DT_REC32):
            if cmp:
                a[...] = ~a
        elif dt == _lib.DT_F64:
            u = a.view(np.uint64)
            top = np.uint64(1 << 63)
            if not inverse:
                neg = (u >> np.uint64(63)) == 1
                u[...] = np.where(neg, ~u, u | top)
                if cmp:
                    u[...] = ~u
            else:
                if cmp:
                    u[...] = ~u
                pos = (u >> np.uint64(63)) == 1
                u[...] = np.where(pos, u & ~top, ~u)

    def sample(self, t, core, s, seed):
        n = t.shape[0]
        if n == 0:
            return t[:0].clone()
        idx = [((sm_mix((seed + (i + 1) * GAMMA) & MASK64)) * n) >> 64 for i in range(s)]
        return t[torch.tensor(idx, dtype=torch.long)].clone()

    def _order(self, a, core):
        if core == _lib.DT_REC32:
            return np.lexsort(a.T[::-1])
        return np.argsort(a.view(np.uint32 if core == _lib.DT_U32 else np.uint64), kind="stable")

    def sort(self, t, core):
        a = _np(t)
        a[...] = a[self._order(a, core)]

    def partition(self, t, core, spl):
        a, s = _np(t), _np(spl)
        if core == _lib.DT_REC32:
            keys = [tuple(r) for r in a.tolist()]
            ss = [tuple(r) for r in s.tolist()]
            import bisect
            b = np.array([bisect.bisect_left(ss, k) for k in keys], dtype=np.int64)
        else:
            ut = np.uint32 if core == _lib.DT_U32 else np.uint64
            b = np.searchsorted(s.view(ut), a.view(ut), side="left")
        order = np.argsort(b, kind="stable")
        counts = np.bincount(b, minlength=s.shape[0] + 1).astype(np.int64)
        return torch.from_numpy(a[order].copy()), torch.from_numpy(counts)
