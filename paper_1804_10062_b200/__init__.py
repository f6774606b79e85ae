"""qmsort-b200: a B200-native drop-in for the reference QuickMergesort entry point.

Python mirror of the reference API (``/root/reference/proj/core/include/qmsort``):

=====================================  ============================================
reference (C++)                        here
=====================================  ============================================
``enum class Variant`` (sort.hpp:17)   :class:`Variant`
``enum class PivotStrategy`` (:19)     :class:`PivotStrategy`
``enum class BaseCase`` (merge.hpp:14) :class:`BaseCase`
``BaseCasePolicy`` (merge.hpp:26-31)   :class:`BaseCasePolicy`
``SortConfig`` (sort.hpp:25-34)        :class:`SortConfig` (+ GPU knobs)
``qms/qmqs/momqms/hqms`` (:37-66)      :func:`qms` :func:`qmqs` :func:`momqms` :func:`hqms`
``Metrics`` (metrics.hpp:14-24)        :class:`Metrics`
``qmsort::sort(first, last, cfg,       :func:`sort` (device tensor in place, or host
  less)`` (sort.hpp:215-226)             array through the host drop-in call)
``sort_range_counted`` (:207-211)      :func:`sort_range_counted`
``Element<PayloadBytes>``              :func:`sort_elements` (key-only ordering,
  (element.hpp:13-20)                    payload moved; stable on the GPU)
``select_nth(first, last, k, cmp, m)`` :func:`select_nth` (1-based k, returns the
  (selection.hpp:207-212)                position; range partitioned around it)
``PartitionResult``                    :class:`PartitionResult`, :func:`partition`
  (partition_result.hpp:12-17)           (three-way, around a pivot value)
=====================================  ============================================

All compute goes through the CUDA library (``libqmsort_gpu.so``) via the C-ABI
in ``include/qmsort_gpu.h``; nothing here sorts on the CPU.
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
from typing import Any

from . import _lib
from ._lib import DT_F64, DT_I32, DT_I64, DT_REC32, DT_U32, DT_U64, GREATER, LESS, QmsortError

__all__ = [
    "Variant", "PivotStrategy", "BaseCase", "MergesortSide", "BaseCasePolicy", "SortConfig",
    "Metrics", "qms", "qmqs", "momqms", "hqms", "sort", "sort_batch", "sort_range_counted",
    "QmsortError",
    "DT_I32", "DT_U32", "DT_U64", "DT_F64", "DT_REC32", "DT_I64", "LESS", "GREATER",
    "workspace_bytes", "generate", "check", "dtype_of", "sort_elements", "select_nth",
    "PartitionResult", "partition",
]


class Variant(enum.IntEnum):
    qms = 0
    qmqs = 1
    momqms = 2
    hqms = 3


class PivotStrategy(enum.IntEnum):
    median_of_3 = 0
    median_of_sqrt_n = 1
    mom_of_thirds = 2
    hybrid = 3


class BaseCase(enum.IntEnum):
    insertion = 0
    hardcoded_small = 1
    clever_quicksort = 2


class MergesortSide(enum.IntEnum):
    smaller_always = 0
    larger_when_feasible = 1


@dataclasses.dataclass
class BaseCasePolicy:
    """merge.hpp:26-31.  On the GPU every kind maps to the block sorter (K5)."""

    kind: BaseCase = BaseCase.hardcoded_small
    size_threshold: int = 10
    use_levels: bool = False


class Algorithm(enum.IntEnum):
    samplesort = 0  # sampled multi-splitter partition + block sort (default)
    mergesort = 1   # block sort + merge-path passes only


@dataclasses.dataclass
class SortConfig:
    """SortConfig (sort.hpp:25-34) plus the GPU-only knobs (GpuSortOptions)."""

    variant: Variant = Variant.qms
    pivot: PivotStrategy = PivotStrategy.median_of_3
    base_case: BaseCasePolicy = dataclasses.field(default_factory=BaseCasePolicy)
    beta: float = 0.5
    delta: float = 1.0 / 16.0
    side: MergesortSide = MergesortSide.larger_when_feasible
    three_way: bool = False
    block: int = 128
    # GPU knobs
    algorithm: Algorithm = Algorithm.samplesort
    seed: int = 42
    max_levels: int = 8
    profile: bool = False  # time every kernel launch (Metrics.phase_ns)

    def to_c(self) -> _lib.GpuConfig:
        c = _lib.GpuConfig()
        c.variant = int(self.variant)
        c.pivot = int(self.pivot)
        c.base_case_kind = int(self.base_case.kind)
        c.base_case_size_threshold = int(self.base_case.size_threshold)
        c.base_case_use_levels = int(bool(self.base_case.use_levels))
        c.beta = float(self.beta)
        c.delta = float(self.delta)
        c.side = int(self.side)
        c.three_way = int(bool(self.three_way))
        c.block = int(self.block)
        c.algorithm = int(self.algorithm)
        c.seed = int(self.seed) & ((1 << 64) - 1)
        c.max_levels = int(self.max_levels)
        c.profile = int(bool(self.profile))
        return c


def qms() -> SortConfig:
    """Median-of-3 pivots, hard-coded small base case (sort.hpp:37)."""
    return SortConfig()


def qmqs() -> SortConfig:
    """sort.hpp:41-48."""
    return SortConfig(variant=Variant.qmqs,
                      base_case=BaseCasePolicy(BaseCase.clever_quicksort, 16, True))


def momqms() -> SortConfig:
    """sort.hpp:52-57."""
    return SortConfig(variant=Variant.momqms, pivot=PivotStrategy.mom_of_thirds)


def hqms() -> SortConfig:
    """sort.hpp:61-66."""
    return SortConfig(variant=Variant.hqms, pivot=PivotStrategy.hybrid)


@dataclasses.dataclass
class Metrics:
    """metrics.hpp:14-24.  comparisons/moves are not instrumented on the GPU (0);
    max_depth = partition levels; elapsed_ns = device time (CUDA events)."""

    comparisons: int = 0
    moves: int = 0
    max_depth: int = 0
    elapsed_ns: int = 0
    # GPU pass ledger
    alg_bytes: int = 0
    levels: int = 0
    merge_passes: int = 0
    kernel_launches: int = 0
    host_syncs: int = 0
    phase_bytes: list = dataclasses.field(default_factory=lambda: [0] * _lib.NUM_PHASES)
    phase_ns: list = dataclasses.field(default_factory=lambda: [0] * _lib.NUM_PHASES)
    phase_launches: list = dataclasses.field(default_factory=lambda: [0] * _lib.NUM_PHASES)
    resplits: int = 0  # hybrid pivot: buckets re-sampled with triple medians (f1)
    sample_keys: int = 0  # splitter-sample keys drawn (median_of_sqrt_n: the reference's s per segment)
    table_buckets: int = 0  # integer-key buckets sent to the comparison-free table / cell sorts (tablesort.cuh)

    @classmethod
    def from_c(cls, m: _lib.GpuMetrics) -> "Metrics":
        kw = {}
        for f in dataclasses.fields(cls):
            v = getattr(m, f.name)
            kw[f.name] = [int(x) for x in v] if f.name.startswith("phase_") else int(v)
        return cls(**kw)

    def phases(self) -> dict:
        """{family: (launches, alg_bytes, ns)} for the families that ran."""
        return {name: (self.phase_launches[i], self.phase_bytes[i], self.phase_ns[i])
                for i, name in enumerate(_lib.PHASE_NAMES) if self.phase_launches[i]}


def _cmp_code(less: Any) -> int:
    if less in (None, "less", LESS):
        return LESS
    if less in ("greater", GREATER):
        return GREATER
    raise ValueError(f"unsupported comparator {less!r}: use 'less' or 'greater'")


def dtype_of(data: Any) -> int:
    """Map a torch tensor / numpy array to a qmsort dtype code.

    int32 -> I32, uint32 -> U32, uint64 -> U64, int64 -> I64, float64 -> F64,
    and an (n, 4) array of 64-bit words -> REC32 (records compared
    lexicographically).
    """
    name = str(data.dtype).replace("torch.", "")
    shape = tuple(data.shape)
    if len(shape) == 2 and shape[1] == 4 and name in ("uint64", "int64"):
        return DT_REC32
    if len(shape) != 1:
        raise ValueError(f"expected a 1-D array or an (n, 4) record array, got shape {shape}")
    table = {"int32": DT_I32, "uint32": DT_U32, "uint64": DT_U64, "int64": DT_I64,
             "float64": DT_F64}
    if name not in table:
        raise ValueError(f"unsupported dtype {name}")
    return table[name]


def _is_torch_cuda(x: Any) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _stream_ptr(stream: Any) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def workspace_bytes(dtype: int, n: int, cfg: SortConfig | None = None) -> int:
    lib = _lib.load()
    c = (cfg or SortConfig()).to_c()
    return int(lib.qmsort_gpu_workspace_bytes(dtype, n, ctypes.byref(c)))


def sort(data: Any, cfg: SortConfig | None = None, less: Any = "less", *, workspace: Any = None,
         stream: Any = None, dtype: int | None = None) -> Metrics:
    """Sort ``data`` ascending under ``less`` in place and return the Metrics.

    * CUDA torch tensor: sorted on its device (``qmsort_gpu_sort``); the
      optional ``workspace`` is a uint8 CUDA tensor of at least
      :func:`workspace_bytes`.
    * numpy array / CPU tensor (C-contiguous): the host drop-in call
      ``qmsort_gpu_sort_host`` copies it to the GPU, sorts and copies back.
    ``dtype`` overrides the element type inferred from the array (e.g. an
    int32 tensor holding uint32 keys).
    """
    lib = _lib.load()
    cfg = cfg or SortConfig()
    c = cfg.to_c()
    m = _lib.GpuMetrics()
    dt = dtype_of(data) if dtype is None else int(dtype)
    if lib.qmsort_gpu_dtype_size(dt) == 0:
        raise ValueError(f"unknown dtype code {dt}")
    cmp = _cmp_code(less)
    n = int(data.shape[0])
    if _is_torch_cuda(data):
        if not data.is_contiguous():
            raise ValueError("tensor must be contiguous")
        ws_ptr, ws_bytes = None, 0
        if workspace is not None:
            ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
        rc = lib.qmsort_gpu_sort(dt, cmp, data.data_ptr(), n, ctypes.byref(c), ws_ptr, ws_bytes,
                                 ctypes.byref(m), _stream_ptr(stream))
        _lib.check(rc, "qmsort_gpu_sort")
    else:
        ptr = _host_ptr(data)
        rc = lib.qmsort_gpu_sort_host(dt, cmp, ptr, n, ctypes.byref(c), ctypes.byref(m))
        _lib.check(rc, "qmsort_gpu_sort_host")
    return Metrics.from_c(m)


def sort_batch(arrays: list, cfg: SortConfig | None = None, less: Any = "less", *,
               dtype: int | None = None) -> Metrics:
    """Sort a list of independent host arrays (numpy / CPU tensors, ideally
    pinned) in place through ``qmsort_gpu_sort_host_batch``: a ring of three
    device arenas overlaps array i+1's host-to-device copy, array i's sort and
    array i-1's device-to-host copy.  Returns summed Metrics."""
    lib = _lib.load()
    c = (cfg or SortConfig()).to_c()
    m = _lib.GpuMetrics()
    if not arrays:
        return Metrics()
    dt = dtype_of(arrays[0]) if dtype is None else int(dtype)
    for a in arrays:
        if _is_torch_cuda(a):
            raise ValueError("sort_batch takes host arrays; use sort() for device tensors")
        if (dtype_of(a) if dtype is None else dt) != dt:
            raise ValueError("all arrays of a batch must share one dtype")
    ptrs = (ctypes.c_void_p * len(arrays))(*[_host_ptr(a) for a in arrays])
    ns = (ctypes.c_size_t * len(arrays))(*[int(a.shape[0]) for a in arrays])
    rc = lib.qmsort_gpu_sort_host_batch(dt, _cmp_code(less), ptrs, ns, len(arrays), ctypes.byref(c),
                                        ctypes.byref(m))
    _lib.check(rc, "qmsort_gpu_sort_host_batch")
    return Metrics.from_c(m)


def sort_range_counted(data: Any, cfg: SortConfig, metrics: Metrics, less: Any = "less") -> None:
    """sort.hpp:207-211: sort and accumulate into a caller-owned Metrics."""
    r = sort(data, cfg, less)
    metrics.elapsed_ns += r.elapsed_ns
    metrics.max_depth = max(metrics.max_depth, r.max_depth)
    metrics.alg_bytes += r.alg_bytes
    metrics.levels += r.levels
    metrics.merge_passes += r.merge_passes
    metrics.kernel_launches += r.kernel_launches
    metrics.host_syncs += r.host_syncs


def _nbytes_rows(data: Any) -> tuple[int, int]:
    """(n elements, bytes per element) of a record array: a numpy structured /
    void array, or a 2-D uint8 array or tensor of shape (n, elem_bytes)."""
    shape = tuple(data.shape)
    if type(data).__module__.startswith("torch"):
        if len(shape) != 2 or str(data.dtype) != "torch.uint8":
            raise ValueError("element tensors must be uint8 of shape (n, elem_bytes)")
        return shape[0], shape[1]
    if len(shape) == 1:
        return shape[0], int(data.dtype.itemsize)
    if len(shape) == 2 and data.dtype.itemsize == 1:
        return shape[0], shape[1]
    raise ValueError(f"unsupported element array of shape {shape} and dtype {data.dtype}")


def sort_elements(data: Any, key_dtype: int = DT_I64, cfg: SortConfig | None = None,
                  less: Any = "less", *, key_offset: int = 0, stream: Any = None) -> Metrics:
    """Sort key + payload elements in place by key alone (Element<PayloadBytes>,
    element.hpp:13-20).  ``key_dtype`` is the type of the key at byte
    ``key_offset`` of every element (int64 in the reference profile).  Equal
    keys keep their input order; the key sequence equals the reference's."""
    lib = _lib.load()
    c = (cfg or SortConfig()).to_c()
    m = _lib.GpuMetrics()
    cmp = _cmp_code(less)
    n, eb = _nbytes_rows(data)
    if _is_torch_cuda(data):
        if not data.is_contiguous():
            raise ValueError("tensor must be contiguous")
        rc = lib.qmsort_gpu_sort_elements(int(key_dtype), cmp, data.data_ptr(), n, eb, key_offset,
                                          ctypes.byref(c), None, 0, ctypes.byref(m),
                                          _stream_ptr(stream))
        _lib.check(rc, "qmsort_gpu_sort_elements")
    else:
        rc = lib.qmsort_gpu_sort_elements_host(int(key_dtype), cmp, _host_ptr(data), n, eb,
                                               key_offset, ctypes.byref(c), ctypes.byref(m))
        _lib.check(rc, "qmsort_gpu_sort_elements_host")
    return Metrics.from_c(m)


def select_nth(data: Any, k: int, cmp: Any = "less", metrics: Metrics | None = None,
               cfg: SortConfig | None = None, *, dtype: int | None = None,
               stream: Any = None) -> int:
    """selection.hpp:207-212: place the k-th smallest (1-based k) under ``cmp``
    at its sorted position, with everything left of it <= and right of it >=,
    and return that position (k - 1).  Accumulates into ``metrics`` if given."""
    lib = _lib.load()
    c = (cfg or SortConfig()).to_c()
    m = _lib.GpuMetrics()
    dt = dtype_of(data) if dtype is None else int(dtype)
    n = int(data.shape[0])
    pos = ctypes.c_size_t(0)
    if _is_torch_cuda(data):
        if not data.is_contiguous():
            raise ValueError("tensor must be contiguous")
        rc = lib.qmsort_gpu_select_nth(dt, _cmp_code(cmp), data.data_ptr(), n, int(k),
                                       ctypes.byref(pos), ctypes.byref(c), None, 0,
                                       ctypes.byref(m), _stream_ptr(stream))
        _lib.check(rc, "qmsort_gpu_select_nth")
    else:
        rc = lib.qmsort_gpu_select_nth_host(dt, _cmp_code(cmp), _host_ptr(data), n, int(k),
                                            ctypes.byref(pos), ctypes.byref(c), ctypes.byref(m))
        _lib.check(rc, "qmsort_gpu_select_nth_host")
    if metrics is not None:
        r = Metrics.from_c(m)
        metrics.elapsed_ns += r.elapsed_ns
        metrics.max_depth = max(metrics.max_depth, r.max_depth)
        metrics.levels += r.levels
        metrics.kernel_launches += r.kernel_launches
    return int(pos.value)


@dataclasses.dataclass
class PartitionResult:
    """partition_result.hpp:12-17: [0, lt_end) < pivot, [lt_end, gt_begin) ==
    pivot, [gt_begin, n) > pivot under the comparator."""

    lt_end: int = 0
    gt_begin: int = 0
    left_size: int = 0
    right_size: int = 0


def partition(data: Any, pivot: Any, less: Any = "less", cfg: SortConfig | None = None, *,
              dtype: int | None = None, stream: Any = None) -> PartitionResult:
    """Three-way partition of ``data`` around the pivot value in place on the
    GPU (``qmsort_gpu_partition3``; the contract of three_way_partition,
    partition.hpp:196-230).  ``pivot`` is a scalar (or a 4-word record)."""
    import numpy as np
    lib = _lib.load()
    c = (cfg or SortConfig()).to_c()
    m = _lib.GpuMetrics()
    dt = dtype_of(data) if dtype is None else int(dtype)
    npdt = {DT_I32: np.int32, DT_U32: np.uint32, DT_U64: np.uint64, DT_F64: np.float64, DT_I64: np.int64,
            DT_REC32: np.uint64}[dt]
    pv = np.ascontiguousarray(np.asarray(pivot, dtype=npdt).reshape(-1))
    if pv.nbytes != lib.qmsort_gpu_dtype_size(dt):
        raise ValueError("pivot must be one element of the array's type")
    cnt = (ctypes.c_uint64 * 3)()
    n = int(data.shape[0])
    if _is_torch_cuda(data):
        if not data.is_contiguous():
            raise ValueError("tensor must be contiguous")
        rc = lib.qmsort_gpu_partition3(dt, _cmp_code(less), data.data_ptr(), n, pv.ctypes.data, cnt,
                                       ctypes.byref(c), None, 0, ctypes.byref(m), _stream_ptr(stream))
        _lib.check(rc, "qmsort_gpu_partition3")
    else:
        rc = lib.qmsort_gpu_partition3_host(dt, _cmp_code(less), _host_ptr(data), n, pv.ctypes.data, cnt,
                                            ctypes.byref(c), ctypes.byref(m))
        _lib.check(rc, "qmsort_gpu_partition3_host")
    c0, c1, c2 = int(cnt[0]), int(cnt[1]), int(cnt[2])
    return PartitionResult(c0, c0 + c1, c0, c2)


def _host_ptr(data: Any) -> int:
    if type(data).__module__.startswith("torch"):
        if not data.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return data.data_ptr()
    if not data.flags["C_CONTIGUOUS"] or not data.flags["WRITEABLE"]:
        raise ValueError("array must be C-contiguous and writeable")
    return data.ctypes.data


# ---------------------------------------------------------------------------
# Harness helpers (K9 generators and verification), used by bench.py / tests.
# ---------------------------------------------------------------------------
GEN_U32, GEN_U64, GEN_REC32 = 0, 1, 2
GEN_F64_SORTED, GEN_F64_REVERSE, GEN_F64_DISTINCT16, GEN_F64_GAUSS, GEN_F64_ORGAN = 10, 11, 12, 13, 14


def generate(kind: int, out: Any, seed: int, start: int = 0, total: int | None = None,
             stream: Any = None) -> None:
    """Fill CUDA tensor ``out`` with global elements [start, start+n) of a seeded config."""
    lib = _lib.load()
    n = int(out.shape[0])
    rc = lib.qmsort_gpu_generate(kind, out.data_ptr(), n, seed, start, total or n,
                                 _stream_ptr(stream))
    _lib.check(rc, "qmsort_gpu_generate")


def check(data: Any, less: Any = "less", order: bool = True, stream: Any = None) -> tuple[int, int, int]:
    """(order violations, multiset sum fingerprint, multiset xor fingerprint) of a CUDA tensor."""
    lib = _lib.load()
    out = (ctypes.c_uint64 * 3)()
    rc = lib.qmsort_gpu_check(dtype_of(data), _cmp_code(less), data.data_ptr(), int(data.shape[0]),
                              int(order), out, _stream_ptr(stream))
    _lib.check(rc, "qmsort_gpu_check")
    return int(out[0]), int(out[1]), int(out[2])
