"""ctypes binding of the C-ABI in include/qmsort_gpu.h.

The shared library ``libqmsort_gpu.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, sm_100a).  There is no CPU fallback: if the
library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QMSORT_GPU_LIB") or os.path.join(_HERE, "libqmsort_gpu.so")

QMSORT_OK = 0
QMSORT_EINVAL = 1
QMSORT_ENOWS = 2
QMSORT_ECUDA = 3
QMSORT_ENCCL = 4
QMSORT_EINTERNAL = 5

DT_I32, DT_U32, DT_U64, DT_F64, DT_REC32, DT_I64 = 0, 1, 2, 3, 4, 5
LESS, GREATER = 0, 1


class GpuConfig(ctypes.Structure):
    """qmsort_gpu_config (mirrors SortConfig, sort.hpp:25-34)."""

    _fields_ = [
        ("variant", ctypes.c_int),
        ("pivot", ctypes.c_int),
        ("base_case_kind", ctypes.c_int),
        ("base_case_size_threshold", ctypes.c_uint64),
        ("base_case_use_levels", ctypes.c_int),
        ("beta", ctypes.c_double),
        ("delta", ctypes.c_double),
        ("side", ctypes.c_int),
        ("three_way", ctypes.c_int),
        ("block", ctypes.c_uint64),
        ("algorithm", ctypes.c_int),
        ("seed", ctypes.c_uint64),
        ("max_levels", ctypes.c_int),
        ("profile", ctypes.c_int),
    ]


NUM_PHASES = 8
PHASE_NAMES = ["transform", "sample", "count", "plan", "scatter", "blocksort", "merge", "fill"]


class GpuMetrics(ctypes.Structure):
    """qmsort_gpu_metrics (Metrics, metrics.hpp:14-24, plus the pass ledger)."""

    _fields_ = [
        ("comparisons", ctypes.c_uint64),
        ("moves", ctypes.c_uint64),
        ("max_depth", ctypes.c_uint64),
        ("elapsed_ns", ctypes.c_uint64),
        ("alg_bytes", ctypes.c_uint64),
        ("levels", ctypes.c_uint32),
        ("merge_passes", ctypes.c_uint32),
        ("kernel_launches", ctypes.c_uint32),
        ("host_syncs", ctypes.c_uint32),
        ("phase_bytes", ctypes.c_uint64 * 8),
        ("phase_ns", ctypes.c_uint64 * 8),
        ("phase_launches", ctypes.c_uint32 * 8),
        ("resplits", ctypes.c_uint32),
        ("sample_keys", ctypes.c_uint64),
        ("table_buckets", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]


EXPORTED = [
    "qmsort_gpu_config_init",
    "qmsort_gpu_workspace_bytes",
    "qmsort_gpu_sort",
    "qmsort_gpu_sort_host",
    "qmsort_gpu_last_error",
    "qmsort_gpu_dtype_size",
    "qmsort_gpu_transform",
    "qmsort_gpu_core_dtype",
    "qmsort_gpu_sample",
    "qmsort_gpu_partition_workspace_bytes",
    "qmsort_gpu_partition",
    "qmsort_gpu_generate",
    "qmsort_gpu_check",
    "qmsort_gpu_version",
    "qmsort_gpu_abi_sizes",
    "qmsort_gpu_elements_workspace_bytes",
    "qmsort_gpu_sort_elements",
    "qmsort_gpu_sort_elements_host",
    "qmsort_gpu_select_workspace_bytes",
    "qmsort_gpu_select_nth",
    "qmsort_gpu_select_nth_host",
    "qmsort_gpu_sort_host_batch",
    "qmsort_gpu_ipc_handle",
    "qmsort_gpu_ipc_open",
    "qmsort_gpu_ipc_close",
    "qmsort_gpu_sort_sharded",
    "qmsort_gpu_shard_workspace_bytes",
    "qmsort_gpu_shard_sample",
    "qmsort_gpu_shard_splitters",
    "qmsort_gpu_shard_count",
    "qmsort_gpu_shard_plan",
    "qmsort_gpu_shard_scatter",
    "qmsort_gpu_shard_finish",
    "qmsort_gpu_shard_subbuckets",
    "qmsort_gpu_shard_plan_folded",
    "qmsort_gpu_shard_finish_presplit",
    "qmsort_gpu_partition3_workspace_bytes",
    "qmsort_gpu_partition3",
    "qmsort_gpu_partition3_host",
]

_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"qmsort-b200 CUDA library not built: {p} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
        )
    lib = ctypes.CDLL(p)
    vp, sz, u64, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int
    u32, i32 = ctypes.c_uint32, ctypes.c_int32
    cfgp, mp = ctypes.POINTER(GpuConfig), ctypes.POINTER(GpuMetrics)
    sig = {
        "qmsort_gpu_config_init": (None, [cfgp, i]),
        "qmsort_gpu_workspace_bytes": (sz, [i, sz, cfgp]),
        "qmsort_gpu_sort": (i, [i, i, vp, sz, cfgp, vp, sz, mp, vp]),
        "qmsort_gpu_sort_host": (i, [i, i, vp, sz, cfgp, mp]),
        "qmsort_gpu_last_error": (ctypes.c_char_p, []),
        "qmsort_gpu_dtype_size": (sz, [i]),
        "qmsort_gpu_transform": (i, [i, i, vp, sz, i, vp]),
        "qmsort_gpu_core_dtype": (i, [i]),
        "qmsort_gpu_sample": (i, [i, vp, sz, sz, u64, vp, vp]),
        "qmsort_gpu_partition_workspace_bytes": (sz, [i, sz]),
        "qmsort_gpu_partition": (i, [i, vp, sz, vp, ctypes.c_uint32, vp, vp, vp, sz, vp]),
        "qmsort_gpu_generate": (i, [i, vp, sz, u64, u64, u64, vp]),
        "qmsort_gpu_check": (i, [i, i, vp, sz, i, ctypes.POINTER(u64), vp]),
        "qmsort_gpu_version": (ctypes.c_char_p, []),
        "qmsort_gpu_elements_workspace_bytes": (sz, [sz, sz]),
        "qmsort_gpu_sort_elements": (i, [i, i, vp, sz, sz, sz, cfgp, vp, sz, mp, vp]),
        "qmsort_gpu_sort_elements_host": (i, [i, i, vp, sz, sz, sz, cfgp, mp]),
        "qmsort_gpu_select_workspace_bytes": (sz, [i, sz]),
        "qmsort_gpu_select_nth": (i, [i, i, vp, sz, sz, ctypes.POINTER(sz), cfgp, vp, sz, mp, vp]),
        "qmsort_gpu_select_nth_host": (i, [i, i, vp, sz, sz, ctypes.POINTER(sz), cfgp, mp]),
        "qmsort_gpu_sort_host_batch": (i, [i, i, ctypes.POINTER(vp), ctypes.POINTER(sz), sz, cfgp, mp]),
        "qmsort_gpu_ipc_handle": (i, [vp, vp, ctypes.POINTER(u64)]),
        "qmsort_gpu_ipc_open": (i, [vp, u64, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "qmsort_gpu_ipc_close": (i, [vp]),
        "qmsort_gpu_sort_sharded": (i, [i, i, u32, ctypes.POINTER(i), ctypes.POINTER(vp), ctypes.POINTER(sz),
                                        ctypes.POINTER(vp), ctypes.POINTER(sz), ctypes.POINTER(sz), cfgp, mp]),
        "qmsort_gpu_shard_workspace_bytes": (sz, [i, sz]),
        "qmsort_gpu_shard_sample": (i, [i, i, vp, sz, sz, u64, vp, vp]),
        "qmsort_gpu_shard_splitters": (i, [i, vp, sz, u32, vp, ctypes.POINTER(u32), ctypes.POINTER(u32)]),
        "qmsort_gpu_shard_count": (i, [i, i, vp, sz, vp, u32, i, vp, vp, sz, vp]),
        "qmsort_gpu_shard_plan": (i, [u32, u32, ctypes.POINTER(u32), ctypes.POINTER(u64), ctypes.POINTER(i32),
                                      ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64),
                                      ctypes.POINTER(u64), ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "qmsort_gpu_shard_scatter": (i, [i, i, vp, sz, u32, i, ctypes.POINTER(i32), ctypes.POINTER(u64),
                                         ctypes.POINTER(vp), ctypes.POINTER(u64), u32, i, vp, sz, vp]),
        "qmsort_gpu_shard_subbuckets": (u32, [i, u32, u64]),
        "qmsort_gpu_shard_plan_folded": (i, [u32, u32, u32, ctypes.POINTER(u32), ctypes.POINTER(u64),
                                             ctypes.POINTER(i32), ctypes.POINTER(u64), ctypes.POINTER(u64),
                                             ctypes.POINTER(u32), ctypes.POINTER(i32), ctypes.POINTER(u64)]),
        "qmsort_gpu_shard_finish_presplit": (i, [i, i, vp, sz, vp, u32, ctypes.POINTER(u64), cfgp, vp, sz, mp, vp]),
        "qmsort_gpu_shard_finish": (i, [i, i, vp, sz, vp, i32, u64, i32, u64, vp, cfgp, vp, sz, mp, vp]),
        "qmsort_gpu_partition3_workspace_bytes": (sz, [i, sz]),
        "qmsort_gpu_partition3": (i, [i, i, vp, sz, vp, ctypes.POINTER(u64), cfgp, vp, sz, mp, vp]),
        "qmsort_gpu_partition3_host": (i, [i, i, vp, sz, vp, ctypes.POINTER(u64), cfgp, mp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


class QmsortError(RuntimeError):
    """A nonzero C-ABI status, like the reference harness's runtime_error (trial.hpp:116)."""

    def __init__(self, code: int, where: str):
        msg = load().qmsort_gpu_last_error().decode(errors="replace")
        super().__init__(f"{where} failed with status {code}: {msg}")
        self.code = code


def check(code: int, where: str) -> None:
    if code != QMSORT_OK:
        raise QmsortError(code, where)
