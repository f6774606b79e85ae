#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for qmsort-b200.

Workload (BASELINE.json metric, config 2): sort n = 2^28 uint32 keys drawn
i.i.d. uniform by the seeded SplitMix64 recipe, Median-of-3
preset qms(), one sort per step, keys resident in HBM.  Output:
one JSON line with the metric "sorted Gkeys/s at n=2^28 uint32" plus the
roofline of the dominant kernel, the pass-ledger roofline of the whole sort,
the reference CPU QuickMergesort timed on the host cores (cpu_baseline) and
the end-to-end number through the host-array drop-in call (e2e).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With N > 1 every rank is one process on one GPU (launched by the driver under
torchrun, or -- when WORLD_SIZE is unset -- by bench.py re-executing itself
under torch.distributed.run) and the ranks run the distributed samplesort
(sharded.py): global splitters, the exchange fused into the partition's
scatter (peer stores over NVLink), local sorts.  Default: the C2 recipe with
2^28 uint32 keys per GPU (weak scaling, whole-job keys/s); --config c3 / c5:
the north-star sharded configs, 2^30 uint64 keys / 2^26 32-byte records in
total (strong scaling).  --sharded runs that path at N = 1 too.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted Gkeys/s at n=2^28 uint32 (1-8 B200); achieved HBM GB/s vs roofline"
UNIT = "Gkeys/s"
N_DEFAULT = 1 << 28
SEED = 42
CPU_WARM = 1 << 24  # reference-arm warm-up sorts: a 2^24 prefix
# BASELINE.json configs runnable with device generators: (dtype attr, torch dtype,
# row shape, generator attr, n, key bytes, description)
CONFIGS = {
    "c2": ("DT_U32", "uint32", (), "GEN_U32", 1 << 28, 4, "C2: sort n=2^28 uint32 i.i.d. uniform"),
    "c3": ("DT_U64", "uint64", (), "GEN_U64", 1 << 30, 8, "C3: sort n=2^30 uint64 i.i.d. uniform"),
    "c4a": ("DT_F64", "float64", (), "GEN_F64_SORTED", 1 << 27, 8, "C4a: 2^27 float64 sorted"),
    "c4b": ("DT_F64", "float64", (), "GEN_F64_REVERSE", 1 << 27, 8, "C4b: 2^27 float64 reverse"),
    "c4c": ("DT_F64", "float64", (), "GEN_F64_DISTINCT16", 1 << 27, 8, "C4c: 2^27 float64 16 distinct"),
    "c4d": ("DT_F64", "float64", (), "GEN_F64_GAUSS", 1 << 27, 8, "C4d: 2^27 float64 gaussian"),
    "c4e": ("DT_F64", "float64", (), "GEN_F64_ORGAN", 1 << 27, 8, "C4e: 2^27 float64 organ-pipe"),
    "c5": ("DT_REC32", "uint64", (4,), "GEN_REC32", 1 << 26, 32, "C5: 2^26 32-byte records"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", "--keys", dest="n", type=int, default=N_DEFAULT, help="keys per GPU")
    ap.add_argument("--algorithm", choices=["samplesort", "mergesort"], default="samplesort")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling runs: skip extras")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2",
                    help="BASELINE config (c2 is the headline; the others are informational; "
                         "c3 / c5 are the sharded north-star configs with --gpus N / --sharded)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the distributed samplesort path even on one GPU (exercises NCCL)")
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                    help="sharded path: exchange fused into the scatter (CUDA IPC peer stores) "
                         "or a NCCL all-to-all after the partition")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in rows),
                "sm_max_mhz": max(int(r[1]) for r in rows), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU legs: the reference QuickMergesort (oracle/_ref) or the C restatement
# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_lib():
    """The reference QuickMergesort on this host: the reference headers
    compiled here with -O3 -march=native -funroll-loops from the preprocessed
    translation unit (oracle/_ref/ref_shim.ii, `make -C oracle native`), else
    the prebuilt -O3 build (oracle/_ref/libqmsref.so), else the C restatement."""
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    paths = []
    if os.path.exists(os.path.join(ref_dir, "ref_shim.ii")):
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "native"],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        if r.returncode == 0:
            paths.append((os.path.join(ref_dir, "libqmsref_native.so"), "-O3 -march=native -funroll-loops"))
    paths.append((os.path.join(ref_dir, "libqmsref.so"), "-O3 (prebuilt)"))
    for ref, flags in paths:
        if os.path.exists(ref):
            lib = ctypes.CDLL(ref)
            lib.qmsref_sort.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
            return "reference", flags, lambda a, std=False: lib.qmsref_sort(
                1, 0, 0, 0, int(std), a.ctypes.data_as(ctypes.c_void_p), a.shape[0], None)
    port = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = ctypes.CDLL(port)
    lib.qmso_sort.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    return "port", "-O3", lambda a, std=False: lib.qmso_sort(1, 0, 0, a.ctypes.data_as(ctypes.c_void_p), a.shape[0])


def host_input(n: int):
    """C2 recipe on the host: u32[i] = SplitMix64(seed)_i >> 32 (numpy, vectorised, in blocks)."""
    import numpy as np
    out = np.empty(n, dtype=np.uint32)
    blk = 1 << 24
    for s0 in range(0, n, blk):
        m = min(blk, n - s0)
        j = np.arange(s0 + 1, s0 + m + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(SEED) + j * np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        out[s0:s0 + m] = (z >> np.uint64(32)).astype(np.uint32)
    return out


class PinnedCore:
    """Run the single-threaded reference on one host core (the reference
    cannot use more than one thread per sort)."""

    def __init__(self):
        self.core = None
        self.prev = None

    def __enter__(self):
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = max(self.prev)  # the last allowed core (core 0 takes the interrupts)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)


def cpu_baseline(n: int = N_DEFAULT) -> dict:
    """The reference qms() and std::sort on the SAME host array the GPU sorts
    (the full C2 input), one sort each, pinned to one core."""
    kind, flags, fn = cpu_lib()
    base = host_input(n)
    a = base.copy()
    with PinnedCore() as pc:
        t = time.perf_counter()
        fn(a)
        qms_s = time.perf_counter() - t
        a[:] = base
        t = time.perf_counter()
        if kind == "reference":
            fn(a, std=True)
        std_s = time.perf_counter() - t if kind == "reference" else None
    return {"value": n / qms_s / 1e9, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"qmsort::sort(qms(), std::less) on the full C2 array (2^{n.bit_length() - 1} uint32, the "
                      f"GPU's input), one sort, single-threaded reference built {flags}, pinned to core "
                      f"{pc.core} of {os.cpu_count()} ({cpu_model()})",
            "seconds": qms_s, "std_sort_value": (n / std_s / 1e9) if std_s else None,
            "std_sort_seconds": std_s, "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
            "build_flags": flags}


def run_reference(args) -> None:
    """--impl reference: the reference CPU QuickMergesort on the host, on our
    arm's workload: every timed step sorts a fresh copy of the full 2^28 C2
    array (single-threaded, pinned to one core).  The W warm-up steps sort a
    2^24 prefix (a CPU sort has nothing to warm beyond caches and pages)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind, flags, fn = cpu_lib()
    n = args.n
    base = host_input(n)
    a = base.copy()
    times, std_s = [], None
    with PinnedCore() as pc:
        for _ in range(args.warmup):
            w = base[: min(n, CPU_WARM)].copy()
            fn(w)
        for _ in range(args.steps):
            a[:] = base
            t = time.perf_counter()
            fn(a)
            times.append(time.perf_counter() - t)
        if kind == "reference":
            a[:] = base
            t = time.perf_counter()
            fn(a, std=True)
            std_s = time.perf_counter() - t
    ms = statistics.mean(times) * 1e3
    value = n / (ms / 1e3) / 1e9
    sample = (f"each step: qmsort::sort(qms(), std::less) of a fresh copy of the full C2 array (2^{n.bit_length() - 1} "
              f"uint32, the workload our arm sorts); single-threaded reference built {flags}, pinned to core "
              f"{pc.core} of {os.cpu_count()} ({cpu_model()}); warm-up steps sort a 2^24 prefix")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded SplitMix64, SURVEY.md 8(d) C2 recipe, seed 42)",
            "config": workload_config(n),
            "impl": "reference",
            "step_ms": [round(t * 1e3, 1) for t in times],
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
                             "cpu_model": cpu_model(), "host_cores": os.cpu_count(), "build_flags": flags,
                             "std_sort_value": (n / std_s / 1e9) if std_s else None},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(n: int) -> dict:
    """The workload both arms run (BASELINE.json configs[1])."""
    return {"workload": f"C2: sort n=2^{n.bit_length() - 1} uint32 i.i.d. uniform (seeded SplitMix64, seed 42), "
                        "qms() preset", "n": n, "key_bytes": 4}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args) -> None:
    import torch

    import paper_1804_10062_b200 as q

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if os.environ.get("QMSORT_BENCH_ONE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        from paper_1804_10062_b200 import sharded
        sharded.bench_main(args, METRIC, UNIT)
        return

    dt_name, tdt, rowshape, gen_name, n_cfg, kb, desc = CONFIGS[args.config]
    dt = getattr(q, dt_name)
    n = args.n if args.config == "c2" else (n_cfg if args.n == N_DEFAULT else args.n)
    if args.config != "c2":  # informational configs: device numbers only
        args.no_e2e = args.no_cpu_baseline = True
    dev = torch.device("cuda", local)
    pristine = torch.empty((n,) + rowshape, dtype=getattr(torch, tdt), device=dev)
    q.generate(getattr(q, gen_name), pristine, seed=SEED)
    x = torch.empty_like(pristine)
    cfg = q.qms()
    if args.algorithm == "mergesort":
        cfg.algorithm = q.Algorithm.mergesort
    ws = torch.empty(q.workspace_bytes(dt, n, cfg), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step():
        x.copy_(pristine)
        flush.zero_()
        torch.cuda.synchronize()
        e0.record(stream)
        m = q.sort(x, cfg, workspace=ws, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), m

    for _ in range(max(1, args.warmup)):  # at least one untimed sort to verify
        step()
    # correctness of the benchmarked sort (untimed): sorted + same multiset
    viol, s_out, x_out = q.check(x)
    _, s_in, x_in = q.check(pristine, order=False)
    if viol != 0 or s_out != s_in or x_out != x_in:
        raise RuntimeError(f"benchmarked sort is wrong: {viol} order violations / multiset mismatch")

    torch.cuda.synchronize()
    clocks = Clocks(local)
    times, launches, metrics = [], 0, None
    for _ in range(args.steps):
        t, m = step()
        times.append(t)
        launches += m.kernel_launches
        metrics = m
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = statistics.mean(times)
    value = n / (ms / 1e3) / 1e9

    # per-kernel-family device time (untimed profiling run with events per launch)
    pcfg = q.qms()
    pcfg.algorithm = cfg.algorithm
    pcfg.profile = True
    prof = None
    for _ in range(2):
        x.copy_(pristine)
        flush.zero_()
        torch.cuda.synchronize()
        prof = q.sort(x, pcfg, workspace=ws, stream=stream)
    peak, peak_src = peaks()
    phases = prof.phases()
    dom = max(phases.items(), key=lambda kv: kv[1][2])
    dom_name, (dom_launches, dom_bytes, dom_ns) = dom
    achieved = dom_bytes / dom_ns if dom_ns else 0.0  # bytes/ns == GB/s
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(dom_name)
    sort_bytes = metrics.alg_bytes
    sort_gbs = sort_bytes / (ms * 1e6)
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "alg_bytes_per_launch": dom_bytes / max(1, dom_launches),
                "launches": dom_launches, "avg_launch_us": dom_ns / max(1, dom_launches) / 1e3,
                "peak_source": peak_src}
    sort_roofline = {"alg_bytes": sort_bytes, "achieved": sort_gbs, "peak": peak, "unit": "GB/s",
                     "frac": sort_gbs / peak,
                     "floor_frac": 4 * n * kb / (ms * 1e6) / peak,
                     "ledger_bytes_over_nw": sort_bytes / (n * kb),
                     "levels": metrics.levels,
                     "phases": {k: {"launches": v[0], "alg_bytes": v[1], "us": v[2] / 1e3,
                                    "GBps": (v[1] / v[2]) if v[2] else None}
                                for k, v in phases.items()}}

    metric = METRIC if args.config == "c2" else f"sorted Gkeys/s, {desc} (informational)"
    line = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": {"DT_U32": "u32", "DT_U64": "u64", "DT_F64": "f64", "DT_REC32": "4xu64"}[dt_name],
            "data": f"synthetic (seeded SplitMix64, SURVEY.md 8(d) {args.config.upper()} recipe, seed 42)",
            "config": (workload_config(n) if args.config == "c2"
                       else {"workload": f"{desc}, qms() preset", "n": n, "key_bytes": kb}),
            "setup": {"algorithm": args.algorithm, "parallelism": "single B200",
                      "l2": "flushed (256 MiB write) before every timed step; input > L2"},
            "step_ms": [round(t, 4) for t in times],
            "gpu_launches": launches, "clocks": clk, "roofline": roofline,
            "sort_roofline": sort_roofline}

    if not args.no_e2e:
        line["e2e"] = e2e(q, torch, n, pristine, cfg, args)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(n)
    print(json.dumps(line), flush=True)


def e2e(q, torch, n, pristine, cfg, args) -> dict:
    """Same metric through the host-array API: every step sorts its own pinned
    host copy of the input and H2D + sort + D2H of every step lie inside the
    timed region.  The steps go through qmsort_gpu_sort_host_batch (a stream of
    independent sort requests): a ring of three device arenas keeps both PCIe
    copy engines busy (step i+1 in, step i sorting, step i-1 out).  The single-call latency of
    qmsort_gpu_sort_host is reported alongside (sync_ms_per_step)."""
    host_src = pristine.cpu()
    # up to 12 arrays per batch call (the ring's fill and drain -- one H2D and
    # one D2H that overlap nothing -- are part of the timed call: over 6 arrays
    # they add 1/6 to the per-step time, over 12 1/12); 6 if the host cannot
    # pin that much memory
    steps = max(2, min(args.steps, 12))
    try:
        bufs = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(steps)]
    except RuntimeError:
        bufs = None
        torch.cuda.empty_cache()
        steps = max(2, min(args.steps, 6))
    if bufs is None:
        bufs = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(steps)]
    for b in bufs:
        b.copy_(host_src)
    warm = [torch.empty(n, dtype=torch.uint32, pin_memory=True) for _ in range(2)]
    for w in warm:
        w.copy_(host_src)
    q.sort_batch(warm, cfg)  # allocates the batch arenas
    t = time.perf_counter()
    q.sort_batch(bufs, cfg)
    ms = (time.perf_counter() - t) / steps * 1e3
    # correctness of what came back: sorted + same multiset as the input
    for b in bufs[:2]:
        d = b.cuda()
        viol, s_out, x_out = q.check(d)
        _, s_in, x_in = q.check(pristine, order=False)
        if viol or s_out != s_in or x_out != x_in:
            raise RuntimeError("e2e sort returned a wrong result")
    # single-call latency (one thread, nothing overlapped); the first call
    # allocates the calling thread's device arena, so warm it up once
    warm[1].copy_(host_src)
    q.sort(warm[1], cfg)
    warm[0].copy_(host_src)
    t = time.perf_counter()
    q.sort(warm[0], cfg)
    sync_ms = (time.perf_counter() - t) * 1e3
    return {"value": n / (ms / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": n * 4, "d2h_bytes_per_step": n * 4,
            "steps": steps, "sync_ms_per_step": sync_ms,
            "api": "qmsort_gpu_sort_host_batch (C-ABI, host arrays) over pinned host buffers, "
                   "one array per step"}


def relaunch_under_torchrun(args) -> None:
    """--gpus N > 1 without a torchrun environment: re-execute this script as N
    ranks (one process per GPU) through torch.distributed.run; rank 0 prints
    the line."""
    import socket

    import torch
    have = torch.cuda.device_count() if args.impl == "ours" else args.gpus
    if os.environ.get("QMSORT_BENCH_ONE_GPU") == "1":  # test aid: every rank on GPU 0
        have = args.gpus
    if have < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} GPU(s) visible")
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    # "--n" would be taken for an abbreviation of torchrun's own options
    own = ["--keys" if a == "--n" else ("--keys=" + a[4:] if a.startswith("--n=") else a) for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *own]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.quick:
        args.no_cpu_baseline = True
        args.no_e2e = True
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
