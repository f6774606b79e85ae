"""Where the sharded path's time goes at P = 1 (exchange to itself): the
phases of sharded.sort_sharded(force_exchange=True), timed with a device
sync around each (so the sum exceeds the pipelined step time)."""
import os, sys, time
import torch
import torch.distributed as dist
sys.path.insert(0, ".")
import paper_1804_10062_b200 as q
from paper_1804_10062_b200 import sharded as S

for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533")):
    os.environ.setdefault(k, v)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = 1 << 28
src = torch.empty(n, dtype=torch.uint32, device="cuda")
q.generate(q.GEN_U32, src, seed=42)
ex, ops = S.PeerExchange(), S.GpuOps()
core, dt, cmp = q.DT_U32, q.DT_U32, 0
T = {}
def tick(name, t0):
    torch.cuda.synchronize(); T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3; return time.perf_counter()
for rep in range(4):
    if rep == 1: T.clear()
    x = src.clone(); torch.cuda.synchronize(); dist.barrier()
    t = time.perf_counter(); t00 = t
    w = S._wire(x, core); ops.to_core(w, dt, cmp); t = tick("to_core", t)
    smp = ops.sample(w, core, 64, 42); t = tick("sample", t)
    all_smp = ex.all_gather(smp).contiguous(); t = tick("all_gather samples", t)
    ops.sort(all_smp, core); spl = S.pick_splitters(all_smp, 1); t = tick("sort samples + splitters", t)
    counts = ops.partition_count(w, core, spl); t = tick("partition_count", t)
    allc = ex.all_gather(counts); C = allc.view(1, 1).cpu().tolist(); t = tick("all_gather counts", t)
    totals, offs = S._bucket_offsets(C, 1, 0); ex.ensure_capacity(max(totals) * 4, w.device); ex.barrier(); t = tick("capacity + barrier", t)
    ops.scatter_peers(w, core, 0, ex.ptrs, offs); t = tick("scatter_peers", t)
    ex.barrier(); t = tick("barrier", t)
    got = ex.recv[: totals[0] * 4].view(w.dtype).view((totals[0],))
    ops.sort(got, core); t = tick("local sort", t)
    ops.to_core(got, dt, cmp, inverse=True); t = tick("inverse", t)
    T["TOTAL"] = T.get("TOTAL", 0) + (t - t00) * 1e3
for k, v in T.items(): print(f"{k:26s} {v / 3:8.3f} ms")
