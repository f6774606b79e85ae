"""Probe: do two independent sorts on two streams overlap on one B200?
Times S sequential sorts of n keys vs the same sorts split over two host
threads / streams (the kernels are pipe-bound on different pipes: the
partition on shared memory, the block sort on the ALU)."""
import sys, threading, time
import torch
sys.path.insert(0, ".")
import paper_1804_10062_b200 as q

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
S = 8
src = torch.empty(n, dtype=torch.uint32, device="cuda")
q.generate(q.GEN_U32, src, seed=42)
xs = [torch.empty_like(src) for _ in range(S)]
cfg = q.qms()
streams = [torch.cuda.Stream() for _ in range(2)]
ws = [torch.empty(q.workspace_bytes(q.DT_U32, n, cfg), dtype=torch.uint8, device="cuda") for _ in range(2)]

def run(ids, k):
    for i in ids:
        q.sort(xs[i], cfg, workspace=ws[k], stream=streams[k])
    streams[k].synchronize()

for rep in range(3):
    for x in xs: x.copy_(src)
    torch.cuda.synchronize(); t = time.perf_counter(); run(range(S), 0); torch.cuda.synchronize()
    seq = time.perf_counter() - t
    for x in xs: x.copy_(src)
    torch.cuda.synchronize(); t = time.perf_counter()
    th = [threading.Thread(target=run, args=(range(k, S, 2), k)) for k in range(2)]
    [h.start() for h in th]; [h.join() for h in th]
    torch.cuda.synchronize()
    par = time.perf_counter() - t
    print(f"n={n} {S} sorts: sequential {seq*1e3/S:.3f} ms/sort, two streams {par*1e3/S:.3f} ms/sort ({seq/par:.2f}x)")
