"""Debug helper: C2 sort through the library in QMSORT_GPU_LIB, locate order violations."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1804_10062_b200 as q
n = 1 << 28
p = torch.empty(n, dtype=torch.uint32, device="cuda")
q.generate(q.GEN_U32, p, seed=42)
ref = torch.sort(p.view(torch.int32) ^ torch.tensor(-2**31, dtype=torch.int32, device="cuda")).values ^ torch.tensor(-2**31, dtype=torch.int32, device="cuda")
for trial in range(3):
    x = p.clone()
    q.sort(x, q.qms())
    bad = torch.nonzero(x.view(torch.int32) != ref).flatten()
    print("trial", trial, "mismatches", bad.numel(), bad[:10].tolist())
    if bad.numel():
        i = bad[0].item()
        print(" got", x[i-3:i+4].tolist(), "\n want", ref[i-3:i+4].view(torch.uint32).tolist() if False else (ref[i-3:i+4].to(torch.int64) & 0xFFFFFFFF).tolist())
