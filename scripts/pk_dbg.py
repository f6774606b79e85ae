import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1804_10062_b200 as q
bad = 0
rng = np.random.default_rng(1)
for m in [2, 3, 31, 32, 33, 500, 511, 512, 513, 1000, 1024, 1025, 1500, 2047, 2048, 2049, 3000, 4095, 4096, 4097, 6000, 8192, 8193, 12000, 16384]:
    for span in [1, 100, 65535, 65536]:
        for rep in range(3):
            base = int(rng.integers(0, 2**32 - 70000))
            a = (base + rng.integers(0, span + 1, size=m)).astype(np.uint32)
            t = torch.from_numpy(a.copy()).cuda()
            q.sort(t, q.qms())
            g = t.cpu().numpy()
            w = np.sort(a)
            if not np.array_equal(g, w):
                bad += 1
                d = np.nonzero(g != w)[0]
                print("BAD m", m, "span", span, "first diff", d[:5], g[d[:3]], w[d[:3]])
print("bad", bad)
