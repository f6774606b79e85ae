"""GPU parity at the FULL BASELINE.json sizes, bit-exact against the reference.

tests/golden/golden_full.json holds SHA-256 digests of the reference
QuickMergesort's output (compiled from /root/reference, seed 42) for every
config at its full size: C1 2^20 int32 permutation, C2 2^28 uint32, C3 2^30
uint64, C4a-e 2^27 float64 stress cases, C5 2^26 32-byte records.  Here the
same inputs are produced (device generators, bit-identical to the host
recipe; the Gaussian case on the host and uploaded), sorted on the B200
through the C-ABI, and the digest of the device output must match.  The
size-independent properties (sortedness, multiset fingerprint) are checked on
the device as well.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1804_10062_b200 as q

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_full.json")))
GEN = {"u32": (q.GEN_U32, torch.uint32, ()), "u64": (q.GEN_U64, torch.uint64, ()),
       "rec32": (q.GEN_REC32, torch.uint64, (4,)), "f64_sorted": (q.GEN_F64_SORTED, torch.float64, ()),
       "f64_reverse": (q.GEN_F64_REVERSE, torch.float64, ()),
       "f64_distinct16": (q.GEN_F64_DISTINCT16, torch.float64, ()),
       "f64_organ": (q.GEN_F64_ORGAN, torch.float64, ())}


def sha_tensor(t) -> str:
    h = hashlib.sha256()
    a = t.cpu().numpy()
    mv = memoryview(np.ascontiguousarray(a)).cast("B")
    for i in range(0, len(mv), 1 << 28):
        h.update(mv[i:i + (1 << 28)])
    return h.hexdigest()


@pytest.mark.parametrize("name", sorted(GOLD))
def test_full_size_bit_exact(oracle, name):
    """Every digest of golden_full.json: the nine configs at seed 42, C2 and C5
    at seeds 1 and 2, and C3 digested from the reference's own qms() as well as
    from std::sort."""
    g = GOLD[name]
    n = g["n"]
    cfg = g.get("config", name)
    if cfg in GEN:
        kind, tdt, tail = GEN[cfg]
        x = torch.empty((n,) + tail, dtype=tdt, device="cuda")
        q.generate(kind, x, seed=g["seed"], total=n)
    else:  # C1 permutation (sequential Fisher-Yates) and C4d Gaussian (host libm)
        x = torch.from_numpy(oracle.gen(cfg, n, seed=g["seed"])).cuda()
    torch.cuda.synchronize()
    assert sha_tensor(x) == g["input_sha256"], "input recipe drifted"
    _, s_in, x_in = q.check(x, order=False)
    m = q.sort(x, q.qms())
    viol, s_out, x_out = q.check(x)
    assert viol == 0 and (s_out, x_out) == (s_in, x_in)
    assert sha_tensor(x) == g["sorted_sha256"], "device output differs from the reference"
    assert m.elapsed_ns > 0


def test_c2_descending_full_size():
    """C2 with std::greater: sortedness + multiset at 2^28 (no reference digest)."""
    n = 1 << 28
    x = torch.empty(n, dtype=torch.uint32, device="cuda")
    q.generate(q.GEN_U32, x, seed=1)
    _, s_in, x_in = q.check(x, order=False)
    q.sort(x, q.qms(), "greater")
    viol, s_out, x_out = q.check(x, "greater")
    assert viol == 0 and (s_out, x_out) == (s_in, x_in)


@pytest.mark.parametrize("name,k_frac", [("u32", 0.5), ("u32", 1e-6), ("u64", 0.9), ("rec32", 0.3)])
def test_full_size_select_nth(name, k_frac):
    """select_nth at the full config size: the k-th key equals position k-1 of
    the full sort, whose digest matches the reference's (test above)."""
    g = GOLD[name]
    n = g["n"]
    kind, tdt, tail = GEN[name]
    x = torch.empty((n,) + tail, dtype=tdt, device="cuda")
    q.generate(kind, x, seed=g["seed"], total=n)
    y = x.clone()
    k = max(1, int(n * k_frac))
    _, s_in, x_in = q.check(x, order=False)
    p = q.select_nth(x, k)
    assert p == k - 1
    _, s_out, x_out = q.check(x, order=False)
    assert (s_out, x_out) == (s_in, x_in)  # a permutation of the input
    q.sort(y, q.qms())
    assert sha_tensor(y) == g["sorted_sha256"]
    assert torch.equal(x[p], y[p])
    del y
    # partition around position k-1 (unsigned order for the integer configs)
    if not tail:
        xv = x.view(torch.int64 if x.element_size() == 8 else torch.int32)
        pv = int(xv[p].item()) & ((1 << (8 * x.element_size())) - 1)
        lo = x[:p].cpu().numpy()
        hi = x[p + 1:].cpu().numpy()
        assert (lo <= np.array(pv, dtype=lo.dtype)).all() and (hi >= np.array(pv, dtype=hi.dtype)).all()


def _sha_slices(slices) -> str:
    h = hashlib.sha256()
    for t in slices:
        a = t.cpu().numpy()
        mv = memoryview(np.ascontiguousarray(a)).cast("B")
        for i in range(0, len(mv), 1 << 28):
            h.update(mv[i:i + (1 << 28)])
    return h.hexdigest()


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name,path", [("u64", "c"), ("rec32", "c"), ("rec32", "emulated_fused")])
def test_sharded_full_size_bit_exact(name, path, P):
    """The north-star sharded configs at full size -- C3 (2^30 uint64, 8 GiB)
    and C5 (2^26 32-byte records) -- sorted by P ranks (here all on one
    B200: same kernels, same peer-store exchange).  Shard r generates global
    elements [r n/P, (r+1) n/P); the concatenated slices must hash to the
    reference QuickMergesort's digest of the whole array."""
    from paper_1804_10062_b200 import sharded
    g = GOLD[name]
    n = g["n"]
    kind, tdt, tail = GEN[name]
    shards = []
    for r in range(P):
        a, b = r * n // P, (r + 1) * n // P
        t = torch.empty((b - a,) + tail, dtype=tdt, device="cuda")
        q.generate(kind, t, seed=g["seed"], start=a, total=n)
        shards.append(t)
    torch.cuda.synchronize()
    if path == "c":
        out, m = sharded.sort_sharded_devices(shards, [0] * P, "less")
    else:
        out = sharded.sort_sharded_emulated_fused(shards, "less")
    del shards
    sizes = [o.shape[0] for o in out]
    assert sum(sizes) == n and max(sizes) < 1.2 * n / P, sizes
    for o in out:
        assert q.check(o)[0] == 0
    assert _sha_slices(out) == g["sorted_sha256"], "concatenated slices differ from the reference"
