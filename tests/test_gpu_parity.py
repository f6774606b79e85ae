"""GPU parity: the B200 sort through the C-ABI vs the CPU QuickMergesort oracle.

Mirrors the reference's own suites (test_sort.cpp:37-77, 356-362;
acceptance.cpp:86-114): every variant x distribution x size must give output
byte-identical to the oracle on the same seeded input.  Bit-exact (integer /
record / IEEE bit patterns): there is no tolerance.
"""
import numpy as np
import pytest

import paper_1804_10062_b200 as q
from oracle_lib import DT_F64, DT_I32, DT_I64, DT_REC32, DT_U32, DT_U64

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DTYPES = [DT_I32, DT_U32, DT_U64, DT_F64, DT_REC32, DT_I64]


def rand_input(dt, n, seed, dist="uniform"):
    rng = np.random.default_rng(seed)
    shape = (n, 4) if dt == DT_REC32 else (n,)
    if dist == "uniform":
        raw = rng.integers(0, 2**63, size=shape, dtype=np.uint64) * 2 + rng.integers(0, 2, size=shape, dtype=np.uint64)
    elif dist == "fewdistinct":
        raw = (rng.integers(0, 7, size=shape, dtype=np.uint64) + 1) * np.uint64(0x0101010101)
    elif dist == "allequal":
        raw = np.full(shape, 0x123456789, dtype=np.uint64)
    elif dist == "sorted":
        raw = np.arange(n, dtype=np.uint64) * np.uint64(3)
        if dt == DT_REC32:
            raw = np.repeat(raw[:, None], 4, axis=1)
    elif dist == "reverse":
        raw = (np.arange(n, dtype=np.uint64)[::-1] * np.uint64(3)).copy()
        if dt == DT_REC32:
            raw = np.repeat(raw[:, None], 4, axis=1)
    elif dist == "organpipe":
        i = np.arange(n, dtype=np.uint64)
        raw = np.minimum(i + 1, np.uint64(n) - i)
        if dt == DT_REC32:
            raw = np.repeat(raw[:, None], 4, axis=1)
    else:
        raise ValueError(dist)
    if dt == DT_I32:
        return (raw & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    if dt == DT_U32:
        return (raw >> np.uint64(7) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    if dt == DT_U64:
        return raw.astype(np.uint64)
    if dt == DT_I64:  # the reference profile's key type (test_sort.cpp:22)
        return (raw - np.uint64(1 << 62) if dist != "uniform" else raw).astype(np.uint64).view(np.int64)
    if dt == DT_F64:
        # finite doubles, no NaN / -0.0: scale signed integers
        s = (raw >> np.uint64(11)).astype(np.int64) - (1 << 51)
        x = s.astype(np.float64) * 1.25e-3
        x[x == 0] = 0.0
        return x
    if dt == DT_REC32:
        r = raw.astype(np.uint64).copy()
        if dist == "uniform":
            r[:, 0] >>= np.uint64(52)  # word 0 from 2^12 values, as config 5
        return r
    raise ValueError(dt)


def gpu_sort(a, cfg=None, less="less"):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    m = q.sort(t, cfg or q.qms(), less)
    torch.cuda.synchronize()
    return t.cpu().numpy(), m


SIZES = [0, 1, 2, 3, 9, 10, 100, 511, 512, 513, 1000, 1024, 2047, 4096, 4097, 8191, 8192,
         8193, 16383, 16384, 16385, 20000, 65536, 100003, 1 << 20]


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n", SIZES)
def test_uniform_sizes_samplesort(oracle, dt, n):
    a = rand_input(dt, n, seed=n + 17 * dt)
    got, _ = gpu_sort(a)
    np.testing.assert_array_equal(got, oracle.sort(dt, a))


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n", [40001, 100003, 1 << 19])  # above every block-sort cap
def test_uniform_sizes_mergesort(oracle, dt, n):
    a = rand_input(dt, n, seed=n + 3 * dt)
    cfg = q.qms()
    cfg.algorithm = q.Algorithm.mergesort
    got, m = gpu_sort(a, cfg)
    np.testing.assert_array_equal(got, oracle.sort(dt, a))
    assert m.merge_passes >= 1


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("dist", ["fewdistinct", "allequal", "sorted", "reverse", "organpipe"])
@pytest.mark.parametrize("n", [5000, 300001])
def test_distributions(oracle, dt, dist, n):
    a = rand_input(dt, n, seed=5, dist=dist)
    got, _ = gpu_sort(a)
    np.testing.assert_array_equal(got, oracle.sort(dt, a))


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("n", [7, 5000, 200000])
def test_descending_greater(oracle, dt, n):
    """std::greater comparator (test_sort.cpp:356-362)."""
    a = rand_input(dt, n, seed=99)
    got, _ = gpu_sort(a, less="greater")
    np.testing.assert_array_equal(got, oracle.sort(dt, a, greater=True))


@pytest.mark.parametrize("preset", [q.qms, q.qmqs, q.momqms, q.hqms])
def test_fig1_all_presets(preset):
    """Worked 12-element example (test_sort.cpp:24,37-45) under every variant."""
    a = np.array([7, 11, 4, 5, 6, 10, 9, 2, 3, 1, 0, 8], dtype=np.int32)
    got, _ = gpu_sort(a, preset())
    np.testing.assert_array_equal(got, np.arange(12, dtype=np.int32))


def test_host_dropin_matches(oracle):
    """qmsort_gpu_sort_host: the host-array drop-in (sort.hpp:215-226)."""
    a = rand_input(DT_U32, 300000, seed=3)
    b = a.copy()
    m = q.sort(b)  # numpy -> host path
    np.testing.assert_array_equal(b, oracle.sort(DT_U32, a))
    assert m.elapsed_ns > 0


def test_fuzz_all_variants(oracle):
    """Fuzz over random n < 3000 and the six reference distributions
    (test_sort.cpp:59-77)."""
    rng = np.random.default_rng(1001)
    for trial in range(60):
        n = int(rng.integers(0, 3000))
        dt = DTYPES[trial % len(DTYPES)]
        dist = ["uniform", "sorted", "reverse", "organpipe", "fewdistinct", "allequal"][trial % 6]
        a = rand_input(dt, n, seed=trial, dist=dist)
        for preset in (q.qms, q.qmqs, q.momqms, q.hqms):
            got, _ = gpu_sort(a, preset())
            np.testing.assert_array_equal(got, oracle.sort(dt, a))


@pytest.mark.parametrize("cfgname", ["i32_perm", "u32", "u64", "f64_sorted", "f64_reverse",
                                     "f64_distinct16", "f64_gauss", "f64_organ", "rec32", "i64"])
def test_config_shapes_reduced(oracle, cfgname):
    """The five BASELINE configs at 2^20 elements, seeded recipes of SURVEY.md 8(d)."""
    n = 1 << 20
    a = oracle.gen(cfgname, n, seed=42)
    dt = {"i32_perm": DT_I32, "u32": DT_U32, "u64": DT_U64, "rec32": DT_REC32,
          "i64": DT_I64}.get(cfgname, DT_F64)
    got, _ = gpu_sort(a)
    if cfgname == "i32_perm":
        np.testing.assert_array_equal(got, np.arange(n, dtype=np.int32))  # closed form
    np.testing.assert_array_equal(got, oracle.sort(dt, a))


@pytest.mark.parametrize("kind,dt,cfgname", [(q.GEN_U32, DT_U32, "u32"), (q.GEN_U64, DT_U64, "u64"),
                                             (q.GEN_REC32, DT_REC32, "rec32"),
                                             (q.GEN_F64_DISTINCT16, DT_F64, "f64_distinct16"),
                                             (q.GEN_F64_ORGAN, DT_F64, "f64_organ")])
def test_device_generators_match_host(oracle, kind, dt, cfgname):
    n = 100000
    shape = (n, 4) if dt == DT_REC32 else (n,)
    tdt = {DT_U32: torch.uint32, DT_U64: torch.uint64, DT_REC32: torch.uint64, DT_F64: torch.float64}[dt]
    t = torch.empty(shape, dtype=tdt, device="cuda")
    q.generate(kind, t, seed=7, start=0, total=n)
    np.testing.assert_array_equal(t.cpu().numpy(), oracle.gen(cfgname, n, seed=7))


@pytest.mark.parametrize("dt", [DT_U32, DT_I64, DT_F64, DT_REC32])
def test_host_batch_pipeline(oracle, dt):
    """qmsort_gpu_sort_host_batch: a stream of independent host arrays (sizes
    0 .. 2^21, pinned and pageable) -- each equals the oracle's sort."""
    sizes = [0, 1, 5000, 1 << 21, 777, 1 << 20, 3]
    arrays = [rand_input(dt, n, seed=n + 7) for n in sizes]
    want = [oracle.sort(dt, a) for a in arrays]
    work = [a.copy() for a in arrays]
    m = q.sort_batch(work)
    for g, w in zip(work, want):
        np.testing.assert_array_equal(g, w)
    assert m.kernel_launches > 0 and m.elapsed_ns > 0
    # pinned torch buffers, descending
    pins = [torch.from_numpy(a.copy()).pin_memory() for a in arrays[2:5]]
    q.sort_batch(pins, less="greater")
    for p, a in zip(pins, arrays[2:5]):
        np.testing.assert_array_equal(p.numpy(), oracle.sort(dt, a, greater=True))


@pytest.mark.parametrize("case", ["w1_const", "w1_low_bits", "w0_wide", "w0_span2", "mixed"])
@pytest.mark.parametrize("n", [3000, 200000])
def test_rec32_prefix_ties(oracle, case, n):
    """Record block sort: the (prefix | index) fast path must hand every tile
    whose 52-bit prefixes tie to the full-record sorter -- records equal in
    w0/w1 (or in w1's top bits) that differ only in later words, a w0 range
    wider than 64 bits of prefix, two w0 values per tile, and a mix."""
    rng = np.random.default_rng(n + len(case))
    r = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64)
    if case == "w1_const":
        r[:, 0] = rng.integers(0, 3, size=n, dtype=np.uint64)
        r[:, 1] = np.uint64(0xDEADBEEF)
    elif case == "w1_low_bits":
        r[:, 0] >>= np.uint64(60)
        r[:, 1] = (r[:, 1] >> np.uint64(52) << np.uint64(52)) | rng.integers(0, 4096, size=n, dtype=np.uint64)
        r[:, 1] &= np.uint64(0xFFF00000000FFFFF)
    elif case == "w0_wide":
        r[:, 0] = r[:, 0] * np.uint64(2) + np.uint64(1)
    elif case == "w0_span2":
        r[:, 0] = rng.integers(7, 9, size=n, dtype=np.uint64)
    else:
        r[:, 0] >>= np.uint64(58)
        r[: n // 2, 1] = np.uint64(5)
    got, _ = gpu_sort(r)
    np.testing.assert_array_equal(got, oracle.sort(DT_REC32, r))
    got, _ = gpu_sort(r, less="greater")
    np.testing.assert_array_equal(got, oracle.sort(DT_REC32, r, greater=True))


@pytest.mark.parametrize("base", [0, 12345, (1 << 32) - 65535, (1 << 32) - 70000, (1 << 32) - 1 - 65534])
@pytest.mark.parametrize("span", [1, 2, 1000, 65533, 65534, 65535, 65536])
@pytest.mark.parametrize("n", [2, 1000, 1024, 1025, 2048, 3000, 4096, 9000, 16384, 300000])
def test_u32_packed_spans(oracle, base, span, n):
    """uint32 block sort: tiles whose keys span < 2^16 - 1 values are sorted
    two keys per register -- spans at and around the limit, keys touching 0
    and 2^32 - 1 (the padding must stay above every real key), both orders."""
    rng = np.random.default_rng(n * 7 + span)
    hi = min((1 << 32) - 1, base + span - 1)
    a = rng.integers(base, hi + 1, size=n, dtype=np.uint64).astype(np.uint32)
    if n > 2:
        a[0], a[1] = base, hi  # the full span is present
    got, _ = gpu_sort(a)
    np.testing.assert_array_equal(got, np.sort(a))
    got, _ = gpu_sort(a, less="greater")
    np.testing.assert_array_equal(got, np.sort(a)[::-1])


@pytest.mark.parametrize("dt", [DT_U64, DT_I64, DT_U32])
@pytest.mark.parametrize("n", [5482783, 3000001])
def test_skewed_window(oracle, dt, n):
    """90 % of the keys in a window of 100 values, the rest spread wide: the
    lower levels get segments whose key range is a single value or two, and
    the padding keys of a partial tile fall into LUT cells past the range
    (once read as a negative splitter count -- an out-of-bounds search)."""
    rng = np.random.default_rng(n)
    raw = rng.integers(0, 2**62, size=n, dtype=np.uint64)
    m = rng.random(n) < 0.9
    raw[m] = rng.integers(1000, 1100, size=int(m.sum()), dtype=np.uint64)
    a = raw.astype(np.uint32) if dt == DT_U32 else (raw.view(np.int64) if dt == DT_I64 else raw)
    got, _ = gpu_sort(a)
    np.testing.assert_array_equal(got, oracle.sort(dt, a))


def dense_u32(rng, n, density_inv, base=0):
    """n uint32 keys uniform over n * density_inv values starting at base."""
    return (rng.integers(0, n * density_inv, size=n, dtype=np.uint64) + np.uint64(base)).astype(np.uint32)


@pytest.mark.parametrize("density_inv", [3, 4, 5, 16, 33, 64, 65, 200])
@pytest.mark.parametrize("n", [1 << 20, 3000001])
@pytest.mark.parametrize("dt", [DT_U32, DT_I32])
def test_table_sort_dense_keys(oracle, dt, density_inv, n):
    """Dense uint32 / int32 key sets: the last level's buckets span a few 10^4
    values and go through the comparison-free table sort (K5t) when the span
    is between 4 and 64 values per key; sparser buckets go through the
    wide-span table sort (K5c), denser ones keep the network.  Both orders, keys touching both ends of the key space."""
    rng = np.random.default_rng(n + density_inv)
    for base in (0, (1 << 32) - n * density_inv, 0x7FFFFFFF - n * density_inv // 2):
        a = dense_u32(rng, n, density_inv, base)
        if dt == DT_I32:
            a = a.view(np.int32)
        got, m = gpu_sort(a)
        np.testing.assert_array_equal(got, np.sort(a))
        if 5 <= density_inv <= 16:
            assert m.table_buckets > 0
        if density_inv <= 3:  # too dense for either table sort (a segment's end buckets aside)
            assert m.table_buckets <= 4
        got, _ = gpu_sort(a, less="greater")
        np.testing.assert_array_equal(got, np.sort(a)[::-1])


@pytest.mark.parametrize("copies", [2, 3, 4, 5, 9])
@pytest.mark.parametrize("hot", [1, 40, 2000, 40000])
def test_table_sort_repeated_values(oracle, copies, hot):
    """Table sort with second, third, fourth and later copies of a value:
    `hot` values of a dense key set appear `copies` times (planes 1 and 2, the
    overflow list, and -- 40000 x 5 and up -- more fourth copies per bucket
    than the list holds, which sends the bucket back to the network)."""
    n = 1 << 20
    rng = np.random.default_rng(copies * 1000 + hot)
    a = dense_u32(rng, n, 16, 123456)
    idx = rng.choice(n, size=hot, replace=False)
    for c in range(1, copies):
        a[(idx + c * 7919) % n] = a[idx]
    got, m = gpu_sort(a)
    np.testing.assert_array_equal(got, np.sort(a))
    assert m.table_buckets > 0
    got, _ = gpu_sort(a, less="greater")
    np.testing.assert_array_equal(got, np.sort(a)[::-1])


def test_table_sort_clustered_buckets(oracle):
    """Buckets whose keys crowd one end of their splitter range (a staircase of
    dense clusters separated by gaps) and buckets made of a few long runs."""
    n = 1 << 21
    rng = np.random.default_rng(5)
    steps = rng.integers(0, 1 << 12, size=n // 4096, dtype=np.uint64).cumsum() * np.uint64(4096)
    a = (np.repeat(steps, 4096)[:n] + rng.integers(0, 9000, size=n, dtype=np.uint64)).astype(np.uint32)
    got, m = gpu_sort(a)
    np.testing.assert_array_equal(got, np.sort(a))
    b = np.repeat(rng.integers(0, 1 << 24, size=n // 3, dtype=np.uint64), 3)[:n].astype(np.uint32)
    rng.shuffle(b)
    got, m = gpu_sort(b)
    np.testing.assert_array_equal(got, np.sort(b))


def _as_dtype(raw, dt):
    """uint64 bit patterns -> an array of dt (float64: finite, no NaN / -0.0)."""
    if dt == DT_U64:
        return raw.astype(np.uint64)
    if dt == DT_I64:
        return raw.astype(np.uint64).view(np.int64)
    if dt == DT_U32:
        return (raw & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    if dt == DT_I32:
        return (raw & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    raise ValueError(dt)


@pytest.mark.parametrize("n", [1 << 18, 1 << 20, (1 << 21) + 12345, 1 << 22])
@pytest.mark.parametrize("dt", [DT_U64, DT_I64, DT_F64, DT_U32])
def test_cell_sort_wide_span_keys(oracle, dt, n):
    """Sparse keys (64-bit keys, uint32 keys over the full range at small n):
    the last level's buckets span far more than 2^16 values and go through
    the wide-span table sort (K5c: cells of 2^sh values, in-cell ordering).
    2^20 8-byte keys leave buckets of about 2048 keys (small shape), 2^21 of
    about 4096 (big shape).  Both orders."""
    a = rand_input(dt, n, seed=n + dt)
    got, m = gpu_sort(a)
    np.testing.assert_array_equal(got, np.sort(a))
    if not (dt == DT_U32 and n == 1 << 22):  # (512 even buckets of 8192 uint32 keys: over the cell sort's 4096)
        assert m.table_buckets > 0
    got, _ = gpu_sort(a, less="greater")
    np.testing.assert_array_equal(got, np.sort(a)[::-1])


@pytest.mark.parametrize("dist", ["gaussian", "exponential", "near_zero", "binades", "lattice"])
def test_cell_sort_float_shapes(oracle, dist):
    """float64 shapes whose bit patterns are far from uniform inside a bucket:
    a bucket that straddles zero or many binades crowds its keys into a few
    cells (overflow list / fix list full -> the network sorts it)."""
    n = 1 << 21
    rng = np.random.default_rng(11)
    if dist == "gaussian":
        x = rng.standard_normal(n)
    elif dist == "exponential":
        x = rng.exponential(1.0, n) * rng.choice([-1.0, 1.0], n)
    elif dist == "near_zero":
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, -280, n)
    elif dist == "binades":
        x = np.ldexp(rng.random(n) + 0.5, rng.integers(-40, 40, n)) * rng.choice([-1.0, 1.0], n)
    else:  # values on a coarse lattice: a few thousand distinct doubles, each many times
        x = rng.integers(-3000, 3000, n).astype(np.float64) * 0.37
    x[x == 0] = 0.0
    got, _ = gpu_sort(x)
    np.testing.assert_array_equal(got, np.sort(x))
    got, _ = gpu_sort(x, less="greater")
    np.testing.assert_array_equal(got, np.sort(x)[::-1])


@pytest.mark.parametrize("dt", [DT_U64, DT_I64, DT_U32])
@pytest.mark.parametrize("shape", ["pairs", "triples", "quads", "runs9", "clusters", "two_scales", "hot_cell"])
def test_cell_sort_crowded_cells(oracle, dt, shape):
    """Cells holding several keys: exact duplicates (2, 3, 4, 9 copies of every
    value: planes, overflow list), tight clusters (distinct keys that share a
    cell and must be ordered inside it), two scales in one bucket, and one
    cell that takes a large share of its bucket (fallback to the network)."""
    n = 1 << 20
    rng = np.random.default_rng(dt * 100 + len(shape))
    wide = rng.integers(0, 2**63, size=n, dtype=np.uint64) * np.uint64(2)
    if shape in ("pairs", "triples", "quads", "runs9"):
        c = {"pairs": 2, "triples": 3, "quads": 4, "runs9": 9}[shape]
        raw = np.repeat(wide[: n // c + 1], c)[:n].copy()
        rng.shuffle(raw)
    elif shape == "clusters":  # 2..6 distinct keys a few values apart around every centre
        raw = wide.copy()
        k = n // 4
        for j in range(1, 4):
            raw[j * k:(j + 1) * k] = raw[:k] + rng.integers(1, 50, size=k, dtype=np.uint64)
    elif shape == "two_scales":  # half the keys spread out, half within 2^20 values of 64 centres
        raw = wide.copy()
        centres = rng.integers(0, 2**63, size=64, dtype=np.uint64)
        raw[: n // 2] = centres[rng.integers(0, 64, n // 2)] + rng.integers(0, 1 << 20, size=n // 2, dtype=np.uint64)
    else:  # hot_cell: 30 % of the keys within 1000 consecutive values
        raw = wide.copy()
        raw[: n * 3 // 10] = np.uint64(1 << 61) + rng.integers(0, 1000, size=n * 3 // 10, dtype=np.uint64)
    if dt in (DT_U32, DT_I32):
        raw = raw >> np.uint64(32)
    a = _as_dtype(raw, dt)
    got, m = gpu_sort(a)
    np.testing.assert_array_equal(got, np.sort(a))
    got, _ = gpu_sort(a, less="greater")
    np.testing.assert_array_equal(got, np.sort(a)[::-1])


@pytest.mark.parametrize("shape", ["c5", "const_w0", "wide_w0", "outliers", "narrow_outliers", "two_w0", "dup_prefix"])
@pytest.mark.parametrize("n", [1 << 18, (1 << 20) + 777])
def test_record_even_splitters(oracle, shape, n):
    """Records under even splitters (K1 cuts the sampled prefix range into
    equal parts): the C5 shape (12-bit w0), one w0 for all records (the prefix
    is w1), w0 over all 64 bits, a few records far outside the sampled prefix
    range on both sides (they clamp into the end buckets; narrow_outliers: so
    far outside that the 32-bit range index saturates), two distant w0
    values (an uneven sample: quantile splitters), and records that agree on
    the whole prefix and differ only in w2 / w3."""
    rng = np.random.default_rng(n + len(shape))
    r = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64) * np.uint64(2)
    if shape == "c5":
        r[:, 0] >>= np.uint64(52)
    elif shape == "const_w0":
        r[:, 0] = np.uint64(0xABCDEF)
    elif shape == "outliers":
        r[:, 0] = np.uint64(1 << 40) + (r[:, 0] >> np.uint64(44))
        r[:3, 0] = np.uint64(5)
        r[3:6, 0] = np.uint64(0xFFFFFFFFFFFFFF00)
    elif shape == "narrow_outliers":
        # one w0 and a narrow w1 range (a small prefix span), plus records the
        # sample misses whose prefix lies 2^34 spans above / below the range
        r[:, 0] = np.uint64(7)
        r[:, 1] >>= np.uint64(34)
        r[:5, 0] = np.uint64(8)
        r[5:8, 0] = np.uint64(6)
        r[8:11, 1] = np.array([(1 << 40) + (1 << 29), (1 << 50) + (1 << 28), (1 << 63) + 12345], dtype=np.uint64)
    elif shape == "two_w0":
        r[:, 0] = np.where(rng.integers(0, 2, n) == 1, np.uint64(7), np.uint64(1 << 62))
    elif shape == "dup_prefix":
        r[:, 0] >>= np.uint64(56)
        r[:, 1] = r[:, 0] * np.uint64(0x0101010101010101)
    want = oracle.sort(DT_REC32, r)
    got, _ = gpu_sort(r)
    np.testing.assert_array_equal(got, want)
    got, _ = gpu_sort(r, less="greater")
    np.testing.assert_array_equal(got, want[::-1])


@pytest.mark.parametrize("dt", [DT_U32, DT_U64, DT_I64])
@pytest.mark.parametrize("share", [0.08, 0.12, 0.15, 0.25, 0.6])
def test_even_splitters_near_the_acceptance_threshold(oracle, dt, share):
    """Mixtures around K1's even-splitter test: most keys uniform over the full
    range plus `share` of them uniform over one eighth of it, so the ranges
    inside that eighth hold 1.6 ... 5 times their share -- samples just under
    the threshold are accepted (uneven buckets, deeper levels for the big
    ones), samples over it keep the quantile splitters; and a last level whose
    segments are dense in one half and empty in the other."""
    n = 1 << 22
    rng = np.random.default_rng(int(share * 100) + dt)
    full = np.uint64(0xFFFFFFFF if dt == DT_U32 else 0xFFFFFFFFFFFFFFFF)
    raw = rng.integers(0, 2**63, size=n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n, dtype=np.uint64)
    raw &= full
    k = int(n * share)
    raw[:k] = (raw[:k] >> np.uint64(3)) + (full >> np.uint64(2))
    rng.shuffle(raw)
    a = _as_dtype(raw, dt)
    got, _ = gpu_sort(a)
    np.testing.assert_array_equal(got, np.sort(a))
    # every other 2^16-value stripe empty (uint32) / every other 2^40-value stripe (64-bit)
    stripe = np.uint64(16 if dt == DT_U32 else 40)
    b = _as_dtype(raw & ~(np.uint64(1) << stripe) & full, dt)
    got, _ = gpu_sort(b)
    np.testing.assert_array_equal(got, np.sort(b))
    got, _ = gpu_sort(b, less="greater")
    np.testing.assert_array_equal(got, np.sort(b)[::-1])
