// shim_demo.cpp -- TEST: the C++ drop-in include/qmsort_gpu.hpp used exactly
// like the reference call qmsort::sort(v.begin(), v.end(), cfg, less)
// (sort.hpp:215-226).  With WITH_REFERENCE the reference's own SortConfig
// presets (qmsort::qms(), qmsort::hqms()) are passed straight through.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <deque>
#include <functional>
#include <numeric>
#include <vector>

#include "qmsort_gpu.hpp"
#ifdef WITH_REFERENCE
#include "qmsort/qmsort.hpp"
#endif

static int fails = 0;
#define CHECK(c)                                              \
    do {                                                      \
        if (!(c)) {                                           \
            std::printf("CHECK failed: %s (line %d)\n", #c, __LINE__); \
            ++fails;                                          \
        }                                                     \
    } while (0)

struct Rec {
    std::uint64_t w[4];
};
// a record comparator functor, declared as the lexicographic word order
struct RecLess {
    bool operator()(const Rec& a, const Rec& b) const {
        return std::lexicographical_compare(a.w, a.w + 4, b.w, b.w + 4);
    }
};
namespace qmsort::gpu {
template <>
struct is_rec32<Rec> : std::true_type {};
template <>
struct rec32_order<RecLess, Rec> : std::integral_constant<int, QMSORT_LESS> {};
}  // namespace qmsort::gpu

int main() {
    // Fig. 1 worked example (test_sort.cpp:24,37-45) under every preset
    for (auto cfg : {qmsort::gpu::qms(), qmsort::gpu::qmqs(), qmsort::gpu::momqms(), qmsort::gpu::hqms()}) {
        std::vector<std::int32_t> v{7, 11, 4, 5, 6, 10, 9, 2, 3, 1, 0, 8};
        qmsort::gpu::sort(v.begin(), v.end(), cfg);
        std::vector<std::int32_t> e(12);
        std::iota(e.begin(), e.end(), 0);
        CHECK(v == e);
    }
    // seeded uint32 / double / rec32, ascending and descending
    std::vector<std::uint32_t> u(1 << 20);
    std::uint64_t s = 42;
    for (auto& x : u) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        x = (std::uint32_t)(s >> 32);
    }
    auto u2 = u;
    qmsort::gpu::sort(u.begin(), u.end());
    std::sort(u2.begin(), u2.end());
    CHECK(u == u2);
    qmsort::gpu::sort(u.begin(), u.end(), qmsort::gpu::qms(), std::greater<>{});
    CHECK(std::is_sorted(u.begin(), u.end(), std::greater<>{}));
    std::vector<double> d(100000);
    for (std::size_t i = 0; i < d.size(); ++i) d[i] = (double)((i * 7919) % 1000) - 499.5;
    auto d2 = d;
    qmsort::gpu::sort(d.begin(), d.end(), qmsort::gpu::qms(), std::less<double>{});
    std::sort(d2.begin(), d2.end());
    CHECK(d == d2);
    std::vector<Rec> r(50000);
    for (std::size_t i = 0; i < r.size(); ++i) r[i] = Rec{{(i * 37) % 4096, (i * 2654435761u) % 1000003, i, 7}};
    qmsort::gpu::sort(r.begin(), r.end());
    CHECK(std::is_sorted(r.begin(), r.end(), [](const Rec& a, const Rec& b) {
        return std::lexicographical_compare(a.w, a.w + 4, b.w, b.w + 4);
    }));
    {
        auto r2 = r;
        std::reverse(r2.begin(), r2.end());
        qmsort::gpu::sort(r2.begin(), r2.end(), qmsort::gpu::qms(), RecLess{});
        CHECK(std::equal(r.begin(), r.end(), r2.begin(), [](const Rec& a, const Rec& b) {
            return std::equal(a.w, a.w + 4, b.w);
        }));
    }
    // a non-contiguous random-access range (std::deque) is gathered, sorted, written back
    {
        std::deque<std::int64_t> dq;
        for (int i = 0; i < 100000; ++i) dq.push_back((std::int64_t)((i * 7919LL) % 100003) - 50000);
        qmsort::gpu::sort(dq.begin(), dq.end());
        CHECK(std::is_sorted(dq.begin(), dq.end()) && dq.size() == 100000);
    }
    // sort_range_counted (sort.hpp:207-211): counters accumulate into a caller Metrics
    {
        qmsort::gpu::Metrics acc;
        std::less<> cmp;
        std::vector<std::uint32_t> a(u.begin(), u.begin() + 300000);
        qmsort::gpu::sort_range_counted(a.begin(), a.end(), qmsort::gpu::qms(), cmp, acc);
        CHECK(std::is_sorted(a.begin(), a.end()));
        const auto t1 = acc.elapsed_ns;
        std::reverse(a.begin(), a.end());
        qmsort::gpu::sort_range_counted(a.begin(), a.end(), qmsort::gpu::qms(), cmp, acc);
        CHECK(std::is_sorted(a.begin(), a.end()) && t1 > 0 && acc.elapsed_ns > t1 && acc.comparisons == 0);
    }
    // PartitionResult (partition_result.hpp:12-17): three-way partition around a pivot value
    {
        std::vector<std::int32_t> v{7, 11, 4, 5, 6, 10, 9, 2, 3, 1, 0, 8, 7, 7};
        const auto pr = qmsort::gpu::partition(v.begin(), v.end(), 7);
        CHECK(pr.lt_end == 7 && pr.gt_begin == 10 && pr.left_size == 7 && pr.right_size == 4);
        CHECK(std::all_of(v.begin(), v.begin() + 7, [](int x) { return x < 7; }));
        CHECK(std::all_of(v.begin() + 7, v.begin() + 10, [](int x) { return x == 7; }));
        CHECK(std::all_of(v.begin() + 10, v.end(), [](int x) { return x > 7; }));
        std::vector<double> dv(200000);
        for (std::size_t i = 0; i < dv.size(); ++i) dv[i] = (double)((i * 7919) % 1001) - 500.0;
        const auto pd = qmsort::gpu::partition(dv.begin(), dv.end(), 0.0, std::greater<>{});
        CHECK(std::all_of(dv.begin(), dv.begin() + pd.lt_end, [](double x) { return x > 0.0; }));
        CHECK(std::all_of(dv.begin() + pd.lt_end, dv.begin() + pd.gt_begin, [](double x) { return x == 0.0; }));
        CHECK(std::all_of(dv.begin() + pd.gt_begin, dv.end(), [](double x) { return x < 0.0; }));
        CHECK(pd.gt_begin - pd.lt_end == (std::size_t)std::count(dv.begin(), dv.end(), 0.0));
    }
    // int64 keys (the reference profile's Vec, test_sort.cpp:22)
    std::vector<std::int64_t> q64(200000);
    for (auto& x : q64) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        x = (std::int64_t)s;
    }
    auto q64b = q64;
    qmsort::gpu::sort(q64.begin(), q64.end());
    std::sort(q64b.begin(), q64b.end());
    CHECK(q64 == q64b);
    // key + payload elements: ordered on the key alone, equal keys stay in input order
    struct Elem {
        std::int64_t key;
        unsigned char payload[16];
    };
    std::vector<Elem> ev(30000);
    for (std::size_t i = 0; i < ev.size(); ++i) {
        ev[i].key = (std::int64_t)((i * 7919) % 97) - 48;
        for (int b = 0; b < 16; ++b) ev[i].payload[b] = (unsigned char)(i >> (b % 3 * 8));
    }
    auto ev2 = ev;
    qmsort::gpu::sort(ev.begin(), ev.end());
    std::stable_sort(ev2.begin(), ev2.end(), [](const Elem& a, const Elem& b) { return a.key < b.key; });
    CHECK(std::equal(ev.begin(), ev.end(), ev2.begin(), [](const Elem& a, const Elem& b) {
        return a.key == b.key && std::equal(a.payload, a.payload + 16, b.payload);
    }));
    // select_nth (selection.hpp:207-212), 1-based k
    {
        auto a = q64b;
        std::reverse(a.begin(), a.end());
        const std::size_t p = qmsort::gpu::select_nth(a.begin(), a.end(), 777);
        CHECK(p == 776 && a[p] == q64b[776]);
        CHECK(std::all_of(a.begin(), a.begin() + p, [&](std::int64_t x) { return x <= a[p]; }));
        CHECK(std::all_of(a.begin() + p + 1, a.end(), [&](std::int64_t x) { return x >= a[p]; }));
    }
#ifdef WITH_REFERENCE
    {
        // the reference's own Element<16> (test_sort.cpp:328-339)
        std::vector<qmsort::Element<16>> re(5000);
        for (std::size_t i = 0; i < re.size(); ++i) {
            re[i].key = (std::int64_t)((i * 31) % 50);
            re[i].payload[0] = std::byte{(unsigned char)i};
        }
        qmsort::gpu::sort(re.begin(), re.end(), qmsort::qms());
        CHECK(std::is_sorted(re.begin(), re.end()));
    }
    // the reference's own config objects and comparator types drop straight in
    std::vector<std::int32_t> v{7, 11, 4, 5, 6, 10, 9, 2, 3, 1, 0, 8};
    qmsort::gpu::sort(v.begin(), v.end(), qmsort::hqms(), std::greater<>{});
    CHECK(std::is_sorted(v.begin(), v.end(), std::greater<>{}));
    std::vector<std::int32_t> w{7, 11, 4, 5, 6, 10, 9, 2, 3, 1, 0, 8};
    qmsort::SortConfig rc = qmsort::qms();
    rc.pivot = qmsort::PivotStrategy::median_of_sqrt_n;
    qmsort::gpu::sort(w.begin(), w.end(), rc);
    CHECK(std::is_sorted(w.begin(), w.end()));
#endif
    std::printf(fails ? "shim FAILED (%d)\n" : "shim ok\n", fails);
    return fails ? 1 : 0;
}
