// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (include path
// /root/reference/proj/core/include, passed by oracle/Makefile) into
// oracle/_ref/libqmsref.so so that tests and bench.py's reference arm can call
// the reference QuickMergesort itself through ctypes.  No reference source is
// copied into this repository; the .so is a build product (git-ignored).
//
// Entry points mirror the reference call the north star names:
//   qmsort::sort(v.begin(), v.end(), preset, less)          sort.hpp:215-226
//   std::sort(v.begin(), v.end(), less)                      trial.hpp:106
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>

#include "qmsort/qmsort.hpp"

namespace {
struct Rec32 {
    std::uint64_t w[4];
};
struct RecLess {
    bool operator()(const Rec32& a, const Rec32& b) const {
        for (int i = 0; i < 4; ++i)
            if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
        return false;
    }
};
struct RecGreater {
    bool operator()(const Rec32& a, const Rec32& b) const { return RecLess{}(b, a); }
};

qmsort::SortConfig preset(int variant, int pivot) {
    qmsort::SortConfig c;
    switch (variant) {
        case 1: c = qmsort::qmqs(); break;
        case 2: c = qmsort::momqms(); break;
        case 3: c = qmsort::hqms(); break;
        default: c = qmsort::qms(); break;
    }
    if (pivot == 1) c.pivot = qmsort::PivotStrategy::median_of_sqrt_n;
    return c;
}

template <class T, class L>
void run(void* data, std::size_t n, int variant, int pivot, int use_std, std::uint64_t* m4) {
    T* p = static_cast<T*>(data);
    if (use_std) {
        std::sort(p, p + n, L{});
        return;
    }
    qmsort::Metrics m = qmsort::sort(p, p + n, preset(variant, pivot), L{});
    if (m4) {
        m4[0] = m.comparisons;
        m4[1] = m.moves;
        m4[2] = m.max_depth;
        m4[3] = m.elapsed_ns;
    }
}

template <class T>
int run_t(void* data, std::size_t n, int greater, int variant, int pivot, int use_std,
          std::uint64_t* m4) {
    if (greater)
        run<T, std::greater<>>(data, n, variant, pivot, use_std, m4);
    else
        run<T, std::less<>>(data, n, variant, pivot, use_std, m4);
    return 0;
}
}  // namespace

extern "C" {

// dtype: 0 i32, 1 u32, 2 u64, 3 f64, 4 rec32, 5 i64.  variant: 0 qms, 1 qmqs,
// 2 momqms, 3 hqms.  pivot: 0 preset, 1 median_of_sqrt_n.  use_std: std::sort.
int qmsref_sort(int dtype, int greater, int variant, int pivot, int use_std, void* data,
                std::size_t n, std::uint64_t* metrics4) {
    switch (dtype) {
        case 0: return run_t<std::int32_t>(data, n, greater, variant, pivot, use_std, metrics4);
        case 1: return run_t<std::uint32_t>(data, n, greater, variant, pivot, use_std, metrics4);
        case 2: return run_t<std::uint64_t>(data, n, greater, variant, pivot, use_std, metrics4);
        case 3: return run_t<double>(data, n, greater, variant, pivot, use_std, metrics4);
        case 5: return run_t<std::int64_t>(data, n, greater, variant, pivot, use_std, metrics4);
        case 4:
            if (greater)
                run<Rec32, RecGreater>(data, n, variant, pivot, use_std, metrics4);
            else
                run<Rec32, RecLess>(data, n, variant, pivot, use_std, metrics4);
            return 0;
    }
    return -1;
}

// generate_input(spec, n, seed) (dataset.hpp:62-99) -> int64 buffer.
// kind: 0 random_perm, 1 sorted, 2 reverse, 3 organ_pipe, 4 few_distinct, 5 random_dup
int qmsref_generate(int kind, std::size_t param, std::size_t n, std::uint64_t seed,
                    std::int64_t* out) {
    qmsort::DataSpec d{static_cast<qmsort::Distribution>(kind), param};
    auto v = qmsort::generate_input(d, n, seed);
    std::memcpy(out, v.data(), n * sizeof(std::int64_t));
    return 0;
}

std::uint64_t qmsref_splitmix(std::uint64_t seed, std::uint64_t j) {
    qmsort::SplitMix64 g(seed);
    std::uint64_t x = 0;
    for (std::uint64_t i = 0; i <= j; ++i) x = g.next();
    return x;
}

// mix_seed (rng.hpp:41-44), the per-trial seed stream of the CLI harness.
std::uint64_t qmsref_mix_seed(std::uint64_t seed, std::uint64_t stream) {
    return qmsort::mix_seed(seed, stream);
}

// kCsvHeader and to_csv (trial.hpp:62-77) of a record with the given fields;
// returns the length written into buf (cap bytes).
int qmsref_csv(char* buf, int cap, const char* algo, std::size_t n, const char* dist,
               std::uint64_t seed, std::uint64_t trial, std::uint64_t comparisons,
               std::uint64_t moves, std::uint64_t time_ns, std::uint64_t depth, double lin,
               double ratio, int header) {
    std::string s;
    if (header) {
        s = qmsort::kCsvHeader;
    } else {
        qmsort::TrialRecord r;
        r.algorithm = algo;
        r.n = n;
        r.distribution = dist;
        r.seed = seed;
        r.trial = trial;
        r.metrics.comparisons = comparisons;
        r.metrics.moves = moves;
        r.metrics.elapsed_ns = time_ns;
        r.metrics.max_depth = depth;
        r.cmp_norm_linear = lin;
        r.cmp_over_nlogn = ratio;
        s = qmsort::to_csv(r);
    }
    std::snprintf(buf, (std::size_t)cap, "%s", s.c_str());
    return (int)s.size();
}

// qmsort::sort over Element<16> (element.hpp:13-20, test_sort.cpp:328-339):
// data is n raw 24-byte elements {int64 key, 16 payload bytes}.
int qmsref_sort_elem16(void* data, std::size_t n, int greater) {
    using E = qmsort::Element<16>;
    static_assert(sizeof(E) == 24, "Element<16> layout");
    E* p = static_cast<E*>(data);
    if (greater)
        qmsort::sort(p, p + n, qmsort::qms(), [](const E& a, const E& b) { return b < a; });
    else
        qmsort::sort(p, p + n, qmsort::qms());
    return 0;
}

// select_nth (selection.hpp:207-212) on an int64 array; returns the position.
std::size_t qmsref_select_nth_i64(std::int64_t* a, std::size_t n, std::size_t k, int greater) {
    qmsort::Metrics m;
    if (greater) {
        qmsort::CountingComparator<std::greater<>> cmp(m);
        return qmsort::select_nth(a, a + n, k, cmp, m);
    }
    qmsort::CountingComparator<std::less<>> cmp(m);
    return qmsort::select_nth(a, a + n, k, cmp, m);
}

// swap_merge (merge.hpp:64-97) on an int64 array, indices as in the tests.
void qmsref_swap_merge_i64(std::int64_t* a, std::size_t b1, std::size_t e1, std::size_t t,
                           std::size_t te) {
    qmsort::Metrics m;
    qmsort::CountingComparator<std::less<>> cmp(m);
    qmsort::swap_merge(a + b1, a + e1, a + t, a + te, cmp, m);
}
}
