// qmsort_gpu.hpp -- C++ drop-in over the C-ABI (qmsort_gpu.h).
//
// Mirrors the reference entry point
//     template <class It, class Less = std::less<>>
//     Metrics qmsort::sort(It first, It last, const SortConfig& cfg = {}, Less less = {},
//                          SortObserver* obs = nullptr);          // sort.hpp:215-226
// as qmsort::gpu::sort with the same argument meaning: a contiguous range of
// int32 / uint32 / uint64 / double / 32-byte records, a SortConfig (ours, or the
// reference's own qmsort::SortConfig -- any type with the same member names),
// and std::less / std::greater.  The range is copied to the B200, sorted there
// and copied back; failures throw std::runtime_error (as trial.hpp:116 does),
// never fall back to the CPU.  SortObserver hooks are accepted and ignored
// (the GPU pipeline has no QuickXsort steps to observe).
#pragma once

#include <cstdint>
#include <functional>
#include <iterator>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "qmsort_gpu.h"

namespace qmsort {
namespace gpu {

enum class Variant { qms, qmqs, momqms, hqms };                           // sort.hpp:17
enum class PivotStrategy { median_of_3, median_of_sqrt_n, mom_of_thirds, hybrid };  // :19
enum class MergesortSide { smaller_always, larger_when_feasible };        // :21
enum class BaseCase { insertion, hardcoded_small, clever_quicksort };     // merge.hpp:14

struct BaseCasePolicy {  // merge.hpp:26-31
    BaseCase kind = BaseCase::hardcoded_small;
    std::size_t size_threshold = 10;
    bool use_levels = false;
};

struct SortConfig {  // sort.hpp:25-34
    Variant variant = Variant::qms;
    PivotStrategy pivot = PivotStrategy::median_of_3;
    BaseCasePolicy base_case{};
    double beta = 0.5;
    double delta = 1.0 / 16.0;
    MergesortSide side = MergesortSide::larger_when_feasible;
    bool three_way = false;
    std::size_t block = 128;
};

inline SortConfig qms() { return SortConfig{}; }  // sort.hpp:37
inline SortConfig qmqs() {                         // sort.hpp:41-48
    SortConfig c;
    c.variant = Variant::qmqs;
    c.base_case.kind = BaseCase::clever_quicksort;
    c.base_case.size_threshold = 16;
    c.base_case.use_levels = true;
    return c;
}
inline SortConfig momqms() {  // sort.hpp:52-57
    SortConfig c;
    c.variant = Variant::momqms;
    c.pivot = PivotStrategy::mom_of_thirds;
    return c;
}
inline SortConfig hqms() {  // sort.hpp:61-66
    SortConfig c;
    c.variant = Variant::hqms;
    c.pivot = PivotStrategy::hybrid;
    return c;
}

struct Metrics {  // metrics.hpp:14-24 (comparisons/moves are not counted on the GPU)
    std::uint64_t comparisons = 0;
    std::uint64_t moves = 0;
    std::uint64_t max_depth = 0;
    std::uint64_t elapsed_ns = 0;
};

// Element type -> qmsort_dtype.  A user-defined 32-byte record is enabled by
// specialising qmsort::gpu::is_rec32<T> (lexicographic over four uint64 words).
template <class T>
struct is_rec32 : std::false_type {};
template <class T>
constexpr int dtype_code() {
    if constexpr (std::is_same_v<T, std::int32_t>) return QMSORT_DT_I32;
    else if constexpr (std::is_same_v<T, std::uint32_t>) return QMSORT_DT_U32;
    else if constexpr (std::is_same_v<T, std::uint64_t>) return QMSORT_DT_U64;
    else if constexpr (std::is_same_v<T, double>) return QMSORT_DT_F64;
    else if constexpr (is_rec32<T>::value) {
        static_assert(sizeof(T) == 32 && std::is_trivially_copyable_v<T>, "rec32 must be 32 trivially copyable bytes");
        return QMSORT_DT_REC32;
    } else {
        static_assert(sizeof(T) == 0, "qmsort::gpu::sort supports int32, uint32, uint64, double and rec32");
        return -1;
    }
}

template <class Less, class T>
constexpr int cmp_code() {
    if constexpr (std::is_same_v<Less, std::less<>> || std::is_same_v<Less, std::less<T>>) return QMSORT_LESS;
    else if constexpr (std::is_same_v<Less, std::greater<>> || std::is_same_v<Less, std::greater<T>>)
        return QMSORT_GREATER;
    else if constexpr (is_rec32<T>::value) return QMSORT_LESS;  // the record's lexicographic order
    else {
        static_assert(sizeof(Less) == 0, "comparator must be std::less or std::greater");
        return -1;
    }
}

// Any config type with SortConfig's member names (ours or the reference's).
template <class Cfg>
inline qmsort_gpu_config to_c(const Cfg& c) {
    qmsort_gpu_config g;
    qmsort_gpu_config_init(&g, static_cast<int>(c.variant));
    g.variant = static_cast<int>(c.variant);
    g.pivot = static_cast<int>(c.pivot);
    g.base_case_kind = static_cast<int>(c.base_case.kind);
    g.base_case_size_threshold = c.base_case.size_threshold;
    g.base_case_use_levels = c.base_case.use_levels ? 1 : 0;
    g.beta = c.beta;
    g.delta = c.delta;
    g.side = static_cast<int>(c.side);
    g.three_way = c.three_way ? 1 : 0;
    g.block = c.block;
    return g;
}

inline void throw_on(int rc, const char* where) {
    if (rc != QMSORT_OK)
        throw std::runtime_error(std::string(where) + " failed (" + std::to_string(rc) +
                                 "): " + qmsort_gpu_last_error());
}

// Host-range drop-in for qmsort::sort(first, last, cfg, less).
template <class It, class Cfg = SortConfig, class Less = std::less<>, class Observer = void>
Metrics sort(It first, It last, const Cfg& cfg = Cfg{}, Less = Less{}, Observer* = nullptr) {
    using T = typename std::iterator_traits<It>::value_type;
    static_assert(std::is_base_of_v<std::random_access_iterator_tag,
                                    typename std::iterator_traits<It>::iterator_category>,
                  "contiguous random-access range required");
    const std::size_t n = static_cast<std::size_t>(last - first);
    Metrics m;
    if (n == 0) return m;
    qmsort_gpu_config c = to_c(cfg);
    qmsort_gpu_metrics gm{};
    throw_on(qmsort_gpu_sort_host(dtype_code<T>(), cmp_code<Less, T>(), &*first, n, &c, &gm),
             "qmsort_gpu_sort_host");
    m.max_depth = gm.max_depth;
    m.elapsed_ns = gm.elapsed_ns;
    return m;
}

// Device-range variant: d_first..d_last in GPU memory, optional stream.
template <class T, class Cfg = SortConfig, class Less = std::less<>>
Metrics sort_device(T* d_first, T* d_last, const Cfg& cfg = Cfg{}, Less = Less{},
                    void* stream = nullptr) {
    Metrics m;
    qmsort_gpu_config c = to_c(cfg);
    qmsort_gpu_metrics gm{};
    throw_on(qmsort_gpu_sort(dtype_code<T>(), cmp_code<Less, T>(), d_first,
                             static_cast<std::size_t>(d_last - d_first), &c, nullptr, 0, &gm, stream),
             "qmsort_gpu_sort");
    m.max_depth = gm.max_depth;
    m.elapsed_ns = gm.elapsed_ns;
    return m;
}

}  // namespace gpu
}  // namespace qmsort
