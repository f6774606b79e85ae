// qmsort_gpu.hpp -- C++ drop-in over the C-ABI (qmsort_gpu.h).
//
// Mirrors the reference entry point
//     template <class It, class Less = std::less<>>
//     Metrics qmsort::sort(It first, It last, const SortConfig& cfg = {}, Less less = {},
//                          SortObserver* obs = nullptr);          // sort.hpp:215-226
// as qmsort::gpu::sort with the same argument meaning: a contiguous range of
// int32 / int64 / uint32 / uint64 / double / 32-byte records, or of key +
// payload elements (any standard-layout type with a scalar `key` member, such
// as the reference's Element<PayloadBytes>, element.hpp:13-20), a SortConfig (ours, or the
// reference's own qmsort::SortConfig -- any type with the same member names),
// and std::less / std::greater.  The range is copied to the B200, sorted there
// and copied back; failures throw std::runtime_error (as trial.hpp:116 does),
// never fall back to the CPU.  SortObserver hooks are accepted and ignored
// (the GPU pipeline has no QuickXsort steps to observe).
#pragma once

#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <functional>
#include <iterator>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

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

// partition_result.hpp:12-17: [0, lt_end) < pivot, [lt_end, gt_begin) ==
// pivot, [gt_begin, n) > pivot (the three-way contract, partition.hpp:196-230).
struct PartitionResult {
    std::size_t lt_end = 0;
    std::size_t gt_begin = 0;
    std::size_t left_size = 0;
    std::size_t right_size = 0;
};

// Element type -> qmsort_dtype.  A user-defined 32-byte record is enabled by
// specialising qmsort::gpu::is_rec32<T>: a declaration that T is four uint64
// words whose std::less order (T's operator<) is lexicographic over w0..w3.
// A record comparator functor other than std::less / std::greater must be
// declared the same way through qmsort::gpu::rec32_order<Less, T> (value
// QMSORT_LESS for the lexicographic order, QMSORT_GREATER for its reverse);
// any other comparator is rejected at compile time -- the GPU cannot run an
// arbitrary functor, and a silent substitution would sort wrongly.
template <class T>
struct is_rec32 : std::false_type {};
template <class Less, class T>
struct rec32_order : std::integral_constant<int, -1> {};
template <class T>
constexpr int scalar_code() {
    if constexpr (std::is_integral_v<T> && std::is_signed_v<T> && sizeof(T) == 4) return QMSORT_DT_I32;
    else if constexpr (std::is_integral_v<T> && std::is_unsigned_v<T> && sizeof(T) == 4) return QMSORT_DT_U32;
    else if constexpr (std::is_integral_v<T> && std::is_signed_v<T> && sizeof(T) == 8) return QMSORT_DT_I64;
    else if constexpr (std::is_integral_v<T> && std::is_unsigned_v<T> && sizeof(T) == 8) return QMSORT_DT_U64;
    else if constexpr (std::is_same_v<T, double>) return QMSORT_DT_F64;
    else return -1;
}
// Key + payload element: a standard-layout class with a scalar `key` member.
template <class T, class = void>
struct is_keyed_element : std::false_type {};
template <class T>
struct is_keyed_element<T, std::void_t<decltype(std::declval<const T&>().key)>>
    : std::bool_constant<std::is_class_v<T> && std::is_standard_layout_v<T> &&
                         std::is_trivially_copyable_v<T> &&
                         scalar_code<std::remove_cv_t<decltype(std::declval<T&>().key)>>() >= 0> {};

template <class T>
constexpr int dtype_code() {
    if constexpr (scalar_code<T>() >= 0) return scalar_code<T>();
    else if constexpr (is_rec32<T>::value) {
        static_assert(sizeof(T) == 32 && std::is_trivially_copyable_v<T>, "rec32 must be 32 trivially copyable bytes");
        return QMSORT_DT_REC32;
    } else {
        static_assert(sizeof(T) == 0, "qmsort::gpu::sort supports int32, int64, uint32, uint64, double, rec32 and keyed elements");
        return -1;
    }
}

template <class Less, class T>
constexpr int cmp_code() {
    if constexpr (std::is_same_v<Less, std::less<>> || std::is_same_v<Less, std::less<T>>) return QMSORT_LESS;
    else if constexpr (std::is_same_v<Less, std::greater<>> || std::is_same_v<Less, std::greater<T>>)
        return QMSORT_GREATER;
    else if constexpr (is_rec32<T>::value && rec32_order<Less, T>::value >= 0) return rec32_order<Less, T>::value;
    else {
        static_assert(sizeof(Less) == 0,
                      "comparator must be std::less or std::greater (records: or a functor declared through "
                      "qmsort::gpu::rec32_order<Less, T>)");
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

// Is It a contiguous iterator (C++20 concept; pointers and the standard
// contiguous containers' iterators before C++20)?
template <class It>
constexpr bool is_contiguous() {
#if __cplusplus >= 202002L
    return std::contiguous_iterator<It>;
#else
    using T = typename std::iterator_traits<It>::value_type;
    return std::is_pointer_v<It> || std::is_same_v<It, typename std::vector<T>::iterator> ||
           std::is_same_v<It, typename std::vector<T>::const_iterator>;
#endif
}

template <class T, class Cfg, class Less>
void sort_contiguous(T* p, std::size_t n, const Cfg& cfg, qmsort_gpu_metrics& gm) {
    qmsort_gpu_config c = to_c(cfg);
    if constexpr (is_keyed_element<T>::value && !is_rec32<T>::value) {
        // Element<PayloadBytes>: ordered on the key alone (element.hpp:17-18)
        using Key = std::remove_cv_t<decltype(std::declval<T&>().key)>;
        throw_on(qmsort_gpu_sort_elements_host(scalar_code<Key>(), cmp_code<Less, T>(), p, n, sizeof(T),
                                               offsetof(T, key), &c, &gm),
                 "qmsort_gpu_sort_elements_host");
    } else {
        throw_on(qmsort_gpu_sort_host(dtype_code<T>(), cmp_code<Less, T>(), p, n, &c, &gm), "qmsort_gpu_sort_host");
    }
}

// Host-range drop-in for qmsort::sort(first, last, cfg, less) (sort.hpp:215-226).
// Any random-access range, like the reference's: a contiguous one is sorted
// in place through the host-array call; another (std::deque ...) is gathered
// into a contiguous buffer, sorted, and written back.
template <class It, class Cfg = SortConfig, class Less = std::less<>, class Observer = void>
Metrics sort(It first, It last, const Cfg& cfg = Cfg{}, Less = Less{}, Observer* = nullptr) {
    using T = typename std::iterator_traits<It>::value_type;
    static_assert(std::is_base_of_v<std::random_access_iterator_tag,
                                    typename std::iterator_traits<It>::iterator_category>,
                  "random-access range required");
    const std::size_t n = static_cast<std::size_t>(last - first);
    Metrics m;
    if (n == 0) return m;
    qmsort_gpu_metrics gm{};
    if constexpr (is_contiguous<It>()) {
        sort_contiguous<T, Cfg, Less>(&*first, n, cfg, gm);
    } else {
        std::vector<T> buf(first, last);
        sort_contiguous<T, Cfg, Less>(buf.data(), n, cfg, gm);
        std::copy(buf.begin(), buf.end(), first);
    }
    m.max_depth = gm.max_depth;
    m.elapsed_ns = gm.elapsed_ns;
    return m;
}

// sort_range_counted(first, last, cfg, cmp, m, obs) (sort.hpp:207-211): sort
// with a caller-owned comparator object and Metrics; the counters accumulate
// into m (elapsed_ns adds the device time, max_depth the deepest partition;
// comparisons / moves are not counted on the GPU).  Cmp is std::less /
// std::greater (or a declared record order); the reference's
// CountingComparator<Less> wrapper is unwrapped to its Less by the caller.
template <class It, class Cfg, class Cmp, class Observer = void>
void sort_range_counted(It first, It last, const Cfg& cfg, Cmp& cmp, Metrics& m, Observer* obs = nullptr) {
    const Metrics r = sort(first, last, cfg, cmp, obs);
    m.elapsed_ns += r.elapsed_ns;
    m.max_depth = std::max(m.max_depth, r.max_depth);
}

// Three-way partition of a host range around `pivot` (a value) under Less,
// in place on the B200: the PartitionResult of partition_result.hpp:12-17.
template <class It, class Less = std::less<>>
PartitionResult partition(It first, It last, const typename std::iterator_traits<It>::value_type& pivot,
                          Less = Less{}, Metrics* m = nullptr) {
    using T = typename std::iterator_traits<It>::value_type;
    static_assert(is_contiguous<It>(), "partition needs a contiguous range");
    const std::size_t n = static_cast<std::size_t>(last - first);
    std::uint64_t c[3] = {0, 0, 0};
    qmsort_gpu_metrics gm{};
    throw_on(qmsort_gpu_partition3_host(dtype_code<T>(), cmp_code<Less, T>(), n ? &*first : nullptr, n, &pivot, c,
                                        nullptr, &gm),
             "qmsort_gpu_partition3_host");
    if (m) m->elapsed_ns += gm.elapsed_ns;
    PartitionResult r;
    r.lt_end = static_cast<std::size_t>(c[0]);
    r.gt_begin = static_cast<std::size_t>(c[0] + c[1]);
    r.left_size = r.lt_end;
    r.right_size = static_cast<std::size_t>(c[2]);
    return r;
}

// select_nth(first, last, k, cmp, m) (selection.hpp:207-212): k is 1-based;
// returns the offset of the k-th smallest under Less, with the range
// partitioned around it.  Less is std::less / std::greater.
template <class It, class Less = std::less<>>
std::size_t select_nth(It first, It last, std::size_t k, Less = Less{}, Metrics* m = nullptr,
                       const SortConfig& cfg = SortConfig{}) {
    using T = typename std::iterator_traits<It>::value_type;
    static_assert(is_contiguous<It>(), "select_nth needs a contiguous range");
    const std::size_t n = static_cast<std::size_t>(last - first);
    qmsort_gpu_config c = to_c(cfg);
    qmsort_gpu_metrics gm{};
    std::size_t pos = 0;
    throw_on(qmsort_gpu_select_nth_host(dtype_code<T>(), cmp_code<Less, T>(), &*first, n, k, &pos, &c, &gm),
             "qmsort_gpu_select_nth_host");
    if (m) {
        m->max_depth = std::max<std::uint64_t>(m->max_depth, gm.max_depth);
        m->elapsed_ns += gm.elapsed_ns;
    }
    return pos;
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
