// qmsort_gpu.cu -- host orchestration and the C-ABI (include/qmsort_gpu.h).
//
// Maps the reference QuickXsort driver (detail::quickmergesort_impl,
// sort.hpp:128-201) onto B200 kernels:
//   reference step                         B200 replacement
//   pivot (median_of_3 / median_of_sqrt)   K1 sample_kernel: K-1 sampled splitters
//   block_partition (two sides)            K2-K4 count / plan / scatter (K buckets)
//   "continue on the other side" loop      level loop over device segment lists
//   mergesort_with_temp + base case X      K5 block sort of every bucket <= cap
//   swap_merge recursion (large ranges)    K6/K7 merge-path passes (fallback and
//                                          algorithm = mergesort)
// Buffers: the caller's array A and a workspace array B of the same size are
// used ping-pong.  Every scatter writes each bucket at its FINAL offset, so the
// two buffers share one coordinate system and the sorted result always ends
// in A.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <chrono>
#include <map>
#include <set>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/qmsort_gpu.h"
#include "aux_kernels.cuh"
#include "blocksort.cuh"
#include "common.cuh"
#include "elements.cuh"
#include "mergepass.cuh"
#include "samplesort.cuh"
#include "tablesort.cuh"

namespace qmsort_b200 {

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define QCK(x)                                                                               \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess)                                                               \
            return fail(QMSORT_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
    } while (0)
// QMSORT_DEBUG_SYNC=1: synchronise after every launch and name the failing
// one (source line) -- a debugging aid, off by default.
static bool debug_sync() {
    static const bool on = [] {
        const char* e = std::getenv("QMSORT_DEBUG_SYNC");
        return e && e[0] == '1';
    }();
    return on;
}
#define QCK_LAUNCH(led)                                                                      \
    do {                                                                                     \
        ++(led).launches;                                                                    \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ == cudaSuccess && debug_sync()) {                                             \
            e_ = cudaDeviceSynchronize();                                                    \
            std::fprintf(stderr, "qmsort debug: launch %d at qmsort_gpu.cu:%d %s\n",         \
                         (led).launches, __LINE__, cudaGetErrorString(e_));                  \
        }                                                                                    \
        if (e_ != cudaSuccess)                                                               \
            return fail(QMSORT_ECUDA, std::string("kernel launch (qmsort_gpu.cu:") +         \
                                          std::to_string(__LINE__) + "): " + cudaGetErrorString(e_)); \
    } while (0)
#define QLAUNCH(led, ph, bytes, ...) \
    do {                             \
        (led).pre(ph);               \
        __VA_ARGS__;                 \
        (led).post(bytes);           \
        QCK_LAUNCH(led);             \
    } while (0)
#define QTRY(x)                      \
    do {                             \
        int r_ = (x);                \
        if (r_ != QMSORT_OK) return r_; \
    } while (0)

// Per-key-type tile shapes.  Class c of the block sorter sorts buckets of up to
// CLS_T[c] * BI keys with CLS_T[c] threads; the largest class is the cap.
template <class K>
struct Tune;
template <>
struct Tune<uint32_t> {
    static constexpr int LOGKMAX = 9;
    static constexpr int BI = 32;                                 // block sort keys / thread
    // block sort classes (96: tiles just over 2048 keys keep all three warps
    // busy; trailing repeats are never chosen -- kNumClasses is the widest list)
    static constexpr int CLS_T[kNumClasses] = {64, 96, 128, 256, 512, 512, 512, 512, 512};
    // task list 5 (a repeat the size rule never picks): the buckets the plan
    // finds eligible for the table sort (tablesort.cuh)
#ifndef QMSORT_TABLE_SORT
#define QMSORT_TABLE_SORT 1
#endif
    static constexpr int TABLE_CLASS = QMSORT_TABLE_SORT ? 5 : kNumClasses;
    // task list 6: buckets for the wide-span table sort (CellSort)
#ifndef QMSORT_CELL_SORT
#define QMSORT_CELL_SORT 1
#endif
    static constexpr int CELL_CLASS = QMSORT_CELL_SORT ? 6 : kNumClasses;
    static constexpr int CELL_BIG_CLASS = kNumClasses;  // (none)
    // even splitters at a last level: ranges of about EVEN_TARGET keys and at
    // most EVEN_SPAN values -- table-sort buckets filling 15 of its 16 rows
#ifndef QMSORT_U32_EVEN_TARGET
#define QMSORT_U32_EVEN_TARGET 3700
#endif
    static constexpr int EVEN_TARGET = QMSORT_TABLE_SORT ? QMSORT_U32_EVEN_TARGET : 0, EVEN_SPAN = 65535,
                         EVEN_OVER = 0;
    static constexpr int TARGET_DIV = 4;                          // target bucket = cap / 4
    // last level: 3/4 of the target, so most tiles stay inside the packed
    // 16-bit block sort's span (measured: block sort 1817 -> 1716 us on C2)
#ifndef QMSORT_U32_LAST_NUM
#define QMSORT_U32_LAST_NUM 3
#define QMSORT_U32_LAST_DEN 4
#endif
    static constexpr int LAST_NUM = QMSORT_U32_LAST_NUM, LAST_DEN = QMSORT_U32_LAST_DEN;
#ifndef QMSORT_U32_SAMPLE_THREADS
#define QMSORT_U32_SAMPLE_THREADS 512
#endif
    static constexpr int ST = QMSORT_U32_SAMPLE_THREADS, SI = 16;  // sampler
    static constexpr int XT = 512, XI = 16;  // scatter tile
    static constexpr int CT = 256, CU = 16;  // count
    static constexpr int MT = 512, MI = 16;  // merge pass
    static constexpr int BMI = 16;  // bulk merge pass (two stages of MT x BMI keys)
    // merge pass kernel: the plain one (measured on C2, 14 passes: 9.9 ms
    // against 12.2 ms staged by the bulk-copy engine, 11.9 ms with 16-byte
    // register stores; 8 keys per thread 13.7 ms)
    static constexpr bool MERGE_BULK = false;
};
template <>
struct Tune<uint64_t> {
    static constexpr int LOGKMAX = 9;
    static constexpr int BI = 16;
    static constexpr int CLS_T[kNumClasses] = {64, 96, 128, 192, 256, 384, 512, 512, 512};  // measured: C3 block sort -7 %
    static constexpr int TABLE_CLASS = kNumClasses;  // no dense table sort
    static constexpr int CELL_CLASS = QMSORT_CELL_SORT ? 7 : kNumClasses;
    static constexpr int CELL_BIG_CLASS = QMSORT_CELL_SORT ? 8 : kNumClasses;  // buckets beyond 2048 keys
#ifndef QMSORT_U64_EVEN_TARGET
#define QMSORT_U64_EVEN_TARGET 7600
#endif
    // even splitters: K ranges; a last level that K ranges would leave with
    // buckets over the small cell-sort tile (2048 keys) takes ranges of 7600
    // keys instead -- the big tile 15/16 full (measured: C3 42.6 -> 45.1 Gkeys/s;
    // applied to every last level C4 loses 7 %)
    static constexpr int EVEN_TARGET = QMSORT_U64_EVEN_TARGET, EVEN_SPAN = 0, EVEN_OVER = 2048;
    static constexpr int TARGET_DIV = 4;
#ifndef QMSORT_U64_LAST_NUM
#define QMSORT_U64_LAST_NUM 1
#define QMSORT_U64_LAST_DEN 1
#endif
    static constexpr int LAST_NUM = QMSORT_U64_LAST_NUM, LAST_DEN = QMSORT_U64_LAST_DEN;  // measured with the cell sort: 1/1 (C4a +1.5 %, C4d +2.7 %, C3 +0.4 % over 3/4)
    static constexpr int ST = 512, SI = 16;
    static constexpr int XT = 512, XI = 12;  // measured: C3 scatter 14.8 -> 13.7 ms, C4a 2.55 -> 2.17 ms (was 256 x 16)
    static constexpr int CT = 256, CU = 8;
    static constexpr int MT = 512, MI = 16;
    static constexpr int BMI = 16;
    static constexpr bool MERGE_BULK = true;  // measured on C3, 17 passes: 84.2 ms against 101.2 ms plain
};
template <>
struct Tune<Rec32> {
    static constexpr int LOGKMAX = 8;
    static constexpr int BI = 8;
    static constexpr int CLS_T[kNumClasses] = {64, 96, 128, 256, 512, 512, 512, 512, 512};
#ifndef QMSORT_REC_CELL_SORT
#define QMSORT_REC_CELL_SORT 1
#endif
    // task list 7: buckets of 256..2048 records for the cell sort on record prefixes
    static constexpr int TABLE_CLASS = kNumClasses, CELL_CLASS = QMSORT_REC_CELL_SORT ? 7 : kNumClasses,
                         CELL_BIG_CLASS = kNumClasses;
    static constexpr int EVEN_TARGET = 0, EVEN_SPAN = 0, EVEN_OVER = 0;
    static constexpr int TARGET_DIV = 2;
    static constexpr int LAST_NUM = 1, LAST_DEN = 2;  // measured: C5 block sort 2.55 -> 2.32 ms
    static constexpr int ST = 512, SI = 8;
    static constexpr int XT = 512, XI = 4;  // measured: C5 scatter 2.84 -> 2.73 ms (was 256 x 8)
    static constexpr int CT = 256, CU = 4;
    static constexpr int MT = 512, MI = 8;
    static constexpr int BMI = 4;  // 2 x 64 KB stages
    static constexpr bool MERGE_BULK = true;  // measured on C5: 24.8 ms against 27.9 ms plain
};
template <class K>
constexpr uint32_t class_cap(int c) {
    return (uint32_t)Tune<K>::CLS_T[c] * Tune<K>::BI;
}

// Kernel families for the per-phase ledger (qmsort_gpu_metrics.phase_*).
enum Phase {
    kPhTransform = 0,
    kPhSample = 1,
    kPhCount = 2,
    kPhPlan = 3,
    kPhScatter = 4,
    kPhBlocksort = 5,
    kPhMerge = 6,
    kPhFill = 7,
};

// Pass ledger: algorithmic bytes per kernel family and, when profiling is on,
// CUDA-event device time of every launch.
struct Ledger {
    uint64_t alg_bytes = 0;
    uint32_t launches = 0, syncs = 0, levels = 0, merge_passes = 0, resplits = 0;
    uint64_t sample_keys = 0;
    uint32_t table_buckets = 0;
    uint64_t ph_bytes[QMSORT_NUM_PHASES] = {};
    uint32_t ph_launches[QMSORT_NUM_PHASES] = {};
    bool prof = false;
    cudaStream_t st = nullptr;
    int cur = 0;
    cudaEvent_t pending = nullptr;
    struct Rec {
        int ph;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    void pre(int ph) {
        cur = ph;
        if (prof) {
            cudaEventCreate(&pending);
            cudaEventRecord(pending, st);
        }
    }
    void post(uint64_t bytes) {
        ph_bytes[cur] += bytes;
        alg_bytes += bytes;
        ++ph_launches[cur];
        if (prof) {
            cudaEvent_t b;
            cudaEventCreate(&b);
            cudaEventRecord(b, st);
            recs.push_back({cur, pending, b});
            pending = nullptr;
        }
    }
    // After the stream is synchronised: per-phase device time.
    void collect(uint64_t* ph_ns) {
        for (const Rec& r : recs) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) ph_ns[r.ph] += (uint64_t)((double)ms * 1e6);
        }
    }
    ~Ledger() {
        for (const Rec& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        if (pending) cudaEventDestroy(pending);
    }
};

// Raise the dynamic shared-memory limit of a kernel once per (device,
// kernel): the attribute belongs to the device context, so a process that
// sorts on several GPUs sets it on each.
static int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
static cudaError_t allow_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    if (bytes <= 48 * 1024) return cudaSuccess;
    const auto key = std::make_pair(current_device(), fn);
    std::lock_guard<std::mutex> g(mu);
    if (done.count(key)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Waits inside a sort poll instead of blocking: the host thread never sleeps,
// so the launches that follow a control read go out at once (the wake-up of a
// blocking wait occasionally left milliseconds of idle GPU between kernels).
static cudaError_t spin_sync(cudaStream_t st) {
    cudaError_t e;
    while ((e = cudaStreamQuery(st)) == cudaErrorNotReady) {
    }
    return e;
}
static cudaError_t spin_event(cudaEvent_t ev) {
    cudaError_t e;
    while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
    }
    return e;
}

// Pool of small mapped pinned host buffers for control reads (read_small).
constexpr uint32_t kMappedBytes = 8192;
static std::mutex g_mapped_mu;
static std::vector<unsigned char*> g_mapped_free;
struct MappedBuf {
    unsigned char* host = nullptr;
    unsigned char* dev = nullptr;
    ~MappedBuf() {
        if (host) {
            std::lock_guard<std::mutex> g(g_mapped_mu);
            g_mapped_free.push_back(host);
        }
    }
};

// Copy up to two small device regions (<= kMappedBytes in total) to the host:
// a store kernel on `st` writes them into mapped pinned memory, then the
// stream is synchronised.  Unlike a device-to-host cudaMemcpyAsync this never
// waits behind a bulk copy of another stream on the copy engine.
static int read_small(cudaStream_t st, void* dst0, const void* src0, size_t b0,
                      void* dst1 = nullptr, const void* src1 = nullptr, size_t b1 = 0) {
    if (b0 + b1 > kMappedBytes) return fail(QMSORT_EINTERNAL, "read_small: too many bytes");
    MappedBuf mb;
    {
        std::lock_guard<std::mutex> g(g_mapped_mu);
        if (!g_mapped_free.empty()) {
            mb.host = g_mapped_free.back();
            g_mapped_free.pop_back();
        }
    }
    if (!mb.host) {
        void* h = nullptr;
        QCK(cudaHostAlloc(&h, kMappedBytes, cudaHostAllocMapped));
        mb.host = static_cast<unsigned char*>(h);
    }
    void* dptr = nullptr;
    QCK(cudaHostGetDevicePointer(&dptr, mb.host, 0));
    mb.dev = static_cast<unsigned char*>(dptr);
    SmallRead r0{static_cast<const unsigned char*>(src0), (uint32_t)b0, 0};
    SmallRead r1{static_cast<const unsigned char*>(src1), (uint32_t)b1, (uint32_t)align_up(b0, 16)};
    store_mapped_kernel<<<1, 256, 0, st>>>(r0, r1, mb.dev);
    QCK(cudaGetLastError());
    QCK(spin_sync(st));
    std::memcpy(dst0, mb.host, b0);
    if (b1) std::memcpy(dst1, mb.host + r1.dst_off, b1);
    return QMSORT_OK;
}

// Grid size of a persistent kernel: resident CTAs per SM x SMs (cached per
// device and kernel).
static unsigned resident_grid(const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, unsigned> cache;
    const int dev = current_device();
    const auto key = std::make_pair(dev, fn);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const unsigned r = (unsigned)(per_sm * sms);
    cache[key] = r;
    return r;
}

constexpr int kCntSlots = 18;  // LevelCounters of one sort: one per partition level (+1)

struct WsLayout {
    size_t b_off = 0, segs_off[2] = {0, 0}, chunks_off[2] = {0, 0}, cnt_off[2] = {0, 0};
    size_t tree_off[2] = {0, 0}, sorted_off[2] = {0, 0}, lut_off[2] = {0, 0};
    size_t hist_off = 0, tasks_off = 0, fills_off = 0, misc_off = 0, total = 0;
    uint32_t seg_cap = 0, chunk_cap = 0, split_cap = 0, task_cap = 0, fill_cap = 0, hist_cap = 0;
    uint32_t min_cap = 0;  // smallest block-sort takeover size the work lists are sized for
    uint64_t chunk_elems = 0;
};

// The largest bucket the block sorter takes: every bucket that fits one CTA,
// or -- beta with base_case.use_levels (base_case_levels, sort.hpp:91-96:
// X on blocks of about n^beta) -- n^beta clamped to the size classes.
template <class K>
static uint32_t takeover_cap(size_t n, const qmsort_gpu_config* cfg) {
    constexpr uint32_t cap_max = class_cap<K>(kNumClasses - 1);
    if (!cfg || !cfg->base_case_use_levels || !(cfg->beta > 0.0 && cfg->beta < 1.0)) return cap_max;
    const double t = std::pow((double)std::max<size_t>(n, 2), cfg->beta);
    return (uint32_t)std::min<double>(cap_max, std::max<double>(class_cap<K>(0), t));
}

template <class K>
static WsLayout make_layout(size_t n, uint32_t min_cap = class_cap<K>(kNumClasses - 1)) {
    using TU = Tune<K>;
    const uint64_t cap = min_cap;
    const uint64_t target = cap / TU::TARGET_DIV;
    constexpr uint64_t tile = (uint64_t)TU::XT * TU::XI;
    WsLayout L;
    // chunks of 16 tiles, dispensed dynamically to persistent CTAs
    const uint64_t ch = tile * 16;
    L.chunk_elems = ch;
    L.min_cap = min_cap;
    L.seg_cap = (uint32_t)(n / cap + 2);
    L.chunk_cap = (uint32_t)(L.seg_cap + n / ch + 2);
    const uint64_t last_target = target * TU::LAST_NUM / TU::LAST_DEN;  // choose_logk's last level
    L.split_cap = (uint32_t)(2 * n / last_target + 2 * (uint64_t)L.seg_cap + 2 * (1u << TU::LOGKMAX) + 64);
    L.task_cap = 4 * L.split_cap + 64;  // per class, all levels of one sort
    L.fill_cap = 2 * L.split_cap;  // small fills from the front, large from the back (each <= split_cap)
    // histogram words of one level: a segment of len keys takes (nch + 1) 2K
    // words with nch <= len/ch + 1 and 2K <= min(2 K_max, 4 len/last_target + 4)
    // (choose_logk), so a level needs at most
    //   2 K_max n/ch + 8 n/last_target + 8 segments
    L.hist_cap = (uint32_t)(2ull * (1u << TU::LOGKMAX) * (n / ch + 4) + 8ull * (n / last_target + 1) +
                            8ull * L.seg_cap + 4096);
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o = align_up(o + bytes, 256);
        return at;
    };
    L.b_off = take(n * sizeof(K));
    for (int i = 0; i < 2; ++i) {
        L.segs_off[i] = take(sizeof(SegDesc) * L.seg_cap);
        L.chunks_off[i] = take(sizeof(ChunkDesc) * L.chunk_cap);
        L.cnt_off[i] = take(sizeof(LevelCounters) * (i == 0 ? kCntSlots : 1));
        L.tree_off[i] = take(sizeof(K) * L.split_cap);
        L.sorted_off[i] = take(sizeof(K) * L.split_cap);
        L.lut_off[i] = take(KeyTraits<K>::kLut ? sizeof(uint32_t) * kLutPerSplitter * (size_t)L.split_cap : 0);
    }
    L.hist_off = take(sizeof(uint32_t) * (size_t)L.hist_cap);
    L.tasks_off = take(sizeof(SortTask) * (size_t)kNumClasses * L.task_cap);
    L.fills_off = take(sizeof(FillTask) * (size_t)L.fill_cap);
    L.misc_off = take(4096);
    L.total = o;
    return L;
}

template <class K, int T, int I>
static int launch_tiles(const K* src, K* dst, uint64_t off, uint64_t len, cudaStream_t st,
                        Ledger& led) {
    using BS = BlockSorter<K, T, I>;
    if (len == 0) return QMSORT_OK;
    auto fn = blocksort_tiles_kernel<K, T, I>;
    QCK(allow_smem((const void*)fn, BS::kSmemBytes));
    const uint64_t tiles = (len + BS::kCap - 1) / BS::kCap;
    QLAUNCH(led, kPhBlocksort, 2 * len * sizeof(K),
            fn<<<(unsigned)tiles, T, BS::kSmemBytes, st>>>(src, dst, off, len));
    return QMSORT_OK;
}

template <class K, int C>
static int blocksort_one_from(const K* src, K* dst, uint64_t off, uint64_t len, cudaStream_t st,
                              Ledger& led) {
    if constexpr (C + 1 < kNumClasses) {
        if (len > class_cap<K>(C)) return blocksort_one_from<K, C + 1>(src, dst, off, len, st, led);
    }
    return launch_tiles<K, Tune<K>::CLS_T[C], Tune<K>::BI>(src, dst, off, len, st, led);
}

// Sort [off, off+len) with len <= the cap: one CTA of the smallest class.
template <class K>
static int blocksort_one(const K* src, K* dst, uint64_t off, uint64_t len, cudaStream_t st,
                         Ledger& led) {
    using TU = Tune<K>;
    return blocksort_one_from<K, 0>(src, dst, off, len, st, led);
}

// Block-sort the `count` tasks of size class C into A: one CTA per task.
template <class K, int C>
static int launch_class(const SortTask* tasks, uint32_t count, K* A, const K* B, cudaStream_t st,
                        Ledger& led, Xf xf) {
    using TU = Tune<K>;
    constexpr int T = TU::CLS_T[C];
    using BS = BlockSorter<K, T, TU::BI>;
    if (count == 0) return QMSORT_OK;
    if constexpr (std::is_same<K, uint32_t>::value && C == TU::TABLE_CLASS) {
        QCK(allow_smem((const void*)tablesort_tasks_kernel, TableSort::kSmemBytes));
        QLAUNCH(led, kPhBlocksort, 0,
                tablesort_tasks_kernel<<<count, TableSort::T, TableSort::kSmemBytes, st>>>(tasks, A, B, xf));
        return QMSORT_OK;
    }
    if constexpr (C == TU::CELL_CLASS || C == TU::CELL_BIG_CLASS) {
        constexpr bool BIG = C == TU::CELL_BIG_CLASS;
        using CS = CellSort<K, BIG>;
        auto fn = cellsort_tasks_kernel<K, BIG>;
        QCK(allow_smem((const void*)fn, CS::kSmemBytes));
        QLAUNCH(led, kPhBlocksort, 0, fn<<<count, CS::T, CS::kSmemBytes, st>>>(tasks, A, B, xf));
        return QMSORT_OK;
    }
    auto fn = blocksort_tasks_kernel<K, T, TU::BI>;
    QCK(allow_smem((const void*)fn, BS::kSmemBytes));
    QLAUNCH(led, kPhBlocksort, 0, fn<<<count, T, BS::kSmemBytes, st>>>(tasks, A, B, xf));
    return QMSORT_OK;
}

// Every size class's task list, smallest first.
template <class K, int C>
static int launch_classes_from(const SortTask* tasks, uint32_t task_cap, const uint32_t* nt, K* A,
                               const K* B, cudaStream_t st, Ledger& led, Xf xf) {
    QTRY((launch_class<K, C>(tasks + (size_t)C * task_cap, nt[C], A, B, st, led, xf)));
    if constexpr (C + 1 < kNumClasses) return launch_classes_from<K, C + 1>(tasks, task_cap, nt, A, B, st, led, xf);
    return QMSORT_OK;
}

// Partition levels a balanced split needs before every bucket fits the block
// sorter: the levels enqueued at once, without a host round trip between them.
static int estimate_levels(uint64_t n, const PlanParams& p) {
    int lv = 0;
    uint64_t len = n;
    while (len > p.cap && lv < 16) {
        const uint32_t k = choose_logk(len, p.target, p.last_target, p.log_kmax, p.cap);
        len = (len + (1ull << k) - 1) >> k;
        ++lv;
    }
    return lv;
}

// Block-sort tiles + merge-path passes over [off, off+len); the range currently
// lives in X (A or B); the result lands in A.
template <class K>
static int xf_range(K* p, uint64_t n, Xf xf, bool inverse, cudaStream_t st, Ledger& led) {
    if (n == 0) return QMSORT_OK;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    QLAUNCH(led, kPhTransform, 2 * n * sizeof(K), xf_kernel<K><<<grid, 256, 0, st>>>(p, n, xf, inverse ? 1 : 0));
    return QMSORT_OK;
}

#ifndef QMSORT_MERGE_BULK
#define QMSORT_MERGE_BULK 1
#endif
// splits (optional, splits_cap entries): device scratch for the Blackwell
// merge pass (K6a split points + K6b bulk-copy staging); without it, or with
// QMSORT_MERGE_BULK=0, the warp-search kernel with plain loads runs.
template <class K>
static int mergesort_range(K* X, K* A, K* B, uint64_t off, uint64_t len, cudaStream_t st,
                           Ledger& led, uint64_t* splits = nullptr, size_t splits_cap = 0) {
    using TU = Tune<K>;
    constexpr uint64_t C = class_cap<K>(kNumClasses - 1);
    constexpr uint64_t MC = (uint64_t)TU::MT * TU::MI;
    static_assert(MC <= 2 * C, "merge tile must fit in one run pair");
    static_assert(C % MC == 0, "merge tiles never straddle a run pair");
    if (len <= C) return blocksort_one<K>(X, A, off, len, st, led);
    const uint64_t tiles = (len + C - 1) / C;
    const uint32_t passes = ceil_log2_u64(tiles);
    K* Y = (passes % 2 == 0) ? A : B;
    QTRY((launch_tiles<K, TU::CLS_T[kNumClasses - 1], TU::BI>(X, Y, off, len, st, led)));
    K* s = Y;
    K* d = (Y == A) ? B : A;
    constexpr uint64_t BC = (uint64_t)TU::MT * TU::BMI;  // bulk merge tile
    static_assert(C % BC == 0, "bulk merge tiles never straddle a run pair");
    const uint64_t mtiles = (len + MC - 1) / MC;
    const uint64_t btiles = (len + BC - 1) / BC;
    if (QMSORT_MERGE_BULK && TU::MERGE_BULK && splits && splits_cap >= btiles) {
        using BM = BulkMerge<K, TU::MT, TU::BMI>;
        auto fn = merge_pass_bulk_kernel<K, TU::MT, TU::BMI>;
        QCK(allow_smem((const void*)fn, BM::kSmemBytes));
        const unsigned grid = (unsigned)std::min<uint64_t>(btiles, resident_grid((const void*)fn, TU::MT, BM::kSmemBytes));
        for (uint64_t run = C; run < len; run *= 2) {
            QLAUNCH(led, kPhMerge, 0,
                    merge_split_kernel<K><<<(unsigned)std::min<uint64_t>((btiles + 255) / 256, 1184), 256, 0, st>>>(
                        s + off, len, run, BC, btiles, splits));
            QLAUNCH(led, kPhMerge, 2 * len * sizeof(K),
                    fn<<<grid, TU::MT, BM::kSmemBytes, st>>>(s + off, d + off, len, run, splits, btiles));
            ++led.merge_passes;
            std::swap(s, d);
        }
    } else {
        using BS = BlockSorter<K, TU::MT, TU::MI>;
        auto fn = merge_pass_kernel<K, TU::MT, TU::MI>;
        QCK(allow_smem((const void*)fn, BS::kSmemBytes));
        for (uint64_t run = C; run < len; run *= 2) {
            QLAUNCH(led, kPhMerge, 2 * len * sizeof(K),
                    fn<<<(unsigned)mtiles, TU::MT, BS::kSmemBytes, st>>>(s + off, d + off, len, run));
            ++led.merge_passes;
            std::swap(s, d);
        }
    }
    if (s != A) return fail(QMSORT_EINTERNAL, "merge passes ended outside the caller buffer");
    return QMSORT_OK;
}

// xf (fused transform): level 0 reads the caller's keys through f, every
// final write (block sort, fills, merge fallback) goes through f^-1.
// A level 0 done elsewhere (the folded sharded exchange): B holds the n core
// keys grouped into the three-way bins of the m distinct splitters uniq
// (device, core keys) -- open, equal, open, ..., open, with the host's
// counts[2m+1] -- equal bins unwritten (they become fills).
template <class K>
struct Presplit {
    const K* uniq;
    uint32_t m;
    const uint64_t* counts;
};

// src0 (optional): level 0 reads the keys from there instead of A (an
// out-of-place sort; src0 is only read).  pre (optional): start at level 1
// from a level 0 done elsewhere.
template <class K>
static int samplesort(K* A, K* B, size_t n, const qmsort_gpu_config& cfg, unsigned char* ws,
                      const WsLayout& L, cudaStream_t st, Ledger& led, Xf xf, const K* src0 = nullptr,
                      const Presplit<K>* pre = nullptr) {
    const bool fused = xf.a != 0 || xf.b != 0;
    using TU = Tune<K>;
    constexpr uint32_t cap_max = class_cap<K>(kNumClasses - 1);
    // beta (sort.hpp:25-34, base_case_levels sort.hpp:91-96): with
    // base_case.use_levels the reference runs X on blocks of about n^beta; here
    // n^beta is the largest bucket the block sorter takes (clamped to the
    // block sorter's classes); otherwise every bucket that fits one CTA does
    // (never below what the work lists were sized for: other entry points
    // lay out their workspace for the default takeover size)
    const uint32_t cap = std::min(cap_max, std::max(takeover_cap<K>(n, &cfg), L.min_cap));
    PlanParams p;
    p.chunk_elems = L.chunk_elems;
    p.cap = cap;
    p.target = cap / TU::TARGET_DIV;
    p.last_target = p.target * TU::LAST_NUM / TU::LAST_DEN;
    p.log_kmax = TU::LOGKMAX;
    for (int c = 0; c < kNumClasses; ++c) p.class_cap[c] = class_cap<K>(c);
    p.task_cap = L.task_cap;
    p.fill_cap = L.fill_cap;
    p.dst_is_a = 0;
    p.xf_fix = fused ? 1u : 0u;
    p.pivot = (uint32_t)std::max(0, cfg.pivot);
    const double dl = std::min(1.0, std::max(1.0 / 65536.0, cfg.delta > 0 ? cfg.delta : 1.0 / 16.0));
    p.delta_q16 = (uint32_t)(dl * 65536.0);
    p.table_class = (uint32_t)TU::TABLE_CLASS;
    p.cell_class = (uint32_t)TU::CELL_CLASS;
    if constexpr (KeyTraits<K>::kLut) {
        p.cell_cap = (uint32_t)CellSort<K>::kCap;
        p.cell_bits = (uint32_t)CellSort<K>::kCellBits;
        p.cell_big_cap = (uint32_t)CellSort<K, true>::kCap;
        p.cell_big_bits = (uint32_t)CellSort<K, true>::kCellBits;
    } else {
        p.cell_cap = (uint32_t)CellSort<K>::kCap;
        p.cell_bits = (uint32_t)CellSort<K>::kCellBits;
        p.cell_big_cap = p.cell_big_bits = 0;
    }
    p.cell_big_class = (uint32_t)TU::CELL_BIG_CLASS;

    LevelBufs lv[2];
    K* tree[2];
    K* sorted[2];
    uint32_t* lut[2];
    LevelCounters* cnts = reinterpret_cast<LevelCounters*>(ws + L.cnt_off[0]);
    // sort-wide block-sort tasks and equal-key fills: every level's small
    // buckets keep their place (later levels never touch them), so they are
    // all sorted once, after the last partition level
    LevelCounters* tot = &cnts[kCntSlots - 1];
    for (int i = 0; i < 2; ++i) {
        lv[i].segs = reinterpret_cast<SegDesc*>(ws + L.segs_off[i]);
        lv[i].chunks = reinterpret_cast<ChunkDesc*>(ws + L.chunks_off[i]);
        lv[i].cnt = &cnts[i];
        lv[i].seg_cap = L.seg_cap;
        lv[i].chunk_cap = L.chunk_cap;
        lv[i].split_cap = L.split_cap;
        lv[i].hist_cap = L.hist_cap;
        tree[i] = reinterpret_cast<K*>(ws + L.tree_off[i]);
        sorted[i] = reinterpret_cast<K*>(ws + L.sorted_off[i]);
        lut[i] = reinterpret_cast<uint32_t*>(ws + L.lut_off[i]);
    }
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist_off);
    SortTask* tasks = reinterpret_cast<SortTask*>(ws + L.tasks_off);
    FillTask* fills = reinterpret_cast<FillTask*>(ws + L.fills_off);

    // every level's counters start at zero; level l reads its segment and
    // chunk counts from cnts[l] (written by level l-1) on the device
    QCK(cudaMemsetAsync(cnts, 0, sizeof(LevelCounters) * kCntSlots, st));
    const uint64_t key_max = ~0ull >> (64 - 8 * (int)std::min<size_t>(8, sizeof(K)));
    if (!pre) QLAUNCH(led, kPhPlan, 0, init_level_kernel<<<16, 256, 0, st>>>(lv[0], n, key_max, p));

    using BSS = BlockSorter<K, TU::ST, TU::SI>;
    auto sample_fn = sample_kernel<K, TU::ST, TU::SI>;
    auto sample_xf_fn = sample_kernel<K, TU::ST, TU::SI, true>;
    QCK(allow_smem((const void*)sample_fn, BSS::kSmemBytes));
    QCK(allow_smem((const void*)sample_xf_fn, BSS::kSmemBytes));
    using SM = ScatterSmem<K, TU::XT, TU::XI, TU::LOGKMAX>;
    auto scatter_fn = scatter_kernel<K, TU::XT, TU::XI, TU::LOGKMAX>;
    QCK(allow_smem((const void*)scatter_fn, sizeof(SM)));
    auto count_fn = count_kernel<K, TU::CT, TU::CU, TU::LOGKMAX>;
    const unsigned scatter_grid = resident_grid((const void*)scatter_fn, TU::XT, sizeof(SM));
    const unsigned count_grid = resident_grid((const void*)count_fn, TU::CT, 0);
    const unsigned sample_grid = resident_grid((const void*)sample_fn, TU::ST, BSS::kSmemBytes);
    auto plan_fn = plan_kernel<K, 512, TU::LOGKMAX>;
    const unsigned plan_grid = resident_grid((const void*)plan_fn, 512, 0);
    const unsigned colsum_grid = resident_grid((const void*)colsum_kernel, 512, 0);

    K* src = src0 ? const_cast<K*>(src0) : A;  // level 0 only reads it
    K* dst = B;
    int level = 0;
    int batch = std::max(1, estimate_levels(n, p));
    if (pre) {
        // level 0's result is in B: its segment (one, three-way, no chunks:
        // the bin totals are the plan's histogram) and the plan of its
        // children, then the level loop from level 1 (B -> A)
        const uint32_t logk = std::max<uint32_t>(1, ceil_log2_u64((uint64_t)pre->m + 1));
        if (logk > (uint32_t)TU::LOGKMAX) return fail(QMSORT_EINVAL, "presplit: too many splitters");
        SegDesc d{};
        d.off = 0;
        d.len = n;
        d.lo = 0;
        d.hi = key_max;
        d.logk = logk;
        d.m = pre->m;
        d.eq = 1;
        d.lutbits = std::min(logk + 4, (uint32_t)kLutMaxBits);
        std::vector<uint32_t> hh(2u << logk, 0);
        uint64_t biggest = 0;
        for (uint32_t b = 0; b < 2 * pre->m + 1; ++b) {
            hh[b] = (uint32_t)pre->counts[b];
            if (!(b & 1)) biggest = std::max<uint64_t>(biggest, pre->counts[b]);
        }
        const uint32_t one = 1;
        QCK(cudaMemcpyAsync(lv[0].segs, &d, sizeof(d), cudaMemcpyHostToDevice, st));
        QCK(cudaMemcpyAsync(hist, hh.data(), hh.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        QCK(cudaMemcpyAsync(&cnts[0].nsegs, &one, sizeof(one), cudaMemcpyHostToDevice, st));
        if (pre->m) QCK(cudaMemcpyAsync(sorted[0], pre->uniq, sizeof(K) * pre->m, cudaMemcpyDeviceToDevice, st));
        p.dst_is_a = 0;  // level 0 "wrote" B
        lv[0].cnt = &cnts[0];
        lv[1].cnt = &cnts[1];
        QLAUNCH(led, kPhPlan, 0,
                plan_fn<<<plan_grid, 512, 0, st>>>(lv[0].segs, hist, sorted[0], lv[1], p, tasks, fills, &cnts[0], tot));
        level = 1;
        src = B;
        dst = A;
        batch = std::max(1, estimate_levels(biggest, p));
        // the fake level 0 adds nothing to the pass ledger (its nkeys is 0)
    }
    // median_of_sqrt_n (median_of_sqrt_pivot, partition.hpp:235-251): level 0
    // draws s = 2 floor(sqrt(n)/2) + 1 strided keys; more than one block sort
    // holds are sorted here first (block sort + merge passes in B, which
    // level 0's scatter only overwrites after its sample kernel has read them)
    const K* presorted = nullptr;
    uint32_t presorted_n = 0;
    {
        const uint64_t s0 = sqrt_sample_size(n);
        if (!pre && cfg.pivot == 1 && s0 > (uint64_t)BSS::kCap && 2 * s0 <= n) {
            const uint64_t stride = n / s0;
            QLAUNCH(led, kPhSample, 0,
                    gather_strided_kernel<K><<<(unsigned)std::min<uint64_t>((s0 + 255) / 256, 1184), 256, 0, st>>>(
                        src, n, s0, stride, B, xf));
            QTRY(mergesort_range<K>(B, B, B + s0, 0, s0, st, led, reinterpret_cast<uint64_t*>(ws + L.hist_off),
                                    L.hist_cap / 2));
            presorted = B;
            presorted_n = (uint32_t)s0;
        }
    }
    const int max_levels = std::max(level + 1, std::min(cfg.max_levels > 0 ? cfg.max_levels : 8, kCntSlots - 2));
    LevelCounters hc[kCntSlots];
    for (;;) {
        // enqueue a batch of levels back to back: every grid is persistent
        // and reads its work counts on the device
        const int stop = std::min(level + batch, max_levels);
        for (; level < stop; ++level) {
            const int cur = level & 1, nxt = cur ^ 1;
            lv[cur].cnt = &cnts[level];
            lv[nxt].cnt = &cnts[level + 1];
            LevelCounters* c = &cnts[level];
            p.dst_is_a = (dst == A) ? 1 : 0;
            const uint64_t seed = cfg.seed ^ (0x5851F42D4C957F2Dull * (uint64_t)(level + 1));
            const Xf lxf = level == 0 ? xf : Xf{0, 0};  // only level 0 reads the caller's keys
            QLAUNCH(led, kPhSample, 0,
                    (level == 0 && fused ? sample_xf_fn : sample_fn)<<<sample_grid, TU::ST, BSS::kSmemBytes, st>>>(
                        lv[cur].segs, &c->nsegs, src, tree[cur], sorted[cur], lut[cur], seed, 32u, lxf,
                        level == 0 ? presorted : nullptr, level == 0 ? presorted_n : 0u,
                        (uint32_t)TU::EVEN_TARGET, (uint32_t)TU::EVEN_SPAN, (uint32_t)TU::EVEN_OVER));
            QLAUNCH(led, kPhCount, 0,
                    count_fn<<<count_grid, TU::CT, 0, st>>>(lv[cur].segs, lv[cur].chunks, 0u, &c->nchunks,
                                                            &c->work_count, src, tree[cur], sorted[cur],
                                                            lut[cur], hist, lxf));
            QLAUNCH(led, kPhPlan, 0,
                    colsum_kernel<<<colsum_grid, 512, 0, st>>>(lv[cur].segs, hist, c));
            QLAUNCH(led, kPhPlan, 0,
                    plan_fn<<<plan_grid, 512, 0, st>>>(lv[cur].segs, hist, sorted[cur], lv[nxt], p, tasks,
                                                      fills, c, tot));
            QLAUNCH(led, kPhScatter, 0,
                    scatter_fn<<<scatter_grid, TU::XT, sizeof(SM), st>>>(
                        lv[cur].segs, lv[cur].chunks, 0u, &c->nchunks, &c->work_scatter, src, dst,
                        tree[cur], sorted[cur], lut[cur], hist, PeerArgs{}, lxf));
            // A and B alternate; an out-of-place source is left after level 0
            K* prev = src;
            src = dst;
            dst = (prev == A || prev == B) ? prev : A;
        }
        // one control read per batch
        QTRY(read_small(st, hc, cnts, sizeof(LevelCounters) * (size_t)(level + 1), &hc[kCntSlots - 1],
                        tot, sizeof(LevelCounters)));
        ++led.launches;
        ++led.syncs;
        for (int l = 0; l <= level; ++l)
            if (hc[l].overflow) return fail(QMSORT_EINTERNAL, "samplesort work-list capacity exceeded");
        if (hc[level].nsegs == 0) break;
        if (level >= max_levels) {
            // K8 fallback: the remaining oversized buckets are merge-sorted.
            std::vector<SegDesc> h(hc[level].nsegs);
            QCK(cudaMemcpyAsync(h.data(), lv[level & 1].segs, sizeof(SegDesc) * h.size(),
                                cudaMemcpyDeviceToHost, st));
            QCK(spin_sync(st));
            ++led.syncs;
            for (const SegDesc& d : h) {
                QTRY(mergesort_range<K>(src, A, B, d.off, d.len, st, led,
                                        reinterpret_cast<uint64_t*>(ws + L.hist_off), L.hist_cap / 2));
                if (fused) QTRY(xf_range<K>(A + d.off, d.len, xf, true, st, led));
            }
            break;
        }
        batch = 1;  // more levels than a balanced split needs: continue one at a time
    }
    // block-sort every bucket that fits one CTA (all levels; counts from the
    // control read), then the fills
    const uint32_t* nt = hc[kCntSlots - 1].ntasks;
    for (int c = 0; c < kNumClasses; ++c)
        if (nt[c] > L.task_cap) return fail(QMSORT_EINTERNAL, "block-sort task list capacity exceeded");
    QTRY((launch_classes_from<K, 0>(tasks, L.task_cap, nt, A, B, st, led, xf)));
    if (TU::TABLE_CLASS < kNumClasses) led.table_buckets += nt[TU::TABLE_CLASS < kNumClasses ? TU::TABLE_CLASS : 0];
    if (TU::CELL_CLASS < kNumClasses) led.table_buckets += nt[TU::CELL_CLASS < kNumClasses ? TU::CELL_CLASS : 0];
    if (TU::CELL_BIG_CLASS < kNumClasses)
        led.table_buckets += nt[TU::CELL_BIG_CLASS < kNumClasses ? TU::CELL_BIG_CLASS : 0];
    if (hc[kCntSlots - 1].nfill || hc[kCntSlots - 1].nfill_big)
        QLAUNCH(led, kPhFill, 0,
                fill_kernel<K><<<1184, 256, 0, st>>>(fills, &tot->nfill, &tot->nfill_big, L.fill_cap, A, xf));
    // pass ledger from the device counters (count 1, scatter 2, block sort 2, fill 1)
    const uint64_t w = sizeof(K);
    for (int l = 0; l < level; ++l) {
        const LevelCounters& c = hc[l];
        if (c.nsegs == 0) continue;
        ++led.levels;
        led.resplits += c.resplits;
        led.sample_keys += c.sample_keys;
        led.ph_bytes[kPhCount] += c.nkeys * w;
        led.ph_bytes[kPhScatter] += 2 * c.nkeys * w;
        led.alg_bytes += 3 * c.nkeys * w;
    }
    const LevelCounters& t = hc[kCntSlots - 1];
    if (t.overflow) return fail(QMSORT_EINTERNAL, "samplesort work-list capacity exceeded");
    led.ph_bytes[kPhBlocksort] += 2 * t.task_keys * w;
    led.ph_bytes[kPhFill] += t.fill_keys * w;
    led.alg_bytes += 2 * t.task_keys * w + t.fill_keys * w;
    return QMSORT_OK;
}

// xf: the caller's keys are f^-1(core keys); the samplesort path fuses f and
// f^-1 into its first reads and last writes, the others run them as passes.
// src0 (optional): sort the n keys at src0 into A (src0 is only read).
template <class K>
static int sort_core(K* A, size_t n, const qmsort_gpu_config& cfg, unsigned char* ws,
                     const WsLayout& L, cudaStream_t st, Ledger& led, Xf xf = Xf{0, 0},
                     const K* src0 = nullptr) {
    constexpr uint64_t cap = class_cap<K>(kNumClasses - 1);
    if (src0 == A) src0 = nullptr;
    if (n <= 1) {
        if (n == 1 && src0) QCK(cudaMemcpyAsync(A, src0, sizeof(K), cudaMemcpyDeviceToDevice, st));
        return QMSORT_OK;
    }
    const bool fused = xf.a != 0 || xf.b != 0;
    K* B = reinterpret_cast<K*>(ws + L.b_off);
    if (n > cap && cfg.algorithm != 1) return samplesort<K>(A, B, n, cfg, ws, L, st, led, xf, src0);
    if (src0) QCK(cudaMemcpyAsync(A, src0, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    if (fused) QTRY(xf_range<K>(A, n, xf, false, st, led));
    if (n <= cap) QTRY(blocksort_one<K>(A, A, 0, n, st, led));
    else QTRY(mergesort_range<K>(A, A, B, 0, n, st, led, reinterpret_cast<uint64_t*>(ws + L.hist_off),
                                 L.hist_cap / 2));
    if (fused) QTRY(xf_range<K>(A, n, xf, true, st, led));
    return QMSORT_OK;
}

static int core_dtype(int dt) {
    if (dt == QMSORT_DT_I32) return QMSORT_DT_U32;
    if (dt == QMSORT_DT_F64 || dt == QMSORT_DT_I64) return QMSORT_DT_U64;
    return dt;
}

static size_t dtype_size(int dt) {
    switch (dt) {
        case QMSORT_DT_I32:
        case QMSORT_DT_U32: return 4;
        case QMSORT_DT_U64:
        case QMSORT_DT_I64:
        case QMSORT_DT_F64: return 8;
        case QMSORT_DT_REC32: return 32;
    }
    return 0;
}

static size_t ws_bytes_for(int dt, size_t n, const qmsort_gpu_config* cfg = nullptr) {
    switch (core_dtype(dt)) {
        case QMSORT_DT_U32: return make_layout<uint32_t>(n, takeover_cap<uint32_t>(n, cfg)).total;
        case QMSORT_DT_U64: return make_layout<uint64_t>(n, takeover_cap<uint64_t>(n, cfg)).total;
        case QMSORT_DT_REC32: return make_layout<Rec32>(n, takeover_cap<Rec32>(n, cfg)).total;
    }
    return 0;
}

// The comparator's transform as an Xf (common.cuh; the same maps as
// transform32/64_kernel).
static Xf make_xf(int dt, int cmp) {
    constexpr uint64_t S = 0x8000000000000000ull, M = 0x7FFFFFFFFFFFFFFFull;
    switch (dt) {
        case QMSORT_DT_I32: return Xf{0, cmp ? 0x7FFFFFFFull : 0x80000000ull};
        case QMSORT_DT_U32: return Xf{0, cmp ? 0xFFFFFFFFull : 0};
        case QMSORT_DT_U64: return Xf{0, cmp ? ~0ull : 0};
        case QMSORT_DT_F64: return Xf{M, cmp ? M : S};
        case QMSORT_DT_I64: return Xf{0, cmp ? M : S};
        case QMSORT_DT_REC32: return Xf{0, cmp ? ~0ull : 0};
    }
    return Xf{0, 0};
}

// Launch the forward / inverse order-preserving transform.
static int run_transform(int dt, int cmp, void* d, size_t n, int inverse, cudaStream_t st,
                         Ledger& led) {
    int mode = kXfNone;
    bool wide = false;
    size_t words = n;
    switch (dt) {
        case QMSORT_DT_I32: mode = cmp ? kXfI32Greater : kXfI32Less; break;
        case QMSORT_DT_U32: mode = cmp ? kXfU32Greater : kXfNone; break;
        case QMSORT_DT_U64: mode = cmp ? kXfU64Greater : kXfNone; wide = true; break;
        case QMSORT_DT_F64: mode = cmp ? kXfF64Greater : kXfF64Less; wide = true; break;
        case QMSORT_DT_I64: mode = cmp ? kXfI64Greater : kXfI64Less; wide = true; break;
        case QMSORT_DT_REC32: mode = cmp ? kXfU64Greater : kXfNone; wide = true; words = 4 * n; break;
    }
    if (mode == kXfNone || n == 0) return QMSORT_OK;
    const unsigned grid = (unsigned)std::min<size_t>((words + 255) / 256, 148 * 16);
    if (wide)
        QLAUNCH(led, kPhTransform, 2 * n * dtype_size(dt),
                transform64_kernel<<<grid, 256, 0, st>>>(static_cast<uint64_t*>(d), words, mode, inverse));
    else
        QLAUNCH(led, kPhTransform, 2 * n * dtype_size(dt),
                transform32_kernel<<<grid, 256, 0, st>>>(static_cast<uint32_t*>(d), words, mode));
    return QMSORT_OK;
}

static int validate(int dt, int cmp, size_t n, const void* p) {
    if (dtype_size(dt) == 0) return fail(QMSORT_EINVAL, "unknown dtype");
    if (cmp != QMSORT_LESS && cmp != QMSORT_GREATER) return fail(QMSORT_EINVAL, "unknown comparator");
    if (n >= (1ull << 32)) return fail(QMSORT_EINVAL, "n must be < 2^32");
    if (n > 0 && p == nullptr) return fail(QMSORT_EINVAL, "null data pointer");
    return QMSORT_OK;
}

static void fill_metrics(qmsort_gpu_metrics* m, Ledger& led, float ms) {
    if (!m) return;
    std::memset(m, 0, sizeof(*m));
    m->elapsed_ns = (uint64_t)((double)ms * 1e6);
    m->max_depth = led.levels;
    m->alg_bytes = led.alg_bytes;
    m->levels = led.levels;
    m->merge_passes = led.merge_passes;
    m->kernel_launches = led.launches;
    m->host_syncs = led.syncs + 1;
    m->resplits = led.resplits;
    m->sample_keys = led.sample_keys;
    m->table_buckets = led.table_buckets;
    for (int i = 0; i < QMSORT_NUM_PHASES; ++i) {
        m->phase_bytes[i] = led.ph_bytes[i];
        m->phase_launches[i] = led.ph_launches[i];
    }
    led.collect(m->phase_ns);
}

// src (optional): sort the n keys at src into d, leaving src untouched.
static int sort_device(int dt, int cmp, void* d, size_t n, const qmsort_gpu_config* cfgp,
                       void* wsp, size_t ws_bytes, qmsort_gpu_metrics* m, cudaStream_t st,
                       const void* src = nullptr) {
    QTRY(validate(dt, cmp, n, d));
    if (src == d) src = nullptr;
    if (src && n > 0 && ((const char*)src < (const char*)d + n * dtype_size(dt)) &&
        ((const char*)d < (const char*)src + n * dtype_size(dt)))
        return fail(QMSORT_EINVAL, "source and destination ranges overlap");
    qmsort_gpu_config cfg;
    if (cfgp) cfg = *cfgp;
    else qmsort_gpu_config_init(&cfg, 0);
    const size_t need = ws_bytes_for(dt, n, &cfg);
    void* ws = wsp;
    bool own = false;
    if (ws == nullptr && n > 1) {
        QCK(cudaMallocAsync(&ws, need, st));
        own = true;
    } else if (n > 1 && ws_bytes < need) {
        return fail(QMSORT_ENOWS, "workspace too small: need " + std::to_string(need) + " bytes");
    }
    if (src && n == 1) QCK(cudaMemcpyAsync(d, src, dtype_size(dt), cudaMemcpyDeviceToDevice, st));
    Ledger led;
    led.prof = cfg.profile != 0;
    led.st = st;
    cudaEvent_t e0, e1;
    QCK(cudaEventCreate(&e0));
    QCK(cudaEventCreate(&e1));
    QCK(cudaEventRecord(e0, st));
    // the comparator's order-preserving transform runs inside the sort
    // (fused into its first reads and last writes), not as extra passes
    const Xf xf = make_xf(dt, cmp);
    int rc = QMSORT_OK;
    unsigned char* w = static_cast<unsigned char*>(ws);
    switch (core_dtype(dt)) {
        case QMSORT_DT_U32:
            rc = sort_core<uint32_t>(static_cast<uint32_t*>(d), n, cfg, w,
                                     make_layout<uint32_t>(n, takeover_cap<uint32_t>(n, &cfg)), st, led, xf,
                                     static_cast<const uint32_t*>(src));
            break;
        case QMSORT_DT_U64:
            rc = sort_core<uint64_t>(static_cast<uint64_t*>(d), n, cfg, w,
                                     make_layout<uint64_t>(n, takeover_cap<uint64_t>(n, &cfg)), st, led, xf,
                                     static_cast<const uint64_t*>(src));
            break;
        case QMSORT_DT_REC32:
            rc = sort_core<Rec32>(static_cast<Rec32*>(d), n, cfg, w, make_layout<Rec32>(n, takeover_cap<Rec32>(n, &cfg)),
                                  st, led, xf,
                                  static_cast<const Rec32*>(src));
            break;
    }
    cudaEventRecord(e1, st);
    cudaError_t se = spin_event(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (own) cudaFreeAsync(ws, st);
    if (rc != QMSORT_OK) return rc;
    if (se != cudaSuccess) return fail(QMSORT_ECUDA, std::string("sort: ") + cudaGetErrorString(se));
    fill_metrics(m, led, ms);
    g_err.clear();
    return QMSORT_OK;
}

// ---------------------------------------------------------------------------
// Sharded building blocks
// ---------------------------------------------------------------------------
template <class K>
__global__ void gather_sample_kernel(const K* __restrict__ src, uint64_t n, uint64_t s,
                                     uint64_t seed, K* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = sm_mix(seed + (i + 1) * kGamma);
        out[i] = src[__umul64hi(h, n)];
    }
}

// Classifier (LUT or Eytzinger tree) of caller-given sorted splitters for one
// segment covering the whole input.  eq = 1 (the sharded exchange, distinct
// splitters): three-way bins, 2j = keys between splitters j-1 and j, 2j+1 =
// keys equal to splitter j.
template <class K>
__global__ void given_splitters_kernel(const K* __restrict__ spl, uint32_t nsplit, uint32_t logk,
                                       SegDesc* seg, K* tree, K* sorted, uint32_t* lut, uint64_t n,
                                       uint32_t nchunks, ChunkDesc* chunks, uint64_t chunk_elems,
                                       uint64_t key_max, uint32_t eq) {
    using KT = KeyTraits<K>;
    const uint32_t K_ = 1u << logk;
    const uint32_t lutbits = min(logk + 4, (uint32_t)kLutMaxBits);
    uint32_t bl = 0;
    while (bl < 64 && (key_max >> bl) != 0) ++bl;
    const uint32_t shift = bl > lutbits ? bl - lutbits : 0;
    for (uint32_t i = threadIdx.x; i < K_; i += blockDim.x) sorted[i] = i < nsplit ? spl[i] : KT::max_key();
    if constexpr (KT::kLut) {
        for (uint32_t c = threadIdx.x; c < (1u << lutbits); c += blockDim.x) {
            const uint64_t cmin = (uint64_t)c << shift;
            uint64_t cmax = cmin + (((uint64_t)1 << shift) - 1);
            if (c == (1u << lutbits) - 1 || cmax > key_max || cmax < cmin) cmax = key_max;
            uint32_t r[2];
            for (int w = 0; w < 2; ++w) {
                const uint64_t v = w == 0 ? cmin : cmax;
                uint32_t lo = 0, cnt = nsplit;
                while (cnt > 0) {
                    const uint32_t half = cnt >> 1;
                    if ((uint64_t)KT::bits(spl[lo + half]) < v) {
                        lo += half + 1;
                        cnt -= half + 1;
                    } else {
                        cnt = half;
                    }
                }
                r[w] = lo;
            }
            if (r[1] < r[0]) r[1] = r[0];  // a cell past key_max: empty range (see sample_segment)
            lut[c] = r[0] | ((r[1] - r[0]) << 16);
        }
    } else {
        for (uint32_t t = threadIdx.x + 1; t < K_; t += blockDim.x) {
            const uint32_t depth = 31 - __clz(t);
            const uint32_t rank = ((2 * (t - (1u << depth)) + 1) << (logk - 1 - depth)) - 1;
            tree[t] = rank < nsplit ? spl[rank] : KT::max_key();
        }
    }
    for (uint32_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
        ChunkDesc cd;
        cd.seg = 0;
        cd.pad = 0;
        cd.begin = (uint64_t)c * chunk_elems;
        cd.end = min(n, cd.begin + chunk_elems);
        chunks[c] = cd;
    }
    if (threadIdx.x == 0) {
        SegDesc d;
        d.off = 0;
        d.len = n;
        d.lo = 0;
        d.hi = key_max;
        d.chunk_begin = 0;
        d.nchunks = nchunks;
        d.logk = logk;
        d.m = nsplit;
        d.eq = eq;
        d.sp = 0;
        d.hist_base = 0;
        d.shift = shift;
        d.lutbits = lutbits;
        d.sampler = kSampleRandom;
        d.arith = d.scale = 0;
        *seg = d;
    }
}

// Offsets only (no children): bucket starts in place of the totals and the
// bucket counts (bin b = bucket j, three-way off).
template <int T, int LOG_KMAX>
__global__ void __launch_bounds__(T) given_plan_kernel(const SegDesc* __restrict__ segs,
                                                       uint32_t* __restrict__ hist,
                                                       uint32_t ncounts, uint64_t* counts) {
    constexpr int NB = 2 << LOG_KMAX;
    __shared__ uint32_t start[NB];
    __shared__ uint32_t warp_sums[32];
    const SegDesc d = segs[0];
    const uint32_t nb = (1u << d.logk) << d.eq;
    const uint32_t stride = d.nchunks + 1;
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        const uint32_t v = hist[b * stride + d.nchunks];
        start[b] = v;
        if (b < ncounts) counts[b] = v;
    }
    __syncthreads();
    block_exclusive_scan_smem<T>(start, (int)nb, warp_sums);
    for (uint32_t b = threadIdx.x; b < nb; b += T) hist[b * stride + d.nchunks] = start[b];
}

// Partition the n keys at `in` by nsplit sorted splitters (count + plan when
// parts & 1, scatter when parts & 2).  eq: distinct splitters, three-way bins
// (2 nsplit + 1 counts).  xf: `in` holds the caller's keys, classified through
// f (the splitters are core keys); local scatters write core keys, the peer
// scatter the caller's.
template <class K>
static int partition_given(const K* in, size_t n, const K* spl, uint32_t nsplit, K* out,
                           uint64_t* counts, unsigned char* ws, const WsLayout& L, cudaStream_t st,
                           Ledger& led, int parts = 3, const PeerArgs* peers = nullptr,
                           bool eq = false, Xf xf = Xf{0, 0}) {
    using TU = Tune<K>;
    const uint32_t logk = std::max<uint32_t>(1, ceil_log2_u64((uint64_t)nsplit + 1));
    if (logk > (uint32_t)TU::LOGKMAX) return fail(QMSORT_EINVAL, "too many splitters");
    SegDesc* seg = reinterpret_cast<SegDesc*>(ws + L.segs_off[0]);
    ChunkDesc* chunks = reinterpret_cast<ChunkDesc*>(ws + L.chunks_off[0]);
    K* tree = reinterpret_cast<K*>(ws + L.tree_off[0]);
    K* sorted = reinterpret_cast<K*>(ws + L.sorted_off[0]);
    uint32_t* lut = reinterpret_cast<uint32_t*>(ws + L.lut_off[0]);
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist_off);
    const uint64_t key_max = ~0ull >> (64 - 8 * (int)std::min<size_t>(8, sizeof(K)));
    const uint32_t nchunks = (uint32_t)std::max<uint64_t>(1, (n + L.chunk_elems - 1) / L.chunk_elems);
    LevelCounters* cnt = reinterpret_cast<LevelCounters*>(ws + L.cnt_off[0]);
    if (parts & 1) {  // classify + count + plan (bucket sizes into counts)
        QLAUNCH(led, kPhSample, 0,
                given_splitters_kernel<K><<<1, 256, 0, st>>>(spl, nsplit, logk, seg, tree, sorted, lut,
                                                             n, nchunks, chunks, L.chunk_elems, key_max,
                                                             eq ? 1u : 0u));
        const uint32_t ncounts = eq ? 2 * nsplit + 1 : nsplit + 1;
        QCK(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * ncounts, st));
        if (n == 0) return QMSORT_OK;
        QCK(cudaMemsetAsync(cnt, 0, sizeof(LevelCounters), st));
        auto count_fn = count_kernel<K, TU::CT, TU::CU, TU::LOGKMAX>;
        QLAUNCH(led, kPhCount, n * sizeof(K),
                count_fn<<<std::min(nchunks, resident_grid((const void*)count_fn, TU::CT, 0)), TU::CT, 0,
                           st>>>(seg, chunks, nchunks, nullptr, &cnt->work_count, in, tree, sorted, lut, hist,
                                 xf));
        QLAUNCH(led, kPhPlan, 0, colsum_kernel<<<64, 512, 0, st>>>(seg, hist, nullptr));
        QLAUNCH(led, kPhPlan, 0, given_plan_kernel<512, TU::LOGKMAX><<<1, 512, 0, st>>>(seg, hist, ncounts, counts));
    }
    if (!(parts & 2) || n == 0) return QMSORT_OK;
    using SM = ScatterSmem<K, TU::XT, TU::XI, TU::LOGKMAX>;
    if (peers) {  // the exchange fused into the scatter: bucket b -> rank b's buffer
        auto fn = scatter_kernel<K, TU::XT, TU::XI, TU::LOGKMAX, true>;
        QCK(allow_smem((const void*)fn, sizeof(SM)));
        QLAUNCH(led, kPhScatter, 2 * n * sizeof(K),
                fn<<<std::min(nchunks, resident_grid((const void*)fn, TU::XT, sizeof(SM))), TU::XT,
                     sizeof(SM), st>>>(seg, chunks, nchunks, nullptr, &cnt->work_scatter, in, out, tree,
                                       sorted, lut, hist, *peers, xf));
        return QMSORT_OK;
    }
    auto scatter_fn = scatter_kernel<K, TU::XT, TU::XI, TU::LOGKMAX>;
    QCK(allow_smem((const void*)scatter_fn, sizeof(SM)));
    QLAUNCH(led, kPhScatter, 2 * n * sizeof(K),
            scatter_fn<<<std::min(nchunks, resident_grid((const void*)scatter_fn, TU::XT, sizeof(SM))),
                         TU::XT, sizeof(SM), st>>>(seg, chunks, nchunks, nullptr, &cnt->work_scatter, in,
                                                   out, tree, sorted, lut, hist, PeerArgs{}, xf));
    return QMSORT_OK;
}

// ---------------------------------------------------------------------------
// Call frame shared by the device entry points: optional library-owned
// workspace, CUDA-event timing and the metrics record.
// ---------------------------------------------------------------------------
struct CallFrame {
    cudaStream_t st;
    Ledger led;
    void* ws = nullptr;
    bool own = false;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    explicit CallFrame(cudaStream_t s) : st(s) { led.st = s; }
    int begin(const qmsort_gpu_config& cfg, void* wsp, size_t ws_bytes, size_t need) {
        led.prof = cfg.profile != 0;
        ws = wsp;
        if (ws == nullptr && need > 0) {
            QCK(cudaMallocAsync(&ws, need, st));
            own = true;
        } else if (need > 0 && ws_bytes < need) {
            return fail(QMSORT_ENOWS, "workspace too small: need " + std::to_string(need) + " bytes");
        }
        QCK(cudaEventCreate(&e0));
        QCK(cudaEventCreate(&e1));
        QCK(cudaEventRecord(e0, st));
        return QMSORT_OK;
    }
    // Synchronises the stream; rc is the status of the work in between.
    int end(int rc, qmsort_gpu_metrics* m) {
        float ms = 0.f;
        cudaError_t se = cudaSuccess;
        if (e1) {
            cudaEventRecord(e1, st);
            se = spin_event(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        if (own) cudaFreeAsync(ws, st);
        own = false;
        if (rc != QMSORT_OK) return rc;
        if (se != cudaSuccess) return fail(QMSORT_ECUDA, std::string("sync: ") + cudaGetErrorString(se));
        fill_metrics(m, led, ms);
        g_err.clear();
        return QMSORT_OK;
    }
    ~CallFrame() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

static const qmsort_gpu_config& cfg_or_default(const qmsort_gpu_config* p, qmsort_gpu_config& tmp) {
    if (p) return *p;
    qmsort_gpu_config_init(&tmp, 0);
    return tmp;
}

// ---------------------------------------------------------------------------
// f3: key + payload elements (element.hpp:13-20).  Workspace: the 32-byte
// records | the Rec32 samplesort workspace | the gathered elements.
// ---------------------------------------------------------------------------
struct ElemLayout {
    size_t recs_off, sort_off, gather_off, total;
};
static ElemLayout elem_layout(size_t n, size_t elem_bytes) {
    ElemLayout E;
    E.recs_off = 0;
    E.sort_off = align_up(n * sizeof(Rec32), 256);
    E.gather_off = E.sort_off + align_up(make_layout<Rec32>(std::max<size_t>(n, 2)).total, 256);
    E.total = E.gather_off + align_up(n * elem_bytes, 256);
    return E;
}

static int validate_elems(int kdt, int cmp, const void* p, size_t n, size_t elem_bytes, size_t key_off) {
    QTRY(validate(kdt, cmp, n, p));
    if (kdt == QMSORT_DT_REC32) return fail(QMSORT_EINVAL, "element keys must be scalar");
    const size_t kw = dtype_size(kdt);
    if (elem_bytes == 0 || elem_bytes % 4 != 0 || elem_bytes > 4096)
        return fail(QMSORT_EINVAL, "elem_bytes must be a multiple of 4 in [4, 4096]");
    if (elem_bytes % kw != 0 || key_off % kw != 0 || key_off + kw > elem_bytes)
        return fail(QMSORT_EINVAL, "key must be naturally aligned inside the element");
    return QMSORT_OK;
}

static int sort_elements_device(int kdt, int cmp, void* d, size_t n, size_t elem_bytes,
                                size_t key_off, const qmsort_gpu_config* cfgp, void* wsp,
                                size_t ws_bytes, qmsort_gpu_metrics* m, cudaStream_t st) {
    QTRY(validate_elems(kdt, cmp, d, n, elem_bytes, key_off));
    qmsort_gpu_config tmp;
    const qmsort_gpu_config& cfg = cfg_or_default(cfgp, tmp);
    CallFrame f(st);
    const ElemLayout E = elem_layout(n, elem_bytes);
    QTRY(f.begin(cfg, wsp, ws_bytes, n > 1 ? E.total : 0));
    int rc = QMSORT_OK;
    if (n > 1) {
        unsigned char* w = static_cast<unsigned char*>(f.ws);
        Rec32* recs = reinterpret_cast<Rec32*>(w + E.recs_off);
        unsigned char* out = w + E.gather_off;
        const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
        QLAUNCH(f.led, kPhTransform, n * (elem_bytes + sizeof(Rec32)),
                make_elem_recs_kernel<<<grid, 256, 0, st>>>(static_cast<const unsigned char*>(d), n,
                                                            (uint32_t)elem_bytes, (uint32_t)key_off,
                                                            kdt, cmp, recs));
        rc = sort_core<Rec32>(recs, n, cfg, w + E.sort_off, make_layout<Rec32>(std::max<size_t>(n, 2)), st, f.led);
        if (rc == QMSORT_OK) {
            const unsigned g2 = (unsigned)std::min<size_t>((n * (elem_bytes / 4) + 255) / 256, 148 * 16);
#define QGATHER(W)                                                                                  \
    QLAUNCH(f.led, kPhTransform, n * (2 * elem_bytes + sizeof(Rec32)),                              \
            gather_elems_kernel<W><<<g2, 256, 0, st>>>(static_cast<const W*>(d), reinterpret_cast<W*>(out), \
                                                      recs, n, (uint32_t)(elem_bytes / sizeof(W))))
            if (elem_bytes % 16 == 0) QGATHER(uint4);
            else if (elem_bytes % 8 == 0) QGATHER(uint2);
            else QGATHER(uint32_t);
#undef QGATHER
            QCK(cudaMemcpyAsync(d, out, n * elem_bytes, cudaMemcpyDeviceToDevice, st));
        }
    }
    return f.end(rc, m);
}

// ---------------------------------------------------------------------------
// f4: select_nth (selection.hpp:207-212).  The reference finds the k-th
// smallest by median-of-medians three-way partitioning (select_kth,
// selection.hpp:131-203) and leaves the range partitioned around it.  Here
// every round draws a sample, brackets rank k between two sampled keys s1 <=
// s2 and partitions the current window into  < s1 | == s1 | (s1, s2] | > s2
// with one count + scatter pass (K2-K4, caller-given splitters); the window
// shrinks to the bucket holding rank k (to a few percent of its size with
// high probability, and always by at least the keys equal to s1).  A window
// of equal keys ends the search; a small window is block-sorted.  Elements
// left of position k-1 are <= it and those right of it >= it, as in the
// reference.
// ---------------------------------------------------------------------------
template <class K>
struct HostKey {
    static bool is_min(const K& k) { return k == 0; }
    static K pred(const K& k) { return k - 1; }
    static bool eq(const K& a, const K& b) { return a == b; }
};
template <>
struct HostKey<Rec32> {
    static bool is_min(const Rec32& k) { return (k.w[0] | k.w[1] | k.w[2] | k.w[3]) == 0; }
    static Rec32 pred(const Rec32& k) {
        Rec32 r = k;
        for (int i = 3; i >= 0; --i) {
            if (r.w[i] != 0) {
                --r.w[i];
                break;
            }
            r.w[i] = ~0ull;
        }
        return r;
    }
    static bool eq(const Rec32& a, const Rec32& b) { return std::memcmp(&a, &b, sizeof(Rec32)) == 0; }
};

constexpr uint32_t kSelectSample = 4096;  // <= the smallest block-sort cap of every key type
constexpr uint32_t kSelectBand = 48;      // sample ranks either side of k (~3 sigma at p = 1/2)
constexpr size_t kSelectSortAt = 1u << 18;

template <class K>
static size_t select_extra_bytes() {
    return align_up(kSelectSample * sizeof(K), 256) + 256 + 256;
}

template <class K>
static int select_core(K* A, size_t n, size_t k0, const qmsort_gpu_config& cfg, unsigned char* ws,
                       const WsLayout& L, cudaStream_t st, Ledger& led) {
    static_assert(kSelectSample <= class_cap<K>(kNumClasses - 1), "sample must fit one block sort");
    K* B = reinterpret_cast<K*>(ws + L.b_off);
    K* smp = reinterpret_cast<K*>(ws + L.total);
    K* dspl = reinterpret_cast<K*>(ws + L.total + align_up(kSelectSample * sizeof(K), 256));
    uint64_t* dcnt = reinterpret_cast<uint64_t*>(ws + L.total + align_up(kSelectSample * sizeof(K), 256) + 256);
    size_t lo = 0, hi = n;
    for (uint32_t round = 0;; ++round) {
        const size_t m = hi - lo;
        if (m <= kSelectSortAt || round >= 64) return sort_core<K>(A + lo, m, cfg, ws, L, st, led);
        const uint64_t seed = cfg.seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(round + 1));
        QLAUNCH(led, kPhSample, 0,
                gather_sample_kernel<K><<<(kSelectSample + 255) / 256, 256, 0, st>>>(A + lo, m, kSelectSample, seed, smp));
        QTRY(blocksort_one<K>(smp, smp, 0, kSelectSample, st, led));
        const double frac = (double)(k0 - lo) / (double)m;
        const int64_t r = (int64_t)(frac * kSelectSample);
        const size_t i1 = (size_t)std::max<int64_t>(0, r - (int64_t)kSelectBand);
        const size_t i2 = (size_t)std::min<int64_t>(kSelectSample - 1, r + (int64_t)kSelectBand);
        K h[2];
        QTRY(read_small(st, &h[0], smp + i1, sizeof(K), &h[1], smp + i2, sizeof(K)));
        ++led.launches;
        ++led.syncs;
        K sp[3];
        uint32_t ns = 0;
        if (!HostKey<K>::is_min(h[0])) sp[ns++] = HostKey<K>::pred(h[0]);  // bucket "< s1"
        const uint32_t eqb = ns;                                            // bucket "== s1"
        sp[ns++] = h[0];
        if (!HostKey<K>::eq(h[0], h[1])) sp[ns++] = h[1];
        QCK(cudaMemcpyAsync(dspl, sp, sizeof(K) * ns, cudaMemcpyHostToDevice, st));
        QTRY(partition_given<K>(A + lo, m, dspl, ns, B + lo, dcnt, ws, L, st, led));
        uint64_t cnt[4] = {0, 0, 0, 0};
        QCK(cudaMemcpyAsync(cnt, dcnt, sizeof(uint64_t) * (ns + 1), cudaMemcpyDeviceToHost, st));
        QCK(cudaMemcpyAsync(A + lo, B + lo, m * sizeof(K), cudaMemcpyDeviceToDevice, st));
        QCK(spin_sync(st));
        ++led.syncs;
        ++led.levels;
        const size_t want = k0 - lo;
        size_t acc = 0;
        uint32_t b = 0;
        while (b < ns && want >= acc + cnt[b]) acc += cnt[b++];
        if (b == eqb) return QMSORT_OK;  // rank k sits among keys equal to s1
        lo += acc;
        hi = lo + cnt[b];
    }
}

static size_t select_ws_bytes(int dt, size_t n) {
    const size_t nn = std::max<size_t>(n, 2);
    switch (core_dtype(dt)) {
        case QMSORT_DT_U32: return make_layout<uint32_t>(nn).total + select_extra_bytes<uint32_t>();
        case QMSORT_DT_U64: return make_layout<uint64_t>(nn).total + select_extra_bytes<uint64_t>();
        case QMSORT_DT_REC32: return make_layout<Rec32>(nn).total + select_extra_bytes<Rec32>();
    }
    return 0;
}

static int select_device(int dt, int cmp, void* d, size_t n, size_t k, size_t* pos,
                         const qmsort_gpu_config* cfgp, void* wsp, size_t ws_bytes,
                         qmsort_gpu_metrics* m, cudaStream_t st) {
    QTRY(validate(dt, cmp, n, d));
    if (k < 1 || k > n) return fail(QMSORT_EINVAL, "k must satisfy 1 <= k <= n (1-based rank)");
    qmsort_gpu_config tmp;
    const qmsort_gpu_config& cfg = cfg_or_default(cfgp, tmp);
    CallFrame f(st);
    QTRY(f.begin(cfg, wsp, ws_bytes, n > 1 ? select_ws_bytes(dt, n) : 0));
    int rc = QMSORT_OK;
    if (n > 1) {
        rc = run_transform(dt, cmp, d, n, 0, st, f.led);
        unsigned char* w = static_cast<unsigned char*>(f.ws);
        const size_t nn = std::max<size_t>(n, 2);
        if (rc == QMSORT_OK) {
            switch (core_dtype(dt)) {
                case QMSORT_DT_U32:
                    rc = select_core<uint32_t>(static_cast<uint32_t*>(d), n, k - 1, cfg, w, make_layout<uint32_t>(nn), st, f.led);
                    break;
                case QMSORT_DT_U64:
                    rc = select_core<uint64_t>(static_cast<uint64_t*>(d), n, k - 1, cfg, w, make_layout<uint64_t>(nn), st, f.led);
                    break;
                case QMSORT_DT_REC32:
                    rc = select_core<Rec32>(static_cast<Rec32*>(d), n, k - 1, cfg, w, make_layout<Rec32>(nn), st, f.led);
                    break;
            }
        }
        if (rc == QMSORT_OK) rc = run_transform(dt, cmp, d, n, 1, st, f.led);
    }
    rc = f.end(rc, m);
    if (rc == QMSORT_OK && pos) *pos = k - 1;
    return rc;
}

// Per-thread cached device arena (grow-only) and stream for the host-array
// entry points.
struct HostArena {
    void* buf = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;
    ~HostArena() {
        if (buf) cudaFree(buf);
        if (st) cudaStreamDestroy(st);
    }
};
// Process-wide state of the batch entry point (one batch at a time, under
// g_batch_mu): a ring of device arenas with their compute streams, one stream
// per copy direction and the events that order them.
constexpr int kBatchArenas = 3;
static std::mutex g_batch_mu;
struct BatchPipe {
    HostArena ar[kBatchArenas];
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t h2d_done[kBatchArenas] = {}, sort_done[kBatchArenas] = {}, d2h_done[kBatchArenas] = {};
    int init(size_t need) {
        if (!h2d) QCK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        if (!d2h) QCK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        for (int a = 0; a < kBatchArenas; ++a) {
            if (!ar[a].st) QCK(cudaStreamCreateWithFlags(&ar[a].st, cudaStreamNonBlocking));
            if (ar[a].bytes < need) {
                if (ar[a].buf) QCK(cudaFree(ar[a].buf));
                ar[a].buf = nullptr;
                ar[a].bytes = 0;
                QCK(cudaMalloc(&ar[a].buf, need));
                ar[a].bytes = need;
            }
            for (cudaEvent_t* e : {&h2d_done[a], &sort_done[a], &d2h_done[a]})
                if (!*e) QCK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        return QMSORT_OK;
    }
};
// One batch pipe per device (the streams, arenas and events of a device
// cannot serve another); created on first use, under g_batch_mu.
static std::map<int, BatchPipe>& batch_pipes() {
    static std::map<int, BatchPipe>* m = new std::map<int, BatchPipe>();  // never destroyed: outlives the CUDA context teardown order
    return *m;
}
// The calling thread's arena on the current device.
static int host_arena(size_t need, unsigned char** base, cudaStream_t* st) {
    static thread_local std::map<int, HostArena> tl;
    HostArena& ar = tl[current_device()];
    if (!ar.st) QCK(cudaStreamCreateWithFlags(&ar.st, cudaStreamNonBlocking));
    if (ar.bytes < need) {
        if (ar.buf) QCK(cudaFree(ar.buf));
        ar.buf = nullptr;
        ar.bytes = 0;
        QCK(cudaMalloc(&ar.buf, need));
        ar.bytes = need;
    }
    *base = static_cast<unsigned char*>(ar.buf);
    *st = ar.st;
    return QMSORT_OK;
}

// Host-array sort through the calling thread's arena: H2D, sort, D2H.
static int sort_host_one(int dtype, int cmp, void* h_data, size_t n, const qmsort_gpu_config* cfg,
                         qmsort_gpu_metrics* metrics) {
    QTRY(validate(dtype, cmp, n, h_data));
    if (n <= 1) {
        if (metrics) std::memset(metrics, 0, sizeof(*metrics));
        return QMSORT_OK;
    }
    const size_t data_bytes = align_up(n * dtype_size(dtype), 256);
    const size_t need = data_bytes + ws_bytes_for(dtype, n, cfg);
    unsigned char* base = nullptr;
    cudaStream_t st = nullptr;
    QTRY(host_arena(need, &base, &st));
    QCK(cudaMemcpyAsync(base, h_data, n * dtype_size(dtype), cudaMemcpyHostToDevice, st));
    int rc = sort_device(dtype, cmp, base, n, cfg, base + data_bytes, need - data_bytes, metrics, st);
    if (rc != QMSORT_OK) return rc;
    QCK(cudaMemcpyAsync(h_data, base, n * dtype_size(dtype), cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    return QMSORT_OK;
}

#include "shard.cuh"

}  // namespace qmsort_b200

using namespace qmsort_b200;

extern "C" {

void qmsort_gpu_config_init(qmsort_gpu_config* c, int variant) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    // SortConfig defaults (sort.hpp:25-34, merge.hpp:26-31)
    c->variant = 0;
    c->pivot = 0;
    c->base_case_kind = 1;
    c->base_case_size_threshold = 10;
    c->base_case_use_levels = 0;
    c->beta = 0.5;
    c->delta = 1.0 / 16.0;
    c->side = 1;
    c->three_way = 0;
    c->block = 128;
    c->algorithm = 0;
    c->seed = 42;
    c->max_levels = 8;
    c->profile = 0;
    switch (variant) {
        case 1:  // qmqs (sort.hpp:41-48)
            c->variant = 1;
            c->base_case_kind = 2;
            c->base_case_size_threshold = 16;
            c->base_case_use_levels = 1;
            break;
        case 2:  // momqms (sort.hpp:52-57)
            c->variant = 2;
            c->pivot = 2;
            break;
        case 3:  // hqms (sort.hpp:61-66)
            c->variant = 3;
            c->pivot = 3;
            break;
        default: break;
    }
}

size_t qmsort_gpu_dtype_size(int dtype) { return dtype_size(dtype); }

int qmsort_gpu_core_dtype(int dtype) { return core_dtype(dtype); }

size_t qmsort_gpu_workspace_bytes(int dtype, size_t n, const qmsort_gpu_config* cfg) {
    if (dtype_size(dtype) == 0) return 0;
    return ws_bytes_for(dtype, n, cfg);
}

int qmsort_gpu_sort(int dtype, int cmp, void* d_data, size_t n, const qmsort_gpu_config* cfg,
                    void* d_ws, size_t ws_bytes, qmsort_gpu_metrics* metrics, void* stream) {
    return sort_device(dtype, cmp, d_data, n, cfg, d_ws, ws_bytes, metrics,
                       static_cast<cudaStream_t>(stream));
}

int qmsort_gpu_sort_host(int dtype, int cmp, void* h_data, size_t n, const qmsort_gpu_config* cfg,
                         qmsort_gpu_metrics* metrics) {
    return sort_host_one(dtype, cmp, h_data, n, cfg, metrics);
}

int qmsort_gpu_sort_host_batch(int dtype, int cmp, void* const* h_arrays, const size_t* ns,
                               size_t count, const qmsort_gpu_config* cfg,
                               qmsort_gpu_metrics* metrics) {
    if (count > 0 && (h_arrays == nullptr || ns == nullptr))
        return fail(QMSORT_EINVAL, "null array list");
    for (size_t i = 0; i < count; ++i) QTRY(validate(dtype, cmp, ns[i], h_arrays[i]));
    if (metrics) std::memset(metrics, 0, sizeof(*metrics));
    std::vector<size_t> todo;  // arrays with something to sort
    size_t need = 0;
    for (size_t i = 0; i < count; ++i) {
        if (ns[i] <= 1) continue;
        todo.push_back(i);
        need = std::max(need, align_up(ns[i] * dtype_size(dtype), 256) + ws_bytes_for(dtype, ns[i], cfg));
    }
    if (todo.empty()) return QMSORT_OK;
    std::lock_guard<std::mutex> batch_lock(g_batch_mu);
    // One host thread, three device arenas in a ring, one stream per copy
    // direction: the host-to-device engine streams array j+1 while array j
    // sorts (its compute stream waits on an event) and array j-1 returns on
    // the device-to-host engine.  Array j+1 reuses the arena of array j-2 once
    // that array's copy back has completed (an event, not a host wait).  The
    // host blocks only inside each sort (its control read) and at the end.
    constexpr int A = kBatchArenas;
    BatchPipe& bp = batch_pipes()[current_device()];
    QTRY(bp.init(need));
    const size_t m = todo.size();
    auto bytes_of = [&](size_t j) { return ns[todo[j]] * dtype_size(dtype); };
    auto h2d = [&](size_t j) -> int {
        const int a = (int)(j % A);
        if (j >= (size_t)A) QCK(cudaStreamWaitEvent(bp.h2d, bp.d2h_done[a], 0));
        QCK(cudaMemcpyAsync(bp.ar[a].buf, h_arrays[todo[j]], bytes_of(j), cudaMemcpyHostToDevice, bp.h2d));
        QCK(cudaEventRecord(bp.h2d_done[a], bp.h2d));
        return QMSORT_OK;
    };
    int rc = h2d(0);
    for (size_t j = 0; j < m && rc == QMSORT_OK; ++j) {
        if (j + 1 < m && (rc = h2d(j + 1)) != QMSORT_OK) break;
        const int a = (int)(j % A);
        const size_t n = ns[todo[j]];
        unsigned char* base = static_cast<unsigned char*>(bp.ar[a].buf);
        const size_t data_bytes = align_up(n * dtype_size(dtype), 256);
        QCK(cudaStreamWaitEvent(bp.ar[a].st, bp.h2d_done[a], 0));
        qmsort_gpu_metrics mj;
        rc = sort_device(dtype, cmp, base, n, cfg, base + data_bytes, bp.ar[a].bytes - data_bytes, &mj,
                         bp.ar[a].st);
        if (rc != QMSORT_OK) break;
        QCK(cudaEventRecord(bp.sort_done[a], bp.ar[a].st));
        QCK(cudaStreamWaitEvent(bp.d2h, bp.sort_done[a], 0));
        QCK(cudaMemcpyAsync(h_arrays[todo[j]], base, bytes_of(j), cudaMemcpyDeviceToHost, bp.d2h));
        QCK(cudaEventRecord(bp.d2h_done[a], bp.d2h));
        if (metrics) {
            metrics->elapsed_ns += mj.elapsed_ns;
            metrics->alg_bytes += mj.alg_bytes;
            metrics->kernel_launches += mj.kernel_launches;
            metrics->host_syncs += mj.host_syncs;
            metrics->max_depth = std::max(metrics->max_depth, mj.max_depth);
            metrics->levels = std::max(metrics->levels, mj.levels);
        }
    }
    // drain both copy streams whatever happened (no copy may outlive the call)
    const cudaError_t e1 = cudaStreamSynchronize(bp.h2d);
    const cudaError_t e2 = cudaStreamSynchronize(bp.d2h);
    if (rc != QMSORT_OK) return rc;
    if (e1 != cudaSuccess || e2 != cudaSuccess)
        return fail(QMSORT_ECUDA, std::string("batch copies: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    g_err.clear();
    return QMSORT_OK;
}

size_t qmsort_gpu_elements_workspace_bytes(size_t n, size_t elem_bytes) {
    return elem_layout(n, elem_bytes).total;
}

int qmsort_gpu_sort_elements(int key_dtype, int cmp, void* d_data, size_t n, size_t elem_bytes,
                             size_t key_offset, const qmsort_gpu_config* cfg, void* d_ws,
                             size_t ws_bytes, qmsort_gpu_metrics* metrics, void* stream) {
    return sort_elements_device(key_dtype, cmp, d_data, n, elem_bytes, key_offset, cfg, d_ws,
                                ws_bytes, metrics, static_cast<cudaStream_t>(stream));
}

int qmsort_gpu_sort_elements_host(int key_dtype, int cmp, void* h_data, size_t n,
                                  size_t elem_bytes, size_t key_offset,
                                  const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics) {
    QTRY(validate_elems(key_dtype, cmp, h_data, n, elem_bytes, key_offset));
    if (n <= 1) {
        if (metrics) std::memset(metrics, 0, sizeof(*metrics));
        return QMSORT_OK;
    }
    const size_t data_bytes = align_up(n * elem_bytes, 256);
    const size_t ws = elem_layout(n, elem_bytes).total;
    unsigned char* base = nullptr;
    cudaStream_t st = nullptr;
    QTRY(host_arena(data_bytes + ws, &base, &st));
    QCK(cudaMemcpyAsync(base, h_data, n * elem_bytes, cudaMemcpyHostToDevice, st));
    QTRY(sort_elements_device(key_dtype, cmp, base, n, elem_bytes, key_offset, cfg, base + data_bytes,
                              ws, metrics, st));
    QCK(cudaMemcpyAsync(h_data, base, n * elem_bytes, cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    return QMSORT_OK;
}

size_t qmsort_gpu_select_workspace_bytes(int dtype, size_t n) {
    if (dtype_size(dtype) == 0) return 0;
    return select_ws_bytes(dtype, n);
}

int qmsort_gpu_select_nth(int dtype, int cmp, void* d_data, size_t n, size_t k, size_t* pos,
                          const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes,
                          qmsort_gpu_metrics* metrics, void* stream) {
    return select_device(dtype, cmp, d_data, n, k, pos, cfg, d_ws, ws_bytes, metrics,
                         static_cast<cudaStream_t>(stream));
}

int qmsort_gpu_select_nth_host(int dtype, int cmp, void* h_data, size_t n, size_t k, size_t* pos,
                               const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics) {
    QTRY(validate(dtype, cmp, n, h_data));
    if (k < 1 || k > n) return fail(QMSORT_EINVAL, "k must satisfy 1 <= k <= n (1-based rank)");
    const size_t data_bytes = align_up(n * dtype_size(dtype), 256);
    const size_t ws = select_ws_bytes(dtype, n);
    unsigned char* base = nullptr;
    cudaStream_t st = nullptr;
    QTRY(host_arena(data_bytes + ws, &base, &st));
    QCK(cudaMemcpyAsync(base, h_data, n * dtype_size(dtype), cudaMemcpyHostToDevice, st));
    QTRY(select_device(dtype, cmp, base, n, k, pos, cfg, base + data_bytes, ws, metrics, st));
    QCK(cudaMemcpyAsync(h_data, base, n * dtype_size(dtype), cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    return QMSORT_OK;
}

const char* qmsort_gpu_last_error(void) { return g_err.c_str(); }

int qmsort_gpu_transform(int dtype, int cmp, void* d_data, size_t n, int inverse, void* stream) {
    QTRY(validate(dtype, cmp, n, d_data));
    Ledger led;
    QTRY(run_transform(dtype, cmp, d_data, n, inverse, static_cast<cudaStream_t>(stream), led));
    return QMSORT_OK;
}

int qmsort_gpu_sample(int core, const void* d, size_t n, size_t s, uint64_t seed, void* out,
                      void* stream) {
    QTRY(validate(core, 0, n, d));
    if (core != core_dtype(core)) return fail(QMSORT_EINVAL, "sample expects a core dtype");
    if (n == 0 || s == 0) return QMSORT_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)std::min<size_t>((s + 255) / 256, 1184);
    switch (core) {
        case QMSORT_DT_U32: gather_sample_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)d, n, s, seed, (uint32_t*)out); break;
        case QMSORT_DT_U64: gather_sample_kernel<uint64_t><<<grid, 256, 0, st>>>((const uint64_t*)d, n, s, seed, (uint64_t*)out); break;
        case QMSORT_DT_REC32: gather_sample_kernel<Rec32><<<grid, 256, 0, st>>>((const Rec32*)d, n, s, seed, (Rec32*)out); break;
    }
    QCK(cudaGetLastError());
    return QMSORT_OK;
}

size_t qmsort_gpu_partition_workspace_bytes(int core, size_t n) {
    if (dtype_size(core) == 0) return 0;
    return ws_bytes_for(core, n);
}

static int partition_entry(int core, const void* d_in, size_t n, const void* spl, uint32_t nsplit,
                           void* d_out, uint64_t* d_counts, void* d_ws, size_t ws_bytes,
                           void* stream, int parts, const PeerArgs* peers) {
    QTRY(validate(core, 0, n, d_in));
    if (core != core_dtype(core)) return fail(QMSORT_EINVAL, "partition expects a core dtype");
    if (nsplit > 1023) return fail(QMSORT_EINVAL, "nsplit must be <= 1023");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t need = ws_bytes_for(core, std::max<size_t>(n, 2));
    void* ws = d_ws;
    bool own = false;
    if (!ws) {
        if (parts != 3) return fail(QMSORT_EINVAL, "split partition calls need a caller workspace");
        QCK(cudaMallocAsync(&ws, need, st));
        own = true;
    } else if (ws_bytes < need) {
        return fail(QMSORT_ENOWS, "partition workspace too small");
    }
    Ledger led;
    unsigned char* w = static_cast<unsigned char*>(ws);
    int rc = QMSORT_OK;
    const size_t nn = std::max<size_t>(n, 2);
    switch (core) {
        case QMSORT_DT_U32:
            rc = partition_given<uint32_t>((const uint32_t*)d_in, n, (const uint32_t*)spl, nsplit,
                                           (uint32_t*)d_out, d_counts, w, make_layout<uint32_t>(nn), st,
                                           led, parts, peers);
            break;
        case QMSORT_DT_U64:
            rc = partition_given<uint64_t>((const uint64_t*)d_in, n, (const uint64_t*)spl, nsplit,
                                           (uint64_t*)d_out, d_counts, w, make_layout<uint64_t>(nn), st,
                                           led, parts, peers);
            break;
        case QMSORT_DT_REC32:
            if (nsplit > 255) rc = fail(QMSORT_EINVAL, "rec32 partition supports <= 255 splitters");
            else
                rc = partition_given<Rec32>((const Rec32*)d_in, n, (const Rec32*)spl, nsplit,
                                            (Rec32*)d_out, d_counts, w, make_layout<Rec32>(nn), st,
                                            led, parts, peers);
            break;
    }
    if (own) cudaFreeAsync(ws, st);
    return rc;
}

int qmsort_gpu_partition(int core, const void* d_in, size_t n, const void* spl, uint32_t nsplit,
                         void* d_out, uint64_t* d_counts, void* d_ws, size_t ws_bytes, void* stream) {
    return partition_entry(core, d_in, n, spl, nsplit, d_out, d_counts, d_ws, ws_bytes, stream, 3,
                           nullptr);
}


size_t qmsort_gpu_partition3_workspace_bytes(int dtype, size_t n) {
    if (dtype_size(dtype) == 0) return 0;
    return ws_bytes_for(dtype, std::max<size_t>(n, 2)) + 256;
}

int qmsort_gpu_partition3(int dtype, int cmp, void* d_data, size_t n, const void* h_pivot, uint64_t* h_counts3,
                          const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes, qmsort_gpu_metrics* metrics,
                          void* stream) {
    return partition3_device(dtype, cmp, d_data, n, h_pivot, h_counts3, cfg, d_ws, ws_bytes, metrics,
                             static_cast<cudaStream_t>(stream));
}

int qmsort_gpu_partition3_host(int dtype, int cmp, void* h_data, size_t n, const void* h_pivot,
                               uint64_t* h_counts3, const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics) {
    QTRY(validate(dtype, cmp, n, h_data));
    const size_t data_bytes = align_up(std::max<size_t>(n, 1) * dtype_size(dtype), 256);
    const size_t ws = qmsort_gpu_partition3_workspace_bytes(dtype, n);
    unsigned char* base = nullptr;
    cudaStream_t st = nullptr;
    QTRY(host_arena(data_bytes + ws, &base, &st));
    if (n) QCK(cudaMemcpyAsync(base, h_data, n * dtype_size(dtype), cudaMemcpyHostToDevice, st));
    QTRY(partition3_device(dtype, cmp, base, n, h_pivot, h_counts3, cfg, base + data_bytes, ws, metrics, st));
    if (n) QCK(cudaMemcpyAsync(h_data, base, n * dtype_size(dtype), cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    return QMSORT_OK;
}

// ---- the distributed samplesort (shard.cuh) ----
int qmsort_gpu_sort_sharded(int dtype, int cmp, uint32_t P, const int* devices, const void* const* d_in,
                            const size_t* n_in, void* const* d_out, const size_t* out_cap, size_t* out_n,
                            const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics) {
    return sort_sharded_sp(dtype, cmp, P, devices, d_in, n_in, d_out, out_cap, out_n, cfg, metrics);
}

size_t qmsort_gpu_shard_workspace_bytes(int dtype, size_t n) {
    if (dtype_size(dtype) == 0) return 0;
    return shard_ws_bytes(dtype, n);
}

int qmsort_gpu_shard_sample(int dtype, int cmp, const void* d_in, size_t n, size_t s, uint64_t seed,
                            void* d_out, void* stream) {
    QTRY(validate(dtype, cmp, n, d_in));
    if (s > 0 && n > 0 && !d_out) return fail(QMSORT_EINVAL, "null output");
    return dispatch_sample(dtype, cmp, d_in, n, s, seed, d_out, static_cast<cudaStream_t>(stream));
}

int qmsort_gpu_shard_splitters(int core, const void* h_sorted, size_t m, uint32_t nbuckets, void* h_uniq,
                               uint32_t* h_mult, uint32_t* nuniq) {
    if (!h_sorted || !h_uniq || !h_mult || !nuniq) return fail(QMSORT_EINVAL, "null argument");
    return shard_splitters_host(core, h_sorted, m, nbuckets, h_uniq, h_mult, nuniq);
}

uint32_t qmsort_gpu_shard_subbuckets(int dtype, uint32_t P, uint64_t n_total) {
    if (dtype_size(dtype) == 0 || P < 1 || P > (uint32_t)kMaxPeers) return 0;
    return shard_subbuckets(dtype, P, n_total);
}

int qmsort_gpu_shard_plan_folded(uint32_t P, uint32_t K0, uint32_t nuniq, const uint32_t* mult,
                                 const uint64_t* counts, int32_t* bin_rank, uint64_t* bin_off, uint64_t* out_n,
                                 uint32_t* loc_m, int32_t* loc_uniq, uint64_t* loc_counts) {
    if ((nuniq && !mult) || !counts || !bin_rank || !bin_off || !out_n || !loc_m || !loc_uniq || !loc_counts)
        return fail(QMSORT_EINVAL, "null argument");
    return shard_plan_folded_host(P, K0, nuniq, mult, counts, bin_rank, bin_off, out_n, loc_m, loc_uniq, loc_counts);
}

int qmsort_gpu_shard_finish_presplit(int dtype, int cmp, void* d_out, size_t n, const void* d_local_uniq,
                                     uint32_t local_m, const uint64_t* h_local_counts, const qmsort_gpu_config* cfg,
                                     void* d_ws, size_t ws_bytes, qmsort_gpu_metrics* metrics, void* stream) {
    if (!h_local_counts) return fail(QMSORT_EINVAL, "null counts");
    uint64_t tot = 0;
    for (uint32_t b = 0; b < 2 * local_m + 1; ++b) tot += h_local_counts[b];
    if (tot != n) return fail(QMSORT_EINVAL, "local bin counts must sum to n");
    return sort_presplit_device(dtype, cmp, d_out, n, d_local_uniq, local_m, h_local_counts, cfg, d_ws, ws_bytes,
                                metrics, static_cast<cudaStream_t>(stream));
}

int qmsort_gpu_shard_count(int dtype, int cmp, const void* d_in, size_t n, const void* d_uniq, uint32_t nuniq,
                           int three_way, uint64_t* d_counts, void* d_ws, size_t ws_bytes, void* stream) {
    if (!d_counts || (nuniq && !d_uniq)) return fail(QMSORT_EINVAL, "null argument");
    Ledger led;
    return shard_partition(dtype, cmp, d_in, n, d_uniq, nuniq, d_counts, d_ws, ws_bytes,
                           static_cast<cudaStream_t>(stream), 1, nullptr, led, three_way != 0);
}

int qmsort_gpu_shard_plan(uint32_t P, uint32_t nuniq, const uint32_t* mult, const uint64_t* counts,
                          int32_t* bin_rank, uint64_t* bin_off, uint64_t* recv_n, uint64_t* lo_fill,
                          uint64_t* hi_fill, int32_t* lo_val, int32_t* hi_val) {
    if ((nuniq && !mult) || !counts || !bin_rank || !bin_off || !recv_n || !lo_fill || !hi_fill || !lo_val ||
        !hi_val)
        return fail(QMSORT_EINVAL, "null argument");
    return shard_plan_host(P, nuniq, mult, counts, bin_rank, bin_off, recv_n, lo_fill, hi_fill, lo_val, hi_val);
}

int qmsort_gpu_shard_scatter(int dtype, int cmp, const void* d_in, size_t n, uint32_t nuniq, int three_way,
                             const int32_t* bin_rank, const uint64_t* bin_off, void* const* rank_dest,
                             const uint64_t* recv_n, uint32_t P, int raw, void* d_ws, size_t ws_bytes, void* stream) {
    if (n == 0) return validate(dtype, cmp, n, d_in);
    if (!bin_rank || !bin_off || !rank_dest || !recv_n) return fail(QMSORT_EINVAL, "null argument");
    const ShardRoute rt{bin_rank, bin_off, rank_dest, recv_n, P, raw != 0};
    Ledger led;
    return shard_partition(dtype, cmp, d_in, n, nullptr, nuniq, nullptr, d_ws, ws_bytes,
                           static_cast<cudaStream_t>(stream), 2, &rt, led, three_way != 0);
}

int qmsort_gpu_shard_finish(int dtype, int cmp, const void* d_recv, size_t n_recv, const void* d_uniq,
                            int32_t lo_val, uint64_t lo_fill, int32_t hi_val, uint64_t hi_fill, void* d_out,
                            const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes,
                            qmsort_gpu_metrics* metrics, void* stream) {
    if (n_recv > 0 && !d_recv) return fail(QMSORT_EINVAL, "null receive buffer");
    return shard_finish(dtype, cmp, d_recv, n_recv, d_uniq, lo_val, lo_fill, hi_val, hi_fill, d_out, cfg, d_ws,
                        ws_bytes, metrics, static_cast<cudaStream_t>(stream));
}

// A handle names the whole allocation (e.g. a block of a caching allocator);
// the offset of d_ptr inside it travels with the handle.
int qmsort_gpu_ipc_handle(void* d_ptr, void* handle_out, uint64_t* offset_out) {
    if (!d_ptr || !handle_out || !offset_out) return fail(QMSORT_EINVAL, "null pointer");
    // the driver entry point through cudart: no link-time dependency on libcuda
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range_fn = nullptr;
    if (!range_fn) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        QCK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(QMSORT_ECUDA, "cuMemGetAddressRange unavailable");
        range_fn = reinterpret_cast<RangeFn>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
        return fail(QMSORT_ECUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    QCK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == QMSORT_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return QMSORT_OK;
}

int qmsort_gpu_ipc_open(const void* handle, uint64_t offset, void** d_ptr, void** d_base) {
    if (!handle || !d_ptr || !d_base) return fail(QMSORT_EINVAL, "null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    QCK(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
    *d_ptr = static_cast<unsigned char*>(*d_base) + offset;
    return QMSORT_OK;
}

int qmsort_gpu_ipc_close(void* d_base) {
    if (!d_base) return fail(QMSORT_EINVAL, "null pointer");
    QCK(cudaIpcCloseMemHandle(d_base));
    return QMSORT_OK;
}

int qmsort_gpu_generate(int kind, void* d_out, size_t n, uint64_t seed, uint64_t start,
                        uint64_t total, void* stream) {
    if (n == 0) return QMSORT_OK;
    if (!d_out) return fail(QMSORT_EINVAL, "null output");
    if (!(kind == 0 || kind == 1 || kind == 2 || (kind >= 10 && kind <= 14)))
        return fail(QMSORT_EINVAL, "unknown generator kind");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    generate_kernel<<<grid, 256, 0, st>>>(d_out, n, seed, start, kind, total ? total : n);
    QCK(cudaGetLastError());
    return QMSORT_OK;
}

int qmsort_gpu_check(int dtype, int cmp, const void* d, size_t n, int check_order, uint64_t* out3,
                     void* stream) {
    QTRY(validate(dtype, cmp, n, d));
    if (!out3) return fail(QMSORT_EINVAL, "null out3");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long* res = nullptr;
    QCK(cudaMallocAsync(&res, 3 * sizeof(unsigned long long), st));
    QCK(cudaMemsetAsync(res, 0, 3 * sizeof(unsigned long long), st));
    const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 8));
    if (n > 0) {
#define QCHK(T)                                                                             \
    (cmp ? check_kernel<T, true><<<grid, 256, 0, st>>>((const T*)d, n, res, check_order)    \
         : check_kernel<T, false><<<grid, 256, 0, st>>>((const T*)d, n, res, check_order))
        switch (dtype) {
            case QMSORT_DT_I32: QCHK(int32_t); break;
            case QMSORT_DT_U32: QCHK(uint32_t); break;
            case QMSORT_DT_U64: QCHK(uint64_t); break;
            case QMSORT_DT_F64: QCHK(double); break;
            case QMSORT_DT_I64: QCHK(int64_t); break;
            case QMSORT_DT_REC32: QCHK(Rec32); break;
        }
#undef QCHK
        QCK(cudaGetLastError());
    }
    unsigned long long h[3];
    QCK(cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, st));
    QCK(cudaFreeAsync(res, st));
    QCK(cudaStreamSynchronize(st));
    out3[0] = h[0];
    out3[1] = h[1];
    out3[2] = h[2];
    return QMSORT_OK;
}

const char* qmsort_gpu_version(void) { return "qmsort-b200 0.1 sm_100a"; }

}  // extern "C"

extern "C" void qmsort_gpu_abi_sizes(size_t* config_bytes, size_t* metrics_bytes) {
    if (config_bytes) *config_bytes = sizeof(qmsort_gpu_config);
    if (metrics_bytes) *metrics_bytes = sizeof(qmsort_gpu_metrics);
}
