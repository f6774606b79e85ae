// samplesort.cuh -- K1..K4 + K8: sampled multi-splitter partition.
//
// Generalises the reference's pivot step (median_of_3_index,
// partition.hpp:21-30; median_of_sqrt_pivot, partition.hpp:235-251) and its
// partition (block_partition, partition.hpp:37-164) from one pivot / two sides
// to K-1 splitters / K (or 2K-1 with equality buckets) buckets per pass:
//   * sample_kernel   (K1) -- per segment, draws a seeded sample, sorts it on
//                             chip (blocksort.cuh) and picks K-1 evenly spaced
//                             splitters: the Median-of-sqrt(n) sample
//                             generalised to K-1 quantiles.  Duplicate
//                             splitters switch the segment to three-way
//                             classification (K8, the "equal block takes no
//                             further part" rule of three_way_partition,
//                             partition.hpp:194-195).
//   * count_kernel    (K2) -- classification of U keys per thread in lock
//                             step, shared-memory bucket histogram per chunk.
//   * colsum_kernel +
//     plan_kernel     (K3) -- per (segment, bucket): exclusive prefix over the
//                             chunks; per segment: bucket totals, starts and
//                             the child work (next-level segments, block-sort
//                             tasks, equal-bucket fills).
//   * scatter_kernel  (K4) -- re-classifies each tile, groups it by bucket in
//                             shared memory and writes every bucket run with
//                             coalesced stores to its final offset.
// Offsets are deterministic (no global atomics on the data path): chunk c of
// a segment writes bucket b at  start[b] + sum_{c' < c} hist[b][c'].
//
// Classification.  The bucket of key x is j = #{splitters < x} -- the same
// comparisons against the same splitters for every key type.  For integer
// keys the search is shortened by a bucket lookup table: the segment's key
// range [lo, hi] (known from the parent's splitters) is cut into 2^lutbits
// cells; cell c stores the bucket range [j_lo, j_hi] its keys can fall in, and
// only keys of cells that straddle a splitter finish with a binary search over
// sorted[j_lo..j_hi).  Records (rec32) walk an Eytzinger search tree.
#pragma once
#include <cstddef>
#include <type_traits>

#include "blocksort.cuh"
#include "common.cuh"

namespace qmsort_b200 {

constexpr int kNumClasses = 9;  // block-sort size classes (Tune<K>::CLS_T)
constexpr int kLutMaxBits = 12;
#ifndef QMSORT_EVEN_SPLITTERS
#define QMSORT_EVEN_SPLITTERS 1
#endif
#ifndef QMSORT_RUN_TALLY
#define QMSORT_RUN_TALLY 1
#endif
#ifndef QMSORT_STAGE_KEY8
#define QMSORT_STAGE_KEY8 1
#endif
#ifndef QMSORT_PREFETCH8
#define QMSORT_PREFETCH8 1
#endif
constexpr int kLutPerSplitter = 16;  // LUT words reserved per splitter slot

struct SegDesc {
    uint64_t off;          // absolute element offset of the segment
    uint64_t len;          // number of keys
    uint64_t lo, hi;       // integer keys: every key of the segment is in [lo, hi]
    uint32_t chunk_begin;  // first chunk in the level's chunk table
    uint32_t nchunks;
    uint32_t logk;         // K = 1 << logk buckets
    uint32_t m;            // unique splitters (set by sample_kernel)
    uint32_t eq;           // three-way classification on: 2K bins, bin = 2j + (key == s_j)
    uint32_t sp;           // base index of this segment's splitter storage
    uint32_t hist_base;    // histogram block: bin b, chunk i at hist_base + b*(nchunks+1) + i;
                           // entry i = nchunks holds the bucket total, then its start
    uint32_t shift;        // LUT cell = (key - lo) >> shift
    uint32_t lutbits;      // 2^lutbits LUT cells
    uint32_t sampler;      // kSampleRandom or kSampleTriples (worst-case policy, f1)
    // Even splitters (integer keys, set by sample_kernel when the sample says
    // the keys are spread evenly over [lo, hi]): splitter j is the largest key
    // with ((key - lo) >> shift) * scale >> 32 <= j, so a key's bucket is that
    // product -- no table, no splitter read.
    uint32_t arith;
    uint32_t scale;
};

// K1 sampling rules.  kSampleRandom: seeded random
// positions (median_of_3 / median_of_sqrt_n presets).  kSampleTriples: the
// median of three adjacent keys at evenly strided positions, no seed -- the
// sample analogue of triple_median_pivot (selection.hpp:219-229), used at
// every level by mom_of_thirds and, under hybrid, for a bucket that came out
// outside the delta band (pivot_outside_band, sort.hpp:114-118).
// kSampleSqrt: median_of_sqrt_n (median_of_sqrt_pivot, partition.hpp:235-251)
// -- s = 2 floor(sqrt(len) / 2) + 1 keys at the strided positions i * floor(len / s),
// at least 1024 so that the K-1 quantiles stay usable, at most one block sort
// (a larger level-0 sample is sorted beforehand by the host path, see
// samplesort()).
enum : uint32_t { kSampleRandom = 0, kSampleTriples = 1, kSampleSqrt = 2 };

__host__ __device__ inline uint64_t isqrt_u64(uint64_t x) {
    uint64_t r = 0;
    for (int b = 31; b >= 0; --b) {
        const uint64_t t = r | (1ull << b);
        if (t * t <= x) r = t;
    }
    return r;
}
// The reference's Median-of-sqrt(n) sample size (partition.hpp:240-241).
__host__ __device__ inline uint64_t sqrt_sample_size(uint64_t len) { return 2 * (isqrt_u64(len) / 2) + 1; }

struct ChunkDesc {
    uint32_t seg;
    uint32_t pad;
    uint64_t begin;  // absolute element range [begin, end)
    uint64_t end;
};

struct SortTask {  // one bucket for the block sorter
    uint64_t off;
    uint32_t len;
    uint32_t in_a;  // the bucket was scattered into A (else into B); it is sorted into A
    // integer keys: every key of the bucket lies in [klo, khi] (the splitters
    // around it within the parent segment's range) -- the table sort's span
    uint64_t klo, khi;
};

constexpr uint64_t kFillWarp = 4096;  // fills up to this many keys get a warp each
struct FillTask {  // equal-key bucket: every key equals the segment's splitter
    uint64_t off;
    uint64_t len;
    alignas(16) unsigned char value[32];  // that key (sizeof(K) bytes)
};

struct LevelCounters {
    uint32_t nsegs;
    uint32_t nchunks;
    uint32_t nsplit;  // splitter storage used
    uint32_t nhist;   // histogram words used
    uint32_t nfill;      // equal-key fills of <= kFillWarp keys, from the front of the list
    uint32_t nfill_big;  // larger fills, from the back
    uint32_t ntasks[kNumClasses];
    uint32_t overflow;  // capacity exceeded somewhere (host reports an error)
    uint32_t work_count, work_scatter;  // dynamic chunk dispensers of this level's kernels
    uint32_t resplits;  // hybrid: children re-sampled with triple medians (f1)
    uint32_t max_logk;  // largest log2 K among this level's segments
    uint32_t max_nchunks;  // most chunks of one of this level's segments
    unsigned long long nkeys;      // keys in this level's segments (pass ledger)
    unsigned long long task_keys;  // keys handed to the block sorter
    unsigned long long fill_keys;  // keys written by equal-bucket fills
    unsigned long long sample_keys;  // keys the level's sample kernel drew (all segments)
};

// K4 staging records carry the bin (the write-out adds the bin's destination
// shift) instead of the destination, with the bins' tile starts and shifts in
// two 4-byte arrays: the staging slot costs a 4-byte instead of an 8-byte
// random shared-memory read, and the write-out's shift reads hit runs of one
// bin (measured on C2: scatter 1960 -> 1895 us, 60.1 -> 61.1 Gkeys/s).
#ifndef QMSORT_SCATTER_BINREC
#define QMSORT_SCATTER_BINREC 1
#endif

// A level whose work lists overflowed (emit_segment / plan_kernel set
// `overflow` after bumping the counts) has counts that cover unwritten
// descriptors: every consumer kernel of that level exits at once and the
// host reports QMSORT_EINTERNAL at its control read.  `field` points at a
// member of the level's LevelCounters (null: a single caller-built segment).
#define QMSORT_LEVEL_OVERFLOWED(field, member)                                                       \
    ((field) != nullptr &&                                                                           \
     reinterpret_cast<const volatile LevelCounters*>(reinterpret_cast<const char*>(field) -          \
                                                     offsetof(LevelCounters, member))->overflow != 0)

static_assert(offsetof(LevelCounters, nsegs) == 0, "sample_kernel finds its LevelCounters from &nsegs");

// Median-of-sqrt(n) at level 0 when s exceeds one block sort: out[i] =
// f(src[i * stride]), sorted afterwards by the host path.
template <class K>
__global__ void gather_strided_kernel(const K* __restrict__ src, uint64_t len, uint64_t s, uint64_t stride,
                                      K* __restrict__ out, Xf xf) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = xf_fwd(src[min(i * stride, len - 1)], xf);
}

struct LevelBufs {  // one partition level's work description (device pointers)
    SegDesc* segs;
    ChunkDesc* chunks;
    LevelCounters* cnt;
    uint32_t seg_cap, chunk_cap, split_cap, hist_cap;
};

struct PlanParams {
    uint64_t chunk_elems;   // chunk granularity (multiple of the tile)
    uint32_t cap;           // largest bucket the block sorter takes
    uint32_t target;        // desired bucket size when choosing K
    uint32_t last_target;   // ... at the last level (Tune<K>::last_target)
    uint32_t xf_fix;        // fused transform: singletons / equal buckets in A still get a writer
    uint32_t log_kmax;      // largest K = 1 << log_kmax
    uint32_t class_cap[kNumClasses];
    uint32_t task_cap, fill_cap;
    int dst_is_a;           // this level's scatter writes the caller's buffer
    uint32_t pivot;         // PivotStrategy (sort.hpp:19): 2 mom_of_thirds, 3 hybrid
    uint32_t delta_q16;     // SortConfig::delta in 1/65536 (hybrid skew band)
    uint32_t table_class;   // task list of the table sort (tablesort.cuh); >= kNumClasses: off
    uint32_t cell_class;    // task list of the wide-span table sort (CellSort); >= kNumClasses: off
    uint32_t cell_cap, cell_bits;  // CellSort<K>: keys per bucket, log2 of its cells
    uint32_t cell_big_class, cell_big_cap, cell_big_bits;  // CellSort<K, true> for the buckets beyond cell_cap
};

// Table-sort eligibility of a bucket of len keys within [klo, khi]
// (TableSort::eligible, tablesort.cuh -- restated here for the plan).
__host__ __device__ inline bool table_sort_eligible(uint32_t len, uint64_t klo, uint64_t khi) {
    if (khi < klo || len > 4096u || len < 256u) return false;
    const uint64_t span = khi - klo;
    return span < 65536ull && span >= 4ull * len && span <= 64ull * len;
}

// Cell width of a bucket of len keys spanning span + 1 values: the smallest
// shift that leaves at most min(2^max_bits, 16 len rounded up to a power of
// two) cells.
__host__ __device__ inline uint32_t cell_shift(uint32_t len, uint64_t span, uint32_t max_bits) {
#ifdef __CUDA_ARCH__
    const uint32_t bits = 64u - (uint32_t)__clzll((long long)span);  // bit length of span
    const uint32_t tb = min(max_bits, 32u - (uint32_t)__clz((int)(16u * len - 1u)));
#else
    uint32_t bits = 0;
    while (bits < 64 && (span >> bits)) ++bits;
    uint32_t tb = 0;
    while (tb < max_bits && (1u << tb) < 16u * len) ++tb;
#endif
    return bits > tb ? bits - tb : 0u;
}
// Buckets the plan sends to the cell sort (CellSort<K>: cap keys, 2^max_bits
// cells): at least 4 cells per key (else most cells hold several keys).
__host__ __device__ inline bool cell_sort_eligible(uint32_t len, uint64_t klo, uint64_t khi, uint32_t cap,
                                                   uint32_t max_bits) {
    if (khi < klo || len > cap || len < 256u) return false;
    const uint64_t span = khi - klo;
    return (span >> cell_shift(len, span, max_bits)) >= 4ull * len;
}

__host__ __device__ inline uint32_t ceil_log2_u64(uint64_t x) {
    uint32_t r = 0;
    while ((1ull << r) < x) ++r;
    return r;
}

// Number of buckets for a segment of len keys.  A segment whose buckets would
// average at most 3/4 of the block sorter's cap with the largest K is split
// once (K = len / last_target rounded up to a power of two, at most K_max): the
// last level then never leaves a sliver for a further level.  Larger segments
// spread log2(len / target) bits evenly over the fewest levels of <= K_max,
// where the last level may leave buckets of up to twice the target when the
// cap allows it (one "slack" bit).
__host__ __device__ inline uint32_t choose_logk(uint64_t len, uint32_t target, uint32_t last_target,
                                                uint32_t log_kmax, uint32_t cap) {
    const uint64_t ratio = (len + target - 1) / target;
    uint32_t r = ceil_log2_u64(ratio);
    if (r < 1) r = 1;
    if (len <= ((uint64_t)cap * 3 / 4) << log_kmax) {
        uint32_t rl = ceil_log2_u64((len + last_target - 1) / last_target);
        if (rl < 1) rl = 1;
        return rl < log_kmax ? rl : log_kmax;
    }
    const uint32_t slack = cap / target >= 4 ? 1u : 0u;
    const uint32_t rs = r > slack ? r - slack : 1;
    const uint32_t levels = (rs + log_kmax - 1) / log_kmax;
    uint32_t k = (r + levels - 1) / levels;
    if (k < 1) k = 1;
    if (k > log_kmax) k = log_kmax;
    return k;
}

// Append a segment (and, unless write_chunks is false, its chunk table) to
// the next level.  Called by one thread.  Returns false on capacity overflow.
__device__ inline bool emit_segment(const LevelBufs& nb, uint64_t off, uint64_t len, uint64_t lo,
                                    uint64_t hi, const PlanParams& p, uint32_t sampler,
                                    bool write_chunks = true) {
    const uint32_t logk = choose_logk(len, p.target, p.last_target, p.log_kmax, p.cap);
    const uint32_t nch = (uint32_t)((len + p.chunk_elems - 1) / p.chunk_elems);
    const uint32_t hwords = (nch + 1) * (2u << logk);
    const uint32_t s = atomicAdd(&nb.cnt->nsegs, 1u);
    atomicMax(&nb.cnt->max_logk, logk);
    atomicMax(&nb.cnt->max_nchunks, nch);
    const uint32_t sp = atomicAdd(&nb.cnt->nsplit, 1u << logk);
    const uint32_t c0 = atomicAdd(&nb.cnt->nchunks, nch);
    const uint32_t hb = atomicAdd(&nb.cnt->nhist, hwords);
    if (s >= nb.seg_cap || sp + (1u << logk) > nb.split_cap || c0 + nch > nb.chunk_cap ||
        hb + hwords > nb.hist_cap) {
        atomicExch(&nb.cnt->overflow, 1u);
        return false;
    }
    SegDesc d;
    d.off = off;
    d.len = len;
    d.lo = lo;
    d.hi = hi;
    d.chunk_begin = c0;
    d.nchunks = nch;
    d.logk = logk;
    d.m = 0;
    d.eq = 0;
    d.sp = sp;
    d.hist_base = hb;
    d.lutbits = min(logk + 4, (uint32_t)kLutMaxBits);
    const uint64_t span = hi - lo;  // keys in [lo, hi]
    uint32_t bl = 0;
    while (bl < 64 && (span >> bl) != 0) ++bl;  // bit length of span
    d.shift = bl > d.lutbits ? bl - d.lutbits : 0;
    d.sampler = sampler;
    d.arith = d.scale = 0;
    nb.segs[s] = d;
    atomicAdd(&nb.cnt->nkeys, (unsigned long long)len);
    for (uint32_t i = 0; write_chunks && i < nch; ++i) {
        ChunkDesc c;
        c.seg = s;
        c.pad = 0;
        c.begin = off + (uint64_t)i * p.chunk_elems;
        c.end = min(off + len, c.begin + p.chunk_elems);
        nb.chunks[c0 + i] = c;
    }
    return true;
}

// Level 0: one segment covering [0, n); its (many) chunks are written by all
// threads of the grid.
__global__ void init_level_kernel(LevelBufs nb, uint64_t n, uint64_t key_max, PlanParams p) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        emit_segment(nb, 0, n, 0, key_max, p,
                     p.pivot == 2 ? kSampleTriples : p.pivot == 1 ? kSampleSqrt : kSampleRandom, false);
    const uint32_t nch = (uint32_t)((n + p.chunk_elems - 1) / p.chunk_elems);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nch && i < nb.chunk_cap;
         i += gridDim.x * blockDim.x) {
        ChunkDesc c;
        c.seg = 0;
        c.pad = 0;
        c.begin = (uint64_t)i * p.chunk_elems;
        c.end = min(n, c.begin + p.chunk_elems);
        nb.chunks[i] = c;
    }
}

// ---------------------------------------------------------------------------
// Classification
// ---------------------------------------------------------------------------
// Shared-memory view of one segment's classifier.
template <class K, int LOG_KMAX>
struct ClassifierSmem {
    static constexpr int KMAX = 1 << LOG_KMAX;
    K sorted[KMAX];                                           // unique splitters
    K tree[KeyTraits<K>::kLut ? 1 : KMAX];                    // rec32: Eytzinger tree
    uint64_t ptree[KeyTraits<K>::kLut ? 1 : KMAX];            // rec32: the tree's 64-bit prefixes
    uint32_t lut[KeyTraits<K>::kLut ? (1 << kLutMaxBits) : 1];  // integers: j_lo | (j_hi-j_lo) << 16
};

// Records: a 64-bit prefix that is monotone (non-decreasing) in the
// lexicographic order -- the top 64 bits of (w0 - base, w1), clamped to
// [0, 2^64) for w0 outside [base, base + 2^(64-psh)).  base and psh come from
// the segment's sample (SegDesc lo / shift); any values keep the prefix
// monotone, they only decide how often two prefixes tie.  p(a) < p(b) implies
// a < b, so a tree step needs the full record compare only on equal prefixes.
__device__ __forceinline__ uint64_t rec_prefix(const Rec32& r, uint64_t base, uint32_t psh) {
    if (r.w[0] < base) return 0;
    const uint64_t d0 = r.w[0] - base;
    if (psh == 0) return d0;
    if (psh >= 64) return d0 ? ~0ull : r.w[1];
    if (d0 >> (64 - psh)) return ~0ull;
    return (d0 << psh) | (r.w[1] >> (64 - psh));
}

// The largest record whose prefix (rec_prefix with base, psh) is p: the upper
// end of an even range of record prefixes as a splitter record.
__device__ __forceinline__ Rec32 rec_from_prefix(uint64_t p, uint64_t base, uint32_t psh) {
    Rec32 r;
    if (psh == 0) {
        r.w[0] = base + p;
        r.w[1] = ~0ull;
    } else if (psh >= 64) {
        r.w[0] = base;
        r.w[1] = p;
    } else {
        r.w[0] = base + (p >> psh);
        r.w[1] = (p << (64 - psh)) | ((1ull << (64 - psh)) - 1);
    }
    r.w[2] = r.w[3] = ~0ull;
    return r;
}

// Bucket of a key in an even-splitter segment (SegDesc::arith): integers
// ((key - lo) >> shift) * scale >> 32; records the same product of their
// prefix's distance from the sample's smallest prefix (hi) >> lutbits.
template <class K>
__device__ __forceinline__ uint32_t even_bucket(const K& key, const SegDesc& d) {
    using KT = KeyTraits<K>;
    if constexpr (KT::kLut) {
        using UI = typename KT::UInt;
        const UI rel = KT::bits(key) - (UI)d.lo;
        const UI r = rel >> d.shift;  // < 2^32 for keys within [lo, hi]; a tile's padding keys saturate
        const uint32_t r32 = sizeof(UI) == 8 && r > (UI)0xFFFFFFFFu ? 0xFFFFFFFFu : (uint32_t)r;
        return min(__umulhi(r32, d.scale), d.m);
    } else {
        // records outside the sampled prefix range clamp into the end
        // buckets: below it rel = 0; above it the 32-bit range index
        // saturates (a truncated index would land in an arbitrary bucket)
        const uint64_t pk = rec_prefix(key, d.lo, d.shift);
        const uint64_t rel = pk > d.hi ? pk - d.hi : 0;
        const uint64_t r = rel >> d.lutbits;
        return min(__umulhi(r > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)r, d.scale), d.m);
    }
}

template <class K, int LOG_KMAX, int T>
__device__ __forceinline__ void load_classifier(ClassifierSmem<K, LOG_KMAX>& c, const SegDesc& d,
                                                const K* __restrict__ tree_store,
                                                const K* __restrict__ sorted_store,
                                                const uint32_t* __restrict__ lut_store) {
    const uint32_t K_ = 1u << d.logk;
    for (uint32_t i = threadIdx.x; i < K_; i += T) c.sorted[i] = sorted_store[d.sp + i];
    if constexpr (KeyTraits<K>::kLut) {
        const uint32_t nc = 1u << d.lutbits;
        const uint32_t* src = lut_store + (size_t)d.sp * kLutPerSplitter;
        if (!d.arith)  // even splitters need no table
            for (uint32_t i = threadIdx.x; i < nc; i += T) c.lut[i] = src[i];
    } else if (!d.arith) {
        for (uint32_t i = threadIdx.x; i < K_; i += T) {
            const K t = tree_store[d.sp + i];
            c.tree[i] = t;
            if constexpr (std::is_same<K, Rec32>::value) c.ptree[i] = rec_prefix(t, d.lo, d.shift);
        }
    }
}

// Warp-aggregated shared-memory increment for segments with few bins (the
// sharded exchange's P buckets): lanes holding the same bin are counted by
// one atomic of their leader (measured at P = 1: K4 1.67 -> 0.89 ms; K2's
// plain increments stay faster, the match costs more than the contention).  valid = false: the
// lane takes part in the vote but adds nothing.  Returns the lane's rank
// among the bin's keys (the pre-increment count plus its peers below it).
__device__ __forceinline__ uint32_t warp_agg_inc(uint32_t* counters, uint32_t b, bool valid) {
    const uint32_t key = valid ? b : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader && valid) base = atomicAdd(&counters[b], (uint32_t)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
}

// Bins of U keys.  bin = j, or 2j + (key == splitter j) with equality buckets.
template <class K, int LOG_KMAX, int U>
__device__ __forceinline__ void classify_keys(const K (&key)[U],
                                              const ClassifierSmem<K, LOG_KMAX>& c,
                                              const SegDesc& d, uint32_t (&bin)[U]) {
    using KT = KeyTraits<K>;
    uint32_t j[U];
    if constexpr (KT::kLut) {
        using UI = typename KT::UInt;
        const UI lo = (UI)d.lo;
        const uint32_t shift = d.shift;
        const UI cmax = (UI)((1u << d.lutbits) - 1);
        uint32_t wide = 0;  // keys whose cell straddles two or more splitters
        if (d.arith) {  // even splitters: the bucket is a product (uniform per segment)
#pragma unroll
            for (int u = 0; u < U; ++u) j[u] = even_bucket<K>(key[u], d);
        } else
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const UI rel = KT::bits(key[u]) - lo;
            const uint32_t cell = (uint32_t)min((UI)(rel >> shift), cmax);
            const uint32_t e = c.lut[cell];
            const uint32_t cnt = e >> 16;
            // branch-free finish for cells straddling at most one splitter
            const uint32_t j0 = e & 0xFFFFu;
            j[u] = j0 + ((cnt != 0 && KT::lt(c.sorted[j0], key[u])) ? 1u : 0u);
            wide |= (cnt > 1 ? 1u : 0u) << u;
        }
        if (wide) {  // rare: binary search #{sorted[j0 .. j0+cnt) < key}
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!((wide >> u) & 1u)) continue;
                const UI rel = KT::bits(key[u]) - lo;
                const uint32_t e = c.lut[(uint32_t)min((UI)(rel >> shift), cmax)];
                uint32_t jj = e & 0xFFFFu, cnt = e >> 16;
                while (cnt > 0) {
                    const uint32_t half = cnt >> 1;
                    const bool less = KT::lt(c.sorted[jj + half], key[u]);
                    jj = less ? jj + half + 1 : jj;
                    cnt = less ? cnt - half - 1 : half;
                }
                j[u] = jj;
            }
        }
    } else if (d.arith) {
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = even_bucket<K>(key[u], d);
    } else {
        // Eytzinger walk on the splitters' prefixes; the full record compare
        // only where a key's prefix equals the node's
        uint32_t t[U];
        uint64_t pk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            t[u] = 1;
            pk[u] = rec_prefix(key[u], d.lo, d.shift);
        }
        for (uint32_t l = 0; l < d.logk; ++l) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t np = c.ptree[t[u]];
                bool right = pk[u] > np;
                if (pk[u] == np) right = KT::lt(c.tree[t[u]], key[u]);
                t[u] = 2 * t[u] + (right ? 1u : 0u);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = t[u] - (1u << d.logk);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) QCHECK(j[u] <= (1u << d.logk), j[u], d.m);
    if (d.eq) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t jj = j[u] < d.m ? j[u] : 0;
            bin[u] = 2 * j[u] + ((j[u] < d.m && KT::eq(key[u], c.sorted[jj])) ? 1u : 0u);
        }
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) bin[u] = j[u];
    }
}

// ---------------------------------------------------------------------------
// K1: per-segment sample + splitter selection.  One CTA per segment.
// ---------------------------------------------------------------------------
template <class K, int T, int ITEMS, bool XF>
__device__ __forceinline__ void sample_segment(uint32_t seg, SegDesc* segs, const K* __restrict__ src,
                                               K* tree_store, K* sorted_store,
                                               uint32_t* lut_store, uint64_t seed,
                                               uint32_t oversample, const Xf& xf,
                                               const K* __restrict__ presorted, uint32_t presorted_n,
                                               unsigned long long* sample_keys, uint32_t even_target,
                                               uint32_t even_span, uint32_t even_over) {
    using BS = BlockSorter<K, T, ITEMS>;
    using P = SmemPad<K>;
    using KT = KeyTraits<K>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s = reinterpret_cast<K*>(smem_raw);
    __shared__ uint32_t flags[1024 + 1];
    __shared__ uint32_t warp_sums[32];

    const SegDesc d = segs[seg];
    const uint32_t K_ = 1u << d.logk;
    // presorted (level 0 of median_of_sqrt_n with s > one block sort): the
    // host sorted the segment's s strided keys beforehand
    const bool pre = presorted != nullptr && seg == 0;
    int S = (int)min((uint32_t)BS::kCap, max(1024u, oversample * K_));
    uint64_t stride = 1;
    if (pre) {
        S = (int)presorted_n;
    } else if (d.sampler == kSampleSqrt) {
        S = (int)min((uint64_t)BS::kCap, max((uint64_t)1024, sqrt_sample_size(d.len)));
        stride = max((uint64_t)1, d.len / (uint64_t)S);
    }
    if (threadIdx.x == 0) atomicAdd(sample_keys, (unsigned long long)S);

    // kSampleRandom: seeded sample with replacement (counter-based SplitMix64
    // of the sample index; uniform position via a 64x64 high multiply).
    // kSampleTriples: median of the three keys at stride position idx.
    // kSampleSqrt: the key at position idx * floor(len / s).
    K k[ITEMS];
    // A cheaper first look (integer keys, random sampler): every thread reads
    // ITEMS consecutive keys at one seeded random position -- 64 bytes in one
    // go instead of ITEMS scattered sectors (level 1 of C2: 8 MB instead of
    // 250 MB of DRAM traffic).  Runs of neighbours are at least as clumped as
    // independent draws, so a run sample that tallies even is accepted; any
    // other is forgotten and the seeded sample below decides.
    auto load_runs = [&]() {
        const uint64_t h = sm_mix(seed + (d.off + 1) * kGamma + (uint64_t)(threadIdx.x + 1) * 0x9E3779B97F4A7C15ull);
        const K* r = src + d.off + __umul64hi(h, d.len - (uint64_t)ITEMS + 1);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) k[i] = XF ? xf_fwd(r[i], xf) : r[i];
    };
    auto load_sample = [&]() {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int idx = (int)threadIdx.x * ITEMS + i;
        if (pre || idx >= S) {
            k[i] = KT::max_key();
        } else if (d.sampler == kSampleSqrt) {
            k[i] = src[d.off + min((uint64_t)idx * stride, d.len - 1)];
            if (XF) k[i] = xf_fwd(k[i], xf);
        } else if (d.sampler == kSampleTriples) {
            const uint64_t p0 = ((uint64_t)idx * d.len) / (uint64_t)S;
            const K* t = src + d.off + min(p0, d.len - 3);
            K a = t[0], b = t[1], c = t[2];
            if (XF) {
                a = xf_fwd(a, xf);
                b = xf_fwd(b, xf);
                c = xf_fwd(c, xf);
            }
            KT::cas(a, b);  // a <= b
            KT::cas(b, c);  // c = max; b = median candidate
            KT::cas(a, b);  // b = median of three
            k[i] = b;
        } else {
            const uint64_t h = sm_mix(seed + (d.off + 1) * kGamma + (uint64_t)(idx + 1) * 0xD1B54A32D192ED03ull);
            k[i] = src[d.off + __umul64hi(h, d.len)];
            if (XF) k[i] = xf_fwd(k[i], xf);
        }
    }
    };
    // Even splitters (integer keys): cut [lo, hi] into equal ranges when the
    // sample says no range would take more than about twice its share --
    // uniform keys then need no lookup table and no splitter compare in K2 /
    // K4 (a bucket is still #{splitters < key}; the splitters are the ranges'
    // upper ends), and the sample is only tallied, not sorted.  Anything else
    // keeps the sample's quantiles.
    __shared__ uint32_t ar_max;
    auto try_even = [&]() -> bool {  // (all threads; true: the segment's splitters are written)
      if constexpr (KT::kLut) {
        const uint64_t span = d.hi - d.lo;
        if (QMSORT_EVEN_SPLITTERS && span >= 2ull * K_ - 1) {
            const uint32_t bl = 64u - (uint32_t)__clzll((long long)span);
            const uint32_t psh = bl > 32 ? bl - 32 : 0;
            const uint32_t span32 = (uint32_t)(span >> psh);
            // ranges: K, or -- a last level -- as few as leave buckets of
            // even_target keys spanning at most even_span values (the table
            // sort's tile and table, tablesort.cuh)
            uint32_t nr = K_;
            // (8-byte keys: only where K ranges would leave buckets over
            // even_over keys, the small cell-sort shape's tile, anyway)
            if (even_target && d.len > (uint64_t)even_over * K_) {
                uint64_t want = (d.len + even_target - 1) / even_target;
                if (even_span) want = max(want, span / even_span + 1);
                nr = (uint32_t)min((uint64_t)K_, max(want, (uint64_t)2));
            }
            const uint32_t scale = (uint32_t)(((uint64_t)nr << 32) / ((uint64_t)span32 + 1));
            const uint32_t m_ar = __umulhi(span32, scale);  // the last key's range = splitters
            for (uint32_t j = threadIdx.x; j <= m_ar; j += T) flags[j] = 0;
            if (threadIdx.x == 0) ar_max = 0;
            __syncthreads();
            auto tally = [&](const K& key) {
                const uint64_t rel = (uint64_t)KT::bits(key) - d.lo;
                atomicAdd(&flags[min(__umulhi((uint32_t)(rel >> psh), scale), m_ar)], 1u);
            };
            if (pre) {
                for (int q = threadIdx.x; q < S; q += T) tally(presorted[q]);
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i)
                    if ((int)threadIdx.x * ITEMS + i < S) tally(k[i]);
            }
            __syncthreads();
            for (uint32_t j = threadIdx.x; j <= m_ar; j += T) atomicMax(&ar_max, flags[j]);
            __syncthreads();
            const bool even = m_ar >= 1 && (uint64_t)ar_max * (m_ar + 1) <= 2ull * (uint64_t)S + 8ull * (m_ar + 1);
            __syncthreads();
            if (even) {
                // upper end of range j (j < m_ar): the largest key with
                // ((key - lo) >> psh) * scale >> 32 <= j
                K* sorted = sorted_store + d.sp;
                for (uint32_t j = threadIdx.x; j < m_ar; j += T) {
                    const uint64_t r = ((((uint64_t)(j + 1)) << 32) - 1) / scale;
                    sorted[j] = (K)(d.lo + ((r + 1) << psh) - 1);
                }
                if (threadIdx.x == 0) {
                    segs[seg].m = m_ar;
                    segs[seg].eq = 0;
                    segs[seg].shift = psh;
                    segs[seg].arith = 1;
                    segs[seg].scale = scale;
                }
                return true;
            }
        }
      }
      return false;
    };
    if constexpr (KT::kLut) {
        if (QMSORT_RUN_TALLY && !pre && d.sampler == kSampleRandom && S == T * ITEMS &&
            d.len >= 16ull * (uint64_t)S) {
            load_runs();
            if (try_even()) return;
            if (threadIdx.x == 0) atomicAdd(sample_keys, (unsigned long long)S);  // a second sample is drawn
            __syncthreads();
        }
    }
    load_sample();
    if (try_even()) return;
    if constexpr (std::is_same<K, Rec32>::value) {
        // Records: the same test on the sample's 64-bit prefixes, over the
        // range [smallest, largest] sampled prefix; the splitters are the
        // largest records of the even prefix ranges, a record's bucket the
        // product of its prefix (records outside the sampled range clamp
        // into the end buckets, which keeps the buckets monotone).
        if (QMSORT_EVEN_SPLITTERS && !pre) {
            __shared__ unsigned long long rmin, rmax;
            __shared__ uint32_t rec_max;
            auto minmax = [&](auto&& f) {
                if (threadIdx.x == 0) {
                    rmin = ~0ull;
                    rmax = 0;
                }
                __syncthreads();
                unsigned long long lo2 = ~0ull, hi2 = 0;
#pragma unroll
                for (int i = 0; i < ITEMS; ++i)
                    if ((int)threadIdx.x * ITEMS + i < S) {
                        const unsigned long long v = f(k[i]);
                        lo2 = min(lo2, v);
                        hi2 = max(hi2, v);
                    }
                if (lo2 <= hi2) {
                    atomicMin(&rmin, lo2);
                    atomicMax(&rmax, hi2);
                }
                __syncthreads();
            };
            minmax([](const Rec32& r) { return (unsigned long long)r.w[0]; });
            const uint64_t base = rmin;
            const uint32_t wsh = rmax > rmin ? (uint32_t)__clzll((long long)(rmax - rmin)) : 64u;
            __syncthreads();
            minmax([&](const Rec32& r) { return (unsigned long long)rec_prefix(r, base, wsh); });
            const uint64_t plo = rmin, span = rmax - rmin;
            __syncthreads();
            if (span >= 2ull * K_ - 1) {
                const uint32_t bl = 64u - (uint32_t)__clzll((long long)span);
                const uint32_t psh2 = bl > 32 ? bl - 32 : 0;
                const uint32_t span32 = (uint32_t)(span >> psh2);
                const uint32_t scale = (uint32_t)(((uint64_t)K_ << 32) / ((uint64_t)span32 + 1));
                const uint32_t m_ar = __umulhi(span32, scale);
                for (uint32_t j = threadIdx.x; j <= m_ar; j += T) flags[j] = 0;
                if (threadIdx.x == 0) rec_max = 0;
                __syncthreads();
#pragma unroll
                for (int i = 0; i < ITEMS; ++i)
                    if ((int)threadIdx.x * ITEMS + i < S) {
                        const uint64_t rel = rec_prefix(k[i], base, wsh) - plo;
                        atomicAdd(&flags[min(__umulhi((uint32_t)(rel >> psh2), scale), m_ar)], 1u);
                    }
                __syncthreads();
                for (uint32_t j = threadIdx.x; j <= m_ar; j += T) atomicMax(&rec_max, flags[j]);
                __syncthreads();
                const bool even =
                    m_ar >= 1 && (uint64_t)rec_max * (m_ar + 1) <= 2ull * (uint64_t)S + 8ull * (m_ar + 1);
                __syncthreads();
                if (even) {
                    K* sorted = sorted_store + d.sp;
                    for (uint32_t j = threadIdx.x; j < m_ar; j += T) {
                        const uint64_t r = ((((uint64_t)(j + 1)) << 32) - 1) / scale;
                        sorted[j] = rec_from_prefix(plo + (((r + 1) << psh2) - 1), base, wsh);
                    }
                    if (threadIdx.x == 0) {
                        segs[seg].m = m_ar;
                        segs[seg].eq = 0;
                        segs[seg].lo = base;
                        segs[seg].shift = wsh;
                        segs[seg].hi = plo;
                        segs[seg].lutbits = psh2;
                        segs[seg].arith = 1;
                        segs[seg].scale = scale;
                    }
                    return;
                }
            }
        }
    }
    if (!pre) BS::sort(k, s, S);  // sorted sample of S keys in s (padded)
    auto at = [&](int q) -> K { return pre ? presorted[q] : s[P::idx(q)]; };
    uint64_t pbase = 0;
    uint32_t psh = 0;
    if constexpr (std::is_same<K, Rec32>::value) {  // prefix window of the sampled w0 range
        const uint64_t w0a = at(0).w[0], w0b = at(S - 1).w[0];
        pbase = w0a;
        psh = w0b > w0a ? (uint32_t)__clzll((long long)(w0b - w0a)) : 64u;
    }

    // candidate splitter j (0 <= j < K-1): sample quantile (j+1)/K
    for (uint32_t j = threadIdx.x; j < K_ - 1; j += T) {
        const int q = (int)(((uint64_t)(j + 1) * S) / K_);
        const K c = at(q);
        const bool keep = (j == 0) || !KT::eq(c, at((int)(((uint64_t)j * S) / K_)));
        flags[j] = keep ? 1u : 0u;
    }
    if (threadIdx.x == 0) flags[K_ - 1] = 0;
    __syncthreads();
    // compact unique splitters (candidates are sorted, so duplicates are adjacent)
    const uint32_t m = block_exclusive_scan_smem<T>(flags, (int)K_, warp_sums);
    K* sorted = sorted_store + d.sp;
    for (uint32_t j = threadIdx.x; j < K_ - 1; j += T) {
        const int q = (int)(((uint64_t)(j + 1) * S) / K_);
        if (flags[j + 1] != flags[j]) sorted[flags[j]] = at(q);
    }
    __syncthreads();  // sorted[] (global) is visible block-wide after the barrier
    for (uint32_t j = threadIdx.x; j < m; j += T) s[P::idx(j)] = sorted[j];  // compacted copy
    __syncthreads();
    if constexpr (KT::kLut) {
        // LUT cell c covers keys [lo + c<<shift, lo + (c+1)<<shift - 1] within [lo, hi]
        const uint32_t nc = 1u << d.lutbits;
        uint32_t* lut = lut_store + (size_t)d.sp * kLutPerSplitter;
        for (uint32_t c = threadIdx.x; c < nc; c += T) {
            const uint64_t cmin = d.lo + ((uint64_t)c << d.shift);
            uint64_t cmax = cmin + (((uint64_t)1 << d.shift) - 1);
            if (c == nc - 1 || cmax > d.hi || cmax < cmin) cmax = d.hi;
            // #{sorted < v} by binary search over the m unique splitters
            uint32_t jl = 0, jh = 0;
            for (int w = 0; w < 2; ++w) {
                const uint64_t v = w == 0 ? cmin : cmax;
                uint32_t lo2 = 0, cnt = m;
                while (cnt > 0) {
                    const uint32_t half = cnt >> 1;
                    if ((uint64_t)KT::bits(s[P::idx(lo2 + half)]) < v) {
                        lo2 += half + 1;
                        cnt -= half + 1;
                    } else {
                        cnt = half;
                    }
                }
                if (w == 0) jl = lo2;
                else jh = lo2;
            }
            // cells past hi (cmin > cmax after the clamp) hold no real key, but
            // the padding keys of a partial tile land in the last one: keep
            // the range empty rather than negative (a negative count read as
            // 0xFFFF sent the wide-cell search far outside the splitters)
            if (jh < jl) jh = jl;
            lut[c] = jl | ((jh - jl) << 16);
        }
    } else {
        // Eytzinger tree over sorted[0..m), padded with the maximum key.
        K* tree = tree_store + d.sp;
        for (uint32_t t = threadIdx.x + 1; t < K_; t += T) {
            const uint32_t depth = 31 - __clz(t);
            const uint32_t rank = ((2 * (t - (1u << depth)) + 1) << (d.logk - 1 - depth)) - 1;
            tree[t] = rank < m ? s[P::idx(rank)] : KT::max_key();
        }
    }
    if (threadIdx.x == 0) {
        segs[seg].m = m;
        segs[seg].eq = (m < K_ - 1) ? 1u : 0u;
        if constexpr (std::is_same<K, Rec32>::value) {
            segs[seg].lo = pbase;
            segs[seg].shift = psh;
        }
    }
}

// The level's segment count is read on the device (written by the previous
// level's plan), so a whole sort is enqueued without host round trips.
template <class K, int T, int ITEMS, bool XF = false>  // XF: level 0 of a fused-transform sort
__global__ void __launch_bounds__(T) sample_kernel(SegDesc* segs, const uint32_t* __restrict__ nsegs,
                                                   const K* __restrict__ src, K* tree_store,
                                                   K* sorted_store, uint32_t* lut_store,
                                                   uint64_t seed, uint32_t oversample,
                                                   Xf xf = Xf{0, 0}, const K* presorted = nullptr,
                                                   uint32_t presorted_n = 0, uint32_t even_target = 0,
                                                   uint32_t even_span = 0, uint32_t even_over = 0) {
    if (QMSORT_LEVEL_OVERFLOWED(nsegs, nsegs)) return;
    const uint32_t ns = *nsegs;
    LevelCounters* lc = reinterpret_cast<LevelCounters*>(const_cast<uint32_t*>(nsegs));  // nsegs is its first member
    for (uint32_t seg = blockIdx.x; seg < ns; seg += gridDim.x) {
        sample_segment<K, T, ITEMS, XF>(seg, segs, src, tree_store, sorted_store, lut_store, seed,
                                        oversample, xf, presorted, presorted_n, &lc->sample_keys, even_target,
                                        even_span, even_over);
        __syncthreads();  // shared memory is reused by the next segment
    }
}

// ---------------------------------------------------------------------------
// K2: per-chunk bucket histogram.
// ---------------------------------------------------------------------------
template <class K, int T, int U, int LOG_KMAX, bool XF>
__device__ __forceinline__ void count_chunk(const ClassifierSmem<K, LOG_KMAX>& cls, uint32_t* shist,
                                            const SegDesc& d, const ChunkDesc& c, uint32_t ck,
                                            const K* __restrict__ src, uint32_t* __restrict__ hist,
                                            const Xf& xf) {
    const uint32_t nb = (1u << d.logk) << d.eq;
    for (uint32_t i = threadIdx.x; i < nb; i += T) shist[i] = 0;
    __syncthreads();
    const K* p = src + c.begin + threadIdx.x;
    const uint32_t len = (uint32_t)(c.end - c.begin);
    constexpr uint32_t STEP = (uint32_t)T * U;
    uint32_t base = 0;
    for (; base + STEP <= len; base += STEP) {  // full tiles: no bounds checks
        K k[U];
        uint32_t bin[U];
#pragma unroll
        for (int u = 0; u < U; ++u) k[u] = XF ? xf_fwd(p[base + u * T], xf) : p[base + u * T];
        classify_keys<K, LOG_KMAX, U>(k, cls, d, bin);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            QCHECK(bin[u] < nb, bin[u], nb);
            atomicAdd(&shist[bin[u]], 1u);
        }
    }
    if (base < len) {
        const uint32_t rem = len - base;
        K k[U];
        uint32_t bin[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = u * T + threadIdx.x;
            k[u] = i < rem ? (XF ? xf_fwd(p[base + u * T], xf) : p[base + u * T]) : KeyTraits<K>::max_key();
        }
        classify_keys<K, LOG_KMAX, U>(k, cls, d, bin);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u * T + threadIdx.x < rem) atomicAdd(&shist[bin[u]], 1u);
    }
    __syncthreads();
    const uint32_t ci = ck - d.chunk_begin;
    const uint32_t stride = d.nchunks + 1;
    for (uint32_t b = threadIdx.x; b < nb; b += T) hist[d.hist_base + b * stride + ci] = shist[b];
    __syncthreads();
}

// Persistent CTAs fetch chunks dynamically from *work (no tail of idle SMs);
// the classifier is reloaded only when the segment changes.
template <class K, int T, int U, int LOG_KMAX>
__global__ void __launch_bounds__(T, 4) count_kernel(const SegDesc* __restrict__ segs,
                                                  const ChunkDesc* __restrict__ chunks,
                                                  uint32_t nchunks, const uint32_t* __restrict__ nchunks_dev,
                                                  uint32_t* __restrict__ work,
                                                  const K* __restrict__ src,
                                                  const K* __restrict__ tree_store,
                                                  const K* __restrict__ sorted_store,
                                                  const uint32_t* __restrict__ lut_store,
                                                  uint32_t* __restrict__ hist, Xf xf = Xf{0, 0}) {
    constexpr int KMAX = 1 << LOG_KMAX;
    __shared__ ClassifierSmem<K, LOG_KMAX> cls;
    __shared__ uint32_t shist[2 * KMAX];
    __shared__ uint32_t next_chunk;
    if (QMSORT_LEVEL_OVERFLOWED(nchunks_dev, nchunks)) return;
    const uint32_t nck = nchunks_dev ? *nchunks_dev : nchunks;  // device count: no host round trip
    uint32_t cur_seg = 0xFFFFFFFFu;
    for (;;) {
        if (threadIdx.x == 0) next_chunk = atomicAdd(work, 1u);
        __syncthreads();
        const uint32_t ck = next_chunk;
        if (ck >= nck) break;
        const ChunkDesc c = chunks[ck];
        const SegDesc d = segs[c.seg];
        if (c.seg != cur_seg) {
            load_classifier<K, LOG_KMAX, T>(cls, d, tree_store, sorted_store, lut_store);
            cur_seg = c.seg;
        }
        if (xf.a | xf.b) count_chunk<K, T, U, LOG_KMAX, true>(cls, shist, d, c, ck, src, hist, xf);
        else count_chunk<K, T, U, LOG_KMAX, false>(cls, shist, d, c, ck, src, hist, xf);
    }
}

// ---------------------------------------------------------------------------
// K3a: per (segment, bin): exclusive prefix over the segment's chunks (in
// place) and the bin total (entry nchunks).  One warp per bin.
// ---------------------------------------------------------------------------
// One warp per (segment, bin) pair, flattened over the level's segments with
// the level's largest bin count (segment count and largest K read on the
// device; null cnt = one segment of up to 1024 bins).
__global__ void __launch_bounds__(512) colsum_kernel(const SegDesc* __restrict__ segs,
                                                     uint32_t* __restrict__ hist,
                                                     const LevelCounters* __restrict__ cnt) {
    if (cnt && cnt->overflow) return;
    const uint32_t ns = cnt ? cnt->nsegs : 1u;
    const uint32_t NBMAX = cnt ? (2u << cnt->max_logk) : 1024u;  // bins incl. equality bins
    if (cnt && cnt->max_nchunks <= 16) {
        // segments of a few chunks (the lower levels): one thread per
        // (segment, bin) walks its column serially -- a warp per column
        // would leave most lanes idle
        const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
        for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (uint64_t)ns * NBMAX;
             idx += nt) {
            const SegDesc d = segs[idx / NBMAX];
            const uint32_t b = (uint32_t)(idx % NBMAX);
            if (b >= ((1u << d.logk) << d.eq)) continue;
            uint32_t* col = hist + d.hist_base + b * (d.nchunks + 1);
            uint32_t v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = c < (int)d.nchunks ? col[c] : 0u;
            uint32_t carry = 0;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                if (c < (int)d.nchunks) col[c] = carry;
                carry += v[c];
            }
            col[d.nchunks] = carry;
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t idx = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
         idx < (uint64_t)ns * NBMAX; idx += nw) {
        const SegDesc d = segs[idx / NBMAX];
        const uint32_t b = (uint32_t)(idx % NBMAX);
        const uint32_t nb = (1u << d.logk) << d.eq;
        if (b >= nb) continue;
        const uint32_t stride = d.nchunks + 1;
        uint32_t* col = hist + d.hist_base + b * stride;
        uint32_t carry = 0;
        for (uint32_t c0 = 0; c0 < d.nchunks; c0 += 128) {
            uint32_t v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // four loads in flight per lane
                const uint32_t c = c0 + q * 32 + lane;
                v[q] = c < d.nchunks ? col[c] : 0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t c = c0 + q * 32 + lane;
                uint32_t x = v[q];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (c < d.nchunks) col[c] = carry + x - v[q];
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
        }
        if (lane == 0) col[d.nchunks] = carry;
    }
}

// Key bounds of bin b of segment d (integer keys): bucket j holds the keys in
// (splitter j-1, splitter j] within the segment's [lo, hi]; with equality
// bins the splitter itself went to bin 2j+1.
template <class K>
__device__ __forceinline__ void bucket_bounds(const SegDesc& d, const K* __restrict__ sp, uint32_t b,
                                              uint64_t& klo, uint64_t& khi) {
    klo = d.lo;
    khi = d.hi;
    if constexpr (KeyTraits<K>::kLut) {
        const uint32_t j = d.eq ? (b >> 1) : b;
        if (j > 0) klo = (uint64_t)KeyTraits<K>::bits(sp[j - 1]) + 1;
        if (j < d.m) khi = (uint64_t)KeyTraits<K>::bits(sp[j]) - (d.eq ? 1u : 0u);
    }
}

// ---------------------------------------------------------------------------
// K3b: per segment: bucket starts and child work.
// ---------------------------------------------------------------------------
template <class K, int T, int LOG_KMAX>
__global__ void __launch_bounds__(T) plan_kernel(const SegDesc* __restrict__ segs,
                                                 uint32_t* __restrict__ hist,
                                                 const K* __restrict__ sorted_store,
                                                 LevelBufs next, PlanParams p,
                                                 SortTask* __restrict__ tasks,
                                                 FillTask* __restrict__ fills,
                                                 LevelCounters* __restrict__ cur_cnt,
                                                 LevelCounters* __restrict__ sort_cnt) {
    constexpr int NB = 2 << LOG_KMAX;
    __shared__ uint32_t tot[NB];
    __shared__ uint32_t start[NB];
    __shared__ uint32_t slot[NB];  // block-sort task: class << 28 | index within the class
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t cls_count[kNumClasses], cls_base[kNumClasses];
    __shared__ unsigned long long cls_keys;
    if (*(volatile const uint32_t*)&cur_cnt->overflow) return;  // uniform: set before this kernel
    const uint32_t ns = cur_cnt->nsegs;  // device count: no host round trip
    for (uint32_t seg = blockIdx.x; seg < ns; seg += gridDim.x) {
    __syncthreads();  // the previous segment's shared arrays are no longer read
    const SegDesc d = segs[seg];
    const uint32_t nb = (1u << d.logk) << d.eq;
    const uint32_t stride = d.nchunks + 1;
    if (threadIdx.x < kNumClasses) cls_count[threadIdx.x] = 0;
    if (threadIdx.x == 0) cls_keys = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        const uint32_t v = hist[d.hist_base + b * stride + d.nchunks];
        tot[b] = v;
        start[b] = v;
    }
    __syncthreads();
    block_exclusive_scan_smem<T>(start, (int)nb, warp_sums);
    // block-sort tasks: reserve per class in shared memory first, then one
    // global atomic per class and CTA (the global counters are contended)
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        const uint32_t len = tot[b];
        uint32_t sl = 0xFFFFFFFFu;
        if (len != 0 && !(d.eq && (b & 1)) && len <= p.cap && !(len == 1 && p.dst_is_a && !p.xf_fix)) {
            uint32_t cls = 0;
            while (cls < kNumClasses - 1 && len > p.class_cap[cls]) ++cls;
            if (KeyTraits<K>::kLut && (p.table_class < (uint32_t)kNumClasses || p.cell_class < (uint32_t)kNumClasses)) {
                uint64_t klo, khi;
                bucket_bounds<K>(d, sorted_store + d.sp, b, klo, khi);
                if (p.table_class < (uint32_t)kNumClasses && table_sort_eligible(len, klo, khi)) cls = p.table_class;
                else if (p.cell_class < (uint32_t)kNumClasses && cell_sort_eligible(len, klo, khi, p.cell_cap, p.cell_bits)) cls = p.cell_class;
                else if (p.cell_big_class < (uint32_t)kNumClasses && len > p.cell_cap &&
                         cell_sort_eligible(len, klo, khi, p.cell_big_cap, p.cell_big_bits)) cls = p.cell_big_class;
            }
            // records: the cell sort finds the bucket's prefix bounds itself
            if (!KeyTraits<K>::kLut && p.cell_class < (uint32_t)kNumClasses && len >= 256u && len <= p.cell_cap)
                cls = p.cell_class;
            sl = (cls << 28) | atomicAdd(&cls_count[cls], 1u);
            atomicAdd(&cls_keys, (unsigned long long)len);
        }
        slot[b] = sl;
    }
    __syncthreads();
    if (threadIdx.x < kNumClasses)
        cls_base[threadIdx.x] = cls_count[threadIdx.x]
                                    ? atomicAdd(&sort_cnt->ntasks[threadIdx.x], cls_count[threadIdx.x])
                                    : 0u;
    if (threadIdx.x == 0 && cls_keys) atomicAdd(&sort_cnt->task_keys, cls_keys);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        hist[d.hist_base + b * stride + d.nchunks] = start[b];
        const uint32_t len = tot[b];
        if (len == 0) continue;
        const uint64_t off = d.off + start[b];
        if (d.eq && (b & 1)) {  // equal-key bucket: final once it is in the caller's buffer
            if (!p.dst_is_a || p.xf_fix) {  // (fused transform: its fill writes f^-1)
                // small fills from the front (a warp each), large ones from the back
                const bool big = len > kFillWarp;
                const uint32_t f = atomicAdd(big ? &sort_cnt->nfill_big : &sort_cnt->nfill, 1u);
                if (f < p.fill_cap / 2) {
                    FillTask ft;
                    ft.off = off;
                    ft.len = len;
                    const K v = sorted_store[d.sp + (b >> 1)];
                    memcpy(ft.value, &v, sizeof(K));
                    fills[big ? p.fill_cap - 1 - f : f] = ft;
                    atomicAdd(&sort_cnt->fill_keys, (unsigned long long)len);
                } else {
                    atomicExch(&cur_cnt->overflow, 1u);
                }
            }
        } else if (len <= p.cap) {
            QCHECK((uint64_t)start[b] + len <= d.len, start[b] + len, d.len);
            const uint32_t sl = slot[b];
            if (sl == 0xFFFFFFFFu) continue;  // single key already in place
            const uint32_t cls = sl >> 28;
            const uint32_t t = cls_base[cls] + (sl & 0x0FFFFFFFu);
            if (t < p.task_cap) {
                SortTask st;
                st.off = off;
                st.len = len;
                st.in_a = p.dst_is_a ? 1u : 0u;
                bucket_bounds<K>(d, sorted_store + d.sp, b, st.klo, st.khi);
                tasks[(size_t)cls * p.task_cap + t] = st;
            } else {
                atomicExch(&cur_cnt->overflow, 1u);
            }
        } else {
            // child key range: (splitter j-1, splitter j] within the parent's [lo, hi]
            const uint32_t j = d.eq ? (b >> 1) : b;
            const K* sp = sorted_store + d.sp;
            uint64_t clo = d.lo, chi = d.hi;
            if (KeyTraits<K>::kLut) {
                if (j > 0) clo = KeyTraits<K>::bits(sp[j - 1]) + 1;
                if (j < d.m) chi = KeyTraits<K>::bits(sp[j]);
            }
            // worst-case policy (f1): mom_of_thirds always samples triple
            // medians; hybrid does so for a child outside the delta band,
            // i.e. larger than (parent / buckets) / delta
            uint32_t sampler = p.pivot == 2 ? kSampleTriples : p.pivot == 1 ? kSampleSqrt : kSampleRandom;
            if (p.pivot == 3 &&
                (uint64_t)len * (uint64_t)(1u << d.logk) * p.delta_q16 > d.len * 65536ull) {
                sampler = kSampleTriples;
                atomicAdd(&cur_cnt->resplits, 1u);
            }
            emit_segment(next, off, len, clo, chi, p, sampler);
        }
    }
    }  // segments
}

// ---------------------------------------------------------------------------
// K4: scatter.  Tile = T * U keys; one CTA walks the tiles of one chunk.
// ---------------------------------------------------------------------------
template <class K, int T, int U, int LOG_KMAX>
struct ScatterSmem {
    static constexpr int KMAX = 1 << LOG_KMAX;
    static constexpr int NB = 2 * KMAX;
    static constexpr int BPT = NB / T;  // bins owned by each thread in the scan
    static_assert(NB % T == 0 && (BPT == 1 || BPT == 2 || BPT == 4), "bins per thread");
    static constexpr int TILE = T * U;
    // a staged key travels with its segment-relative destination, so the
    // write-out reads one record per key and needs no per-bucket lookup
    // 8- and 32-byte keys stage only their index in the tile: the write-out
    // re-reads the key from the tile just loaded (L1/L2), which moves 8
    // instead of 16 / 48 bytes per key through shared memory twice (measured:
    // C5 scatter 3.78 -> 2.87 ms, C4a 2.80 -> 2.56 ms, C3 unchanged).
    static constexpr bool kStageIndex = sizeof(K) >= 8;
    struct alignas(sizeof(K) >= 8 && !kStageIndex ? 16 : 8) Rec {
        typename std::conditional<kStageIndex, uint32_t, K>::type key;  // key, or its tile index
        uint32_t dest;
    };
    ClassifierSmem<K, LOG_KMAX> cls;
    Rec stage[TILE];
    alignas(16) uint32_t hist[NB];
    alignas(16) uint2 sd[NB];  // {bucket start in the tile, destination base}
    uint32_t warp_sums[T / 32];
};

template <int N>
struct VecU32;
template <>
struct VecU32<1> {
    using type = uint32_t;
};
template <>
struct VecU32<2> {
    using type = uint2;
};
template <>
struct VecU32<4> {
    using type = uint4;
};
template <int N>
__device__ __forceinline__ void vec_load(const uint32_t* p, uint32_t (&v)[N]) {
    const typename VecU32<N>::type x = *reinterpret_cast<const typename VecU32<N>::type*>(p);
    memcpy(v, &x, sizeof(x));
}
template <int N>
__device__ __forceinline__ void vec_store(uint32_t* p, const uint32_t (&v)[N]) {
    typename VecU32<N>::type x;
    memcpy(&x, v, sizeof(x));
    *reinterpret_cast<typename VecU32<N>::type*>(p) = x;
}

// One tile of m keys (m == T*U when FULL): classify, rank within the tile's
// bucket (shared-memory counter), exclusive scan of the tile histogram (each
// thread owns BPT consecutive bins and keeps their write cursors in
// registers), group by bucket in shared memory, then write every bucket run
// with coalesced stores.
// Where a scatter writes: the segment's range of the destination buffer
// (every level of the sort), or -- the sharded exchange fused into the
// partition -- every bin's keys straight into its rank's receive buffer, a
// peer GPU's memory mapped through CUDA IPC (or this GPU's own), at that
// rank's offset for this sender.  The ranks' buffers are laid end to end in
// one virtual key space: rank r owns positions [vbase[r], vbase[r+1]); a
// bin's write cursor starts at its virtual position for this sender
// (bin_base, from the host's plan), so the scatter's own position arithmetic
// is unchanged and each store maps its position to (rank, offset).
// Positions >= vbase[nranks] belong to bins that are not sent (equal-key
// runs the receivers fill).
constexpr int kMaxPeers = 8;
constexpr int kMaxPeerBins = 1024;  // bins of one exchange (2 x 512 with equality bins)
struct PeerArgs {
    unsigned long long dest[kMaxPeers];  // receive buffer of rank r (device pointer)
    uint32_t vbase[kMaxPeers + 1];       // virtual key positions of the ranks' buffers
    uint32_t nranks;
    uint32_t raw;                        // ship the caller's bit patterns (else core keys)
    const uint32_t* bin_base;            // device: this sender's first virtual position per bin
};
template <class K>
struct LocalSink {
    K* out;
    uint64_t lim;  // the segment's length (checked builds)
    __device__ __forceinline__ void store(uint32_t dest, const K& key) const {
        QCHECK(dest < lim, dest, lim);
        out[dest] = key;
    }
    __device__ __forceinline__ void store_bin(uint32_t, uint32_t dest, const K& key) const {
        QCHECK(dest < lim, dest, lim);
        out[dest] = key;
    }
};
// The fused exchange: a virtual position -> its rank (a three-step binary
// search over the ranks' bases in shared memory; one rank: none) -> one
// store at dmv[rank] + v * sizeof(K) (dmv = buffer - base * sizeof(K)).
template <class K>
struct PeerSink {
    const unsigned long long* dmv;  // shared memory
    const uint32_t* vb;             // shared memory: kMaxPeers + 1 bases, unused ranks = end
    uint32_t nranks;
    __device__ __forceinline__ void store(uint32_t v, const K& key) const {
        if (v >= vb[kMaxPeers]) return;  // a bin that is not sent
        uint32_t r = 0;
        if (nranks > 1) {
            r = v >= vb[4] ? 4u : 0u;
            r += v >= vb[r + 2] ? 2u : 0u;
            r += v >= vb[r + 1] ? 1u : 0u;
        }
        *reinterpret_cast<K*>(dmv[r] + (unsigned long long)v * sizeof(K)) = key;
    }
    __device__ __forceinline__ void store_bin(uint32_t, uint32_t v, const K& key) const { store(v, key); }
};

// The m keys of a tile into registers (striped: key u of thread t is p[u T + t]).
template <class K, int T, int U, bool XF>
__device__ __forceinline__ void load_tile(K (&k)[U], const K* __restrict__ p, uint32_t m, const Xf& xf) {
    const uint32_t tid = threadIdx.x;
    if (m == (uint32_t)(T * U)) {
#pragma unroll
        for (int u = 0; u < U; ++u) k[u] = XF ? xf_fwd(p[u * T + tid], xf) : p[u * T + tid];
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t li = u * T + tid;
            k[u] = li < m ? (XF ? xf_fwd(p[li], xf) : p[li]) : KeyTraits<K>::max_key();
        }
    }
}

// k: the tile's keys (load_tile); once they are staged the next tile of the
// chunk (pnext, mnext keys; 0: none) is loaded into k, so its global loads
// are in flight during the write-out.
template <class K, int T, int U, int LOG_KMAX, bool FULL, bool XF, class Sink, bool RAW = false>
__device__ __forceinline__ void scatter_tile(ScatterSmem<K, T, U, LOG_KMAX>& sm, const SegDesc& d,
                                             const K* __restrict__ p, uint32_t m,
                                             const Sink& out,
                                             uint32_t (&cursor)[ScatterSmem<K, T, U, LOG_KMAX>::BPT],
                                             const Xf& xf, K (&k)[U], const K* __restrict__ pnext,
                                             uint32_t mnext) {
    using SM = ScatterSmem<K, T, U, LOG_KMAX>;
    constexpr int BPT = SM::BPT;
    const uint32_t tid = threadIdx.x;
    uint32_t bin[U];
    classify_keys<K, LOG_KMAX, U>(k, sm.cls, d, bin);
    // rank within the tile's bucket; pack (bin, rank) into one word
    if (((1u << d.logk) << d.eq) <= 64) {
        // Few bins (the sharded exchange's P buckets, small segments): no
        // staging.  Warp-aggregated ranks give the lanes of one bin
        // consecutive slots after the bin's cursor, so every key is stored
        // straight from its register and each bin's lanes write one
        // contiguous run.
        uint32_t* base = reinterpret_cast<uint32_t*>(sm.sd);  // bin -> destination of its next key
#pragma unroll
        for (int i = 0; i < BPT; ++i) base[tid * BPT + i] = cursor[i];
        __syncthreads();
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool v = FULL || u * T + tid < m;
            const uint32_t r = warp_agg_inc(sm.hist, bin[u], v);
            // the exchange ships the caller's bit patterns (receivers sort
            // them with the fused transform); local levels store core keys
            if (v) out.store_bin(bin[u], base[bin[u]] + r, RAW && XF ? xf_inv(k[u], xf) : k[u]);
        }
        if (mnext) load_tile<K, T, U, XF>(k, pnext, mnext, xf);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            cursor[i] += sm.hist[tid * BPT + i];
            sm.hist[tid * BPT + i] = 0;
        }
        __syncthreads();
        return;
    }
    {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (FULL || u * T + tid < m) bin[u] = (bin[u] << 16) | atomicAdd(&sm.hist[bin[u]], 1u);
    }
    __syncthreads();
    {  // block exclusive scan over all NB bins, BPT per thread
        uint32_t h[BPT];
        vec_load<BPT>(&sm.hist[tid * BPT], h);
        uint32_t local = 0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) local += h[i];
        const uint32_t lane = tid & 31, wid = tid >> 5;
        uint32_t x = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) sm.warp_sums[wid] = x;
        __syncthreads();
        // earlier warps' totals: one load per lane and a warp reduction
        // (not T/32 broadcast loads per thread)
        const uint32_t ws = lane < wid ? sm.warp_sums[lane] : 0u;
        uint32_t excl = x - local + __reduce_add_sync(0xffffffffu, ws);
        uint32_t z[BPT];
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
#if QMSORT_SCATTER_BINREC
            // bin start in the tile / its destination shift, as two arrays:
            // the staging reads 4 random bytes, the write-out reads the shift
            // of runs of equal bins (mostly one address per warp)
            reinterpret_cast<uint32_t*>(sm.sd)[tid * BPT + i] = excl;
            reinterpret_cast<uint32_t*>(sm.sd)[SM::NB + tid * BPT + i] = cursor[i] - excl;
#else
            sm.sd[tid * BPT + i] = make_uint2(excl, cursor[i] - excl);
#endif
            cursor[i] += h[i];
            excl += h[i];
            z[i] = 0;
        }
        vec_store<BPT>(&sm.hist[tid * BPT], z);
    }
    __syncthreads();
    if constexpr (QMSORT_SCATTER_BINREC) {
        // Even splitters: a key's bin is a product of the key, so the staged
        // record is the key alone (8-byte keys: its tile index) -- 4 bytes
        // through shared memory instead of 8; the write-out recomputes the bin.
        if (d.arith) {
            // 4- and 8-byte keys are staged themselves (QMSORT_STAGE_KEY8: 8-byte
            // keys too -- 8 bytes through shared memory, no second read of the
            // tile), records by their tile index
            constexpr bool kKey = sizeof(K) == 4 || (sizeof(K) == 8 && QMSORT_STAGE_KEY8);
            using SlotT = typename std::conditional<kKey && sizeof(K) == 8, uint64_t, uint32_t>::type;
            SlotT* st = reinterpret_cast<SlotT*>(sm.stage);
            const uint32_t* binstart = reinterpret_cast<const uint32_t*>(sm.sd);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (FULL || u * T + tid < m) {
                    const uint32_t pos = binstart[bin[u] >> 16] + (bin[u] & 0xFFFFu);
                    QCHECK(pos < m, pos, m);
                    if constexpr (kKey) memcpy(&st[pos], &k[u], sizeof(SlotT));
                    else st[pos] = u * T + tid;
                }
            }
            if (mnext) load_tile<K, T, U, XF>(k, pnext, mnext, xf);
            __syncthreads();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = u * T + tid;
                if (FULL || i < m) {
                    const SlotT v = st[i];
                    K raw, core;
                    if constexpr (kKey) {
                        memcpy(&core, &v, sizeof(SlotT));
                        raw = XF ? xf_inv(core, xf) : core;
                    } else {
                        raw = p[v];
                        core = XF ? xf_fwd(raw, xf) : raw;
                    }
                    const uint32_t b = even_bucket<K>(core, d);
                    const uint32_t dest = binstart[SM::NB + b] + i;
                    out.store(dest, RAW && XF ? raw : core);
                }
            }
            __syncthreads();
            return;
        }
    }
    typename SM::Rec* stage = sm.stage;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (FULL || u * T + tid < m) {
#if QMSORT_SCATTER_BINREC
            const uint32_t pos = reinterpret_cast<const uint32_t*>(sm.sd)[bin[u] >> 16] + (bin[u] & 0xFFFFu);
#else
            const uint2 sg = sm.sd[bin[u] >> 16];
            const uint32_t pos = sg.x + (bin[u] & 0xFFFFu);
#endif
            QCHECK(pos < m, pos, m);
            typename SM::Rec r;
            if constexpr (SM::kStageIndex) r.key = u * T + tid;
            else r.key = k[u];
#if QMSORT_SCATTER_BINREC
            r.dest = bin[u] >> 16;  // the bin; the write-out adds its shift
#else
            r.dest = sg.y + pos;
#endif
            stage[pos] = r;
        }
    }
    if (mnext) load_tile<K, T, U, XF>(k, pnext, mnext, xf);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t i = u * T + tid;
        if (FULL || i < m) {
            const typename SM::Rec r = stage[i];
#if QMSORT_SCATTER_BINREC
            const uint32_t dest = reinterpret_cast<const uint32_t*>(sm.sd)[SM::NB + r.dest] + i;
#else
            const uint32_t dest = r.dest;
#endif
            if constexpr (SM::kStageIndex) out.store(dest, XF && !RAW ? xf_fwd(p[r.key], xf) : p[r.key]);
            else out.store(dest, RAW && XF ? xf_inv(r.key, xf) : r.key);
        }
    }
    __syncthreads();
    }
}

// The tiles of one chunk, software-pipelined: tile t+1's keys are loaded
// while tile t is written out.
template <class K, int T, int U, int LOG_KMAX, bool XF, class Sink, bool RAW>
__device__ __forceinline__ void scatter_chunk(ScatterSmem<K, T, U, LOG_KMAX>& sm, const SegDesc& d,
                                              const K* __restrict__ p, uint32_t len, const Sink& out,
                                              uint32_t (&cursor)[ScatterSmem<K, T, U, LOG_KMAX>::BPT],
                                              const Xf& xf) {
    constexpr uint32_t TILE = (uint32_t)T * U;
    // 4- and 8-byte keys (measured: C2 scatter 1476 -> 1348 us; C3, with the
    // keys themselves staged under even splitters, 11.5 -> 9.8 ms; records,
    // whose registers the write-out needs, lose 5 %)
    constexpr bool kPrefetch = sizeof(K) == 4 || (sizeof(K) == 8 && QMSORT_PREFETCH8);
    K k[U];
    if (kPrefetch) load_tile<K, T, U, XF>(k, p, min(len, TILE), xf);
    for (uint32_t t0 = 0; t0 < len;) {
        const uint32_t m = min(TILE, len - t0);
        const uint32_t nx = t0 + m;
        const uint32_t mn = kPrefetch ? min(TILE, len - nx) : 0u;  // 0 after the last tile
        if (!kPrefetch) load_tile<K, T, U, XF>(k, p + t0, m, xf);
        if (m == TILE)
            scatter_tile<K, T, U, LOG_KMAX, true, XF, Sink, RAW>(sm, d, p + t0, m, out, cursor, xf, k, p + nx, mn);
        else
            scatter_tile<K, T, U, LOG_KMAX, false, XF, Sink, RAW>(sm, d, p + t0, m, out, cursor, xf, k, p + nx, mn);
        t0 = nx;
    }
}

template <class K, int T, int U, int LOG_KMAX, bool PEER = false>
__global__ void __launch_bounds__(T, T >= 1024 ? 1 : T >= 512 ? 2 : (sizeof(K) >= 8 ? 2 : 3)) scatter_kernel(const SegDesc* __restrict__ segs,
                                                    const ChunkDesc* __restrict__ chunks,
                                                    uint32_t nchunks, const uint32_t* __restrict__ nchunks_dev,
                                                    uint32_t* __restrict__ work,
                                                    const K* __restrict__ src, K* __restrict__ dst,
                                                    const K* __restrict__ tree_store,
                                                    const K* __restrict__ sorted_store,
                                                    const uint32_t* __restrict__ lut_store,
                                                    const uint32_t* __restrict__ hist,
                                                    PeerArgs peers = PeerArgs{}, Xf xf = Xf{0, 0}) {
    using SM = ScatterSmem<K, T, U, LOG_KMAX>;
    constexpr uint32_t TILE = SM::TILE;
    constexpr int BPT = SM::BPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    __shared__ uint32_t next_chunk;
    __shared__ unsigned long long peer_dmv[PEER ? kMaxPeers : 1];
    __shared__ uint32_t peer_vb[PEER ? kMaxPeers + 1 : 1];
    if (PEER && threadIdx.x < kMaxPeers)
        peer_dmv[threadIdx.x] = peers.dest[threadIdx.x] - (unsigned long long)peers.vbase[threadIdx.x] * sizeof(K);
    if (PEER && threadIdx.x <= kMaxPeers) peer_vb[threadIdx.x] = peers.vbase[threadIdx.x];
    if (QMSORT_LEVEL_OVERFLOWED(nchunks_dev, nchunks)) return;
    const uint32_t nck = nchunks_dev ? *nchunks_dev : nchunks;  // device count: no host round trip
    uint32_t cur_seg = 0xFFFFFFFFu;
    // persistent CTAs fetch chunks dynamically (no tail of idle SMs)
    for (;;) {
        if (threadIdx.x == 0) next_chunk = atomicAdd(work, 1u);
        __syncthreads();
        const uint32_t ck = next_chunk;
        if (ck >= nck) break;
        const ChunkDesc c = chunks[ck];
        const SegDesc d = segs[c.seg];
        const uint32_t nb = (1u << d.logk) << d.eq;
        if (c.seg != cur_seg) {
            load_classifier<K, LOG_KMAX, T>(sm.cls, d, tree_store, sorted_store, lut_store);
            cur_seg = c.seg;
        }
        const uint32_t ci = ck - d.chunk_begin;
        const uint32_t stride = d.nchunks + 1;
        uint32_t cursor[BPT];
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            const uint32_t b = threadIdx.x * BPT + i;
            cursor[i] = 0;
            if (b < nb) {
                const uint32_t* col = hist + d.hist_base + b * stride;
                // bucket start (local) or the bin's virtual position (peers) + chunk prefix
                cursor[i] = (PEER ? peers.bin_base[b] : col[d.nchunks]) + col[ci];
            }
            sm.hist[b] = 0;
        }
        __syncthreads();

        const K* p = src + c.begin;
        const uint32_t len = (uint32_t)(c.end - c.begin);
        if constexpr (PEER) {
            const PeerSink<K> out{peer_dmv, peer_vb, peers.nranks};
            if ((xf.a | xf.b) && peers.raw)  // ship the caller's keys
                scatter_chunk<K, T, U, LOG_KMAX, true, PeerSink<K>, true>(sm, d, p, len, out, cursor, xf);
            else if (xf.a | xf.b)  // ship core keys
                scatter_chunk<K, T, U, LOG_KMAX, true, PeerSink<K>, false>(sm, d, p, len, out, cursor, xf);
            else
                scatter_chunk<K, T, U, LOG_KMAX, false, PeerSink<K>, false>(sm, d, p, len, out, cursor, xf);
        } else {
            const LocalSink<K> out{dst + d.off, d.len};
            if (xf.a | xf.b)  // level 0 of a fused-transform sort
                scatter_chunk<K, T, U, LOG_KMAX, true, LocalSink<K>, false>(sm, d, p, len, out, cursor, xf);
            else
                scatter_chunk<K, T, U, LOG_KMAX, false, LocalSink<K>, false>(sm, d, p, len, out, cursor, xf);
        }
    }
}

// Equal-key buckets: write the splitter value (f^-1 of it) over the bucket.
// The fill count is read on the device (written by the level's plan).
// Buckets up to kFillWarp keys get a warp each (many small equal runs, e.g.
// the exchange's equal-key shares); larger ones the whole grid in turn.
template <class K>
__global__ void fill_kernel(const FillTask* __restrict__ fills, const uint32_t* __restrict__ nfill,
                            const uint32_t* __restrict__ nfill_big, uint32_t fill_cap, K* __restrict__ dst,
                            Xf xf = Xf{0, 0}) {
    const uint32_t ns = min(*nfill, fill_cap / 2), nbig = min(*nfill_big, fill_cap / 2);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t f = gw; f < ns; f += nw) {
        const FillTask ft = fills[f];
        K v;
        memcpy(&v, ft.value, sizeof(K));
        v = xf_inv(v, xf);
        for (uint64_t i = lane; i < ft.len; i += 32) dst[ft.off + i] = v;
    }
    for (uint32_t f = 0; f < nbig; ++f) {
        const FillTask ft = fills[fill_cap - 1 - f];
        K v;
        memcpy(&v, ft.value, sizeof(K));
        v = xf_inv(v, xf);
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ft.len;
             i += (uint64_t)gridDim.x * blockDim.x)
            dst[ft.off + i] = v;
    }
}

// Block-sort every task of one size class into A (from A or B, at the same
// offsets): one CTA per task (launched with the sort's task count).
template <class K, int T, int ITEMS>
// 4-byte keys: registers budgeted for 1536 / T resident CTAs (40 per
// thread, a few spills): occupancy beats registers here (measured on C2:
// 64 regs 1735 us, 48-51 regs 1684 us, 40 regs 1673 us).  Other keys: the
// compiler's choice (0) -- an explicit 1 lets it take ~50% more registers
// (measured: u64 and record block sorts 30% slower).
#ifndef QMSORT_BS_U32_THREADS
#define QMSORT_BS_U32_THREADS 1536
#endif
__global__ void __launch_bounds__(T, sizeof(K) == 4 ? QMSORT_BS_U32_THREADS / T : 0) blocksort_tasks_kernel(const SortTask* __restrict__ tasks, K* A,
                                                            const K* B, Xf xf = Xf{0, 0}) {
    using BS = BlockSorter<K, T, ITEMS>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s = reinterpret_cast<K*>(smem_raw);
    const SortTask t = tasks[blockIdx.x];
    QCHECK(t.len <= (uint32_t)BS::kCap, t.len, BS::kCap);
    BS::sort_tile((t.in_a ? A : B) + t.off, A + t.off, (int)t.len, s, xf);
}

// Block-sort consecutive tiles of a range (merge-sort front end / fallback).
template <class K, int T, int ITEMS>
__global__ void __launch_bounds__(T) blocksort_tiles_kernel(const K* src, K* dst, uint64_t off,
                                                            uint64_t len) {
    using BS = BlockSorter<K, T, ITEMS>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s = reinterpret_cast<K*>(smem_raw);
    const uint64_t t0 = (uint64_t)blockIdx.x * BS::kCap;
    const int m = (int)min((uint64_t)BS::kCap, len - t0);
    BS::sort_tile(src + off + t0, dst + off + t0, m, s);
}

}  // namespace qmsort_b200
