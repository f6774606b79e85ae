// samplesort.cuh -- K1..K4 + K8: sampled multi-splitter partition.
//
// Generalises the reference's pivot step (median_of_3_index,
// partition.hpp:21-30; median_of_sqrt_pivot, partition.hpp:235-251) and its
// partition (block_partition, partition.hpp:37-164) from one pivot / two sides
// to K-1 splitters / up to 2K-1 buckets per pass:
//   * sample_kernel   (K1) -- per segment, draws a seeded sample, sorts it on
//                             chip (blocksort.cuh) and picks K-1 evenly spaced
//                             splitters, exactly like the Median-of-sqrt(n)
//                             sample generalised to K-1 quantiles.  Duplicate
//                             splitters switch the segment to three-way
//                             classification (K8, the "equal block takes no
//                             further part" rule of three_way_partition,
//                             partition.hpp:194-195).
//   * count_kernel    (K2) -- branchless search-tree classification, per-chunk
//                             bucket histogram in shared memory.
//   * plan_kernel     (K3) -- per segment: bucket totals, exclusive scan,
//                             per-(chunk, bucket) output offsets; emits the
//                             child work (next-level segments, block-sort
//                             tasks, equal-bucket fills).
//   * scatter_kernel  (K4) -- re-classifies each tile, groups it by bucket in
//                             shared memory and writes every bucket run with
//                             coalesced stores to its final offset.
// Offsets are deterministic (no global atomics on the data path): chunk c of
// a segment writes bucket b at  start[b] + sum_{c' < c} hist[c'][b].
#pragma once
#include "blocksort.cuh"
#include "common.cuh"

namespace qmsort_b200 {

constexpr int kNumClasses = 3;  // block-sort size classes

struct SegDesc {
    uint64_t off;          // absolute element offset of the segment
    uint64_t len;          // number of keys
    uint32_t chunk_begin;  // first chunk in the level's chunk table
    uint32_t nchunks;
    uint32_t logk;         // K = 1 << logk buckets (2K with equality buckets)
    uint32_t m;            // unique splitters (set by sample_kernel)
    uint32_t eq;           // three-way classification on
    uint32_t sp;           // base index of this segment's splitter storage
    uint32_t hist_base;    // first histogram word; chunk i's row is at
                           // hist_base + i * 2K (2K bins per row)
    uint32_t pad;
};

struct ChunkDesc {
    uint32_t seg;
    uint32_t pad;
    uint64_t begin;  // absolute element range [begin, end)
    uint64_t end;
};

struct SortTask {  // one bucket for the block sorter
    uint64_t off;
    uint32_t len;
    uint32_t pad;
};

struct FillTask {  // equal-key bucket: every key equals the segment's splitter j
    uint64_t off;
    uint64_t len;
    uint32_t seg;
    uint32_t j;
};

struct LevelCounters {
    uint32_t nsegs;
    uint32_t nchunks;
    uint32_t nsplit;  // splitter storage used
    uint32_t nhist;   // histogram words used
    uint32_t nfill;
    uint32_t ntasks[kNumClasses];
    uint32_t overflow;  // capacity exceeded somewhere (host reports an error)
    unsigned long long nkeys;      // keys in this level's segments (pass ledger)
    unsigned long long task_keys;  // keys handed to the block sorter
    unsigned long long fill_keys;  // keys written by equal-bucket fills
};

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
    uint32_t log_kmax;      // largest K = 1 << log_kmax
    uint32_t class_cap[kNumClasses];
    uint32_t task_cap, fill_cap;
    int dst_is_a;           // this level's scatter writes the caller's buffer
};

__host__ __device__ inline uint32_t ceil_log2_u64(uint64_t x) {
    uint32_t r = 0;
    while ((1ull << r) < x) ++r;
    return r;
}

// Number of buckets for a segment of len keys: spread the remaining
// log2(len/target) bits evenly over the fewest levels of at most 2^log_kmax.
__host__ __device__ inline uint32_t choose_logk(uint64_t len, uint32_t target, uint32_t log_kmax) {
    const uint64_t ratio = (len + target - 1) / target;
    uint32_t r = ceil_log2_u64(ratio);
    if (r < 1) r = 1;
    const uint32_t levels = (r + log_kmax - 1) / log_kmax;
    uint32_t k = (r + levels - 1) / levels;
    if (k < 1) k = 1;
    if (k > log_kmax) k = log_kmax;
    return k;
}

// Append a segment (and its chunk table) to the next level.  Called by one
// thread.  Returns false on capacity overflow.
__device__ inline bool emit_segment(const LevelBufs& nb, uint64_t off, uint64_t len,
                                    const PlanParams& p) {
    const uint32_t logk = choose_logk(len, p.target, p.log_kmax);
    const uint32_t nch = (uint32_t)((len + p.chunk_elems - 1) / p.chunk_elems);
    const uint32_t s = atomicAdd(&nb.cnt->nsegs, 1u);
    const uint32_t sp = atomicAdd(&nb.cnt->nsplit, 1u << logk);
    const uint32_t c0 = atomicAdd(&nb.cnt->nchunks, nch);
    const uint32_t hb = atomicAdd(&nb.cnt->nhist, nch * (2u << logk));
    if (s >= nb.seg_cap || sp + (1u << logk) > nb.split_cap || c0 + nch > nb.chunk_cap ||
        hb + nch * (2u << logk) > nb.hist_cap) {
        atomicExch(&nb.cnt->overflow, 1u);
        return false;
    }
    SegDesc d;
    d.off = off;
    d.len = len;
    d.chunk_begin = c0;
    d.nchunks = nch;
    d.logk = logk;
    d.m = 0;
    d.eq = 0;
    d.sp = sp;
    d.hist_base = hb;
    d.pad = 0;
    nb.segs[s] = d;
    atomicAdd(&nb.cnt->nkeys, (unsigned long long)len);
    for (uint32_t i = 0; i < nch; ++i) {
        ChunkDesc c;
        c.seg = s;
        c.pad = 0;
        c.begin = off + (uint64_t)i * p.chunk_elems;
        c.end = min(off + len, c.begin + p.chunk_elems);
        nb.chunks[c0 + i] = c;
    }
    return true;
}

__global__ void init_level_kernel(LevelBufs nb, uint64_t n, PlanParams p) {
    if (threadIdx.x == 0 && blockIdx.x == 0) emit_segment(nb, 0, n, p);
}

// Search-tree classification (Eytzinger layout, tree[1..K-1]).  Returns
// 2j + e where j = #{splitters < key} and e = 1 iff three-way mode is on and
// key equals splitter j.
template <class K>
__device__ __forceinline__ uint32_t classify(const K& key, const K* tree, const K* sorted,
                                             uint32_t logk, uint32_t m, uint32_t eq) {
    uint32_t t = 1;
    for (uint32_t l = 0; l < logk; ++l) t = 2 * t + (KeyTraits<K>::lt(tree[t], key) ? 1u : 0u);
    const uint32_t j = t - (1u << logk);
    uint32_t e = 0;
    if (eq && j < m) e = KeyTraits<K>::eq(key, sorted[j]) ? 1u : 0u;
    return 2 * j + e;
}

// ---------------------------------------------------------------------------
// K1: per-segment sample + splitter selection.  One CTA per segment.
// ---------------------------------------------------------------------------
template <class K, int T, int ITEMS>
__global__ void __launch_bounds__(T) sample_kernel(SegDesc* segs, const K* __restrict__ src,
                                                   K* tree_store, K* sorted_store, uint64_t seed) {
    using BS = BlockSorter<K, T, ITEMS>;
    using P = SmemPad<K>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s = reinterpret_cast<K*>(smem_raw);
    __shared__ uint32_t flags[1024 + 1];
    __shared__ uint32_t warp_sums[32];

    const uint32_t seg = blockIdx.x;
    const SegDesc d = segs[seg];
    const uint32_t K_ = 1u << d.logk;

    // Seeded sample with replacement (counter-based SplitMix64 of the sample
    // index; uniform position via a 64x64 high multiply).
    K k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint64_t idx = (uint64_t)threadIdx.x * ITEMS + i;
        const uint64_t h = sm_mix(seed + (d.off + 1) * kGamma + (idx + 1) * 0xD1B54A32D192ED03ull);
        const uint64_t pos = __umul64hi(h, d.len);
        k[i] = src[d.off + pos];
    }
    BS::sort(k, s);  // sorted sample of BS::kCap keys in s (padded)

    // candidate splitter j (0 <= j < K-1): sample quantile (j+1)/K
    const int S = BS::kCap;
    for (uint32_t j = threadIdx.x; j < K_ - 1; j += T) {
        const int q = (int)(((uint64_t)(j + 1) * S) / K_);
        const K c = s[P::idx(q)];
        const bool keep = (j == 0) || !KeyTraits<K>::eq(c, s[P::idx((int)(((uint64_t)j * S) / K_))]);
        flags[j] = keep ? 1u : 0u;
    }
    if (threadIdx.x == 0) flags[K_ - 1] = 0;
    __syncthreads();
    // compact unique splitters (candidates are sorted, so duplicates are adjacent)
    const uint32_t m = block_exclusive_scan_smem<T>(flags, (int)K_, warp_sums);
    K* sorted = sorted_store + d.sp;
    for (uint32_t j = threadIdx.x; j < K_ - 1; j += T) {
        const int q = (int)(((uint64_t)(j + 1) * S) / K_);
        const bool keep = (j + 1 < K_ - 1) ? (flags[j + 1] != flags[j]) : (flags[j] != m);
        if (keep) sorted[flags[j]] = s[P::idx(q)];
    }
    __syncthreads();  // sorted[] (global) is visible block-wide after the barrier
    // Eytzinger tree over sorted[0..m), padded with the maximum key.
    K* tree = tree_store + d.sp;
    for (uint32_t t = threadIdx.x + 1; t < K_; t += T) {
        const uint32_t depth = 31 - __clz(t);
        const uint32_t rank = ((2 * (t - (1u << depth)) + 1) << (d.logk - 1 - depth)) - 1;
        tree[t] = rank < m ? sorted[rank] : KeyTraits<K>::max_key();
    }
    if (threadIdx.x == 0) {
        segs[seg].m = m;
        segs[seg].eq = (m < K_ - 1) ? 1u : 0u;
    }
}

// ---------------------------------------------------------------------------
// K2: per-chunk bucket histogram.
// ---------------------------------------------------------------------------
template <class K, int T, int LOG_KMAX>
__global__ void __launch_bounds__(T) count_kernel(const SegDesc* __restrict__ segs,
                                                  const ChunkDesc* __restrict__ chunks,
                                                  const K* __restrict__ src,
                                                  const K* __restrict__ tree_store,
                                                  const K* __restrict__ sorted_store,
                                                  uint32_t* __restrict__ chunk_hist) {
    constexpr int KMAX = 1 << LOG_KMAX;
    constexpr int NB = 2 * KMAX;
    __shared__ K tree[KMAX];
    __shared__ K sorted[KMAX];
    __shared__ uint32_t hist[NB];
    const ChunkDesc c = chunks[blockIdx.x];
    const SegDesc d = segs[c.seg];
    const uint32_t K_ = 1u << d.logk;
    for (uint32_t i = threadIdx.x; i < K_; i += T) {
        tree[i] = tree_store[d.sp + i];
        sorted[i] = sorted_store[d.sp + i];
    }
    for (uint32_t i = threadIdx.x; i < 2 * K_; i += T) hist[i] = 0;
    __syncthreads();
    constexpr int U = 8;
    uint64_t i = c.begin + threadIdx.x;
    for (; i + (U - 1) * T < c.end; i += U * T) {
        K k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) k[u] = src[i + (uint64_t)u * T];
#pragma unroll
        for (int u = 0; u < U; ++u)
            atomicAdd(&hist[classify<K>(k[u], tree, sorted, d.logk, d.m, d.eq)], 1u);
    }
    for (; i < c.end; i += T)
        atomicAdd(&hist[classify<K>(src[i], tree, sorted, d.logk, d.m, d.eq)], 1u);
    __syncthreads();
    uint32_t* row = chunk_hist + d.hist_base + (size_t)(blockIdx.x - d.chunk_begin) * (2 * K_);
    for (uint32_t b = threadIdx.x; b < 2 * K_; b += T) row[b] = hist[b];
}

// ---------------------------------------------------------------------------
// K3: per-segment plan: totals, bucket starts, per-chunk offsets, children.
// ---------------------------------------------------------------------------
template <class K, int T, int LOG_KMAX>
__global__ void __launch_bounds__(T) plan_kernel(const SegDesc* __restrict__ segs,
                                                 uint32_t* __restrict__ chunk_hist,
                                                 LevelBufs next, PlanParams p,
                                                 SortTask* __restrict__ tasks,
                                                 FillTask* __restrict__ fills,
                                                 LevelCounters* __restrict__ cur_cnt) {
    constexpr int NB = 2 << LOG_KMAX;
    __shared__ uint32_t tot[NB];
    __shared__ uint32_t start[NB];
    __shared__ uint32_t warp_sums[32];
    const uint32_t seg = blockIdx.x;
    const SegDesc d = segs[seg];
    const uint32_t nb = 2u << d.logk;
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        uint32_t sum = 0;
        const uint32_t* col = chunk_hist + d.hist_base + b;
#pragma unroll 8
        for (uint32_t c = 0; c < d.nchunks; ++c) sum += col[(size_t)c * nb];
        tot[b] = sum;
        start[b] = sum;
    }
    __syncthreads();
    block_exclusive_scan_smem<T>(start, (int)nb, warp_sums);
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        uint32_t run = start[b];
        uint32_t* col = chunk_hist + d.hist_base + b;
        for (uint32_t c = 0; c < d.nchunks; ++c) {
            const uint32_t v = col[(size_t)c * nb];
            col[(size_t)c * nb] = run;
            run += v;
        }
        const uint32_t len = tot[b];
        if (len == 0) continue;
        const uint64_t off = d.off + start[b];
        if (b & 1) {  // equal-key bucket: already final when it landed in the caller's buffer
            if (!p.dst_is_a) {
                const uint32_t f = atomicAdd(&cur_cnt->nfill, 1u);
                if (f < p.fill_cap) {
                    FillTask ft;
                    ft.off = off;
                    ft.len = len;
                    ft.seg = seg;
                    ft.j = b >> 1;
                    fills[f] = ft;
                    atomicAdd(&cur_cnt->fill_keys, (unsigned long long)len);
                } else {
                    atomicExch(&cur_cnt->overflow, 1u);
                }
            }
        } else if (len <= p.cap) {
            if (len == 1 && p.dst_is_a) continue;
            int cls = 0;
            while (cls < kNumClasses - 1 && len > p.class_cap[cls]) ++cls;
            const uint32_t t = atomicAdd(&cur_cnt->ntasks[cls], 1u);
            if (t < p.task_cap) {
                SortTask st;
                st.off = off;
                st.len = len;
                st.pad = 0;
                tasks[(size_t)cls * p.task_cap + t] = st;
                atomicAdd(&cur_cnt->task_keys, (unsigned long long)len);
            } else {
                atomicExch(&cur_cnt->overflow, 1u);
            }
        } else {
            emit_segment(next, off, len, p);
        }
    }
}

// ---------------------------------------------------------------------------
// K4: scatter.  Tile = T * ITEMS keys; one CTA walks the tiles of one chunk.
// ---------------------------------------------------------------------------
template <class K, int T, int ITEMS, int LOG_KMAX>
struct ScatterSmem {
    static constexpr int KMAX = 1 << LOG_KMAX;
    static constexpr int NB = 2 * KMAX;
    static constexpr int TILE = T * ITEMS;
    K tree[KMAX];
    K sorted[KMAX];
    K stage[TILE];
    uint16_t stage_bin[TILE];
    uint32_t hist[NB];
    uint32_t start[NB];
    uint64_t gdst[NB];
    uint32_t cursor[NB];
    uint32_t warp_sums[32];
};

template <class K, int T, int ITEMS, int LOG_KMAX>
__global__ void __launch_bounds__(T) scatter_kernel(const SegDesc* __restrict__ segs,
                                                    const ChunkDesc* __restrict__ chunks,
                                                    const K* __restrict__ src, K* __restrict__ dst,
                                                    const K* __restrict__ tree_store,
                                                    const K* __restrict__ sorted_store,
                                                    const uint32_t* __restrict__ chunk_off) {
    using SM = ScatterSmem<K, T, ITEMS, LOG_KMAX>;
    constexpr int TILE = SM::TILE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SM& sm = *reinterpret_cast<SM*>(smem_raw);

    const ChunkDesc c = chunks[blockIdx.x];
    const SegDesc d = segs[c.seg];
    const uint32_t K_ = 1u << d.logk;
    const uint32_t nb = 2 * K_;
    for (uint32_t i = threadIdx.x; i < K_; i += T) {
        sm.tree[i] = tree_store[d.sp + i];
        sm.sorted[i] = sorted_store[d.sp + i];
    }
    const uint32_t* row = chunk_off + d.hist_base + (size_t)(blockIdx.x - d.chunk_begin) * nb;
    for (uint32_t b = threadIdx.x; b < nb; b += T) {
        sm.cursor[b] = row[b];
        sm.hist[b] = 0;
    }
    __syncthreads();

    for (uint64_t t0 = c.begin; t0 < c.end; t0 += TILE) {
        const int m = (int)min((uint64_t)TILE, c.end - t0);
        K k[ITEMS];
        uint32_t bin[ITEMS];
        uint32_t rank[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int li = i * T + threadIdx.x;
            if (li < m) k[i] = src[t0 + li];
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int li = i * T + threadIdx.x;
            if (li < m) {
                bin[i] = classify<K>(k[i], sm.tree, sm.sorted, d.logk, d.m, d.eq);
                rank[i] = atomicAdd(&sm.hist[bin[i]], 1u);
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += T) sm.start[b] = sm.hist[b];
        __syncthreads();
        block_exclusive_scan_smem<T>(sm.start, (int)nb, sm.warp_sums);
        for (uint32_t b = threadIdx.x; b < nb; b += T) {
            const uint32_t h = sm.hist[b];
            sm.gdst[b] = d.off + sm.cursor[b] - sm.start[b];
            sm.cursor[b] += h;
            sm.hist[b] = 0;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int li = i * T + threadIdx.x;
            if (li < m) {
                const uint32_t pos = sm.start[bin[i]] + rank[i];
                sm.stage[pos] = k[i];
                sm.stage_bin[pos] = (uint16_t)bin[i];
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += T) dst[sm.gdst[sm.stage_bin[i]] + i] = sm.stage[i];
        __syncthreads();
    }
}

// Equal-key buckets that landed in the workspace: write the splitter value.
template <class K>
__global__ void fill_kernel(const FillTask* __restrict__ fills, uint32_t nfill,
                            const SegDesc* __restrict__ segs, const K* __restrict__ sorted_store,
                            K* __restrict__ dst) {
    for (uint32_t f = 0; f < nfill; ++f) {
        const FillTask ft = fills[f];
        const K v = sorted_store[segs[ft.seg].sp + ft.j];
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ft.len;
             i += (uint64_t)gridDim.x * blockDim.x)
            dst[ft.off + i] = v;
    }
}

// Block-sort every task of one size class: src -> dst at the same offsets.
template <class K, int T, int ITEMS>
__global__ void __launch_bounds__(T) blocksort_tasks_kernel(const SortTask* __restrict__ tasks,
                                                            const K* src, K* dst) {
    using BS = BlockSorter<K, T, ITEMS>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s = reinterpret_cast<K*>(smem_raw);
    const SortTask t = tasks[blockIdx.x];
    BS::sort_tile(src + t.off, dst + t.off, (int)t.len, s);
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
