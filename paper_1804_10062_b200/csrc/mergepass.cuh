// mergepass.cuh -- K6/K7: merge-path HBM merge passes.
//
// Replaces the upper levels of the reference merge recursion
// (mergesort_with_temp / mergesort_into / swap_merge, merge.hpp:64-135; paper
// Fig. 2).  One pass merges every pair of sorted runs of length `run` into runs
// of 2*run, reading one buffer and writing the other -- the ping-pong through a
// scratch region that the QuickXsort scheme gets from the not-yet-sorted
// partition side.  Each CTA owns T*ITEMS outputs: a warp
// locates the CTA's two merge-path split points with a 32-ary cooperative
// search (a handful of dependent global round trips instead of ~log2(run)),
// the two input slices are staged into shared memory, and the block merges
// them on chip with the same serial merge as the block sort.  Ties take the
// left run first, as swap_merge does (merge.hpp:76).
#pragma once
#include "blocksort.cuh"
#include "common.cuh"

namespace qmsort_b200 {

// Number of elements of A among the first diag outputs of merge(A, B).
// Called by all 32 lanes of a warp; every lane returns the same value.
template <class K>
__device__ __forceinline__ uint64_t merge_path_global_warp(const K* __restrict__ A, uint64_t la,
                                                           const K* __restrict__ B, uint64_t lb,
                                                           uint64_t diag) {
    const int lane = threadIdx.x & 31;
    uint64_t lo = diag > lb ? diag - lb : 0;
    uint64_t hi = diag < la ? diag : la;
    while (lo < hi) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t q = lo + (uint64_t)lane * step;
        bool p = false;
        if (q < hi) p = !KeyTraits<K>::lt(B[diag - 1 - q], A[q]);
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, p));
        const uint64_t nlo = c > 0 ? lo + (uint64_t)(c - 1) * step + 1 : lo;
        const uint64_t nhi = min(hi, lo + (uint64_t)c * step);
        lo = nlo;
        hi = nhi;
    }
    return lo;
}

template <class K, int T, int ITEMS>
__global__ void __launch_bounds__(T) merge_pass_kernel(const K* __restrict__ src,
                                                       K* __restrict__ dst, uint64_t len,
                                                       uint64_t run) {
    using BS = BlockSorter<K, T, ITEMS>;
    using P = SmemPad<K>;
    constexpr int C = BS::kCap;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s = reinterpret_cast<K*>(smem_raw);
    __shared__ uint64_t split[2];

    const uint64_t out0 = (uint64_t)blockIdx.x * C;
    const uint64_t pair = (out0 / (2 * run)) * (2 * run);
    const uint64_t la = min(run, len - pair);
    const uint64_t lb = min(run, len - pair - la);
    const K* A = src + pair;
    const K* B = A + la;
    const uint64_t d0 = out0 - pair;
    const uint64_t d1 = min(d0 + C, la + lb);
    const int wid = threadIdx.x >> 5;
    if (wid < 2) {
        const uint64_t r = merge_path_global_warp<K>(A, la, B, lb, wid == 0 ? d0 : d1);
        if ((threadIdx.x & 31) == 0) split[wid] = r;
    }
    __syncthreads();
    const uint64_t a0 = split[0], a1 = split[1];
    const int na = (int)(a1 - a0);
    const int nb = (int)((d1 - a1) - (d0 - a0));
    const int total = na + nb;
    QCHECK(na >= 0 && nb >= 0 && total <= C, (uint64_t)na, (uint64_t)nb);
    const K* As = A + a0;
    const K* Bs = B + (d0 - a0);
    for (int i = threadIdx.x; i < total; i += T) s[P::idx(i)] = i < na ? As[i] : Bs[i - na];
    __syncthreads();
    K k[ITEMS];
    const int diag = (int)threadIdx.x * ITEMS;
    const bool owner = diag < total;
    if (owner) {
        const int a = merge_path_smem<K>(s, 0, na, na, nb, diag);
        serial_merge_smem<K, ITEMS>(s, a, na, na + diag - a, na + nb, k);
    }
    __syncthreads();
    if (owner) BS::store_blocked(k, s);
    __syncthreads();
    BS::store_striped(dst + pair + d0, total, s);
}

}  // namespace qmsort_b200

#ifndef QMSORT_MERGE_WINDOW
#define QMSORT_MERGE_WINDOW 0  // measured slower (C2 / C3 / C5 merge passes +7-29 %)
#endif
#ifndef QMSORT_MERGE_DIRECT_STORE
#define QMSORT_MERGE_DIRECT_STORE 0  // 16-byte stores from registers instead of the staged write-out
#endif

namespace qmsort_b200 {

// ---------------------------------------------------------------------------
// Blackwell merge pass: split points precomputed by K6a, input slices staged
// by the bulk-copy engine (cp.async.bulk global -> shared, completion counted
// on an mbarrier) into one of two shared-memory buffers while the CTA merges
// the previous tile out of the other -- the copy of tile i+1 overlaps the
// merge and the write-out of tile i.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(mbar)), "r"(count) : "memory");
}
// One arrival that also announces `bytes` of bulk-copy transactions.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(mbar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "QMS_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra QMS_WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(mbar)),
        "r"(phase)
        : "memory");
}
// global [src, src + bytes) -> shared dst; both 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(mbar))
        : "memory");
}
// generic-proxy accesses of shared memory before the async proxy's next write
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// K6a: the merge-path split of every tile start (one thread per tile): the
// number of A elements among the first d outputs of its run pair's merge.
template <class K>
__global__ void merge_split_kernel(const K* __restrict__ src, uint64_t len, uint64_t run, uint64_t C,
                                   uint64_t ntiles, uint64_t* __restrict__ splits) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d0g = t * C;
        const uint64_t pair = d0g / (2 * run) * (2 * run);
        const uint64_t la = min(run, len - pair);
        const uint64_t lb = min(run, len - pair - la);
        const K* A = src + pair;
        const K* B = A + la;
        const uint64_t diag = d0g - pair;
        uint64_t lo = diag > lb ? diag - lb : 0, hi = diag < la ? diag : la;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (KeyTraits<K>::lt(B[diag - 1 - mid], A[mid])) hi = mid;
            else lo = mid + 1;
        }
        splits[t] = lo;
    }
}

template <class K>
struct MergeTile {
    uint64_t pair, d0, d1;   // output range [pair + d0, pair + d1)
    uint64_t a0, a1, b0, b1;  // input slices A[a0, a1), B[b0, b1) of the pair's runs
    const K* A;
    const K* B;
    __device__ __forceinline__ MergeTile(const K* src, uint64_t len, uint64_t run, uint64_t C, uint64_t t,
                                         const uint64_t* splits) {
        const uint64_t d0g = t * C;
        pair = d0g / (2 * run) * (2 * run);
        const uint64_t la = min(run, len - pair);
        const uint64_t lb = min(run, len - pair - la);
        A = src + pair;
        B = A + la;
        d0 = d0g - pair;
        d1 = min(d0 + C, la + lb);
        a0 = splits[t];
        a1 = d1 == la + lb ? la : splits[t + 1];  // tiles never straddle a pair (run % C == 0)
        b0 = d0 - a0;
        b1 = d1 - a1;
    }
};

// One input slice g[0, n).  The bulk-copy engine moves whole 16-byte
// blocks, so the copy covers [floor16(g), ceil16(g + n)) -- a few keys of the
// neighbouring slice on either side, harmless -- whenever that stays inside
// the array [lo_bound, hi_bound); at the array's ends the partial blocks are
// plain loads instead (and every key is, for 8-byte-aligned records).
template <class K>
struct Slice {
    uint64_t h, tl;  // plain-loaded head [0, h) and tail [tl, n)
    uint32_t bytes;  // bulk-copied bytes, starting at element `first` (may be < 0: over-read)
    int32_t first;
    uint32_t lead;   // g's address mod 16: the slice lands at the same offset mod 16
    __device__ __forceinline__ Slice(const K* g, uint64_t n, const K* lo_bound, const K* hi_bound) {
        const uintptr_t ga = reinterpret_cast<uintptr_t>(g), ge = ga + n * sizeof(K);
        const uintptr_t lo = ga & ~(uintptr_t)15, hi = (ge + 15) & ~(uintptr_t)15;
        lead = (uint32_t)(ga & 15u);
        h = tl = n;
        bytes = 0;
        first = 0;
        if (n == 0 || lead % sizeof(K) != 0) {  // nothing to move / records 8 bytes off
            lead = 0;
            return;
        }
        // the bulk range [blo, bhi): over-read where the array allows, else shrink to the interior
        const uintptr_t blo = lo >= reinterpret_cast<uintptr_t>(lo_bound) ? lo : (ga + 15) & ~(uintptr_t)15;
        const uintptr_t bhi = hi <= reinterpret_cast<uintptr_t>(hi_bound) ? hi : ge & ~(uintptr_t)15;
        if (blo >= bhi || (bhi - ga) % sizeof(K) != 0) return;  // all plain loads
        first = (int32_t)(((intptr_t)blo - (intptr_t)ga) / (intptr_t)sizeof(K));
        h = first > 0 ? (uint64_t)first : 0;
        tl = min(n, (uint64_t)((bhi - ga) / sizeof(K)));
        bytes = (uint32_t)(bhi - blo);
    }
    // room before the slice for an over-read head, a whole number of keys
    static constexpr uint32_t kRoom = sizeof(K) > 16 ? (uint32_t)sizeof(K) : 16u;
    // plain loads of head and tail, the bulk copy (one thread)
    __device__ __forceinline__ void stage(const K* g, uint64_t n, unsigned char* dst, uint64_t* mbar) const {
        K* s = reinterpret_cast<K*>(dst + kRoom + lead);
        for (uint64_t i = 0; i < h; ++i) s[i] = g[i];
        for (uint64_t i = tl; i < n; ++i) s[i] = g[i];
        if (bytes) bulk_g2s(s + first, g + first, bytes, mbar);
    }
    __device__ __forceinline__ uint32_t offset() const { return (kRoom + lead) / sizeof(K); }  // element of g[0]
};

template <class K, int T, int ITEMS>
struct BulkMerge {
    static constexpr int C = T * ITEMS;
    // one stage: A slice + B slice, each with up to 16 bytes of alignment slack
    static constexpr size_t kInBytes = (size_t)C * sizeof(K) + 256;
    // the write-out reuses the stage in the block sorter's padded layout
    static constexpr size_t kStageBytes =
        ((kInBytes > sizeof(K) * SmemPad<K>::elems(C) ? kInBytes : sizeof(K) * SmemPad<K>::elems(C)) + 127) / 128 * 128;
    static constexpr size_t kSmemBytes = 2 * kStageBytes;
};

// K6b: persistent CTAs walk the tiles t = blockIdx.x, + gridDim.x, ...
template <class K, int T, int ITEMS>
__global__ void __launch_bounds__(T) merge_pass_bulk_kernel(const K* __restrict__ src, K* __restrict__ dst,
                                                            uint64_t len, uint64_t run,
                                                            const uint64_t* __restrict__ splits,
                                                            uint64_t ntiles) {
    using BM = BulkMerge<K, T, ITEMS>;
    using BS = BlockSorter<K, T, ITEMS>;
    constexpr int C = BM::C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint32_t s_off[2][2];  // element offsets of the A and B slices in each stage
    unsigned char* stage[2] = {smem_raw, smem_raw + BM::kStageBytes};
    const uint64_t first = blockIdx.x;
    if (first >= ntiles) return;
    const K* src_end = src + len;
    auto issue = [&](uint64_t t, int b) {  // one thread: stage tile t into buffer b
        const MergeTile<K> g(src, len, run, C, t, splits);
        const uint64_t na = g.a1 - g.a0, nb = g.b1 - g.b0;
        const Slice<K> sa(g.A + g.a0, na, src, src_end), sb(g.B + g.b0, nb, src, src_end);
        // B's slice region starts after A's (rounded to 16 bytes and to whole keys)
        constexpr uint32_t kAl = sizeof(K) > 16 ? (uint32_t)sizeof(K) : 16u;
        const uint32_t bbyte = (uint32_t)((Slice<K>::kRoom + sa.lead + na * sizeof(K) + 16 + kAl - 1) / kAl * kAl);
        mbar_arrive_expect_tx(&mbar[b], sa.bytes + sb.bytes);  // announce, then start the copies
        sa.stage(g.A + g.a0, na, stage[b], &mbar[b]);
        sb.stage(g.B + g.b0, nb, stage[b] + bbyte, &mbar[b]);
        s_off[b][0] = sa.offset();
        s_off[b][1] = bbyte / sizeof(K) + sb.offset();
    };
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        issue(first, 0);
        if (first + gridDim.x < ntiles) issue(first + gridDim.x, 1);
    }
    uint32_t phase[2] = {0, 0};
    int b = 0;
    for (uint64_t t = first; t < ntiles; t += gridDim.x, b ^= 1) {
        const MergeTile<K> g(src, len, run, C, t, splits);
        mbar_wait(&mbar[b], phase[b]);
        phase[b] ^= 1;
        __syncthreads();  // the plain-load head/tail elements of thread 0 are visible too
        const K* s = reinterpret_cast<const K*>(stage[b]);
        const int na = (int)(g.a1 - g.a0), nb = (int)(g.b1 - g.b0);
        const int oa = (int)s_off[b][0], ob = (int)s_off[b][1];
        QCHECK(na >= 0 && nb >= 0 && na + nb <= C, (uint64_t)na, (uint64_t)nb);
        const int total = na + nb;
        K k[ITEMS];
        const int diag = (int)threadIdx.x * ITEMS;
        const bool owner = diag < total;
        if (owner) {
            // merge path over the dense slices: A at s[oa, oa+na), B at s[ob, ob+nb)
            const int a = merge_path_smem<K, NoPad>(s, oa, na, ob, nb, diag);
            if (QMSORT_MERGE_WINDOW && diag + ITEMS <= total) {  // no serial chain
                const int a_end = merge_path_smem<K, NoPad>(s, oa, na, ob, nb, diag + ITEMS);
                bitonic_merge_window<K, ITEMS, NoPad>(s, oa + a, a_end - a, ob + diag - a, k);
            } else {
                serial_merge_smem<K, ITEMS, NoPad>(s, oa + a, oa + na, ob + diag - a, ob + nb, k);
            }
        }
        K* out = dst + g.pair + g.d0;
        if (QMSORT_MERGE_DIRECT_STORE && total == C && (reinterpret_cast<uintptr_t>(out) & 15u) == 0 &&
            (ITEMS * sizeof(K)) % 16 == 0) {
            // full tile: each thread's ITEMS consecutive outputs as 16-byte stores
            // straight from registers (no staging, no barrier)
            constexpr int NV = ITEMS * (int)sizeof(K) / 16;  // 16-byte vectors per thread
            uint4* o = reinterpret_cast<uint4*>(out + diag);
            const unsigned char* kb = reinterpret_cast<const unsigned char*>(k);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                uint4 x;
                memcpy(&x, kb + 16 * v, 16);
                o[v] = x;
            }
            __syncthreads();  // every merge has read the stage: it is free again
        } else {
            __syncthreads();  // every merge has read the stage
            K* w = reinterpret_cast<K*>(stage[b]);
            if (owner) BS::store_blocked(k, w);
            __syncthreads();
            BS::store_striped(out, total, w);
            __syncthreads();  // the stage is free again
        }
        if (threadIdx.x == T - 32 && t + 2 * (uint64_t)gridDim.x < ntiles) {  // the last warp issues
            fence_proxy_async_smem();  // generic-proxy reads/writes before the bulk copy's writes
            issue(t + 2 * (uint64_t)gridDim.x, b);
        }
    }
}

}  // namespace qmsort_b200
