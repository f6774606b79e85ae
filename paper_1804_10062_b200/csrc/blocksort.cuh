// blocksort.cuh -- K5: shared-memory block sort of register-resident tiles.
//
// Replaces the reference's base case X (small_sort / insertion_sort /
// clever_quicksort, reference small_sort.hpp:13-111, clever.hpp:21-53) and the
// bottom levels of the merge recursion (mergesort_into, merge.hpp:103-119):
// instead of handing blocks below 10 elements to a straight-line sorter, every
// bucket that fits one CTA is sorted entirely on chip:
//   1. each thread sorts ITEMS keys in registers with Batcher's odd-even merge
//      network (compile-time unrolled, no local memory);
//      uint32 tiles whose keys span fewer than 2^16 - 1 values take this and
//      the warp rounds with two 16-bit keys per register (key - min, U16x2:
//      VIMNMX.U16x2 compare-and-swaps, one shuffle per two keys);
//   2. log2(T) merge-path rounds in shared memory double the run length; each
//      thread locates its output diagonal by binary search (merge path) and
//      merges ITEMS outputs serially -- the same "take run1 on ties" rule as
//      swap_merge (merge.hpp:76), so the merge is stable.
// The tile is loaded once from HBM and written once (2 n w bytes per pass).
#pragma once
#include <type_traits>
#include <utility>

#include "common.cuh"

#ifndef QMSORT_SELECT_PRED
#define QMSORT_SELECT_PRED 1
#endif
// the packed path's five warp rounds fully unrolled (compile-time shuffle
// distances and lane masks)
#ifndef QMSORT_UNROLL_WARP_ROUNDS
#define QMSORT_UNROLL_WARP_ROUNDS 0
#endif

#ifndef QMSORT_SELECT_PRED16
#define QMSORT_SELECT_PRED16 0
#endif

namespace qmsort_b200 {

// Batcher odd-even merge sort network on N register-resident keys.  The
// comparator list is computed at compile time and applied through a fold
// expression, so every register index is a constant (no local memory).
template <int N>
struct OddEvenNet {
    static constexpr int count() {
        int c = 0;
        for (int p = 1; p < N; p <<= 1)
            for (int q = p; q >= 1; q >>= 1)
                for (int j = q % p; j + q < N; j += 2 * q)
                    for (int i = 0; i < q; ++i)
                        if (i + j + q < N && (i + j) / (2 * p) == (i + j + q) / (2 * p)) ++c;
        return c;
    }
    static constexpr int kCount = count();
    struct Pairs {
        int a[kCount > 0 ? kCount : 1];
        int b[kCount > 0 ? kCount : 1];
    };
    static constexpr Pairs make() {
        Pairs r{};
        int c = 0;
        for (int p = 1; p < N; p <<= 1)
            for (int q = p; q >= 1; q >>= 1)
                for (int j = q % p; j + q < N; j += 2 * q)
                    for (int i = 0; i < q; ++i)
                        if (i + j + q < N && (i + j) / (2 * p) == (i + j + q) / (2 * p)) {
                            r.a[c] = i + j;
                            r.b[c] = i + j + q;
                            ++c;
                        }
        return r;
    }
    static constexpr Pairs kPairs = make();
};

// Network compare-and-swaps finish on the FMA pipe (KeyTraits<K>::cas_alt:
// the maximum's words by IMADs), relieving the ALU pipe the kernel is bound by.
template <class K>
__device__ __forceinline__ void net_cas(K& a, K& b, int) {
    KeyTraits<K>::cas_alt(a, b);
}

template <class K, int N, size_t... I>
__device__ __forceinline__ void apply_net(K (&k)[N], std::index_sequence<I...>) {
    (net_cas<K>(k[OddEvenNet<N>::kPairs.a[I]], k[OddEvenNet<N>::kPairs.b[I]], (int)I), ...);
}

template <class K, int N>
__device__ __forceinline__ void register_sort(K (&k)[N]) {
    if constexpr (OddEvenNet<N>::kCount > 0)
        apply_net<K, N>(k, std::make_index_sequence<OddEvenNet<N>::kCount>{});
}

// Merge-path split on shared memory: the number of elements taken from run A
// among the first `diag` outputs of merge(A, B) when ties take A first.
// Shared-memory index maps: SmemPad<K> (one pad word per bank row, the block
// sorter) or NoPad (dense, where the bulk-copy engine wrote the keys).
struct NoPad {
    __device__ __forceinline__ static unsigned idx(unsigned i) { return i; }
};

template <class K, class P = SmemPad<K>>
__device__ __forceinline__ int merge_path_smem(const K* s, int a0, int alen, int b0, int blen,
                                               int diag) {
    unsigned lo = diag > blen ? (unsigned)(diag - blen) : 0u;
    unsigned hi = diag < alen ? (unsigned)diag : (unsigned)alen;
    const unsigned bd = (unsigned)(b0 + diag - 1);
    while (lo < hi) {
        const unsigned mid = (lo + hi) >> 1;
        // A[mid] goes first unless B[diag-1-mid] < A[mid]
        const bool a_first = !KeyTraits<K>::lt(s[P::idx(bd - mid)], s[P::idx((unsigned)a0 + mid)]);
        lo = a_first ? mid + 1 : lo;
        hi = a_first ? hi : mid;
    }
    return (int)lo;
}

// Serially merge ITEMS outputs from positions ai (run A, ends at aend) and bi
// (run B, ends at bend) of shared memory into registers.  Branch-free: an
// exhausted run reads as the maximum key, which is also exactly what any
// remaining keys of the other run equal when a tie with it takes run A.
template <class K, int ITEMS, class P = SmemPad<K>>
__device__ __forceinline__ void serial_merge_smem(const K* s, int ai, int aend, int bi, int bend,
                                                  K (&out)[ITEMS]) {
    using KT = KeyTraits<K>;
    K ka = ai < aend ? s[P::idx((unsigned)ai)] : KT::max_key();
    K kb = bi < bend ? s[P::idx((unsigned)bi)] : KT::max_key();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool tb = KT::lt(kb, ka);
        out[i] = tb ? kb : ka;
        ai += tb ? 0 : 1;
        bi += tb ? 1 : 0;
        const int ni = tb ? bi : ai;
        const int ne = tb ? bend : aend;
        K v = s[P::idx((unsigned)ni)];  // at most ITEMS slots past a run end: inside the slack
        v = ni < ne ? v : KT::max_key();
        ka = tb ? ka : v;
        kb = tb ? v : kb;
    }
}

// The same ITEMS outputs without a serial dependency chain: the thread's
// window is A[ai, ai+x) (ascending) and B[bi, bi+ITEMS-x) (also ascending,
// loaded reversed), i.e. a bitonic sequence, which a log2(ITEMS)-stage
// half-cleaner network sorts in registers.  All loads are independent, and the
// compare-and-swaps split over the ALU and FMA pipes (net_cas).  Keys only: the
// output equals the serial merge's (equal keys are indistinguishable).
template <class K, int ITEMS, class P = SmemPad<K>>
__device__ __forceinline__ void bitonic_merge_window(const K* s, int ai, int x, int bi, K (&out)[ITEMS]);

// min (lower = true) or max of a and b.
template <class K>
__device__ __forceinline__ K select_minmax(const K& a, const K& b, bool lower) {
    if constexpr (std::is_same<K, uint32_t>::value && QMSORT_SELECT_PRED) {
        return lower ? min(a, b) : max(a, b);  // two predicated VIMNMX
    } else {
        const bool b_less = KeyTraits<K>::lt(b, a);
        return (b_less == lower) ? b : a;
    }
}

// Two 16-bit keys in one register: the halves are two independent sequences
// that every network step below treats alike (SIMD within a register).  A
// compare-and-swap is one VIMNMX.U16x2 plus the two-IMAD maximum (the halves'
// a + b - min cannot carry: each half's result is that half's maximum), a
// shuffle moves two keys.  Used by the block sorter for tiles whose keys span
// at most 2^16 values (keys stored as key - min).
struct U16x2 {
    uint32_t v;
};
template <>
struct KeyTraits<U16x2> {
    __device__ __forceinline__ static void cas_alt(U16x2& a, U16x2& b) {
        const uint32_t lo = __vminu2(a.v, b.v);
        const uint32_t t = lo * c_neg1 + a.v;
        b.v = t * c_one + b.v;
        a.v = lo;
    }
    __device__ __forceinline__ static U16x2 shfl_xor(U16x2 a, int m) {
        return U16x2{__shfl_xor_sync(0xffffffffu, a.v, m)};
    }
};
// min or max of both halves, chosen per lane: both min and max and one LOP3
// (three issue slots).  QMSORT_SELECT_PRED16: `lower ? vmin : vmax`, which
// ptxas emits as two predicated VIMNMX.U16x2 -- measured slower in the packed
// block sort (C2: 1683 against 1640 us), while the unpacked uint32 select
// (QMSORT_SELECT_PRED) gains (C2 sample kernel 146 -> 130 us).
__device__ __forceinline__ U16x2 select_minmax(const U16x2& a, const U16x2& b, bool lower) {
#if QMSORT_SELECT_PRED16
    return U16x2{lower ? __vminu2(a.v, b.v) : __vmaxu2(a.v, b.v)};
#else
    const uint32_t msk = 0u - (uint32_t)lower;
    const uint32_t mn = __vminu2(a.v, b.v), mx = __vmaxu2(a.v, b.v);
    return U16x2{(mn & msk) | (mx & ~msk)};
#endif
}

// One warp-level merge round: every pair of ascending runs of `lr` lanes x
// ITEMS keys (lane-blocked) becomes one ascending run of 2*lr lanes.  Bitonic
// merge in its all-ascending form: a flip stage pairs position p with its
// mirror p ^ (2*lr*ITEMS - 1), then half-cleaners at distances lr*ITEMS/2 ..
// 1.  Cross-lane distances use register shuffles, in-lane distances plain
// compare-and-swap; no shared memory and no barriers.
template <class K, int ITEMS>
__device__ __forceinline__ void warp_merge_round(K (&k)[ITEMS], int lr) {
    using KT = KeyTraits<K>;
    const int lane = threadIdx.x & 31;
    {
        const int fm = 2 * lr - 1;
        const bool lower = (lane & lr) == 0;
        if constexpr (ITEMS == 1) {
            k[0] = select_minmax(k[0], KT::shfl_xor(k[0], fm), lower);
        } else {
#pragma unroll
            for (int j = 0; j < ITEMS / 2; ++j) {
                const K y0 = KT::shfl_xor(k[ITEMS - 1 - j], fm);
                const K y1 = KT::shfl_xor(k[j], fm);
                k[j] = select_minmax(k[j], y0, lower);
                k[ITEMS - 1 - j] = select_minmax(k[ITEMS - 1 - j], y1, lower);
            }
        }
    }
#if QMSORT_UNROLL_WARP_ROUNDS
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int s = lr >> 1; s >= 1; s >>= 1) {
        const bool lower = (lane & s) == 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) k[j] = select_minmax(k[j], KT::shfl_xor(k[j], s), lower);
    }
#pragma unroll
    for (int s = ITEMS / 2; s >= 1; s >>= 1) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
            if ((j & s) == 0) net_cas<K>(k[j], k[j + s], j + s);
    }
}

template <class K, int ITEMS, class P>
__device__ __forceinline__ void bitonic_merge_window(const K* s, int ai, int x, int bi, K (&out)[ITEMS]) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int idx = i < x ? ai + i : bi + (ITEMS - 1 - i);
        out[i] = s[P::idx((unsigned)idx)];
    }
#pragma unroll
    for (int st = ITEMS / 2; st >= 1; st >>= 1) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
            if ((j & st) == 0) net_cas<K>(out[j], out[j + st], j + st);
    }
}

// Sort the 32*ITEMS keys of a warp (lane-blocked: lane l ends up holding
// positions l*ITEMS .. l*ITEMS+ITEMS-1 of the ascending order).
template <class K, int ITEMS>
__device__ __forceinline__ void warp_sort(K (&k)[ITEMS]) {
    register_sort<K, ITEMS>(k);
#pragma unroll 1
    for (int lr = 1; lr < 32; lr <<= 1) warp_merge_round<K, ITEMS>(k, lr);
}

template <class K, int T, int ITEMS>
struct BlockSorter {
    static constexpr int kThreads = T;
    static constexpr int kItems = ITEMS;
    static constexpr int kCap = T * ITEMS;
    static constexpr int kSmemElems = SmemPad<K>::elems(kCap);
    // records (Rec32) first try the prefix path: the tile unpadded plus a
    // padded array of 64-bit (prefix | index) keys
    static constexpr bool kPrefixPath = std::is_same<K, Rec32>::value && kCap <= 4096;
    static constexpr size_t kPrefixSmemBytes =
        kPrefixPath ? (size_t)kCap * sizeof(K) + sizeof(uint64_t) * SmemPad<uint64_t>::elems(kCap) : 0;
    static constexpr size_t kSmemBytes =
        sizeof(K) * kSmemElems > kPrefixSmemBytes ? sizeof(K) * kSmemElems : kPrefixSmemBytes;
    using P = SmemPad<K>;
    using KT = KeyTraits<K>;

    // Lanes merged by the register-shuffle rounds before the shared-memory
    // merge-path rounds take over (measured: all 32 for 4-byte keys; 8 for
    // 8- and 32-byte keys, whose shuffles move 2 or 8 words per key).
    static constexpr int kWarpLanes = sizeof(K) >= 8 ? 8 : 32;
    // merge-path rounds: bitonic window merge (no serial chain) for records,
    // serial merge otherwise (measured: the window merge is not faster for
    // 4-byte keys)
    static constexpr bool kWindow = sizeof(K) > 8;

    // Keys rounded up to whole threads: threads at or beyond mp / ITEMS own
    // no keys and only take part in the barriers.
    __device__ __forceinline__ static int padded(int m) { return (m + ITEMS - 1) / ITEMS * ITEMS; }
    // Keys rounded up to whole warps (the warp-level rounds need all lanes).
    static constexpr int kWarpKeys = 32 * ITEMS;
    __device__ __forceinline__ static int warp_padded(int m) {
        const int w = (m + kWarpKeys - 1) / kWarpKeys * kWarpKeys;
        return w < kCap ? w : kCap;
    }

    // Coalesced (striped) load of m <= kCap keys into shared memory, padding
    // up to a whole warp with the maximum key.
    __device__ __forceinline__ static void load_striped(const K* __restrict__ src, int m, K* s) {
        const int mw = warp_padded(m);
#pragma unroll 4
        for (int i = threadIdx.x; i < mw; i += T) s[P::idx(i)] = i < m ? src[i] : KT::max_key();
    }
    __device__ __forceinline__ static void store_blocked(const K (&k)[ITEMS], K* s) {
        const int base = threadIdx.x * ITEMS;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) s[P::idx(base + i)] = k[i];
    }
    __device__ __forceinline__ static void load_blocked(K (&k)[ITEMS], const K* s) {
        const int base = threadIdx.x * ITEMS;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) k[i] = s[P::idx(base + i)];
    }
    __device__ __forceinline__ static void store_striped(K* __restrict__ dst, int m, const K* s,
                                                         const Xf& xf = Xf{0, 0}) {
#pragma unroll 4
        for (int i = threadIdx.x; i < m; i += T) dst[i] = xf_inv(s[P::idx(i)], xf);
    }

    // Sort the first m keys held in registers (blocked arrangement; the last
    // owning thread is padded with the maximum key).  Cost scales with m:
    // ceil(log2(m / ITEMS)) merge rounds over the owning threads only.  On
    // return the sorted keys sit in shared memory s (padded indexing).  Must
    // be called by all T threads; s must not be in use.
    __device__ __forceinline__ static void sort(K (&k)[ITEMS], K* s, int m) {
        const int mp = padded(m);
        const int out = threadIdx.x * ITEMS;
        const bool owner = out < mp;
        // warps holding any key (their other lanes hold maximum-key padding)
        const bool warp_active = (int)(threadIdx.x & ~31u) * ITEMS < mp;
        if (warp_active) {
            register_sort<K, ITEMS>(k);
#pragma unroll 1
            for (int lr = 1; lr < kWarpLanes && lr * ITEMS < mp; lr <<= 1) warp_merge_round<K, ITEMS>(k, lr);
        }
#pragma unroll 1
        for (int run = kWarpLanes * ITEMS; run < mp; run <<= 1) {
            if (owner) store_blocked(k, s);
            __syncthreads();
            if (owner) merge_step(k, s, mp, out, run);
            __syncthreads();
        }
        if (owner) store_blocked(k, s);
        __syncthreads();
    }

    // One merge-path round for the thread whose outputs start at `out`: runs of
    // `run` keys in s (padded indexing) pairwise into k.
    __device__ __forceinline__ static void merge_step(K (&k)[ITEMS], const K* s, int mp, int out, int run) {
        const int pair = out & ~(2 * run - 1);
        const int diag = out - pair;
        const int a0 = pair, b0 = pair + run;
        const int alen = min(run, mp - a0);
        const int blen = max(0, min(run, mp - b0));
        const int a = merge_path_smem<K>(s, a0, alen, b0, blen, diag);
        if constexpr (kWindow) {  // records: the wide serial merge is select-heavy
            const int a_end = merge_path_smem<K>(s, a0, alen, b0, blen, diag + ITEMS);
            bitonic_merge_window<K, ITEMS>(s, a0 + a, a_end - a, b0 + diag - a, k);
        } else {
            serial_merge_smem<K, ITEMS>(s, a0 + a, a0 + alen, b0 + diag - a, b0 + blen, k);
        }
    }

    // Merge-path rounds in shared memory from sorted runs of run0 keys up to
    // the whole tile; the result is left in s.  in_smem: the runs are already
    // in s (padded indexing) rather than in the threads' registers.
    __device__ __forceinline__ static void merge_rounds(K (&k)[ITEMS], K* s, int m, int run0, bool in_smem) {
        const int mp = padded(m);
        const int out = threadIdx.x * ITEMS;
        const bool owner = out < mp;
#pragma unroll 1
        for (int run = run0; run < mp; run <<= 1) {
            if (owner && !in_smem) store_blocked(k, s);
            in_smem = false;
            __syncthreads();
            if (owner) merge_step(k, s, mp, out, run);
            __syncthreads();
        }
        if (owner && !in_smem) store_blocked(k, s);
        __syncthreads();
    }

    // Records: sort 64-bit keys (p & ~0xFFF) | i instead of the records, where
    // p is the top 64 bits of the (w0 - min w0, w1) pair over the tile -- a
    // monotone map of the lexicographic order -- and i the record's index in
    // the tile.  If no two keys share their top 52 bits the key order is the
    // record order, and one gather from shared memory writes the sorted tile;
    // otherwise (ties in the prefix) returns false with nothing written and
    // the caller sorts the records themselves.  The uint64 sorter's compare-
    // and-swaps are a few instructions where a record's is ~30.
    __device__ static bool sort_tile_prefix(const K* src, K* dst, int m, K* s, const Xf& xf) {
        using B64 = BlockSorter<uint64_t, T, ITEMS>;
        using P8 = SmemPad<uint64_t>;
        __shared__ unsigned long long red_lo[T / 32], red_hi[T / 32];
        K* rec = s;
        uint64_t* s64 = reinterpret_cast<uint64_t*>(s + kCap);
        const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
        uint64_t w0[ITEMS], w1[ITEMS];
        unsigned long long lo = ~0ull, hi = 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int i = j * T + tid;
            w0[j] = w1[j] = 0;
            if (i < m) {
                const K r = src[i];
                rec[i] = r;
                w0[j] = r.w[0];
                w1[j] = r.w[1];
                lo = min(lo, (unsigned long long)r.w[0]);
                hi = max(hi, (unsigned long long)r.w[0]);
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            red_lo[wid] = lo;
            red_hi[wid] = hi;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < T / 32; ++w) {
            lo = min(lo, red_lo[w]);
            hi = max(hi, red_hi[w]);
        }
        const uint64_t span = hi - lo;
        const int sh = span ? __clzll((long long)span) : 64;  // w1 bits in the prefix
        const int mw = B64::warp_padded(m);
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int i = j * T + tid;
            const uint64_t d = w0[j] - lo;
            const uint64_t p = sh == 64 ? w1[j] : sh == 0 ? d : (d << sh) | (w1[j] >> (64 - sh));
            if (i < mw) s64[P8::idx(i)] = i < m ? (p & ~0xFFFull) | (uint64_t)i : ~0ull;
        }
        __syncthreads();
        uint64_t k[ITEMS];
        if (tid * ITEMS < mw) B64::load_blocked(k, s64);
        __syncthreads();
        B64::sort(k, s64, m);
        int tie = 0;
        for (int i = tid; i + 1 < m; i += T)
            tie |= ((s64[P8::idx(i)] ^ s64[P8::idx(i + 1)]) >> 12) == 0 ? 1 : 0;
        if (__syncthreads_or(tie)) return false;
        for (int i = tid; i < m; i += T) dst[i] = xf_inv(rec[s64[P8::idx(i)] & 0xFFFull], xf);
        return true;
    }

    // uint32 tiles whose keys span < 2^16 - 1 values: the key - min values are
    // sorted two per register (U16x2) through the register network and the
    // warp rounds -- about half the instructions per key -- then unpacked into
    // shared memory for the merge-path rounds.  Warp w's 1024 keys: register
    // j of lane l holds positions w*1024 + l*16 + j (low half) and the same
    // + 512 (high half).  Each half is sorted as a 512-key warp run, then one
    // cross-half round (flip stage: low position p against high position
    // 511 - p, then the half-cleaners of both halves) leaves the low halves
    // holding the warp's 512 smallest keys in order and the high halves the
    // rest: a sorted run of 1024, as the unpacked warp stage produces.
    static constexpr bool kPackedPath = std::is_same<K, uint32_t>::value && ITEMS == 32;
    static constexpr int kPI = ITEMS / 2;  // packed registers per lane
    template <int NPI>
    __device__ __forceinline__ static void cross_half_round(U16x2 (&pk)[NPI]) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < NPI / 2; ++j) {
            const int jj = NPI - 1 - j;
            const uint32_t y0 = __shfl_xor_sync(0xffffffffu, pk[jj].v, 31);
            const uint32_t y1 = __shfl_xor_sync(0xffffffffu, pk[j].v, 31);
            const uint32_t s0 = __byte_perm(y0, 0, 0x1032), s1 = __byte_perm(y1, 0, 0x1032);  // swap halves
            pk[j].v = (__vminu2(pk[j].v, s0) & 0xFFFFu) | (__vmaxu2(pk[j].v, s0) & 0xFFFF0000u);
            pk[jj].v = (__vminu2(pk[jj].v, s1) & 0xFFFFu) | (__vmaxu2(pk[jj].v, s1) & 0xFFFF0000u);
        }
#pragma unroll
        for (int sd = 16; sd >= 1; sd >>= 1) {
            const bool lower = (lane & sd) == 0;
#pragma unroll
            for (int j = 0; j < NPI; ++j) pk[j] = select_minmax(pk[j], KeyTraits<U16x2>::shfl_xor(pk[j], sd), lower);
        }
#pragma unroll
        for (int sd = NPI / 2; sd >= 1; sd >>= 1) {
#pragma unroll
            for (int j = 0; j < NPI; ++j)
                if ((j & sd) == 0) net_cas<U16x2>(pk[j], pk[j + sd], j + sd);
        }
    }
    // One warp sorts positions [wb, wb + 64 NPI) of s (keys - lo, two per
    // register) into a sorted run; positions past the warp's span up to its
    // 32 ITEMS slots get the maximum key.
    template <int NPI>
    __device__ __forceinline__ static void packed_warp_sort(K* s, int m, uint32_t lo, int wb) {
        const int base = wb + (int)(threadIdx.x & 31) * NPI;
        U16x2 pk[NPI];
#pragma unroll
        for (int j = 0; j < NPI; ++j) {
            const int p0 = base + j, p1 = p0 + 32 * NPI;
            const uint32_t k0 = p0 < m ? s[P::idx(p0)] - lo : 0xFFFFu;
            const uint32_t k1 = p1 < m ? s[P::idx(p1)] - lo : 0xFFFFu;
            pk[j].v = k0 | (k1 << 16);
        }
        register_sort<U16x2, NPI>(pk);
#if QMSORT_UNROLL_WARP_ROUNDS
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int lr = 1; lr < 32; lr <<= 1) warp_merge_round<U16x2, NPI>(pk, lr);
        cross_half_round<NPI>(pk);
        // each warp reads and writes only its own positions
#pragma unroll
        for (int j = 0; j < NPI; ++j) {
            const int p0 = base + j;
            const uint32_t v0 = pk[j].v & 0xFFFFu, v1 = pk[j].v >> 16;
            s[P::idx(p0)] = v0 == 0xFFFFu ? KT::max_key() : v0 + lo;  // 0xFFFF: padding only
            s[P::idx(p0 + 32 * NPI)] = v1 == 0xFFFFu ? KT::max_key() : v1 + lo;
        }
        if constexpr (NPI < kPI) {  // the rest of the warp's run: padding
            for (int i = wb + 64 * NPI + (int)(threadIdx.x & 31); i < wb + 32 * ITEMS; i += 32)
                s[P::idx(i)] = KT::max_key();
        }
    }
    __device__ __forceinline__ static void sort_tile_packed(K* s, int m, uint32_t lo) {
        const int wb = (int)(threadIdx.x & ~31u) * ITEMS;  // the warp's first position
        // (a tail warp holding at most half its span sorting it with half the
        // registers, packed_warp_sort<kPI / 2>, measured slower: block sort
        // 1627 -> 1750 us on C2 -- the second instantiation of the unrolled
        // network and warp rounds in one kernel)
        if (wb < m) packed_warp_sort<kPI>(s, m, lo, wb);  // warps holding keys
        K k[ITEMS];
        merge_rounds(k, s, m, 32 * ITEMS, true);
    }

    // Whole tile: global src (m keys) -> sorted -> global dst.  src may alias dst.
    // xf: the inverse order-preserving transform is applied on the way out.
    __device__ __forceinline__ static void sort_tile(const K* src, K* dst, int m, K* s,
                                                     const Xf& xf = Xf{0, 0}) {
        if constexpr (kPrefixPath) {
            if (m > 1 && sort_tile_prefix(src, dst, m, s, xf)) return;
        }
        if constexpr (kPackedPath) {
            // striped load with the tile's key range
            __shared__ uint32_t red_lo[T / 32], red_hi[T / 32];
            const int mw = warp_padded(m);
            uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll 4
            for (int i = threadIdx.x; i < mw; i += T) {
                const K x = i < m ? src[i] : KT::max_key();
                s[P::idx(i)] = x;
                if (i < m) {
                    lo = min(lo, x);
                    hi = max(hi, x);
                }
            }
            lo = __reduce_min_sync(0xffffffffu, lo);
            hi = __reduce_max_sync(0xffffffffu, hi);
            if ((threadIdx.x & 31) == 0) {
                red_lo[threadIdx.x >> 5] = lo;
                red_hi[threadIdx.x >> 5] = hi;
            }
            __syncthreads();
#pragma unroll
            for (int w = 0; w < T / 32; ++w) {
                lo = min(lo, red_lo[w]);
                hi = max(hi, red_hi[w]);
            }
            if (m > 1 && hi - lo < 0xFFFFu) {  // 0xFFFF is reserved for padding
                sort_tile_packed(s, m, lo);
                store_striped(dst, m, s, xf);
                return;
            }
        } else {
            load_striped(src, m, s);
        }
        __syncthreads();
        K k[ITEMS];
        if ((int)threadIdx.x * ITEMS < warp_padded(m)) load_blocked(k, s);
        __syncthreads();
        sort(k, s, m);
        store_striped(dst, m, s, xf);
    }
};

}  // namespace qmsort_b200
