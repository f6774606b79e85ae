// tablesort.cuh -- K5t: comparison-free sort of narrow-span uint32 buckets.
//
// The last partition level leaves buckets whose keys all lie between two
// neighbouring splitters.  On dense key sets (C2: 2^28 keys over 2^32 values)
// that span is a few 10^4 values for a few 10^3 keys, and the bucket can be
// sorted without a single key comparison -- the base-case role of
// small_sort / insertion_sort (reference small_sort.hpp:13-111) and the
// bottom merge levels (merge.hpp:103-119), like K5, for the buckets the plan
// marks eligible (TableSort::eligible):
//   1. a bit table of the span lives in shared memory; every key sets its bit
//      (atomicOr).  A key that finds it set is a second copy: it bumps its
//      word's copy count and sets the same bit of a second plane, a third
//      copy that of a third plane; fourth and later copies go to a short
//      overflow list;
//   2. one scan over the table's words gives every word the number of keys
//      below it (set bits + copy count);
//   3. a key's rank = its word's prefix + the set bits below its own bit
//      (+ its copy number): it is stored at that position of a 16-bit staging
//      tile (key - klo), which goes out with coalesced stores.
// About 50 instructions per key where the comparison network spends 190.
// Buckets that do not fit the scheme after all (a key outside the bounds,
// more than kOvfCap fourth copies) are sorted by the comparison network in
// the same CTA, with the table's memory as its tile.
#pragma once
#include "blocksort.cuh"
#include "samplesort.cuh"

namespace qmsort_b200 {

// Shared-memory accesses of the hot loops by 32-bit shared-window address (one
// base register for the whole kernel instead of a generic-pointer conversion
// per access).
__device__ __forceinline__ uint32_t smem_atom_or(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint2 smem_ld64(uint32_t addr) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr) : "memory");
    return r;
}
__device__ __forceinline__ void smem_st32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" : : "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void smem_st16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" : : "r"(addr), "h"((unsigned short)v) : "memory");
}

#ifndef QMSORT_TS_PLANES
#define QMSORT_TS_PLANES 3  // bit planes: first, second (, third) copies of a value
#endif
#ifndef QMSORT_TS_CTAS
#define QMSORT_TS_CTAS 5  // resident CTAs per SM the kernel is compiled for
#endif

struct TableSort {
    static constexpr int T = 256, ITEMS = 16, kCap = T * ITEMS;  // keys per bucket
    static constexpr int kPlanes = QMSORT_TS_PLANES;
    static_assert(kPlanes == 2 || kPlanes == 3, "planes");
    static constexpr int kWords = 2048;                          // 2^16 values, one bit each
    static constexpr int kWpt = kWords / T;                      // table words per thread in the scan
    static constexpr int kOvfCap = 128;
    static_assert(kWpt == 8, "the cell swizzle assumes 8 words per thread");

    struct Smem {
        // One 8-byte cell per table word (32 values): x = the values present,
        // y = keys below the word (low half, written by the scan) | second and
        // later copies among the word's keys (high half, counted by the
        // insert).  Word w lives in cell w ^ ((w >> 4) & 7): the scan's
        // per-thread walks over 8 consecutive words are conflict-free.
        alignas(16) uint2 cell[kWords];
        // bit b of y2[w] / y3[w]: value 32 w + b has a second / third copy
        // (same swizzle; read only for words whose copy count is not zero)
        uint32_t y2[kWords], y3[kPlanes > 2 ? kWords : 1];
        alignas(16) uint16_t out[kCap];
        uint32_t ovf[kOvfCap];  // fourth and later copies (key - klo)
        uint32_t warp_sums[T / 32];
        uint32_t novf;
    };
    using Net = BlockSorter<uint32_t, T, ITEMS>;  // fallback, in the table's memory
    static_assert(Net::kSmemBytes <= (sizeof(uint2) + sizeof(uint32_t)) * kWords, "fallback tile");
    static constexpr size_t kSmemBytes = sizeof(Smem);

    // Buckets the plan sends here: at most kCap keys, bounds spanning fewer
    // than 2^16 values, and sparse enough that fourth copies stay rare
    // (span >= 4 len) yet dense enough that the table scan pays (span <= 64 len).
    __host__ __device__ static bool eligible(uint32_t len, uint64_t klo, uint64_t khi) {
        return table_sort_eligible(len, klo, khi);
    }

    __device__ __forceinline__ static uint32_t cell_of(uint32_t w) { return w ^ ((w >> 4) & 7u); }

    // The rare paths are kept out of line: the unrolled per-key code stays
    // small (inlined, the kernel stalled on instruction fetch).
    // A key that found its first-copy bit set: returns its copy number (1, 2,
    // or 3 = on the overflow list).
    __device__ __noinline__ static uint32_t later_copy(Smem& sm, uint32_t a, uint32_t bit, uint32_t v) {
        atomicAdd(&sm.cell[a].y, 0x10000u);
        if (!(atomicOr(&sm.y2[a], bit) & bit)) return 1u;
        if (kPlanes > 2 && !(atomicOr(&sm.y3[a], bit) & bit)) return 2u;
        const uint32_t i = atomicAdd(&sm.novf, 1u);
        if (i < (uint32_t)kOvfCap) sm.ovf[i] = v;
        return 3u;
    }
    // overflow entries below v in v's word
    __device__ __noinline__ static uint32_t ovf_below(const Smem& sm, uint32_t v, uint32_t L) {
        uint32_t n = 0;
#pragma unroll 1
        for (uint32_t i = 0; i < L; ++i) {
            const uint32_t o = sm.ovf[i];
            n += ((o >> 5) == (v >> 5) && o < v) ? 1u : 0u;
        }
        return n;
    }
    // later copies of smaller values in the word of cell a
    __device__ __forceinline__ static uint32_t copies_below(const Smem& sm, uint32_t a, uint32_t below, uint32_t v,
                                                            uint32_t L) {
        uint32_t n = (uint32_t)__popc(sm.y2[a] & below);
        if (kPlanes > 2) n += (uint32_t)__popc(sm.y3[a] & below);
        if (L) n += ovf_below(sm, v, L);
        return n;
    }

    // src may alias dst.  Returns false with nothing written when the bucket
    // has to be sorted by the network.
    __device__ __forceinline__ static bool sort(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                const int m, Smem& sm, const uint32_t klo, const uint32_t span,
                                                const Xf& xf) {
        const int tid = threadIdx.x;
        const uint32_t cells = (uint32_t)__cvta_generic_to_shared(sm.cell);
        const uint32_t outs = (uint32_t)__cvta_generic_to_shared(sm.out);
        const uint32_t W = (span >> 5) + 1;    // table words in use
        const uint32_t Wc = (W + 7u) & ~7u;    // cells touched (whole swizzle blocks)
        const int rows = (m + T - 1) / T;
        uint32_t k[ITEMS];
        {
            const uint32_t* p = src + tid;
#pragma unroll
            for (int u = 0; u < ITEMS; ++u) k[u] = u * T + tid < m ? p[u * T] : klo;
        }
        for (uint32_t i = tid; i < Wc; i += T) {
            sm.cell[i] = make_uint2(0, 0);
            sm.y2[i] = 0;
            if (kPlanes > 2) sm.y3[i] = 0;
        }
        if (tid == 0) sm.novf = 0;
        __syncthreads();
        // 1. insert; k[u] becomes (key - klo) | copy number << 16, or ~0 for
        // a slot without a key to place (past the bucket, overflow list)
        uint32_t vmax = 0;
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            if (u < rows) {  // uniform
                const bool valid = u * T + tid < m;
                uint32_t v = k[u] - klo;
                vmax = max(vmax, v);
                v = min(v, span);
                const uint32_t a = cell_of(v >> 5);
                const uint32_t bit = valid ? 1u << (v & 31u) : 0u;
                k[u] = valid ? v : 0xFFFFFFFFu;
                if (smem_atom_or(cells + a * 8u, bit) & bit) {
                    const uint32_t c = later_copy(sm, a, bit, v);
                    k[u] = c == 3u ? 0xFFFFFFFFu : (v | (c << 16));
                }
            }
        }
        const int bad = __syncthreads_or(vmax > span ? 1 : 0);
        const uint32_t L = sm.novf;
        if (bad || L > (uint32_t)kOvfCap) return false;
        // 2. scan: thread t owns words 8t .. 8t+7
        uint32_t nk[kWpt];
        uint32_t cnt = 0;
        const uint32_t w0 = (uint32_t)tid * kWpt;
        const bool owner = w0 < Wc;
        // cell of word w0 + j (w0 is a multiple of 8: the swizzle only permutes the thread's own 8 cells)
        auto own = [&](int j) -> uint32_t { return cells + (w0 | ((((uint32_t)tid >> 1) & 7u) ^ (uint32_t)j)) * 8u; };
        if (owner) {
#pragma unroll
            for (int j = 0; j < kWpt; ++j) {
                const uint2 c = smem_ld64(own(j));
                nk[j] = (uint32_t)__popc(c.x) + (c.y >> 16);
                cnt += nk[j];
            }
        }
        const uint32_t lane = tid & 31, wid = tid >> 5;
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) sm.warp_sums[wid] = x;
        __syncthreads();
        if (owner) {
            uint32_t run = x - cnt;
#pragma unroll
            for (int i = 0; i < T / 32; ++i) run += (uint32_t)i < wid ? sm.warp_sums[i] : 0u;
#pragma unroll
            for (int j = 0; j < kWpt; ++j) {
                // the copy count in the high half stays (prefix < 2^13)
                asm volatile("red.shared.or.b32 [%0], %1;" : : "r"(own(j) + 4u), "r"(run) : "memory");
                run += nk[j];
            }
        }
        __syncthreads();
        // 3. rank and stage: a key's position = the keys below its word + the
        // copies of smaller values in its word + its own copy number
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            if (u < rows) {
                const uint32_t v = k[u] & 0xFFFFu;
                const uint32_t a = cell_of(v >> 5);
                const uint2 c = smem_ld64(cells + a * 8u);
                const uint32_t below = ~(0xFFFFFFFFu << (v & 31u));
                uint32_t pos = (c.y & 0xFFFFu) + (uint32_t)__popc(c.x & below);
                if (c.y >> 16) pos += copies_below(sm, a, below, v, L) + ((k[u] >> 16) & 3u);
                QCHECK(k[u] == 0xFFFFFFFFu || pos < (uint32_t)m, pos, m);
                if (k[u] != 0xFFFFFFFFu) smem_st16(outs + pos * 2u, v);
            }
        }
        for (uint32_t i = tid; i < L; i += T) {  // fourth and later copies
            const uint32_t v = sm.ovf[i];
            const uint32_t a = cell_of(v >> 5);
            const uint2 c = sm.cell[a];
            const uint32_t below = (1u << (v & 31u)) - 1u;
            uint32_t pos = (c.y & 0xFFFFu) + (uint32_t)__popc(c.x & below) + copies_below(sm, a, below, v, L) + (uint32_t)kPlanes;
#pragma unroll 1
            for (uint32_t j = 0; j < i; ++j) pos += sm.ovf[j] == v ? 1u : 0u;
            QCHECK(pos < (uint32_t)m, pos, m);
            sm.out[pos] = (uint16_t)v;
        }
        __syncthreads();
#pragma unroll 4
        for (int i = tid; i < m; i += T) dst[i] = xf_inv((uint32_t)sm.out[i] + klo, xf);
        return true;
    }
};

// One CTA per table-class task (launched with the class's task count).
__global__ void __launch_bounds__(TableSort::T, QMSORT_TS_CTAS) tablesort_tasks_kernel(const SortTask* __restrict__ tasks,
                                                                         uint32_t* A, const uint32_t* B, Xf xf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TableSort::Smem& sm = *reinterpret_cast<TableSort::Smem*>(smem_raw);
    const SortTask t = tasks[blockIdx.x];
    QCHECK(t.len <= (uint32_t)TableSort::kCap, t.len, TableSort::kCap);
    const uint32_t* src = (t.in_a ? A : B) + t.off;
    if (TableSort::sort(src, A + t.off, (int)t.len, sm, (uint32_t)t.klo, (uint32_t)(t.khi - t.klo), xf)) return;
    __syncthreads();
    TableSort::Net::sort_tile(src, A + t.off, (int)t.len, reinterpret_cast<uint32_t*>(smem_raw), xf);
}

// ---------------------------------------------------------------------------
// K5c: the table sort for wide spans (uint32 buckets spanning 2^16 values or
// more, uint64 / int64 / float64 buckets).  The bucket's span is cut into at
// most 2^16 cells of 2^sh values -- about 16 cells per key -- and the table
// holds one bit per cell.  A cell's keys (up to three by the bit planes, more
// through the overflow list) land in the cell's output slots in arrival
// order; cells holding more than one key are then put in order by their
// first arrival with an insertion sort over the slots (the `fix` list: about
// 6 % of the keys on smooth data).  Cells are monotone in the key, so the
// tile is sorted.  Buckets whose keys crowd a few cells (overflow list or fix
// list full) go to the comparison network in the same CTA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void smem_st_key(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" : : "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void smem_st_key(uint32_t addr, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" : : "r"(addr), "l"(v) : "memory");
}

// Shapes (CellShape<K, BIG>): uint32 -- 256 threads, 4096 keys, 2^16 cells;
// 8-byte keys -- 256 threads, 2048 keys, 2^15 cells (38 KB of shared memory,
// 5 CTAs per SM: last-level buckets of 2^27 keys average 1000 keys), and a big
// shape of 512 threads, 8192 keys, 2^16 cells (C3's 2^30 keys leave buckets of
// 4096 keys on average).
template <class K, bool BIG>
struct CellShape {
    static constexpr int T = BIG ? 512 : 256;
    static constexpr int ITEMS = sizeof(K) == 4 || BIG ? 16 : 8;
    static constexpr int kCellBits = sizeof(K) == 4 || BIG ? 16 : 15;
    static constexpr int kMinCtas = BIG || sizeof(K) > 8 ? 2 : (sizeof(K) == 4 ? 4 : 5);
};

// What a key's cell is computed from: integer keys -- their bits, within the
// bounds the plan passes with the task; records -- the 64-bit prefix of
// (w0 - smallest w0, w1) (rec_prefix), within the bucket's smallest and
// largest prefix, both found by the CTA once the bucket is in registers.
template <class K>
struct CellBounds {
    using UI = typename KeyTraits<K>::UInt;
    UI klo, span;
    uint32_t sh;
    template <int ITEMS, class SM>
    __device__ __forceinline__ bool prepare(const K (&)[ITEMS], int, SM&, int, int) {
        return true;
    }
    __device__ __forceinline__ UI proj(const K& k) const { return KeyTraits<K>::bits(k); }
};
template <>
struct CellBounds<Rec32> {
    using UI = uint64_t;
    uint64_t klo, span;
    uint32_t sh;
    uint64_t base;
    uint32_t wsh;
    __device__ __forceinline__ uint64_t proj(const Rec32& r) const { return rec_prefix(r, base, wsh); }
    // block-wide smallest / largest f(key) over the bucket's keys
    template <int ITEMS, class SM, class F>
    __device__ __forceinline__ void minmax(const Rec32 (&k)[ITEMS], int m, SM& sm, int T, F&& f, uint64_t& lo,
                                           uint64_t& hi) {
        if (threadIdx.x == 0) {
            sm.red[0] = ~0ull;
            sm.red[1] = 0;
        }
        __syncthreads();
        unsigned long long a = ~0ull, b = 0;
#pragma unroll
        for (int u = 0; u < ITEMS; ++u)
            if (u * T + (int)threadIdx.x < m) {
                const unsigned long long v = f(k[u]);
                a = min(a, v);
                b = max(b, v);
            }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 31) == 0 && a <= b) {
            atomicMin(&sm.red[0], a);
            atomicMax(&sm.red[1], b);
        }
        __syncthreads();
        lo = sm.red[0];
        hi = sm.red[1];
        __syncthreads();
    }
    template <int ITEMS, class SM>
    __device__ __forceinline__ bool prepare(const Rec32 (&k)[ITEMS], int m, SM& sm, int T, int cell_bits) {
        uint64_t lo, hi;
        minmax(k, m, sm, T, [](const Rec32& r) { return (unsigned long long)r.w[0]; }, lo, hi);
        base = lo;
        wsh = hi > lo ? (uint32_t)__clzll((long long)(hi - lo)) : 64u;
        minmax(k, m, sm, T, [&](const Rec32& r) { return (unsigned long long)rec_prefix(r, base, wsh); }, lo, hi);
        klo = lo;
        span = hi - lo;
        sh = cell_shift((uint32_t)m, span, (uint32_t)cell_bits);
        return (span >> sh) >= 4ull * (uint64_t)m;  // else most cells hold several records
    }
};

template <class K, bool BIG = false>
struct CellSort {
    using KT = KeyTraits<K>;
    using BD = CellBounds<K>;
    using UI = typename BD::UI;
    using SH = CellShape<K, BIG>;
    static constexpr int T = SH::T, ITEMS = SH::ITEMS, kCap = T * ITEMS;
    static constexpr int kPlanes = 3;
    static constexpr int kCellBits = SH::kCellBits;
    static constexpr int kWords = (1 << kCellBits) / 32;
    static constexpr int kWpt = kWords / T;  // table words per thread in the scan
    static constexpr int kOvfCap = 128, kFixCap = 1024;
    static_assert(kWpt == 8 || kWpt == 4, "the cell swizzle");

    struct Smem {
        alignas(16) uint2 cell[kWords];  // as TableSort::Smem
        uint32_t y2[kWords], y3[kWords];
        alignas(16) K out[kCap];
        uint32_t fix[kFixCap];  // first slot | keys << 16 of the cells holding several keys
        K ovfk[kOvfCap];        // fourth and later keys of a cell
        uint32_t ovf[kOvfCap];  // ... and their cells
        unsigned long long red[2];
        uint32_t warp_sums[T / 32];
        uint32_t novf, nfix;
    };
    using Net = BlockSorter<K, T, ITEMS>;
    static_assert(Net::kSmemBytes <= sizeof(Smem), "fallback tile");
    static constexpr size_t kSmemBytes = sizeof(Smem);

    // Word w lives in cell w ^ s(w): the scan's per-thread walks over kWpt
    // consecutive words are conflict-free (8-byte cells: 16 lanes per access).
    // 8 words per thread: lane l reads cell 8 l + (j ^ (l >> 1 & 7)); 4 words:
    // cell 4 l + (j ^ (l >> 2 & 3)).
    __device__ __forceinline__ static uint32_t cell_of(uint32_t w) {
        return kWpt == 8 ? w ^ ((w >> 4) & 7u) : w ^ ((w >> 4) & 3u);
    }

    // A key that found its cell's bit set: its copy number (1, 2), or 3 | the
    // overflow-list slot reserved for it << 2 (the caller stores the key: it
    // stays in registers).
    __device__ __noinline__ static uint32_t later_copy(Smem& sm, uint32_t a, uint32_t bit, uint32_t v) {
        atomicAdd(&sm.cell[a].y, 0x10000u);
        if (!(atomicOr(&sm.y2[a], bit) & bit)) return 1u;
        if (!(atomicOr(&sm.y3[a], bit) & bit)) return 2u;
        const uint32_t i = atomicAdd(&sm.novf, 1u);
        if (i < (uint32_t)kOvfCap) sm.ovf[i] = v;
        return 3u | (i << 2);
    }
    // overflow entries in cells below v of v's word / in cell v
    __device__ __noinline__ static uint32_t ovf_below(const Smem& sm, uint32_t v, uint32_t L) {
        uint32_t n = 0;
#pragma unroll 1
        for (uint32_t i = 0; i < L; ++i) {
            const uint32_t o = sm.ovf[i];
            n += ((o >> 5) == (v >> 5) && o < v) ? 1u : 0u;
        }
        return n;
    }
    __device__ __noinline__ static uint32_t ovf_equal(const Smem& sm, uint32_t v, uint32_t L) {
        uint32_t n = 0;
#pragma unroll 1
        for (uint32_t i = 0; i < L; ++i) n += sm.ovf[i] == v ? 1u : 0u;
        return n;
    }
    // A key in a word that holds later copies: the copies in cells below its
    // own; the first arrival of a cell with several keys queues the cell for
    // the in-cell sort.
    __device__ __noinline__ static uint32_t slow_rank(Smem& sm, uint32_t a, uint32_t v, uint32_t copy, uint32_t pos,
                                                      uint32_t L) {
        const uint32_t bit = 1u << (v & 31u), below = bit - 1u;
        const uint32_t c2 = sm.y2[a], c3 = sm.y3[a];
        uint32_t n = (uint32_t)__popc(c2 & below) + (uint32_t)__popc(c3 & below);
        if (L) n += ovf_below(sm, v, L);
        if (copy == 0 && (c2 & bit)) {
            uint32_t mult = 2u + ((c3 & bit) ? 1u : 0u);
            if (L && (c3 & bit)) mult += ovf_equal(sm, v, L);
            const uint32_t i = atomicAdd(&sm.nfix, 1u);
            if (i < (uint32_t)kFixCap) sm.fix[i] = (pos + n) | (mult << 16);
        }
        return n + copy;
    }

    // src may alias dst.  Returns false with nothing written when the bucket
    // has to be sorted by the network.
    __device__ __forceinline__ static bool sort(const K* __restrict__ src, K* __restrict__ dst, const int m, Smem& sm,
                                                BD& bd, const Xf& xf) {
        const int tid = threadIdx.x;
        const uint32_t cells = (uint32_t)__cvta_generic_to_shared(sm.cell);
        const uint32_t outs = (uint32_t)__cvta_generic_to_shared(sm.out);
        const int rows = (m + T - 1) / T;
        K k[ITEMS];
        {
            const K* p = src + tid;
#pragma unroll
            for (int u = 0; u < ITEMS; ++u)
                if (u * T + tid < m) k[u] = p[u * T];
        }
        if (!bd.prepare(k, m, sm, T, kCellBits)) return false;
        const UI klo = bd.klo, span = bd.span;
        const uint32_t sh = bd.sh;
        const uint32_t vspan = (uint32_t)(span >> sh);  // last cell
        const uint32_t W = (vspan >> 5) + 1;
        const uint32_t Wc = (W + (uint32_t)kWpt - 1u) & ~((uint32_t)kWpt - 1u);
        for (uint32_t i = tid; i < Wc; i += T) {
            sm.cell[i] = make_uint2(0, 0);
            sm.y2[i] = 0;
            sm.y3[i] = 0;
        }
        if (tid == 0) {
            sm.novf = 0;
            sm.nfix = 0;
        }
        __syncthreads();
        // 1. insert; cp = the keys' copy numbers, 2 bits each (3: overflow list)
        uint32_t cp = 0;
        bool oob = false;
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            if (u < rows && u * T + tid < m) {
                const UI rel = bd.proj(k[u]) - klo;
                oob |= rel > span;
                const uint32_t v = (uint32_t)(min(rel, span) >> sh);
                const uint32_t a = cell_of(v >> 5);
                const uint32_t bit = 1u << (v & 31u);
                if (smem_atom_or(cells + a * 8u, bit) & bit) {
                    const uint32_t c = later_copy(sm, a, bit, v);
                    cp |= (c & 3u) << (2 * u);
                    if ((c & 3u) == 3u && (c >> 2) < (uint32_t)kOvfCap) sm.ovfk[c >> 2] = k[u];
                }
            }
        }
        const int bad = __syncthreads_or(oob ? 1 : 0);
        const uint32_t L = sm.novf;
        if (bad || L > (uint32_t)kOvfCap) return false;
        // 2. scan: thread t owns words 8t .. 8t+7
        uint32_t nk[kWpt];
        uint32_t cnt = 0;
        const uint32_t w0 = (uint32_t)tid * kWpt;
        const bool owner = w0 < Wc;
        auto own = [&](int j) -> uint32_t { return cells + cell_of(w0 + (uint32_t)j) * 8u; };
        if (owner) {
#pragma unroll
            for (int j = 0; j < kWpt; ++j) {
                const uint2 c = smem_ld64(own(j));
                nk[j] = (uint32_t)__popc(c.x) + (c.y >> 16);
                cnt += nk[j];
            }
        }
        const uint32_t lane = tid & 31, wid = tid >> 5;
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) sm.warp_sums[wid] = x;
        __syncthreads();
        if (owner) {
            uint32_t run = x - cnt;
#pragma unroll
            for (int i = 0; i < T / 32; ++i) run += (uint32_t)i < wid ? sm.warp_sums[i] : 0u;
#pragma unroll
            for (int j = 0; j < kWpt; ++j) {
                asm volatile("red.shared.or.b32 [%0], %1;" : : "r"(own(j) + 4u), "r"(run) : "memory");
                run += nk[j];
            }
        }
        __syncthreads();
        // 3. stage every key at its cell's slots
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            if (u < rows && u * T + tid < m) {
                const uint32_t copy = (cp >> (2 * u)) & 3u;
                const uint32_t v = (uint32_t)((bd.proj(k[u]) - klo) >> sh);
                const uint32_t a = cell_of(v >> 5);
                const uint2 c = smem_ld64(cells + a * 8u);
                const uint32_t below = ~(0xFFFFFFFFu << (v & 31u));
                uint32_t pos = (c.y & 0xFFFFu) + (uint32_t)__popc(c.x & below);
                if (c.y >> 16) pos += slow_rank(sm, a, v, copy, pos, L);
                QCHECK(copy == 3u || pos < (uint32_t)m, pos, m);
                if (copy != 3u) {
                    if constexpr (sizeof(K) <= 8) smem_st_key(outs + pos * (uint32_t)sizeof(K), k[u]);
                    else sm.out[pos] = k[u];
                }
            }
        }
        for (uint32_t i = tid; i < L; i += T) {  // fourth and later keys of a cell
            const uint32_t v = sm.ovf[i];
            const uint32_t a = cell_of(v >> 5);
            const uint2 c = sm.cell[a];
            const uint32_t below = (1u << (v & 31u)) - 1u;
            uint32_t pos = (c.y & 0xFFFFu) + (uint32_t)__popc(c.x & below) + (uint32_t)__popc(sm.y2[a] & below) +
                           (uint32_t)__popc(sm.y3[a] & below) + ovf_below(sm, v, L) + (uint32_t)kPlanes;
#pragma unroll 1
            for (uint32_t j = 0; j < i; ++j) pos += sm.ovf[j] == v ? 1u : 0u;
            QCHECK(pos < (uint32_t)m, pos, m);
            sm.out[pos] = sm.ovfk[i];
        }
        __syncthreads();
        // 4. cells with several keys: order their slots
        const uint32_t F = sm.nfix;
        if (F > (uint32_t)kFixCap) return false;
        for (uint32_t i = tid; i < F; i += T) {
            const uint32_t f = sm.fix[i];
            const uint32_t p0 = f & 0xFFFFu, mult = f >> 16;
            QCHECK(p0 + mult <= (uint32_t)m, p0, mult);
#pragma unroll 1
            for (uint32_t j = 1; j < mult; ++j) {
                const K key = sm.out[p0 + j];
                uint32_t q = j;
                while (q > 0 && KT::lt(key, sm.out[p0 + q - 1])) {
                    sm.out[p0 + q] = sm.out[p0 + q - 1];
                    --q;
                }
                sm.out[p0 + q] = key;
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int i = tid; i < m; i += T) dst[i] = xf_inv(sm.out[i], xf);
        return true;
    }
};

template <class K, bool BIG>
__global__ void __launch_bounds__(CellShape<K, BIG>::T, CellShape<K, BIG>::kMinCtas)
    cellsort_tasks_kernel(const SortTask* __restrict__ tasks, K* A, const K* B, Xf xf) {
    using CS = CellSort<K, BIG>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typename CS::Smem& sm = *reinterpret_cast<typename CS::Smem*>(smem_raw);
    const SortTask t = tasks[blockIdx.x];
    QCHECK(t.len <= (uint32_t)CS::kCap, t.len, CS::kCap);
    const K* src = (t.in_a ? A : B) + t.off;
    typename CS::BD bd;
    if constexpr (KeyTraits<K>::kLut) {
        using UI = typename CS::UI;
        const uint64_t span = t.khi - t.klo;
        bd.klo = (UI)t.klo;
        bd.span = (UI)span;
        bd.sh = cell_shift(t.len, span, CS::kCellBits);
    }
    if (CS::sort(src, A + t.off, (int)t.len, sm, bd, xf)) return;
    __syncthreads();
    CS::Net::sort_tile(src, A + t.off, (int)t.len, reinterpret_cast<K*>(smem_raw), xf);
}

}  // namespace qmsort_b200
