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

struct TableSort {
    static constexpr int T = 256, ITEMS = 16, kCap = T * ITEMS;  // keys per bucket
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
        uint32_t y2[kWords], y3[kWords];
        alignas(16) uint16_t out[kCap];
        uint32_t ovf[kOvfCap];  // fourth and later copies (key - klo)
        uint32_t warp_sums[T / 32];
        uint32_t novf;
    };
    using Net = BlockSorter<uint32_t, T, ITEMS>;  // fallback, in the table's memory
    static_assert(Net::kSmemBytes <= (sizeof(uint2) + 2 * sizeof(uint32_t)) * kWords, "fallback tile");
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
        if (!(atomicOr(&sm.y3[a], bit) & bit)) return 2u;
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
        uint32_t n = (uint32_t)__popc(sm.y2[a] & below) + (uint32_t)__popc(sm.y3[a] & below);
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
            sm.y3[i] = 0;
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
            uint32_t pos = (c.y & 0xFFFFu) + (uint32_t)__popc(c.x & below) + copies_below(sm, a, below, v, L) + 3u;
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
__global__ void __launch_bounds__(TableSort::T, 5) tablesort_tasks_kernel(const SortTask* __restrict__ tasks,
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

}  // namespace qmsort_b200
