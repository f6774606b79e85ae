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
