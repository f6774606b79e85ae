// elements.cuh -- device kernels for SURVEY.md 8(f) rows f3 (key + payload
// elements) and f4 (select_nth).
//
// f3: the reference's Element<PayloadBytes> (element.hpp:13-20) orders on an
// int64 key alone; the payload is moved, never compared.  On the GPU each
// element becomes a 32-byte sort record {order-preserving key, input index, 0,
// 0} that the Rec32 samplesort orders lexicographically, so equal keys keep
// their input order (a stable sort -- one of the arrangements the reference's
// unstable qms may return, test_sort.cpp:328-339).  The payload is then
// gathered once by the sorted indices: one read and one write of every element.
#pragma once
#include <cstdint>

#include "aux_kernels.cuh"
#include "common.cuh"

namespace qmsort_b200 {

// Order-preserving 64-bit image of one key of the element at e.  dtype codes
// follow qmsort_dtype; greater flips the order.
__device__ __forceinline__ uint64_t elem_key_bits(const unsigned char* e, int dtype, int greater) {
    uint64_t k = 0;
    switch (dtype) {
        case 0: k = (uint64_t)(*reinterpret_cast<const uint32_t*>(e) ^ 0x80000000u); break;  // int32
        case 1: k = *reinterpret_cast<const uint32_t*>(e); break;                             // uint32
        case 2: k = *reinterpret_cast<const uint64_t*>(e); break;                             // uint64
        case 3: k = f64_fwd(*reinterpret_cast<const uint64_t*>(e)); break;                    // double
        case 5: k = *reinterpret_cast<const uint64_t*>(e) ^ 0x8000000000000000ull; break;      // int64
        default: break;
    }
    return greater ? ~k : k;
}

__global__ void make_elem_recs_kernel(const unsigned char* __restrict__ data, uint64_t n,
                                      uint32_t elem_bytes, uint32_t key_off, int dtype,
                                      int greater, Rec32* __restrict__ recs) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        Rec32 r;
        r.w[0] = elem_key_bits(data + i * elem_bytes + key_off, dtype, greater);
        r.w[1] = i;
        r.w[2] = 0;
        r.w[3] = 0;
        recs[i] = r;
    }
}

// dst element j = src element recs[j].w[1]; W-sized words, `words` per
// element.  Consecutive threads write consecutive words (coalesced stores).
template <class W>
__global__ void gather_elems_kernel(const W* __restrict__ src, W* __restrict__ dst,
                                    const Rec32* __restrict__ recs, uint64_t n, uint32_t words) {
    const uint64_t total = n * words;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = t / words;
        const uint64_t w = t - e * words;
        dst[t] = src[recs[e].w[1] * words + w];
    }
}

}  // namespace qmsort_b200
