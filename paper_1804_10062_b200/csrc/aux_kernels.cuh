// aux_kernels.cuh -- order-preserving key transforms, K9 harness generators and
// the device-side verification pass.
//
// Transforms: the reference sorts under an arbitrary `less` (sort.hpp:215-217).
// For the five supported (dtype, comparator) pairs the order is mapped onto
// unsigned integer / word-lexicographic order by a bijection f with
// less(a, b) <=> f(a) <u f(b); the sort core runs on f(x) and f^-1 restores the
// caller's bit patterns.  float64 uses the IEEE total-order trick, which equals
// operator< on NaN-free input without -0.0 (BASELINE.json config 4).
#pragma once
#include "common.cuh"

namespace qmsort_b200 {

enum TransformMode : int {
    kXfNone = 0,
    kXfI32Less = 1,      // x ^ 0x80000000
    kXfI32Greater = 2,   // x ^ 0x7FFFFFFF
    kXfU32Greater = 3,   // ~x
    kXfU64Greater = 4,   // ~x (also rec32 words)
    kXfF64Less = 5,      // sign-magnitude -> biased
    kXfF64Greater = 6,   // f64less then ~
    kXfI64Less = 7,      // x ^ 0x8000000000000000
    kXfI64Greater = 8,   // x ^ 0x7FFFFFFFFFFFFFFF
};

__device__ __forceinline__ uint64_t f64_fwd(uint64_t b) {
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ uint64_t f64_inv(uint64_t u) {
    return (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
}

// In-place transform over `words` 32- or 64-bit words.
__global__ void transform32_kernel(uint32_t* p, uint64_t words, int mode) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = p[i];
        if (mode == kXfI32Less) x ^= 0x80000000u;
        else if (mode == kXfI32Greater) x ^= 0x7FFFFFFFu;
        else if (mode == kXfU32Greater) x = ~x;
        p[i] = x;
    }
}
__global__ void transform64_kernel(uint64_t* p, uint64_t words, int mode, int inverse) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = p[i];
        if (mode == kXfU64Greater) x = ~x;
        else if (mode == kXfF64Less) x = inverse ? f64_inv(x) : f64_fwd(x);
        else if (mode == kXfF64Greater) x = inverse ? f64_inv(~x) : ~f64_fwd(x);
        else if (mode == kXfI64Less) x ^= 0x8000000000000000ull;
        else if (mode == kXfI64Greater) x ^= 0x7FFFFFFFFFFFFFFFull;
        p[i] = x;
    }
}

// The same maps as an Xf (common.cuh) over a range of core keys: the
// stand-alone passes the fused samplesort path does not need (direct block
// sort of a small n, merge sort, merge fallback ranges).
template <class K>
__global__ void xf_kernel(K* p, uint64_t n, Xf xf, int inverse) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = inverse ? xf_inv(p[i], xf) : xf_fwd(p[i], xf);
}

// ---------------------------------------------------------------------------
// K9: counter-based SplitMix64 generators, bit-identical to the host recipes
// (reference rng.hpp:10-23).  Element j of SplitMix64(seed) is
// mix(seed + (j+1) * gamma).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t sm_at(uint64_t seed, uint64_t j) {
    return sm_mix(seed + (j + 1) * kGamma);
}

// kind: 0 u32 uniform (C2), 1 u64 uniform (C3), 2 rec32 (C5),
//       10 f64 sorted, 11 f64 reverse, 12 f64 16-distinct, 13 f64 gaussian,
//       14 f64 organ-pipe (C4 a..e; `total` = full n for 11 / 14).
__global__ void generate_kernel(void* out, uint64_t n, uint64_t seed, uint64_t start, int kind,
                                uint64_t total) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = start + i;
        switch (kind) {
            case 0: static_cast<uint32_t*>(out)[i] = (uint32_t)(sm_at(seed, g) >> 32); break;
            case 1: static_cast<uint64_t*>(out)[i] = sm_at(seed, g); break;
            case 2: {
                ulonglong2* o = static_cast<ulonglong2*>(out) + 2 * i;
                o[0] = make_ulonglong2(sm_at(seed, 4 * g) >> 52, sm_at(seed, 4 * g + 1));
                o[1] = make_ulonglong2(sm_at(seed, 4 * g + 2), sm_at(seed, 4 * g + 3));
                break;
            }
            case 10: static_cast<double*>(out)[i] = (double)(g + 1); break;
            case 11: static_cast<double*>(out)[i] = (double)(total - g); break;
            case 12: static_cast<double*>(out)[i] = (double)((sm_at(seed, g) >> 60) + 1); break;
            case 13: {
                const uint64_t k = g / 2;
                const double u1 = (double)((sm_at(seed, 2 * k) >> 11) + 1) * 0x1.0p-53;
                const double u2 = (double)(sm_at(seed, 2 * k + 1) >> 11) * 0x1.0p-53;
                const double r = sqrt(-2.0 * log(u1));
                double x = (g & 1) ? r * sin(6.283185307179586 * u2) : r * cos(6.283185307179586 * u2);
                static_cast<double*>(out)[i] = (x == 0.0) ? 0.0 : x;
                break;
            }
            case 14: {
                const uint64_t a = g + 1, b = total - g;
                static_cast<double*>(out)[i] = (double)(a < b ? a : b);
                break;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Verification on the caller's raw dtype and comparator: adjacent-pair order
// violations and an order-independent multiset fingerprint of the raw bits
// (sum and xor of mixed words).  res[0] += violations, res[1] += sum,
// res[2] ^= xor.
// ---------------------------------------------------------------------------
template <class T>
struct RawOrder {
    __device__ __forceinline__ static bool lt(const T& a, const T& b) { return a < b; }
    __device__ __forceinline__ static uint64_t bits(const T& a) {
        uint64_t u = 0;
        memcpy(&u, &a, sizeof(T));
        return u;
    }
};
template <>
struct RawOrder<Rec32> {
    __device__ __forceinline__ static bool lt(const Rec32& a, const Rec32& b) {
        return KeyTraits<Rec32>::lt(a, b);
    }
    __device__ __forceinline__ static uint64_t bits(const Rec32& a) {
        return KeyTraits<Rec32>::hash(a);
    }
};

template <class T, bool GREATER>
__global__ void check_kernel(const T* __restrict__ a, uint64_t n, unsigned long long* res,
                             int check_order) {
    uint64_t bad = 0, sum = 0, x = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const T v = a[i];
        const uint64_t h = sm_mix(RawOrder<T>::bits(v) + kGamma);
        sum += h;
        x ^= h;
        if (check_order && i + 1 < n) {
            const T w = a[i + 1];
            if (GREATER ? RawOrder<T>::lt(v, w) : RawOrder<T>::lt(w, v)) ++bad;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        x ^= __shfl_xor_sync(0xffffffffu, x, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&res[0], (unsigned long long)bad);
        atomicAdd(&res[1], (unsigned long long)sum);
        atomicXor(&res[2], (unsigned long long)x);
    }
}

// Small control reads (counters, a few keys) into mapped pinned host memory:
// one warp stores the words over PCIe (posted writes), so these reads never
// queue on a copy engine behind another stream's bulk transfer.
struct SmallRead {
    const unsigned char* src;
    uint32_t bytes, dst_off;
};
__global__ void store_mapped_kernel(SmallRead r0, SmallRead r1, unsigned char* dst) {
    for (uint32_t i = threadIdx.x; i < r0.bytes; i += blockDim.x) dst[r0.dst_off + i] = r0.src[i];
    for (uint32_t i = threadIdx.x; i < r1.bytes; i += blockDim.x) dst[r1.dst_off + i] = r1.src[i];
}

}  // namespace qmsort_b200
