// common.cuh -- key types, orderings and small device helpers shared by every
// qmsort-b200 kernel.
//
// The sort core works on three UNSIGNED key types whose natural order is the
// sort order: uint32 (C1/C2 after the order-preserving transform), uint64
// (C3/C4) and Rec32 = four uint64 words compared lexicographically (C5, the
// rec32 comparator of SURVEY.md 8(d)).  The reference's comparator `less`
// (sort.hpp:215-217) is folded into an order-preserving bijection applied on
// the way in and out (transform.cuh), so one kernel family serves every
// (dtype, less/greater) pair bit-exactly.
#pragma once
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace qmsort_b200 {

struct alignas(16) Rec32 {
    uint64_t w[4];
};

template <class K>
struct KeyTraits;

// Constants the compiler cannot fold (constant bank).  They let a
// compare-and-swap finish on the FMA pipe -- max = (a - min) + b with two
// IMADs -- so sorting networks, which are otherwise pure ALU-pipe min/max,
// split their work over both integer pipes (B300_MICROARCH.md "Pipe rates").
__constant__ uint32_t c_neg1 = 0xFFFFFFFFu;
__constant__ uint32_t c_one = 1u;

// x + y - m (mod 2^32) with two IMADs: given the 32-bit word m of the smaller
// of two keys, the same word of the larger one (the words of {min, max} are a
// permutation of the words of {a, b}, so their sums agree mod 2^32).
__device__ __forceinline__ uint32_t other_word(uint32_t x, uint32_t y, uint32_t m) {
    const uint32_t t = m * c_neg1 + x;  // x - m
    return t * c_one + y;
}

template <>
struct KeyTraits<uint32_t> {
    static constexpr int kBytes = 4;
    __device__ __forceinline__ static uint32_t max_key() { return 0xFFFFFFFFu; }
    __device__ __forceinline__ static bool lt(uint32_t a, uint32_t b) { return a < b; }
    __device__ __forceinline__ static bool eq(uint32_t a, uint32_t b) { return a == b; }
    // compare-and-swap: a <- min, b <- max
    __device__ __forceinline__ static void cas(uint32_t& a, uint32_t& b) {
        uint32_t lo = min(a, b), hi = max(a, b);
        a = lo;
        b = hi;
    }
    // same result; min on the ALU pipe, max by two IMADs on the FMA pipe
    __device__ __forceinline__ static void cas_alt(uint32_t& a, uint32_t& b) {
        const uint32_t lo = min(a, b);
        const uint32_t t = lo * c_neg1 + a;  // a - lo
        b = t * c_one + b;                   // a + b - lo = max (mod 2^32)
        a = lo;
    }
    __device__ __forceinline__ static uint64_t hash(uint32_t a) { return a; }
    __device__ __forceinline__ static uint32_t shfl_xor(uint32_t a, int m) {
        return __shfl_xor_sync(0xffffffffu, a, m);
    }
    // bucket lookup table (LUT) support: keys are unsigned integers
    static constexpr bool kLut = true;
    using UInt = uint32_t;
    __device__ __forceinline__ static uint32_t bits(uint32_t a) { return a; }
};

template <>
struct KeyTraits<uint64_t> {
    static constexpr int kBytes = 8;
    __device__ __forceinline__ static uint64_t max_key() { return ~0ull; }
    __device__ __forceinline__ static bool lt(uint64_t a, uint64_t b) { return a < b; }
    __device__ __forceinline__ static bool eq(uint64_t a, uint64_t b) { return a == b; }
    __device__ __forceinline__ static void cas(uint64_t& a, uint64_t& b) {
        bool s = b < a;
        uint64_t lo = s ? b : a, hi = s ? a : b;
        a = lo;
        b = hi;
    }
    // same result: the minimum selected on the ALU pipe, the maximum's two
    // words by IMADs on the FMA pipe (other_word)
    __device__ __forceinline__ static void cas_alt(uint64_t& a, uint64_t& b) {
        const uint64_t mn = (b < a) ? b : a;
        const uint32_t xl = other_word((uint32_t)a, (uint32_t)b, (uint32_t)mn);
        const uint32_t xh = other_word((uint32_t)(a >> 32), (uint32_t)(b >> 32), (uint32_t)(mn >> 32));
        b = ((uint64_t)xh << 32) | xl;
        a = mn;
    }
    __device__ __forceinline__ static uint64_t hash(uint64_t a) { return a; }
    __device__ __forceinline__ static uint64_t shfl_xor(uint64_t a, int m) {
        return __shfl_xor_sync(0xffffffffu, a, m);
    }
    static constexpr bool kLut = true;
    using UInt = uint64_t;
    __device__ __forceinline__ static uint64_t bits(uint64_t a) { return a; }
};

template <>
struct KeyTraits<Rec32> {
    static constexpr int kBytes = 32;
    __device__ __forceinline__ static Rec32 max_key() {
        Rec32 r;
        r.w[0] = r.w[1] = r.w[2] = r.w[3] = ~0ull;
        return r;
    }
    __device__ __forceinline__ static bool lt(const Rec32& a, const Rec32& b) {
        // lexicographic over (w0,w1,w2,w3) as unsigned 64-bit words
        if (a.w[0] != b.w[0]) return a.w[0] < b.w[0];
        if (a.w[1] != b.w[1]) return a.w[1] < b.w[1];
        if (a.w[2] != b.w[2]) return a.w[2] < b.w[2];
        return a.w[3] < b.w[3];
    }
    __device__ __forceinline__ static bool eq(const Rec32& a, const Rec32& b) {
        return a.w[0] == b.w[0] && a.w[1] == b.w[1] && a.w[2] == b.w[2] && a.w[3] == b.w[3];
    }
    __device__ __forceinline__ static void cas(Rec32& a, Rec32& b) {
        bool s = lt(b, a);
        Rec32 lo, hi;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            lo.w[i] = s ? b.w[i] : a.w[i];
            hi.w[i] = s ? a.w[i] : b.w[i];
        }
        a = lo;
        b = hi;
    }
    __device__ __forceinline__ static void cas_alt(Rec32& a, Rec32& b) {
        const bool s = lt(b, a);
        Rec32 mn, mx;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            mn.w[i] = s ? b.w[i] : a.w[i];
            const uint32_t xl = other_word((uint32_t)a.w[i], (uint32_t)b.w[i], (uint32_t)mn.w[i]);
            const uint32_t xh = other_word((uint32_t)(a.w[i] >> 32), (uint32_t)(b.w[i] >> 32),
                                           (uint32_t)(mn.w[i] >> 32));
            mx.w[i] = ((uint64_t)xh << 32) | xl;
        }
        a = mn;
        b = mx;
    }
    __device__ __forceinline__ static Rec32 shfl_xor(const Rec32& a, int m) {
        Rec32 r;
#pragma unroll
        for (int i = 0; i < 4; ++i) r.w[i] = __shfl_xor_sync(0xffffffffu, a.w[i], m);
        return r;
    }
    __device__ __forceinline__ static uint64_t hash(const Rec32& a) {
        return a.w[0] * 0x9E3779B97F4A7C15ull ^ a.w[1] * 0xBF58476D1CE4E5B9ull ^
               a.w[2] * 0x94D049BB133111EBull ^ a.w[3];
    }
    static constexpr bool kLut = false;  // classified by the search tree only
    using UInt = uint64_t;
    __device__ __forceinline__ static uint64_t bits(const Rec32& a) { return a.w[0]; }
};

// Shared-memory padding: one spare element every 128 bytes so that a thread
// that owns ITEMS consecutive keys ("blocked" arrangement) can store them
// without bank conflicts when ITEMS*sizeof(K) is a multiple of 128 bytes.
// elems() leaves 64 elements of slack so that merge loops may read a few
// slots past the end of a run without leaving the allocation.
template <class K>
struct SmemPad {
    static constexpr int kPer = (128 / KeyTraits<K>::kBytes) > 0 ? (128 / KeyTraits<K>::kBytes) : 1;
    static constexpr int kShift = kPer >= 32 ? 5 : kPer >= 16 ? 4 : kPer >= 8 ? 3 : kPer >= 4 ? 2 : kPer >= 2 ? 1 : 0;
    __device__ __forceinline__ static unsigned idx(unsigned i) { return i + (i >> kShift); }
    static constexpr int elems(int n) { return n + n / kPer + 64; }
};

// Device-side invariant checks, compiled in with -DQMSORT_DEVICE_CHECKS=1 only
// (compute-sanitizer is not available on the bench pool): a violated bound
// prints the file, line and the two values involved and traps, so a bad index
// stops the call with QMSORT_ECUDA instead of corrupting memory.  The checked
// build runs the sanitizer workload (scripts/device_checks.sh).
#ifndef QMSORT_DEVICE_CHECKS
#define QMSORT_DEVICE_CHECKS 0
#endif
#if QMSORT_DEVICE_CHECKS
#define QCHECK(cond, a, b)                                                                            \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("qmsort device check failed %s:%d: %s (%llu, %llu)\n", __FILE__, __LINE__, #cond,  \
                   (unsigned long long)(a), (unsigned long long)(b));                                 \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define QCHECK(cond, a, b) \
    do {                   \
    } while (0)
#endif

// Order-preserving transform fused into the sort's first reads and last
// writes (aux_kernels.cuh has the standalone passes):
//   f(x) = x ^ b ^ (sext(x) & a),   f^-1(u) = u ^ b ^ (sext(u ^ b) & a)
// where sext(x) is all ones when x's top bit is set and a never has the top
// bit (so the top bit of f(x) is top(x) ^ top(b)).  a = b = 0: identity.
// int32/int64: b = sign bit (less) or its complement (greater), a = 0;
// unsigned greater: b = ~0; float64: a = 0x7FF..F, b = sign bit (less) or
// 0x7FF..F (greater); records: every word ^ b.
struct Xf {
    uint64_t a, b;
};
__device__ __forceinline__ uint32_t xf_fwd(uint32_t x, const Xf& f) { return x ^ (uint32_t)f.b; }
__device__ __forceinline__ uint32_t xf_inv(uint32_t u, const Xf& f) { return u ^ (uint32_t)f.b; }
__device__ __forceinline__ uint64_t xf_fwd(uint64_t x, const Xf& f) {
    return x ^ f.b ^ ((uint64_t)((int64_t)x >> 63) & f.a);
}
__device__ __forceinline__ uint64_t xf_inv(uint64_t u, const Xf& f) {
    const uint64_t v = u ^ f.b;
    return v ^ ((uint64_t)((int64_t)v >> 63) & f.a);
}
__device__ __forceinline__ Rec32 xf_fwd(Rec32 x, const Xf& f) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x.w[i] ^= f.b;
    return x;
}
__device__ __forceinline__ Rec32 xf_inv(Rec32 u, const Xf& f) { return xf_fwd(u, f); }

// SplitMix64 finaliser (reference rng.hpp:14-19) -- also used as a hash.
__host__ __device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

// Block-wide exclusive scan of `n` uint32 counters held in shared memory
// (in place).  Returns the total.  All threads of the block must call it.
// `warp_sums` needs blockDim.x/32 entries.
template <int T>
__device__ __forceinline__ uint32_t block_exclusive_scan_smem(uint32_t* data, int n,
                                                              uint32_t* warp_sums) {
    constexpr int kWarps = T / 32;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n + T - 1) / T;  // consecutive items per thread
    const int beg = tid * per;
    uint32_t local = 0;
    for (int i = 0; i < per; ++i)
        if (beg + i < n) local += data[beg + i];
    // warp inclusive scan
    uint32_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < kWarps ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kWarps) warp_sums[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    uint32_t excl = x - local + (wid > 0 ? warp_sums[wid - 1] : 0);
    const uint32_t total = warp_sums[kWarps - 1];
    for (int i = 0; i < per; ++i) {
        if (beg + i < n) {
            uint32_t v = data[beg + i];
            data[beg + i] = excl;
            excl += v;
        }
    }
    __syncthreads();
    return total;
}

}  // namespace qmsort_b200
