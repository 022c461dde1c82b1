// Shared device helpers for libitq3 (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cmath>

#include "../../include/itq3.h"

namespace itq3 {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kSubBlocks = 8;  // packing.py:31

// ---- error plumbing (host) ------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute belongs to
// the device context, so a process driving several GPUs sets it on each (bit d of `done` = device d).
template <typename K>
inline int ensure_smem_attr(K* kernel, int smem, std::atomic<unsigned long long>& done, const char* what) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return ITQ3_OK;
    if (cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return check_launch(what);
    done.fetch_or(bit, std::memory_order_acq_rel);
    return ITQ3_OK;
}
inline int device_sms() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

__host__ __device__ inline int block_nbytes(int n, int ss) { return 3 * n / 8 + 4 + (ss ? 16 : 0); }
inline bool valid_block_n(int n) { return n == 32 || n == 64 || n == 128 || n == 256 || n == 512; }

// ---- binary16 <-> double, exactly as packing.py:87-109 -----------------------------------
// encode_f16: RNE single rounding from binary64, finite overflow saturates to +-65504
// (0x7BFF), NaN -> 0x7E00, +-inf pass through.
__host__ __device__ __forceinline__ uint16_t f64_to_f16_bits(double x) {
#ifdef __CUDA_ARCH__
    const uint64_t b = (uint64_t)__double_as_longlong(x);
#else
    uint64_t b;
    memcpy(&b, &x, sizeof(b));
#endif
    const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
    const int exp = (int)((b >> 52) & 0x7ff);
    const uint64_t mant = b & 0xFFFFFFFFFFFFFull;
    if (exp == 0x7ff) return mant ? (uint16_t)0x7E00 : (uint16_t)(sign | 0x7C00);
    const double ax = fabs(x);
    if (ax >= 65504.0) return (uint16_t)(sign | 0x7BFF);  // saturate (incl. values that round to inf)
    if (exp == 0) return sign;                            // binary64 zero / subnormal -> +-0
    const int e = exp - 1023;
    if (e >= -14) {  // normal binary16
        uint32_t m = (uint32_t)(mant >> 42);
        const uint64_t rem = mant & ((1ull << 42) - 1);
        const uint64_t half = 1ull << 41;
        uint32_t h = ((uint32_t)(e + 15) << 10) + m;
        if (rem > half || (rem == half && (m & 1u))) h += 1;  // carry into exponent is correct
        return (uint16_t)(sign | h);
    }
    const uint64_t M = mant | (1ull << 52);
    const int s = 28 - e;  // value in units of 2^-24 = M * 2^(e-52+24)
    if (s > 63) return sign;
    const uint64_t m = M >> s;
    const uint64_t rem = M & ((1ull << s) - 1);
    const uint64_t half = 1ull << (s - 1);
    uint64_t h = m;
    if (rem > half || (rem == half && (m & 1u))) h += 1;
    return (uint16_t)(sign | (uint16_t)h);
}

// decode_f16: exact value of any binary16 pattern
__host__ __device__ __forceinline__ double f16_bits_to_f64(uint16_t h) {
    const int sign = h >> 15;
    const int exp = (h >> 10) & 0x1f;
    const int man = h & 0x3ff;
    double v;
    if (exp == 0) {
        v = (double)man * 5.9604644775390625e-08;  // 2^-24
    } else if (exp == 31) {
#ifdef __CUDA_ARCH__
        v = man ? __longlong_as_double(0x7ff8000000000000ll) : __longlong_as_double(0x7ff0000000000000ll);
#else
        v = man ? __builtin_nan("") : __builtin_inf();
#endif
    } else {
        v = (double)(man | 0x400) * ldexp(1.0, exp - 25);
    }
    return sign ? -v : v;
}

__device__ __forceinline__ float f16_bits_to_f32(uint16_t h) {
    return __half2float(__ushort_as_half(h));
}

// ---- numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src) -------------------
// add.reduce starts from the identity 0.0 and adds pairwise_sum(v, n):
//   n < 8: sequential; n <= 128: 8 strided accumulators then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7));
//   n > 128: split at n/2 (multiple of 8) and recurse.  All block sizes here are powers of two.
// Warp-cooperative for n in [8, 512]: lane group g = lane/8 owns 128-chunk g, lane k = lane%8
// owns accumulator k; the tree and the chunk recursion map onto xor shuffles 1,2,4 | 8,16.
// Returns the sum on every lane.  v is in shared memory (or any generic memory).
__device__ __forceinline__ double warp_pairwise_sum(const double* v, int n, int lane) {
    const int L = n < 128 ? n : 128;
    const int chunks = n / L;
    const int g = lane >> 3, k = lane & 7;
    double r = 0.0;
    if (g < chunks) {
        const double* p = v + g * L;
        r = p[k];
        for (int i = 8; i < L; i += 8) r = __dadd_rn(r, p[i + k]);
    }
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
    if (chunks >= 2) r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 8));
    if (chunks >= 4) r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 16));
    r = __shfl_sync(FULL, r, 0);
    return __dadd_rn(0.0, r);  // reduce identity (turns -0 into +0 like numpy)
}

// Serial form of the same recursion for a single thread (used for short sub-block sums).
__device__ __forceinline__ double serial_pairwise_sum(const double* v, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, v[i]);
        return __dadd_rn(0.0, res);
    }
    // n in {8,16,32,64} here
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = v[k];
    for (int i = 8; i < n; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], v[i + k]);
    }
    const double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                 __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    return __dadd_rn(0.0, res);
}

// copysign(floor(|v| + 0.5), v) with the addition rounded, as numpy does (quantizer.py:152-153)
__device__ __forceinline__ double round_half_away(double v) {
    return copysign(floor(__dadd_rn(fabs(v), 0.5)), v);
}

__device__ __forceinline__ double clip1(double v) { return fmin(fmax(v, -1.0), 1.0); }

// ------------------------------------------------------------------------------------------
// Butterfly helpers (generic over float / double)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
// p + sg * v with sg = +-1: the product is exact, so this is v + p (sg = 1) or p - v (sg = -1) with ONE
// rounding -- bit-identical to add_rn / sub_rn (signed zeros included), one instruction instead of
// two adds and a select
__device__ __forceinline__ double pm_rn(double sg, double v, double p) { return __fma_rn(sg, v, p); }
__device__ __forceinline__ float pm_rn(float sg, float v, float p) { return __fmaf_rn(sg, v, p); }

// Unnormalised butterfly over N = 32*E elements held in stride layout.
template <int E, typename T>
__device__ __forceinline__ void warp_butterfly(T (&v)[E], int lane) {
#pragma unroll
    for (int h = 1; h < 32 && h < 32 * E; h <<= 1) {
        const T sg = (lane & h) ? T(-1) : T(1);  // high lane: lo - hi = p - v
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const T p = __shfl_xor_sync(FULL, v[e], h);
            v[e] = pm_rn(sg, v[e], p);
        }
    }
#pragma unroll
    for (int hh = 1; hh < E; hh <<= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e & hh) == 0) {
                const T lo = v[e], hi = v[e + hh];
                v[e] = add_rn(lo, hi);
                v[e + hh] = sub_rn(lo, hi);
            }
        }
    }
}

}  // namespace itq3
