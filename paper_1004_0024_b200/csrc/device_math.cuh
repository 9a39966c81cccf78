// Device restatements of the reference's scalar numeric primitives.  Every floating-point
// step is spelled with a round-to-nearest intrinsic so that nvcc can neither contract a
// multiply-add (the reference is built with -ffp-contract=off, ref: proj/src/CMakeLists.txt:23-29)
// nor re-associate; the library is additionally compiled with -fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace isingb200 {

constexpr uint32_t kMtN = 624;  // ref: kMtStateSize, rng.hpp:11
constexpr uint32_t kMtM = 397;
constexpr uint32_t kInitSpinSeedMix = 0x9E3779B9u;  // ref: sweep_state.cpp:48
constexpr uint32_t kSwapSeedMix = 0x85EBCA6Bu;      // new: swap draws stay off the sweep streams

enum : int { kExpExact = 1, kExpFast = 2, kExpAccurate = 3 };

// ref: recurrence(), rng.cpp:22-25.  cur/next are consecutive old words, far is word i+397.
__device__ __forceinline__ uint32_t mt_recurrence(uint32_t cur, uint32_t next, uint32_t far) {
    const uint32_t y = (cur & 0x80000000u) | (next & 0x7fffffffu);
    return far ^ (y >> 1) ^ ((0u - (next & 1u)) & 0x9908b0dfu);
}

// ref: temper_one(), rng.cpp:27-33
__device__ __forceinline__ uint32_t mt_temper(uint32_t y) {
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

// ref: u32_to_unit, rng.hpp:87-92 — x/2^32 truncated toward zero.  cvt.rz keeps the top 24
// significant bits exactly as the reference's mask does; the power-of-two product is exact.
__device__ __forceinline__ float u32_to_unit(uint32_t x) {
    return __fmul_rn(__uint2float_rz(x), 0x1p-32f);
}

// ref: fastexp.hpp:15-23
__device__ constexpr float kTwoLnSq2 = 0.9609060278364028f;
__device__ constexpr float kLog2eP23 = 12102203.161561485f;
__device__ constexpr float kLog2eP25 = 48408812.64624594f;
__device__ constexpr float kAccCutoff = -21.834136187592387f;
__device__ constexpr float kImageLo = -1056964608.0f;
__device__ constexpr float kImageHi = 1073741760.0f;

// ref: exp_fast, fastexp.hpp:27-32 (lrintf in the default rounding mode == cvt.rni)
__device__ __forceinline__ float image_to_float(float t) {
    t = fminf(fmaxf(t, kImageLo), kImageHi);
    const int i = __float2int_rn(t) + 0x3F800000;
    return __fmul_rn(__int_as_float(i), kTwoLnSq2);
}
__device__ __forceinline__ float exp_fast(float x) { return image_to_float(__fmul_rn(x, kLog2eP23)); }

// ref: exp_accurate, fastexp.hpp:37-51 (IEEE sqrt: __fsqrt_rn)
__device__ __forceinline__ float exp_accurate(float x) {
    const float core = __fsqrt_rn(__fsqrt_rn(image_to_float(__fmul_rn(x, kLog2eP25))));
    return x >= 0.0f ? 1.0f : (x < kAccCutoff ? 0.0f : core);
}

// ref: eval_exp<exact>, sweep_kernels.hpp:22 — float(std::exp(double(x))).  CUDA's f64 exp and
// glibc's both stay within 1 ulp of the true value; after the rounding to f32 they can differ
// only when that value sits within ~1e-16 (relative) of an f32 rounding boundary.
__device__ __forceinline__ float exp_exact(float x) { return __double2float_rn(exp(double(x))); }

// Wait statistics of one lockstep attempt of 32 chains: adds, for w = 1, 2, 4, 8, 16, 32, the
// number of aligned w-lane groups of `ballot` that hold at least one accepting lane.
__device__ __forceinline__ void wait_fold(uint32_t ballot, uint32_t (&c)[6]) {
    const uint32_t a2 = (ballot | (ballot >> 1)) & 0x55555555u;
    const uint32_t a4 = (a2 | (a2 >> 2)) & 0x11111111u;
    const uint32_t a8 = (a4 | (a4 >> 4)) & 0x01010101u;
    const uint32_t a16 = (a8 | (a8 >> 8)) & 0x00010001u;
    c[0] += __popc(ballot);
    c[1] += __popc(a2);
    c[2] += __popc(a4);
    c[3] += __popc(a8);
    c[4] += __popc(a16);
    c[5] += ballot != 0u ? 1u : 0u;
}

template <int EXP>
__device__ __forceinline__ float exp_kind(float x) {
    if constexpr (EXP == kExpExact) return exp_exact(x);
    else if constexpr (EXP == kExpFast) return exp_fast(x);
    else return exp_accurate(x);
}

__device__ __forceinline__ float exp_kind_dyn(int kind, float x) {
    return kind == kExpExact ? exp_exact(x) : (kind == kExpFast ? exp_fast(x) : exp_accurate(x));
}

// ref: flip_exponent, sweep_kernels.hpp:14-16: -beta * ((2*s) * (hs + gamma*ht)).
// neg_beta = -beta, two_s = +/-2.
__device__ __forceinline__ float flip_exponent(float neg_beta, float gamma, float two_s, float hs,
                                               float ht) {
    return __fmul_rn(neg_beta, __fmul_rn(two_s, __fadd_rn(hs, __fmul_rn(gamma, ht))));
}

}  // namespace isingb200
