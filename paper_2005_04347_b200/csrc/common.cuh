// common.cuh -- shared device helpers of the ASNN engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "exp_glibc.h"

namespace asnn_b200 {


// Row segments (uint4 {row, first edge, end edge, aux}): a heavy row's stored
// edges split across the levels whose sources they need.  aux: kAccLoad =
// start from the partial sum in accbuf[slot], kAccStore = leave the partial
// sum there instead of finishing the row; slot = aux & kSlotMask.  The fp32
// accumulation is the same sequence of roundings as one uninterrupted sum.
constexpr uint32_t kAccLoad = 0x80000000u;
constexpr uint32_t kAccStore = 0x40000000u;
constexpr uint32_t kSlotMask = 0x3FFFFFFFu;

// The 2^(i/128) table of exp_glibc (tools/gen_exp_table.py).
static __device__ const uint64_t kExpTab[256] = {
#include "exp_table.inc"
};

// sigmoid32 of the reference (network.hpp:44-59), bit for bit: the logistic
// 1/(1+exp(-4.97 x)) in double, clamped into (0,1), rounded to float, clamped
// again.  Explicit _rn intrinsics keep every step a single IEEE operation (no
// contraction), the build never enables FTZ (sigmoid32 returns the float
// denormal 0x1p-149 at negative saturation), and exp is the
// restatement of the host glibc exp (exp_glibc.h) -- identical doubles, so
// identical floats: checked for all 2^32 inputs (oracle/exp_check.c,
// tests/test_gpu_sigmoid.py).
__device__ __forceinline__ float sigmoid32(float x) {
    const double e = exp_glibc(__dmul_rn(-4.97, static_cast<double>(x)), kExpTab);
    double v = __ddiv_rn(1.0, __dadd_rn(1.0, e));
    if (v <= 0.0) v = 4.9406564584124654e-324;         // DBL_TRUE_MIN
    if (v >= 1.0) v = 1.0 - 1.1102230246251565e-16;     // 1 - DBL_EPSILON/2
    float f = __double2float_rn(v);
    if (f <= 0.0f) f = 1.40129846e-45f;                  // FLT_TRUE_MIN
    if (f >= 1.0f) f = 1.0f - 5.96046448e-08f;           // 1 - FLT_EPSILON/2
    return f;
}

// One multiply-add of the reference accumulation (eval.cpp:20-21):
// x86 mulss then addss, never an FMA.
__device__ __forceinline__ float mac(float acc, float w, float a) {
    return __fadd_rn(acc, __fmul_rn(w, a));
}

template <int V>
struct Vec;
template <>
struct Vec<1> {
    using T = float;
};
template <>
struct Vec<2> {
    using T = float2;
};
template <>
struct Vec<4> {
    using T = float4;
};

template <int V>
__device__ __forceinline__ void load_cols(float (&r)[V], const float* p) {
    if constexpr (V == 1) {
        r[0] = __ldg(p);
    } else if constexpr (V == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        r[0] = t.x;
        r[1] = t.y;
    } else {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        r[0] = t.x;
        r[1] = t.y;
        r[2] = t.z;
        r[3] = t.w;
    }
}

// Plain (coherent) load for data written earlier in the same kernel.
template <int V>
__device__ __forceinline__ void load_cols_cg(float (&r)[V], const float* p) {
    if constexpr (V == 1) {
        r[0] = *p;
    } else if constexpr (V == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        r[0] = t.x;
        r[1] = t.y;
    } else {
        const float4 t = *reinterpret_cast<const float4*>(p);
        r[0] = t.x;
        r[1] = t.y;
        r[2] = t.z;
        r[3] = t.w;
    }
}

template <int V>
__device__ __forceinline__ void store_cols(float* p, const float (&r)[V]) {
    if constexpr (V == 1) {
        *p = r[0];
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(r[0], r[1]);
    } else {
        *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
    }
}

}  // namespace asnn_b200
