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
// sigmoid32's fast path reduces by 2^(i/32) instead (tools/gen_exp_table.py
// --n 32): one 16-byte {tail, scale} load per evaluation from a 512-byte
// table, four L1 lines for a warp's 32 random indices where the glibc table
// takes two 8-byte loads over up to sixteen (profiles/r1_light_variants.txt).
static __device__ __align__(16) const uint64_t kExp32Tab[64] = {
#include "exp32_table.inc"
};

// sigmoid32 of the reference (network.hpp:44-59), bit for bit: the logistic
// 1/(1+exp(-4.97 x)) in double, clamped into (0,1), rounded to float, clamped
// again.  Explicit _rn intrinsics keep every step a single IEEE operation (no
// contraction), the build never enables FTZ (sigmoid32 returns the float
// denormal 0x1p-149 at negative saturation), and exp is the
// restatement of the host glibc exp (exp_glibc.h) -- identical doubles, so
// identical floats: checked for all 2^32 inputs (oracle/exp_check.c,
// tests/test_gpu_sigmoid.py).
__device__ __forceinline__ float sigmoid32_exact(float x) {
    const double e = exp_glibc(__dmul_rn(-4.97, static_cast<double>(x)), kExpTab);
    double v = __ddiv_rn(1.0, __dadd_rn(1.0, e));
    if (v <= 0.0) v = 4.9406564584124654e-324;         // DBL_TRUE_MIN
    if (v >= 1.0) v = 1.0 - 1.1102230246251565e-16;     // 1 - DBL_EPSILON/2
    float f = __double2float_rn(v);
    if (f <= 0.0f) f = 1.40129846e-45f;                  // FLT_TRUE_MIN
    if (f >= 1.0f) f = 1.0f - 5.96046448e-08f;           // 1 - FLT_EPSILON/2
    return f;
}

// sigmoid32 with a short double-precision fast path and an exact rounding
// test (Ziv): the fast path evaluates 1/(1+exp(-4.97 x)) to a relative error
// below 2^-47 (exp(t) = 2^(k/32) exp(r), |r| <= ln2/64, degree-5 Taylor
// polynomial; reciprocal by MUFU.RCP64H refined by one third-order step
// y (1 + e + e^2), e = 1 - d y, which triples the bits where two Newton steps
// chain four dependent DFMAs) -- about half the FP64 operations of the
// correctly rounded exp + division.  Whenever that value lies within 2^12
// double ulps (2^-40 relative) of a float rounding boundary, or the result
// leaves the normal float range, the exact restatement above decides.  Both
// results then round to the same float: the reference's double is within
// ~1 ulp of the true value too.  Checked for all 2^32 inputs against
// sigmoid32_exact on the device (asnn_dev_sigmoid_selfcheck) and against the
// reference's host sigmoid32 (tests/test_gpu_sigmoid.py).
//
// The fast path is straight-line code (selects, no branches) so that the V
// evaluations of a column group interleave their FP64 dependency chains;
// sigmoid32_v takes the exact restatement in one rarely-taken branch after
// all of them.  Saturated (x > 10) and out-of-range (x <= -17, NaN) inputs
// run the same straight line on their unclamped t -- whatever it computes is
// replaced by the clamp constant or sent to the exact path, so no clamp sits
// on the latency chain of the latency-bound sweeps (K-chain).
//
// TabLoad: how the {tail, scale} pair of 2^(i/32) is read -- global memory
// through L1 (default) or a shared-memory copy (K-chain's finish warps).
struct ExpTabGlobal {
    __device__ __forceinline__ ulonglong2 operator()(uint32_t i) const {
        return __ldg(reinterpret_cast<const ulonglong2*>(kExp32Tab) + i);
    }
};
template <class TabLoad = ExpTabGlobal>
__device__ __forceinline__ float sigmoid32_fast(float x, bool& exact, TabLoad tab = TabLoad()) {
    const double t = __dmul_rn(-4.97, static_cast<double>(x));
    // decided on x with FP32 compares (the FP64 pipe binds populations):
    // sat: x > 10 (t < -49.7): the true value is within 2^-71 of 1, the float
    // rounds to 1 and clamps to 1 - FLT_EPSILON/2 -- and the fast path gives
    // that same clamp on the band below (t in [-49.7, -40]) too;
    // out: x <= -17 or NaN (t >= 84.49): float subnormal / clamped results
    // go to the exact restatement (a superset of what needs it)
    const bool sat = x > 10.0f;
    const bool out = !(x > -17.0f);
    // k = round(t 32/ln2) in the low bits of zs; r = t - k ln2/32 with the hi
    // part of ln2/32 exact against k (|k| < 2^12 on the accepted range)
    const double zs = __fma_rn(t, 0x1.71547652b82fep5, XG_SHIFT);
    const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(zs));
    const double kd = __dsub_rn(zs, XG_SHIFT);
    double r = __fma_rn(kd, -0x1.62e42fefa0000p-6, t);
    r = __fma_rn(kd, -0x1.cf79abc9e3b3ap-45, r);
    const ulonglong2 e = tab(static_cast<uint32_t>(ki & 31u));
    const double tail = __longlong_as_double(static_cast<long long>(e.x));
    const uint64_t sbits = e.y + (ki << 47);
    // exp(r) - 1 = r + r^2 (1/2 + r/6 + r^2 (1/24 + r/120)) + O(r^6/720),
    // 2^-48.6 at |r| = ln2/64; the bracket by Estrin (two FMA levels where
    // Horner chains three -- the sweeps of deep networks wait on this chain)
    const double r2 = __dmul_rn(r, r);
    const double q0 = __fma_rn(r, 0x1.5555555555555p-3, 0.5);
    const double q1 = __fma_rn(r, 0x1.1111111111111p-7, 0x1.5555555555555p-5);
    const double p = __fma_rn(r2, q1, q0);
    const double tmp = __fma_rn(r2, p, __dadd_rn(r, tail));
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    // 1 + scale (1 + tmp) as scale tmp + (1 + scale): the sum 1 + scale is
    // formed while the polynomial runs (one rounding of ~2^-53 more, inside
    // the fast path's 2^-47 budget)
    const double d = __fma_rn(scale, tmp, __dadd_rn(1.0, scale));
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    // third-order refinement: e = 1 - d y; y (1 + e + e^2) has error e^3
    const double er = __fma_rn(-d, y, 1.0);
    y = __fma_rn(y, __fma_rn(er, er, er), y);
    // y in (2^-125, 1]: distance of its low 29 mantissa bits from the float
    // rounding midpoint 2^28 (in double ulps of y), in 32-bit arithmetic:
    // near <=> |low29 - 2^28| < 2^12 <=> low29 - (2^28 - 2^12 + 1) < 2^13 - 1
    const uint32_t low29 = static_cast<uint32_t>(__double_as_longlong(y)) & ((1u << 29) - 1);
    const bool near = low29 - ((1u << 28) - (1u << 12) + 1) < (1u << 13) - 1;
    float f = __double2float_rn(y);
    f = (sat || f >= 1.0f) ? 1.0f - 5.96046448e-08f : f;
    exact = out || (near && !sat);
    return f;
}

__device__ __forceinline__ float sigmoid32_path(float x, bool& exact) {
    const float f = sigmoid32_fast(x, exact);
    return exact ? sigmoid32_exact(x) : f;
}

// The exact restatement out of line, for single-value call sites: the
// latency-bound one-column sweeps (config 3: 2.82 -> 2.70 ms) run a tighter
// loop without its inlined body; column groups (V = 4) keep it inline
// (config 5 measured 4% slower out of line, profiles/r1_light_variants.txt).
static __device__ __noinline__ float sigmoid32_exact_call(float x) { return sigmoid32_exact(x); }

template <class TabLoad = ExpTabGlobal>
__device__ __forceinline__ float sigmoid32(float x, TabLoad tab = TabLoad()) {
    bool exact;
    const float f = sigmoid32_fast(x, exact, tab);
    return exact ? sigmoid32_exact_call(x) : f;
}

// V independent sigmoid32 in place: fast paths first, then the exact
// restatement for whichever values need it.
template <int V>
__device__ __forceinline__ void sigmoid32_v(float (&a)[V]) {
    float f[V];
    bool ex[V];
    bool any = false;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        f[j] = sigmoid32_fast(a[j], ex[j]);
        any |= ex[j];
    }
    if (any) {
#pragma unroll
        for (int j = 0; j < V; ++j)
            if (ex[j]) f[j] = (V == 1 ? sigmoid32_exact_call(a[j]) : sigmoid32_exact(a[j]));
    }
#pragma unroll
    for (int j = 0; j < V; ++j) a[j] = f[j];
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

// Debug write-count mode (build flag ASNN_WRITE_COUNT, libasnn_b200_wc.so):
// every producer of an activation value -- the op slot of eval.cpp:16-23,
// in A or in K-cta's shared-memory rows -- adds 1 to g_wc[pos][col], so a
// test can assert that each slot is written exactly once per sweep
// (proj/tests/test_eval.cpp:199-213), segmented heavy rows
// included.  The normal build compiles the notes away.
#ifdef ASNN_WRITE_COUNT
static __device__ uint32_t* g_wc = nullptr;
static __device__ uint32_t g_wc_ld = 0;
#endif
__device__ __forceinline__ void wc_note(uint32_t pos, uint32_t col, int n) {
#ifdef ASNN_WRITE_COUNT
    if (g_wc)
        for (int v = 0; v < n; ++v) atomicAdd(&g_wc[static_cast<uint64_t>(pos) * g_wc_ld + col + v], 1u);
#else
    (void)pos, (void)col, (void)n;
#endif
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
