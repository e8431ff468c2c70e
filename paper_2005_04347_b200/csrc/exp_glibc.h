/*
 * exp_glibc.h -- the reference's exp, bit for bit.
 *
 * sigmoid32 (network.hpp:44-59) calls std::exp(double), i.e. glibc's exp.  On
 * x86-64 CPUs with FMA and AVX2 glibc >= 2.28 dispatches (ifunc) to its FMA
 * build of the table-driven algorithm from Arm's optimized-routines:
 *
 *   k = round(x * 128/ln2),  r = x - k*ln2/128 (two-constant reduction),
 *   exp(x) = 2^(k/128) * (1 + tail + r + C2 r^2 + C3 r^3 + C4 r^4 + C5 r^5),
 *
 * compiled with every a*b+c contracted to one fused multiply-add.  This header
 * restates that operation sequence -- each step one IEEE operation, fused
 * where the FMA build fuses and nowhere else -- so the device computes the
 * SAME double as the host libm, hence the same float after sigmoid32's
 * rounding (bitwise parity instead of CUDA exp's <= 1-ulp agreement).  The
 * 2^(i/128) table is generated from exact arithmetic (tools/gen_exp_table.py,
 * which also checks it against the host libm) and the constants are the
 * published ones of the algorithm.  Verified exhaustively against the host
 * libm for all 2^32 float inputs of sigmoid32 (oracle/exp_check.c).
 *
 * Usable from C (host; compile with -ffp-contract=off) and CUDA (device).
 */
#ifndef ASNN_EXP_GLIBC_H
#define ASNN_EXP_GLIBC_H

#include <stdint.h>

#if defined(__CUDACC__)
#define XG_FN __device__ __forceinline__ static
#define XG_FMA(a, b, c) __fma_rn((a), (b), (c))
#define XG_MUL(a, b) __dmul_rn((a), (b))
#define XG_ADD(a, b) __dadd_rn((a), (b))
#define XG_SUB(a, b) __dsub_rn((a), (b))
#define XG_ASDOUBLE(u) __longlong_as_double((long long)(u))
#define XG_ASUINT(d) ((uint64_t)__double_as_longlong(d))
#define XG_TAB(T, i) __ldg(&(T)[i])
#else
#include <math.h>
#include <string.h>
#define XG_FN static inline
#define XG_FMA(a, b, c) fma((a), (b), (c))
#define XG_MUL(a, b) ((a) * (b))
#define XG_ADD(a, b) ((a) + (b))
#define XG_SUB(a, b) ((a) - (b))
static inline double xg_asdouble(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static inline uint64_t xg_asuint(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
#define XG_ASDOUBLE(u) xg_asdouble(u)
#define XG_ASUINT(d) xg_asuint(d)
#define XG_TAB(T, i) ((T)[i])
#endif

#define XG_INVLN2N 0x1.71547652b82fep7 /* 128/ln2 */
#define XG_SHIFT 0x1.8p52
#define XG_NEGLN2HIN -0x1.62e42fefa0000p-8
#define XG_NEGLN2LON -0x1.cf79abc9e3b3ap-47
#define XG_C2 0x1.ffffffffffdbdp-2
#define XG_C3 0x1.555555555543cp-3
#define XG_C4 0x1.55555cf172b91p-5
#define XG_C5 0x1.1111167a4d017p-7

/* |x| >= 512 (k outside the normal exponent range): scale the result in two
 * steps, and round subnormal results once (the reference's specialcase). */
XG_FN double xg_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    double scale, y;
    if ((ki & 0x80000000u) == 0) {
        sbits -= 1009ull << 52;
        scale = XG_ASDOUBLE(sbits);
        y = XG_FMA(scale, tmp, scale);
        return XG_MUL(y, 0x1p1009);
    }
    sbits += 1022ull << 52;
    scale = XG_ASDOUBLE(sbits);
    const double st = XG_MUL(tmp, scale); /* shared by y and lo: not fused */
    y = XG_ADD(scale, st);
    if (1.0 > y) {
        const double hi = XG_ADD(y, 1.0);
        double lo = XG_ADD(XG_SUB(scale, y), st);
        lo = XG_ADD(XG_ADD(XG_SUB(1.0, hi), y), lo);
        y = XG_SUB(XG_ADD(lo, hi), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return XG_MUL(y, 0x1p-1022);
}

/* T: the 256-entry table of exp_table.inc. */
XG_FN double exp_glibc(double x, const uint64_t* T) {
    const uint64_t ix = XG_ASUINT(x);
    uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return XG_ADD(1.0, x); /* |x| < 2^-54 */
        if (abstop >= 0x409u) {                                     /* |x| >= 1024 */
            if (ix == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return XG_ADD(1.0, x);
            return (ix >> 63) ? 0.0 : XG_ASDOUBLE(0x7ff0000000000000ull);
        }
        abstop = 0; /* large |x|: the special case below */
    }
    const double zs = XG_FMA(x, XG_INVLN2N, XG_SHIFT);
    const uint64_t ki = XG_ASUINT(zs);
    const double kd = XG_SUB(zs, XG_SHIFT);
    double r = XG_FMA(kd, XG_NEGLN2HIN, x);
    r = XG_FMA(kd, XG_NEGLN2LON, r);
    const uint32_t idx = 2u * (uint32_t)(ki & 127u);
    const uint64_t top = ki << 45;
    const double tail = XG_ASDOUBLE(XG_TAB(T, idx));
    const uint64_t sbits = XG_TAB(T, idx + 1) + top;
    const double p23 = XG_FMA(r, XG_C3, XG_C2);
    const double tr = XG_ADD(r, tail);
    const double r2 = XG_MUL(r, r);
    const double p45 = XG_FMA(r, XG_C5, XG_C4);
    const double t1 = XG_FMA(p23, r2, tr);
    const double r4 = XG_MUL(r2, r2);
    const double tmp = XG_FMA(r4, p45, t1);
    if (abstop == 0) return xg_specialcase(tmp, sbits, ki);
    const double scale = XG_ASDOUBLE(sbits);
    return XG_FMA(scale, tmp, scale);
}

#endif /* ASNN_EXP_GLIBC_H */
