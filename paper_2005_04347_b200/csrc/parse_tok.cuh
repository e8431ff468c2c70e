// parse_tok.cuh -- device token parsers for the `asnn 1` text format.
//
// parse_id / parse_weight of the reference (io.cpp:66-80) are std::from_chars
// calls that must consume the whole token.  libstdc++ (GCC 13) implements
// from_chars<float> with correct rounding (round to nearest, ties to even),
// accepts an optional '-', "inf"/"infinity"/"nan"/"nan(chars)" in any case,
// decimal digits with an optional '.' and exponent, and reports
// result_out_of_range when a nonzero value rounds to 0 or to infinity (both
// rejected by parse_weight).  The device restates that contract:
//   * Clinger's exact path for <= 2^24 with |q| <= 10 (one IEEE operation);
//   * otherwise a double-precision candidate (error < 2^-50) rounded to
//     float, then the rounding decided EXACTLY by comparing the decimal
//     value with the neighbouring float midpoint in big-integer arithmetic
//     (w * 5^q * 2^q against (2m +- 1) * 2^e, 320-bit);
//   * tokens whose value needs more than 19 significant digits at a rounding
//     boundary, or falls in the float subnormal range, take the exact slow
//     path (parse_f32_exact): the first 200 significant digits as a
//     1152-bit integer plus a sticky bit for the rest, compared with the
//     candidate's neighbouring midpoints -- a float midpoint has fewer than
//     200 significant decimal digits, so the comparison is exact.  No token
//     goes back to the host.
// Checked against the reference's from_chars on random and adversarial
// tokens (tests/test_gpu_parse.py).
#pragma once

#include <stdint.h>

namespace asnn_b200 {
namespace parse {

#include "pow_tables.inc"

enum : uint8_t { kTokOk = 0, kTokErr = 1 };

__device__ __forceinline__ bool is_digit(char c) { return c >= '0' && c <= '9'; }
__device__ __forceinline__ bool is_ws(char c) { return c == ' ' || c == '\t'; }

// std::from_chars<uint32_t> over the whole token.
__device__ __forceinline__ uint8_t parse_u32(const char* p, const char* e, uint32_t& v) {
    if (p == e) return kTokErr;
    uint64_t x = 0;
    for (; p < e; ++p) {
        if (!is_digit(*p)) return kTokErr;
        x = x * 10 + static_cast<uint64_t>(*p - '0');
        if (x > 0xFFFFFFFFull) return kTokErr;
    }
    v = static_cast<uint32_t>(x);
    return kTokOk;
}

// 320-bit unsigned integers for exact comparisons.
struct Big {
    uint64_t l[5];
};

__device__ __forceinline__ void big_u64(Big& b, uint64_t v) {
    b.l[0] = v;
    b.l[1] = b.l[2] = b.l[3] = b.l[4] = 0;
}

// b = a * 5^k (k <= 95)
__device__ __forceinline__ void big_mul_pow5(Big& b, uint64_t a, int k) {
    uint64_t carry = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint64_t m = kPow5[k][i];
        const uint64_t lo = a * m;
        const uint64_t hi = __umul64hi(a, m);
        const uint64_t s = lo + carry;
        b.l[i] = s;
        carry = hi + (s < lo ? 1 : 0);
    }
    b.l[4] = carry;
}

__device__ __forceinline__ void big_shl(Big& b, int s) {
    const int w = s >> 6, r = s & 63;
    for (int i = 4; i >= 0; --i) {
        const int j = i - w;
        uint64_t v = j >= 0 ? b.l[j] : 0;
        if (r) {
            v <<= r;
            if (j - 1 >= 0) v |= b.l[j - 1] >> (64 - r);
        }
        b.l[i] = v;
    }
}

__device__ __forceinline__ int big_cmp(const Big& a, const Big& b) {
    for (int i = 4; i >= 0; --i)
        if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}

// sign of (w * 10^q - m * 2^e), exactly (1 <= w < 2^64, m < 2^27).
__device__ __forceinline__ int cmp_decimal_dyadic(uint64_t w, int q, uint64_t m, int e) {
    Big L, R;
    if (q >= 0) {  // w 5^q 2^q  vs  m 2^e
        big_mul_pow5(L, w, q);
        big_u64(R, m);
        const int s = q - e;
        if (s >= 0) big_shl(L, s);
        else big_shl(R, -s);
    } else {       // w  vs  m 5^k 2^(e+k)
        const int k = -q;
        big_u64(L, w);
        big_mul_pow5(R, m, k);
        const int s = e + k;
        if (s >= 0) big_shl(R, s);
        else big_shl(L, -s);
    }
    return big_cmp(L, R);
}

// Correctly rounded positive normal float of w * 10^q (w >= 1, 19 digits at
// most, -95 <= q <= 38), given a candidate float c whose value is within a
// small fraction of an ulp of it.  sticky: the true value exceeds w*10^q by
// a nonzero amount smaller than 10^q (truncated digits); returns false when
// an exact tie with the sticky tail makes the answer undecidable here.
__device__ __forceinline__ bool round_exact(uint64_t w, int q, float c, bool sticky, float& out) {
    const uint32_t cb = __float_as_uint(c);
    const uint32_t be = cb >> 23;                       // biased exponent, 1..254
    const uint64_t mant = (cb & 0x7FFFFFu) | 0x800000u;
    const int e = static_cast<int>(be) - 150;           // c = mant * 2^e
    // upper midpoint (2 mant + 1) 2^(e-1)
    int cu = cmp_decimal_dyadic(w, q, 2 * mant + 1, e - 1);
    if (cu == 0 && sticky) cu = 1;
    if (cu > 0 || (cu == 0 && (mant & 1))) {
        out = __uint_as_float(cb + 1);  // next float up (exponent carry included)
        return true;
    }
    if (cu == 0) {
        out = c;
        return true;
    }
    // lower midpoint: below a power of two the neighbour is twice as close
    const bool pow2 = mant == 0x800000u && be > 1;
    const int cl = pow2 ? cmp_decimal_dyadic(w, q, 4 * mant - 1, e - 2)
                        : cmp_decimal_dyadic(w, q, 2 * mant - 1, e - 1);
    if (cl == 0 && sticky) {  // strictly above the midpoint: stays c
        out = c;
        return true;
    }
    if (cl < 0 || (cl == 0 && (mant & 1))) {
        out = __uint_as_float(cb - 1);
        return true;
    }
    out = c;
    return true;
}

// ---- exact slow path -------------------------------------------------------
// 1152-bit unsigned integers (36 x 32-bit limbs), single thread, rare tokens.
constexpr int kXL = 36;
struct BigX {
    uint32_t l[kXL];
};
__device__ __noinline__ void bx_set(BigX& b, uint32_t v) {
    b.l[0] = v;
    for (int i = 1; i < kXL; ++i) b.l[i] = 0;
}
// b = b * m + a (m, a < 2^32)
__device__ __noinline__ void bx_muladd(BigX& b, uint32_t m, uint32_t a) {
    uint64_t carry = a;
    for (int i = 0; i < kXL; ++i) {
        const uint64_t t = static_cast<uint64_t>(b.l[i]) * m + carry;
        b.l[i] = static_cast<uint32_t>(t);
        carry = t >> 32;
    }
}
__device__ __noinline__ void bx_mul_pow5(BigX& b, int k) {
    for (; k >= 13; k -= 13) bx_muladd(b, 1220703125u, 0);  // 5^13
    uint32_t m = 1;
    for (; k > 0; --k) m *= 5;
    if (m != 1) bx_muladd(b, m, 0);
}
__device__ __noinline__ void bx_shl(BigX& b, int s) {
    const int w = s >> 5, r = s & 31;
    for (int i = kXL - 1; i >= 0; --i) {
        const int j = i - w;
        uint32_t v = j >= 0 ? b.l[j] : 0u;
        if (r) {
            v <<= r;
            if (j - 1 >= 0) v |= b.l[j - 1] >> (32 - r);
        }
        b.l[i] = v;
    }
}
__device__ __noinline__ int bx_cmp(const BigX& a, const BigX& b) {
    for (int i = kXL - 1; i >= 0; --i)
        if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}
// sign of (D 10^q + sticky - M 2^F), D the digit integer, sticky a positive
// amount below 10^q (truncated nonzero digits)
__device__ __noinline__ int bx_cmp_dyadic(const BigX& D, int q, bool sticky, uint32_t M, int F) {
    BigX L = D, R;
    bx_set(R, M);
    if (q >= 0) {  // D 5^q 2^q  vs  M 2^F
        bx_mul_pow5(L, q);
        if (q >= F) bx_shl(L, q - F);
        else bx_shl(R, F - q);
    } else {       // D  vs  M 5^-q 2^(F - q)
        bx_mul_pow5(R, -q);
        if (F - q >= 0) bx_shl(R, F - q);
        else bx_shl(L, q - F);
    }
    const int c = bx_cmp(L, R);
    return c == 0 && sticky ? 1 : c;
}

// std::from_chars<float> for the tokens the fast path cannot decide: the
// decimal digits of [p, e) (a well-formed finite decimal, sign excluded)
// rounded exactly, ties to even; kTokErr when the result is 0 or infinity
// (result_out_of_range, as libstdc++ reports for parse_weight).  `approx` is
// the fast path's double candidate (relative error < 2^-49).
__device__ __noinline__ uint8_t parse_f32_exact(const char* p, const char* e, double approx, uint32_t sign,
                                                float& out) {
    constexpr int kDigits = 200;
    BigX D;
    bx_set(D, 0);
    int nd = 0, q = 0;
    bool sticky = false, point = false;
    for (; p < e; ++p) {
        const char ch = *p;
        if (ch == '.') {
            point = true;
            continue;
        }
        if (!is_digit(ch)) break;
        const uint32_t d = static_cast<uint32_t>(ch - '0');
        if (nd == 0 && d == 0) {
            if (point) --q;
            continue;
        }
        if (nd < kDigits) {
            bx_muladd(D, 10u, d);
            ++nd;
            if (point) --q;
        } else {
            sticky |= d != 0;
            if (!point) ++q;
        }
    }
    if (p < e && (*p | 0x20) == 'e') {
        const char* t = p + 1;
        bool eneg = false;
        if (t < e && (*t == '+' || *t == '-')) {
            eneg = *t == '-';
            ++t;
        }
        int64_t x = 0;
        for (; t < e && is_digit(*t); ++t)
            if (x < 1000000) x = x * 10 + (*t - '0');
        q += static_cast<int>(eneg ? -x : x);
    }
    // candidate: a float bit pattern within one step of the answer
    uint32_t cb;
    if (approx >= 0x1p-126) {
        const float c = __double2float_rn(approx);
        cb = __float_as_uint(c);
        if ((cb & 0x7F800000u) == 0x7F800000u) cb = 0x7F7FFFFFu;  // FLT_MAX, decided below
    } else {
        cb = static_cast<uint32_t>(__double2uint_rn(__dmul_rn(approx, 0x1p149)));  // subnormal count
    }
    // value of a positive pattern b: m 2^E
    auto mant = [](uint32_t b) -> uint32_t { return (b & 0x7FFFFFu) | ((b >> 23) ? 0x800000u : 0u); };
    auto expo = [](uint32_t b) -> int { return static_cast<int>((b >> 23) ? (b >> 23) : 1u) - 150; };
    // upper midpoint of cb: (2m + 1) 2^(E-1)
    const uint32_t m = mant(cb);
    const int E = expo(cb);
    int cu = bx_cmp_dyadic(D, q, sticky, 2 * m + 1, E - 1);
    uint32_t r = cb;
    if (cu > 0 || (cu == 0 && (m & 1))) {
        r = cb + 1;  // (a pattern past FLT_MAX is infinity)
    } else if (cu < 0) {
        // lower midpoint: below a power of two the neighbour is twice as close
        if (cb == 0) {
            r = 0;
        } else {
            const bool pow2 = (cb & 0x7FFFFFu) == 0 && (cb >> 23) > 1;
            const int cl = pow2 ? bx_cmp_dyadic(D, q, sticky, 4 * m - 1, E - 2)
                                : bx_cmp_dyadic(D, q, sticky, 2 * m - 1, E - 1);
            if (cl < 0 || (cl == 0 && (m & 1))) r = cb - 1;
        }
    }
    if (r == 0 || (r & 0x7F800000u) == 0x7F800000u) return kTokErr;  // rounds to 0 or infinity
    out = __uint_as_float(r | sign);
    return kTokOk;
}

// std::from_chars<float> (chars_format::general) over the whole token.
__device__ __forceinline__ uint8_t parse_f32(const char* p, const char* e, float& out) {
    bool neg = false;
    if (p < e && *p == '-') {
        neg = true;
        ++p;
    }
    if (p == e) return kTokErr;
    const uint32_t sign = neg ? 0x80000000u : 0u;
    const char* const digits0 = p;  // the decimal's first character (after the sign)
    const char c0 = static_cast<char>(*p | 0x20);
    if (c0 == 'i') {  // "inf" or "infinity", any case
        const char* kw = "infinity";
        int n = 0;
        while (n < 8 && p + n < e && static_cast<char>(p[n] | 0x20) == kw[n]) ++n;
        if (!((n == 3 && p + 3 == e) || (n == 8 && p + 8 == e))) return kTokErr;
        out = __uint_as_float(sign | 0x7F800000u);
        return kTokOk;
    }
    if (c0 == 'n') {  // "nan" or "nan(" [A-Za-z0-9_]* ")"
        if (e - p < 3 || static_cast<char>(p[1] | 0x20) != 'a' || static_cast<char>(p[2] | 0x20) != 'n')
            return kTokErr;
        const char* t = p + 3;
        if (t < e) {
            if (*t != '(') return kTokErr;
            ++t;
            while (t < e && (is_digit(*t) || (*t >= 'a' && *t <= 'z') || (*t >= 'A' && *t <= 'Z') || *t == '_'))
                ++t;
            if (t >= e || *t != ')' || t + 1 != e) return kTokErr;
        }
        out = __uint_as_float(sign | 0x7FC00000u);
        return kTokOk;
    }
    uint64_t w = 0;
    int nd = 0, q = 0;
    bool trunc = false, any = false;
    for (; p < e && is_digit(*p); ++p) {
        any = true;
        const uint32_t d = static_cast<uint32_t>(*p - '0');
        if (w == 0 && d == 0) continue;
        if (nd < 19) {
            w = w * 10 + d;
            ++nd;
        } else {
            ++q;
            trunc |= d != 0;
        }
    }
    if (p < e && *p == '.') {
        ++p;
        for (; p < e && is_digit(*p); ++p) {
            any = true;
            const uint32_t d = static_cast<uint32_t>(*p - '0');
            if (w == 0 && d == 0) {
                --q;
                continue;
            }
            if (nd < 19) {
                w = w * 10 + d;
                ++nd;
                --q;
            } else {
                trunc |= d != 0;
            }
        }
    }
    if (!any) return kTokErr;
    if (p < e && (*p | 0x20) == 'e') {
        const char* t = p + 1;
        bool eneg = false;
        if (t < e && (*t == '+' || *t == '-')) {
            eneg = *t == '-';
            ++t;
        }
        if (t < e && is_digit(*t)) {
            int64_t x = 0;
            for (; t < e && is_digit(*t); ++t)
                if (x < 1000000) x = x * 10 + (*t - '0');
            q += static_cast<int>(eneg ? -x : x);
            p = t;
        }
    }
    if (p != e) return kTokErr;
    if (w == 0) {
        out = __uint_as_float(sign);
        return kTokOk;
    }
    if (q > 38) return kTokErr;    // >= 10^39: rounds to infinity
    if (q < -100) return kTokErr;  // < 10^-81: rounds to zero
    // Clinger: one exact IEEE operation
    if (!trunc && w <= (1ull << 24) && q >= -10 && q <= 10) {
        const float pw = static_cast<float>(kPow10[100 + (q < 0 ? -q : q)]);
        const float fw = static_cast<float>(w);
        const float r = q >= 0 ? __fmul_rn(fw, pw) : __fdiv_rn(fw, pw);
        out = __uint_as_float(__float_as_uint(r) | sign);
        return kTokOk;
    }
    // candidate: (double)w * 10^q, relative error < 2^-50
    const double d = __dmul_rn(static_cast<double>(w), kPow10[100 + q]);
    if (d < 0x1p-151) return kTokErr;                     // rounds to zero
    if (d < 0x1.0000000001p-126) return parse_f32_exact(digits0, e, d, sign, out);  // subnormals (and their edge)
    float c = __double2float_rn(d);
    if ((__float_as_uint(c) & 0x7F800000u) == 0x7F800000u) {
        // candidate overflowed: the value rounds to infinity iff it reaches
        // the midpoint between FLT_MAX and 2^128, (2^25 - 1) 2^103 (a tie
        // rounds to the even 2^128)
        if (cmp_decimal_dyadic(w, q, (1ull << 25) - 1, 103) >= 0) return kTokErr;
        c = __uint_as_float(0x7F7FFFFFu);
    }
    float r;
    if (!round_exact(w, q, c, trunc, r)) return parse_f32_exact(digits0, e, d, sign, out);
    if (trunc) {  // the value lies in (w 10^q, (w+1) 10^q): both ends must agree
        float r2;
        const uint64_t w1 = w + 1;
        const double d1 = __dmul_rn(static_cast<double>(w1), kPow10[100 + q]);
        const float c1 = __double2float_rn(d1);
        if ((__float_as_uint(c1) & 0x7F800000u) == 0x7F800000u) return parse_f32_exact(digits0, e, d, sign, out);
        if (!round_exact(w1, q, c1, false, r2)) return parse_f32_exact(digits0, e, d, sign, out);
        // (w+1) 10^q exactly on a midpoint would round toward it from below
        if (__float_as_uint(r2) != __float_as_uint(r)) return parse_f32_exact(digits0, e, d, sign, out);
        const uint32_t rb = __float_as_uint(r2);
        const uint64_t m2 = (rb & 0x7FFFFFu) | 0x800000u;
        const int e2 = static_cast<int>(rb >> 23) - 150;
        if (cmp_decimal_dyadic(w1, q, 2 * m2 - 1, e2 - 1) == 0 ||
            cmp_decimal_dyadic(w1, q, 2 * m2 + 1, e2 - 1) == 0)
            return parse_f32_exact(digits0, e, d, sign, out);
    }
    if ((__float_as_uint(r) & 0x7F800000u) == 0x7F800000u) return kTokErr;  // rounded to infinity
    out = __uint_as_float(__float_as_uint(r) | sign);
    return kTokOk;
}

}  // namespace parse
}  // namespace asnn_b200
