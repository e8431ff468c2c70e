// gen_core.h -- the bench corpora's per-node generator steps, shared verbatim
// by the host generators (netgen.cpp, g++ -ffp-contract=off) and the device
// generators (gen.cu, nvcc -fmad=false): same integer RNG, same IEEE double
// operations in the same order, so host and device produce byte-identical
// networks (tests/test_gpu_gen.py).
//
//  * Rng: SplitMix64 (rng.hpp:10-38 of the reference), counter-seeded per node;
//  * det_pow: u^e for u in (0, 1], e < 0, from +, -, *, / and exact bit
//    manipulation only (no libm): identical on both sides, ~1e-15 relative
//    (the Pareto draw only keeps floor(xm * u^e));
//  * pl_draw: config 4's per-target source draws;
//  * mlp_draw: config 2's per-target edges.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define ASNN_HD __host__ __device__ __forceinline__
#else
#define ASNN_HD inline
#endif

namespace asnn_gen {

struct Rng {
    uint64_t s;
    ASNN_HD uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    ASNN_HD uint64_t bounded(uint64_t n) {  // rejection sampling, unbiased
        const uint64_t threshold = (0 - n) % n;
        for (;;) {
            const uint64_t r = next();
            if (r >= threshold) return r % n;
        }
    }
    ASNN_HD double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    ASNN_HD float uniform(float lo, float hi) {
        return static_cast<float>(lo + uniform01() * (static_cast<double>(hi) - lo));
    }
};

ASNN_HD Rng node_rng(uint64_t seed, uint32_t v, uint64_t salt) {
    return Rng{seed ^ (0x9E3779B97F4A7C15ull * (static_cast<uint64_t>(v) + 1)) ^ salt};
}

ASNN_HD double bits_to_double(uint64_t b) {
    union {
        uint64_t u;
        double d;
    } x;
    x.u = b;
    return x.d;
}
ASNN_HD uint64_t double_to_bits(double d) {
    union {
        uint64_t u;
        double d;
    } x;
    x.d = d;
    return x.u;
}

constexpr double kLn2Hi = 6.93147180369123816490e-01;  // trailing zeros: k * kLn2Hi exact for |k| < 2^11
constexpr double kLn2Lo = 1.90821492927058770002e-10;
constexpr double kInvLn2 = 1.44269504088896338700e+00;
constexpr double kSqrt2 = 1.41421356237309514547e+00;

// ln(u) for a normal u > 0: u = m * 2^k with m in [sqrt(1/2), sqrt(2)),
// ln(m) = 2 atanh(s), s = (m - 1) / (m + 1), |s| < 0.1716 (series to s^25).
ASNN_HD double det_log(double u) {
    const uint64_t b = double_to_bits(u);
    int k = static_cast<int>((b >> 52) & 0x7FF) - 1023;
    double m = bits_to_double((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
    if (m > kSqrt2) {
        m = m * 0.5;
        k += 1;
    }
    const double s = (m - 1.0) / (m + 1.0);
    const double s2 = s * s;
    double p = 1.0 / 25.0;
    p = p * s2 + 1.0 / 23.0;
    p = p * s2 + 1.0 / 21.0;
    p = p * s2 + 1.0 / 19.0;
    p = p * s2 + 1.0 / 17.0;
    p = p * s2 + 1.0 / 15.0;
    p = p * s2 + 1.0 / 13.0;
    p = p * s2 + 1.0 / 11.0;
    p = p * s2 + 1.0 / 9.0;
    p = p * s2 + 1.0 / 7.0;
    p = p * s2 + 1.0 / 5.0;
    p = p * s2 + 1.0 / 3.0;
    const double lm = 2.0 * s + 2.0 * s * (s2 * p);
    return static_cast<double>(k) * kLn2Hi + (lm + static_cast<double>(k) * kLn2Lo);
}

// e^t for |t| < 700: t = j ln2 + r, |r| <= ln2 / 2, Taylor series to r^17.
ASNN_HD double det_exp(double t) {
    const double jf = t * kInvLn2;
    const int j = static_cast<int>(jf < 0.0 ? jf - 0.5 : jf + 0.5);
    const double r = (t - static_cast<double>(j) * kLn2Hi) - static_cast<double>(j) * kLn2Lo;
    double p = 1.0 / 355687428096000.0;  // 1/17!
    p = p * r + 1.0 / 20922789888000.0;  // 1/16!
    p = p * r + 1.0 / 1307674368000.0;
    p = p * r + 1.0 / 87178291200.0;
    p = p * r + 1.0 / 6227020800.0;
    p = p * r + 1.0 / 479001600.0;
    p = p * r + 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    return p * bits_to_double(static_cast<uint64_t>(j + 1023) << 52);
}

// u^e, u in (0, 1], e < 0 (the Pareto inverse CDF; result in [1, 2^(53/alpha)]).
ASNN_HD double det_pow(double u, double e) { return det_exp(e * det_log(u)); }

// ---- config 4: banded power-law ASNN ---------------------------------------------------
struct PowerlawSpec {
    const uint32_t* starts;  // [bands + 1] band boundaries (band 0 = inputs, last = outputs)
    uint32_t bands;
    double xm;               // Pareto scale of the extra-source count
    double alpha;
    uint64_t seed;
};

constexpr uint64_t kSaltSucc = 0x5A5A5A5A5A5A5A5Aull;
constexpr uint64_t kSaltSrc = 0xC3C3C3C3C3C3C3C3ull;
constexpr uint64_t kSaltMlp = 0x3C3C3C3C3C3C3C3Cull;

ASNN_HD uint32_t band_of(const uint32_t* starts, uint32_t bands, uint32_t id) {
    // upper_bound(starts[0..bands], id) - 1
    uint32_t lo = 0, hi = bands + 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (starts[mid] <= id) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

// Mandatory successor of non-output node v (pins every node to an output).
ASNN_HD uint32_t pl_succ(const PowerlawSpec& s, uint32_t v) {
    const uint32_t b = band_of(s.starts, s.bands, v);
    Rng r = node_rng(s.seed, v, kSaltSucc);
    return s.starts[b + 1] + static_cast<uint32_t>(r.bounded(s.starts[b + 2] - s.starts[b + 1]));
}

// Sources of non-input target t other than the nodes that picked t as their
// mandatory successor: emit(src) for the mandatory predecessor (band b-1)
// and the Pareto(alpha)-many extra sources drawn from [0, start(b)) (dense
// Bernoulli scan when that is more than half of them).  Returns the stream
// after the source draws (the weights follow it).
template <class Emit>
ASNN_HD Rng pl_draw(const PowerlawSpec& s, uint32_t t, Emit&& emit) {
    const uint32_t b = band_of(s.starts, s.bands, t);
    const uint32_t avail = s.starts[b];
    Rng r = node_rng(s.seed, t, kSaltSrc);
    emit(s.starts[b - 1] + static_cast<uint32_t>(r.bounded(s.starts[b] - s.starts[b - 1])));
    const double u = 1.0 - r.uniform01();  // (0, 1]
    // min(floor(xm * u^(-1/alpha)), cap) -- floor of a value in [0, cap) is exact
    const double cap = static_cast<double>(avail < (1u << 20) ? avail : (1u << 20));
    double d = 0.0;
    if (s.xm > 0.0) {
        const double y = s.xm * det_pow(u, -1.0 / s.alpha);
        d = y >= cap ? cap : static_cast<double>(static_cast<uint64_t>(y));
    }
    const uint32_t k = static_cast<uint32_t>(d);
    if (k >= avail / 2) {
        const double q = static_cast<double>(k) / avail;
        for (uint32_t x = 0; x < avail; ++x)
            if (r.uniform01() < q) emit(x);
    } else {
        for (uint32_t i = 0; i < k; ++i) emit(static_cast<uint32_t>(r.bounded(avail)));
    }
    return r;
}

// ---- config 2: pruned-MLP-style network --------------------------------------------------
// Target t (layer t / width >= 1) links to each node of the previous layer
// with probability p (ascending sources, a weight drawn right after each
// accepted link), at least one (a uniform pick if none was accepted).
template <class Emit>
ASNN_HD uint32_t mlp_draw(uint64_t seed, uint32_t width, double p, uint32_t t, Emit&& emit) {
    const uint32_t base = (t / width - 1) * width;
    Rng r = node_rng(seed, t, kSaltMlp);
    uint32_t n = 0;
    for (uint32_t j = 0; j < width; ++j)
        if (r.uniform01() < p) {
            const float w = r.uniform(-1.0f, 1.0f);
            emit(base + j, w);
            ++n;
        }
    if (n == 0) {
        const uint32_t j = static_cast<uint32_t>(r.bounded(width));
        emit(base + j, r.uniform(-1.0f, 1.0f));
        n = 1;
    }
    return n;
}

}  // namespace asnn_gen
