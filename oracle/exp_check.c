/*
 * oracle/exp_check.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Exhaustive check that the device exp restatement
 * (paper_2005_04347_b200/csrc/exp_glibc.h, here compiled for the host with
 * the same operation sequence) returns the host libm's exp(t) bit for bit for
 * every argument sigmoid32 can produce, t = -4.97 * (double)f over all 2^32
 * float bit patterns f (network.hpp:45), and that sigmoid32 built on it equals
 * the reference's sigmoid32 (network.hpp:54-59) for all of them.
 *
 *   gcc -O2 -fopenmp -ffp-contract=off -mfma -Ipaper_2005_04347_b200/csrc \
 *       oracle/exp_check.c -o oracle/_ref/exp_check -lm && oracle/_ref/exp_check
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "exp_glibc.h"

static const uint64_t kTab[256] = {
#include "exp_table.inc"
};

static float sig32(double e) {
    /* network.hpp:44-59 given e = exp(-4.97 x) */
    double v = 1.0 / (1.0 + e);
    if (v <= 0.0) v = DBL_TRUE_MIN;
    if (v >= 1.0) v = 1.0 - DBL_EPSILON / 2;
    float f = (float)v;
    if (f <= 0.0f) f = FLT_TRUE_MIN;
    if (f >= 1.0f) f = 1.0f - FLT_EPSILON / 2;
    return f;
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (1ull << 32);
    unsigned long long exp_diff = 0, sig_diff = 0, first = ~0ull;
#pragma omp parallel for schedule(static, 1 << 16) reduction(+ : exp_diff, sig_diff) reduction(min : first)
    for (long long i = 0; i < (long long)n; ++i) {
        uint32_t b = (uint32_t)i;
        float f;
        memcpy(&f, &b, 4);
        if (isnan(f)) continue;
        const double t = -4.97 * (double)f;
        const double a = exp(t);
        const double g = exp_glibc(t, kTab);
        uint64_t ua, ug;
        memcpy(&ua, &a, 8);
        memcpy(&ug, &g, 8);
        if (ua != ug) {
            ++exp_diff;
            if ((unsigned long long)i < first) first = (unsigned long long)i;
        }
        const float sa = sig32(a), sg = sig32(g);
        uint32_t fa, fg;
        memcpy(&fa, &sa, 4);
        memcpy(&fg, &sg, 4);
        sig_diff += fa != fg;
    }
    printf("{\"inputs\": %llu, \"exp_mismatches\": %llu, \"sigmoid32_mismatches\": %llu, "
           "\"first_mismatch_bits\": %lld}\n",
           (unsigned long long)n, exp_diff, sig_diff, exp_diff ? (long long)first : -1);
    return exp_diff || sig_diff;
}
