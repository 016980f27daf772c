// Counter-based synthetic IMDP generator for the workloads the reference's
// random_imdp (random_model.hpp:42-101) cannot express: BASELINE config 4
// (10M states x 8 actions x 64 successors, 5.12e9 transitions: int64
// colptr, > 100 GB) and config 5 (power-law successor counts on [1, 4096]).
// See DESIGN.md "Workloads".
//
// Every random draw is a pure function of (seed, column, stream, index), so
// a column can be produced by any thread on any device — or on the host, for
// sampled parity checks — without generating its predecessors.  The same
// source compiles for host and device; every floating-point operation is an
// explicit round-to-nearest op (no FMA contraction on either side), so host
// and device produce bit-identical columns.
//
// Laws (per column c of state s = c / actions):
//   law 0 (fixed support k): rows = one uniform draw in each of k equal
//     strata of [0, n) — distinct and increasing by construction;
//     lower = u * lower_scale, upper = min(lower + v * upper_scale, 1)
//     (the reference generator's value law with scale = lower_scale).
//   law 1 (power law): k ~ P(k) ~ k^-alpha on [1, kmax] by inverse CDF over
//     an integer threshold table (identical on host and device); rows
//     stratified as above; lower = u * lower_scale / k,
//     upper = min(lower + v * upper_scale / k, 1), k = 1 -> upper = 1.
//     A draw whose upper bounds sum below 1 is redrawn with the next
//     attempt counter (the reference generator's rejection, random_model.hpp:62-86).
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#ifdef __CUDACC__
#define RIMDP_HD __host__ __device__ __forceinline__
#else
#define RIMDP_HD inline
#endif

namespace rimdp_gen {

constexpr int kMaxK = 1 << 13;       // largest power-law support
constexpr int kCdfSize = kMaxK + 1;  // thresholds for k = 1 .. kmax

RIMDP_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
RIMDP_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
RIMDP_HD double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}

RIMDP_HD uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Independent 64-bit draw for (seed, column, stream, index).
RIMDP_HD uint64_t draw(uint64_t seed, uint64_t col, uint32_t stream, uint32_t idx) {
    uint64_t h = mix64(seed ^ 0x243f6a8885a308d3ull);
    h = mix64(h ^ col);
    h = mix64(h ^ ((static_cast<uint64_t>(stream) << 32) | idx));
    return h;
}

// Uniform [0, 1) with 53 random bits (random_model.hpp:34-36 convention).
RIMDP_HD double u01(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

struct Params {
    int32_t num_states;
    int32_t actions;
    int32_t law;
    int32_t support;       // law 0
    int32_t kmax;          // law 1
    double lower_scale;
    double upper_scale;
    uint64_t seed;
};

enum Stream : uint32_t { kLen = 1, kRow = 2, kLow = 3, kUp = 4 };

// Number of entries of column c.  cdf[k-1] = floor(2^64 * P(K <= k)) for law 1.
RIMDP_HD int column_length(const Params& p, const uint64_t* cdf, int64_t c) {
    if (p.law == 0) return p.support < p.num_states ? p.support : p.num_states;
    const uint64_t u = draw(p.seed, static_cast<uint64_t>(c), kLen, 0);
    // smallest k with u < cdf[k-1]
    int lo = 0, hi = p.kmax - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (u < cdf[mid]) hi = mid;
        else lo = mid + 1;
    }
    const int k = lo + 1;
    return k < p.num_states ? k : p.num_states;
}

// Row of entry i of a k-entry column: one draw in stratum i of [0, n).
RIMDP_HD int32_t column_row(const Params& p, int64_t c, int k, int i, uint32_t attempt) {
    const int64_t n = p.num_states;
    const int64_t a = (static_cast<int64_t>(i) * n) / k, b = (static_cast<int64_t>(i + 1) * n) / k;
    const uint64_t u = draw(p.seed, static_cast<uint64_t>(c), kRow + 8u * attempt, static_cast<uint32_t>(i));
    return static_cast<int32_t>(a + static_cast<int64_t>(u % static_cast<uint64_t>(b - a)));
}

RIMDP_HD void column_bounds(const Params& p, int64_t c, int k, int i, uint32_t attempt, double& lo, double& up) {
    const double u = u01(draw(p.seed, static_cast<uint64_t>(c), kLow + 8u * attempt, static_cast<uint32_t>(i)));
    const double v = u01(draw(p.seed, static_cast<uint64_t>(c), kUp + 8u * attempt, static_cast<uint32_t>(i)));
    if (p.law == 0) {
        lo = dmul(u, p.lower_scale);
        up = dadd(lo, dmul(v, p.upper_scale));
    } else {
        const double kk = static_cast<double>(k);
        lo = ddiv(dmul(u, p.lower_scale), kk);
        up = k == 1 ? 1.0 : dadd(lo, ddiv(dmul(v, p.upper_scale), kk));
    }
    if (up > 1.0) up = 1.0;
}

// Writes column c (k entries) and returns the attempt used; the upper bounds
// of the returned draw sum to >= 1 (feasible, Sum lower <= 1 by the laws).
template <class T>
RIMDP_HD uint32_t write_column(const Params& p, int64_t c, int k, int32_t* rows, T* lower, T* upper) {
    for (uint32_t attempt = 0;; ++attempt) {
        double us = 0.0, ls = 0.0;
        for (int i = 0; i < k; ++i) {
            double lo, up;
            column_bounds(p, c, k, i, attempt, lo, up);
            const T l = static_cast<T>(lo), u = static_cast<T>(up);
            ls = dadd(ls, static_cast<double>(l));
            us = dadd(us, static_cast<double>(u));
        }
        if ((us >= 1.0 && ls <= 1.0) || attempt >= 64) {
            for (int i = 0; i < k; ++i) {
                double lo, up;
                column_bounds(p, c, k, i, attempt, lo, up);
                rows[i] = column_row(p, c, k, i, attempt);
                lower[i] = static_cast<T>(lo);
                upper[i] = attempt >= 64 ? static_cast<T>(1) : static_cast<T>(up);
            }
            return attempt;
        }
    }
}

// Host only: the law-1 threshold table, cdf[k-1] = floor(2^64 P(K <= k)) with
// P(K = k) ~ k^-alpha on [1, kmax] (long double accumulation; the last
// threshold saturates so every draw lands in [1, kmax]).  Shared by the
// engine (csrc/engine.cu) and the CPU checker's workload builder
// (oracle/ref_capi.cpp), so both produce the same columns.
inline std::vector<uint64_t> power_law_cdf(int kmax, double alpha) {
    std::vector<long double> w(kmax);
    long double z = 0;
    for (int k = 1; k <= kmax; ++k) z += (w[k - 1] = powl((long double)k, -(long double)alpha));
    std::vector<uint64_t> cdf(kmax);
    long double acc = 0;
    for (int k = 1; k <= kmax; ++k) {
        acc += w[k - 1];
        const long double f = acc / z * 18446744073709551616.0L;
        cdf[k - 1] = (k == kmax || f >= 18446744073709551615.0L) ? ~0ull : (uint64_t)f;
    }
    return cdf;
}

} // namespace rimdp_gen
