// Scalar policy for the device kernels: explicit round-to-nearest operations
// (no FMA contraction, so every multiply and add rounds exactly like the
// reference built for x86-64 without -march), the feasibility tolerance of
// NumericTraits (numeric.hpp:53-81), and an order-preserving integer key for
// the adversary ordering of omax.hpp:41-58.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rimdp_dev {

template <class T>
struct Num;

template <>
struct Num<double> {
    using Bits = unsigned long long;
    static constexpr int kKeyWords = 2;
    __host__ __device__ static double tol() { return 1e-9; }
    __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
    __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
    // Value -> unsigned key whose integer order is the ordering the reference
    // sorts by: ascending V for the pessimistic adversary, descending for the
    // optimistic one.  -0.0 and +0.0 map to the same key because the
    // reference compares values with != (ties then fall back to the row).
    __device__ __forceinline__ static Bits key(double v, bool pessimistic) {
        Bits b = static_cast<Bits>(__double_as_longlong(v == 0.0 ? 0.0 : v));
        b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
        return pessimistic ? b : ~b;
    }
    // Inverse of key (a key of -0.0 gives +0.0).
    __device__ __forceinline__ static double value(Bits k, bool pessimistic) {
        if (!pessimistic) k = ~k;
        k = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        return __longlong_as_double(static_cast<long long>(k));
    }
    // Non-negative residuals compare like their bit patterns.
    __device__ __forceinline__ static unsigned long long res_bits(double r) {
        return static_cast<unsigned long long>(__double_as_longlong(r));
    }
    __host__ __device__ static double from_res_bits(unsigned long long b) {
        double d;
        memcpy(&d, &b, sizeof d);
        return d;
    }
};

template <>
struct Num<float> {
    using Bits = unsigned int;
    static constexpr int kKeyWords = 1;
    __host__ __device__ static float tol() { return 1e-5f; }
    __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
    __device__ __forceinline__ static float sub(float a, float b) { return __fsub_rn(a, b); }
    __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ __forceinline__ static Bits key(float v, bool pessimistic) {
        Bits b = static_cast<Bits>(__float_as_int(v == 0.0f ? 0.0f : v));
        b = (b >> 31) ? ~b : (b | 0x80000000u);
        return pessimistic ? b : ~b;
    }
    __device__ __forceinline__ static float value(Bits k, bool pessimistic) {
        if (!pessimistic) k = ~k;
        k = (k >> 31) ? (k & 0x7fffffffu) : ~k;
        return __int_as_float(static_cast<int>(k));
    }
    __device__ __forceinline__ static unsigned long long res_bits(float r) {
        return static_cast<unsigned long long>(static_cast<unsigned>(__float_as_int(r)));
    }
    __host__ __device__ static float from_res_bits(unsigned long long b) {
        unsigned u = static_cast<unsigned>(b);
        float f;
        memcpy(&f, &u, sizeof f);
        return f;
    }
};

// ---------------------------------------------------------------------------
// L2 residency of the value vector.  Per iteration the column kernels stream
// the transition store once (20 B / transition, far larger than the 126 MB
// L2) while gathering V[row] at random (n x 8 B).  Streaming loads carry an
// evict-first policy and the gathers evict-last, so V stays resident in L2
// instead of being evicted by the stream (config 4: V is 80 MB).
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_hint(const float* a, unsigned long long pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_hint(const int* a, unsigned long long pol) {
    int v;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}

// 128-bit (64-bit) vector forms of ld_hint: E consecutive entries of one lane
// in one load.  The caller guarantees the alignment (column offset % E == 0).
__device__ __forceinline__ void ld_hint_vec(const double* a, unsigned long long pol, double (&v)[2]) {
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v[0]), "=d"(v[1]) : "l"(a), "l"(pol));
}
__device__ __forceinline__ void ld_hint_vec(const double* a, unsigned long long pol, double (&v)[4]) {
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v[0]), "=d"(v[1]) : "l"(a), "l"(pol));
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v[2]), "=d"(v[3]) : "l"(a + 2), "l"(pol));
}
__device__ __forceinline__ void ld_hint_vec(const float* a, unsigned long long pol, float (&v)[2]) {
    asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v[0]), "=f"(v[1]) : "l"(a), "l"(pol));
}
__device__ __forceinline__ void ld_hint_vec(const float* a, unsigned long long pol, float (&v)[4]) {
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(a), "l"(pol));
}
__device__ __forceinline__ void ld_hint_vec(const int* a, unsigned long long pol, int (&v)[2]) {
    asm("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v[0]), "=r"(v[1]) : "l"(a), "l"(pol));
}
__device__ __forceinline__ void ld_hint_vec(const int* a, unsigned long long pol, int (&v)[4]) {
    asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(a), "l"(pol));
}

// Entries [j0, j0 + E) of a column (base pointer p, length L) into v: one
// vector load when the run is whole and aligned, else guarded scalar loads.
template <int E, class U>
__device__ __forceinline__ void ld_run(const U* p, int j0, int L, bool aligned, unsigned long long pol, U (&v)[E]) {
    if (aligned && j0 + E <= L) {
        ld_hint_vec(p + j0, pol, v);
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = j0 + e < L ? ld_hint(p + j0 + e, pol) : U(0);
    }
}

// Programmatic dependent launch: the kernels
// of an iteration are launched with programmatic stream serialization, so a
// kernel's blocks can become resident while its predecessor drains.  Every
// such kernel first waits for the predecessor grid to complete (its writes
// are then visible), then lets its own successor launch.  Without the launch
// attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

} // namespace rimdp_dev
