// TEST INFRASTRUCTURE ONLY — compile-time stand-in for Boost.Multiprecision.
//
// The reference's numeric.hpp:3 includes <boost/multiprecision/cpp_int.hpp>
// for its exact `Rational` scalar (numeric.hpp:17-18, 83-101, 105-170).
// Boost is not installed in this image.  The oracle build only instantiates
// the f64/f32 solver path, which never executes Rational code, but the
// non-template Rational members in numeric.hpp must still compile.  This
// stub supplies those symbols with a fixed-width (__int128) representation.
// It is NOT arbitrary precision and must never be used for rational solves.
#pragma once

#include <cstdint>
#include <limits>
#include <string>
#include <type_traits>

namespace boost {
namespace multiprecision {

class cpp_int {
public:
    __int128 v = 0;
    cpp_int() = default;
    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    cpp_int(I x) : v(static_cast<__int128>(x)) {}

    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) { return fromraw(a.v * b.v); }
    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) { return fromraw(a.v + b.v); }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return fromraw(a.v - b.v); }
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) { return fromraw(a.v / b.v); }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) { return fromraw(a.v % b.v); }
    cpp_int operator-() const { return fromraw(-v); }
    friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v == b.v; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v != b.v; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v < b.v; }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v > b.v; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return a.v <= b.v; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return a.v >= b.v; }

    std::string str() const {
        __int128 x = v;
        bool neg = x < 0;
        if (neg) x = -x;
        std::string s;
        do {
            s.insert(s.begin(), static_cast<char>('0' + static_cast<int>(x % 10)));
            x /= 10;
        } while (x != 0);
        return neg ? "-" + s : s;
    }
    template <class T>
    T convert_to() const { return static_cast<T>(v); }

    static cpp_int fromraw(__int128 x) {
        cpp_int r;
        r.v = x;
        return r;
    }
};

inline cpp_int pow(const cpp_int& b, unsigned e) {
    cpp_int r(1);
    for (unsigned i = 0; i < e; ++i) r = r * b;
    return r;
}

class cpp_rational {
public:
    cpp_int n{0}, d{1};
    cpp_rational() = default;
    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    cpp_rational(I x) : n(x), d(1) {}
    cpp_rational(const cpp_int& x) : n(x), d(1) {}
    cpp_rational(const cpp_int& a, const cpp_int& b) : n(a), d(b) { norm(); }
    explicit cpp_rational(double x) {
        // Exact for dyadic values that fit the 128-bit stand-in.
        int e = 0;
        while (x != static_cast<double>(static_cast<long long>(x)) && e < 60) {
            x *= 2;
            ++e;
        }
        n = cpp_int(static_cast<long long>(x));
        d = cpp_int::fromraw(static_cast<__int128>(1) << e);
        norm();
    }

    cpp_rational operator-() const { return cpp_rational(-n, d); }
    friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.n * b.d + b.n * a.d, a.d * b.d);
    }
    friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.n * b.d - b.n * a.d, a.d * b.d);
    }
    friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.n * b.n, a.d * b.d);
    }
    friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.n * b.d, a.d * b.n);
    }
    cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
    cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
    cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
    cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

    friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
        return a.n == b.n && a.d == b.d;
    }
    friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return !(a == b); }
    friend bool operator<(const cpp_rational& a, const cpp_rational& b) {
        return a.n * b.d < b.n * a.d;
    }
    friend bool operator>(const cpp_rational& a, const cpp_rational& b) { return b < a; }
    friend bool operator<=(const cpp_rational& a, const cpp_rational& b) { return !(b < a); }
    friend bool operator>=(const cpp_rational& a, const cpp_rational& b) { return !(a < b); }

    template <class T>
    T convert_to() const {
        return static_cast<T>(static_cast<long double>(n.v) / static_cast<long double>(d.v));
    }

private:
    void norm() {
        if (d < cpp_int(0)) {
            n = -n;
            d = -d;
        }
        __int128 a = n.v < 0 ? -n.v : n.v, b = d.v;
        while (b != 0) {
            __int128 t = a % b;
            a = b;
            b = t;
        }
        if (a > 1) {
            n.v /= a;
            d.v /= a;
        }
    }
};

inline cpp_int numerator(const cpp_rational& r) { return r.n; }
inline cpp_int denominator(const cpp_rational& r) { return r.d; }

} // namespace multiprecision
} // namespace boost
