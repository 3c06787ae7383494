// fdweights.hpp -- exact centred finite-difference weights (host).
//
// Replaces fd_weights / centered_offsets of the reference (proj/src/fdcoeff.cpp:12-18,
// 60-95), which solves the moment system in Boost rationals.  For the centred stencils
// the hot path uses, the solution has a closed form (Fornberg):
//   d/dx   : w_j = (-1)^(j+1)   (K!)^2 / (j   (K-j)! (K+j)!),  w_-j = -w_j, w_0 = 0
//   d2/dx2 : w_j = 2(-1)^(j+1) (K!)^2 / (j^2 (K-j)! (K+j)!),  w_-j =  w_j, w_0 = -2 sum w_j
// evaluated here in exact 128-bit rational arithmetic and rounded once to double, which
// is what the reference's to_double(Rational) yields (proj/include/sf/rational.hpp:15).
// Pinned against proj/tests/test_symbolic.cpp:52-74 by tests/test_capi_cpu.py.
#pragma once

#include <cstdlib>
#include <vector>

namespace sfb {

struct Frac {
    __int128 n = 0, d = 1;
};

inline __int128 gcd128(__int128 a, __int128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        __int128 t = a % b;
        a = b;
        b = t;
    }
    return a ? a : 1;
}

inline Frac make_frac(__int128 n, __int128 d) {
    if (d < 0) {
        n = -n;
        d = -d;
    }
    __int128 g = gcd128(n, d);
    return Frac{n / g, d / g};
}

inline Frac add(const Frac& a, const Frac& b) {
    __int128 g = gcd128(a.d, b.d);
    return make_frac(a.n * (b.d / g) + b.n * (a.d / g), a.d * (b.d / g));
}

inline double to_double(const Frac& f) {
    // numerators/denominators of the orders supported here stay below 2^53, so one
    // IEEE division rounds correctly
    return double(f.n) / double(f.d);
}

inline __int128 fact(int n) {
    __int128 r = 1;
    for (int i = 2; i <= n; ++i) r *= i;
    return r;
}

// w_0..w_K of the centred stencil of accuracy `order` for derivative 1 or 2.
inline bool centred_weights(int deriv, int order, std::vector<Frac>& out) {
    if (order < 2 || order % 2 != 0 || order > 16 || (deriv != 1 && deriv != 2)) return false;
    const int K = order / 2;
    out.assign(K + 1, Frac{});
    const __int128 kf2 = fact(K) * fact(K);
    Frac sum{0, 1};
    for (int j = 1; j <= K; ++j) {
        __int128 num = (deriv == 2 ? 2 : 1) * kf2 * ((j % 2) ? 1 : -1);
        __int128 den = (deriv == 2 ? __int128(j) * j : __int128(j)) * fact(K - j) * fact(K + j);
        out[j] = make_frac(num, den);
        sum = add(sum, out[j]);
    }
    out[0] = deriv == 2 ? make_frac(-2 * sum.n, sum.d) : Frac{0, 1};
    return true;
}

}  // namespace sfb
