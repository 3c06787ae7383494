// verify.hpp -- the reference's verification recipes as first-class calls on the GPU
// operators.  Mirrors the seismic part of proj/include/sf/verify.hpp
// (adjoint_test :66-85, gradient_test :92-119, bench :123-138) and
// proj/include/sf/slopefit.hpp; the analytic convergence sweeps need FFTW and stay out of
// scope.
#pragma once

#include <vector>

#include "sfb/seismic_ops.hpp"

namespace sfb {

// proj/include/sf/slopefit.hpp:12-50
struct SlopeFit {
    std::vector<double> log_x, log_y;
    double slope = 0.0, intercept = 0.0, residual = 0.0;
};
SlopeFit fit_loglog(const std::vector<double>& x, const std::vector<double>& y);

// <F q, d> vs <q, F^T d> with d = F q (proj/src/verify.cpp:201-253).  fp32 arithmetic on the
// device: rel_err sits at ~1e-6 instead of the reference's 1e-16.
struct AdjointConfig {
    int ndim = 2;
    long n = 64;
    int space_order = 8;
    double h = 10.0;
    long nbl = 10;
    double tn = 300.0;
    double f0 = 0.01;
};
struct AdjointReport {
    double forward_dot = 0, adjoint_dot = 0, rel_err = 0;
};
AdjointReport adjoint_test(const AdjointConfig& cfg = {});

// Taylor remainders of the FWI objective (proj/src/verify.cpp:255-331): eps0 ~ s, eps1 ~ s^2.
// The floating-point floor that removes eps1 points from the second fit is fp32's here.
struct GradientConfig {
    long nx = 81, nz = 61;
    double h = 10.0;
    int space_order = 8;
    long nbl = 30;
    double tn = 450.0;
    double f0 = 0.012;
    // the reference sweeps 1 .. 1e-6 in f64; in fp32 the second-order remainder drowns in
    // round-off below s ~ 1e-2, and s ~ 1 is outside the asymptotic regime
    std::vector<double> steps = {0.32, 0.16, 0.08, 0.04, 0.02, 0.01};
};
struct GradientReport {
    double phi0 = 0, dphi = 0;
    std::vector<double> steps, eps0, eps1;
    std::vector<bool> eps1_fitted;
    SlopeFit fit0{}, fit1{};
    bool fit1_valid = false;
};
GradientReport gradient_test(const GradientConfig& cfg = {});

// Operator metrics per space order in the reference's accounting (proj/src/passes.cpp:
// 318-356: flops = adds + muls of the optimised dense block, bytes = 8 B x distinct
// fields) plus a wall-clock scaling probe n^3 vs (2n)^3 (proj/src/verify.cpp:338-393).
struct BenchConfig {
    std::vector<int> orders = {2, 4, 6, 8, 12};
    long n = 32;
    long steps = 800;
    int wall_order = 8;
    int repeats = 3;
};
struct BenchReport {
    std::vector<int> orders;
    std::vector<double> oi, flops;
    double wall_small = 0, wall_big = 0, wall_ratio = 0;
};
BenchReport bench(const BenchConfig& cfg = {});

}  // namespace sfb
