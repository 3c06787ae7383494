// verify.cpp -- adjoint_test / gradient_test / bench of the host layer (include/sfb/verify.hpp).
#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <numeric>

#include "engine.hpp"
#include "sfb/verify.hpp"

namespace sfb {

// Least-squares line through (log x, log y) -- the contract of proj/include/sf/slopefit.hpp
// (positive values, strictly monotone abscissae, at least three points; residual = rms
// distance of the points from the line).  Computed from centred sums.
SlopeFit fit_loglog(const std::vector<double>& x, const std::vector<double>& y) {
    const std::size_t n = x.size();
    if (y.size() != n) throw ParameterError("fit_loglog: x and y differ in length");
    if (n < 3) throw ParameterError("fit_loglog: a slope needs three points or more");
    auto positive = [](double v) { return v > 0.0; };
    if (!std::all_of(x.begin(), x.end(), positive) || !std::all_of(y.begin(), y.end(), positive))
        throw ParameterError("fit_loglog: logarithms need positive values");
    const bool up = std::adjacent_find(x.begin(), x.end(), std::greater_equal<double>()) == x.end();
    const bool down = std::adjacent_find(x.begin(), x.end(), std::less_equal<double>()) == x.end();
    if (!up && !down) throw ParameterError("fit_loglog: abscissae must be strictly monotone");
    SlopeFit f;
    f.log_x.resize(n);
    f.log_y.resize(n);
    std::transform(x.begin(), x.end(), f.log_x.begin(), [](double v) { return std::log(v); });
    std::transform(y.begin(), y.end(), f.log_y.begin(), [](double v) { return std::log(v); });
    const double mx = std::accumulate(f.log_x.begin(), f.log_x.end(), 0.0) / double(n);
    const double my = std::accumulate(f.log_y.begin(), f.log_y.end(), 0.0) / double(n);
    double cxx = 0.0, cxy = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        cxx += (f.log_x[i] - mx) * (f.log_x[i] - mx);
        cxy += (f.log_x[i] - mx) * (f.log_y[i] - my);
    }
    f.slope = cxy / cxx;
    f.intercept = my - f.slope * mx;
    double miss = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        const double off = f.log_y[i] - (f.intercept + f.slope * f.log_x[i]);
        miss += off * off;
    }
    f.residual = std::sqrt(miss / double(n));
    return f;
}

// ---- verification recipes -------------------------------------------------------------------
// The two recipes are the reference's (proj/src/verify.cpp:201-331, pinned by
// proj/tests/test_verify.cpp): same media, acquisition and time steps, so the numbers are
// comparable.  They run differently here: each recipe builds ONE engine and drives it through
// the C-ABI, rebinding the model between evaluations, instead of rebuilding an operator (and a
// device plan) for every run.

namespace {

// depth-only velocity profile broadcast over a grid whose LAST axis is depth
std::vector<double> layered(const std::vector<long>& shape, double h,
                            const std::function<double(double)>& v_of_depth) {
    const long nz = shape.back();
    std::vector<double> column(static_cast<std::size_t>(nz));
    for (long z = 0; z < nz; ++z) column[std::size_t(z)] = v_of_depth(double(z) * h);
    std::size_t columns = 1;
    for (std::size_t a = 0; a + 1 < shape.size(); ++a) columns *= std::size_t(shape[a]);
    std::vector<double> vel;
    vel.reserve(columns * column.size());
    for (std::size_t c = 0; c < columns; ++c) vel.insert(vel.end(), column.begin(), column.end());
    return vel;
}

// a line of receivers along axis 0 at fixed values of the other coordinates
std::vector<double> receiver_line(long n, double h, std::vector<double> other) {
    std::vector<double> rec;
    for (long i = 0; i < n; ++i) {
        rec.push_back(double(i) * h);
        rec.insert(rec.end(), other.begin(), other.end());
    }
    return rec;
}

double dot(const std::vector<double>& a, const std::vector<double>& b) {
    return std::inner_product(a.begin(), a.end(), b.begin(), 0.0);
}

}  // namespace

// <F q, d> against <q, F^T d> for d = F q: a two-layer medium (interface at half depth),
// an off-lattice source near the top, one receiver per lattice column at depth 4.5 h,
// dt = 0.8 of the stable limit.
AdjointReport adjoint_test(const AdjointConfig& cfg) {
    if (cfg.ndim != 2 && cfg.ndim != 3) throw ParameterError("adjoint_test: ndim must be 2 or 3");
    const std::size_t rank = std::size_t(cfg.ndim);
    const std::vector<long> shape(rank, cfg.n);
    const long half = cfg.n / 2;
    SeismicModel model(shape, std::vector<double>(rank, cfg.h), std::vector<double>(rank, 0.0),
                       layered(shape, cfg.h, [&](double depth) { return depth < double(half) * cfg.h ? 1.5 : 2.5; }),
                       cfg.nbl, cfg.space_order);
    const double mid = 0.5 * double(cfg.n - 1) * cfg.h;
    std::vector<double> src(rank, mid), fixed;
    src.front() += 0.37 * cfg.h;
    src.back() = 2.13 * cfg.h;
    if (rank == 3) fixed.push_back(mid);
    fixed.push_back(4.5 * cfg.h);
    AcquisitionGeometry geom(model, src, receiver_line(cfg.n, cfg.h, fixed), 0.0, cfg.tn,
                             0.8 * model.critical_dt(cfg.space_order), cfg.f0);

    Engine eng(model, geom, cfg.space_order);   // forward and adjoint share the plan
    const std::vector<double>& q = geom.src()->traces();
    std::vector<double>& d = geom.rec()->traces();
    std::vector<double> back(q.size());
    eng.check(sfb_forward(eng.plan(), q.data(), d.data(), 0, nullptr));
    eng.check(sfb_adjoint(eng.plan(), d.data(), back.data(), nullptr));
    AdjointReport rep;
    rep.forward_dot = dot(d, d);
    rep.adjoint_dot = dot(q, back);
    rep.rel_err = std::abs(rep.forward_dot - rep.adjoint_dot) /
                  std::max(std::abs(rep.forward_dot), std::numeric_limits<double>::min());
    return rep;
}

// Taylor test of the FWI gradient.  phi(m0 + s dm) - phi(m0) must shrink like s, and the
// remainder after the gradient term like s^2; dm points from a smooth background (tanh, 80 m
// transition) to the two-layer truth that produced the data.  Source at mid-width, depth 2 h;
// one receiver per lattice column at the same depth; dt = 0.75 of the stable limit.
GradientReport gradient_test(const GradientConfig& cfg) {
    const std::vector<long> shape{cfg.nx, cfg.nz};
    const double width = double(cfg.nx - 1) * cfg.h, interface = 0.5 * double(cfg.nz - 1) * cfg.h;
    SeismicModel model(shape, {cfg.h, cfg.h}, {0.0, 0.0},
                       layered(shape, cfg.h, [&](double z) { return z < interface ? 1.5 : 2.5; }),
                       cfg.nbl, cfg.space_order);
    const std::vector<double> m_true = model.physical_m();
    AcquisitionGeometry geom(model, {0.5 * width, 2.0 * cfg.h},
                             receiver_line(cfg.nx, cfg.h, {2.0 * cfg.h}), 0.0, cfg.tn,
                             0.75 * model.critical_dt(cfg.space_order), cfg.f0);
    Engine eng(model, geom, cfg.space_order);
    const double* wavelet = geom.src()->traces().data();
    std::vector<double>& predicted = geom.rec()->traces();

    // data of the true medium
    eng.check(sfb_forward(eng.plan(), wavelet, predicted.data(), 0, nullptr));
    const std::vector<double> observed = predicted;

    // objective and gradient at the background
    model.set_velocity(layered(shape, cfg.h, [&](double z) {
        return 2.0 + 0.5 * std::tanh((z - interface) / 80.0);
    }));
    const std::vector<double> m0 = model.physical_m();
    std::vector<double> dm(m0.size());
    std::transform(m_true.begin(), m_true.end(), m0.begin(), dm.begin(), std::minus<double>());
    const GradientResult at_m0 = fwi_gradient(model, geom, observed, cfg.space_order);
    GradientReport rep;
    rep.phi0 = at_m0.objective;
    rep.dphi = dot(at_m0.gradient, dm);
    rep.steps = cfg.steps;

    // objective along the line m0 + s dm, on the one engine
    std::vector<double> m_s(m0.size());
    for (double s : cfg.steps) {
        std::transform(m0.begin(), m0.end(), dm.begin(), m_s.begin(),
                       [s](double base, double dir) { return base + s * dir; });
        model.set_physical_m(m_s);
        eng.rebind_model(model);
        eng.check(sfb_forward(eng.plan(), wavelet, predicted.data(), 0, nullptr));
        const double change = objective(*geom.rec(), observed) - rep.phi0;
        rep.eps0.push_back(std::abs(change));
        rep.eps1.push_back(std::abs(change - s * rep.dphi));
    }
    model.set_physical_m(m0);

    // Second-order remainders at the round-off level of phi0 say nothing about the gradient.
    // The device computes in fp32, so the floor is 100 fp32 ulps of phi0 (the f64 reference
    // uses 100 f64 ulps); points under it stay out of the quadratic fit.
    const double floor = 100.0 * double(std::numeric_limits<float>::epsilon()) * rep.phi0;
    std::vector<double> s_kept, eps1_kept;
    for (std::size_t i = 0; i < rep.eps1.size(); ++i) {
        rep.eps1_fitted.push_back(rep.eps1[i] > floor);
        if (rep.eps1_fitted.back()) {
            s_kept.push_back(cfg.steps[i]);
            eps1_kept.push_back(rep.eps1[i]);
        }
    }
    rep.fit0 = fit_loglog(cfg.steps, rep.eps0);
    rep.fit1_valid = s_kept.size() >= 3;
    if (rep.fit1_valid) rep.fit1 = fit_loglog(s_kept, eps1_kept);
    return rep;
}

namespace {

// bare acoustic stencil on an n^3 grid, m = 1/2.25, no damping (proj/src/verify.cpp:338-376);
// seconds of `steps` dense updates, median of `repeats`
double timed_run(long n, int order, long steps, int repeats) {
    std::vector<double> vel(std::size_t(n) * n * n, 1.5);
    SeismicModel model({n, n, n}, {10.0, 10.0, 10.0}, {0.0, 0.0, 0.0}, vel, 0, order);
    const double dt = 0.5 * model.critical_dt(order);
    const double c = 5.0 * double(n - 1);
    AcquisitionGeometry geom(model, {c, c, c}, {c, c, 10.0}, 0.0, double(steps + 1) * dt + 0.5 * dt,
                             dt, 0.01);
    Engine eng(model, geom, order);
    std::vector<double> times;
    for (int r = 0; r < std::max(repeats, 1); ++r) {
        eng.check(sfb_upload_traces(eng.plan(), SFB_CLOUD_SRC, geom.src()->traces().data()));
        eng.check(sfb_step_begin(eng.plan(), SFB_OP_FORWARD, 0));
        sfb_report rep{};
        eng.check(sfb_time_stencil(eng.plan(), SFB_OP_FORWARD, 1, 1 + steps, &rep));
        times.push_back(rep.seconds);
    }
    auto median = times.begin() + long(times.size() / 2);
    std::nth_element(times.begin(), median, times.end());
    return *median;
}

}  // namespace

BenchReport bench(const BenchConfig& cfg) {
    BenchReport rep;
    for (int k : cfg.orders) {
        check_space_order(k);
        // reference accounting for the 3-D damped acoustic update:
        // 3 K D + 3 D + 11 flops, 8 B x {u, m, damp, inv0}
        const double flops = 3.0 * (k / 2) * 3 + 3.0 * 3 + 11.0;
        rep.orders.push_back(k);
        rep.flops.push_back(flops);
        rep.oi.push_back(flops / 32.0);
    }
    rep.wall_small = timed_run(cfg.n, cfg.wall_order, cfg.steps, cfg.repeats);
    rep.wall_big = timed_run(2 * cfg.n, cfg.wall_order, cfg.steps, cfg.repeats);
    rep.wall_ratio = rep.wall_big / std::max(rep.wall_small, 1e-12);
    return rep;
}

}  // namespace sfb
