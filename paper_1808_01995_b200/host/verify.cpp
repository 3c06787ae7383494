// verify.cpp -- adjoint_test / gradient_test / bench of the host layer (include/sfb/verify.hpp).
#include <algorithm>
#include <cmath>
#include <limits>

#include "engine.hpp"
#include "sfb/verify.hpp"

namespace sfb {

// proj/include/sf/slopefit.hpp:20-50: least-squares line through (log x, log y)
SlopeFit fit_loglog(const std::vector<double>& x, const std::vector<double>& y) {
    if (x.size() != y.size()) throw ParameterError("fit_loglog: size mismatch");
    if (x.size() < 3) throw ParameterError("fit_loglog: need at least 3 points");
    const bool rising = x[1] > x[0];
    for (std::size_t i = 0; i < x.size(); ++i) {
        if (!(x[i] > 0.0) || !(y[i] > 0.0)) throw ParameterError("fit_loglog: values must be positive");
        if (i > 0 && (x[i] == x[i - 1] || (x[i] > x[i - 1]) != rising))
            throw ParameterError("fit_loglog: x must be strictly monotone");
    }
    SlopeFit f;
    const double n = double(x.size());
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (std::size_t i = 0; i < x.size(); ++i) {
        f.log_x.push_back(std::log(x[i]));
        f.log_y.push_back(std::log(y[i]));
        sx += f.log_x[i];
        sy += f.log_y[i];
        sxx += f.log_x[i] * f.log_x[i];
        sxy += f.log_x[i] * f.log_y[i];
    }
    f.slope = (n * sxy - sx * sy) / (n * sxx - sx * sx);
    f.intercept = (sy - f.slope * sx) / n;
    double ss = 0;
    for (std::size_t i = 0; i < x.size(); ++i) {
        const double d = f.log_y[i] - (f.slope * f.log_x[i] + f.intercept);
        ss += d * d;
    }
    f.residual = std::sqrt(ss / n);
    return f;
}

// proj/src/verify.cpp:201-253: two layers split on the last axis, off-lattice source, a
// receiver line at depth 4.5 h, dt = 0.8 critical
AdjointReport adjoint_test(const AdjointConfig& cfg) {
    if (cfg.ndim != 2 && cfg.ndim != 3) throw ParameterError("adjoint_test: ndim must be 2 or 3");
    const long n = cfg.n;
    const std::size_t nd = std::size_t(cfg.ndim);
    std::size_t npts = 1;
    for (std::size_t d = 0; d < nd; ++d) npts *= std::size_t(n);
    std::vector<double> vel(npts);
    for (std::size_t i = 0; i < npts; ++i) vel[i] = long(i % std::size_t(n)) < n / 2 ? 1.5 : 2.5;
    SeismicModel model(std::vector<long>(nd, n), std::vector<double>(nd, cfg.h),
                       std::vector<double>(nd, 0.0), vel, cfg.nbl, cfg.space_order);
    const double L = double(n - 1) * cfg.h;
    std::vector<double> src, rec;
    if (cfg.ndim == 2) {
        src = {0.5 * L + 0.37 * cfg.h, 2.13 * cfg.h};
        for (long i = 0; i < n; ++i) rec.insert(rec.end(), {double(i) * cfg.h, 4.5 * cfg.h});
    } else {
        src = {0.5 * L + 0.37 * cfg.h, 0.5 * L, 2.13 * cfg.h};
        for (long i = 0; i < n; ++i) rec.insert(rec.end(), {double(i) * cfg.h, 0.5 * L, 4.5 * cfg.h});
    }
    const double dt = 0.8 * model.critical_dt(cfg.space_order);
    AcquisitionGeometry geom(model, src, rec, 0.0, cfg.tn, dt, cfg.f0);
    WaveOp fwd = forward_operator(model, geom, cfg.space_order);
    run_wave(fwd);
    AdjointReport rep;
    for (double d : geom.rec()->traces()) rep.forward_dot += d * d;
    WaveOp adj = adjoint_operator(model, geom, cfg.space_order);  // injects rec = F q
    run_wave(adj);
    const std::vector<double>& q = geom.src()->traces();
    const std::vector<double>& a = adj.smp->traces();
    for (std::size_t i = 0; i < q.size(); ++i) rep.adjoint_dot += q[i] * a[i];
    rep.rel_err = std::abs(rep.forward_dot - rep.adjoint_dot) /
                  std::max(std::abs(rep.forward_dot), std::numeric_limits<double>::min());
    return rep;
}

// proj/src/verify.cpp:255-331
GradientReport gradient_test(const GradientConfig& cfg) {
    const long nx = cfg.nx, nz = cfg.nz;
    const double h = cfg.h, lx = double(nx - 1) * h, lz = double(nz - 1) * h;
    std::vector<double> vel_true(std::size_t(nx) * nz), vel_start(vel_true.size());
    for (long x = 0; x < nx; ++x)
        for (long z = 0; z < nz; ++z) {
            const double depth = double(z) * h;
            const std::size_t i = std::size_t(x) * nz + z;
            vel_true[i] = depth < 0.5 * lz ? 1.5 : 2.5;
            vel_start[i] = 2.0 + 0.5 * std::tanh((depth - 0.5 * lz) / 80.0);  // smooth background
        }
    SeismicModel model({nx, nz}, {h, h}, {0.0, 0.0}, vel_true, cfg.nbl, cfg.space_order);
    const std::vector<double> m_true = model.physical_m();
    const double dt = 0.75 * model.critical_dt(cfg.space_order);
    std::vector<double> src = {0.5 * lx, 2.0 * h}, rec;
    for (long i = 0; i < nx; ++i) rec.insert(rec.end(), {double(i) * h, 2.0 * h});
    AcquisitionGeometry geom(model, src, rec, 0.0, cfg.tn, dt, cfg.f0);
    WaveOp obs_op = forward_operator(model, geom, cfg.space_order);
    run_wave(obs_op);
    const std::vector<double> observed = geom.rec()->traces();

    model.set_velocity(vel_start);
    const std::vector<double> m0 = model.physical_m();
    std::vector<double> dm(m0.size());
    for (std::size_t i = 0; i < m0.size(); ++i) dm[i] = m_true[i] - m0[i];
    GradientResult base = fwi_gradient(model, geom, observed, cfg.space_order);
    GradientReport rep;
    rep.phi0 = base.objective;
    for (std::size_t i = 0; i < dm.size(); ++i) rep.dphi += base.gradient[i] * dm[i];
    rep.steps = cfg.steps;
    std::vector<double> m_s(m0.size());
    for (double s : cfg.steps) {
        for (std::size_t i = 0; i < m0.size(); ++i) m_s[i] = m0[i] + s * dm[i];
        model.set_physical_m(m_s);
        WaveOp fwd = forward_operator(model, geom, cfg.space_order);
        run_wave(fwd);
        const double phi = objective(*geom.rec(), observed);
        rep.eps0.push_back(std::abs(phi - rep.phi0));
        rep.eps1.push_back(std::abs(phi - rep.phi0 - s * rep.dphi));
    }
    model.set_physical_m(m0);
    // below ~100 ulp of phi0 the remainder is cancellation noise; the device computes in
    // fp32, so the ulp is fp32's
    const double noise = 100.0 * double(std::numeric_limits<float>::epsilon()) * rep.phi0;
    std::vector<double> x0, y0, x1, y1;
    rep.eps1_fitted.resize(rep.eps1.size());
    for (std::size_t i = 0; i < cfg.steps.size(); ++i) {
        x0.push_back(cfg.steps[i]);
        y0.push_back(rep.eps0[i]);
        const bool ok = rep.eps1[i] > noise;
        rep.eps1_fitted[i] = ok;
        if (ok) {
            x1.push_back(cfg.steps[i]);
            y1.push_back(rep.eps1[i]);
        }
    }
    rep.fit0 = fit_loglog(x0, y0);
    rep.fit1_valid = x1.size() >= 3;
    if (rep.fit1_valid) rep.fit1 = fit_loglog(x1, y1);
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
    std::sort(times.begin(), times.end());
    return times[times.size() / 2];
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
