// test_seismic_dropin.cpp -- the reference's hot-path integration tests
// (proj/tests/test_seismic.cpp:154-313, proj/tests/test_verify.cpp:68-77), written the way
// the reference writes them, compiled against include/sfb/*.hpp with `namespace sf = sfb;`.
// It is the drop-in claim made executable: only the namespace alias and the tolerances of
// the identities that depend on f64 round-off (dot test 1e-12 -> 1e-4) differ.
// doctest is not available in this image, so a minimal CHECK macro stands in for it.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "sfb/geometry.hpp"
#include "sfb/gridio.hpp"
#include "sfb/model.hpp"
#include "sfb/seismic_ops.hpp"
#include "sfb/verify.hpp"

namespace sf = sfb;
using namespace sf;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_failed;                                                          \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                        \
    } while (0)
#define TEST_CASE(name) static void name()

namespace {
SeismicModel constant_model(long n, double h, double c, long nbl, int order = 8) {
    std::vector<double> vel(size_t(n) * size_t(n), c);
    return SeismicModel({n, n}, {h, h}, {0.0, 0.0}, vel, nbl, order);
}
}  // namespace

TEST_CASE(forward_adjoint_dot_test_at_order_4) {  // test_seismic.cpp:154-163
    AdjointConfig cfg;
    cfg.ndim = 2;
    cfg.n = 48;
    cfg.space_order = 4;
    cfg.tn = 200.0;
    AdjointReport r = adjoint_test(cfg);
    CHECK(r.forward_dot > 0.0);
    CHECK(r.rel_err <= 1e-4);
}

TEST_CASE(adjoint_dot_test_in_3d) {  // test_verify.cpp:68-77
    AdjointConfig cfg;
    cfg.ndim = 3;
    cfg.n = 24;
    cfg.space_order = 6;
    cfg.tn = 150.0;
    AdjointReport r = adjoint_test(cfg);
    CHECK(r.forward_dot > 0.0);
    CHECK(r.rel_err <= 1e-4);
}

TEST_CASE(zero_source_produces_zero_receivers) {  // test_seismic.cpp:165-174
    SeismicModel m = constant_model(31, 10.0, 1.5, 8);
    AcquisitionGeometry g(m, {150.0, 150.0}, {50.0, 100.0, 250.0, 100.0}, 0.0, 150.0,
                          0.9 * m.critical_dt(), 0.01);
    for (long t = 0; t < g.nt(); ++t) g.src()->trace(t, 0) = 0.0;
    WaveOp w = forward_operator(m, g, 8);
    run_wave(w);
    for (long t = 0; t < g.nt(); ++t)
        for (long p = 0; p < g.n_rec(); ++p) CHECK(g.rec()->trace(t, p) == 0.0);
}

TEST_CASE(absorbing_layer_dissipates_the_wavefield) {  // test_seismic.cpp:176-197
    SeismicModel m = constant_model(41, 10.0, 1.5, 20);
    double dt = 0.9 * m.critical_dt();
    AcquisitionGeometry g(m, {200.0, 200.0}, {200.0, 300.0}, 0.0, 900.0, dt, 0.01);
    WaveOp w = forward_operator(m, g, 8, true);
    run_wave(w);
    auto& u = *w.wavefield;
    std::vector<long> shape = u.grid()->shape();
    auto energy = [&](long t) {
        double e = 0;
        for (long i = 0; i < shape[0]; ++i)
            for (long j = 0; j < shape[1]; ++j) {
                double v = u.at({t, i, j});
                e += v * v;
            }
        return e;
    };
    double peak = 0;
    for (long t = 0; t < g.nt(); ++t) peak = std::max(peak, energy(t));
    CHECK(peak > 0.0);
    CHECK(energy(g.nt() - 1) < 0.05 * peak);
}

TEST_CASE(zero_residual_gives_zero_objective_and_zero_gradient) {  // test_seismic.cpp:247-260
    SeismicModel m = constant_model(21, 10.0, 1.5, 6);
    AcquisitionGeometry g(m, {100.0, 20.0}, {40.0, 40.0, 160.0, 40.0}, 0.0, 120.0,
                          0.8 * m.critical_dt(), 0.01);
    WaveOp w = forward_operator(m, g, 8);
    run_wave(w);
    std::vector<double> observed(size_t(g.nt()) * size_t(g.n_rec()));
    for (long t = 0; t < g.nt(); ++t)
        for (long p = 0; p < g.n_rec(); ++p)
            observed[size_t(t) * size_t(g.n_rec()) + size_t(p)] = g.rec()->trace(t, p);
    GradientResult res = fwi_gradient(m, g, observed, 8);
    CHECK(res.objective == 0.0);
    for (double v : res.gradient) CHECK(v == 0.0);
}

TEST_CASE(unstable_dt_and_missing_history_are_rejected) {  // test_seismic.cpp:108-114, seismic_ops.cpp:113-114
    SeismicModel m = constant_model(21, 10.0, 1.5, 4);
    bool threw = false;
    try {
        AcquisitionGeometry(m, {100.0, 100.0}, {50.0, 50.0}, 0.0, 100.0, m.critical_dt() * 1.5, 0.01);
    } catch (const StabilityError&) {
        threw = true;
    }
    CHECK(threw);
    AcquisitionGeometry g(m, {100.0, 100.0}, {50.0, 50.0}, 0.0, 60.0, 0.8 * m.critical_dt(), 0.01);
    WaveOp fwd = forward_operator(m, g, 8);
    run_wave(fwd);
    threw = false;
    try {
        gradient_operator(m, g, 8, fwd.wavefield);
    } catch (const ParameterError&) {
        threw = true;
    }
    CHECK(threw);
}

TEST_CASE(fwi_returns_immediately_when_started_at_the_true_model) {  // test_seismic.cpp:262-285
    SeismicModel m = constant_model(21, 10.0, 1.5, 6);
    std::vector<AcquisitionGeometry> shots;
    shots.emplace_back(m, std::vector<double>{100.0, 20.0},
                       std::vector<double>{40.0, 40.0, 160.0, 40.0}, 0.0, 120.0,
                       0.8 * m.critical_dt(), 0.01);
    WaveOp w = forward_operator(m, shots[0], 8);
    run_wave(w);
    std::vector<std::vector<double>> observed(1);
    observed[0] = shots[0].rec()->traces();
    FwiConfig cfg;
    cfg.n_iter = 5;
    cfg.m_min = 0.1;
    cfg.m_max = 1.0;
    std::vector<double> m_true = m.physical_m();
    FwiResult res = fwi(m, shots, observed, cfg, &m_true);
    CHECK(res.objectives.size() == 1);
    CHECK(res.objectives[0] == 0.0);
    CHECK(res.final_m == m_true);
}

int main() {
    struct {
        const char* name;
        void (*fn)();
    } tests[] = {
        {"forward/adjoint dot test at order 4", forward_adjoint_dot_test_at_order_4},
        {"adjoint dot test in 3-D", adjoint_dot_test_in_3d},
        {"zero source produces zero receivers", zero_source_produces_zero_receivers},
        {"absorbing layer dissipates the wavefield", absorbing_layer_dissipates_the_wavefield},
        {"zero residual gives zero objective and zero gradient",
         zero_residual_gives_zero_objective_and_zero_gradient},
        {"unstable dt / missing history rejected", unstable_dt_and_missing_history_are_rejected},
        {"fwi returns immediately at the true model",
         fwi_returns_immediately_when_started_at_the_true_model},
    };
    for (auto& t : tests) {
        int before = g_failed;
        try {
            t.fn();
        } catch (const std::exception& e) {
            ++g_failed;
            std::printf("EXCEPTION in '%s': %s\n", t.name, e.what());
        }
        std::printf("[%s] %s\n", g_failed == before ? "ok" : "FAIL", t.name);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
