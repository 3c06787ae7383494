// ref_driver.cpp -- C-ABI driver around the REFERENCE's own public API ("sf",
// /root/reference/proj/include/sf/*.hpp), compiled together with the reference's unmodified
// sources by oracle/Makefile into oracle/_ref/libsf_ref.so.
//
// TEST INFRASTRUCTURE ONLY: it exists so that tests/ can check the oracle (and through it
// the CUDA path) against outputs of the real reference, and so that bench.py's
// `--impl reference` arm can time the reference's own CPU engines.  Everything numerical
// below happens inside the reference; this file only marshals arrays.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "sf/emit.hpp"
#include "sf/error.hpp"
#include "sf/execute.hpp"
#include "sf/geometry.hpp"
#include "sf/gridio.hpp"
#include "sf/lower.hpp"
#include "sf/model.hpp"
#include "sf/seismic_ops.hpp"
#include "sf/solve.hpp"

namespace {

thread_local std::string g_err;

struct Problem {
    int ndim;
    const long* shape;        // physical
    const double* spacing;
    const double* origin;
    const double* velocity;   // physical, row-major
    long nbl;
    int model_order, op_order;
    long nsrc, nrec;
    const double* src_coords;
    const double* rec_coords;
    double t0, tn, dt, f0;
};

sf::Backend backend_of(int b) {
    return b == 0 ? sf::Backend::Interpreter : (b == 1 ? sf::Backend::Emitted : sf::Backend::Auto);
}

sf::SeismicModel make_model(const Problem& p) {
    std::vector<long> shape(p.shape, p.shape + p.ndim);
    std::vector<double> h(p.spacing, p.spacing + p.ndim), o(p.origin, p.origin + p.ndim);
    size_t n = 1;
    for (long e : shape) n *= size_t(e);
    std::vector<double> vel(p.velocity, p.velocity + n);
    return sf::SeismicModel(shape, h, o, vel, p.nbl, p.model_order);
}

sf::AcquisitionGeometry make_geom(const Problem& p, const sf::SeismicModel& m) {
    std::vector<double> s(p.src_coords, p.src_coords + p.nsrc * p.ndim);
    std::vector<double> r(p.rec_coords, p.rec_coords + p.nrec * p.ndim);
    return sf::AcquisitionGeometry(m, s, r, p.t0, p.tn, p.dt, p.f0);
}

// compact copy of one time level (interior nodes only)
void copy_level(const sf::TimeFunction& u, long level, double* out) {
    const auto& shape = u.grid()->shape();
    std::vector<long> idx(shape.size() + 1, 0);
    idx[0] = u.time_buffered() ? level % u.time_slots() : level;
    size_t k = 0;
    for (;;) {
        out[k++] = u.at(idx);
        size_t d = idx.size();
        bool done = true;
        while (d > 1) {
            --d;
            if (++idx[d] < shape[d - 1]) {
                done = false;
                break;
            }
            idx[d] = 0;
        }
        if (done) break;
    }
}

void copy_field(const sf::Function& f, double* out) {
    const auto& shape = f.grid()->shape();
    std::vector<long> idx(shape.size(), 0);
    size_t k = 0;
    for (;;) {
        out[k++] = f.at(idx);
        size_t d = idx.size();
        bool done = true;
        while (d > 0) {
            --d;
            if (++idx[d] < shape[d]) {
                done = false;
                break;
            }
            idx[d] = 0;
        }
        if (done) break;
    }
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const sf::StabilityError& e) {
        g_err = e.what();
        return 2;
    } catch (const sf::LocationError& e) {
        g_err = e.what();
        return 3;
    } catch (const sf::ParameterError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* sfr_last_error() { return g_err.c_str(); }

// SeismicModel: padded m, damp (compact [N...]), critical dt
int sfr_model(const Problem* p, double* m_out, double* damp_out, double* crit_dt) {
    return guarded([&] {
        sf::SeismicModel m = make_model(*p);
        if (m_out) copy_field(*m.m(), m_out);
        if (damp_out) copy_field(*m.damp(), damp_out);
        if (crit_dt) *crit_dt = m.critical_dt(p->op_order);
    });
}

// AcquisitionGeometry: nt, base / weight tables of both clouds, the Ricker source traces
int sfr_geometry(const Problem* p, long* nt, long* src_base, double* src_w, long* rec_base,
                 double* rec_w, double* src_traces) {
    return guarded([&] {
        sf::SeismicModel m = make_model(*p);
        sf::AcquisitionGeometry g = make_geom(*p, m);
        if (nt) *nt = g.nt();
        auto put = [&](const sf::SparseFunction& s, long* base, double* w) {
            if (base) std::copy(s.base_table().begin(), s.base_table().end(), base);
            if (w)
                std::memcpy(w, s.weight_table()->values(),
                            size_t(s.npoints()) * size_t(s.corners()) * sizeof(double));
        };
        put(*g.src(), src_base, src_w);
        put(*g.rec(), rec_base, rec_w);
        if (src_traces)
            std::memcpy(src_traces, g.src()->traces()->values(),
                        size_t(g.nt()) * size_t(g.n_src()) * sizeof(double));
    });
}

// forward_operator + run_wave.  src_traces (nullable) overrides the Ricker preload.
// Outputs: rec [nt][nrec]; level_a = level nt-1, level_b = level nt-2 (compact, nullable).
int sfr_forward(const Problem* p, const double* src_traces, int backend, int nthreads,
                double* rec, double* level_a, double* level_b, double* seconds) {
    return guarded([&] {
        sf::SeismicModel m = make_model(*p);
        sf::AcquisitionGeometry g = make_geom(*p, m);
        if (src_traces)
            std::memcpy(g.src()->traces()->values(), src_traces,
                        size_t(g.nt()) * size_t(g.n_src()) * sizeof(double));
        sf::WaveOp w = sf::forward_operator(m, g, p->op_order);
        sf::ExecutionReport rep = sf::run_wave(w, backend_of(backend), nthreads);
        if (seconds) *seconds = rep.seconds;
        std::memcpy(rec, g.rec()->traces()->values(),
                    size_t(g.nt()) * size_t(g.n_rec()) * sizeof(double));
        if (level_a) copy_level(*w.wavefield, g.nt() - 1, level_a);
        if (level_b) copy_level(*w.wavefield, g.nt() - 2, level_b);
    });
}

// adjoint_operator + run_wave: rec_in [nt][nrec] injected, srca [nt][nsrc] sampled
int sfr_adjoint(const Problem* p, const double* rec_in, int backend, int nthreads, double* srca,
                double* level0) {
    return guarded([&] {
        sf::SeismicModel m = make_model(*p);
        sf::AcquisitionGeometry g = make_geom(*p, m);
        std::memcpy(g.rec()->traces()->values(), rec_in,
                    size_t(g.nt()) * size_t(g.n_rec()) * sizeof(double));
        sf::WaveOp w = sf::adjoint_operator(m, g, p->op_order);
        sf::run_wave(w, backend_of(backend), nthreads);
        std::memcpy(srca, w.smp->traces()->values(),
                    size_t(g.nt()) * size_t(g.n_src()) * sizeof(double));
        if (level0) copy_level(*w.wavefield, 0, level0);
    });
}

// fwi_gradient: observed [nt][nrec] -> objective, gradient over the physical cells
int sfr_fwi_gradient(const Problem* p, const double* observed, int backend, double* objective,
                     double* gradient, double* residual) {
    return guarded([&] {
        sf::SeismicModel m = make_model(*p);
        sf::AcquisitionGeometry g = make_geom(*p, m);
        std::vector<double> obs(observed, observed + size_t(g.nt()) * size_t(g.n_rec()));
        sf::GradientResult r = sf::fwi_gradient(m, g, obs, p->op_order, backend_of(backend));
        if (objective) *objective = r.objective;
        if (gradient) std::copy(r.gradient.begin(), r.gradient.end(), gradient);
        if (residual) std::copy(r.residual.begin(), r.residual.end(), residual);
    });
}

// The reference's bare acoustic stencil (the recipe of its `bench`, src/verify.cpp:338-376,
// restated through the public API because verify.cpp needs FFTW): n^3 grid, m = 1/2.25,
// zero damping, `steps` updates on the chosen engine.  Returns the engine's own timing.
int sfr_dense_bench(long n, int order, long steps, int backend, int nthreads, double* seconds,
                    double* flops_per_point) {
    return guarded([&] {
        auto grid = std::make_shared<sf::Grid>(std::vector<long>{n, n, n},
                                               std::vector<double>{10.0, 10.0, 10.0},
                                               std::vector<double>{0.0, 0.0, 0.0});
        auto u = sf::TimeFunction::create("u", grid, order, 2);
        auto m = sf::Function::create("m", grid, 2);
        auto damp = sf::Function::create("damp", grid, 2);
        std::fill(m->values(), m->values() + m->storage_size(), 1.0 / 2.25);
        sf::Equation pde(m->ref() * u->dt2() + damp->ref() * u->dt(2), u->laplace());
        std::vector<sf::Equation> eqs;
        eqs.emplace_back(u->forward(), sf::solve_linear(pde, u->forward()));
        sf::Operator op = sf::compile("acoustic", eqs, sf::CompileOptions{});
        // a non-zero state so the arithmetic is not all zeros
        for (size_t i = 0; i < u->storage_size(); i += 7) u->values()[i] = 1e-3 * double(i % 13);
        sf::RunArgs args;
        args.t_from = 1;
        args.t_to = 1 + steps;
        args.bind.set("dt", 1.0);
        args.check_finite = false;
        args.nthreads = nthreads;
        sf::ExecutionReport rep = (backend == 1) ? sf::run_emitted(op, args) : sf::run(op, args);
        if (seconds) *seconds = rep.seconds;
        if (flops_per_point) *flops_per_point = double(op.metrics.flops_per_point.total());
    });
}

// the reference's own file writers / readers (proj/src/gridio.cpp, proj/src/sparse.cpp)
int sfr_write_grid(const char* path, int ndim, const long* shape, const double* data) {
    return guarded([&] {
        std::vector<long> sh(shape, shape + ndim);
        size_t n = 1;
        for (long e : sh) n *= size_t(e);
        sf::write_grid(path, sh, std::vector<double>(data, data + n));
    });
}

int sfr_read_grid(const char* path, int* ndim, long* shape, double* data, long capacity) {
    return guarded([&] {
        sf::GridData g = sf::read_grid(path);
        *ndim = int(g.shape.size());
        std::copy(g.shape.begin(), g.shape.end(), shape);
        if (long(g.data.size()) > capacity) throw sf::ParameterError("buffer too small");
        std::copy(g.data.begin(), g.data.end(), data);
    });
}

int sfr_write_traces_table(const char* path, long nt, long np, const double* tr, double t0,
                           double dt) {
    return guarded([&] {
        sf::write_traces_csv(path, nt, np, std::vector<double>(tr, tr + nt * np), t0, dt);
    });
}

// SparseFunction CSV pair: coords [np][ndim] + traces [nt][np] on a unit grid of `n` nodes
int sfr_write_cloud_csv(const char* traces_path, const char* coords_path, int ndim, long n,
                        long np, long nt, const double* coords, const double* tr,
                        const double* times) {
    return guarded([&] {
        auto grid = std::make_shared<sf::Grid>(std::vector<long>(size_t(ndim), n),
                                               std::vector<double>(size_t(ndim), 1.0),
                                               std::vector<double>(size_t(ndim), 0.0));
        auto s = sf::SparseFunction::create("s", grid, std::vector<double>(coords, coords + np * ndim), nt);
        for (long t = 0; t < nt; ++t)
            for (long p = 0; p < np; ++p) s->trace(t, p) = tr[t * np + p];
        sf::write_traces_csv(traces_path, *s, std::vector<double>(times, times + nt));
        sf::write_coords_csv(coords_path, *s);
    });
}

int sfr_emit_available() { return sf::emit_backend_available() ? 1 : 0; }

}  // extern "C"
