// ops.cpp -- forward / adjoint / gradient operators of the host layer on top of the C-ABI
// engine (include/sfb200.h).  Structure follows the reference's entry points
// (proj/src/seismic_ops.cpp:58-286); what the reference hands to its compiler and its
// run_window (proj/src/seismic_ops.cpp:44-54) is handed to sfb_forward / sfb_adjoint /
// sfb_gradient here.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <thread>

#include "engine.hpp"
#include "sfb/seismic_ops.hpp"
#include "sfb200.h"

namespace sfb {

namespace {
thread_local int g_device = 0;
}

void set_device(int ordinal) { g_device = ordinal; }
int device() { return g_device; }

namespace {

// proj/src/seismic_ops.cpp:15-22
void check_cfl(const SeismicModel& model, const AcquisitionGeometry& geom, int space_order) {
    const double crit = model.critical_dt(space_order);
    if (geom.dt() > crit * (1.0 + 1e-12))
        throw StabilityError("dt " + std::to_string(geom.dt()) + " exceeds the stable limit " +
                             std::to_string(crit) + " at order " + std::to_string(space_order));
}

ExecutionReport to_report(const sfb_report& r) {
    ExecutionReport e;
    e.seconds = r.seconds;
    e.flops = r.flops;
    e.gflops = r.gflops;
    e.steps = r.steps;
    e.gpts_per_s = r.gpts_per_s;
    e.kernel_launches = r.kernel_launches;
    return e;
}

std::vector<double> cloud_coords(const SparseFunction& s) { return s.coords(); }

}  // namespace

// proj/src/seismic_ops.cpp:58-82
WaveOp forward_operator(const SeismicModel& model, const AcquisitionGeometry& geom,
                        int space_order, bool save, std::vector<long> /*tiles*/) {
    check_space_order(space_order);
    check_cfl(model, geom, space_order);
    WaveOp w;
    w.dt = geom.dt();
    w.nt = geom.nt();
    w.space_order = space_order;
    w.inj = geom.src();
    w.smp = geom.rec();
    w.save_every = save ? 1 : 0;
    w.wavefield = save ? TimeFunction::create("u", model.grid(), space_order, 2, geom.nt())
                       : TimeFunction::create("u", model.grid(), space_order, 2);
    w.engine = std::make_shared<Engine>(model, geom, space_order);
    return w;
}

// proj/src/seismic_ops.cpp:84-107: receiver traces are injected, the field is sampled at
// the source coordinates into a fresh cloud "srca".
WaveOp adjoint_operator(const SeismicModel& model, const AcquisitionGeometry& geom,
                        int space_order) {
    check_space_order(space_order);
    check_cfl(model, geom, space_order);
    WaveOp w;
    w.dt = geom.dt();
    w.nt = geom.nt();
    w.space_order = space_order;
    w.adjoint = true;
    w.inj = geom.rec();
    w.smp = SparseFunction::create("srca", model.grid(), cloud_coords(*geom.src()), geom.nt());
    w.smp->locate();
    w.wavefield = TimeFunction::create("v", model.grid(), space_order, 2);
    w.engine = std::make_shared<Engine>(model, geom, space_order);
    return w;
}

// ---- TTI ----------------------------------------------------------------------------------

TtiModel::TtiModel(const SeismicModel& model, const std::vector<double>& eps,
                   const std::vector<double>& del, const std::vector<double>& th,
                   const std::vector<double>& ph) {
    const std::vector<long>& ps = model.physical_shape();
    std::size_t n = 1;
    for (long e : ps) n *= std::size_t(e);
    if (eps.size() != n || del.size() != n || th.size() != n || ph.size() != n)
        throw ParameterError("TtiModel: field size does not match the physical shape");
    const int nd = int(ps.size()), off = 3 - nd;
    auto extend = [&](const char* name, const std::vector<double>& v) {
        auto f = Function::create(name, model.grid(), model.space_order());
        long N[3] = {1, 1, 1}, pn[3] = {1, 1, 1}, pad[3] = {0, 0, 0}, st[3] = {0, 0, 0};
        for (int a = 0; a < nd; ++a) {
            N[off + a] = model.grid()->shape()[std::size_t(a)];
            pn[off + a] = ps[std::size_t(a)];
            pad[off + a] = model.nbl();
            st[off + a] = f->stride(a);
        }
        std::vector<long> zero(std::size_t(nd), 0);
        double* origin = f->values() + f->flat_index(zero);
        for (long i = 0; i < N[0]; ++i)
            for (long j = 0; j < N[1]; ++j)
                for (long l = 0; l < N[2]; ++l) {
                    const long pi = std::clamp(i - pad[0], 0L, pn[0] - 1);
                    const long pj = std::clamp(j - pad[1], 0L, pn[1] - 1);
                    const long pl = std::clamp(l - pad[2], 0L, pn[2] - 1);
                    origin[i * st[0] + j * st[1] + l * st[2]] =
                        v[(std::size_t(pi) * pn[1] + pj) * pn[2] + pl];
                }
        return f;
    };
    epsilon = extend("epsilon", eps);
    delta = extend("delta", del);
    theta = extend("theta", th);
    phi = extend("phi", ph);
}

double TtiModel::epsilon_max() const {
    double m = 0.0;
    const double* p = epsilon->values();
    for (std::size_t i = 0; i < epsilon->storage_size(); ++i) m = std::max(m, p[i]);
    return m;
}

double tti_critical_dt(const SeismicModel& model, const TtiModel& tti, int space_order) {
    return 0.9 * model.critical_dt(space_order) / std::sqrt(1.0 + 2.0 * tti.epsilon_max());
}

WaveOp tti_forward_operator(const SeismicModel& model, const TtiModel& tti,
                            const AcquisitionGeometry& geom, int space_order) {
    check_space_order(space_order);
    const double crit = tti_critical_dt(model, tti, space_order);
    if (geom.dt() > crit * (1.0 + 1e-12))
        throw StabilityError("dt " + std::to_string(geom.dt()) + " exceeds the TTI stable limit " +
                             std::to_string(crit) + " at order " + std::to_string(space_order));
    WaveOp w;
    w.dt = geom.dt();
    w.nt = geom.nt();
    w.space_order = space_order;
    w.tti = true;
    w.inj = geom.src();
    w.smp = geom.rec();
    w.wavefield = TimeFunction::create("p", model.grid(), space_order, 2);
    w.wavefield_r = TimeFunction::create("r", model.grid(), space_order, 2);
    w.engine = std::make_shared<Engine>(model, geom, space_order);
    sfb_field_view ev = Engine::view(*tti.epsilon), dv = Engine::view(*tti.delta),
                   tv = Engine::view(*tti.theta), pv = Engine::view(*tti.phi);
    w.engine->check(sfb_set_model_tti(w.engine->plan(), &ev, &dv, &tv, &pv));
    return w;
}

// proj/src/seismic_ops.cpp:109-135
GradientOp gradient_operator(const SeismicModel& model, const AcquisitionGeometry& geom,
                             int space_order, std::shared_ptr<TimeFunction> saved_u) {
    check_space_order(space_order);
    check_cfl(model, geom, space_order);
    if (!saved_u || saved_u->time_buffered() || saved_u->time_slots() != geom.nt())
        throw ParameterError("gradient_operator: saved forward history required");

    GradientOp g;
    g.dt = geom.dt();
    g.nt = geom.nt();
    g.space_order = space_order;
    g.resid = SparseFunction::create("resid", model.grid(), cloud_coords(*geom.rec()), geom.nt());
    g.resid->locate();
    g.v = TimeFunction::create("v", model.grid(), space_order, 2);
    g.grad = Function::create("grad", model.grid(), space_order);
    if (saved_u->device_history) {
        // the forward operator's engine holds the history, the model and both clouds
        g.engine = std::static_pointer_cast<Engine>(saved_u->device_history);
    } else {
        // a history that exists in host memory only (filled by the caller, or produced by
        // another engine): bind every level, as the reference reads u_saved[t] from RAM
        g.engine = std::make_shared<Engine>(model, geom, space_order);
        for (long t = 0; t < geom.nt(); ++t) {
            sfb_field_mview mv = Engine::mview(*saved_u, t);
            sfb_field_view v{};
            v.ptr = mv.ptr;
            for (int a = 0; a < 3; ++a) v.stride[a] = mv.stride[a];
            g.engine->check(sfb_put_history(g.engine->plan(), 1, t, &v));
        }
    }
    return g;
}

// proj/src/seismic_ops.cpp:137-141 (+ run_window :44-54)
ExecutionReport run_wave(WaveOp& w, Backend, int) {
    if (!w.engine) throw BindingError("run_wave: operator was not built");
    Engine& e = *w.engine;
    sfb_report rep{};
    w.wavefield->zero();
    if (w.tti) {
        w.wavefield_r->zero();
        e.check(sfb_tti_forward(e.plan(), w.inj->traces().data(), w.smp->traces().data(), &rep));
        if (w.nt >= 3)
            for (int field = 0; field < 2; ++field)
                for (long lvl : {w.nt - 1, w.nt - 2}) {
                    TimeFunction& f = field ? *w.wavefield_r : *w.wavefield;
                    sfb_field_mview mv = Engine::mview(f, lvl % f.time_slots());
                    e.check(sfb_get_wavefield(e.plan(), field, lvl, &mv));
                }
        return to_report(rep);
    }
    const bool ckpt = !w.adjoint && w.save_every > 0 && w.checkpoint_every > 0;
    if (ckpt) {
        e.check(sfb_forward_checkpointed(e.plan(), w.inj->traces().data(),
                                         w.smp->traces().data(), w.checkpoint_every, &rep));
    } else if (!w.adjoint) {
        e.check(sfb_forward(e.plan(), w.inj->traces().data(), w.smp->traces().data(),
                            w.save_every, &rep));
    } else {
        e.check(sfb_adjoint(e.plan(), w.inj->traces().data(), w.smp->traces().data(), &rep));
    }
    // mirror the live time levels into the host TimeFunction (slot rules of
    // proj/src/execute.cpp:187-199)
    TimeFunction& u = *w.wavefield;
    if (w.save_every > 0) {
        u.device_history = w.engine;
        u.device_save_every = ckpt ? 1 : w.save_every;
        if (w.host_history && !ckpt && !u.time_buffered())
            for (long t = 2; t < w.nt; t += 1) {
                if (t % w.save_every != 0) continue;
                sfb_field_mview mv = Engine::mview(u, t);
                e.check(sfb_get_wavefield(e.plan(), 0, t, &mv));
            }
    } else if (w.nt >= 3) {
        const long a = w.adjoint ? 0 : w.nt - 1, b = w.adjoint ? 1 : w.nt - 2;
        for (long lvl : {a, b}) {
            sfb_field_mview mv = Engine::mview(u, u.time_buffered() ? lvl % u.time_slots() : lvl);
            e.check(sfb_get_wavefield(e.plan(), 0, lvl, &mv));
        }
    }
    return to_report(rep);
}

// SURVEY.md 8e through the operator interface: one process, one plan per slab, fused halo push
ExecutionReport run_wave_slabs(WaveOp& w, const SeismicModel& model,
                               const AcquisitionGeometry& geom, const std::vector<int>& devices) {
    if (w.tti) throw CapabilityError("run_wave_slabs: acoustic operators only");
    if (devices.empty()) throw ParameterError("run_wave_slabs: empty device list");
    if (model.grid()->ndim() != 3) throw CapabilityError("run_wave_slabs: 3-D grids only");
    const long n0 = model.grid()->shape()[0];
    const long K = w.space_order / 2, nslab = long(devices.size());
    if (n0 / nslab < 2 * K)
        throw ParameterError("run_wave_slabs: slabs thinner than two halo widths");
    const int op = w.adjoint ? SFB_OP_ADJOINT : SFB_OP_FORWARD;
    const int inj_cloud = w.adjoint ? SFB_CLOUD_REC : SFB_CLOUD_SRC;
    const int smp_cloud = w.adjoint ? SFB_CLOUD_SRC : SFB_CLOUD_REC;
    std::vector<std::unique_ptr<Engine>> eng;
    long lo = 0;
    for (long i = 0; i < nslab; ++i) {   // balanced contiguous split (slabs.split_slabs)
        const long hi = lo + n0 / nslab + (i < n0 % nslab ? 1 : 0);
        eng.emplace_back(new Engine(model, geom, w.space_order, lo, hi, devices[std::size_t(i)]));
        lo = hi;
    }
    for (long i = 0; i < nslab; ++i) {
        Engine& e = *eng[std::size_t(i)];
        e.check(sfb_upload_traces(e.plan(), inj_cloud, w.inj->traces().data()));
        e.check(sfb_link_peers(e.plan(), i > 0 ? eng[std::size_t(i - 1)]->plan() : nullptr,
                               i + 1 < nslab ? eng[std::size_t(i + 1)]->plan() : nullptr));
        e.check(sfb_step_begin(e.plan(), op, 0));
    }
    for (auto& e : eng) e->check(sfb_stream_sync(e->plan()));
    const auto t0 = std::chrono::steady_clock::now();
    for (long s = 0; s < w.nt - 2; ++s) {
        const long t = w.adjoint ? w.nt - 2 - s : 1 + s;
        for (auto& e : eng) {
            e->check(sfb_step_slab_boundary(e->plan(), op, t));
            e->check(sfb_step_slab_interior(e->plan(), op, t));
        }
        for (long i = 0; i < nslab; ++i) {
            Engine& e = *eng[std::size_t(i)];
            if (i > 0) e.check(sfb_peer_wait(e.plan(), eng[std::size_t(i - 1)]->plan()));
            if (i + 1 < nslab) e.check(sfb_peer_wait(e.plan(), eng[std::size_t(i + 1)]->plan()));
        }
    }
    for (auto& e : eng) e->check(sfb_step_end(e->plan(), op));
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // sampled traces: every point is sampled by the slab that owns its base plane, the
    // others hold zeros, so the record is the sum; wavefield: each slab writes its planes
    std::vector<double>& out = w.smp->traces();
    std::fill(out.begin(), out.end(), 0.0);
    std::vector<double> part(out.size());
    w.wavefield->zero();
    for (auto& e : eng) {
        e->check(sfb_download_traces(e->plan(), smp_cloud, part.data()));
        for (std::size_t i = 0; i < out.size(); ++i) out[i] += part[i];
        if (w.nt >= 3) {
            TimeFunction& u = *w.wavefield;
            const long a = w.adjoint ? 0 : w.nt - 1, b = w.adjoint ? 1 : w.nt - 2;
            for (long lvl : {a, b}) {
                sfb_field_mview mv = Engine::mview(u, u.time_buffered() ? lvl % u.time_slots() : lvl);
                e->check(sfb_get_wavefield(e->plan(), 0, lvl, &mv));
            }
        }
    }
    ExecutionReport rep;
    const long steps = std::max(0L, w.nt - 2);
    double pts = 1;
    for (long e : model.grid()->shape()) pts *= double(e);
    rep.seconds = sec;
    rep.steps = steps;
    rep.gpts_per_s = sec > 0 ? pts * double(steps) / sec / 1e9 : 0.0;
    return rep;
}

ExecutionReport run_wave_slabs(WaveOp& w, const SeismicModel& model, const TtiModel& tti,
                               const AcquisitionGeometry& geom, const std::vector<int>& devices) {
    if (!w.tti) throw ParameterError("run_wave_slabs: not a TTI operator");
    if (devices.empty()) throw ParameterError("run_wave_slabs: empty device list");
    if (model.grid()->ndim() != 3) throw CapabilityError("run_wave_slabs: 3-D grids only");
    const long n0 = model.grid()->shape()[0];
    const long K = w.space_order / 2, nslab = long(devices.size());
    if (n0 / nslab < 2 * K)
        throw ParameterError("run_wave_slabs: slabs thinner than two halo widths");
    const int op = SFB_OP_TTI_FORWARD;
    std::vector<std::unique_ptr<Engine>> eng;
    long lo = 0;
    sfb_field_view ev = Engine::view(*tti.epsilon), dv = Engine::view(*tti.delta),
                   tv = Engine::view(*tti.theta), pv = Engine::view(*tti.phi);
    for (long i = 0; i < nslab; ++i) {
        const long hi = lo + n0 / nslab + (i < n0 % nslab ? 1 : 0);
        eng.emplace_back(new Engine(model, geom, w.space_order, lo, hi, devices[std::size_t(i)]));
        Engine& e = *eng.back();
        e.check(sfb_set_model_tti(e.plan(), &ev, &dv, &tv, &pv));
        e.check(sfb_upload_traces(e.plan(), SFB_CLOUD_SRC, w.inj->traces().data()));
        e.check(sfb_step_begin(e.plan(), op, 0));
        lo = hi;
    }
    auto sync_all = [&] {
        for (auto& e : eng) e->check(sfb_stream_sync(e->plan()));
    };
    // ghost planes of `which` between every pair of neighbouring slabs
    auto exchange = [&](int which, long t) {
        sync_all();
        for (long i = 0; i + 1 < nslab; ++i) {
            Engine &a = *eng[std::size_t(i)], &b = *eng[std::size_t(i + 1)];
            void *a_slo, *a_shi, *a_rlo, *a_rhi, *b_slo, *b_shi, *b_rlo, *b_rhi;
            int64_t n = 0;
            a.check(sfb_tti_halo_blocks(a.plan(), which, t, &a_slo, &a_shi, &a_rlo, &a_rhi, &n));
            b.check(sfb_tti_halo_blocks(b.plan(), which, t, &b_slo, &b_shi, &b_rlo, &b_rhi, &n));
            b.check(sfb_copy_halo(b.plan(), b_rlo, a_shi, n));
            a.check(sfb_copy_halo(a.plan(), a_rhi, b_slo, n));
        }
        sync_all();
    };
    sync_all();
    const auto t0 = std::chrono::steady_clock::now();
    for (long t = 1; t < w.nt - 1; ++t) {
        for (auto& e : eng) e->check(sfb_tti_step_rot(e->plan(), t, SFB_PART_ALL));
        exchange(SFB_TTI_HALO_G_P, t);
        exchange(SFB_TTI_HALO_G_R, t);
        for (auto& e : eng) e->check(sfb_tti_step_update(e->plan(), t, SFB_PART_ALL));
        exchange(SFB_TTI_HALO_P, t);
        exchange(SFB_TTI_HALO_R, t);
    }
    for (auto& e : eng) e->check(sfb_step_end(e->plan(), op));
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<double>& out = w.smp->traces();
    std::fill(out.begin(), out.end(), 0.0);
    std::vector<double> part(out.size());
    w.wavefield->zero();
    w.wavefield_r->zero();
    for (auto& e : eng) {
        e->check(sfb_download_traces(e->plan(), SFB_CLOUD_REC, part.data()));
        for (std::size_t i = 0; i < out.size(); ++i) out[i] += part[i];
        if (w.nt >= 3)
            for (int field = 0; field < 2; ++field)
                for (long lvl : {w.nt - 1, w.nt - 2}) {
                    TimeFunction& f = field ? *w.wavefield_r : *w.wavefield;
                    sfb_field_mview mv = Engine::mview(f, lvl % f.time_slots());
                    e->check(sfb_get_wavefield(e->plan(), field, lvl, &mv));
                }
    }
    ExecutionReport rep;
    double pts = 1;
    for (long e : model.grid()->shape()) pts *= double(e);
    rep.seconds = sec;
    rep.steps = std::max(0L, w.nt - 2);
    rep.gpts_per_s = sec > 0 ? pts * double(rep.steps) / sec / 1e9 : 0.0;
    return rep;
}

// proj/src/seismic_ops.cpp:143-147
ExecutionReport run_gradient(GradientOp& g, Backend, int) {
    if (!g.engine) throw BindingError("run_gradient: operator was not built");
    Engine& e = *g.engine;
    sfb_report rep{};
    g.v->zero();
    g.grad->zero();
    sfb_field_mview gv = Engine::mview(*g.grad);
    e.check(sfb_gradient(e.plan(), g.resid->traces().data(), &gv, &rep));
    return to_report(rep);
}

// proj/src/seismic_ops.cpp:149-160
double objective(const SparseFunction& pred, const std::vector<double>& observed) {
    const std::size_t n = std::size_t(pred.nt()) * std::size_t(pred.npoints());
    if (observed.size() != n) throw ParameterError("objective: observed trace shape mismatch");
    double phi = 0;
    const std::vector<double>& p = pred.traces();
    for (std::size_t i = 0; i < n; ++i) {
        const double r = p[i] - observed[i];
        phi += 0.5 * r * r;
    }
    return phi;
}

namespace {

// adjoint of the edge-clamped extension, proj/src/seismic_ops.cpp:166-193: every padded
// cell is summed onto the physical cell it copies, padded cells visited in row-major order
std::vector<double> fold_gradient(const SeismicModel& model, const Function& grad) {
    const std::vector<long>& ps = model.physical_shape();
    const std::vector<long>& shape = model.grid()->shape();
    const int nd = int(shape.size()), off = 3 - nd;
    long N[3] = {1, 1, 1}, pn[3] = {1, 1, 1}, pad[3] = {0, 0, 0}, st[3] = {0, 0, 0};
    for (int a = 0; a < nd; ++a) {
        N[off + a] = shape[std::size_t(a)];
        pn[off + a] = ps[std::size_t(a)];
        pad[off + a] = model.nbl();
        st[off + a] = grad.stride(a);
    }
    std::vector<long> zero(std::size_t(nd), 0);
    const double* origin = grad.values() + grad.flat_index(zero);
    std::vector<double> out(std::size_t(pn[0]) * pn[1] * pn[2], 0.0);
    for (long i = 0; i < N[0]; ++i) {
        const long pi = std::clamp(i - pad[0], 0L, pn[0] - 1);
        for (long j = 0; j < N[1]; ++j) {
            const long pj = std::clamp(j - pad[1], 0L, pn[1] - 1);
            const double* row = origin + i * st[0] + j * st[1];
            double* orow = out.data() + (std::size_t(pi) * pn[1] + pj) * pn[2];
            for (long l = 0; l < N[2]; ++l) orow[std::clamp(l - pad[2], 0L, pn[2] - 1)] += row[l];
        }
    }
    return out;
}

}  // namespace

// proj/src/seismic_ops.cpp:197-216
GradientResult fwi_gradient(const SeismicModel& model, AcquisitionGeometry& geom,
                            const std::vector<double>& observed, int space_order, Backend backend,
                            long save_every, long checkpoint_every) {
    if (save_every < 1) throw ParameterError("fwi_gradient: save_every must be >= 1");
    if (checkpoint_every != 0 && (checkpoint_every < 2 || save_every != 1))
        throw ParameterError("fwi_gradient: checkpoint_every must be >= 2 (with save_every 1)");
    WaveOp fwd = forward_operator(model, geom, space_order, true);
    fwd.save_every = save_every;
    fwd.checkpoint_every = checkpoint_every;
    fwd.host_history = false;  // the history stays in HBM
    run_wave(fwd, backend);
    GradientResult res;
    res.objective = objective(*geom.rec(), observed);
    GradientOp g = gradient_operator(model, geom, space_order, fwd.wavefield);
    const std::size_t n = std::size_t(geom.nt()) * std::size_t(geom.n_rec());
    res.residual.resize(n);
    const std::vector<double>& pred = geom.rec()->traces();
    for (std::size_t i = 0; i < n; ++i) res.residual[i] = pred[i] - observed[i];
    g.resid->traces() = res.residual;
    run_gradient(g, backend);
    res.gradient = fold_gradient(model, *g.grad);
    return res;
}

// proj/src/seismic_ops.cpp:218-286: fixed-step projected gradient descent; shot gradients
// computed cfg.nthreads at a time (one engine per shot) and reduced in shot order.
FwiResult fwi(SeismicModel& model, std::vector<AcquisitionGeometry>& shots,
              const std::vector<std::vector<double>>& observed, const FwiConfig& cfg,
              const std::vector<double>* true_m) {
    if (shots.empty() || shots.size() != observed.size())
        throw ParameterError("fwi: one observed record per shot required");
    if (!(cfg.m_min > 0.0) || !(cfg.m_max > cfg.m_min)) throw ParameterError("fwi: bad model box");
    FwiResult out;
    std::vector<double> m = model.physical_m();
    double alpha = 0;
    auto rms_error = [&](const std::vector<double>& cur) {
        if (!true_m) return 0.0;
        double s = 0;
        for (std::size_t i = 0; i < cur.size(); ++i) s += (cur[i] - (*true_m)[i]) * (cur[i] - (*true_m)[i]);
        return std::sqrt(s / double(cur.size()));
    };
    const int dev = device();
    for (long it = 0; it < cfg.n_iter; ++it) {
        std::vector<GradientResult> parts(shots.size());
        std::vector<std::string> failures(shots.size());
        const std::size_t width = cfg.nthreads > 1 ? std::size_t(cfg.nthreads) : 1;
        for (std::size_t lo = 0; lo < shots.size(); lo += width) {
            const std::size_t hi = std::min(shots.size(), lo + width);
            std::vector<std::thread> pool;
            for (std::size_t s = lo; s < hi; ++s)
                pool.emplace_back([&, s] {
                    set_device(cfg.devices.empty() ? dev : cfg.devices[s % cfg.devices.size()]);
                    try {
                        parts[s] = fwi_gradient(model, shots[s], observed[s], cfg.space_order,
                                                cfg.backend, cfg.save_every, cfg.checkpoint_every);
                    } catch (const Error& e) {
                        failures[s] = e.what();
                    }
                });
            for (auto& th : pool) th.join();
        }
        for (const auto& f : failures)
            if (!f.empty()) throw StabilityError("fwi: shot failed: " + f);
        double phi = 0;
        std::vector<double> g(m.size(), 0.0);
        for (const auto& p : parts) {
            phi += p.objective;
            for (std::size_t i = 0; i < g.size(); ++i) g[i] += p.gradient[i];
        }
        if (!std::isfinite(phi))
            throw StabilityError("fwi: non-finite objective at iteration " + std::to_string(it));
        out.objectives.push_back(phi);
        out.model_rms.push_back(rms_error(m));
        if (it == 0) {
            double gmax = 0, mmax = 0;
            for (double v : g) gmax = std::max(gmax, std::abs(v));
            for (double v : m) mmax = std::max(mmax, std::abs(v));
            if (gmax == 0.0) {
                out.final_m = m;
                return out;
            }
            alpha = cfg.step_scale * mmax / gmax;
        }
        for (std::size_t i = 0; i < m.size(); ++i)
            m[i] = std::clamp(m[i] - alpha * g[i], cfg.m_min, cfg.m_max);
        model.set_physical_m(m);
    }
    out.model_rms.push_back(rms_error(m));
    out.final_m = m;
    return out;
}

}  // namespace sfb
