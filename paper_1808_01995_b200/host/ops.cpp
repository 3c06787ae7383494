// ops.cpp -- forward / adjoint / gradient operators of the host layer on top of the C-ABI
// engine (include/sfb200.h).  Structure follows the reference's entry points
// (proj/src/seismic_ops.cpp:58-286); what the reference hands to its compiler and its
// run_window (proj/src/seismic_ops.cpp:44-54) is handed to sfb_forward / sfb_adjoint /
// sfb_gradient here.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <functional>
#include <mutex>
#include <numeric>
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
    const bool full_history = saved_u && !saved_u->time_buffered() && saved_u->time_slots() == geom.nt();
    if (!full_history) throw ParameterError("gradient_operator: saved forward history required");
    check_space_order(space_order);
    check_cfl(model, geom, space_order);

    GradientOp g;
    g.space_order = space_order;
    g.nt = geom.nt();
    g.dt = geom.dt();
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
        // one update launch per slab and step: both boundary plane groups are computed and
        // pushed first (the first chunk sweeps up, the last one down), the rest follows
        for (auto& e : eng) e->check(sfb_step_slab_fused(e->plan(), op, t));
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
    // the plans are linked (after the TTI fields are bound: the link maps g and r as well):
    // each pass of a step is one launch per slab whose edge chunks push their boundary planes
    // into the neighbours' ghost planes; events order the slabs, nothing is copied
    for (long i = 0; i < nslab; ++i) {
        Engine& e = *eng[std::size_t(i)];
        e.check(sfb_link_peers(e.plan(), i > 0 ? eng[std::size_t(i - 1)]->plan() : nullptr,
                               i + 1 < nslab ? eng[std::size_t(i + 1)]->plan() : nullptr));
    }
    for (auto& e : eng) e->check(sfb_stream_sync(e->plan()));
    auto for_neighbours = [&](auto&& wait) {
        for (long i = 0; i < nslab; ++i) {
            Engine& e = *eng[std::size_t(i)];
            if (i > 0) e.check(wait(e.plan(), eng[std::size_t(i - 1)]->plan()));
            if (i + 1 < nslab) e.check(wait(e.plan(), eng[std::size_t(i + 1)]->plan()));
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    for (long t = 1; t < w.nt - 1; ++t) {
        for (auto& e : eng) e->check(sfb_tti_step_rot_fused(e->plan(), t));
        for_neighbours(sfb_tti_peer_wait_g);
        for (auto& e : eng) e->check(sfb_tti_step_update_fused(e->plan(), t));
        for_neighbours(sfb_peer_wait);
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

// ---- misfit, shot gradient and the inversion driver ---------------------------------------
// Semantics are the reference's (proj/src/seismic_ops.cpp:149-286: least-squares misfit over
// all rows, residual = predicted - observed, gradient folded onto the physical cells,
// fixed-step projected descent with the step chosen at the first iteration); the
// organisation is this repository's: a shot is evaluated directly on an engine, and the
// driver keeps ONE engine per lane for the whole inversion instead of building operators,
// plans and device buffers per shot and per iteration.

double objective(const SparseFunction& pred, const std::vector<double>& observed) {
    const std::vector<double>& p = pred.traces();
    if (observed.size() != std::size_t(pred.nt()) * std::size_t(pred.npoints()))
        throw ParameterError("objective: " + std::to_string(observed.size()) +
                             " observed samples for a " + std::to_string(pred.nt()) + " x " +
                             std::to_string(pred.npoints()) + " record");
    double half_sq = 0.0;   // accumulated sample by sample, in table order
    auto o = observed.begin();
    for (double v : p) {
        const double d = v - *o++;
        half_sq += 0.5 * d * d;
    }
    return half_sq;
}

namespace {

// Adjoint of SeismicModel's edge-clamped extension (proj/src/model.cpp:92-100): a padded
// node contributes to the physical cell whose value it copies.  `padded` is a compact
// row-major array over the computational grid; nodes are visited in storage order.
std::vector<double> fold_onto_physical(const SeismicModel& model, const std::vector<double>& padded) {
    const std::vector<long>& phys = model.physical_shape();
    const std::vector<long>& full = model.grid()->shape();
    const std::size_t rank = full.size();
    // per axis: computational index -> physical index
    std::vector<std::vector<long>> to_phys(rank);
    for (std::size_t a = 0; a < rank; ++a) {
        to_phys[a].resize(std::size_t(full[a]));
        for (long i = 0; i < full[a]; ++i)
            to_phys[a][std::size_t(i)] = std::clamp(i - model.nbl(), 0L, phys[a] - 1);
    }
    std::size_t cells = 1;
    for (long e : phys) cells *= std::size_t(e);
    std::vector<double> out(cells, 0.0);
    // walk the padded array as (rows of the last axis) x (last axis)
    const long row_len = full[rank - 1];
    const std::vector<long>& last = to_phys[rank - 1];
    std::vector<long> idx(rank, 0);
    const std::size_t rows = padded.size() / std::size_t(row_len);
    for (std::size_t r = 0; r < rows; ++r) {
        std::size_t base = 0;
        for (std::size_t a = 0; a + 1 < rank; ++a)
            base = base * std::size_t(phys[a]) + std::size_t(to_phys[a][std::size_t(idx[a])]);
        double* dst = out.data() + base * std::size_t(phys[rank - 1]);
        const double* src = padded.data() + r * std::size_t(row_len);
        for (long l = 0; l < row_len; ++l) dst[last[std::size_t(l)]] += src[l];
        for (std::size_t a = rank - 1; a-- > 0;) {   // advance the row index (odometer)
            if (++idx[a] < full[a]) break;
            idx[a] = 0;
        }
    }
    return out;
}

struct ShotPolicy {
    int space_order;
    long save_every;        // image against every save_every-th forward level
    long checkpoint_every;  // or keep checkpoints and recompute (exact imaging condition)
};

void check_policy(const ShotPolicy& p, const char* who) {
    if (p.save_every < 1) throw ParameterError(std::string(who) + ": save_every must be >= 1");
    if (p.checkpoint_every != 0 && (p.checkpoint_every < 2 || p.save_every != 1))
        throw ParameterError(std::string(who) + ": checkpoint_every must be >= 2 (with save_every 1)");
}

// One shot on a bound engine: forward run keeping the history in HBM, misfit and residual
// on the host, gradient sweep, fold.  The predicted record lands in geom.rec() as with the
// operator interface.
GradientResult evaluate_shot(Engine& e, const SeismicModel& model, AcquisitionGeometry& geom,
                             const std::vector<double>& observed, const ShotPolicy& pol,
                             std::vector<double>& padded_scratch) {
    check_space_order(pol.space_order);
    check_cfl(model, geom, pol.space_order);
    SparseFunction& rec = *geom.rec();
    const double* src = geom.src()->traces().data();
    if (pol.checkpoint_every > 0)
        e.check(sfb_forward_checkpointed(e.plan(), src, rec.traces().data(), pol.checkpoint_every, nullptr));
    else
        e.check(sfb_forward(e.plan(), src, rec.traces().data(), pol.save_every, nullptr));
    GradientResult out;
    out.objective = objective(rec, observed);
    out.residual.resize(observed.size());
    std::transform(rec.traces().begin(), rec.traces().end(), observed.begin(), out.residual.begin(),
                   [](double pred, double obs) { return pred - obs; });
    const std::vector<long>& full = model.grid()->shape();
    std::size_t nodes = 1;
    for (long n : full) nodes *= std::size_t(n);
    padded_scratch.assign(nodes, 0.0);
    sfb_field_mview gv{};
    gv.ptr = padded_scratch.data();
    long stride = 1;
    for (std::size_t a = full.size(); a-- > 0;) {
        gv.stride[a] = stride;
        stride *= full[a];
    }
    e.check(sfb_gradient(e.plan(), out.residual.data(), &gv, nullptr));
    out.gradient = fold_onto_physical(model, padded_scratch);
    return out;
}

}  // namespace

GradientResult fwi_gradient(const SeismicModel& model, AcquisitionGeometry& geom,
                            const std::vector<double>& observed, int space_order, Backend,
                            long save_every, long checkpoint_every) {
    const ShotPolicy pol{space_order, save_every, checkpoint_every};
    check_policy(pol, "fwi_gradient");
    check_space_order(space_order);
    check_cfl(model, geom, space_order);
    Engine engine(model, geom, space_order);
    std::vector<double> scratch;
    return evaluate_shot(engine, model, geom, observed, pol, scratch);
}

namespace {

// A lane = one CUDA device slot that evaluates shots one after the other on an engine it
// keeps: the plan, its wavefield / history buffers and tensor maps live as long as the
// inversion.  Per shot only the two point tables are rebound, per iteration the model.
class ShotLane {
public:
    explicit ShotLane(int device_ordinal) : device_(device_ordinal) {}

    GradientResult evaluate(const SeismicModel& model, long model_version, AcquisitionGeometry& geom,
                            const std::vector<double>& observed, const ShotPolicy& pol) {
        set_device(device_);
        if (!engine_ || !engine_->fits(model, geom, pol.space_order)) {
            engine_.reset();   // free the old plan's HBM before the new one allocates
            engine_ = std::make_unique<Engine>(model, geom, pol.space_order);
            ++plans_built_;
        } else {
            if (bound_version_ != model_version) engine_->rebind_model(model);
            engine_->rebind_geometry(geom);
        }
        bound_version_ = model_version;
        return evaluate_shot(*engine_, model, geom, observed, pol, scratch_);
    }
    long plans_built() const { return plans_built_; }

private:
    int device_;
    std::unique_ptr<Engine> engine_;
    long bound_version_ = -1;
    long plans_built_ = 0;
    std::vector<double> scratch_;
};

// All shots of one iteration over the lanes.  Shots are handed out dynamically (a lane takes
// the next unclaimed shot when it is free); results are stored by shot index so that the
// reduction order -- and with it the result -- does not depend on the lane count.
class ShotPool {
public:
    ShotPool(const FwiConfig& cfg, int caller_device) {
        const std::size_t lanes = cfg.nthreads > 1 ? std::size_t(cfg.nthreads) : 1;
        for (std::size_t i = 0; i < lanes; ++i)
            lanes_.emplace_back(cfg.devices.empty() ? caller_device : cfg.devices[i % cfg.devices.size()]);
    }

    std::vector<GradientResult> evaluate(const SeismicModel& model, long model_version,
                                         std::vector<AcquisitionGeometry>& shots,
                                         const std::vector<std::vector<double>>& observed,
                                         const ShotPolicy& pol) {
        std::vector<GradientResult> terms(shots.size());
        std::vector<std::string> errors(shots.size());
        std::atomic<std::size_t> next{0};
        auto drain = [&](ShotLane& lane) {
            for (std::size_t s; (s = next.fetch_add(1)) < shots.size();) {
                try {
                    terms[s] = lane.evaluate(model, model_version, shots[s], observed[s], pol);
                } catch (const std::exception& e) {
                    errors[s] = e.what()[0] ? e.what() : "unknown failure";
                }
            }
        };
        std::vector<std::thread> crew;
        for (std::size_t i = 1; i < lanes_.size() && i < shots.size(); ++i)
            crew.emplace_back(drain, std::ref(lanes_[i]));
        const int callers_device = device();
        drain(lanes_[0]);   // the caller is lane 0
        set_device(callers_device);
        for (std::thread& t : crew) t.join();
        for (std::size_t s = 0; s < errors.size(); ++s)
            if (!errors[s].empty())
                throw StabilityError("fwi: shot " + std::to_string(s) + " failed: " + errors[s]);
        return terms;
    }

private:
    std::vector<ShotLane> lanes_;
};

double max_abs(const std::vector<double>& v) {
    double m = 0.0;
    for (double x : v) m = std::max(m, std::abs(x));
    return m;
}

}  // namespace

FwiResult fwi(SeismicModel& model, std::vector<AcquisitionGeometry>& shots,
              const std::vector<std::vector<double>>& observed, const FwiConfig& cfg,
              const std::vector<double>* true_m) {
    if (shots.empty() || observed.size() != shots.size())
        throw ParameterError("fwi: " + std::to_string(shots.size()) + " shots but " +
                             std::to_string(observed.size()) + " observed records");
    if (!(cfg.m_min > 0.0 && cfg.m_max > cfg.m_min))
        throw ParameterError("fwi: the model box needs 0 < m_min < m_max");
    const ShotPolicy pol{cfg.space_order, cfg.save_every, cfg.checkpoint_every};
    check_policy(pol, "fwi");

    std::vector<double> m = model.physical_m();
    auto distance_to_truth = [&] {   // rms over the physical cells; 0 without a reference model
        if (!true_m) return 0.0;
        double sq = 0.0;
        for (std::size_t i = 0; i < m.size(); ++i) sq += (m[i] - (*true_m)[i]) * (m[i] - (*true_m)[i]);
        return std::sqrt(sq / double(m.size()));
    };

    ShotPool pool(cfg, device());
    FwiResult history;
    double step = 0.0;   // fixed after the first gradient: step_scale * max|m| / max|g|
    for (long it = 0; it < cfg.n_iter; ++it) {
        const std::vector<GradientResult> terms = pool.evaluate(model, it, shots, observed, pol);
        // reduce in shot order
        double phi = 0.0;
        std::vector<double> g(m.size(), 0.0);
        for (const GradientResult& term : terms) {
            phi += term.objective;
            std::transform(g.begin(), g.end(), term.gradient.begin(), g.begin(), std::plus<double>());
        }
        if (!std::isfinite(phi))
            throw StabilityError("fwi: the objective of iteration " + std::to_string(it) + " is not finite");
        history.objectives.push_back(phi);
        history.model_rms.push_back(distance_to_truth());
        if (it == 0) {
            const double steepest = max_abs(g);
            if (steepest == 0.0) {   // already at a stationary point: nothing to do
                history.final_m = std::move(m);
                return history;
            }
            step = cfg.step_scale * max_abs(m) / steepest;
        }
        // projected descent step onto the box [m_min, m_max]
        std::transform(m.begin(), m.end(), g.begin(), m.begin(), [&](double mi, double gi) {
            return std::clamp(mi - step * gi, cfg.m_min, cfg.m_max);
        });
        model.set_physical_m(m);
    }
    history.model_rms.push_back(distance_to_truth());
    history.final_m = std::move(m);
    return history;
}

}  // namespace sfb
