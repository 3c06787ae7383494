// engine_step.cu -- the acoustic time loops behind the C-ABI.
//
// They restate run_wave / run_gradient / run_window of the reference
// (proj/src/seismic_ops.cpp:44-54,137-147): zero the wavefield and the sampled traces,
// then step t over [1, nt-1), ascending for the forward operator and descending for the
// adjoint and gradient operators, each step being dense update -> scatter -> gather in
// that order (proj/tests/test_compiler.cpp:109-120).
#include <cstdlib>

#include "engine.hpp"
#include "point_kernels.cuh"

namespace sfb {

// ---- stepping ------------------------------------------------------------------------------


OpRoles roles(int op) {
    switch (op) {
    case SFB_OP_FORWARD: return {false, SFB_CLOUD_SRC, SFB_CLOUD_REC, false};
    case SFB_OP_ADJOINT: return {true, SFB_CLOUD_REC, SFB_CLOUD_SRC, false};
    case SFB_OP_GRADIENT: return {true, SFB_CLOUD_REC, -1, true};
    case SFB_OP_TTI_FORWARD: return {false, SFB_CLOUD_SRC, SFB_CLOUD_REC, false};
    default: throw Failure(SFB_ERR_PARAMETER, "unknown operator id");
    }
}

void step_begin(Plan& P, int op, long long save_every) {
    const OpRoles ro = roles(op);
    require(P.model_set, SFB_ERR_BINDING, "model fields are not bound (sfb_set_model)");
    require(P.cloud[ro.inj].set, SFB_ERR_BINDING, "injected point cloud is not bound");
    require(ro.smp < 0 || P.cloud[ro.smp].set, SFB_ERR_BINDING,
            "sampled point cloud is not bound");
    require(save_every >= 0, SFB_ERR_PARAMETER, "save_every must be >= 0");
    // run_wave / run_gradient: zero the wavefield and the sampled traces
    SFB_CUDA(cudaMemsetAsync(P.u[0].p, 0, size_t(P.ucount) * 4, P.s_main));
    SFB_CUDA(cudaMemsetAsync(P.u[1].p, 0, size_t(P.ucount) * 4, P.s_main));
    if (ro.smp >= 0) {
        Cloud& c = P.cloud[ro.smp];
        SFB_CUDA(cudaMemsetAsync(c.tr_out.p, 0, size_t(P.desc.nt) * c.np * 4, P.s_main));
    }
    if (op == SFB_OP_FORWARD) {
        P.history_valid = false;
        P.ckpt_valid = false;
        P.save_every = save_every;
        if (save_every > 0) {
            P.nslots = (P.desc.nt - 1) / save_every + 1;
            P.snaps.alloc(size_t(P.nslots) * P.ccount * 4, false);
            SFB_CUDA(cudaMemsetAsync(P.snaps.p, 0, size_t(P.nslots) * P.ccount * 4, P.s_main));
        }
    }
    if (ro.imaging) {
        require(P.history_valid && P.save_every > 0, SFB_ERR_PARAMETER,
                "gradient_operator: saved forward history required");
        P.grad.alloc(size_t(P.ccount) * 4, false);
        SFB_CUDA(cudaMemsetAsync(P.grad.p, 0, size_t(P.ccount) * 4, P.s_main));
    }
    P.live_level[0] = P.live_level[1] = -1;
    P.launches = 0;
    P.main_pending = P.bnd_pending = false;
}


void part_range(const Plan& P, int part, int& lo, int& hi) {
    const int K = P.K, n0 = P.n0;
    switch (part) {
    case SFB_PART_ALL: lo = 0; hi = n0; break;
    case SFB_PART_LOW: lo = 0; hi = std::min(K, n0); break;
    case SFB_PART_HIGH: lo = std::max(n0 - K, std::min(K, n0)); hi = n0; break;
    case SFB_PART_INTERIOR: lo = std::min(K, n0); hi = std::max(n0 - K, std::min(K, n0)); break;
    default: throw Failure(SFB_ERR_PARAMETER, "unknown slab part");
    }
}

// d0 chunk of the single-launch slab step: at least two chunks (the first sweeps up, the last
// down), whole waves of the resident blocks, every chunk charged half a plane per queue-fill
// plane like select_variant does
int fused_chunk(const Plan& P) {
    const StepVariant& v = *P.variant;
    const void* fn = v.func_push ? v.func_push : v.func;
    int bps = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, v.nthreads, v.smem) != cudaSuccess || bps < 1)
        bps = 1;
    const long long tiles = ((P.N[2] + v.tile_x - 1) / v.tile_x) * ((P.N[1] + v.tile_y - 1) / v.tile_y);
    const long long slots = (long long)P.sm_count * bps;
    int best = 2;
    double best_score = -1;
    const int max_nch = std::max(2, P.n0 / std::max(1, 2 * P.K));
    for (int nch = 2; nch <= max_nch; ++nch) {
        const int chunk = (P.n0 + nch - 1) / nch;
        if (chunk < P.K) break;
        const int real = (P.n0 + chunk - 1) / chunk;
        if (real < 2) continue;
        const long long total = tiles * real;
        const long long waves = (total + slots - 1) / slots;
        const double fill = double(total) / double(waves * slots);
        const double score = fill / (1.0 + (2.0 * P.K / chunk) * 0.5);
        if (score > best_score + 1e-9) {
            best_score = score;
            best = real;
        }
        if (total > 16 * slots) break;
    }
    return (P.n0 + best - 1) / best;
}

cudaStream_t part_stream(Plan& P, int part) {
    const bool bnd = part == SFB_PART_LOW || part == SFB_PART_HIGH || part == kPartBoundaryPair;
    cudaStream_t st = bnd ? P.s_bnd : P.s_main;
    // the other stream's last work of the previous step wrote planes this launch reads
    if (bnd && P.main_pending) {
        SFB_CUDA(cudaStreamWaitEvent(P.s_bnd, P.ev_main, 0));
        P.main_pending = false;
    }
    if (!bnd && P.bnd_pending) {
        SFB_CUDA(cudaStreamWaitEvent(P.s_main, P.ev_bnd, 0));
        P.bnd_pending = false;
    }
    return st;
}

void mark_stream(Plan& P, int part) {
    // whole-domain launches have no other stream to order against, and an event record
    // between two kernels would break their programmatic dependent launch
    if (part == SFB_PART_ALL || part == kPartSlabFused) return;
    const bool bnd = part == SFB_PART_LOW || part == SFB_PART_HIGH || part == kPartBoundaryPair;
    if (P.s_bnd == P.s_main) return;
    if (bnd) {
        SFB_CUDA(cudaEventRecord(P.ev_bnd, P.s_bnd));
        P.bnd_pending = true;
    } else {
        SFB_CUDA(cudaEventRecord(P.ev_main, P.s_main));
        P.main_pending = true;
    }
}


// the acoustic stepping entry points: no TTI state, and imaging needs a bound history
// (t % save_every below must not divide by zero across the C ABI)
static void check_step_op(const Plan& P, int, const OpRoles& ro, const StepExtras* ex) {
    require(!ro.imaging || (ex && ex->usave) || (P.history_valid && P.save_every > 0),
            SFB_ERR_PARAMETER, "gradient_operator: saved forward history required");
}

void step_compute(Plan& P, int op, long long t, int part, const StepExtras* ex) {
    const OpRoles ro = roles(op);
    // the TTI pair has its own update launches (engine_tti.cu); only its point work comes here
    require(op != SFB_OP_TTI_FORWARD, SFB_ERR_PARAMETER,
            "the TTI operator steps through sfb_tti_step_rot / sfb_tti_step_update");
    check_step_op(P, op, ro, ex);
    require(t >= 1 && t <= P.desc.nt - 2, SFB_ERR_PARAMETER, "time index outside [1, nt-1)");
    int lo, hi;
    const bool pair = part == kPartBoundaryPair;   // needs n0 >= 2K (split_slabs guarantees it)
    const bool fused = part == kPartSlabFused;
    if (pair || fused) {
        require(P.n0 >= 2 * P.K, SFB_ERR_PARAMETER, "slab thinner than two halo widths");
        lo = 0;
        hi = P.n0;
    } else {
        part_range(P, part, lo, hi);
    }
    if (hi <= lo) return;
    const int cur = int(t & 1), oth = cur ^ 1;
    const long long tnew = ro.backward ? t - 1 : t + 1;
    StepParams sp{};
    sp.k = P.coef;
    sp.dz = P.dz.as<float>();
    sp.dy = P.dy.as<float>();
    sp.dx = P.dx.as<float>();
    sp.uo = (ex && ex->alt) ? P.f[oth].as<float>() : P.u[oth].as<float>();
    sp.N1 = int(P.N[1]);
    sp.N2 = int(P.N[2]);
    sp.pitch = P.pitch;
    sp.plane = P.plane;
    sp.z_lo = lo;
    sp.z_hi = hi;
    sp.chunk = pair ? P.K
               : fused ? fused_chunk(P)
               : (part == SFB_PART_ALL || part == SFB_PART_INTERIOR) ? P.chunk : (hi - lo);
    sp.z_jump = pair ? P.n0 - 2 * P.K : 0;   // block z = 1 starts at plane n0 - K
    sp.push_planes = fused ? P.K : sp.chunk;   // boundary launches push all they compute
    sp.desc_last = fused ? 1 : 0;
    // linked slabs: the boundary plane groups are also written into the neighbours' ghosts
    if (!(ex && ex->alt)) {
        // mirror of owned plane z: low group -> peer_lo + z planes, high group -> peer_hi +
        // (z - (n0 - K)) planes; owned plane z itself sits at uo + (z + K) planes
        const long long d_lo = P.peer_lo[oth] ? P.peer_lo[oth] - (sp.uo + (long long)P.K * P.plane) : 0;
        const long long d_hi = P.peer_hi[oth] ? P.peer_hi[oth] - (sp.uo + (long long)P.n0 * P.plane) : 0;
        if (pair || fused) {
            sp.peer_delta0 = d_lo;
            sp.peer_delta1 = d_hi;
        } else if (part == SFB_PART_LOW) {
            sp.peer_delta0 = d_lo;
        } else if (part == SFB_PART_HIGH) {
            sp.peer_delta0 = d_hi;
        }
    }
    if (ex) {
        sp.snap = ex->snap;
        sp.usave = ex->usave;
        if (ex->usave) sp.grad = P.grad.as<float>();
    } else {
        if (op == SFB_OP_FORWARD && P.save_every > 0 && tnew % P.save_every == 0)
            sp.snap = P.snaps.as<float>() + (tnew / P.save_every) * P.ccount;
        if (ro.imaging && t % P.save_every == 0) {
            sp.usave = P.snaps.as<float>() + (t / P.save_every) * P.ccount;
            sp.grad = P.grad.as<float>();
        }
    }
    const StepVariant& v = *P.variant;
    dim3 grid(unsigned((P.N[2] + v.tile_x - 1) / v.tile_x),
              unsigned((P.N[1] + v.tile_y - 1) / v.tile_y),
              pair ? 2u : unsigned((hi - lo + sp.chunk - 1) / sp.chunk));
    cudaStream_t st = part_stream(P, part);
    StepMaps maps;
    const bool alt = ex && ex->alt;
    maps.u = alt ? P.tm_fu[cur] : P.tm_u[cur];
    maps.f = alt ? P.tm_fo[cur] : P.tm_o[cur];
    maps.o = alt ? P.tm_fo[oth] : P.tm_o[oth];
    maps.r = P.tm_r;
    maps.d = P.sep ? P.tm_r : P.tm_d;
    if (sp.peer_delta0 || sp.peer_delta1 || fused) {
        require(v.launch_push != nullptr, SFB_ERR_CAPABILITY,
                "the selected tile shape has no halo-push kernel (sfb_link_peers picks one that has)");
        SFB_CUDA(v.launch_push(maps, sp, grid, st));
    } else {
        SFB_CUDA(v.launch(maps, sp, grid, st));
    }
    ++P.launches;
    mark_stream(P, part);
    if (!alt && (part == SFB_PART_ALL || part == SFB_PART_INTERIOR || fused)) {
        P.live_level[cur] = t;
        P.live_level[oth] = tnew;
    }
}

// part: SFB_PART_ALL = every node + gather; SFB_PART_LOW = nodes of both boundary plane
// groups (boundary stream); SFB_PART_INTERIOR = remaining nodes + gather
void step_points(Plan& P, int op, long long t, int part, float* target_override, bool allow_gather,
                 const StepExtras* ex, float* peer_lo, float* peer_hi) {
    const OpRoles ro = roles(op);
    check_step_op(P, op, ro, ex);
    const int cur = int(t & 1), oth = cur ^ 1;
    const long long tnew = ro.backward ? t - 1 : t + 1;
    Cloud& ci = P.cloud[ro.inj];
    require(ci.has_in, SFB_ERR_BINDING, "no traces uploaded for the injected cloud");
    struct Range {
        long long b, e;
    };
    Range rg[2] = {{0, 0}, {0, 0}};
    int nr = 1;
    bool gather = false;
    if (part == SFB_PART_ALL || part == kPartSlabFused) {
        rg[0] = {0, ci.ncell};
        gather = ro.smp >= 0 && allow_gather;
    } else if (part == SFB_PART_LOW || part == SFB_PART_HIGH) {
        rg[0] = {0, ci.cell_lo_end};
        rg[1] = {ci.cell_hi_begin, ci.ncell};
        nr = 2;
    } else {
        rg[0] = {ci.cell_lo_end, ci.cell_hi_begin};
        gather = ro.smp >= 0;
    }
    cudaStream_t st = part_stream(P, part);
    for (int i = 0; i < nr; ++i) {
        const bool do_gather = gather && i == 0;
        const long long ncell = std::max<long long>(0, rg[i].e - rg[i].b);
        if (ncell == 0 && !do_gather) continue;
        PointParams pp{};
        pp.ncell = int(ncell);
        pp.cell_start = ci.cell_start.as<int>() + rg[i].b;
        pp.cell_u = ci.cell_u.as<long long>() + rg[i].b;
        pp.cell_c = ci.cell_c.as<long long>() + rg[i].b;
        pp.ent_point = ci.ent_point.as<int>();
        pp.ent_w = ci.ent_w.as<float>();
        pp.inj_row = ci.tr_in.as<float>() + t * ci.np;
        pp.target = target_override ? target_override : P.u[oth].as<float>();
        pp.r = P.r.as<float>();
        pp.inv_dt2 = P.coef.inv_dt2;
        if (part == SFB_PART_LOW || part == SFB_PART_HIGH || part == kPartSlabFused) {
            pp.peer_lo = target_override ? peer_lo : P.peer_lo[oth];
            pp.peer_hi = target_override ? peer_hi : P.peer_hi[oth];
            pp.plane = P.plane;
            pp.K = P.K;
            pp.n0 = P.n0;
        }
        if (ex) {
            pp.snap = ex->snap;
            pp.usave = ex->usave;
            if (ex->usave) pp.grad = P.grad.as<float>();
        } else {
            if (op == SFB_OP_FORWARD && P.save_every > 0 && tnew % P.save_every == 0)
                pp.snap = P.snaps.as<float>() + (tnew / P.save_every) * P.ccount;
            if (ro.imaging && t % P.save_every == 0) {
                pp.usave = P.snaps.as<float>() + (t / P.save_every) * P.ccount;
                pp.grad = P.grad.as<float>();
            }
        }
        int nb_smp = 0;
        if (do_gather) {
            Cloud& cs = P.cloud[ro.smp];
            pp.nsmp = int(cs.np);
            pp.smp_idx = cs.smp_idx.as<long long>();
            pp.smp_w = cs.smp_w.as<float>();
            pp.field = P.u[cur].as<float>();
            pp.smp_row = cs.tr_out.as<float>() + t * cs.np;
            pp.ncorner = 1 << P.ndim;
            const int off = 3 - P.ndim;
            for (int c = 0; c < pp.ncorner; ++c) {
                long long o = 0;
                for (int a = 0; a < P.ndim; ++a)
                    if ((c >> a) & 1) o += (off + a == 0) ? P.plane : (off + a == 1 ? P.pitch : 1);
                pp.corner_off[c] = o;
            }
            nb_smp = int((cs.np + kPointThreads - 1) / kPointThreads);
        }
        const int nb_inj = int((ncell + kPointThreads - 1) / kPointThreads);
        if (nb_inj + nb_smp == 0) continue;
        SFB_CUDA(launch_pdl(&point_step_kernel, dim3(unsigned(nb_inj + nb_smp)), kPointThreads, 0, st,
                            pp, nb_inj));
        ++P.launches;
    }
    mark_stream(P, part);
}

void finite_guard(Plan& P, const char* what, int only) {
    P.flag.alloc(sizeof(int), false);
    SFB_CUDA(cudaMemsetAsync(P.flag.p, 0, sizeof(int), P.s_main));
    for (int b = 0; b < 2; ++b) {
        if (only >= 0 && b != only) continue;
        finite_check_kernel<<<P.sm_count * 8, 256, 0, P.s_main>>>(P.u[b].as<float>(), P.ucount,
                                                                 P.flag.as<int>());
        SFB_CUDA(cudaGetLastError());
    }
    int bad = 0;
    SFB_CUDA(cudaMemcpyAsync(&bad, P.flag.p, sizeof(int), cudaMemcpyDeviceToHost, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    if (bad) throw Failure(SFB_ERR_STABILITY, std::string(what) + ": wavefield went non-finite");
}

void run_op(Plan& P, int op, long long save_every, sfb_report* rep, double* stream_out,
            const double* stream_in) {
    const OpRoles ro = roles(op);
    std::unique_ptr<RowFeeder> feed;
    if (stream_in) {
        feed.reset(new RowFeeder(P, P.cloud[ro.inj], stream_in, ro.backward));
        P.cloud[ro.inj].has_in = true;   // every row a step reads is sent before that step
    }
    step_begin(P, op, save_every);
    const long long nt = P.desc.nt;
    std::unique_ptr<RowStreamer> rs;
    if (stream_out && ro.smp >= 0) rs.reset(new RowStreamer(P, P.cloud[ro.smp], stream_out));
    SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
    for (long long i = 0; i < nt - 2; ++i) {
        const long long t = ro.backward ? nt - 2 - i : 1 + i;
        if (feed) feed->before_step(t);
        step_compute(P, op, t, SFB_PART_ALL);
        step_points(P, op, t, SFB_PART_ALL);
        if (rs) rs->row_done(t);
    }
    SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    if (feed) feed->finish();
    if (rs) rs->flush();   // the last rows travel while the NaN guard scans the fields
    // a non-finite value of one level stays in place in the next one (the update adds twice the
    // centre value), so the level computed last holds every node that ever went bad
    int newest = -1;
    for (int b = 0; b < 2; ++b)
        if (nt > 2 && P.live_level[b] == (ro.backward ? 0 : nt - 1)) newest = b;
    finite_guard(P, op == SFB_OP_FORWARD ? "forward" : (op == SFB_OP_ADJOINT ? "adjoint" : "gradient"),
                 newest);
    float ms = 0.f;
    SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
    if (op == SFB_OP_FORWARD && save_every > 0) P.history_valid = true;
    if (rs) rs->finish();
    if (rep) {
        const long steps = long(std::max<long long>(0, nt - 2));
        int D = P.ndim;
        const long long fpp = 3LL * P.K * D + 3LL * D + 11 + (ro.imaging ? 7 : 0);
        const double pts = double(P.N[0]) * double(P.N[1]) * double(P.N[2]);
        const double own = double(P.n0) * double(P.N[1]) * double(P.N[2]);
        rep->seconds = ms * 1e-3;
        rep->steps = steps;
        rep->flops = (long long)(double(fpp) * own * steps);
        rep->gflops = rep->seconds > 0 ? double(rep->flops) / rep->seconds / 1e9 : 0.0;
        rep->gpts_per_s = rep->seconds > 0 ? own * steps / rep->seconds / 1e9 : 0.0;
        rep->kernel_launches = P.launches;
        (void)pts;
    }
}

// ---- checkpointed history: recompute instead of store ------------------
// The reference keeps the whole forward history in RAM (proj/src/seismic_ops.cpp:66-68) and
// marks checkpointing out of scope.  At config-3 size the full history is
// 415 GB; save_every thins it, this removes the limit: the forward run keeps only the state
// (levels kC-1 and kC) at every C-th level, and the backward sweep recomputes one segment of
// C levels at a time into a small buffer before imaging against it -- every level, i.e. the
// reference's exact imaging condition -- at the price of one extra forward pass.

void forward_checkpointed(Plan& P, long long C, sfb_report* rep, double* stream_out) {
    require(C >= 2, SFB_ERR_PARAMETER, "checkpoint_every must be >= 2");
    require(P.n0 == P.N[0], SFB_ERR_CAPABILITY, "checkpointed runs are single-slab in this round");
    const int op = SFB_OP_FORWARD;
    step_begin(P, op, 0);
    const long long nt = P.desc.nt;
    P.ckpt_valid = false;
    P.ckpt_every = C;
    P.nseg = (nt - 1 + C - 1) / C;
    P.ckpt.alloc(size_t(P.nseg + 1) * 2 * P.ccount * 4, false);
    SFB_CUDA(cudaMemsetAsync(P.ckpt.p, 0, size_t(P.nseg + 1) * 2 * P.ccount * 4, P.s_main));
    std::unique_ptr<RowStreamer> rs;
    if (stream_out) rs.reset(new RowStreamer(P, P.cloud[SFB_CLOUD_REC], stream_out));
    SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
    for (long long t = 1; t < nt - 1; ++t) {
        const long long tnew = t + 1;
        StepExtras ex;
        if (tnew % C == 0) ex.snap = P.ckpt.as<float>() + ((tnew / C) * 2 + 1) * P.ccount;
        if (tnew % C == C - 1) ex.snap = P.ckpt.as<float>() + (((tnew + 1) / C) * 2 + 0) * P.ccount;
        step_compute(P, op, t, SFB_PART_ALL, &ex);
        step_points(P, op, t, SFB_PART_ALL, nullptr, true, &ex);
        if (rs) rs->row_done(t);
    }
    SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    float ms = 0.f;
    SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
    finite_guard(P, "forward");
    if (rs) rs->finish();
    P.ckpt_valid = true;
    P.history_valid = false;
    if (rep) {
        const double own = double(P.n0) * double(P.N[1]) * double(P.N[2]);
        rep->seconds = ms * 1e-3;
        rep->steps = long(std::max<long long>(0, nt - 2));
        rep->flops = (long long)(double(3LL * P.K * P.ndim + 3LL * P.ndim + 11) * own * rep->steps);
        rep->gflops = ms > 0 ? double(rep->flops) / (ms * 1e-3) / 1e9 : 0.0;
        rep->gpts_per_s = ms > 0 ? own * rep->steps / (ms * 1e-3) / 1e9 : 0.0;
        rep->kernel_launches = P.launches;
    }
}

void gradient_checkpointed(Plan& P, sfb_report* rep) {
    require(P.ckpt_valid, SFB_ERR_PARAMETER, "gradient_operator: saved forward history required");
    const long long nt = P.desc.nt, C = P.ckpt_every;
    const int G = SFB_OP_GRADIENT, F = SFB_OP_FORWARD;
    // v (the adjoint wavefield) lives in u[2]; the recomputed forward pair in f[2]
    const bool new_f = !P.f[0].p;
    for (int b = 0; b < 2; ++b) P.f[b].alloc(size_t(P.ucount) * 4, true);
    if (new_f) make_tensor_maps(P);
    P.seg.alloc(size_t(C) * P.ccount * 4, false);
    P.grad.alloc(size_t(P.ccount) * 4, false);
    SFB_CUDA(cudaMemsetAsync(P.grad.p, 0, size_t(P.ccount) * 4, P.s_main));
    SFB_CUDA(cudaMemsetAsync(P.u[0].p, 0, size_t(P.ucount) * 4, P.s_main));
    SFB_CUDA(cudaMemsetAsync(P.u[1].p, 0, size_t(P.ucount) * 4, P.s_main));
    P.launches = 0;
    P.main_pending = P.bnd_pending = false;
    Cloud& cr = P.cloud[SFB_CLOUD_REC];
    require(cr.has_in && P.cloud[SFB_CLOUD_SRC].has_in, SFB_ERR_BINDING,
            "checkpointed gradient needs the source and residual traces on the device");
    const size_t lvl = size_t(P.ccount) * 4, ghost = size_t(P.K) * P.plane;
    SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
    for (long long k = P.nseg - 1; k >= 0; --k) {
        const long long t_lo = k * C, t_top = std::min((k + 1) * C, nt - 2);
        if (t_top <= t_lo) continue;
        // restore the forward state (levels t_lo - 1, t_lo) of this segment
        const float* ck = P.ckpt.as<float>() + (k * 2) * P.ccount;
        SFB_CUDA(cudaMemcpyAsync(P.f[(t_lo + 1) & 1].as<float>() + ghost, ck, lvl,
                                 cudaMemcpyDeviceToDevice, P.s_main));
        SFB_CUDA(cudaMemcpyAsync(P.f[t_lo & 1].as<float>() + ghost, ck + P.ccount, lvl,
                                 cudaMemcpyDeviceToDevice, P.s_main));
        if (k == 0)  // level 1 is never produced by a step: it is identically zero
            SFB_CUDA(cudaMemsetAsync(P.seg.p, 0, lvl, P.s_main));
        // recompute levels t_lo+1 .. t_top into the segment buffer
        for (long long t = std::max<long long>(t_lo, 1); t < t_top; ++t) {
            StepExtras ex;
            ex.alt = true;
            ex.snap = P.seg.as<float>() + (t + 1 - t_lo - 1) * P.ccount;
            step_compute(P, F, t, SFB_PART_ALL, &ex);
            step_points(P, F, t, SFB_PART_ALL, P.f[(t & 1) ^ 1].as<float>(), false, &ex);
        }
        // backward sweep over the segment, imaging against every recomputed level
        for (long long t = t_top; t > t_lo; --t) {
            StepExtras ex;
            ex.usave = P.seg.as<float>() + (t - t_lo - 1) * P.ccount;
            step_compute(P, G, t, SFB_PART_ALL, &ex);
            step_points(P, G, t, SFB_PART_ALL, nullptr, true, &ex);
        }
    }
    SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    float ms = 0.f;
    SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
    finite_guard(P, "gradient");
    if (rep) {
        const double own = double(P.n0) * double(P.N[1]) * double(P.N[2]);
        rep->seconds = ms * 1e-3;
        rep->steps = long(std::max<long long>(0, nt - 2));
        rep->flops = (long long)(double(2 * (3LL * P.K * P.ndim + 3LL * P.ndim + 11) + 7) * own * rep->steps);
        rep->gflops = ms > 0 ? double(rep->flops) / (ms * 1e-3) / 1e9 : 0.0;
        rep->gpts_per_s = ms > 0 ? own * rep->steps / (ms * 1e-3) / 1e9 : 0.0;
        rep->kernel_launches = P.launches;
    }
}

void run_window(Plan& P, int op, long long t_from, long long t_to, bool with_points,
                sfb_report* report) {
    const OpRoles ro = roles(op);
    require(t_from >= 1 && t_to <= P.desc.nt - 1 && t_from <= t_to, SFB_ERR_PARAMETER,
            "run_steps: window outside [1, nt-1)");
    const long before = P.launches;
    const bool tti = op == SFB_OP_TTI_FORWARD;
    if (tti) {
        require(P.tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
        require(P.n0 == P.N[0], SFB_ERR_CAPABILITY, "TTI windows run one whole domain");
        require(P.tti_chunk[0] > 0, SFB_ERR_PARAMETER, "call sfb_step_begin(SFB_OP_TTI_FORWARD) first");
    }
    auto enqueue = [&] {
        for (long long i = 0; i < t_to - t_from; ++i) {
            const long long t = ro.backward ? t_to - 1 - i : t_from + i;
            if (tti) {   // the two launches of the rotated pair (engine_tti.cu)
                tti_rot(P, t, SFB_PART_ALL);
                tti_update(P, t, SFB_PART_ALL, with_points);
                continue;
            }
            step_compute(P, op, t, SFB_PART_ALL);
            if (with_points) step_points(P, op, t, SFB_PART_ALL);
        }
    };
    // SFB_GRAPH=1 (measurement aid): the window is captured into a CUDA graph and replayed as
    // one graph launch.  The loop is device-bound (the host enqueues a step several times
    // faster than the device runs it), so this is not the default: see DESIGN.md 3.2.
    static const bool use_graph = std::getenv("SFB_GRAPH") != nullptr;
    if (use_graph) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        SFB_CUDA(cudaStreamBeginCapture(P.s_main, cudaStreamCaptureModeThreadLocal));
        enqueue();
        SFB_CUDA(cudaStreamEndCapture(P.s_main, &graph));
        SFB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
        SFB_CUDA(cudaGraphLaunch(exec, P.s_main));
        SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
    } else {
        SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
        enqueue();
        SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    }
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    float ms = 0.f;
    SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
    if (report) {
        const double own = double(P.n0) * double(P.N[1]) * double(P.N[2]);
        const long long fpp = tti ? 57LL * P.K + 29
                                  : 3LL * P.K * P.ndim + 3LL * P.ndim + 11 + (ro.imaging ? 7 : 0);
        report->seconds = ms * 1e-3;
        report->steps = long(t_to - t_from);
        report->flops = (long long)(double(fpp) * own * double(report->steps));
        report->gflops = ms > 0 ? double(report->flops) / (ms * 1e-3) / 1e9 : 0.0;
        report->gpts_per_s = ms > 0 ? own * double(report->steps) / (ms * 1e-3) / 1e9 : 0.0;
        report->kernel_launches = P.launches - before;
    }
}

}  // namespace sfb
