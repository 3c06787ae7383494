// engine_tti.cu -- host side of the TTI forward operator (kernels: tti_kernels.cuh): tensor
// maps, per-launch d0 chunking, the two launches of a step per plane group, the whole-run loop.
#include "engine.hpp"

namespace sfb {

// ---- TTI forward ---------------------------------------------------------------------------

void tti_coef(const Plan& P, TtiCoef& k) {
    double ih[3], ih2[3], c0 = 0.0;
    for (int d = 0; d < 3; ++d) {
        ih[d] = P.act[d] ? 1.0 / P.h[d] : 0.0;
        ih2[d] = ih[d] * ih[d];
        c0 += P.w2[0] * ih2[d];
    }
    k.c0 = float(c0);
    for (int j = 1; j <= P.K; ++j) {
        k.lz[j - 1] = float(P.w2[j] * ih2[0]);
        k.ly[j - 1] = float(P.w2[j] * ih2[1]);
        k.lx[j - 1] = float(P.w2[j] * ih2[2]);
        k.fz[j - 1] = float(P.w1[j] * ih[0]);
        k.fy[j - 1] = float(P.w1[j] * ih[1]);
        k.fx[j - 1] = float(P.w1[j] * ih[2]);
    }
    k.qscale = P.coef.qscale;
}

// tensor maps of every TTI field for the (fixed) TTI tile shape
void tti_make_maps(Plan& P) {
    const TtiVariant& v = *P.tti_variant;
    void* wf[Plan::TF_COUNT] = {P.u[0].p, P.u[1].p, P.t_r[0].p, P.t_r[1].p,
                                P.t_a.p,  P.t_b.p,  P.t_c.p};
    for (int i = 0; i < Plan::TF_COUNT; ++i) {
        encode_map(&P.tt_halo[i], wf[i], P.N[2], P.N[1], P.n0 + 2 * P.K, P.pitch, P.plane, v.box_w,
                   v.box_h);
        encode_map(&P.tt_plain[i], wf[i], P.N[2], P.N[1], P.n0 + 2 * P.K, P.pitch, P.plane,
                   v.tile_x, v.tile_y);
    }
    const long long n0g = P.n0 + 2 * P.K;
    for (int f = 0; f < 2; ++f) {
        encode_map(&P.tt_g[f], P.t_g[f].p, P.N[2], P.N[1], n0g, P.pitch, P.plane, v.tile_x,
                   v.tile_y);
        encode_map(&P.tt_bg[f], P.t_bg[f].p, P.N[2], P.N[1], n0g, P.pitch, P.plane, v.tile_x,
                   v.box_h);
        encode_map(&P.tt_gx[f], P.t_g[f].p, P.N[2], P.N[1], n0g, P.pitch, P.plane, v.box_w,
                   v.tile_y);
    }
    encode_map(&P.tt_cx, P.t_c.p, P.N[2], P.N[1], n0g, P.pitch, P.plane, v.box_w, v.tile_y);
    void* cf[Plan::TC_COUNT] = {P.r.p, P.t_e1.p, P.t_e2.p, P.t_lp.p, P.sep ? P.r.p : P.damp.p};
    for (int i = 0; i < Plan::TC_COUNT; ++i)
        encode_map(&P.tt_c[i], cf[i], P.N[2], P.N[1], P.n0, P.pitch, P.plane, v.tile_x, v.tile_y);
}

// d0 chunk length of one TTI launch: the grid should be a whole number of waves of the
// kernel's resident blocks; every chunk re-reads 2K planes to fill its register queues,
// charged at half a plane
int tti_chunk_for(Plan& P, const void* func, int nthreads, size_t smem) {
    const TtiVariant& v = *P.tti_variant;
    const long long tiles = ((P.N[2] + v.tile_x - 1) / v.tile_x) * ((P.N[1] + v.tile_y - 1) / v.tile_y);
    int bps = 1;
    SFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, func, nthreads, smem));
    const long long slots = (long long)P.sm_count * std::max(1, bps);
    int nch = 1;
    double best = -1;
    const int max_nch = std::max(1, P.n0 / std::max(1, 4 * P.K));
    for (int c = 1; c <= max_nch; ++c) {
        const int ch = (P.n0 + c - 1) / c;
        const long long total = tiles * ((P.n0 + ch - 1) / ch);
        const long long waves = (total + slots - 1) / slots;
        const double fill = double(total) / double(waves * slots);
        const double score = fill / (1.0 + (2.0 * P.K / ch) * 0.5);
        if (score > best + 1e-9) {
            best = score;
            nch = c;
        }
        if (total > 16 * slots) break;
    }
    return (P.n0 + nch - 1) / nch;
}

// run_wave for the TTI pair: zero p, r, the products between the passes and the traces
void tti_begin(Plan& P) {
    require(P.tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
    step_begin(P, SFB_OP_TTI_FORWARD, 0);
    for (int b = 0; b < 2; ++b)
        SFB_CUDA(cudaMemsetAsync(P.t_r[b].p, 0, size_t(P.ucount) * 4, P.s_main));
    for (DevBuf* d : {&P.t_g[0], &P.t_g[1], &P.t_bg[0], &P.t_bg[1]})
        SFB_CUDA(cudaMemsetAsync(d->p, 0, size_t(P.ucount) * 4, P.s_main));
    const TtiVariant& v = *P.tti_variant;
    const int sepi = P.sep ? 1 : 0;
    P.tti_chunk[0] = tti_chunk_for(P, v.f_rot, v.threads, v.smem_rot);
    P.tti_chunk[1] = tti_chunk_for(P, v.f_div[sepi], v.threads, v.smem_div[sepi]);
}

dim3 tti_grid(const Plan& P, int lo, int hi, int chunk) {
    const TtiVariant& v = *P.tti_variant;
    return dim3(unsigned((P.N[2] + v.tile_x - 1) / v.tile_x),
                unsigned((P.N[1] + v.tile_y - 1) / v.tile_y), unsigned((hi - lo + chunk - 1) / chunk));
}

// d0 chunk of a single-launch slab pass: at least two chunks (the first sweeps up, the last
// down), whole waves of the one resident block per SM
int tti_fused_chunk(const Plan& P) {
    const TtiVariant& v = *P.tti_variant;
    const long long tiles = ((P.N[2] + v.tile_x - 1) / v.tile_x) * ((P.N[1] + v.tile_y - 1) / v.tile_y);
    const long long slots = P.sm_count;
    int best = 2;
    double best_score = -1;
    const int max_nch = std::max(2, P.n0 / std::max(1, 2 * P.K));
    for (int c = 2; c <= max_nch; ++c) {
        const int ch = (P.n0 + c - 1) / c;
        if (ch < P.K) break;
        const int real = (P.n0 + ch - 1) / ch;
        if (real < 2) continue;
        const long long total = tiles * real;
        const long long waves = (total + slots - 1) / slots;
        const double score = double(total) / double(waves * slots) / (1.0 + (2.0 * P.K / ch) * 0.5);
        if (score > best_score + 1e-9) {
            best_score = score;
            best = real;
        }
        if (total > 16 * slots) break;
    }
    return (P.n0 + best - 1) / best;
}

int tti_part_chunk(const Plan& P, int which, int part, int lo, int hi) {
    if (part == kPartSlabFused) return tti_fused_chunk(P);
    return (part == SFB_PART_ALL || part == SFB_PART_INTERIOR) ? std::min(P.tti_chunk[which], hi - lo)
                                                               : (hi - lo);
}

static void tti_part_bounds(const Plan& P, int part, int& lo, int& hi) {
    if (part == kPartSlabFused) {
        require(P.n0 >= 2 * P.K, SFB_ERR_PARAMETER, "slab thinner than two halo widths");
        lo = 0;
        hi = P.n0;
    } else {
        part_range(P, part, lo, hi);
    }
}

// pass 1 on the planes of `part`: the products a g, b g, c g of p and r (level t)
void tti_rot(Plan& P, long long t, int part) {
    require(t >= 1 && t <= P.desc.nt - 2, SFB_ERR_PARAMETER, "time index outside [1, nt-1)");
    int lo, hi;
    tti_part_bounds(P, part, lo, hi);
    if (hi <= lo) return;
    const bool fused = part == kPartSlabFused;
    const TtiVariant& v = *P.tti_variant;
    const int cur = int(t & 1);
    RotParams rp{};
    tti_coef(P, rp.k);
    rp.N1 = int(P.N[1]);
    rp.N2 = int(P.N[2]);
    rp.pitch = P.pitch;
    rp.plane = P.plane;
    rp.z_lo = lo;
    rp.z_hi = hi;
    rp.chunk = tti_part_chunk(P, 0, part, lo, hi);
    for (int f = 0; f < 2; ++f) {
        rp.g[f] = P.t_g[f].as<float>();
        rp.bg[f] = P.t_bg[f].as<float>();
    }
    rp.lp = P.t_lp.as<float>();
    rp.out_off = (long long)P.K * P.plane;
    RotMaps m1;
    m1.f0_feed = P.tt_plain[Plan::TF_P0 + cur];
    m1.f1_feed = P.tt_plain[Plan::TF_R0 + cur];
    m1.f0_ctr = P.tt_halo[Plan::TF_P0 + cur];
    m1.f1_ctr = P.tt_halo[Plan::TF_R0 + cur];
    m1.a = P.tt_plain[Plan::TF_A];
    m1.b = P.tt_plain[Plan::TF_B];
    m1.c = P.tt_plain[Plan::TF_C];
    cudaStream_t st = part_stream(P, part);
    if (fused) {
        // mirrors of the boundary planes of g in the neighbours' ghost planes: owned plane z of
        // g[f] sits at g[f] + (z + K) planes; low group -> peer_g_lo + z planes, high group ->
        // peer_g_hi + (z - (n0 - K)) planes
        for (int f = 0; f < 2; ++f) {
            float* g = P.t_g[f].as<float>();
            rp.peer_lo[f] = P.peer_g_lo[f] ? P.peer_g_lo[f] - (g + (long long)P.K * P.plane) : 0;
            rp.peer_hi[f] = P.peer_g_hi[f] ? P.peer_g_hi[f] - (g + (long long)P.n0 * P.plane) : 0;
        }
        rp.push_planes = P.K;
        rp.desc_last = 1;
        SFB_CUDA(v.rot_push(m1, rp, tti_grid(P, lo, hi, rp.chunk), st));
    } else {
        SFB_CUDA(v.rot(m1, rp, tti_grid(P, lo, hi, rp.chunk), st));
    }
    ++P.launches;
    mark_stream(P, part);
}

// pass 2 and the update on the planes of `part`, then the point work of the part: Hz(p),
// Hz(r) from the products (ghost planes of a g included), L(p), both leapfrog updates in
// place over level t-1, injection into p and r, sampling of p
void tti_update(Plan& P, long long t, int part, bool with_points) {
    require(t >= 1 && t <= P.desc.nt - 2, SFB_ERR_PARAMETER, "time index outside [1, nt-1)");
    int lo, hi;
    tti_part_bounds(P, part, lo, hi);
    const bool fused = part == kPartSlabFused;
    const TtiVariant& v = *P.tti_variant;
    const int cur = int(t & 1), oth = cur ^ 1;
    const int sepi = P.sep ? 1 : 0;
    cudaStream_t st = part_stream(P, part);
    if (hi > lo) {
        DivParams dp{};
        tti_coef(P, dp.k);
        dp.dz = P.dz.as<float>();
        dp.dy = P.dy.as<float>();
        dp.dx = P.dx.as<float>();
        dp.N1 = int(P.N[1]);
        dp.N2 = int(P.N[2]);
        dp.pitch = P.pitch;
        dp.plane = P.plane;
        dp.z_lo = lo;
        dp.z_hi = hi;
        dp.chunk = tti_part_chunk(P, 1, part, lo, hi);
        dp.po = P.u[oth].as<float>();
        dp.ro = P.t_r[oth].as<float>();
        DivMaps m2;
        m2.g0 = P.tt_g[0];
        m2.g1 = P.tt_g[1];
        m2.a = P.tt_plain[Plan::TF_A];
        m2.bg0 = P.tt_bg[0];
        m2.bg1 = P.tt_bg[1];
        m2.g0x = P.tt_gx[0];
        m2.g1x = P.tt_gx[1];
        m2.cx = P.tt_cx;
        m2.lp = P.tt_c[Plan::TC_LP];
        m2.po = P.tt_plain[Plan::TF_P0 + oth];
        m2.ro = P.tt_plain[Plan::TF_R0 + oth];
        m2.pc = P.tt_plain[Plan::TF_P0 + cur];
        m2.rc = P.tt_plain[Plan::TF_R0 + cur];
        m2.rm = P.tt_c[Plan::TC_RM];
        m2.e1 = P.tt_c[Plan::TC_E1];
        m2.e2 = P.tt_c[Plan::TC_E2];
        m2.d = P.tt_c[Plan::TC_DAMP];
        if (fused) {
            float* bufs[2] = {dp.po, dp.ro};
            float* plo[2] = {P.peer_lo[oth], P.peer_r_lo[oth]};
            float* phi[2] = {P.peer_hi[oth], P.peer_r_hi[oth]};
            for (int f = 0; f < 2; ++f) {
                dp.peer_lo[f] = plo[f] ? plo[f] - (bufs[f] + (long long)P.K * P.plane) : 0;
                dp.peer_hi[f] = phi[f] ? phi[f] - (bufs[f] + (long long)P.n0 * P.plane) : 0;
            }
            dp.push_planes = P.K;
            dp.desc_last = 1;
            SFB_CUDA(v.div_push[sepi](m2, dp, tti_grid(P, lo, hi, dp.chunk), st));
        } else {
            SFB_CUDA(v.div[sepi](m2, dp, tti_grid(P, lo, hi, dp.chunk), st));
        }
        ++P.launches;
        mark_stream(P, part);
    }
    if (with_points && part != SFB_PART_LOW) {
        // HIGH (called after LOW) carries the point work of both boundary plane groups, so
        // the injections land after both groups have been overwritten by the update
        const int op = SFB_OP_TTI_FORWARD;
        const int pp = part == SFB_PART_HIGH ? SFB_PART_LOW : part;
        step_points(P, op, t, pp);                                    // p: scatter + gather
        step_points(P, op, t, pp, P.t_r[oth].as<float>(), false, nullptr,   // r: scatter
                    P.peer_r_lo[oth], P.peer_r_hi[oth]);
    }
    if (part == SFB_PART_ALL || part == SFB_PART_INTERIOR || fused) {
        P.live_level[cur] = t;
        P.live_level[oth] = t + 1;
    }
}

void run_tti(Plan& P, sfb_report* rep, double* stream_out) {
    require(P.n0 == P.N[0], SFB_ERR_CAPABILITY,
            "sfb_tti_forward runs one whole domain; slabs step with sfb_tti_step_*");
    tti_begin(P);
    const long long nt = P.desc.nt;
    std::unique_ptr<RowStreamer> rs;
    if (stream_out) rs.reset(new RowStreamer(P, P.cloud[SFB_CLOUD_REC], stream_out));
    SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
    for (long long t = 1; t < nt - 1; ++t) {
        tti_rot(P, t, SFB_PART_ALL);
        tti_update(P, t, SFB_PART_ALL);
        if (rs) rs->row_done(t);
    }
    SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    float ms = 0.f;
    SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
    finite_guard(P, "tti_forward");
    if (rs) rs->finish();
    if (rep) {
        const long steps = long(std::max<long long>(0, nt - 2));
        const double own = double(P.n0) * double(P.N[1]) * double(P.N[2]);
        // adds + multiplies per node, counted as the reference counts its operators
        // (proj/src/passes.cpp:318-327), D = 3: g(p), g(r): 2 (9K + 2); Hz(p), Hz(r):
        // 2 (15K - 1); L(p): 9K + 3; right-hand sides and the two leapfrog updates: 24
        const long long fpp = 57LL * P.K + 29;
        rep->seconds = ms * 1e-3;
        rep->steps = steps;
        rep->flops = (long long)(double(fpp) * own * steps);
        rep->gflops = ms > 0 ? double(rep->flops) / (ms * 1e-3) / 1e9 : 0.0;
        rep->gpts_per_s = ms > 0 ? own * steps / (ms * 1e-3) / 1e9 : 0.0;
        rep->kernel_launches = P.launches;
    }
}

}  // namespace sfb
