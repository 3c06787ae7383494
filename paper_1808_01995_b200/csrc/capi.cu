// capi.cu -- the extern "C" boundary of libsfb200.so (declared in include/sfb200.h).  The
// host logic behind it lives in engine_setup.cu, engine_step.cu and engine_tti.cu.
#include "engine.hpp"
#include "point_kernels.cuh"
#include "tti_kernels.cuh"

namespace sfb {

thread_local std::string g_create_err;

std::vector<StepVariant>& step_variant_registry() {
    static std::vector<StepVariant> reg;
    return reg;
}

std::vector<TtiVariant>& tti_variant_registry() {
    static std::vector<TtiVariant> reg;
    return reg;
}

}  // namespace sfb

using namespace sfb;

namespace {

// stream memory operations of the driver API (no link-time libcuda dependency)
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValueFn stream_value_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
        throw Failure(SFB_ERR_CAPABILITY, std::string("driver lacks ") + name);
    return reinterpret_cast<StreamValueFn>(p);
}

struct PeerBlob {   // what sfb_peer_export writes into the caller's SFB_PEER_BLOB_BYTES
    cudaIpcMemHandle_t u[2];
    cudaIpcMemHandle_t flag;
    int64_t z_lo, z_hi, n1, n2, pitch, plane, K;
    // TTI pair (has_tti != 0): g(p), g(r) and the two levels of r
    int64_t has_tti;
    cudaIpcMemHandle_t g[2];
    cudaIpcMemHandle_t r[2];
};
static_assert(sizeof(PeerBlob) <= SFB_PEER_BLOB_BYTES, "peer blob");

// test aid (sfb_debug_stall): occupy a stream for a given time
__global__ void stall_kernel(unsigned long long ns) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    } while (t1 - t0 < ns);
}

void close_ipc(Plan& P) {
    for (int side = 0; side < 2; ++side) {
        for (int b = 0; b < 2; ++b)
            if (P.ipc_u[side][b]) cudaIpcCloseMemHandle(P.ipc_u[side][b]);
        if (P.ipc_flag[side]) cudaIpcCloseMemHandle(P.ipc_flag[side]);
        for (int b = 0; b < 2; ++b) {
            if (P.ipc_g[side][b]) cudaIpcCloseMemHandle(P.ipc_g[side][b]);
            if (P.ipc_r[side][b]) cudaIpcCloseMemHandle(P.ipc_r[side][b]);
            P.ipc_g[side][b] = P.ipc_r[side][b] = nullptr;
        }
        P.ipc_u[side][0] = P.ipc_u[side][1] = P.ipc_flag[side] = nullptr;
    }
}

}  // namespace


extern "C" {

SFB_API int sfb_abi_version(void) { return SFB_ABI_VERSION; }

SFB_API const char* sfb_last_error(const sfb_plan* plan) {
    return plan ? plan->err.c_str() : g_create_err.c_str();
}

SFB_API int sfb_device_count(int* count) {
    if (!count) return SFB_ERR_PARAMETER;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *count = n;
    return SFB_OK;
}

SFB_API int sfb_fd_weights(int deriv_order, int space_order, double* out) {
    std::vector<Frac> w;
    if (!out || !centred_weights(deriv_order, space_order, w)) {
        g_create_err = "centered stencils require an even accuracy order in [2, 16]";
        return SFB_ERR_ORDER;
    }
    for (size_t j = 0; j < w.size(); ++j) out[j] = to_double(w[j]);
    return SFB_OK;
}

SFB_API int sfb_critical_dt(int ndim, const double* spacing, double v_max, int space_order,
                    double* out) {
    // SeismicModel::critical_dt, proj/src/model.cpp:103-111 (gamma = 1)
    std::vector<Frac> w;
    if (!out || !spacing || ndim < 1 || ndim > 3 || !(v_max > 0.0) ||
        !centred_weights(2, space_order, w)) {
        g_create_err = "critical_dt: bad arguments";
        return SFB_ERR_PARAMETER;
    }
    double wsum = std::abs(to_double(w[0]));
    for (size_t j = 1; j < w.size(); ++j) wsum += 2.0 * std::abs(to_double(w[j]));
    double h_min = spacing[0];
    for (int a = 1; a < ndim; ++a) h_min = std::min(h_min, spacing[a]);
    const double m_min = 1.0 / (v_max * v_max);
    *out = h_min * std::sqrt(m_min) / std::sqrt(double(ndim) * wsum / 2.0);
    return SFB_OK;
}

SFB_API int sfb_locate(const sfb_plan_desc* desc, const double* origin, int64_t np,
               const double* coords, int64_t* base, double* w) {
    // SparseFunction::locate, proj/src/sparse.cpp:36-70
    if (!desc || !origin || !coords || !base || !w || desc->ndim < 1 || desc->ndim > 3) {
        g_create_err = "locate: bad arguments";
        return SFB_ERR_PARAMETER;
    }
    const int nd = desc->ndim, nc = 1 << nd;
    for (int64_t p = 0; p < np; ++p) {
        double frac[3];
        for (int d = 0; d < nd; ++d) {
            double rel = (coords[p * nd + d] - origin[d]) / desc->spacing[d];
            const double last = double(desc->shape[d] - 1);
            const double tol = 1e-9 * std::max(1.0, last);
            if (rel < -tol || rel > last + tol) {
                char buf[160];
                std::snprintf(buf, sizeof buf, "point %ld axis %d: coordinate %g outside domain",
                              long(p), d, coords[p * nd + d]);
                g_create_err = buf;
                return SFB_ERR_LOCATION;
            }
            rel = std::min(std::max(rel, 0.0), last);
            int64_t b = int64_t(std::floor(rel));
            if (b > desc->shape[d] - 2) b = desc->shape[d] - 2;
            base[p * nd + d] = b;
            frac[d] = rel - double(b);
        }
        for (int c = 0; c < nc; ++c) {
            double ww = 1.0;
            for (int d = 0; d < nd; ++d) ww *= ((c >> d) & 1) ? frac[d] : 1.0 - frac[d];
            w[p * nc + c] = ww;
        }
    }
    return SFB_OK;
}

SFB_API int sfb_plan_create(const sfb_plan_desc* desc, sfb_plan** out) {
    if (out) *out = nullptr;
    sfb_plan* plan = nullptr;
    int rc = guarded(nullptr, [&] {
        require(desc && out, SFB_ERR_PARAMETER, "plan_create: null argument");
        require(desc->ndim >= 1 && desc->ndim <= 3, SFB_ERR_PARAMETER,
                "grid rank must be 1, 2 or 3");
        for (int a = 0; a < desc->ndim; ++a) {
            require(desc->shape[a] >= 2, SFB_ERR_PARAMETER, "grid extent must be >= 2 nodes");
            require(desc->spacing[a] > 0.0, SFB_ERR_PARAMETER, "grid spacing must be positive");
            require(desc->shape[a] < (1LL << 30), SFB_ERR_PARAMETER, "grid extent too large");
        }
        if (desc->space_order < 2 || desc->space_order % 2 != 0)
            throw Failure(SFB_ERR_ORDER, "space order must be a positive even number");
        if (desc->space_order > 2 * kMaxK)
            throw Failure(SFB_ERR_ORDER, "space orders above 16 are not built");
        require(desc->dt > 0.0 && desc->nt >= 1, SFB_ERR_PARAMETER, "bad time axis");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw Failure(SFB_ERR_CAPABILITY,
                          "no CUDA device: this engine has no CPU fallback");
        }
        require(desc->device >= 0 && desc->device < ndev, SFB_ERR_PARAMETER,
                "device ordinal out of range");
        cudaDeviceProp prop;
        SFB_CUDA(cudaGetDeviceProperties(&prop, desc->device));
        if (prop.major != 10)
            throw Failure(SFB_ERR_CAPABILITY,
                          std::string("device ") + prop.name +
                              " is not sm_100: kernels are built for sm_100a only");
        SFB_CUDA(cudaSetDevice(desc->device));

        plan = new sfb_plan_s();
        Plan& P = *plan;
        P.desc = *desc;
        P.device = desc->device;
        P.sm_count = prop.multiProcessorCount;
        P.ndim = desc->ndim;
        P.K = desc->space_order / 2;
        const int off = 3 - P.ndim;
        for (int a = 0; a < P.ndim; ++a) {
            P.N[off + a] = desc->shape[a];
            P.h[off + a] = desc->spacing[a];
            P.act[off + a] = true;
        }
        P.z_lo = desc->slab_lo;
        P.z_hi = desc->slab_hi;
        if (P.z_lo == 0 && P.z_hi == 0) P.z_hi = P.N[0];
        require(P.z_lo >= 0 && P.z_lo < P.z_hi && P.z_hi <= P.N[0], SFB_ERR_PARAMETER,
                "slab range outside the slowest axis");
        P.n0 = int(P.z_hi - P.z_lo);
        if (P.n0 != P.N[0])
            require(P.n0 >= 2 * P.K, SFB_ERR_PARAMETER,
                    "a slab must hold at least space_order planes");
        P.pitch = int(round_up(P.N[2], 32));
        P.plane = (long long)P.N[1] * P.pitch;
        P.ucount = (long long)(P.n0 + 2 * P.K) * P.plane;
        P.ccount = (long long)P.n0 * P.plane;

        std::vector<Frac> w;
        centred_weights(2, desc->space_order, w);
        for (int j = 0; j <= P.K; ++j) P.w2[j] = to_double(w[j]);
        double ih2[3];
        double c0 = 0.0;
        for (int d = 0; d < 3; ++d) {
            ih2[d] = P.act[d] ? 1.0 / (P.h[d] * P.h[d]) : 0.0;
            c0 += P.w2[0] * ih2[d];
        }
        P.coef.c0 = float(c0);
        for (int j = 1; j <= P.K; ++j) {
            P.coef.cz[j - 1] = float(P.w2[j] * ih2[0]);
            P.coef.cy[j - 1] = float(P.w2[j] * ih2[1]);
            P.coef.cx[j - 1] = float(P.w2[j] * ih2[2]);
        }
        P.coef.qscale = float(0.5 / desc->dt);
        P.coef.inv_dt2 = float(1.0 / (desc->dt * desc->dt));

        SFB_CUDA(cudaStreamCreateWithFlags(&P.s_main, cudaStreamNonBlocking));
        int lo_pri = 0, hi_pri = 0;
        SFB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
        SFB_CUDA(cudaStreamCreateWithPriority(&P.s_bnd, cudaStreamNonBlocking, hi_pri));
        SFB_CUDA(cudaEventCreateWithFlags(&P.ev_main, cudaEventDisableTiming));
        SFB_CUDA(cudaEventCreateWithFlags(&P.ev_bnd, cudaEventDisableTiming));
        SFB_CUDA(cudaEventCreateWithFlags(&P.ev_push, cudaEventDisableTiming));
        SFB_CUDA(cudaEventCreateWithFlags(&P.ev_done, cudaEventDisableTiming));
        SFB_CUDA(cudaEventCreateWithFlags(&P.ev_g, cudaEventDisableTiming));
        SFB_CUDA(cudaEventCreate(&P.ev_t0));
        SFB_CUDA(cudaEventCreate(&P.ev_t1));
        P.u[0].alloc(size_t(P.ucount) * 4);
        P.u[1].alloc(size_t(P.ucount) * 4);
        select_variant(P, 0, 0, 0);
        *out = plan;
    });
    if (rc != SFB_OK && plan) {
        std::string keep = g_create_err;
        sfb_plan_destroy(plan);
        g_create_err = keep;
    }
    return rc;
}

SFB_API int sfb_plan_destroy(sfb_plan* plan) {
    if (!plan) return SFB_OK;
    cudaSetDevice(plan->device);
    cudaDeviceSynchronize();
    if (plan->own_streams) {
        if (plan->s_main) cudaStreamDestroy(plan->s_main);
        if (plan->s_bnd) cudaStreamDestroy(plan->s_bnd);
    }
    if (plan->ev_main) cudaEventDestroy(plan->ev_main);
    if (plan->ev_bnd) cudaEventDestroy(plan->ev_bnd);
    if (plan->ev_push) cudaEventDestroy(plan->ev_push);
    if (plan->ev_done) cudaEventDestroy(plan->ev_done);
    if (plan->ev_g) cudaEventDestroy(plan->ev_g);
    close_ipc(*plan);
    if (plan->ev_t0) cudaEventDestroy(plan->ev_t0);
    if (plan->ev_t1) cudaEventDestroy(plan->ev_t1);
    delete plan;
    return SFB_OK;
}

namespace {

// slab_local: the views cover the plan's own planes only (index 0 = global plane slab_lo);
// they are rebased so that the global plane indices used below land inside them
void bind_model(Plan& P, const sfb_field_view* m, const sfb_field_view* damp, double v_max,
                bool slab_local) {
    require(m && damp && m->ptr && damp->ptr, SFB_ERR_PARAMETER, "set_model: null field");
    if (v_max > 0.0) {
        // check_cfl, proj/src/seismic_ops.cpp:15-22
        double crit = 0;
        sfb_critical_dt(P.ndim, P.desc.spacing, v_max, P.desc.space_order, &crit);
        if (P.desc.dt > crit * (1.0 + 1e-12))
            throw Failure(SFB_ERR_STABILITY,
                          "dt " + std::to_string(P.desc.dt) + " exceeds the stable limit " +
                              std::to_string(crit) + " at order " +
                              std::to_string(P.desc.space_order));
    }
    IntView mv = embed_view(P, m->ptr, m->stride), dv = embed_view(P, damp->ptr, damp->stride);
    if (slab_local) {
        mv.ptr -= P.z_lo * mv.s[0];
        dv.ptr -= P.z_lo * dv.s[0];
    }
    P.v_max = v_max;
    const long long rows = (long long)P.n0 * P.N[1];
    DevBuf tmp;
    P.r.alloc(size_t(P.ccount) * 4);
    P.damp.alloc(size_t(P.ccount) * 4);
    upload_f64(P, mv, tmp);
    convert_r_kernel<<<row_grid(P, rows), 256, 0, P.s_main>>>(
        tmp.as<double>(), P.r.as<float>(), rows, int(P.N[2]), P.pitch, P.desc.dt * P.desc.dt);
    SFB_CUDA(cudaGetLastError());
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    upload_f64(P, dv, tmp);
    convert_f64_f32_pitched<<<row_grid(P, rows), 256, 0, P.s_main>>>(
        tmp.as<double>(), P.damp.as<float>(), rows, int(P.N[2]), P.pitch);
    SFB_CUDA(cudaGetLastError());
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    // reference plane of the profile extraction: the global centre plane when the whole
    // field is visible (every slab of a decomposed run then derives bit-identical profiles),
    // the slab's own centre plane otherwise
    detect_separable_damping(P, dv, tmp, slab_local ? P.z_lo + P.n0 / 2 : P.N[0] / 2);
    if (P.sep) P.damp.release();
    select_variant(P, P.variant->TXV, P.variant->TY, P.variant->NST, variant_kind(*P.variant));
    P.model_set = true;
    P.history_valid = false;
}

}  // namespace

SFB_API int sfb_set_model(sfb_plan* plan, const sfb_field_view* m, const sfb_field_view* damp,
                  double v_max) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] { bind_model(*plan, m, damp, v_max, false); });
}

SFB_API int sfb_set_model_slab(sfb_plan* plan, const sfb_field_view* m_slab,
                               const sfb_field_view* damp_slab, double v_max) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] { bind_model(*plan, m_slab, damp_slab, v_max, true); });
}

SFB_API int sfb_set_model_tti(sfb_plan* plan, const sfb_field_view* epsilon,
                              const sfb_field_view* delta, const sfb_field_view* theta,
                              const sfb_field_view* phi) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(epsilon && delta && theta && phi && epsilon->ptr && delta->ptr && theta->ptr &&
                    phi->ptr, SFB_ERR_PARAMETER, "set_model_tti: null field");
        require(P.model_set, SFB_ERR_BINDING, "bind m and damp first (sfb_set_model)");
        // stability gates of the builder's formulation: eps >= delta everywhere (the
        // pseudo-acoustic system is ill-posed otherwise) and the acoustic CFL rule with
        // v_max sqrt(1 + 2 eps_max), times 0.9 for the twice-applied first derivatives
        const IntView ev = embed_view(P, epsilon->ptr, epsilon->stride);
        const IntView dv = embed_view(P, delta->ptr, delta->stride);
        double eps_max = 0.0;
        bool ordered = true;
        for (long long i = 0; i < P.N[0]; ++i)
            for (long long j = 0; j < P.N[1]; ++j)
                for (long long l = 0; l < P.N[2]; ++l) {
                    const double e = ev.ptr[i * ev.s[0] + j * ev.s[1] + l * ev.s[2]];
                    const double d = dv.ptr[i * dv.s[0] + j * dv.s[1] + l * dv.s[2]];
                    eps_max = std::max(eps_max, e);
                    ordered = ordered && e >= d && (1.0 + 2.0 * d) > 0.0;
                }
        if (!ordered)
            throw Failure(SFB_ERR_STABILITY, "TTI medium needs epsilon >= delta > -1/2 everywhere");
        if (P.v_max > 0.0) {
            double crit = 0;
            sfb_critical_dt(P.ndim, P.desc.spacing, P.v_max, P.desc.space_order, &crit);
            crit *= 0.9 / std::sqrt(1.0 + 2.0 * eps_max);
            if (P.desc.dt > crit * (1.0 + 1e-12))
                throw Failure(SFB_ERR_STABILITY, "dt " + std::to_string(P.desc.dt) +
                                                     " exceeds the TTI stable limit " +
                                                     std::to_string(crit));
        }
        std::vector<Frac> w;
        centred_weights(1, P.desc.space_order, w);
        for (int j = 0; j <= P.K; ++j) P.w1[j] = to_double(w[j]);
        DevBuf te, td, tt, tph;
        upload_f64(P, ev, te);
        upload_f64(P, dv, td);
        upload_f64(P, embed_view(P, theta->ptr, theta->stride), tt);
        upload_f64(P, embed_view(P, phi->ptr, phi->stride), tph);
        for (int b = 0; b < 2; ++b) P.t_r[b].alloc(size_t(P.ucount) * 4);
        for (DevBuf* d : {&P.t_a, &P.t_b, &P.t_c, &P.t_g[0], &P.t_g[1], &P.t_bg[0], &P.t_bg[1]})
            d->alloc(size_t(P.ucount) * 4);
        for (DevBuf* d : {&P.t_e1, &P.t_e2, &P.t_lp}) d->alloc(size_t(P.ccount) * 4);
        P.tti_variant = nullptr;
        for (const TtiVariant& tv : tti_variant_registry())
            if (tv.K == P.K) P.tti_variant = &tv;
        require(P.tti_variant != nullptr, SFB_ERR_CAPABILITY, "no TTI kernel image for this order");
        SFB_CUDA(cudaFuncSetAttribute(P.tti_variant->f_rot,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(P.tti_variant->smem_rot)));
        SFB_CUDA(cudaFuncSetAttribute(P.tti_variant->f_rot_push,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(P.tti_variant->smem_rot)));
        for (int i = 0; i < 2; ++i) {
            SFB_CUDA(cudaFuncSetAttribute(P.tti_variant->f_div[i],
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(P.tti_variant->smem_div[i])));
            SFB_CUDA(cudaFuncSetAttribute(P.tti_variant->f_div_push[i],
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(P.tti_variant->smem_div[i])));
        }
        tti_make_maps(P);
        const long long rows = (long long)P.n0 * P.N[1];
        tti_setup_kernel<<<row_grid(P, rows), 256, 0, P.s_main>>>(
            te.as<double>(), td.as<double>(), tt.as<double>(), tph.as<double>(), P.t_a.as<float>(),
            P.t_b.as<float>(), P.t_c.as<float>(), P.t_e1.as<float>(), P.t_e2.as<float>(), rows,
            int(P.N[2]), P.pitch, (long long)P.K * P.plane);
        SFB_CUDA(cudaGetLastError());
        // a slab's second pass forms a g on the ghost planes of g too: the axis component a
        // is static, so its ghost planes are filled here from the caller's global arrays
        for (int side = 0; side < 2; ++side) {
            const long long g0 = side == 0 ? std::max<long long>(0, P.z_lo - P.K) : P.z_hi;
            const long long g1 = side == 0 ? P.z_lo : std::min<long long>(P.N[0], P.z_hi + P.K);
            if (g1 <= g0) continue;
            DevBuf gt, gp;
            upload_f64_planes(P, embed_view(P, theta->ptr, theta->stride), gt, g0, g1 - g0);
            upload_f64_planes(P, embed_view(P, phi->ptr, phi->stride), gp, g0, g1 - g0);
            const long long grow = (g1 - g0) * P.N[1];
            tti_axis_a_kernel<<<row_grid(P, grow), 256, 0, P.s_main>>>(
                gt.as<double>(), gp.as<double>(), P.t_a.as<float>(), grow, int(P.N[2]), P.pitch,
                (g0 - P.z_lo + P.K) * P.plane);
            SFB_CUDA(cudaGetLastError());
            SFB_CUDA(cudaStreamSynchronize(P.s_main));
        }
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
        P.tti_set = true;
    });
}

SFB_API int sfb_set_points(sfb_plan* plan, int cloud, int64_t np, const int64_t* base,
                   const double* w) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(cloud == SFB_CLOUD_SRC || cloud == SFB_CLOUD_REC, SFB_ERR_PARAMETER,
                "unknown cloud id");
        require(np >= 1 && base && w, SFB_ERR_PARAMETER, "set_points: empty point table");
        require(np < (1LL << 31), SFB_ERR_PARAMETER, "too many points");
        Cloud& c = P.cloud[cloud];
        c.np = np;
        c.base.assign(base, base + np * P.ndim);
        c.w.assign(w, w + np * (1 << P.ndim));
        build_cloud(P, c);
    });
}

SFB_API int sfb_upload_traces(sfb_plan* plan, int cloud, const double* traces) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        require(cloud == 0 || cloud == 1, SFB_ERR_PARAMETER, "unknown cloud id");
        require(plan->cloud[cloud].set && traces, SFB_ERR_BINDING, "point cloud is not bound");
        upload_traces(*plan, plan->cloud[cloud], traces);
    });
}

SFB_API int sfb_download_traces(sfb_plan* plan, int cloud, double* traces) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        require(cloud == 0 || cloud == 1, SFB_ERR_PARAMETER, "unknown cloud id");
        require(plan->cloud[cloud].set && traces, SFB_ERR_BINDING, "point cloud is not bound");
        download_traces(*plan, plan->cloud[cloud], traces);
    });
}

SFB_API int sfb_run_resident(sfb_plan* plan, int op, int64_t save_every, sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        if (op == SFB_OP_TTI_FORWARD)
            run_tti(*plan, report, nullptr);
        else
            run_op(*plan, op, save_every, report);
    });
}


SFB_API int sfb_run_steps(sfb_plan* plan, int op, int64_t t_from, int64_t t_to, sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] { run_window(*plan, op, t_from, t_to, true, report); });
}

SFB_API int sfb_time_stencil(sfb_plan* plan, int op, int64_t t_from, int64_t t_to,
                             sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] { run_window(*plan, op, t_from, t_to, false, report); });
}

SFB_API int sfb_forward(sfb_plan* plan, const double* src, double* rec, int64_t save_every,
                sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(src && rec, SFB_ERR_PARAMETER, "forward: null trace table");
        require(P.cloud[0].set && P.cloud[1].set, SFB_ERR_BINDING, "point clouds are not bound");
        upload_traces(P, P.cloud[SFB_CLOUD_SRC], src);
        run_op(P, SFB_OP_FORWARD, save_every, report, rec);
    });
}

SFB_API int sfb_forward_checkpointed(sfb_plan* plan, const double* src, double* rec,
                                     int64_t checkpoint_every, sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(src && rec, SFB_ERR_PARAMETER, "forward: null trace table");
        require(P.cloud[0].set && P.cloud[1].set, SFB_ERR_BINDING, "point clouds are not bound");
        upload_traces(P, P.cloud[SFB_CLOUD_SRC], src);
        forward_checkpointed(P, checkpoint_every, report, rec);
    });
}

SFB_API int sfb_adjoint(sfb_plan* plan, const double* rec, double* srca, sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(rec && srca, SFB_ERR_PARAMETER, "adjoint: null trace table");
        require(P.cloud[0].set && P.cloud[1].set, SFB_ERR_BINDING, "point clouds are not bound");
        // the receiver table is fed to the device row by row while the sweep runs
        run_op(P, SFB_OP_ADJOINT, 0, report, srca, rec);
    });
}

SFB_API int sfb_gradient(sfb_plan* plan, const double* resid, const sfb_field_mview* grad,
                 sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(resid && grad && grad->ptr, SFB_ERR_PARAMETER, "gradient: null argument");
        require(P.cloud[1].set, SFB_ERR_BINDING, "receiver cloud is not bound");
        require((P.history_valid && P.save_every > 0) || P.ckpt_valid, SFB_ERR_PARAMETER,
                "gradient_operator: saved forward history required");
        if (P.ckpt_valid && !P.history_valid) {
            upload_traces(P, P.cloud[SFB_CLOUD_REC], resid);
            gradient_checkpointed(P, report);
        } else {
            run_op(P, SFB_OP_GRADIENT, P.save_every, report, nullptr, resid);
        }
        download_field(P, P.grad.as<float>(), grad);
    });
}

SFB_API int sfb_tti_forward(sfb_plan* plan, const double* src, double* rec, sfb_report* report) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(src && rec, SFB_ERR_PARAMETER, "tti_forward: null trace table");
        require(P.cloud[0].set && P.cloud[1].set, SFB_ERR_BINDING, "point clouds are not bound");
        upload_traces(P, P.cloud[SFB_CLOUD_SRC], src);
        run_tti(P, report, rec);
    });
}

SFB_API int sfb_get_wavefield(sfb_plan* plan, int field, int64_t level, const sfb_field_mview* out) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(out && out->ptr && (field == 0 || (field == 1 && P.tti_set)), SFB_ERR_PARAMETER,
                "get_wavefield: bad argument");
        for (int b = 0; b < 2; ++b)
            if (P.live_level[b] == level) {
                const DevBuf& buf = field == 1 ? P.t_r[b] : P.u[b];
                download_field(P, buf.as<float>() + (long long)P.K * P.plane, out);
                return;
            }
        if (P.history_valid && P.save_every > 0 && level >= 0 && level % P.save_every == 0 &&
            level / P.save_every < P.nslots) {
            download_field(P, P.snaps.as<float>() + (level / P.save_every) * P.ccount, out);
            return;
        }
        throw Failure(SFB_ERR_PARAMETER, "time level " + std::to_string(level) +
                                             " is neither live nor saved");
    });
}

SFB_API int sfb_put_history(sfb_plan* plan, int64_t save_every, int64_t level,
                            const sfb_field_view* u) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(u && u->ptr && save_every >= 1, SFB_ERR_PARAMETER, "put_history: bad argument");
        require(level >= 0 && level < P.desc.nt && level % save_every == 0, SFB_ERR_PARAMETER,
                "put_history: level is not a saved level");
        const long long nslots = (P.desc.nt - 1) / save_every + 1;
        if (P.save_every != save_every || P.nslots != nslots || !P.snaps.p) {
            P.save_every = save_every;
            P.nslots = nslots;
            P.snaps.alloc(size_t(nslots) * P.ccount * 4, true);
        }
        DevBuf tmp;
        upload_f64(P, embed_view(P, u->ptr, u->stride), tmp);
        const long long rows = (long long)P.n0 * P.N[1];
        convert_f64_f32_pitched<<<row_grid(P, rows), 256, 0, P.s_main>>>(
            tmp.as<double>(), P.snaps.as<float>() + (level / save_every) * P.ccount, rows,
            int(P.N[2]), P.pitch);
        SFB_CUDA(cudaGetLastError());
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
        P.history_valid = true;
    });
}

SFB_API int sfb_get_gradient(sfb_plan* plan, const sfb_field_mview* out) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        require(out && out->ptr, SFB_ERR_PARAMETER, "get_gradient: null view");
        require(plan->grad.p != nullptr, SFB_ERR_BINDING, "no gradient sweep has run on this plan");
        SFB_CUDA(cudaStreamSynchronize(plan->s_main));
        download_field(*plan, plan->grad.as<float>(), out);
    });
}

SFB_API int sfb_step_begin(sfb_plan* plan, int op, int64_t save_every) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        if (op == SFB_OP_TTI_FORWARD) {
            tti_begin(*plan);
            return;
        }
        if (op == SFB_OP_GRADIENT) save_every = plan->save_every;
        step_begin(*plan, op, save_every);
    });
}

SFB_API int sfb_tti_step_rot(sfb_plan* plan, int64_t t, int part) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        require(plan->tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
        tti_rot(*plan, t, part);
    });
}

SFB_API int sfb_tti_step_update(sfb_plan* plan, int64_t t, int part) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        require(plan->tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
        tti_update(*plan, t, part);
    });
}

SFB_API int sfb_tti_halo_blocks(sfb_plan* plan, int which, int64_t t, void** send_lo,
                                void** send_hi, void** recv_lo, void** recv_hi, int64_t* count) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(P.tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
        float* u = nullptr;
        switch (which) {
        case SFB_TTI_HALO_G_P: u = P.t_g[0].as<float>(); break;
        case SFB_TTI_HALO_G_R: u = P.t_g[1].as<float>(); break;
        case SFB_TTI_HALO_P: u = P.u[(t + 1) & 1].as<float>(); break;
        case SFB_TTI_HALO_R: u = P.t_r[(t + 1) & 1].as<float>(); break;
        default: throw Failure(SFB_ERR_PARAMETER, "unknown TTI halo field");
        }
        const long long blk = (long long)P.K * P.plane;
        if (recv_lo) *recv_lo = u;
        if (send_lo) *send_lo = u + blk;
        if (send_hi) *send_hi = u + (long long)P.n0 * P.plane;
        if (recv_hi) *recv_hi = u + (long long)(P.n0 + P.K) * P.plane;
        if (count) *count = blk;
    });
}

SFB_API int sfb_step_compute(sfb_plan* plan, int op, int64_t t, int part) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] { step_compute(*plan, op, t, part); });
}

SFB_API int sfb_step_points(sfb_plan* plan, int op, int64_t t, int part) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        require(op != SFB_OP_TTI_FORWARD, SFB_ERR_PARAMETER,
                "the TTI operator steps through sfb_tti_step_rot / sfb_tti_step_update");
        step_points(*plan, op, t, part);
    });
}

SFB_API int sfb_step_slab_boundary(sfb_plan* plan, int op, int64_t t) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        if (plan->n0 >= 2 * plan->K) {
            step_compute(*plan, op, t, kPartBoundaryPair);   // both plane groups, one launch
        } else {
            step_compute(*plan, op, t, SFB_PART_LOW);
            step_compute(*plan, op, t, SFB_PART_HIGH);
        }
        step_points(*plan, op, t, SFB_PART_LOW);
        if (plan->peer_lo[0] || plan->peer_hi[0]) {   // linked: the push of this step ends here
            SFB_CUDA(cudaEventRecord(plan->ev_push, plan->s_bnd));
            if (plan->ipc_flag[0] || plan->ipc_flag[1]) {   // neighbours in other processes
                static StreamValueFn write_value = stream_value_fn("cuStreamWriteValue32");
                CUresult rc = write_value(plan->s_bnd,
                                          reinterpret_cast<CUdeviceptr>(plan->push_flag.p),
                                          ++plan->push_count, 0);
                if (rc != CUDA_SUCCESS)
                    throw Failure(SFB_ERR_CUDA, "cuStreamWriteValue32 failed with code " +
                                                    std::to_string(int(rc)));
            }
        }
    });
}

SFB_API int sfb_step_slab_fused(sfb_plan* plan, int op, int64_t t) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        static StreamValueFn write_value = stream_value_fn("cuStreamWriteValue32");
        step_compute(P, op, t, kPartSlabFused);     // pushes both boundary plane groups first
        step_points(P, op, t, kPartSlabFused);      // every injection (mirrored) + the gather
        if (P.peer_lo[0] || P.peer_hi[0]) {
            // one stream: the pushes have landed AND the ghost-plane readers are done
            SFB_CUDA(cudaEventRecord(P.ev_push, P.s_main));
            SFB_CUDA(cudaEventRecord(P.ev_done, P.s_main));
            if (P.ipc_flag[0] || P.ipc_flag[1]) {
                const CUdeviceptr f = reinterpret_cast<CUdeviceptr>(P.push_flag.p);
                CUresult rc = write_value(P.s_main, f, ++P.push_count, 0);
                if (rc == CUDA_SUCCESS) rc = write_value(P.s_main, f + 4, ++P.done_count, 0);
                if (rc != CUDA_SUCCESS)
                    throw Failure(SFB_ERR_CUDA, "cuStreamWriteValue32 failed with code " +
                                                    std::to_string(int(rc)));
            }
        }
    });
}

namespace {
void signal_word(Plan& P, int word, unsigned value) {
    static StreamValueFn write_value = stream_value_fn("cuStreamWriteValue32");
    CUresult rc = write_value(P.s_main, reinterpret_cast<CUdeviceptr>(P.push_flag.p) + 4 * word,
                              value, 0);
    if (rc != CUDA_SUCCESS)
        throw Failure(SFB_ERR_CUDA, "cuStreamWriteValue32 failed with code " + std::to_string(int(rc)));
}
bool tti_linked(const Plan& P) {
    return P.peer_g_lo[0] || P.peer_g_hi[0];
}
}  // namespace

SFB_API int sfb_tti_step_rot_fused(sfb_plan* plan, int64_t t) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(P.tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
        require(!(P.peer_lo[0] || P.peer_hi[0]) || tti_linked(P), SFB_ERR_BINDING,
                "link the plans after sfb_set_model_tti so that the TTI buffers are mapped");
        tti_rot(P, t, kPartSlabFused);   // pushes both boundary plane groups of g first
        if (tti_linked(P)) {
            SFB_CUDA(cudaEventRecord(P.ev_g, P.s_main));
            if (P.ipc_flag[0] || P.ipc_flag[1]) signal_word(P, 2, ++P.g_count);
        }
    });
}

SFB_API int sfb_tti_peer_wait_g(sfb_plan* plan, sfb_plan* neighbour) {
    if (!plan || !neighbour) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        SFB_CUDA(cudaStreamWaitEvent(plan->s_main, neighbour->ev_g, 0));
    });
}

SFB_API int sfb_tti_peer_wait_g_ipc(sfb_plan* plan) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        static StreamValueFn wait_value = stream_value_fn("cuStreamWaitValue32");
        for (int side = 0; side < 2; ++side) {
            if (!P.ipc_flag[side]) continue;
            CUresult rc = wait_value(P.s_main, reinterpret_cast<CUdeviceptr>(P.ipc_flag[side]) + 8,
                                     P.g_count, CU_STREAM_WAIT_VALUE_GEQ);
            if (rc != CUDA_SUCCESS)
                throw Failure(SFB_ERR_CUDA, "cuStreamWaitValue32 failed with code " +
                                                std::to_string(int(rc)));
        }
    });
}

SFB_API int sfb_tti_step_update_fused(sfb_plan* plan, int64_t t) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(P.tti_set, SFB_ERR_BINDING, "TTI fields are not bound (sfb_set_model_tti)");
        tti_update(P, t, kPartSlabFused);   // pushes the new p and r boundary planes first
        if (tti_linked(P)) {
            SFB_CUDA(cudaEventRecord(P.ev_push, P.s_main));
            SFB_CUDA(cudaEventRecord(P.ev_done, P.s_main));
            if (P.ipc_flag[0] || P.ipc_flag[1]) {
                signal_word(P, 0, ++P.push_count);
                signal_word(P, 1, ++P.done_count);
            }
        }
    });
}

SFB_API int sfb_link_peers(sfb_plan* plan, sfb_plan* lo, sfb_plan* hi) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        auto compatible = [&](const Plan& Q) {
            return Q.K == P.K && Q.N[1] == P.N[1] && Q.N[2] == P.N[2] && Q.pitch == P.pitch &&
                   Q.plane == P.plane;
        };
        for (int b = 0; b < 2; ++b)
            P.peer_lo[b] = P.peer_hi[b] = P.peer_g_lo[b] = P.peer_g_hi[b] = P.peer_r_lo[b] =
                P.peer_r_hi[b] = nullptr;
        if ((lo || hi) && !P.variant->launch_push) {
            select_variant(P, 0, 0, 0);   // the default shape of the order carries the push kernel
            require(P.variant->launch_push != nullptr, SFB_ERR_CAPABILITY,
                    "link_peers: no halo-push kernel for this order");
        }
        if (lo) {
            require(compatible(*lo) && lo->z_hi == P.z_lo, SFB_ERR_PARAMETER,
                    "link_peers: the lower plan is not the slab below this one");
            const long long hg = (long long)(lo->n0 + lo->K) * lo->plane;
            for (int b = 0; b < 2; ++b)   // its high ghost planes: buffer planes n0 + K ...
                P.peer_lo[b] = lo->u[b].as<float>() + hg;
            if (P.tti_set && lo->tti_set)
                for (int b = 0; b < 2; ++b) {
                    P.peer_g_lo[b] = lo->t_g[b].as<float>() + hg;
                    P.peer_r_lo[b] = lo->t_r[b].as<float>() + hg;
                }
        }
        if (hi) {
            require(compatible(*hi) && hi->z_lo == P.z_hi, SFB_ERR_PARAMETER,
                    "link_peers: the upper plan is not the slab above this one");
            for (int b = 0; b < 2; ++b) P.peer_hi[b] = hi->u[b].as<float>();   // planes 0 .. K-1
            if (P.tti_set && hi->tti_set)
                for (int b = 0; b < 2; ++b) {
                    P.peer_g_hi[b] = hi->t_g[b].as<float>();
                    P.peer_r_hi[b] = hi->t_r[b].as<float>();
                }
        }
        if ((lo && lo->device != P.device) || (hi && hi->device != P.device)) {
            // one process driving several GPUs: map the neighbours' memory
            for (sfb_plan* q : {lo, hi}) {
                if (!q || q->device == P.device) continue;
                int can = 0;
                SFB_CUDA(cudaDeviceCanAccessPeer(&can, P.device, q->device));
                require(can != 0, SFB_ERR_CAPABILITY, "link_peers: no peer access between the devices");
                cudaError_t e = cudaDeviceEnablePeerAccess(q->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SFB_CUDA(e);
                (void)cudaGetLastError();
            }
        }
    });
}

SFB_API int sfb_peer_export(sfb_plan* plan, void* blob) {
    if (!plan || !blob) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        if (!P.push_flag.p) P.push_flag.alloc(256, true);
        PeerBlob pb{};
        for (int b = 0; b < 2; ++b) SFB_CUDA(cudaIpcGetMemHandle(&pb.u[b], P.u[b].p));
        SFB_CUDA(cudaIpcGetMemHandle(&pb.flag, P.push_flag.p));
        pb.z_lo = P.z_lo;
        pb.z_hi = P.z_hi;
        pb.n1 = P.N[1];
        pb.n2 = P.N[2];
        pb.pitch = P.pitch;
        pb.plane = P.plane;
        pb.K = P.K;
        pb.has_tti = P.tti_set ? 1 : 0;
        if (P.tti_set)
            for (int b = 0; b < 2; ++b) {
                SFB_CUDA(cudaIpcGetMemHandle(&pb.g[b], P.t_g[b].p));
                SFB_CUDA(cudaIpcGetMemHandle(&pb.r[b], P.t_r[b].p));
            }
        std::memset(blob, 0, SFB_PEER_BLOB_BYTES);
        std::memcpy(blob, &pb, sizeof pb);
    });
}

SFB_API int sfb_link_peers_ipc(sfb_plan* plan, const void* lo_blob, const void* hi_blob) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        close_ipc(P);
        for (int b = 0; b < 2; ++b)
            P.peer_lo[b] = P.peer_hi[b] = P.peer_g_lo[b] = P.peer_g_hi[b] = P.peer_r_lo[b] =
                P.peer_r_hi[b] = nullptr;
        if (!lo_blob && !hi_blob) return;
        if (!P.variant->launch_push) {
            select_variant(P, 0, 0, 0);
            require(P.variant->launch_push != nullptr, SFB_ERR_CAPABILITY,
                    "link_peers_ipc: no halo-push kernel for this order");
        }
        if (!P.push_flag.p) P.push_flag.alloc(256, true);
        const void* blobs[2] = {lo_blob, hi_blob};
        for (int side = 0; side < 2; ++side) {
            if (!blobs[side]) continue;
            PeerBlob pb;
            std::memcpy(&pb, blobs[side], sizeof pb);
            require(pb.K == P.K && pb.n1 == P.N[1] && pb.n2 == P.N[2] && pb.pitch == P.pitch &&
                        pb.plane == P.plane &&
                        (side == 0 ? pb.z_hi == P.z_lo : pb.z_lo == P.z_hi),
                    SFB_ERR_PARAMETER, "link_peers_ipc: the blob is not the neighbouring slab");
            for (int b = 0; b < 2; ++b)
                SFB_CUDA(cudaIpcOpenMemHandle(&P.ipc_u[side][b], pb.u[b],
                                              cudaIpcMemLazyEnablePeerAccess));
            SFB_CUDA(cudaIpcOpenMemHandle(&P.ipc_flag[side], pb.flag, cudaIpcMemLazyEnablePeerAccess));
            const long long n0q = pb.z_hi - pb.z_lo;
            const long long hg = (n0q + pb.K) * pb.plane;
            for (int b = 0; b < 2; ++b) {
                float* base = static_cast<float*>(P.ipc_u[side][b]);
                if (side == 0)
                    P.peer_lo[b] = base + hg;   // its high ghost planes
                else
                    P.peer_hi[b] = base;        // its low ghost planes
            }
            if (P.tti_set && pb.has_tti) {
                for (int b = 0; b < 2; ++b) {
                    SFB_CUDA(cudaIpcOpenMemHandle(&P.ipc_g[side][b], pb.g[b],
                                                  cudaIpcMemLazyEnablePeerAccess));
                    SFB_CUDA(cudaIpcOpenMemHandle(&P.ipc_r[side][b], pb.r[b],
                                                  cudaIpcMemLazyEnablePeerAccess));
                    float* gb = static_cast<float*>(P.ipc_g[side][b]);
                    float* rb = static_cast<float*>(P.ipc_r[side][b]);
                    if (side == 0) {
                        P.peer_g_lo[b] = gb + hg;
                        P.peer_r_lo[b] = rb + hg;
                    } else {
                        P.peer_g_hi[b] = gb;
                        P.peer_r_hi[b] = rb;
                    }
                }
            }
        }
        P.push_count = P.done_count = P.g_count = 0;
        SFB_CUDA(cudaMemsetAsync(P.push_flag.p, 0, 256, P.s_main));
        // the ordering of the ranks rests on stream waits on the NEIGHBOURS' counters: prove
        // here, where the caller can still fall back to send/recv, that this driver accepts
        // such a wait on peer-mapped memory (>= 0 holds at once, whatever the neighbour does)
        static StreamValueFn wait_value = stream_value_fn("cuStreamWaitValue32");
        for (int side = 0; side < 2; ++side) {
            if (!P.ipc_flag[side]) continue;
            const CUresult rc = wait_value(P.s_main, reinterpret_cast<CUdeviceptr>(P.ipc_flag[side]),
                                           0u, CU_STREAM_WAIT_VALUE_GEQ);
            if (rc != CUDA_SUCCESS)
                throw Failure(SFB_ERR_CAPABILITY,
                              "link_peers_ipc: stream wait on the neighbour's counter refused "
                              "(code " + std::to_string(int(rc)) + ")");
        }
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
    });
}

SFB_API int sfb_peer_wait_ipc(sfb_plan* plan) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        static StreamValueFn wait_value = stream_value_fn("cuStreamWaitValue32");
        auto wait = [&](cudaStream_t st, CUdeviceptr word, unsigned value) {
            CUresult rc = wait_value(st, word, value, CU_STREAM_WAIT_VALUE_GEQ);
            if (rc != CUDA_SUCCESS)
                throw Failure(SFB_ERR_CUDA, "cuStreamWaitValue32 failed with code " +
                                                std::to_string(int(rc)));
        };
        // every slab has made the same number of half-steps when its neighbours may go on
        for (int side = 0; side < 2; ++side) {
            if (!P.ipc_flag[side]) continue;
            const CUdeviceptr f = reinterpret_cast<CUdeviceptr>(P.ipc_flag[side]);
            // (1) their pushes of this step have landed in this plan's ghost planes: both
            // streams read those next step
            wait(P.s_main, f, P.push_count);
            if (P.s_bnd != P.s_main) wait(P.s_bnd, f, P.push_count);
            // (2) they have finished READING their own ghost planes of the level this plan's
            // next step overwrites (their last reader is the gather of the interior
            // half-step, on their main stream).  The split protocol stores into peer memory
            // from the boundary stream, the single-launch step from the main stream.
            wait(P.s_bnd, f + 4, P.done_count);
            if (P.s_bnd != P.s_main) wait(P.s_main, f + 4, P.done_count);
        }
    });
}

SFB_API int sfb_peer_wait(sfb_plan* plan, sfb_plan* neighbour) {
    if (!plan || !neighbour) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        // (1) the neighbour's pushes of this step have landed (both streams read them)
        SFB_CUDA(cudaStreamWaitEvent(plan->s_main, neighbour->ev_push, 0));
        if (plan->s_bnd != plan->s_main)
            SFB_CUDA(cudaStreamWaitEvent(plan->s_bnd, neighbour->ev_push, 0));
        // (2) the neighbour's gather has finished reading the ghost planes this plan's next
        // step overwrites (from the boundary stream in the split protocol, from the main
        // stream in the single-launch step)
        SFB_CUDA(cudaStreamWaitEvent(plan->s_bnd, neighbour->ev_done, 0));
        if (plan->s_bnd != plan->s_main)
            SFB_CUDA(cudaStreamWaitEvent(plan->s_main, neighbour->ev_done, 0));
    });
}

SFB_API int sfb_step_slab_interior(sfb_plan* plan, int op, int64_t t) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        step_compute(P, op, t, SFB_PART_INTERIOR);
        step_points(P, op, t, SFB_PART_INTERIOR);
        if (P.peer_lo[0] || P.peer_hi[0]) {   // linked: the ghost planes of level t are free
            SFB_CUDA(cudaEventRecord(P.ev_done, P.s_main));
            if (P.ipc_flag[0] || P.ipc_flag[1]) {
                static StreamValueFn write_value = stream_value_fn("cuStreamWriteValue32");
                CUresult rc = write_value(P.s_main,
                                          reinterpret_cast<CUdeviceptr>(P.push_flag.p) + 4,
                                          ++P.done_count, 0);
                if (rc != CUDA_SUCCESS)
                    throw Failure(SFB_ERR_CUDA, "cuStreamWriteValue32 failed with code " +
                                                    std::to_string(int(rc)));
            }
        }
    });
}

SFB_API int sfb_step_end(sfb_plan* plan, int op) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        if (P.s_bnd != P.s_main) SFB_CUDA(cudaStreamSynchronize(P.s_bnd));
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
        finite_guard(P, "slab step");
        if (op == SFB_OP_FORWARD && P.save_every > 0) P.history_valid = true;
    });
}

SFB_API int sfb_halo_blocks(sfb_plan* plan, int op, int64_t t, void** send_lo, void** send_hi,
                    void** recv_lo, void** recv_hi, int64_t* count) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        roles(op);
        // both operators write the new level into the buffer of parity (t+1)&1
        float* u = P.u[(t + 1) & 1].as<float>();
        const long long blk = (long long)P.K * P.plane;
        if (recv_lo) *recv_lo = u;
        if (send_lo) *send_lo = u + blk;
        if (send_hi) *send_hi = u + (long long)P.n0 * P.plane;
        if (recv_hi) *recv_hi = u + (long long)(P.n0 + P.K) * P.plane;
        if (count) *count = blk;
    });
}

namespace {
// a C-ABI call made from inside another one: its failure becomes this call's failure
void chain(sfb_plan* plan, int rc) {
    if (rc != SFB_OK) throw Failure(rc, plan->err);
}
}  // namespace

SFB_API int sfb_slab_run(sfb_plan* plan, int op, int64_t t_from, int64_t t_to, const double* inj,
                         double* smp) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        const OpRoles ro = roles(op);
        require(t_from >= 1 && t_from <= t_to && t_to <= P.desc.nt - 1, SFB_ERR_PARAMETER,
                "slab_run: steps must lie in [1, nt - 1)");
        const bool linked = P.peer_lo[0] || P.peer_hi[0];
        require(!linked || P.ipc_flag[0] || P.ipc_flag[1], SFB_ERR_CAPABILITY,
                "slab_run: plans linked in-process are stepped call by call "
                "(sfb_step_slab_fused + sfb_peer_wait)");
        const bool tti = op == SFB_OP_TTI_FORWARD;
        std::unique_ptr<RowStreamer> rs;
        if (smp && ro.smp >= 0) rs.reset(new RowStreamer(P, P.cloud[ro.smp], smp));
        std::unique_ptr<RowFeeder> feed;
        if (inj) {
            feed.reset(new RowFeeder(P, P.cloud[ro.inj], inj, ro.backward, t_from, t_to - 1));
            P.cloud[ro.inj].has_in = true;
        }
        for (int64_t i = 0; i < t_to - t_from; ++i) {
            const int64_t t = ro.backward ? t_to - 1 - i : t_from + i;
            if (feed) feed->before_step(t);
            if (tti) {
                chain(plan, sfb_tti_step_rot_fused(plan, t));
                chain(plan, sfb_tti_peer_wait_g_ipc(plan));
                chain(plan, sfb_tti_step_update_fused(plan, t));
            } else {
                chain(plan, sfb_step_slab_fused(plan, op, t));
            }
            chain(plan, sfb_peer_wait_ipc(plan));
            if (rs) rs->row_done(t);
        }
        if (feed) feed->finish();
        if (rs) rs->finish();
    });
}

SFB_API int sfb_debug_stall(sfb_plan* plan, int boundary_stream, int64_t microseconds) {
    if (!plan || microseconds < 0 || microseconds > 1000000) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        stall_kernel<<<1, 1, 0, boundary_stream ? plan->s_bnd : plan->s_main>>>(
            (unsigned long long)microseconds * 1000ull);
        SFB_CUDA(cudaGetLastError());
    });
}

SFB_API int sfb_stream_sync(sfb_plan* plan) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        if (plan->s_bnd != plan->s_main) SFB_CUDA(cudaStreamSynchronize(plan->s_bnd));
        SFB_CUDA(cudaStreamSynchronize(plan->s_main));
    });
}

SFB_API int sfb_streams(sfb_plan* plan, void** main_stream, void** boundary_stream) {
    if (!plan) return SFB_ERR_PARAMETER;
    if (main_stream) *main_stream = plan->s_main;
    if (boundary_stream) *boundary_stream = plan->s_bnd;
    return SFB_OK;
}

SFB_API int sfb_set_streams(sfb_plan* plan, void* main_stream, void* boundary_stream) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        SFB_CUDA(cudaDeviceSynchronize());
        if (P.own_streams) {
            cudaStreamDestroy(P.s_main);
            cudaStreamDestroy(P.s_bnd);
        }
        P.own_streams = false;
        P.s_main = static_cast<cudaStream_t>(main_stream);
        P.s_bnd = static_cast<cudaStream_t>(boundary_stream);
    });
}

SFB_API int sfb_copy_halo(sfb_plan* dst_plan, void* dst, const void* src, int64_t count) {
    if (!dst_plan) return SFB_ERR_PARAMETER;
    return guarded(dst_plan, [&] {
        SFB_CUDA(cudaMemcpyAsync(dst, src, size_t(count) * 4, cudaMemcpyDeviceToDevice,
                                 dst_plan->s_main));
    });
}

SFB_API int sfb_autotune(sfb_plan* plan, int steps) {
    // the counterpart of the reference's autotune (proj/include/sf/execute.hpp:56): time
    // every compiled tile shape of this order on the plan's own (zeroed) buffers, keep the
    // fastest.  Destroys the wavefield state; call before a run.
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
        require(P.model_set, SFB_ERR_BINDING, "autotune needs the model (sfb_set_model)");
        require(P.desc.nt >= 4, SFB_ERR_PARAMETER, "autotune needs nt >= 4");
        if (steps < 1) steps = 6;
        const StepVariant* best = nullptr;
        float best_ms = 0.f;
        for (const StepVariant& v : step_variant_registry()) {
            if (v.K != P.K || v.sep != P.sep) continue;
            select_variant(P, v.TXV, v.TY, v.NST, variant_kind(v));
            SFB_CUDA(cudaMemsetAsync(P.u[0].p, 0, size_t(P.ucount) * 4, P.s_main));
            SFB_CUDA(cudaMemsetAsync(P.u[1].p, 0, size_t(P.ucount) * 4, P.s_main));
            P.save_every = 0;
            for (int rep = 0; rep < 2; ++rep) {  // first round warms up
                SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
                for (int i = 0; i < steps; ++i) step_compute(P, SFB_OP_FORWARD, 1 + (i & 1), SFB_PART_ALL);
                SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
                SFB_CUDA(cudaStreamSynchronize(P.s_main));
            }
            float ms = 0.f;
            SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
            if (!best || ms < best_ms) {
                best = &v;
                best_ms = ms;
            }
        }
        require(best != nullptr, SFB_ERR_CAPABILITY, "no kernel image for this space order");
        select_variant(P, best->TXV, best->TY, best->NST, variant_kind(*best));
        P.history_valid = false;
        P.live_level[0] = P.live_level[1] = -1;
    });
}

SFB_API int sfb_launch_count(sfb_plan* plan, int64_t* count) {
    if (!plan || !count) return SFB_ERR_PARAMETER;
    *count = plan->launches;
    return SFB_OK;
}

SFB_API int sfb_set_dense_damping(sfb_plan* plan, int on) {
    if (!plan) return SFB_ERR_PARAMETER;
    plan->force_dense_damp = on != 0;
    return SFB_OK;
}

SFB_API int sfb_set_tile(sfb_plan* plan, int txv, int ty, int stages, int chunk) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        // stages < 0 selects the dual-stream kernel with |stages| stages; |stages| > 100 its
        // rotated-queue variant with |stages| - 100 stages; |stages| > 200 the 2 x 2 patch
        // variant with |stages| - 200 stages; |stages| > 300 the sliding-window variant;
        // |stages| > 400 the tall variant (two rows of four nodes per thread)
        const int a = stages < 0 ? -stages : stages;
        select_variant(*plan, txv, ty, a % 100,
                       stages < 0 ? (a > 400 ? 5 : a > 300 ? 4 : (a > 200 ? 3 : (a > 100 ? 2 : 1))) : 0);
        if (chunk > 0) plan->chunk = std::min(chunk, plan->n0);
    });
}

SFB_API int sfb_get_tile(sfb_plan* plan, int* txv, int* ty, int* nst, int* chunk, int* sep) {
    if (!plan || !plan->variant) return SFB_ERR_PARAMETER;
    if (txv) *txv = plan->variant->TXV;
    if (ty) *ty = plan->variant->TY;
    if (nst)
        *nst = plan->variant->dual ? -(plan->variant->NST + (plan->variant->tall ? 400
                                                             : plan->variant->slide ? 300
                                                             : plan->variant->patch ? 200
                                                             : plan->variant->rotate ? 100 : 0))
                                   : plan->variant->NST;
    if (chunk) *chunk = plan->chunk;
    if (sep) *sep = plan->variant->sep ? 1 : 0;
    return SFB_OK;
}

}  // extern "C"
