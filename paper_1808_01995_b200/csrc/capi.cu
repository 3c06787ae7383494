// capi.cu -- the extern "C" boundary of libsfb200.so (declared in include/sfb200.h) and
// the host logic behind it: plan set-up, model / point-table upload, the time loops.
//
// The time loops restate run_wave / run_gradient / run_window of the reference
// (proj/src/seismic_ops.cpp:44-54,137-147): zero the wavefield and the sampled traces,
// then step t over [1, nt-1), ascending for the forward operator and descending for the
// adjoint and gradient operators, each step being dense update -> scatter -> gather in
// that order (proj/tests/test_compiler.cpp:109-120).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <thread>

#include "fdweights.hpp"
#include "plan.hpp"
#include "point_kernels.cuh"
#include "tti_kernels.cuh"

namespace sfb {

std::vector<StepVariant>& step_variant_registry() {
    static std::vector<StepVariant> reg;
    return reg;
}

std::vector<TtiVariant>& tti_variant_registry() {
    static std::vector<TtiVariant> reg;
    return reg;
}

namespace {

thread_local std::string g_create_err;

template <typename F>
int guarded(sfb_plan* plan, F&& f) {
    try {
        if (plan) {
            cudaError_t e = cudaSetDevice(plan->device);
            if (e != cudaSuccess)
                throw Failure(SFB_ERR_CAPABILITY,
                              std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        }
        f();
        return SFB_OK;
    } catch (const Failure& e) {
        (plan ? plan->err : g_create_err) = e.what();
        return e.code;
    } catch (const std::exception& e) {
        (plan ? plan->err : g_create_err) = e.what();
        return SFB_ERR_CUDA;
    }
}

void require(bool ok, int code, const char* msg) {
    if (!ok) throw Failure(code, msg);
}

long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

// ---- driver entry point for tensor maps (no link-time libcuda dependency) -------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw Failure(SFB_ERR_CAPABILITY, "driver lacks cuTensorMapEncodeTiled");
    return fn;
}

void encode_map(CUtensorMap* tm, void* base, long long n2, long long n1, long long n0,
                long long pitch, long long plane, int box_w, int box_h) {
    cuuint64_t dims[3] = {cuuint64_t(n2), cuuint64_t(n1), cuuint64_t(n0)};
    cuuint64_t strides[2] = {cuuint64_t(pitch) * 4, cuuint64_t(plane) * 4};
    cuuint32_t box[3] = {cuuint32_t(box_w), cuuint32_t(box_h), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult rc = encode_tiled()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS)
        throw Failure(SFB_ERR_CUDA, "cuTensorMapEncodeTiled failed with code " +
                                        std::to_string(int(rc)));
}

// (re)build every tensor map of the plan for the current tile shape
void make_tensor_maps(Plan& P) {
    const StepVariant& v = *P.variant;
    for (int b = 0; b < 2; ++b) {
        if (!P.u[b].p) continue;
        encode_map(&P.tm_u[b], P.u[b].p, P.N[2], P.N[1], P.n0 + 2 * P.K, P.pitch, P.plane,
                   v.box_w, v.box_h);
        encode_map(&P.tm_o[b], P.u[b].p, P.N[2], P.N[1], P.n0 + 2 * P.K, P.pitch, P.plane,
                   v.tile_x, v.tile_y);
    }
    for (int b = 0; b < 2; ++b) {
        if (!P.f[b].p) continue;
        encode_map(&P.tm_fu[b], P.f[b].p, P.N[2], P.N[1], P.n0 + 2 * P.K, P.pitch, P.plane,
                   v.box_w, v.box_h);
        encode_map(&P.tm_fo[b], P.f[b].p, P.N[2], P.N[1], P.n0 + 2 * P.K, P.pitch, P.plane,
                   v.tile_x, v.tile_y);
    }
    if (P.r.p)
        encode_map(&P.tm_r, P.r.p, P.N[2], P.N[1], P.n0, P.pitch, P.plane, v.tile_x, v.tile_y);
    if (P.damp.p)
        encode_map(&P.tm_d, P.damp.p, P.N[2], P.N[1], P.n0, P.pitch, P.plane, v.tile_x,
                   v.tile_y);
}

// ---- tile shape / chunk choice ----------------------------------------------------------

// dual: -1 any, 0 ring kernel, 1 dual-stream, 2 dual-stream with the rotated (unrolled) queue
void select_variant(Plan& P, int txv, int ty, int nst, int dual = -1) {
    const StepVariant* best = nullptr;
    for (const StepVariant& v : step_variant_registry()) {
        if (v.K != P.K || v.sep != P.sep) continue;
        if (dual >= 0 && (int(v.dual) + int(v.rotate)) != dual) continue;
        if (txv > 0 && (v.TXV != txv || v.TY != ty || (nst > 0 && v.NST != nst))) continue;
        if (txv <= 0) {
            // default shape (measured on B200, tools/probe_tiles.py): the ring kernel up to
            // order 8, the dual-stream kernel (4 stages) above, 64 x 16 tiles
            const bool want_dual = P.K >= 5;
            if (v.dual != want_dual || v.rotate || v.TXV != 16 || v.TY != 16) continue;
            if (v.NST != (want_dual ? 4 : P.K + 3)) continue;
        }
        if (!best) best = &v;
    }
    if (!best && txv <= 0)  // fall back to any compiled shape of this order
        for (const StepVariant& v : step_variant_registry())
            if (v.K == P.K && v.sep == P.sep) {
                best = &v;
                break;
            }
    if (!best)
        throw Failure(SFB_ERR_CAPABILITY, "no kernel image for space order " +
                                              std::to_string(2 * P.K));
    P.variant = best;
    SFB_CUDA(cudaFuncSetAttribute(best->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(best->smem)));
    int bps = 1;
    SFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, best->func, best->nthreads,
                                                           best->smem));
    if (bps < 1) bps = 1;
    // split d0 into chunks so the grid fills whole waves; every chunk spends 2K extra
    // iterations filling its register queue (re-reading 2K planes of u[t]), which the score
    // charges at half an output plane each (measured on the 208-plane order-16 slab of
    // config 5: tools/run_config5.py)
    const long long tiles = ((P.N[2] + best->tile_x - 1) / best->tile_x) *
                            ((P.N[1] + best->tile_y - 1) / best->tile_y);
    const long long slots = (long long)P.sm_count * bps;
    int best_nch = 1;
    double best_score = -1;
    const int max_nch = std::max(1, P.n0 / std::max(1, 2 * P.K));
    for (int nch = 1; nch <= max_nch; ++nch) {
        const int chunk = (P.n0 + nch - 1) / nch;
        const int real = (P.n0 + chunk - 1) / chunk;
        const long long total = tiles * real;
        const long long waves = (total + slots - 1) / slots;
        const double fill = double(total) / double(waves * slots);
        const double extra = 1.0 + (2.0 * P.K / chunk) * 0.5;
        const double score = fill / extra;
        if (score > best_score + 1e-9) {
            best_score = score;
            best_nch = real;
        }
        if (total > 16 * slots) break;
    }
    P.chunk = (P.n0 + best_nch - 1) / best_nch;
    make_tensor_maps(P);
}

// ---- host <-> device field movement --------------------------------------------------------

struct IntView {
    const double* ptr;
    long long s[3];
};

IntView embed_view(const Plan& P, const double* ptr, const int64_t* stride) {
    IntView v{ptr, {0, 0, 0}};
    const int off = 3 - P.ndim;
    for (int a = 0; a < P.ndim; ++a) v.s[off + a] = stride[a];
    return v;
}

// planes [gz0, gz0 + cnt) of a strided host f64 field -> compact device f64 [cnt][N1][N2]
void upload_f64_planes(Plan& P, const IntView& v, DevBuf& tmp, long long gz0, long long cnt) {
    const size_t rowb = size_t(P.N[2]) * 8;
    tmp.alloc(size_t(cnt) * P.N[1] * rowb, false);
    double* d = tmp.as<double>();
    if (v.s[2] == 1 || P.N[2] == 1) {
        for (long long z = 0; z < cnt; ++z) {
            const double* src = v.ptr + (gz0 + z) * v.s[0];
            const size_t spitch = P.N[1] > 1 ? size_t(v.s[1]) * 8 : rowb;
            SFB_CUDA(cudaMemcpy2DAsync(d + z * P.N[1] * P.N[2], rowb, src, spitch, rowb,
                                       size_t(P.N[1]), cudaMemcpyHostToDevice, P.s_main));
        }
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
    } else {
        std::vector<double> row(size_t(P.N[1]) * P.N[2]);
        for (long long z = 0; z < cnt; ++z) {
            for (long long j = 0; j < P.N[1]; ++j)
                for (long long l = 0; l < P.N[2]; ++l)
                    row[j * P.N[2] + l] = v.ptr[(gz0 + z) * v.s[0] + j * v.s[1] + l * v.s[2]];
            SFB_CUDA(cudaMemcpyAsync(d + z * P.N[1] * P.N[2], row.data(), row.size() * 8,
                                     cudaMemcpyHostToDevice, P.s_main));
            SFB_CUDA(cudaStreamSynchronize(P.s_main));
        }
    }
}

// owned planes of a strided host f64 field -> compact device f64 [n0][N1][N2]
void upload_f64(Plan& P, const IntView& v, DevBuf& tmp) {
    upload_f64_planes(P, v, tmp, P.z_lo, P.n0);
}

// compact device f64 [n0][N1][N2] -> owned planes of a strided host f64 field
void download_f64(Plan& P, const DevBuf& tmp, double* ptr, const int64_t* stride) {
    long long s[3] = {0, 0, 0};
    const int off = 3 - P.ndim;
    for (int a = 0; a < P.ndim; ++a) s[off + a] = stride[a];
    const size_t rowb = size_t(P.N[2]) * 8;
    const double* d = tmp.as<double>();
    if (s[2] == 1 || P.N[2] == 1) {
        for (long long z = 0; z < P.n0; ++z) {
            double* dst = ptr + (P.z_lo + z) * s[0];
            const size_t dpitch = P.N[1] > 1 ? size_t(s[1]) * 8 : rowb;
            SFB_CUDA(cudaMemcpy2DAsync(dst, dpitch, d + z * P.N[1] * P.N[2], rowb, rowb,
                                       size_t(P.N[1]), cudaMemcpyDeviceToHost, P.s_main));
        }
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
    } else {
        std::vector<double> row(size_t(P.N[1]) * P.N[2]);
        for (long long z = 0; z < P.n0; ++z) {
            SFB_CUDA(cudaMemcpyAsync(row.data(), d + z * P.N[1] * P.N[2], row.size() * 8,
                                     cudaMemcpyDeviceToHost, P.s_main));
            SFB_CUDA(cudaStreamSynchronize(P.s_main));
            for (long long j = 0; j < P.N[1]; ++j)
                for (long long l = 0; l < P.N[2]; ++l)
                    ptr[(P.z_lo + z) * s[0] + j * s[1] + l * s[2]] = row[j * P.N[2] + l];
        }
    }
}

dim3 row_grid(const Plan& P, long long rows) {
    unsigned gy = unsigned(std::min<long long>(rows, 32768));
    unsigned gz = unsigned((rows + gy - 1) / gy);
    unsigned gx = unsigned(std::max<long long>(1, std::min<long long>(8, (P.N[2] + 255) / 256)));
    return dim3(gx, gy, gz);
}

// fp32 pitched compact array (no ghost planes) or wavefield level -> strided host f64
void download_field(Plan& P, const float* dev, const sfb_field_mview* out) {
    DevBuf tmp;
    const long long rows = (long long)P.n0 * P.N[1];
    tmp.alloc(size_t(rows) * P.N[2] * 8, false);
    convert_f32_pitched_f64<<<row_grid(P, rows), 256, 0, P.s_main>>>(dev, tmp.as<double>(), rows,
                                                                   int(P.N[2]), P.pitch);
    SFB_CUDA(cudaGetLastError());
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    download_f64(P, tmp, out->ptr, out->stride);
}

// ---- separable damping -----------------------------------------------------------------------
// build_damping (proj/src/model.cpp:35-56) is a sum of three 1-D profiles.  When the bound
// damp field has that structure (checked on the device against the field itself), the
// kernel rebuilds it from the profiles and never streams the dense array.
__global__ void sep_check_kernel(const double* __restrict__ damp, const double* __restrict__ pz,
                                 const double* __restrict__ py, const double* __restrict__ px,
                                 long long n0, long long n1, long long n2,
                                 unsigned long long* maxdev, unsigned long long* maxabs) {
    const long long total = n0 * n1 * n2;
    double dev = 0.0, mx = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long l = i % n2, j = (i / n2) % n1, z = i / (n2 * n1);
        const double v = damp[i];
        dev = fmax(dev, fabs(v - (pz[z] + py[j] + px[l])));
        mx = fmax(mx, fabs(v));
    }
    atomicMax(maxdev, (unsigned long long)__double_as_longlong(dev));
    atomicMax(maxabs, (unsigned long long)__double_as_longlong(mx));
}

void detect_separable_damping(Plan& P, const IntView& v, const DevBuf& damp_f64) {
    P.sep = false;
    if (P.force_dense_damp) return;
    // lines through the grid centre; the centre value is counted once (in px)
    const long long c[3] = {P.N[0] / 2, P.N[1] / 2, P.N[2] / 2};
    auto at = [&](long long i, long long j, long long l) {
        return v.ptr[i * v.s[0] + j * v.s[1] + l * v.s[2]];
    };
    const double base = at(c[0], c[1], c[2]);
    std::vector<double> pz(P.n0), py(P.N[1]), px(P.pitch, 0.0);
    for (long long z = 0; z < P.n0; ++z) pz[z] = at(P.z_lo + z, c[1], c[2]) - base;
    for (long long j = 0; j < P.N[1]; ++j) py[j] = at(c[0], j, c[2]) - base;
    for (long long l = 0; l < P.N[2]; ++l) px[l] = at(c[0], c[1], l);
    DevBuf dpz, dpy, dpx, stat;
    auto put = [&P](DevBuf& d, const void* src, size_t bytes) {
        d.alloc(bytes, false);
        SFB_CUDA(cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, P.s_main));
    };
    put(dpz, pz.data(), pz.size() * 8);
    put(dpy, py.data(), py.size() * 8);
    put(dpx, px.data(), px.size() * 8);
    stat.alloc(16, false);
    SFB_CUDA(cudaMemsetAsync(stat.p, 0, 16, P.s_main));
    sep_check_kernel<<<P.sm_count * 8, 256, 0, P.s_main>>>(
        damp_f64.as<double>(), dpz.as<double>(), dpy.as<double>(), dpx.as<double>(), P.n0, P.N[1],
        P.N[2], stat.as<unsigned long long>(), stat.as<unsigned long long>() + 1);
    SFB_CUDA(cudaGetLastError());
    double res[2];
    SFB_CUDA(cudaMemcpyAsync(res, stat.p, 16, cudaMemcpyDeviceToHost, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    if (!(res[0] <= 1e-7 * res[1] || res[1] == 0.0)) return;
    std::vector<float> fz(pz.begin(), pz.end()), fy(py.begin(), py.end()), fx(px.begin(), px.end());
    put(P.dz, fz.data(), fz.size() * 4);
    put(P.dy, fy.data(), fy.size() * 4);
    put(P.dx, fx.data(), fx.size() * 4);
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    P.sep = true;
}

// ---- point tables ------------------------------------------------------------------------

void build_cloud(Plan& P, Cloud& c) {
    const int nd = P.ndim, nc = 1 << nd, off = 3 - nd;
    struct Ent {
        long long key;  // compact node index
        long long u;
        int point;
        float w;
    };
    std::vector<Ent> ents;
    ents.reserve(size_t(c.np) * 2);
    std::vector<long long> smp_idx(c.np, -1);
    std::vector<float> smp_w(size_t(c.np) * nc);
    for (long long p = 0; p < c.np; ++p) {
        long long b[3] = {0, 0, 0};
        for (int a = 0; a < nd; ++a) {
            b[off + a] = c.base[p * nd + a];
            if (b[off + a] < 0 || b[off + a] > P.N[off + a] - 2)
                throw Failure(SFB_ERR_LOCATION, "point " + std::to_string(p) +
                                                    ": base cell outside the grid");
        }
        if (b[0] >= P.z_lo && b[0] < P.z_hi)
            smp_idx[p] = (b[0] - P.z_lo + P.K) * P.plane + b[1] * P.pitch + b[2];
        for (int cc = 0; cc < nc; ++cc) {
            const double w = c.w[p * nc + cc];
            smp_w[p * nc + cc] = float(w);
            if (w == 0.0) continue;
            long long id[3] = {b[0], b[1], b[2]};
            for (int a = 0; a < nd; ++a) id[off + a] += (cc >> a) & 1;
            if (id[0] < P.z_lo || id[0] >= P.z_hi) continue;  // node owned by a neighbour slab
            const long long z = id[0] - P.z_lo;
            Ent e;
            e.key = z * P.plane + id[1] * P.pitch + id[2];
            e.u = (z + P.K) * P.plane + id[1] * P.pitch + id[2];
            e.point = int(p);
            e.w = float(w);
            ents.push_back(e);
        }
    }
    std::stable_sort(ents.begin(), ents.end(),
                     [](const Ent& a, const Ent& b) { return a.key < b.key; });
    std::vector<int> start;
    std::vector<long long> cu, ck;
    std::vector<int> ep(ents.size());
    std::vector<float> ew(ents.size());
    for (size_t i = 0; i < ents.size(); ++i) {
        if (i == 0 || ents[i].key != ents[i - 1].key) {
            start.push_back(int(i));
            cu.push_back(ents[i].u);
            ck.push_back(ents[i].key);
        }
        ep[i] = ents[i].point;
        ew[i] = ents[i].w;
    }
    start.push_back(int(ents.size()));
    c.ncell = (long long)cu.size();
    c.nent = (long long)ents.size();
    c.h_cell_start = start;
    // node ranges lying in the low / high K boundary planes (slab stepping)
    const long long lo_lim = (long long)std::min(P.K, P.n0) * P.plane;
    const long long hi_lim = (long long)std::max(P.n0 - P.K, std::min(P.K, P.n0)) * P.plane;
    c.cell_lo_end = std::lower_bound(ck.begin(), ck.end(), lo_lim) - ck.begin();
    c.cell_hi_begin = std::lower_bound(ck.begin(), ck.end(), hi_lim) - ck.begin();

    auto put = [&P](DevBuf& d, const void* src, size_t bytes) {
        d.alloc(bytes, false);
        if (bytes) SFB_CUDA(cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, P.s_main));
    };
    put(c.cell_start, start.data(), start.size() * sizeof(int));
    put(c.cell_u, cu.data(), cu.size() * 8);
    put(c.cell_c, ck.data(), ck.size() * 8);
    put(c.ent_point, ep.data(), ep.size() * sizeof(int));
    put(c.ent_w, ew.data(), ew.size() * sizeof(float));
    put(c.smp_idx, smp_idx.data(), smp_idx.size() * 8);
    put(c.smp_w, smp_w.data(), smp_w.size() * sizeof(float));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));  // the host tables above are locals
    const size_t trb = size_t(P.desc.nt) * size_t(c.np) * sizeof(float);
    c.tr_in.alloc(trb, true);
    c.tr_out.alloc(trb, true);
    c.has_in = false;
    c.set = true;
}

// ---- trace traffic: fp32 on the wire, repacked to/from the caller's f64 on host threads ----

constexpr size_t kStageBytes = 32u << 20;  // per half

template <typename Fn>
void parallel_chunks(long long n, Fn&& fn) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nthr = unsigned(std::max<long long>(1, std::min<long long>(hw, n / 65536)));
    if (nthr <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> pool;
    const long long per = (n + nthr - 1) / nthr;
    for (unsigned i = 0; i < nthr; ++i) {
        const long long b = i * per, e = std::min(n, b + per);
        if (b < e) pool.emplace_back([=, &fn] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}

void widen(const float* src, double* dst, long long n) {
    parallel_chunks(n, [=](long long b, long long e) {
        for (long long i = b; i < e; ++i) dst[i] = double(src[i]);
    });
}

void narrow(const double* src, float* dst, long long n) {
    parallel_chunks(n, [=](long long b, long long e) {
        for (long long i = b; i < e; ++i) dst[i] = float(src[i]);
    });
}

// host f64 [n] -> device fp32 [n], chunked through the pinned halves
void upload_f32(Plan& P, const double* host, float* dev, long long n) {
    PinnedStage& st = P.stage;
    const long long cap = (long long)std::min<size_t>(kStageBytes / 4, size_t(std::max<long long>(n, 1)));
    st.ensure(size_t(cap));
    int b = 0;
    bool used[2] = {false, false};
    for (long long off = 0; off < n; off += cap, b ^= 1) {
        const long long len = std::min(cap, n - off);
        if (used[b]) SFB_CUDA(cudaEventSynchronize(st.moved[b]));
        narrow(host + off, st.p[b], len);
        SFB_CUDA(cudaMemcpyAsync(dev + off, st.p[b], size_t(len) * 4, cudaMemcpyHostToDevice,
                                 P.s_main));
        SFB_CUDA(cudaEventRecord(st.moved[b], P.s_main));
        used[b] = true;
    }
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
}

// device fp32 [n] -> host f64 [n]; the device data must be complete on s_main
void download_f32(Plan& P, const float* dev, double* host, long long n) {
    PinnedStage& st = P.stage;
    const long long cap = (long long)std::min<size_t>(kStageBytes / 4, size_t(std::max<long long>(n, 1)));
    st.ensure(size_t(cap));
    long long pend_off[2] = {0, 0}, pend_len[2] = {0, 0};
    int b = 0;
    for (long long off = 0; off < n; off += cap, b ^= 1) {
        const long long len = std::min(cap, n - off);
        SFB_CUDA(cudaMemcpyAsync(st.p[b], dev + off, size_t(len) * 4, cudaMemcpyDeviceToHost,
                                 P.s_main));
        SFB_CUDA(cudaEventRecord(st.moved[b], P.s_main));
        pend_off[b] = off;
        pend_len[b] = len;
        if (pend_len[b ^ 1]) {  // repack the previous chunk while this one is in flight
            SFB_CUDA(cudaEventSynchronize(st.moved[b ^ 1]));
            widen(st.p[b ^ 1], host + pend_off[b ^ 1], pend_len[b ^ 1]);
            pend_len[b ^ 1] = 0;
        }
    }
    for (int i = 0; i < 2; ++i)
        if (pend_len[i]) {
            SFB_CUDA(cudaEventSynchronize(st.moved[i]));
            widen(st.p[i], host + pend_off[i], pend_len[i]);
        }
}

void upload_traces(Plan& P, Cloud& c, const double* host) {
    upload_f32(P, host, c.tr_in.as<float>(), P.desc.nt * c.np);
    c.has_in = true;
}

void download_traces(Plan& P, Cloud& c, double* host) {
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    download_f32(P, c.tr_out.as<float>(), host, P.desc.nt * c.np);
}

// ---- stepping ------------------------------------------------------------------------------

struct OpRoles {
    bool backward;
    int inj, smp;  // cloud indices, -1 = none
    bool imaging;
};

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

constexpr int kPartBoundaryPair = 100;   // internal: LOW and HIGH plane groups in one launch

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

// explicit fused outputs / buffer set of one step (checkpointed runs); without it the
// save_every rules of the plain runs apply
struct StepExtras {
    bool alt = false;            // step the recompute pair f[2] instead of u[2]
    float* snap = nullptr;       // copy of the new level
    const float* usave = nullptr;  // forward level to image against
};

void step_compute(Plan& P, int op, long long t, int part, const StepExtras* ex = nullptr) {
    const OpRoles ro = roles(op);
    require(t >= 1 && t <= P.desc.nt - 2, SFB_ERR_PARAMETER, "time index outside [1, nt-1)");
    int lo, hi;
    const bool pair = part == kPartBoundaryPair;   // needs n0 >= 2K (split_slabs guarantees it)
    if (pair) {
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
                    : (part == SFB_PART_ALL || part == SFB_PART_INTERIOR) ? P.chunk : (hi - lo);
    sp.z_jump = pair ? P.n0 - 2 * P.K : 0;   // block z = 1 starts at plane n0 - K
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
    SFB_CUDA(v.launch(maps, sp, grid, st));
    ++P.launches;
    mark_stream(P, part);
    if (!alt && (part == SFB_PART_ALL || part == SFB_PART_INTERIOR)) {
        P.live_level[cur] = t;
        P.live_level[oth] = tnew;
    }
}

// part: SFB_PART_ALL = every node + gather; SFB_PART_LOW = nodes of both boundary plane
// groups (boundary stream); SFB_PART_INTERIOR = remaining nodes + gather
void step_points(Plan& P, int op, long long t, int part, float* target_override = nullptr,
                 bool allow_gather = true, const StepExtras* ex = nullptr) {
    const OpRoles ro = roles(op);
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
    if (part == SFB_PART_ALL) {
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
        point_step_kernel<<<nb_inj + nb_smp, kPointThreads, 0, st>>>(pp, nb_inj);
        SFB_CUDA(cudaGetLastError());
        ++P.launches;
    }
    mark_stream(P, part);
}

void finite_guard(Plan& P, const char* what) {
    P.flag.alloc(sizeof(int), false);
    SFB_CUDA(cudaMemsetAsync(P.flag.p, 0, sizeof(int), P.s_main));
    for (int b = 0; b < 2; ++b) {
        finite_check_kernel<<<P.sm_count * 8, 256, 0, P.s_main>>>(P.u[b].as<float>(), P.ucount,
                                                                 P.flag.as<int>());
        SFB_CUDA(cudaGetLastError());
    }
    int bad = 0;
    SFB_CUDA(cudaMemcpyAsync(&bad, P.flag.p, sizeof(int), cudaMemcpyDeviceToHost, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    if (bad) throw Failure(SFB_ERR_STABILITY, std::string(what) + ": wavefield went non-finite");
}

// Streams the sampled trace rows to the caller's f64 table while the time loop runs: every
// `rows` completed rows are copied (fp32, copy stream, pinned half) and the previous chunk
// is widened on host threads in the shadow of the GPU.
struct RowStreamer {
    Plan& P;
    Cloud& c;
    double* host;
    long long rows;            // rows per chunk
    long long lo = -1, hi = -1;  // rows gathered since the last flush
    int b = 0;
    long long pend_row[2] = {0, 0}, pend_rows[2] = {0, 0};

    RowStreamer(Plan& p, Cloud& cl, double* h) : P(p), c(cl), host(h) {
        rows = std::max<long long>(1, (long long)(kStageBytes / 4) / std::max<long long>(c.np, 1));
        P.stage.ensure(size_t(rows * c.np));
    }
    void drain(int i) {
        if (!pend_rows[i]) return;
        SFB_CUDA(cudaEventSynchronize(P.stage.moved[i]));
        widen(P.stage.p[i], host + pend_row[i] * c.np, pend_rows[i] * c.np);
        pend_rows[i] = 0;
    }
    void flush() {
        if (lo < 0) return;
        PinnedStage& st = P.stage;
        SFB_CUDA(cudaEventRecord(st.ready[b], P.s_main));
        SFB_CUDA(cudaStreamWaitEvent(st.copy, st.ready[b], 0));
        SFB_CUDA(cudaMemcpyAsync(st.p[b], c.tr_out.as<float>() + lo * c.np,
                                 size_t((hi - lo + 1) * c.np) * 4, cudaMemcpyDeviceToHost, st.copy));
        SFB_CUDA(cudaEventRecord(st.moved[b], st.copy));
        pend_row[b] = lo;
        pend_rows[b] = hi - lo + 1;
        lo = hi = -1;
        b ^= 1;
        drain(b);  // the half we are about to reuse: its copy was queued a chunk ago
    }
    void row_done(long long t) {
        lo = lo < 0 ? t : std::min(lo, t);
        hi = hi < 0 ? t : std::max(hi, t);
        if (hi - lo + 1 >= rows) flush();
    }
    void finish() {
        flush();
        drain(0);
        drain(1);
        // rows 0 and nt-1 are never sampled (structural zeros, seismic_ops.hpp:13-16)
        std::fill(host, host + c.np, 0.0);
        if (P.desc.nt > 1) std::fill(host + (P.desc.nt - 1) * c.np, host + P.desc.nt * c.np, 0.0);
    }
};

void run_op(Plan& P, int op, long long save_every, sfb_report* rep, double* stream_out = nullptr) {
    const OpRoles ro = roles(op);
    step_begin(P, op, save_every);
    const long long nt = P.desc.nt;
    std::unique_ptr<RowStreamer> rs;
    if (stream_out && ro.smp >= 0) rs.reset(new RowStreamer(P, P.cloud[ro.smp], stream_out));
    SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
    for (long long i = 0; i < nt - 2; ++i) {
        const long long t = ro.backward ? nt - 2 - i : 1 + i;
        step_compute(P, op, t, SFB_PART_ALL);
        step_points(P, op, t, SFB_PART_ALL);
        if (rs) rs->row_done(t);
    }
    SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    if (rs) rs->flush();   // the last rows travel while the NaN guard scans the fields
    finite_guard(P, op == SFB_OP_FORWARD ? "forward" : (op == SFB_OP_ADJOINT ? "adjoint" : "gradient"));
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

int tti_part_chunk(const Plan& P, int which, int part, int lo, int hi) {
    return (part == SFB_PART_ALL || part == SFB_PART_INTERIOR) ? std::min(P.tti_chunk[which], hi - lo)
                                                               : (hi - lo);
}

// pass 1 on the planes of `part`: the products a g, b g, c g of p and r (level t)
void tti_rot(Plan& P, long long t, int part) {
    require(t >= 1 && t <= P.desc.nt - 2, SFB_ERR_PARAMETER, "time index outside [1, nt-1)");
    int lo, hi;
    part_range(P, part, lo, hi);
    if (hi <= lo) return;
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
    SFB_CUDA(v.rot(m1, rp, tti_grid(P, lo, hi, rp.chunk), st));
    ++P.launches;
    mark_stream(P, part);
}

// pass 2 and the update on the planes of `part`, then the point work of the part: Hz(p),
// Hz(r) from the products (ghost planes of a g included), L(p), both leapfrog updates in
// place over level t-1, injection into p and r, sampling of p
void tti_update(Plan& P, long long t, int part) {
    require(t >= 1 && t <= P.desc.nt - 2, SFB_ERR_PARAMETER, "time index outside [1, nt-1)");
    int lo, hi;
    part_range(P, part, lo, hi);
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
        SFB_CUDA(v.div[sepi](m2, dp, tti_grid(P, lo, hi, dp.chunk), st));
        ++P.launches;
        mark_stream(P, part);
    }
    if (part != SFB_PART_LOW) {
        // HIGH (called after LOW) carries the point work of both boundary plane groups, so
        // the injections land after both groups have been overwritten by the update
        const int op = SFB_OP_TTI_FORWARD;
        const int pp = part == SFB_PART_HIGH ? SFB_PART_LOW : part;
        step_points(P, op, t, pp);                                    // p: scatter + gather
        step_points(P, op, t, pp, P.t_r[oth].as<float>(), false);     // r: scatter
    }
    if (part == SFB_PART_ALL || part == SFB_PART_INTERIOR) {
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

}  // namespace
}  // namespace sfb

using namespace sfb;

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
    if (plan->ev_t0) cudaEventDestroy(plan->ev_t0);
    if (plan->ev_t1) cudaEventDestroy(plan->ev_t1);
    delete plan;
    return SFB_OK;
}

SFB_API int sfb_set_model(sfb_plan* plan, const sfb_field_view* m, const sfb_field_view* damp,
                  double v_max) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        Plan& P = *plan;
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
        P.v_max = v_max;
        const long long rows = (long long)P.n0 * P.N[1];
        DevBuf tmp;
        P.r.alloc(size_t(P.ccount) * 4);
        P.damp.alloc(size_t(P.ccount) * 4);
        upload_f64(P, embed_view(P, m->ptr, m->stride), tmp);
        convert_r_kernel<<<row_grid(P, rows), 256, 0, P.s_main>>>(
            tmp.as<double>(), P.r.as<float>(), rows, int(P.N[2]), P.pitch,
            P.desc.dt * P.desc.dt);
        SFB_CUDA(cudaGetLastError());
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
        upload_f64(P, embed_view(P, damp->ptr, damp->stride), tmp);
        convert_f64_f32_pitched<<<row_grid(P, rows), 256, 0, P.s_main>>>(
            tmp.as<double>(), P.damp.as<float>(), rows, int(P.N[2]), P.pitch);
        SFB_CUDA(cudaGetLastError());
        SFB_CUDA(cudaStreamSynchronize(P.s_main));
        detect_separable_damping(P, embed_view(P, damp->ptr, damp->stride), tmp);
        if (P.sep) P.damp.release();
        select_variant(P, P.variant->TXV, P.variant->TY, P.variant->NST,
                       int(P.variant->dual) + int(P.variant->rotate));
        P.model_set = true;
        P.history_valid = false;
    });
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
        for (int i = 0; i < 2; ++i)
            SFB_CUDA(cudaFuncSetAttribute(P.tti_variant->f_div[i],
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(P.tti_variant->smem_div[i])));
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

namespace {
void run_window(Plan& P, int op, long long t_from, long long t_to, bool with_points,
                sfb_report* report) {
    const OpRoles ro = roles(op);
    require(t_from >= 1 && t_to <= P.desc.nt - 1 && t_from <= t_to, SFB_ERR_PARAMETER,
            "run_steps: window outside [1, nt-1)");
    const long before = P.launches;
    SFB_CUDA(cudaEventRecord(P.ev_t0, P.s_main));
    for (long long i = 0; i < t_to - t_from; ++i) {
        const long long t = ro.backward ? t_to - 1 - i : t_from + i;
        step_compute(P, op, t, SFB_PART_ALL);
        if (with_points) step_points(P, op, t, SFB_PART_ALL);
    }
    SFB_CUDA(cudaEventRecord(P.ev_t1, P.s_main));
    SFB_CUDA(cudaStreamSynchronize(P.s_main));
    float ms = 0.f;
    SFB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
    if (report) {
        const double own = double(P.n0) * double(P.N[1]) * double(P.N[2]);
        const long long fpp = 3LL * P.K * P.ndim + 3LL * P.ndim + 11 + (ro.imaging ? 7 : 0);
        report->seconds = ms * 1e-3;
        report->steps = long(t_to - t_from);
        report->flops = (long long)(double(fpp) * own * double(report->steps));
        report->gflops = ms > 0 ? double(report->flops) / (ms * 1e-3) / 1e9 : 0.0;
        report->gpts_per_s = ms > 0 ? own * double(report->steps) / (ms * 1e-3) / 1e9 : 0.0;
        report->kernel_launches = P.launches - before;
    }
}
}  // namespace

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
        upload_traces(P, P.cloud[SFB_CLOUD_REC], rec);
        run_op(P, SFB_OP_ADJOINT, 0, report, srca);
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
        upload_traces(P, P.cloud[SFB_CLOUD_REC], resid);
        if (P.ckpt_valid && !P.history_valid)
            gradient_checkpointed(P, report);
        else
            run_op(P, SFB_OP_GRADIENT, P.save_every, report);
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
    return guarded(plan, [&] { step_points(*plan, op, t, part); });
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
    });
}

SFB_API int sfb_step_slab_interior(sfb_plan* plan, int op, int64_t t) {
    if (!plan) return SFB_ERR_PARAMETER;
    return guarded(plan, [&] {
        step_compute(*plan, op, t, SFB_PART_INTERIOR);
        step_points(*plan, op, t, SFB_PART_INTERIOR);
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
            select_variant(P, v.TXV, v.TY, v.NST, int(v.dual) + int(v.rotate));
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
        select_variant(P, best->TXV, best->TY, best->NST, int(best->dual) + int(best->rotate));
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
        // rotated-queue variant with |stages| - 100 stages
        const int a = stages < 0 ? -stages : stages;
        select_variant(*plan, txv, ty, a > 100 ? a - 100 : a, stages < 0 ? (a > 100 ? 2 : 1) : 0);
        if (chunk > 0) plan->chunk = std::min(chunk, plan->n0);
    });
}

SFB_API int sfb_get_tile(sfb_plan* plan, int* txv, int* ty, int* nst, int* chunk, int* sep) {
    if (!plan || !plan->variant) return SFB_ERR_PARAMETER;
    if (txv) *txv = plan->variant->TXV;
    if (ty) *ty = plan->variant->TY;
    if (nst)
        *nst = plan->variant->dual ? -(plan->variant->NST + (plan->variant->rotate ? 100 : 0))
                                   : plan->variant->NST;
    if (chunk) *chunk = plan->chunk;
    if (sep) *sep = plan->variant->sep ? 1 : 0;
    return SFB_OK;
}

}  // extern "C"
