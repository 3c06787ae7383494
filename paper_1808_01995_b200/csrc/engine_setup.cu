// engine_setup.cu -- plan set-up and data movement behind the C-ABI: tensor maps, tile-shape
// choice, strided f64 host fields <-> fp32 device fields, separable-damping detection, point
// tables, trace traffic.
#include <cstdint>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "engine.hpp"
#include "point_kernels.cuh"

namespace sfb {

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

// dual: -1 any, 0 ring kernel, 1 dual-stream, 2 dual-stream with the rotated (unrolled) queue,
// 3 dual-stream with 2 x 2 patches per thread, 4 dual-stream with the sliding queue window,
// 5 tall (two rows of four nodes per thread)
void select_variant(Plan& P, int txv, int ty, int nst, int dual) {
    const StepVariant* best = nullptr;
    for (const StepVariant& v : step_variant_registry()) {
        if (v.K != P.K || v.sep != P.sep) continue;
        if (dual >= 0 && variant_kind(v) != dual) continue;
        if (txv > 0 && (v.TXV != txv || v.TY != ty || (nst > 0 && v.NST != nst))) continue;
        if (txv <= 0) {
            // default shape (measured on B200, tools/probe_tiles.py): the ring kernel up to
            // order 8, the dual-stream kernel (4 stages) above -- with the sliding queue
            // window from order 12 up; 64 x 16 tiles, 64 x 14 from order 14 up
            const bool want_dual = P.K >= 5;
            const bool want_slide = P.K >= 6;
            const int want_ty = P.K >= 7 ? 14 : 16;
            if (v.dual != want_dual || v.rotate || v.patch || v.tall || v.slide != want_slide || v.TXV != 16 ||
                v.TY != want_ty)
                continue;
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
    if (best->func_push)
        SFB_CUDA(cudaFuncSetAttribute(best->func_push, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    // a dense host array (numpy, a halo-free Function): move fp32 over the bus through the
    // pinned halves and widen on host threads -- half the PCIe bytes of the general path
    long long hs[3] = {0, 0, 0};
    for (int a = 0; a < P.ndim; ++a) hs[3 - P.ndim + a] = out->stride[a];
    const bool dense = (P.N[2] == 1 || hs[2] == 1) && (P.N[1] == 1 || hs[1] == P.N[2]) &&
                       (P.N[0] == 1 || hs[0] == P.N[1] * P.N[2]);
    if (dense) {
        const float* src = dev;
        if (P.pitch != P.N[2]) {
            tmp.alloc(size_t(rows) * P.N[2] * 4, false);
            pack_f32_kernel<<<row_grid(P, rows), 256, 0, P.s_main>>>(dev, tmp.as<float>(), rows,
                                                                   int(P.N[2]), P.pitch);
            SFB_CUDA(cudaGetLastError());
            src = tmp.as<float>();
        }
        download_f32(P, src, out->ptr + P.z_lo * hs[0], rows * P.N[2]);
        return;
    }
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

void detect_separable_damping(Plan& P, const IntView& v, const DevBuf& damp_f64, long long ref_plane) {
    P.sep = false;
    if (P.force_dense_damp) return;
    // lines through the reference node (grid centre by default); its value is counted once
    // (in px).  Any reference node yields the same sums for a separable field.
    const long long c[3] = {ref_plane, P.N[1] / 2, P.N[2] / 2};
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



void widen(const float* src, double* dst, long long n) {
    // big tables (a gradient, a wavefield) are written once and not read back soon: stream the
    // f64 stores past the cache so that the host moves 12 bytes per value instead of 20
    const bool stream = n >= (1 << 20);
    parallel_chunks(n, [=](long long b, long long e) {
        long long i = b;
#if defined(__SSE2__)
        if (stream) {
            while (i < e && (reinterpret_cast<uintptr_t>(dst + i) & 15)) { dst[i] = double(src[i]); ++i; }
            for (; i + 4 <= e; i += 4) {
                const __m128 f = _mm_loadu_ps(src + i);
                _mm_stream_pd(dst + i, _mm_cvtps_pd(f));
                _mm_stream_pd(dst + i + 2, _mm_cvtps_pd(_mm_movehl_ps(f, f)));
            }
            _mm_sfence();
        }
#endif
        for (; i < e; ++i) dst[i] = double(src[i]);
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

}  // namespace sfb
