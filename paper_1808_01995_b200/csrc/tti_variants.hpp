// tti_variants.hpp -- registry of the compiled TTI kernels (one tile shape per order).
#pragma once

#include <vector>

#include "tti_kernels.cuh"

namespace sfb {

constexpr int kTtiTXV = 16, kTtiTY = 16, kTtiNS = 4;
#ifndef SFB_TTI_NS_DIV
#define SFB_TTI_NS_DIV 6
#endif
constexpr int kTtiNSDiv = SFB_TTI_NS_DIV;
#ifndef SFB_TTI_NS_UPD
#define SFB_TTI_NS_UPD 4
#endif
constexpr int kTtiNSUpd = SFB_TTI_NS_UPD;

struct TtiVariant {
    int K;
    int tile_x, tile_y, box_w, box_h;
    int rot_threads, upd_threads;
    size_t smem_rot, smem_div, smem_upd[2];   // upd: [dense, separable]
    const void* f_rot;
    const void* f_div;
    const void* f_upd[2];
    cudaError_t (*rot)(const RotMaps&, const RotParams&, dim3, cudaStream_t);
    cudaError_t (*div)(const DivMaps&, const DivParams&, dim3, cudaStream_t);
    cudaError_t (*upd[2])(const UpdMaps&, const UpdParams&, dim3, cudaStream_t);
};

std::vector<TtiVariant>& tti_variant_registry();

template <int K>
cudaError_t launch_rot(const RotMaps& tm, const RotParams& p, dim3 grid, cudaStream_t st) {
    using S = RotShape<K, kTtiTXV, kTtiTY, kTtiNS>;
    tti_rot_kernel<K, kTtiTXV, kTtiTY, kTtiNS><<<grid, S::NTHREADS, S::SMEM, st>>>(tm, p);
    return cudaGetLastError();
}

template <int K>
cudaError_t launch_div(const DivMaps& tm, const DivParams& p, dim3 grid, cudaStream_t st) {
    using S = DivShape<K, kTtiTXV, kTtiTY, kTtiNSDiv>;
    tti_div_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv><<<grid, S::NTHREADS, S::SMEM, st>>>(tm, p);
    return cudaGetLastError();
}

template <int K, bool SEP>
cudaError_t launch_upd(const UpdMaps& tm, const UpdParams& p, dim3 grid, cudaStream_t st) {
    using S = UpdShape<K, kTtiTXV, kTtiTY, kTtiNSUpd, SEP>;
    tti_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSUpd, SEP><<<grid, S::NTHREADS, S::SMEM, st>>>(tm, p);
    return cudaGetLastError();
}

template <int K>
void register_tti() {
    using R0 = RotShape<K, kTtiTXV, kTtiTY, kTtiNS>;
    using R1 = DivShape<K, kTtiTXV, kTtiTY, kTtiNSDiv>;
    using U0 = UpdShape<K, kTtiTXV, kTtiTY, kTtiNSUpd, false>;
    using U1 = UpdShape<K, kTtiTXV, kTtiTY, kTtiNSUpd, true>;
    static_assert(R0::SMEM <= 227 * 1024 && R1::SMEM <= 227 * 1024 && U0::SMEM <= 227 * 1024,
                  "TTI rings exceed shared memory");
    TtiVariant v;
    v.K = K;
    v.tile_x = R0::TX; v.tile_y = kTtiTY; v.box_w = R0::SW; v.box_h = R0::SH;
    v.rot_threads = R0::NTHREADS; v.upd_threads = U0::NTHREADS;
    v.smem_rot = R0::SMEM; v.smem_div = R1::SMEM;
    v.smem_upd[0] = U0::SMEM; v.smem_upd[1] = U1::SMEM;
    v.f_rot = reinterpret_cast<const void*>(&tti_rot_kernel<K, kTtiTXV, kTtiTY, kTtiNS>);
    v.f_div = reinterpret_cast<const void*>(&tti_div_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv>);
    v.f_upd[0] = reinterpret_cast<const void*>(&tti_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSUpd, false>);
    v.f_upd[1] = reinterpret_cast<const void*>(&tti_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSUpd, true>);
    v.rot = &launch_rot<K>;
    v.div = &launch_div<K>;
    v.upd[0] = &launch_upd<K, false>;
    v.upd[1] = &launch_upd<K, true>;
    tti_variant_registry().push_back(v);
}

struct TtiRegistrar {
    explicit TtiRegistrar(void (*fn)()) { fn(); }
};

}  // namespace sfb

#define SFB_INSTANTIATE_TTI(KVAL) \
    static sfb::TtiRegistrar sfb_tti_registrar_##KVAL(&sfb::register_tti<KVAL>);
