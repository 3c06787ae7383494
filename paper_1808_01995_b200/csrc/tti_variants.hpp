// tti_variants.hpp -- registry of the compiled TTI kernels (one tile shape per order).
#pragma once

#include <vector>

#include "launch.hpp"
#include "tti_kernels.cuh"

namespace sfb {

// 2 x 7 consumer warps + the producer warp = 15 warps: the register file is allocated in units
// of 4 warps, so 16 x 16 tiles (17 warps -> 20) would cap the kernels at 96 registers per
// thread, which the (2K+1)-plane queue of orders >= 12 does not fit in
#ifndef SFB_TTI_NS_ROT
#define SFB_TTI_NS_ROT 4
#endif
constexpr int kTtiTXV = 16, kTtiTY = 14, kTtiNS = SFB_TTI_NS_ROT;
#ifndef SFB_TTI_NS_DIV
#define SFB_TTI_NS_DIV 3
#endif
constexpr int kTtiNSDiv = SFB_TTI_NS_DIV;

struct TtiVariant {
    int K;
    int tile_x, tile_y, box_w, box_h;
    int threads;
    size_t smem_rot, smem_div[2];   // div: [dense, separable damping]
    const void* f_rot;
    const void* f_div[2];
    cudaError_t (*rot)(const RotMaps&, const RotParams&, dim3, cudaStream_t);
    cudaError_t (*div[2])(const DivMaps&, const DivParams&, dim3, cudaStream_t);
    // the same kernels with the fused halo push (linked slabs)
    const void* f_rot_push;
    const void* f_div_push[2];
    cudaError_t (*rot_push)(const RotMaps&, const RotParams&, dim3, cudaStream_t);
    cudaError_t (*div_push[2])(const DivMaps&, const DivParams&, dim3, cudaStream_t);
};

std::vector<TtiVariant>& tti_variant_registry();

template <int K, bool PUSH = false>
cudaError_t launch_rot(const RotMaps& tm, const RotParams& p, dim3 grid, cudaStream_t st) {
    using S = RotShape<K, kTtiTXV, kTtiTY, kTtiNS>;
    return launch_pdl(&tti_rot_kernel<K, kTtiTXV, kTtiTY, kTtiNS, PUSH>, grid, S::NTHREADS, S::SMEM,
                      st, tm, p);
}

template <int K, bool SEP, bool PUSH = false>
cudaError_t launch_div(const DivMaps& tm, const DivParams& p, dim3 grid, cudaStream_t st) {
    using S = DivShape<K, kTtiTXV, kTtiTY, kTtiNSDiv, SEP>;
    return launch_pdl(&tti_div_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv, SEP, PUSH>, grid,
                      S::NTHREADS, S::SMEM, st, tm, p);
}

template <int K>
void register_tti() {
    using R0 = RotShape<K, kTtiTXV, kTtiTY, kTtiNS>;
    using D0 = DivShape<K, kTtiTXV, kTtiTY, kTtiNSDiv, false>;
    using D1 = DivShape<K, kTtiTXV, kTtiTY, kTtiNSDiv, true>;
    static_assert(R0::SMEM <= 227 * 1024 && D0::SMEM <= 227 * 1024, "TTI rings exceed shared memory");
    TtiVariant v;
    v.K = K;
    v.tile_x = R0::TX; v.tile_y = kTtiTY; v.box_w = R0::SW; v.box_h = R0::SH;
    v.threads = R0::NTHREADS;
    v.smem_rot = R0::SMEM;
    v.smem_div[0] = D0::SMEM; v.smem_div[1] = D1::SMEM;
    v.f_rot = reinterpret_cast<const void*>(&tti_rot_kernel<K, kTtiTXV, kTtiTY, kTtiNS>);
    v.f_div[0] = reinterpret_cast<const void*>(
        &tti_div_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv, false>);
    v.f_div[1] = reinterpret_cast<const void*>(
        &tti_div_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv, true>);
    v.rot = &launch_rot<K>;
    v.div[0] = &launch_div<K, false>;
    v.div[1] = &launch_div<K, true>;
    v.f_rot_push = reinterpret_cast<const void*>(&tti_rot_kernel<K, kTtiTXV, kTtiTY, kTtiNS, true>);
    v.f_div_push[0] = reinterpret_cast<const void*>(
        &tti_div_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv, false, true>);
    v.f_div_push[1] = reinterpret_cast<const void*>(
        &tti_div_update_kernel<K, kTtiTXV, kTtiTY, kTtiNSDiv, true, true>);
    v.rot_push = &launch_rot<K, true>;
    v.div_push[0] = &launch_div<K, false, true>;
    v.div_push[1] = &launch_div<K, true, true>;
    tti_variant_registry().push_back(v);
}

struct TtiRegistrar {
    explicit TtiRegistrar(void (*fn)()) { fn(); }
};

}  // namespace sfb

#define SFB_INSTANTIATE_TTI(KVAL) \
    static sfb::TtiRegistrar sfb_tti_registrar_##KVAL(&sfb::register_tti<KVAL>);
