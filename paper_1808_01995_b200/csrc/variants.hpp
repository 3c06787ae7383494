// variants.hpp -- registry of compiled tile shapes of the acoustic step kernel.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

#include "acoustic_kernel.cuh"

namespace sfb {

struct StepVariant {
    int K, TXV, TY, R, NST;
    bool sep;
    int tile_x, tile_y;   // output tile (d2, d1)
    int box_w, box_h;     // TMA box (d2, d1)
    int halo_x;           // KP
    int nthreads;
    size_t smem;
    const void* func;
    cudaError_t (*launch)(const CUtensorMap&, const StepParams&, dim3, cudaStream_t);
};

std::vector<StepVariant>& step_variant_registry();

template <int K, int TXV, int TY, int R, int NST, bool SEP>
cudaError_t launch_step(const CUtensorMap& tm, const StepParams& p, dim3 grid, cudaStream_t st) {
    using S = StepShape<K, TXV, TY, R, NST>;
    acoustic_step_kernel<K, TXV, TY, R, NST, SEP><<<grid, S::NTHREADS, S::SMEM, st>>>(tm, p);
    return cudaGetLastError();
}

template <int K, int TXV, int TY, int R, int NST, bool SEP>
void register_step() {
    using S = StepShape<K, TXV, TY, R, NST>;
    StepVariant v;
    v.K = K; v.TXV = TXV; v.TY = TY; v.R = R; v.NST = NST; v.sep = SEP;
    v.tile_x = S::TX; v.tile_y = TY; v.box_w = S::SW; v.box_h = S::SH; v.halo_x = S::KP;
    v.nthreads = S::NTHREADS; v.smem = S::SMEM;
    v.func = reinterpret_cast<const void*>(&acoustic_step_kernel<K, TXV, TY, R, NST, SEP>);
    v.launch = &launch_step<K, TXV, TY, R, NST, SEP>;
    step_variant_registry().push_back(v);
}

// the tile shapes built for every half-order K (dense and separable damping)
template <int K>
void register_all_for_K() {
    // the first entry is the default; sfb_set_tile / the autotuner pick among the rest
    register_step<K, 16, 16, 1, K + 3, false>();
    register_step<K, 16, 16, 1, K + 3, true>();
    register_step<K, 16, 32, 1, K + 3, false>();
    register_step<K, 16, 32, 1, K + 3, true>();
    register_step<K, 32, 8, 1, K + 3, false>();
    register_step<K, 32, 8, 1, K + 3, true>();
    if constexpr (K <= 4) {  // two rows per thread: the register queue doubles
        register_step<K, 16, 32, 2, K + 3, false>();
        register_step<K, 16, 32, 2, K + 3, true>();
    }
}

struct VariantRegistrar {
    explicit VariantRegistrar(void (*fn)()) { fn(); }
};

}  // namespace sfb

#define SFB_INSTANTIATE_K(KVAL) \
    static sfb::VariantRegistrar sfb_registrar_##KVAL(&sfb::register_all_for_K<KVAL>);
