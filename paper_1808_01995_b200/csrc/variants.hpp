// variants.hpp -- registry of compiled tile shapes of the acoustic step kernel.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "acoustic_kernel.cuh"
#include "acoustic_patch_kernel.cuh"
#include "acoustic_tall_kernel.cuh"
#include "launch.hpp"

namespace sfb {

struct StepVariant {
    int K, TXV, TY, NST;  // NST: ring stages (ring kernel) or stages of the dual-stream ring
    bool sep;
    bool dual;            // dual-stream kernel (u[t] fetched as feed + centre boxes)
    bool rotate;          // dual-stream kernel unrolled by 2K+1 (queue rotation, no moves)
    bool patch = false;   // dual-stream kernel with 2 x 2 patches per thread (acoustic_patch_kernel.cuh)
    bool slide = false;   // dual-stream kernel with the sliding queue window (unrolled by two)
    bool tall = false;    // dual-stream kernel with two rows of four nodes per thread (acoustic_tall_kernel.cuh)
    int tile_x, tile_y;   // output tile (d2, d1)
    int box_w, box_h;     // TMA box of u[t] (d2, d1)
    int halo_x;           // KP
    int nthreads;
    size_t smem;
    const void* func;
    cudaError_t (*launch)(const StepMaps&, const StepParams&, dim3, cudaStream_t);
    // the same kernel with the fused halo push (default shapes only, else null)
    const void* func_push = nullptr;
    cudaError_t (*launch_push)(const StepMaps&, const StepParams&, dim3, cudaStream_t) = nullptr;
};

std::vector<StepVariant>& step_variant_registry();

// kernel family of a variant: 0 ring, 1 dual-stream, 2 dual-stream with rotated queue, 3 patch,
// 4 dual-stream with the sliding queue window, 5 tall (2 x 4 nodes per thread)
inline int variant_kind(const StepVariant& v) {
    return v.tall ? 5 : v.slide ? 4 : v.patch ? 3 : int(v.dual) + int(v.rotate);
}

template <int K, int TXV, int TY, int NST, bool SEP, bool PUSH = false>
cudaError_t launch_step(const StepMaps& tm, const StepParams& p, dim3 grid, cudaStream_t st) {
    using S = StepShape<K, TXV, TY, NST, SEP>;
    return launch_pdl(&acoustic_step_kernel<K, TXV, TY, NST, SEP, PUSH>, grid, S::NTHREADS, S::SMEM,
                      st, tm, p);
}

template <int K, int TXV, int TY, int NST, bool SEP>
void register_step() {
    using S = StepShape<K, TXV, TY, NST, SEP>;
    if constexpr (S::SMEM <= 227 * 1024) {
        StepVariant v;
        v.K = K; v.TXV = TXV; v.TY = TY; v.NST = NST; v.sep = SEP; v.dual = false; v.rotate = false;
        v.tile_x = S::TX; v.tile_y = TY; v.box_w = S::SW; v.box_h = S::SH; v.halo_x = S::KP;
        v.nthreads = S::NTHREADS; v.smem = S::SMEM;
        v.func = reinterpret_cast<const void*>(&acoustic_step_kernel<K, TXV, TY, NST, SEP>);
        v.launch = &launch_step<K, TXV, TY, NST, SEP>;
        if constexpr (K <= 4 && TXV == 16 && TY == 16 && NST == K + 3) {   // the default shape
            v.func_push = reinterpret_cast<const void*>(
                &acoustic_step_kernel<K, TXV, TY, NST, SEP, true>);
            v.launch_push = &launch_step<K, TXV, TY, NST, SEP, true>;
        }
        step_variant_registry().push_back(v);
    }
}

template <int K, int TXV, int TY, int NS, bool SEP, int MINB, bool ROT, bool PUSH = false>
cudaError_t launch_dual(const StepMaps& tm, const StepParams& p, dim3 grid, cudaStream_t st) {
    using S = DualShape<K, TXV, TY, NS, SEP>;
    return launch_pdl(&acoustic_step_dual_kernel<K, TXV, TY, NS, SEP, MINB, ROT, PUSH>, grid,
                      S::NTHREADS, S::SMEM, st, tm, p);
}

template <int K, int TXV, int TY, int NS, bool SEP, int MINB, bool ROT = false>
void register_dual() {
    using S = DualShape<K, TXV, TY, NS, SEP>;
    if constexpr (S::SMEM * MINB <= 227 * 1024) {
        StepVariant v;
        v.K = K; v.TXV = TXV; v.TY = TY; v.NST = NS; v.sep = SEP; v.dual = true; v.rotate = ROT;
        v.tile_x = S::TX; v.tile_y = TY; v.box_w = S::SW; v.box_h = S::SH; v.halo_x = S::KP;
        v.nthreads = S::NTHREADS; v.smem = S::SMEM;
        v.func = reinterpret_cast<const void*>(
            &acoustic_step_dual_kernel<K, TXV, TY, NS, SEP, MINB, ROT>);
        v.launch = &launch_dual<K, TXV, TY, NS, SEP, MINB, ROT>;
        if constexpr (K >= 5 && TXV == 16 && TY == (K >= 7 ? 14 : 16) && NS == 4 && !ROT) {   // default
            v.func_push = reinterpret_cast<const void*>(
                &acoustic_step_dual_kernel<K, TXV, TY, NS, SEP, MINB, ROT, true>);
            v.launch_push = &launch_dual<K, TXV, TY, NS, SEP, MINB, ROT, true>;
        }
        step_variant_registry().push_back(v);
    }
}

template <int K, int TXV, int TY, int NS, bool SEP, int MINB, bool PUSH = false>
cudaError_t launch_slide(const StepMaps& tm, const StepParams& p, dim3 grid, cudaStream_t st) {
    using S = DualShape<K, TXV, TY, NS, SEP>;
    return launch_pdl(&acoustic_step_dual_kernel<K, TXV, TY, NS, SEP, MINB, false, PUSH, true>, grid,
                      S::NTHREADS, S::SMEM, st, tm, p);
}

template <int K, int TXV, int TY, int NS, bool SEP, int MINB>
void register_slide() {
    using S = DualShape<K, TXV, TY, NS, SEP>;
    if constexpr (S::SMEM * MINB <= 227 * 1024) {
        StepVariant v;
        v.K = K; v.TXV = TXV; v.TY = TY; v.NST = NS; v.sep = SEP; v.dual = true; v.rotate = false;
        v.slide = true;
        v.tile_x = S::TX; v.tile_y = TY; v.box_w = S::SW; v.box_h = S::SH; v.halo_x = S::KP;
        v.nthreads = S::NTHREADS; v.smem = S::SMEM;
        v.func = reinterpret_cast<const void*>(
            &acoustic_step_dual_kernel<K, TXV, TY, NS, SEP, MINB, false, false, true>);
        v.launch = &launch_slide<K, TXV, TY, NS, SEP, MINB>;
        v.func_push = reinterpret_cast<const void*>(
            &acoustic_step_dual_kernel<K, TXV, TY, NS, SEP, MINB, false, true, true>);
        v.launch_push = &launch_slide<K, TXV, TY, NS, SEP, MINB, true>;
        step_variant_registry().push_back(v);
    }
}

template <int K, int NS, bool SEP, int MINB, bool PUSH = false>
cudaError_t launch_patch(const StepMaps& tm, const StepParams& p, dim3 grid, cudaStream_t st) {
    using S = PatchShape<K, NS, SEP>;
    return launch_pdl(&acoustic_step_patch_kernel<K, NS, SEP, MINB, PUSH>, grid, S::NTHREADS,
                      S::SMEM, st, tm, p);
}

template <int K, int NS, bool SEP, int MINB>
void register_patch() {
    using S = PatchShape<K, NS, SEP>;
    if constexpr (S::SMEM * MINB <= 227 * 1024) {
        StepVariant v;
        v.K = K; v.TXV = 16; v.TY = 14; v.NST = NS; v.sep = SEP; v.dual = true; v.rotate = false;
        v.patch = true;
        v.tile_x = S::TX; v.tile_y = 14; v.box_w = S::SW; v.box_h = S::SH; v.halo_x = S::KP;
        v.nthreads = S::NTHREADS; v.smem = S::SMEM;
        v.func = reinterpret_cast<const void*>(&acoustic_step_patch_kernel<K, NS, SEP, MINB>);
        v.launch = &launch_patch<K, NS, SEP, MINB>;
        v.func_push = reinterpret_cast<const void*>(&acoustic_step_patch_kernel<K, NS, SEP, MINB, true>);
        v.launch_push = &launch_patch<K, NS, SEP, MINB, true>;
        step_variant_registry().push_back(v);
    }
}

template <int K, int NS, bool SEP, int TYT, bool PUSH = false>
cudaError_t launch_tall(const StepMaps& tm, const StepParams& p, dim3 grid, cudaStream_t st) {
    using S = TallShape<K, NS, SEP, TYT>;
    return launch_pdl(&acoustic_step_tall_kernel<K, NS, SEP, PUSH, TYT>, grid, S::NTHREADS, S::SMEM,
                      st, tm, p);
}

template <int K, int NS, bool SEP, int TYT = 14>
void register_tall() {
    using S = TallShape<K, NS, SEP, TYT>;
    if constexpr (S::SMEM <= 227 * 1024) {
        StepVariant v;
        v.K = K; v.TXV = 16; v.TY = 2 * TYT; v.NST = NS; v.sep = SEP; v.dual = true; v.rotate = false;
        v.tall = true;
        v.tile_x = S::TX; v.tile_y = 2 * TYT; v.box_w = S::SW; v.box_h = S::SH; v.halo_x = S::KP;
        v.nthreads = S::NTHREADS; v.smem = S::SMEM;
        v.func = reinterpret_cast<const void*>(&acoustic_step_tall_kernel<K, NS, SEP, false, TYT>);
        v.launch = &launch_tall<K, NS, SEP, TYT>;
        v.func_push = reinterpret_cast<const void*>(&acoustic_step_tall_kernel<K, NS, SEP, true, TYT>);
        v.launch_push = &launch_tall<K, NS, SEP, TYT, true>;
        step_variant_registry().push_back(v);
    }
}

template <int K, int TXV, int TY, int NST>
void register_pair() {
    register_step<K, TXV, TY, NST, false>();
    register_step<K, TXV, TY, NST, true>();
}

template <int K, int TXV, int TY, int NS>
void register_dual_pair() {
    // ask for as many resident blocks as the register file can hold with the queue of this K
    constexpr int MINB = K <= 4 ? 3 : 2;
    register_dual<K, TXV, TY, NS, false, MINB>();
    register_dual<K, TXV, TY, NS, true, MINB>();
}

template <int K, int TXV, int TY, int NS>
void register_rotated_pair() {
    constexpr int MINB = K <= 4 ? 3 : 2;
    register_dual<K, TXV, TY, NS, false, MINB, true>();
    register_dual<K, TXV, TY, NS, true, MINB, true>();
}

// the tile shapes built for every half-order K (dense and separable damping); the first
// entry is the default, sfb_set_tile / sfb_autotune pick among the rest
template <int K>
void register_all_for_K() {
    register_pair<K, 16, 16, K + 3>();
    register_pair<K, 16, 16, K + 4>();
    register_pair<K, 32, 8, K + 3>();
    register_pair<K, 16, 32, K + 3>();
    register_pair<K, 32, 16, K + 3>();
    register_dual_pair<K, 16, 16, 3>();
    register_dual_pair<K, 16, 16, 4>();
    // 14 rows: 7 consumer warps + the producer = 8 warps, so two resident blocks get 128
    // registers per thread where the 9-warp 16-row block is capped at 96 (the register file
    // is allocated in units of 4 warps); pays from order 14 up (order 16: +11 %)
    if constexpr (K >= 7) register_dual_pair<K, 16, 14, 4>();
    register_dual_pair<K, 32, 8, 3>();
    // 2 x 2 patches per thread: half the shared-memory wavefronts of the d1 part (orders >= 12)
    if constexpr (K >= 5) {   // sliding queue window: half the register moves per plane
        register_slide<K, 16, K >= 7 ? 14 : 16, 4, false, 2>();
        register_slide<K, 16, K >= 7 ? 14 : 16, 4, true, 2>();
    }
    if constexpr (K >= 6) {
        register_patch<K, 4, false, 2>();
        register_patch<K, 4, true, 2>();
    }
    // two rows of four nodes per thread: 15 LDS.128 per four nodes instead of 23 at order 16
    if constexpr (K >= 7) {
        register_tall<K, 4, false>();
        register_tall<K, 4, true>();
    }
    if constexpr (K <= 4) {  // unrolling by 2K+1 overflows the instruction cache above
        register_rotated_pair<K, 16, 16, 3>();
    }
}

struct VariantRegistrar {
    explicit VariantRegistrar(void (*fn)()) { fn(); }
};

}  // namespace sfb

#define SFB_INSTANTIATE_K(KVAL) \
    static sfb::VariantRegistrar sfb_registrar_##KVAL(&sfb::register_all_for_K<KVAL>);
