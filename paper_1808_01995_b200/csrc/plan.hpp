// plan.hpp -- host-side state behind an sfb_plan handle.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfb200.h"
#include "acoustic_kernel.cuh"
#include "tti_variants.hpp"
#include "variants.hpp"

namespace sfb {

struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SFB_CUDA(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw sfb::Failure(SFB_ERR_CUDA, std::string(#expr) + ": " +                \
                                                 cudaGetErrorString(e_));               \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void alloc(size_t n, bool zero = true) {
        if (n > bytes || !p) {
            release();
            if (n == 0) n = 16;
            cudaError_t e = cudaMalloc(&p, n);
            if (e != cudaSuccess)
                throw Failure(SFB_ERR_CUDA, "cudaMalloc of " + std::to_string(n) +
                                                " bytes: " + cudaGetErrorString(e));
            bytes = n;
        }
        if (zero) {
            SFB_CUDA(cudaMemsetAsync(p, 0, bytes, cudaStreamPerThread));
            SFB_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
        }
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Pinned host staging for trace traffic: two halves so a transfer overlaps the host-side
// f32<->f64 repacking of the previous chunk.
struct PinnedStage {
    float* p[2] = {nullptr, nullptr};
    size_t floats = 0;  // per half
    cudaStream_t copy = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, moved[2] = {nullptr, nullptr};
    PinnedStage() = default;
    PinnedStage(const PinnedStage&) = delete;
    PinnedStage& operator=(const PinnedStage&) = delete;
    ~PinnedStage() {
        for (int i = 0; i < 2; ++i) {
            if (p[i]) cudaFreeHost(p[i]);
            if (ready[i]) cudaEventDestroy(ready[i]);
            if (moved[i]) cudaEventDestroy(moved[i]);
        }
        if (copy) cudaStreamDestroy(copy);
    }
    void ensure(size_t n) {
        if (!copy) {
            SFB_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                SFB_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
                SFB_CUDA(cudaEventCreateWithFlags(&moved[i], cudaEventDisableTiming));
            }
        }
        if (n <= floats) return;
        for (int i = 0; i < 2; ++i) {
            if (p[i]) cudaFreeHost(p[i]);
            p[i] = nullptr;
            SFB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p[i]), n * sizeof(float),
                                   cudaHostAllocDefault));
        }
        floats = n;
    }
};

// One sparse point cloud (sources or receivers) in both of its roles.
struct Cloud {
    long long np = 0;
    bool set = false;
    std::vector<long long> base;  // [np][ndim] global
    std::vector<double> w;        // [np][2^ndim]
    // scatter role (CSR by destination node, nodes sorted by compact index)
    long long ncell = 0, nent = 0;
    long long cell_lo_end = 0, cell_hi_begin = 0;  // nodes in the low / high boundary planes
    DevBuf cell_start, cell_u, cell_c, ent_point, ent_w;
    std::vector<int> h_cell_start;
    // gather role
    DevBuf smp_idx, smp_w;
    // traces, fp32 [nt][np]
    DevBuf tr_in, tr_out;
    bool has_in = false;
};

struct Plan {
    sfb_plan_desc desc{};
    int K = 0;
    int ndim = 0;
    long long N[3] = {1, 1, 1};   // embedded global extents
    double h[3] = {1, 1, 1};
    bool act[3] = {false, false, false};
    long long z_lo = 0, z_hi = 0; // owned planes of embedded axis 0
    int n0 = 0;                   // owned plane count
    int pitch = 0;
    long long plane = 0;          // floats per plane
    long long ucount = 0;         // floats per wavefield buffer (with ghost planes)
    long long ccount = 0;         // floats per compact array
    double w2[kMaxK + 1] = {0};
    StencilCoef coef{};

    int device = 0;
    int sm_count = 0;
    cudaStream_t s_main = nullptr, s_bnd = nullptr;
    bool own_streams = true;
    cudaEvent_t ev_main = nullptr, ev_bnd = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    // fused halo push (sfb_link_peers): the neighbours' wavefield buffers by level parity,
    // offset to the ghost planes this slab fills, and the event that closes a boundary
    // half-step (the neighbours wait on it before their next step)
    float* peer_lo[2] = {nullptr, nullptr};
    float* peer_hi[2] = {nullptr, nullptr};
    cudaEvent_t ev_push = nullptr;
    // ... and the event that closes the interior half-step, whose gather is the last reader
    // of this slab's ghost planes of the current level: a neighbour may overwrite them (the
    // push of its next boundary half-step) only after it
    cudaEvent_t ev_done = nullptr;
    // TTI pair on linked slabs: the neighbours' ghost planes of g(p), g(r) (one buffer per
    // field) and of r (by level parity; those of p are peer_lo / peer_hi), and the event that
    // closes the first pass of a step (the neighbours' second pass waits on it)
    float* peer_g_lo[2] = {nullptr, nullptr};
    float* peer_g_hi[2] = {nullptr, nullptr};
    float* peer_r_lo[2] = {nullptr, nullptr};
    float* peer_r_hi[2] = {nullptr, nullptr};
    cudaEvent_t ev_g = nullptr;
    // neighbours in other processes (sfb_peer_export / sfb_link_peers_ipc): their buffers are
    // mapped through CUDA IPC, and the boundary half-steps are counted in a device word per
    // plan that the neighbours' streams wait on (stream memory operations: no host handshake)
    DevBuf push_flag;                    // [0]: boundary half-steps completed since linking,
                                         // [1]: interior half-steps (ghost-plane readers done)
    unsigned push_count = 0, done_count = 0, g_count = 0;   // g: word [2], TTI first passes
    void* ipc_u[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [lo/hi][parity], opened
    void* ipc_g[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [lo/hi][field]
    void* ipc_r[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [lo/hi][parity]
    void* ipc_flag[2] = {nullptr, nullptr};                         // [lo/hi], opened
    bool main_pending = false, bnd_pending = false;

    DevBuf u[2], r, damp, dz, dy, dx, grad, snaps, flag;
    CUtensorMap tm_u[2], tm_o[2], tm_r, tm_d;  // halo box on u[b]; plain box on u[b], r, damp
    bool model_set = false, sep = false;
    bool force_dense_damp = false;              // keep streaming the dense damp array
    double v_max = 0;

    Cloud cloud[2];
    PinnedStage stage;
    PinnedStage stage_in;   // rows fed to the injected cloud while a run is under way

    // TTI operator state (builder-defined formulation, csrc/tti_kernels.cuh)
    bool tti_set = false;
    DevBuf t_r[2], t_a, t_b, t_c, t_e1, t_e2, t_lp;  // p lives in u[2]; t_lp = L(p)
    DevBuf t_g[2], t_bg[2];             // g and b g of p and r between the two passes
    const TtiVariant* tti_variant = nullptr;
    // tensor maps for the TTI tile: wavefield-layout fields (haloed / plain box) ...
    enum { TF_P0, TF_P1, TF_R0, TF_R1, TF_A, TF_B, TF_C, TF_COUNT };
    CUtensorMap tt_halo[TF_COUNT], tt_plain[TF_COUNT];
    CUtensorMap tt_g[2], tt_bg[2], tt_gx[2], tt_cx;   // plain / d1-haloed / d2-haloed boxes
    // ... and compact fields (plain box)
    enum { TC_RM, TC_E1, TC_E2, TC_LP, TC_DAMP, TC_COUNT };
    CUtensorMap tt_c[TC_COUNT];
    double w1[kMaxK + 1] = {0};                             // first-derivative weights
    int tti_chunk[2] = {0, 0};                              // d0 chunk of the two launches

    const StepVariant* variant = nullptr;       // chosen tile shape
    int chunk = 0;                              // output planes per block

    // checkpointed history (recompute strategy): levels (kC-1, kC) of
    // the forward run for every segment start, a second wavefield pair for the recomputed
    // forward segment, and the levels of one segment
    DevBuf f[2], ckpt, seg;
    CUtensorMap tm_fu[2], tm_fo[2];
    long long ckpt_every = 0, nseg = 0;
    bool ckpt_valid = false;

    // history of the last forward run
    long long save_every = 0, nslots = 0;
    bool history_valid = false;
    long long live_level[2] = {-1, -1};         // time level held by u[0], u[1]
    long long step_save_every = 0;              // save_every of the op being stepped
    long launches = 0;

    std::string err;
};

}  // namespace sfb

struct sfb_plan_s : sfb::Plan {};
