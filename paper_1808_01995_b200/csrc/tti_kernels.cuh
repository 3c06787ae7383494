// tti_kernels.cuh -- TTI (tilted transverse isotropy) pseudo-acoustic forward step, sm_100a.
//
// The reference has no anisotropic operator; this is the builder's
// formulation:
//   m p_tt + damp p_t = (1+2 eps) H0(p) + sqrt(1+2 delta) Hz(r)
//   m r_tt + damp r_t = sqrt(1+2 delta) H0(p) + Hz(r)
//   g(f)  = a D0 f + b D1 f + c D2 f,   (a,b,c) = (sin th cos ph, sin th sin ph, cos th)
//   Hz(f) = D0(a g) + D1(b g) + D2(c g) = -Dbar^T Dbar f,     H0 = L - Hz
// with D_i the centred order-k first derivative and L the acoustic order-k Laplacian, time
// stepping / damping / injection / sampling as in the acoustic operator.
//
// One time step is three launches, all streamed along d0 with TMA boxes, shared-memory
// stage rings and register queues exactly like the acoustic kernel (acoustic_kernel.cuh):
//   1. tti_rot_kernel: g(p), g(r), written as the products a g, b g, c g
//   2. tti_div_kernel: Hz(p), Hz(r), each product differentiated along its own axis
//   3. tti_update_kernel: L(p), the two right-hand sides and both leapfrog updates
// In the rot kernels the two fields are handled by two groups of consumer warps of the same
// block ("field-parallel warps"): each thread carries the d0 queue of ONE field, and both
// groups share the boxes of the symmetry-axis components.  The intermediates g and Hz go
// through HBM (28 + 28 + 44 = 100 bytes per node against the 48 of a fully fused kernel);
// keeping them on chip needs a (2K+1)-plane ring of a haloed region per field, which does
// not fit in 227 KB at order 12 -- see DESIGN.md section 3.4 for the arithmetic.
#pragma once

#include <cuda_runtime.h>

#include "acoustic_kernel.cuh"

namespace sfb {

struct TtiCoef {
    float c0;                                  // Laplacian centre weight * sum 1/h^2
    float lx[kMaxK], ly[kMaxK], lz[kMaxK];     // Laplacian weights / h^2 per axis
    float fx[kMaxK], fy[kMaxK], fz[kMaxK];     // first-derivative weights / h per axis
    float qscale;                              // 1/(2 dt)
};

// ---- pass 1: g(f) = a D0 f + b D1 f + c D2 f, stored as the three products -------------

struct RotMaps {
    CUtensorMap f0_feed, f1_feed, f0_ctr, f1_ctr;  // the two input fields: plain / haloed box
    CUtensorMap a, b, c;                           // axis components, plain box
};

struct RotParams {
    TtiCoef k;
    float* ag[2];       // a g, b g, c g of field 0 / field 1 (wavefield layout)
    float* bg[2];
    float* cg[2];
    long long out_off;  // element offset of local plane 0 inside the outputs
    int N1, N2, pitch;
    long long plane;
    int z_lo, z_hi, chunk;
};

template <int K, int TXV, int TY, int NS>
struct RotShape {
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;
    static constexpr int SH = TY + 2 * K;
    static constexpr int CBOX = SW * SH;
    static constexpr int CPAD = ((CBOX + 31) / 32) * 32;
    static constexpr int ABOX = TX * TY;
    // stage: feed f0,f1 | centre f0,f1 | plain a,b,c
    static constexpr int STAGE = 2 * ABOX + 2 * CPAD + 3 * ABOX;
    static constexpr int GROUP = TXV * TY;            // consumer threads per field
    static constexpr int NTHREADS = 2 * GROUP + 32;
    static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8 + 128;
    static_assert(GROUP % 32 == 0 && (ABOX * 4) % 128 == 0, "tile shape");
};

template <int K, int TXV, int TY, int NS>
__global__ void __launch_bounds__(RotShape<K, TXV, TY, NS>::NTHREADS)
tti_rot_kernel(const __grid_constant__ RotMaps tm, const __grid_constant__ RotParams p) {
    using S = RotShape<K, TXV, TY, NS>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int ABOX = S::ABOX, CPAD = S::CPAD, TX = S::TX;
    constexpr int NCW = 2 * S::GROUP / 32;
    constexpr int OFF_CTR = 2 * ABOX;
    constexpr int OFF_PLAIN = OFF_CTR + 2 * CPAD;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
    uint64_t* done = full + NS;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk;
    const int ze = min(zb + p.chunk, p.z_hi);
    const int nplanes = (ze - zb) + 2 * K;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(done + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= 2 * S::GROUP) {
        if (tid == 2 * S::GROUP) {
            int s = 0;
            uint32_t dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NS) mbar_wait(done + s, dph);
                const bool out = n >= 2 * K;
                float* st = ring + s * STAGE;
                const int feed_b = 2 * ABOX, rest_b = 2 * S::CBOX + 3 * ABOX;
                mbar_arrive_expect_tx(full + s, (feed_b + (out ? rest_b : 0)) * 4);
                // every field lives in the wavefield layout: buffer plane = local plane + K
                tma_load_3d(st, &tm.f0_feed, x0, y0, zb + n, full + s);
                tma_load_3d(st + ABOX, &tm.f1_feed, x0, y0, zb + n, full + s);
                if (out) {
                    const int zc = zb + n - K;  // centre plane (buffer index)
                    tma_load_3d(st + OFF_CTR, &tm.f0_ctr, x0 - KP, y0 - K, zc, full + s);
                    tma_load_3d(st + OFF_CTR + CPAD, &tm.f1_ctr, x0 - KP, y0 - K, zc, full + s);
                    tma_load_3d(st + OFF_PLAIN, &tm.a, x0, y0, zc, full + s);
                    tma_load_3d(st + OFF_PLAIN + ABOX, &tm.b, x0, y0, zc, full + s);
                    tma_load_3d(st + OFF_PLAIN + 2 * ABOX, &tm.c, x0, y0, zc, full + s);
                }
                if (++s == NS) {
                    s = 0;
                    if (n >= NS) dph ^= 1;
                }
            }
        }
        return;
    }

    // ---- consumers: group 0 differentiates field 0, group 1 field 1 ----------------------
    const int field = tid / S::GROUP;
    const int lt = tid - field * S::GROUP;
    const int tx = lt % TXV, ty = lt / TXV;
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool rin = x < p.N2 && y < p.N1;
    const bool lane0 = (tid & 31) == 0;
    long long go = p.out_off + (long long)zb * p.plane + (long long)y * p.pitch + x;
    float* const oa = p.ag[field];
    float* const ob = p.bg[field];
    float* const oc = p.cg[field];

    float q[Q][4];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int aown = ty * TX + 4 * tx;
    int s = 0;
    uint32_t fph = 0;
    for (int n = 0; n < nplanes; ++n) {
        mbar_wait(full + s, fph);
        const float* st = ring + s * STAGE;
        {
            const float4 v = *reinterpret_cast<const float4*>(st + field * ABOX + aown);
#pragma unroll
            for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) q[j][c] = q[j + 1][c];
            q[Q - 1][0] = v.x;
            q[Q - 1][1] = v.y;
            q[Q - 1][2] = v.z;
            q[Q - 1][3] = v.w;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release(done + s, q[Q - 1][0]);
        } else {
            const float* cp = st + OFF_CTR + field * CPAD;  // haloed centre box of this field
            float d0[4], d1[4], d2[4];
            {   // d0 from the register queue, two nodes per instruction
                float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 1; j <= K; ++j) {
                    const float2 w = f2_splat(p.k.fz[j - 1]);
                    a01 = f2_fma(w, f2_sub(make_float2(q[K + j][0], q[K + j][1]),
                                           make_float2(q[K - j][0], q[K - j][1])), a01);
                    a23 = f2_fma(w, f2_sub(make_float2(q[K + j][2], q[K + j][3]),
                                           make_float2(q[K - j][2], q[K - j][3])), a23);
                }
                d0[0] = a01.x;
                d0[1] = a01.y;
                d0[2] = a23.x;
                d0[3] = a23.y;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) d2[c] = 0.f;
            {   // d2: one aligned row segment
                float xr[2 * KP + 4];
                const float* rowp = cp + (ty + K) * SW + 4 * tx;
#pragma unroll
                for (int v = 0; v < (2 * KP + 4) / 4; ++v) {
                    const float4 t4 = *reinterpret_cast<const float4*>(rowp + 4 * v);
                    xr[4 * v + 0] = t4.x;
                    xr[4 * v + 1] = t4.y;
                    xr[4 * v + 2] = t4.z;
                    xr[4 * v + 3] = t4.w;
                }
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 1; j <= K; ++j)
                        d2[c] = fmaf(p.k.fx[j - 1], xr[KP + c + j] - xr[KP + c - j], d2[c]);
            }
            {   // d1: column strip above and below (register-aligned pairs: packed)
                const float* colp = cp + ty * SW + KP + 4 * tx;
                float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 1; j <= K; ++j) {
                    const float4 lo = *reinterpret_cast<const float4*>(colp + (K - j) * SW);
                    const float4 hi = *reinterpret_cast<const float4*>(colp + (K + j) * SW);
                    const float2 w = f2_splat(p.k.fy[j - 1]);
                    a01 = f2_fma(w, f2_sub(make_float2(hi.x, hi.y), make_float2(lo.x, lo.y)), a01);
                    a23 = f2_fma(w, f2_sub(make_float2(hi.z, hi.w), make_float2(lo.z, lo.w)), a23);
                }
                d1[0] = a01.x;
                d1[1] = a01.y;
                d1[2] = a23.x;
                d1[3] = a23.y;
            }
            const float* np = st + OFF_PLAIN + aown;
            const float4 a4 = *reinterpret_cast<const float4*>(np);
            const float4 b4 = *reinterpret_cast<const float4*>(np + ABOX);
            const float4 c4 = *reinterpret_cast<const float4*>(np + 2 * ABOX);
            float g[4];
            g[0] = fmaf(a4.x, d0[0], fmaf(b4.x, d1[0], c4.x * d2[0]));
            g[1] = fmaf(a4.y, d0[1], fmaf(b4.y, d1[1], c4.y * d2[1]));
            g[2] = fmaf(a4.z, d0[2], fmaf(b4.z, d1[2], c4.z * d2[2]));
            g[3] = fmaf(a4.w, d0[3], fmaf(b4.w, d1[3], c4.w * d2[3]));
            // g[0] depends on every shared-memory load of the iteration (see mbar_release)
            __syncwarp();
            if (lane0) mbar_release(done + s, g[0]);
            if (rin) {
                // the second pass differentiates each product along one axis only
                __stcs(reinterpret_cast<float4*>(oa + go),
                       make_float4(a4.x * g[0], a4.y * g[1], a4.z * g[2], a4.w * g[3]));
                __stcs(reinterpret_cast<float4*>(ob + go),
                       make_float4(b4.x * g[0], b4.y * g[1], b4.z * g[2], b4.w * g[3]));
                __stcs(reinterpret_cast<float4*>(oc + go),
                       make_float4(c4.x * g[0], c4.y * g[1], c4.z * g[2], c4.w * g[3]));
            }
            go += p.plane;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
    }
}

// ---- pass 2: Hz(f) = D0(a g) + D1(b g) + D2(c g) ------------------------------------------

struct DivMaps {
    CUtensorMap ag0, ag1;   // plain box (feeds the d0 queue)
    CUtensorMap bg0, bg1;   // box with a d1 halo only
    CUtensorMap cg0, cg1;   // box with a d2 halo only
};

struct DivParams {
    TtiCoef k;
    float* out0;        // Hz of field 0 / field 1 (compact layout)
    float* out1;
    int N1, N2, pitch;
    long long plane;
    int z_lo, z_hi, chunk;
};

template <int K, int TXV, int TY, int NS>
struct DivShape {
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;
    static constexpr int SH = TY + 2 * K;
    static constexpr int ABOX = TX * TY;
    static constexpr int YBOX = TX * SH;            // d1-haloed box
    static constexpr int XBOX = SW * TY;            // d2-haloed box
    static constexpr int XPAD = ((XBOX + 31) / 32) * 32;
    // stage: feed ag0, ag1 | bg0, bg1 | cg0, cg1
    static constexpr int STAGE = 2 * ABOX + 2 * YBOX + 2 * XPAD;
    static constexpr int GROUP = TXV * TY;
    static constexpr int NTHREADS = 2 * GROUP + 32;
    static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8 + 128;
    static_assert(GROUP % 32 == 0 && (ABOX * 4) % 128 == 0 && (YBOX * 4) % 128 == 0, "tile shape");
};

template <int K, int TXV, int TY, int NS>
__global__ void __launch_bounds__(DivShape<K, TXV, TY, NS>::NTHREADS)
tti_div_kernel(const __grid_constant__ DivMaps tm, const __grid_constant__ DivParams p) {
    using S = DivShape<K, TXV, TY, NS>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int ABOX = S::ABOX, YBOX = S::YBOX, XPAD = S::XPAD, TX = S::TX;
    constexpr int NCW = 2 * S::GROUP / 32;
    constexpr int OFF_Y = 2 * ABOX, OFF_X = OFF_Y + 2 * YBOX;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
    uint64_t* done = full + NS;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk;
    const int ze = min(zb + p.chunk, p.z_hi);
    const int nplanes = (ze - zb) + 2 * K;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(done + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= 2 * S::GROUP) {
        if (tid == 2 * S::GROUP) {
            int s = 0;
            uint32_t dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NS) mbar_wait(done + s, dph);
                const bool out = n >= 2 * K;
                float* st = ring + s * STAGE;
                mbar_arrive_expect_tx(full + s,
                                      (2 * ABOX + (out ? 2 * YBOX + 2 * S::XBOX : 0)) * 4);
                tma_load_3d(st, &tm.ag0, x0, y0, zb + n, full + s);
                tma_load_3d(st + ABOX, &tm.ag1, x0, y0, zb + n, full + s);
                if (out) {
                    const int zc = zb + n - K;  // centre plane (buffer index)
                    tma_load_3d(st + OFF_Y, &tm.bg0, x0, y0 - K, zc, full + s);
                    tma_load_3d(st + OFF_Y + YBOX, &tm.bg1, x0, y0 - K, zc, full + s);
                    tma_load_3d(st + OFF_X, &tm.cg0, x0 - KP, y0, zc, full + s);
                    tma_load_3d(st + OFF_X + XPAD, &tm.cg1, x0 - KP, y0, zc, full + s);
                }
                if (++s == NS) {
                    s = 0;
                    if (n >= NS) dph ^= 1;
                }
            }
        }
        return;
    }

    const int field = tid / S::GROUP;
    const int lt = tid - field * S::GROUP;
    const int tx = lt % TXV, ty = lt / TXV;
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool rin = x < p.N2 && y < p.N1;
    const bool lane0 = (tid & 31) == 0;
    float* outp = (field ? p.out1 : p.out0) + (long long)zb * p.plane + (long long)y * p.pitch + x;

    float q[Q][4];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int aown = ty * TX + 4 * tx;
    int s = 0;
    uint32_t fph = 0;
    for (int n = 0; n < nplanes; ++n) {
        mbar_wait(full + s, fph);
        const float* st = ring + s * STAGE;
        {
            const float4 v = *reinterpret_cast<const float4*>(st + field * ABOX + aown);
#pragma unroll
            for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) q[j][c] = q[j + 1][c];
            q[Q - 1][0] = v.x;
            q[Q - 1][1] = v.y;
            q[Q - 1][2] = v.z;
            q[Q - 1][3] = v.w;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release(done + s, q[Q - 1][0]);
        } else {
            float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 1; j <= K; ++j) {   // D0 (a g): register queue
                const float2 w = f2_splat(p.k.fz[j - 1]);
                a01 = f2_fma(w, f2_sub(make_float2(q[K + j][0], q[K + j][1]),
                                       make_float2(q[K - j][0], q[K - j][1])), a01);
                a23 = f2_fma(w, f2_sub(make_float2(q[K + j][2], q[K + j][3]),
                                       make_float2(q[K - j][2], q[K - j][3])), a23);
            }
            {   // D1 (b g): rows above and below in the d1-haloed box
                const float* colp = st + OFF_Y + field * YBOX + ty * TX + 4 * tx;
#pragma unroll
                for (int j = 1; j <= K; ++j) {
                    const float4 lo = *reinterpret_cast<const float4*>(colp + (K - j) * TX);
                    const float4 hi = *reinterpret_cast<const float4*>(colp + (K + j) * TX);
                    const float2 w = f2_splat(p.k.fy[j - 1]);
                    a01 = f2_fma(w, f2_sub(make_float2(hi.x, hi.y), make_float2(lo.x, lo.y)), a01);
                    a23 = f2_fma(w, f2_sub(make_float2(hi.z, hi.w), make_float2(lo.z, lo.w)), a23);
                }
            }
            float d2[4] = {0.f, 0.f, 0.f, 0.f};
            {   // D2 (c g): one aligned row segment of the d2-haloed box
                float xr[2 * KP + 4];
                const float* rowp = st + OFF_X + field * XPAD + ty * SW + 4 * tx;
#pragma unroll
                for (int v = 0; v < (2 * KP + 4) / 4; ++v) {
                    const float4 t4 = *reinterpret_cast<const float4*>(rowp + 4 * v);
                    xr[4 * v + 0] = t4.x;
                    xr[4 * v + 1] = t4.y;
                    xr[4 * v + 2] = t4.z;
                    xr[4 * v + 3] = t4.w;
                }
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 1; j <= K; ++j)
                        d2[c] = fmaf(p.k.fx[j - 1], xr[KP + c + j] - xr[KP + c - j], d2[c]);
            }
            float o[4];
            o[0] = a01.x + d2[0];
            o[1] = a01.y + d2[1];
            o[2] = a23.x + d2[2];
            o[3] = a23.y + d2[3];
            // o[0] depends on every shared-memory load of the iteration (see mbar_release)
            __syncwarp();
            if (lane0) mbar_release(done + s, o[0]);
            if (rin) __stcs(reinterpret_cast<float4*>(outp), make_float4(o[0], o[1], o[2], o[3]));
            outp += p.plane;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
    }
}

#ifndef SFB_TTI_UPD_MINB
#define SFB_TTI_UPD_MINB 1   // (2 with a 2-stage ring was tried: spills at high order, no gain)
#endif

// ---- update: L(p), right-hand sides, leapfrog of p and r -----------------------------------

struct UpdMaps {
    CUtensorMap p_feed, p_ctr;               // u[t] = p: plain / haloed box
    CUtensorMap po, ro, rc, rm, e1, e2, hzp, hzr, d;  // plain boxes of the output plane
};

struct UpdParams {
    TtiCoef k;
    const float *dz, *dy, *dx;   // separable damping profiles
    float* po;                   // p level being overwritten (ghost planes)
    float* ro;                   // r level being overwritten
    int N1, N2, pitch;
    long long plane;
    int z_lo, z_hi, chunk;
};

template <int K, int TXV, int TY, int NS, bool SEP>
struct UpdShape {
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;
    static constexpr int SH = TY + 2 * K;
    static constexpr int CBOX = SW * SH;
    static constexpr int CPAD = ((CBOX + 31) / 32) * 32;
    static constexpr int ABOX = TX * TY;
    static constexpr int NARR = SEP ? 8 : 9;   // po ro rc rm e1 e2 hzp hzr (damp)
    static constexpr int STAGE = ABOX + CPAD + NARR * ABOX;
    static constexpr int NCONS = TXV * TY;
    static constexpr int NTHREADS = NCONS + 32;
    static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8 + 128;
};

template <int K, int TXV, int TY, int NS, bool SEP>
__global__ void __launch_bounds__(UpdShape<K, TXV, TY, NS, SEP>::NTHREADS, SFB_TTI_UPD_MINB)
tti_update_kernel(const __grid_constant__ UpdMaps tm, const __grid_constant__ UpdParams p) {
    using S = UpdShape<K, TXV, TY, NS, SEP>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int NARR = S::NARR, ABOX = S::ABOX, CPAD = S::CPAD, TX = S::TX;
    constexpr int NCW = S::NCONS / 32;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
    uint64_t* done = full + NS;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk;
    const int ze = min(zb + p.chunk, p.z_hi);
    const int nplanes = (ze - zb) + 2 * K;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(done + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= S::NCONS) {
        if (tid == S::NCONS) {
            int s = 0;
            uint32_t dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NS) mbar_wait(done + s, dph);
                const bool out = n >= 2 * K;
                float* st = ring + s * STAGE;
                mbar_arrive_expect_tx(full + s, (ABOX + (out ? S::CBOX + NARR * ABOX : 0)) * 4);
                tma_load_3d(st, &tm.p_feed, x0, y0, zb + n, full + s);
                if (out) {
                    const int zo = zb + n - 2 * K;   // local output plane; buffer plane zo + K
                    tma_load_3d(st + ABOX, &tm.p_ctr, x0 - KP, y0 - K, zo + K, full + s);
                    float* ad = st + ABOX + CPAD;
                    tma_load_3d(ad + 0 * ABOX, &tm.po, x0, y0, zo + K, full + s);
                    tma_load_3d(ad + 1 * ABOX, &tm.ro, x0, y0, zo + K, full + s);
                    tma_load_3d(ad + 2 * ABOX, &tm.rc, x0, y0, zo + K, full + s);
                    tma_load_3d(ad + 3 * ABOX, &tm.rm, x0, y0, zo, full + s);
                    tma_load_3d(ad + 4 * ABOX, &tm.e1, x0, y0, zo, full + s);
                    tma_load_3d(ad + 5 * ABOX, &tm.e2, x0, y0, zo, full + s);
                    tma_load_3d(ad + 6 * ABOX, &tm.hzp, x0, y0, zo, full + s);
                    tma_load_3d(ad + 7 * ABOX, &tm.hzr, x0, y0, zo, full + s);
                    if (!SEP) tma_load_3d(ad + 8 * ABOX, &tm.d, x0, y0, zo, full + s);
                }
                if (++s == NS) {
                    s = 0;
                    if (n >= NS) dph ^= 1;
                }
            }
        }
        return;
    }

    const int tx = tid % TXV, ty = tid / TXV;
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool rin = x < p.N2 && y < p.N1;
    const bool lane0 = (tid & 31) == 0;
    float dxy[4] = {0.f, 0.f, 0.f, 0.f};
    if (SEP && rin) {
        const float4 dx4 = __ldg(reinterpret_cast<const float4*>(p.dx + x));
        const float dyv = __ldg(p.dy + y);
        dxy[0] = dx4.x + dyv;
        dxy[1] = dx4.y + dyv;
        dxy[2] = dx4.z + dyv;
        dxy[3] = dx4.w + dyv;
    }
    float q[Q][4];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    StencilCoef lk;
    lk.c0 = p.k.c0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        lk.cx[j] = p.k.lx[j];
        lk.cy[j] = p.k.ly[j];
        lk.cz[j] = p.k.lz[j];
    }

    const int aown = ty * TX + 4 * tx;
    const long long g0 = (long long)(zb + K) * p.plane + (long long)y * p.pitch + x;
    float* pp = p.po + g0;
    float* rp = p.ro + g0;
    int s = 0;
    uint32_t fph = 0;
    for (int n = 0; n < nplanes; ++n) {
        mbar_wait(full + s, fph);
        const float* st = ring + s * STAGE;
        {
            const float4 v = *reinterpret_cast<const float4*>(st + aown);
#pragma unroll
            for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) q[j][c] = q[j + 1][c];
            q[Q - 1][0] = v.x;
            q[Q - 1][1] = v.y;
            q[Q - 1][2] = v.z;
            q[Q - 1][3] = v.w;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release(done + s, q[Q - 1][0]);
        } else {
            const float* ap = st + ABOX + CPAD + aown;
            float a[NARR][4];
#pragma unroll
            for (int i = 0; i < NARR; ++i) {
                const float4 v = *reinterpret_cast<const float4*>(ap + i * ABOX);
                a[i][0] = v.x;
                a[i][1] = v.y;
                a[i][2] = v.z;
                a[i][3] = v.w;
            }
            float dzv = 0.f;
            if (SEP) dzv = __ldg(p.dz + (zb + n - 2 * K));
            float lap[4];
            stencil_acc<K, KP, SW>(lk, q, st + ABOX, tx, ty, lap);
            float pn[4], rn[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float po = a[0][c], ro = a[1][c], rc = a[2][c], rm = a[3][c];
                const float e1 = a[4][c], e2 = a[5][c], hzp = a[6][c], hzr = a[7][c];
                const float dmp = SEP ? (dxy[c] + dzv) : a[NARR - 1][c];
                const float h0 = lap[c] - hzp;
                const float rhs_p = fmaf(e1, h0, e2 * hzr);
                const float rhs_r = fmaf(e2, h0, hzr);
                const float qq = dmp * rm * p.k.qscale;
                const float c1 = fast_rcp(1.f + qq), c2 = (1.f - qq) * c1;
                pn[c] = fmaf(c1, fmaf(rm, rhs_p, 2.f * q[K][c]), -c2 * po);
                rn[c] = fmaf(c1, fmaf(rm, rhs_r, 2.f * rc), -c2 * ro);
            }
            // pn[0] + rn[0] depends on every shared-memory load of the iteration
            __syncwarp();
            if (lane0) mbar_release(done + s, pn[0] + rn[0]);
            if (rin) {
                __stcs(reinterpret_cast<float4*>(pp), make_float4(pn[0], pn[1], pn[2], pn[3]));
                __stcs(reinterpret_cast<float4*>(rp), make_float4(rn[0], rn[1], rn[2], rn[3]));
            }
            pp += p.plane;
            rp += p.plane;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
    }
}

// set-up: unit symmetry axis and Thomsen factors from the f64 inputs
static __global__ void tti_setup_kernel(const double* __restrict__ eps, const double* __restrict__ delta,
                                 const double* __restrict__ theta, const double* __restrict__ phi,
                                 float* a, float* b, float* c, float* e1, float* e2,
                                 long long rows, int n2, int pitch, long long ghost_off) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x) {
        const long long s = row * n2 + x, d = row * pitch + x;
        double st, ct, sp, cp;
        sincos(theta[s], &st, &ct);
        sincos(phi[s], &sp, &cp);
        a[ghost_off + d] = (float)(st * cp);
        b[ghost_off + d] = (float)(st * sp);
        c[ghost_off + d] = (float)ct;
        e1[d] = (float)(1.0 + 2.0 * eps[s]);
        e2[d] = (float)sqrt(1.0 + 2.0 * delta[s]);
    }
}

}  // namespace sfb
