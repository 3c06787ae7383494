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
// One time step is two launches, both streamed along d0 with TMA boxes, shared-memory
// stage rings and register queues exactly like the acoustic kernel (acoustic_kernel.cuh):
//   1. tti_rot_kernel: g(p), g(r) -- stored as g and the product b g -- and L(p)
//   2. tti_div_update_kernel: Hz(p), Hz(r) -- each product differentiated along its own
//      axis -- the two right-hand sides and both leapfrog updates
// In both kernels the two fields are handled by two groups of consumer warps of the same
// block ("field-parallel warps"): each thread carries the d0 queue of ONE field.  The
// intermediates and L(p) go through HBM once (40 + 64 = 104 bytes per node against the 48 of a
// fully fused kernel); keeping g on chip needs a (2K+1)-plane ring of a haloed region per
// field, which does not fit in 227 KB at order 12 -- see DESIGN.md section 3.4.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

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
    float* g[2];        // g and b g of field 0 / field 1 (wavefield layout)
    float* bg[2];
    float* lp;          // L(field 0) (compact layout): its operands are all on chip here
    long long out_off;  // element offset of local plane 0 inside the outputs
    int N1, N2, pitch;
    long long plane;
    int z_lo, z_hi, chunk;
    // PUSH kernels (linked slabs, single-launch step): the first `push_planes` planes of g
    // that the edge block rows output -- block row 0 sweeping up, the last one sweeping down
    // with desc_last -- are also stored into the neighbour's ghost planes of g: distance in
    // floats from a node of g[field] to its mirror, low / high group (0 = no neighbour)
    long long peer_lo[2], peer_hi[2];
    int push_planes, desc_last;
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

template <int K, int TXV, int TY, int NS, bool PUSH = false>
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
    // sweep direction (PUSH kernels only; see acoustic_step_kernel): iteration n loads buffer
    // plane zl0 + dir n and, from n = 2K on, outputs local plane zo0 + dir (n - 2K)
    const bool desc = PUSH && p.desc_last && gridDim.z > 1 && blockIdx.z == gridDim.z - 1;
    const int dir = desc ? -1 : 1;
    const int zl0 = desc ? ze - 1 + 2 * K : zb;
    const int zo0 = desc ? ze - 1 : zb;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(done + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_enter();

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
                tma_load_3d(st, &tm.f0_feed, x0, y0, zl0 + dir * n, full + s);
                tma_load_3d(st + ABOX, &tm.f1_feed, x0, y0, zl0 + dir * n, full + s);
                if (out) {
                    const int zc = zo0 + dir * (n - 2 * K) + K;  // centre plane (buffer index)
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
    long long go = p.out_off + (long long)zo0 * p.plane + (long long)y * p.pitch + x;
    float* const og = p.g[field];
    float* const ob = p.bg[field];
    long long lo_off = (long long)zo0 * p.plane + (long long)y * p.pitch + x;   // compact
    const long long zstep = desc ? -p.plane : p.plane;
    long long peer_delta = 0;
    if constexpr (PUSH)
        peer_delta = blockIdx.z == 0 ? p.peer_lo[field]
                                     : (blockIdx.z == gridDim.z - 1 ? p.peer_hi[field] : 0);

    // the d0 queue is a sliding window of 2K+2 slots: the plane loop is unrolled by two (plane
    // n uses slots [0, 2K], plane n+1 slots [1, 2K+1]) and the window moves by two slots
    // afterwards -- half the register moves of a queue shifted every plane
    float q[Q + 1][4];
#pragma unroll
    for (int j = 0; j < Q + 1; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int aown = ty * TX + 4 * tx;
    int s = 0;
    uint32_t fph = 0;
    auto iteration = [&](auto off, int n) {
        constexpr int OFF = decltype(off)::value;
#define SFB_TQ(i) q[(i) + OFF]
        mbar_wait(full + s, fph);
        const float* st = ring + s * STAGE;
        {
            const float4 v = *reinterpret_cast<const float4*>(st + field * ABOX + aown);
            SFB_TQ(Q - 1)[0] = v.x;
            SFB_TQ(Q - 1)[1] = v.y;
            SFB_TQ(Q - 1)[2] = v.z;
            SFB_TQ(Q - 1)[3] = v.w;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release(done + s, SFB_TQ(Q - 1)[0]);
        } else {
            const float* cp = st + OFF_CTR + field * CPAD;  // haloed centre box of this field
            const float* np = st + OFF_PLAIN + aown;
            // one pass over the operands: first derivatives for g and -- for p (warp group 0)
            // -- the Laplacian from the same loads (sums instead of differences)
            auto body = [&](auto with_lap) {
                constexpr bool LAP = decltype(with_lap)::value;
                float2 g01 = make_float2(0.f, 0.f), g23 = make_float2(0.f, 0.f);   // a D0 f ...
                float2 l01 = make_float2(0.f, 0.f), l23 = make_float2(0.f, 0.f);
                const float4 a4 = *reinterpret_cast<const float4*>(np);
                const float4 b4 = *reinterpret_cast<const float4*>(np + ABOX);
                const float4 c4 = *reinterpret_cast<const float4*>(np + 2 * ABOX);
                {   // d0 from the register queue, two nodes per instruction
                    float2 d01 = make_float2(0.f, 0.f), d23 = make_float2(0.f, 0.f);
                    if (LAP) {
                        l01 = f2_mul(f2_splat(p.k.c0), make_float2(SFB_TQ(K)[0], SFB_TQ(K)[1]));
                        l23 = f2_mul(f2_splat(p.k.c0), make_float2(SFB_TQ(K)[2], SFB_TQ(K)[3]));
                    }
#pragma unroll
                    for (int j = 1; j <= K; ++j) {
                        const float2 hi01 = make_float2(SFB_TQ(K + j)[0], SFB_TQ(K + j)[1]);
                        const float2 hi23 = make_float2(SFB_TQ(K + j)[2], SFB_TQ(K + j)[3]);
                        const float2 lo01 = make_float2(SFB_TQ(K - j)[0], SFB_TQ(K - j)[1]);
                        const float2 lo23 = make_float2(SFB_TQ(K - j)[2], SFB_TQ(K - j)[3]);
                        const float2 w = f2_splat(p.k.fz[j - 1]);
                        d01 = f2_fma(w, f2_sub(hi01, lo01), d01);
                        d23 = f2_fma(w, f2_sub(hi23, lo23), d23);
                        if (LAP) {
                            const float2 wl = f2_splat(p.k.lz[j - 1]);
                            l01 = f2_fma(wl, f2_add(hi01, lo01), l01);
                            l23 = f2_fma(wl, f2_add(hi23, lo23), l23);
                        }
                    }
                    // a downward sweep holds the queue in reverse: the first derivative (odd in
                    // d0, unlike the Laplacian) comes out with the opposite sign, exactly
                    if (PUSH && desc) {
                        d01 = make_float2(-d01.x, -d01.y);
                        d23 = make_float2(-d23.x, -d23.y);
                    }
                    g01 = f2_mul(make_float2(a4.x, a4.y), d01);
                    g23 = f2_mul(make_float2(a4.z, a4.w), d23);
                }
                {   // d1: column strip above and below (register-aligned pairs: packed)
                    const float* colp = cp + ty * SW + KP + 4 * tx;
                    float2 d01 = make_float2(0.f, 0.f), d23 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 1; j <= K; ++j) {
                        const float4 lo = *reinterpret_cast<const float4*>(colp + (K - j) * SW);
                        const float4 hi = *reinterpret_cast<const float4*>(colp + (K + j) * SW);
                        const float2 w = f2_splat(p.k.fy[j - 1]);
                        d01 = f2_fma(w, f2_sub(make_float2(hi.x, hi.y), make_float2(lo.x, lo.y)), d01);
                        d23 = f2_fma(w, f2_sub(make_float2(hi.z, hi.w), make_float2(lo.z, lo.w)), d23);
                        if (LAP) {
                            const float2 wl = f2_splat(p.k.ly[j - 1]);
                            l01 = f2_fma(wl, f2_add(make_float2(hi.x, hi.y), make_float2(lo.x, lo.y)), l01);
                            l23 = f2_fma(wl, f2_add(make_float2(hi.z, hi.w), make_float2(lo.z, lo.w)), l23);
                        }
                    }
                    g01 = f2_fma(make_float2(b4.x, b4.y), d01, g01);
                    g23 = f2_fma(make_float2(b4.z, b4.w), d23, g23);
                }
                float g[4], lap[4];
                {   // d2: one aligned row segment; even j: the operand pairs are register-aligned
                    // and run packed, odd j: they straddle two pairs and stay scalar
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
                    float2 e01 = make_float2(0.f, 0.f), e23 = make_float2(0.f, 0.f);   // D2 f
                    float2 m01 = make_float2(0.f, 0.f), m23 = make_float2(0.f, 0.f);   // D22 f
#pragma unroll
                    for (int j = 1; j <= K; ++j) {
                        if (j % 2 == 0) {
                            const float2 h01 = make_float2(xr[KP + j], xr[KP + 1 + j]);
                            const float2 h23 = make_float2(xr[KP + 2 + j], xr[KP + 3 + j]);
                            const float2 o01 = make_float2(xr[KP - j], xr[KP + 1 - j]);
                            const float2 o23 = make_float2(xr[KP + 2 - j], xr[KP + 3 - j]);
                            const float2 w = f2_splat(p.k.fx[j - 1]);
                            e01 = f2_fma(w, f2_sub(h01, o01), e01);
                            e23 = f2_fma(w, f2_sub(h23, o23), e23);
                            if (LAP) {
                                const float2 wl = f2_splat(p.k.lx[j - 1]);
                                m01 = f2_fma(wl, f2_add(h01, o01), m01);
                                m23 = f2_fma(wl, f2_add(h23, o23), m23);
                            }
                        } else {
                            e01.x = fmaf(p.k.fx[j - 1], xr[KP + j] - xr[KP - j], e01.x);
                            e01.y = fmaf(p.k.fx[j - 1], xr[KP + 1 + j] - xr[KP + 1 - j], e01.y);
                            e23.x = fmaf(p.k.fx[j - 1], xr[KP + 2 + j] - xr[KP + 2 - j], e23.x);
                            e23.y = fmaf(p.k.fx[j - 1], xr[KP + 3 + j] - xr[KP + 3 - j], e23.y);
                            if (LAP) {
                                m01.x = fmaf(p.k.lx[j - 1], xr[KP + j] + xr[KP - j], m01.x);
                                m01.y = fmaf(p.k.lx[j - 1], xr[KP + 1 + j] + xr[KP + 1 - j], m01.y);
                                m23.x = fmaf(p.k.lx[j - 1], xr[KP + 2 + j] + xr[KP + 2 - j], m23.x);
                                m23.y = fmaf(p.k.lx[j - 1], xr[KP + 3 + j] + xr[KP + 3 - j], m23.y);
                            }
                        }
                    }
                    g01 = f2_fma(make_float2(c4.x, c4.y), e01, g01);
                    g23 = f2_fma(make_float2(c4.z, c4.w), e23, g23);
                    g[0] = g01.x;
                    g[1] = g01.y;
                    g[2] = g23.x;
                    g[3] = g23.y;
                    l01 = f2_add(m01, l01);
                    l23 = f2_add(m23, l23);
                    lap[0] = l01.x;
                    lap[1] = l01.y;
                    lap[2] = l23.x;
                    lap[3] = l23.y;
                }
                // g[0] (+ lap[0]) depends on every shared-memory load of the iteration
                __syncwarp();
                if (lane0) mbar_release(done + s, LAP ? g[0] + lap[0] : g[0]);
                if (rin) {
                    if (LAP)
                        __stcs(reinterpret_cast<float4*>(p.lp + lo_off),
                               make_float4(lap[0], lap[1], lap[2], lap[3]));
                    // the second pass needs b g at 2K neighbours per node (the expensive
                    // product: stored); a g and c g are rebuilt there from g
                    __stcs(reinterpret_cast<float4*>(og + go), make_float4(g[0], g[1], g[2], g[3]));
                    __stcs(reinterpret_cast<float4*>(ob + go),
                           make_float4(b4.x * g[0], b4.y * g[1], b4.z * g[2], b4.w * g[3]));
                    if constexpr (PUSH) {   // the neighbour differentiates a g along d0: g only
                        if (peer_delta && n - 2 * K < p.push_planes)
                            *reinterpret_cast<float4*>(og + go + peer_delta) =
                                make_float4(g[0], g[1], g[2], g[3]);
                    }
                }
            };
            if (field == 0)   // warp-uniform
                body(std::true_type{});
            else
                body(std::false_type{});
            lo_off += zstep;
            go += zstep;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
#undef SFB_TQ
    };
    for (int n = 0; n < nplanes; n += 2) {
        iteration(std::integral_constant<int, 0>{}, n);
        if (n + 1 < nplanes) iteration(std::integral_constant<int, 1>{}, n + 1);
#pragma unroll
        for (int j = 0; j < Q - 1; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[j][c] = q[j + 2][c];
    }
}

// ---- pass 2 + update ------------------------------------------------------------------
// Hz(f) = D0(a g) + D1(b g) + D2(c g) for f = p (warp group 0) and f = r (group 1) -- a g is
// formed when a plane of g enters the register queue, c g along the row segment -- then the
// point-wise rest of the step in the same threads: the groups swap Hz(p) / Hz(r) through
// the feed boxes of the stage they have just consumed, form the two right-hand sides from
// L(p) (written by pass 1) and update p (group 0) and r (group 1) in place.

struct DivMaps {
    CUtensorMap g0, g1, a;      // plain boxes of the newest plane: a g feeds the d0 queue
    CUtensorMap bg0, bg1;       // box with a d1 halo only
    CUtensorMap g0x, g1x, cx;   // g and c in a box with a d2 halo only
    CUtensorMap lp, po, ro, pc, rc, rm, e1, e2, d;   // plain boxes of the output plane
};

struct DivParams {
    TtiCoef k;
    const float *dz, *dy, *dx;   // separable damping profiles
    float* po;                   // p level being overwritten (wavefield layout)
    float* ro;                   // r level being overwritten
    int N1, N2, pitch;
    long long plane;
    int z_lo, z_hi, chunk;
    // PUSH kernels: mirrors of the new p (index 0) / r (index 1) planes in the neighbours'
    // ghost planes, as in RotParams
    long long peer_lo[2], peer_hi[2];
    int push_planes, desc_last;
};

template <int K, int TXV, int TY, int NS, bool SEP>
struct DivShape {
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;
    static constexpr int SH = TY + 2 * K;
    static constexpr int ABOX = TX * TY;
    static constexpr int YBOX = TX * SH;            // d1-haloed box
    static constexpr int XBOX = SW * TY;            // d2-haloed box
    static constexpr int XPAD = ((XBOX + 31) / 32) * 32;
    static constexpr int NPL = SEP ? 8 : 9;         // lp po ro pc rc rm e1 e2 (damp)
    // stage: feed g0, g1, a | bg0, bg1 | g0x, g1x, cx | plain boxes
    static constexpr int STAGE = 3 * ABOX + 2 * YBOX + 3 * XPAD + NPL * ABOX;
    static constexpr int GROUP = TXV * TY;
    static constexpr int NTHREADS = 2 * GROUP + 32;
    static constexpr size_t SMEM = size_t(NS) * STAGE * 4 + 2 * NS * 8 + 128;
    static_assert(GROUP % 32 == 0 && (ABOX * 4) % 128 == 0 && (YBOX * 4) % 128 == 0, "tile shape");
};

template <int K, int TXV, int TY, int NS, bool SEP, bool PUSH = false>
__global__ void __launch_bounds__(DivShape<K, TXV, TY, NS, SEP>::NTHREADS)
tti_div_update_kernel(const __grid_constant__ DivMaps tm, const __grid_constant__ DivParams p) {
    using S = DivShape<K, TXV, TY, NS, SEP>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int ABOX = S::ABOX, YBOX = S::YBOX, XPAD = S::XPAD, TX = S::TX, NPL = S::NPL;
    constexpr int NCW = 2 * S::GROUP / 32;
    constexpr int OFF_Y = 3 * ABOX, OFF_X = OFF_Y + 2 * YBOX, OFF_P = OFF_X + 3 * XPAD;
    enum { A_LP, A_PO, A_RO, A_PC, A_RC, A_RM, A_E1, A_E2, A_D };

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
    const bool desc = PUSH && p.desc_last && gridDim.z > 1 && blockIdx.z == gridDim.z - 1;
    const int dir = desc ? -1 : 1;
    const int zl0 = desc ? ze - 1 + 2 * K : zb;
    const int zo0 = desc ? ze - 1 : zb;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(done + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    pdl_enter();

    if (tid >= 2 * S::GROUP) {
        if (tid == 2 * S::GROUP) {
            int s = 0;
            uint32_t dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NS) mbar_wait(done + s, dph);
                const bool out = n >= 2 * K;
                float* st = ring + s * STAGE;
                mbar_arrive_expect_tx(
                    full + s, (3 * ABOX + (out ? 2 * YBOX + 3 * S::XBOX + NPL * ABOX : 0)) * 4);
                tma_load_3d(st, &tm.g0, x0, y0, zl0 + dir * n, full + s);
                tma_load_3d(st + ABOX, &tm.g1, x0, y0, zl0 + dir * n, full + s);
                tma_load_3d(st + 2 * ABOX, &tm.a, x0, y0, zl0 + dir * n, full + s);
                if (out) {
                    const int zo = zo0 + dir * (n - 2 * K);  // output plane (compact); buffer plane zo + K
                    const int zc = zo + K;
                    tma_load_3d(st + OFF_Y, &tm.bg0, x0, y0 - K, zc, full + s);
                    tma_load_3d(st + OFF_Y + YBOX, &tm.bg1, x0, y0 - K, zc, full + s);
                    tma_load_3d(st + OFF_X, &tm.g0x, x0 - KP, y0, zc, full + s);
                    tma_load_3d(st + OFF_X + XPAD, &tm.g1x, x0 - KP, y0, zc, full + s);
                    tma_load_3d(st + OFF_X + 2 * XPAD, &tm.cx, x0 - KP, y0, zc, full + s);
                    float* ad = st + OFF_P;
                    tma_load_3d(ad + A_LP * ABOX, &tm.lp, x0, y0, zo, full + s);
                    tma_load_3d(ad + A_PO * ABOX, &tm.po, x0, y0, zc, full + s);
                    tma_load_3d(ad + A_RO * ABOX, &tm.ro, x0, y0, zc, full + s);
                    tma_load_3d(ad + A_PC * ABOX, &tm.pc, x0, y0, zc, full + s);
                    tma_load_3d(ad + A_RC * ABOX, &tm.rc, x0, y0, zc, full + s);
                    tma_load_3d(ad + A_RM * ABOX, &tm.rm, x0, y0, zo, full + s);
                    tma_load_3d(ad + A_E1 * ABOX, &tm.e1, x0, y0, zo, full + s);
                    tma_load_3d(ad + A_E2 * ABOX, &tm.e2, x0, y0, zo, full + s);
                    if (!SEP) tma_load_3d(ad + A_D * ABOX, &tm.d, x0, y0, zo, full + s);
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
    float* outp = (field ? p.ro : p.po) + (long long)(zo0 + K) * p.plane + (long long)y * p.pitch + x;
    const long long zstep = desc ? -p.plane : p.plane;
    long long peer_delta = 0;
    if constexpr (PUSH)
        peer_delta = blockIdx.z == 0 ? p.peer_lo[field]
                                     : (blockIdx.z == gridDim.z - 1 ? p.peer_hi[field] : 0);

    float dxy[4] = {0.f, 0.f, 0.f, 0.f};
    if (SEP && rin) {
        const float4 dx4 = __ldg(reinterpret_cast<const float4*>(p.dx + x));
        const float dyv = __ldg(p.dy + y);
        dxy[0] = dx4.x + dyv;
        dxy[1] = dx4.y + dyv;
        dxy[2] = dx4.z + dyv;
        dxy[3] = dx4.w + dyv;
    }

    // sliding queue window, plane loop unrolled by two (see tti_rot_kernel)
    float q[Q + 1][4];
#pragma unroll
    for (int j = 0; j < Q + 1; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int aown = ty * TX + 4 * tx;
    int s = 0;
    uint32_t fph = 0;
    auto iteration = [&](auto off, int n) {
        constexpr int OFF = decltype(off)::value;
#define SFB_TQ(i) q[(i) + OFF]
        mbar_wait(full + s, fph);
        float* st = ring + s * STAGE;
        {
            const float4 v = *reinterpret_cast<const float4*>(st + field * ABOX + aown);
            const float4 a4 = *reinterpret_cast<const float4*>(st + 2 * ABOX + aown);
            // the queue holds a g
            const float2 p01 = f2_mul(make_float2(v.x, v.y), make_float2(a4.x, a4.y));
            const float2 p23 = f2_mul(make_float2(v.z, v.w), make_float2(a4.z, a4.w));
            SFB_TQ(Q - 1)[0] = p01.x;
            SFB_TQ(Q - 1)[1] = p01.y;
            SFB_TQ(Q - 1)[2] = p23.x;
            SFB_TQ(Q - 1)[3] = p23.y;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release(done + s, SFB_TQ(Q - 1)[0]);
        } else {
            float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 1; j <= K; ++j) {   // D0 (a g): register queue
                const float2 w = f2_splat(p.k.fz[j - 1]);
                a01 = f2_fma(w, f2_sub(make_float2(SFB_TQ(K + j)[0], SFB_TQ(K + j)[1]),
                                       make_float2(SFB_TQ(K - j)[0], SFB_TQ(K - j)[1])), a01);
                a23 = f2_fma(w, f2_sub(make_float2(SFB_TQ(K + j)[2], SFB_TQ(K + j)[3]),
                                       make_float2(SFB_TQ(K - j)[2], SFB_TQ(K - j)[3])), a23);
            }
            if (PUSH && desc) {   // reversed queue: D0 is odd in d0 (see tti_rot_kernel)
                a01 = make_float2(-a01.x, -a01.y);
                a23 = make_float2(-a23.x, -a23.y);
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
            float2 e01 = make_float2(0.f, 0.f), e23 = make_float2(0.f, 0.f);
            {   // D2 (c g): one aligned row segment of g and of c in the d2-haloed boxes; the
                // products and the even-j differences run packed
                float xr[2 * KP + 4];
                const float* rowp = st + OFF_X + field * XPAD + ty * SW + 4 * tx;
                const float* crow = st + OFF_X + 2 * XPAD + ty * SW + 4 * tx;
#pragma unroll
                for (int v = 0; v < (2 * KP + 4) / 4; ++v) {
                    const float4 t4 = *reinterpret_cast<const float4*>(rowp + 4 * v);
                    const float4 n4 = *reinterpret_cast<const float4*>(crow + 4 * v);
                    const float2 m01 = f2_mul(make_float2(t4.x, t4.y), make_float2(n4.x, n4.y));
                    const float2 m23 = f2_mul(make_float2(t4.z, t4.w), make_float2(n4.z, n4.w));
                    xr[4 * v + 0] = m01.x;
                    xr[4 * v + 1] = m01.y;
                    xr[4 * v + 2] = m23.x;
                    xr[4 * v + 3] = m23.y;
                }
#pragma unroll
                for (int j = 1; j <= K; ++j) {
                    if (j % 2 == 0) {
                        const float2 w = f2_splat(p.k.fx[j - 1]);
                        e01 = f2_fma(w, f2_sub(make_float2(xr[KP + j], xr[KP + 1 + j]),
                                               make_float2(xr[KP - j], xr[KP + 1 - j])), e01);
                        e23 = f2_fma(w, f2_sub(make_float2(xr[KP + 2 + j], xr[KP + 3 + j]),
                                               make_float2(xr[KP + 2 - j], xr[KP + 3 - j])), e23);
                    } else {
                        e01.x = fmaf(p.k.fx[j - 1], xr[KP + j] - xr[KP - j], e01.x);
                        e01.y = fmaf(p.k.fx[j - 1], xr[KP + 1 + j] - xr[KP + 1 - j], e01.y);
                        e23.x = fmaf(p.k.fx[j - 1], xr[KP + 2 + j] - xr[KP + 2 - j], e23.x);
                        e23.y = fmaf(p.k.fx[j - 1], xr[KP + 3 + j] - xr[KP + 3 - j], e23.y);
                    }
                }
            }
            a01 = f2_add(a01, e01);
            a23 = f2_add(a23, e23);
            const float hz[4] = {a01.x, a01.y, a23.x, a23.y};
            // swap with the other group through this thread's own (already consumed) slot
            // of the feed box; the named barrier covers the 2 * GROUP consumer threads
            *reinterpret_cast<float4*>(st + field * ABOX + aown) =
                make_float4(hz[0], hz[1], hz[2], hz[3]);
            asm volatile("bar.sync 1, %0;" ::"n"(2 * S::GROUP) : "memory");
            const float4 ot = *reinterpret_cast<const float4*>(st + (1 - field) * ABOX + aown);
            const float other[4] = {ot.x, ot.y, ot.z, ot.w};

            const float* ap = st + OFF_P + aown;
            const float4 lp4 = *reinterpret_cast<const float4*>(ap + A_LP * ABOX);
            const float4 rm4 = *reinterpret_cast<const float4*>(ap + A_RM * ABOX);
            const float4 e14 = *reinterpret_cast<const float4*>(ap + A_E1 * ABOX);
            const float4 e24 = *reinterpret_cast<const float4*>(ap + A_E2 * ABOX);
            const float4 ol4 = *reinterpret_cast<const float4*>(ap + (field ? A_RO : A_PO) * ABOX);
            const float4 cu4 = *reinterpret_cast<const float4*>(ap + (field ? A_RC : A_PC) * ABOX);
            float4 dm4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!SEP) dm4 = *reinterpret_cast<const float4*>(ap + A_D * ABOX);
            float dzv = 0.f;
            if (SEP) dzv = __ldg(p.dz + (zo0 + dir * (n - 2 * K)));
            const float lpv[4] = {lp4.x, lp4.y, lp4.z, lp4.w}, rmv[4] = {rm4.x, rm4.y, rm4.z, rm4.w};
            const float e1v[4] = {e14.x, e14.y, e14.z, e14.w}, e2v[4] = {e24.x, e24.y, e24.z, e24.w};
            const float olv[4] = {ol4.x, ol4.y, ol4.z, ol4.w}, cuv[4] = {cu4.x, cu4.y, cu4.z, cu4.w};
            const float dmv[4] = {dm4.x, dm4.y, dm4.z, dm4.w};
            float un[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float hzp = field ? other[c] : hz[c];
                const float hzr = field ? hz[c] : other[c];
                const float h0 = lpv[c] - hzp;
                const float rhs = field ? fmaf(e2v[c], h0, hzr) : fmaf(e1v[c], h0, e2v[c] * hzr);
                const float dmp = SEP ? (dxy[c] + dzv) : dmv[c];
                const float qq = dmp * rmv[c] * p.k.qscale;
                const float c1 = fast_rcp(1.f + qq), c2 = (1.f - qq) * c1;
                un[c] = fmaf(c1, fmaf(rmv[c], rhs, 2.f * cuv[c]), -c2 * olv[c]);
            }
            // the slot written above is refilled by the async proxy after the release
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // un[0] depends on every shared-memory load of the iteration (see mbar_release)
            __syncwarp();
            if (lane0) mbar_release(done + s, un[0]);
            if (rin) {
                __stcs(reinterpret_cast<float4*>(outp), make_float4(un[0], un[1], un[2], un[3]));
                if constexpr (PUSH) {
                    if (peer_delta && n - 2 * K < p.push_planes)
                        *reinterpret_cast<float4*>(outp + peer_delta) =
                            make_float4(un[0], un[1], un[2], un[3]);
                }
            }
            outp += zstep;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
#undef SFB_TQ
    };
    for (int n = 0; n < nplanes; n += 2) {
        iteration(std::integral_constant<int, 0>{}, n);
        if (n + 1 < nplanes) iteration(std::integral_constant<int, 1>{}, n + 1);
#pragma unroll
        for (int j = 0; j < Q - 1; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[j][c] = q[j + 2][c];
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

// a = sin(theta) cos(phi) on extra planes (the ghost planes of a slab)
static __global__ void tti_axis_a_kernel(const double* __restrict__ theta,
                                         const double* __restrict__ phi, float* a, long long rows,
                                         int n2, int pitch, long long off) {
    const long long row = blockIdx.y * (long long)gridDim.z + blockIdx.z;
    if (row >= rows) return;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n2; x += gridDim.x * blockDim.x) {
        double st, ct, sp, cp;
        sincos(theta[row * n2 + x], &st, &ct);
        sincos(phi[row * n2 + x], &sp, &cp);
        a[off + row * pitch + x] = (float)(st * cp);
    }
}

}  // namespace sfb
