// acoustic_tall_kernel.cuh -- "tall" variant of the dual-stream acoustic step kernel for the
// highest space orders (K >= 7), sm_100a.
//
// From order 14 up the dual-stream kernel sits on the shared-memory pipe: a thread owns one
// row of four nodes and pays 2K LDS.128 for the d1 part of those four nodes
// (profiles/r02_acoustic_so16_592_slide.md: l1tex 84 % busy, DRAM at 54 %).  Here a thread
// owns TWO rows of four nodes.  Every row loaded for the d1 part feeds both of them, so the
// column strip costs 2K+2 LDS.128 for EIGHT nodes; with the two row segments of the d2 part
// that is (2K + 2 + 2 * 4) / 2 = 13 LDS.128 per four nodes at order 16 instead of 20.  The
// price is the register queue: 2K+2 planes of eight values, 144 registers at order 16, so a
// block is 7 consumer warps (a 64 x 28 tile) + the producer warp at 255 registers per
// thread, one block per SM.
//
// Queue window, stage layout, TMA boxes, barriers and the arithmetic per node (and its
// order) are the dual-stream kernel's: the kernels produce identical bits.
#pragma once

#include "acoustic_kernel.cuh"
#include "acoustic_patch_kernel.cuh"

namespace sfb {

// release carrying a dependency on four values (the corner nodes of the thread's 2 x 4 block
// together depend on every shared-memory load of the iteration)
__device__ __forceinline__ void mbar_release4(uint64_t* bar, float d0, float d1, float d2, float d3) {
    const uint32_t zero = blockDim.z - 1u;
    const uint32_t bits = (__float_as_uint(d0) | __float_as_uint(d1)) |
                          (__float_as_uint(d2) | __float_as_uint(d3));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar) + (bits & zero))
                 : "memory");
}

// TYT: thread rows, two node rows each (14: 7 consumer warps, a 64 x 28 tile; 16: 8 warps, 64 x 32)
template <int K, int NS, bool SEP, int TYT = 14>
struct TallShape : DualShape<K, 16, 2 * TYT, NS, SEP> {
    static constexpr int NCONS = 16 * TYT;
    static constexpr int NTHREADS = NCONS + 32;
    static_assert(NCONS % 32 == 0, "whole consumer warps");
};

// L(u) of one 2 x 4 block.  Queue window offset OFF: logical plane i of the queue is
// q[i + OFF]; values [0..3] are the upper row, [4..7] the lower one.  Per node the order is
// stencil_acc's: centre, d0 pairs, d1 pairs, then the d2 sum (accumulated apart) added last.
template <int K, int KP, int SW, int OFF>
__device__ __forceinline__ void tall_stencil(const StencilCoef& k, const float (&q)[2 * K + 2][8],
                                             const float* cp, int tx, int ty2, float (&acc)[8]) {
#define SFB_Q(i) q[(i) + OFF]
    float2 a[4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
        a[h] = f2_mul(f2_splat(k.c0), make_float2(SFB_Q(K)[2 * h], SFB_Q(K)[2 * h + 1]));
#pragma unroll
    for (int j = 1; j <= K; ++j) {
        const float2 w = f2_splat(k.cz[j - 1]);
#pragma unroll
        for (int h = 0; h < 4; ++h)
            a[h] = f2_fma(w, f2_add(make_float2(SFB_Q(K - j)[2 * h], SFB_Q(K - j)[2 * h + 1]),
                                    make_float2(SFB_Q(K + j)[2 * h], SFB_Q(K + j)[2 * h + 1])), a[h]);
    }
    {   // d1: rows above (L_j = upper row - j) and below (H_j = lower row + j); the upper row
        // pairs L_j with H_{j-1}, the lower one L_{j-1} with H_j: every loaded row is used twice
        const float* colp = cp + (ty2 + K) * SW + KP + 4 * tx;   // upper row, own columns
        float4 lprev = make_float4(SFB_Q(K)[0], SFB_Q(K)[1], SFB_Q(K)[2], SFB_Q(K)[3]);
        float4 hprev = make_float4(SFB_Q(K)[4], SFB_Q(K)[5], SFB_Q(K)[6], SFB_Q(K)[7]);
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const float4 lj = *reinterpret_cast<const float4*>(colp - j * SW);
            const float4 hj = *reinterpret_cast<const float4*>(colp + (1 + j) * SW);
            const float2 w = f2_splat(k.cy[j - 1]);
            a[0] = f2_fma(w, f2_add(make_float2(lj.x, lj.y), make_float2(hprev.x, hprev.y)), a[0]);
            a[1] = f2_fma(w, f2_add(make_float2(lj.z, lj.w), make_float2(hprev.z, hprev.w)), a[1]);
            a[2] = f2_fma(w, f2_add(make_float2(lprev.x, lprev.y), make_float2(hj.x, hj.y)), a[2]);
            a[3] = f2_fma(w, f2_add(make_float2(lprev.z, lprev.w), make_float2(hj.z, hj.w)), a[3]);
            lprev = lj;
            hprev = hj;
        }
    }
    // d2: one aligned row segment per node row; even j packed, odd j scalar (stencil_acc)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        float2 x01 = make_float2(0.f, 0.f), x23 = make_float2(0.f, 0.f);
        float xr[2 * KP + 4];
        const float* rowp = cp + (ty2 + K + r) * SW + 4 * tx;
#pragma unroll
        for (int v = 0; v < (2 * KP + 4) / 4; ++v) {
            if (v == KP / 4) {  // own float4: already in the queue
#pragma unroll
                for (int c = 0; c < 4; ++c) xr[4 * v + c] = SFB_Q(K)[4 * r + c];
            } else {
                const float4 t4 = *reinterpret_cast<const float4*>(rowp + 4 * v);
                xr[4 * v + 0] = t4.x;
                xr[4 * v + 1] = t4.y;
                xr[4 * v + 2] = t4.z;
                xr[4 * v + 3] = t4.w;
            }
        }
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            if (j % 2 == 0) {
                const float2 w = f2_splat(k.cx[j - 1]);
                x01 = f2_fma(w, f2_add(make_float2(xr[KP - j], xr[KP + 1 - j]),
                                       make_float2(xr[KP + j], xr[KP + 1 + j])), x01);
                x23 = f2_fma(w, f2_add(make_float2(xr[KP + 2 - j], xr[KP + 3 - j]),
                                       make_float2(xr[KP + 2 + j], xr[KP + 3 + j])), x23);
            } else {
                x01.x = fmaf(k.cx[j - 1], xr[KP - j] + xr[KP + j], x01.x);
                x01.y = fmaf(k.cx[j - 1], xr[KP + 1 - j] + xr[KP + 1 + j], x01.y);
                x23.x = fmaf(k.cx[j - 1], xr[KP + 2 - j] + xr[KP + 2 + j], x23.x);
                x23.y = fmaf(k.cx[j - 1], xr[KP + 3 - j] + xr[KP + 3 + j], x23.y);
            }
        }
        a[2 * r] = f2_add(a[2 * r], x01);
        a[2 * r + 1] = f2_add(a[2 * r + 1], x23);
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        acc[2 * h] = a[h].x;
        acc[2 * h + 1] = a[h].y;
    }
#undef SFB_Q
}

template <int K, int NS, bool SEP, bool PUSH = false, int TYT = 14>
__global__ void __launch_bounds__(TallShape<K, NS, SEP, TYT>::NTHREADS, 1)
acoustic_step_tall_kernel(const __grid_constant__ StepMaps tm,
                          const __grid_constant__ StepParams p) {
    using S = TallShape<K, NS, SEP, TYT>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int NARR = S::NARR, ABOX = S::ABOX, CPAD = S::CPAD, TX = S::TX, TY = 2 * TYT;
    constexpr int NCW = S::NCONS / 32;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
    uint64_t* done = full + NS;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk + (blockIdx.z ? p.z_jump : 0);
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

    if (tid >= S::NCONS) {
        // producer: the dual-stream kernel's (same boxes per stage, 28 rows tall)
        if (tid == S::NCONS) {
            int s = 0;
            uint32_t dph = 0;
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NS) mbar_wait(done + s, dph);
                const bool out = n >= 2 * K;
                float* st = ring + s * STAGE;
                mbar_arrive_expect_tx(full + s, (ABOX + (out ? S::CBOX + NARR * ABOX : 0)) * 4);
                tma_load_3d(st, &tm.f, x0, y0, zl0 + dir * n, full + s);
                if (out) {
                    const int zo = zo0 + dir * (n - 2 * K);
                    tma_load_3d(st + ABOX, &tm.u, x0 - KP, y0 - K, zo + K, full + s);
                    float* ad = st + ABOX + CPAD;
                    tma_load_3d(ad, &tm.o, x0, y0, zo + K, full + s);
                    tma_load_3d(ad + ABOX, &tm.r, x0, y0, zo, full + s);
                    if (!SEP) tma_load_3d(ad + 2 * ABOX, &tm.d, x0, y0, zo, full + s);
                }
                if (++s == NS) {
                    s = 0;
                    if (n >= NS) dph ^= 1;
                }
            }
        }
        return;
    }

    const int tx = tid & 15, ty2 = 2 * (tid >> 4);
    const int x = x0 + 4 * tx, y = y0 + ty2;
    const bool rin0 = x < p.N2 && y < p.N1, rin1 = x < p.N2 && y + 1 < p.N1;
    const bool lane0 = (tid & 31) == 0;

    float dxy[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    bool warp_dxy = false;
    if (SEP) {
        if (rin0) {
            const float4 dx4 = __ldg(reinterpret_cast<const float4*>(p.dx + x));
            const float dy0 = __ldg(p.dy + y);
            const float dy1 = rin1 ? __ldg(p.dy + y + 1) : 0.f;
            dxy[0] = dx4.x + dy0;
            dxy[1] = dx4.y + dy0;
            dxy[2] = dx4.z + dy0;
            dxy[3] = dx4.w + dy0;
            dxy[4] = dx4.x + dy1;
            dxy[5] = dx4.y + dy1;
            dxy[6] = dx4.z + dy1;
            dxy[7] = dx4.w + dy1;
        }
        warp_dxy = __any_sync(0xffffffffu, ((dxy[0] + dxy[1]) + (dxy[2] + dxy[3])) +
                                               ((dxy[4] + dxy[5]) + (dxy[6] + dxy[7])) != 0.f);
    }

    float q[Q + 1][8];
#pragma unroll
    for (int j = 0; j < Q + 1; ++j)
#pragma unroll
        for (int c = 0; c < 8; ++c) q[j][c] = 0.f;

    const int aown = ty2 * TX + 4 * tx;   // own float4 of the upper row in a plain box
    long long gc = (long long)zo0 * p.plane + (long long)y * p.pitch + x;
    float* po = p.uo + gc + (long long)K * p.plane;
    const long long zstep = desc ? -p.plane : p.plane;
    float dzn = 0.f;
    if (SEP) dzn = __ldg(p.dz + zo0);
    int s = 0;
    uint32_t fph = 0;

    // one plane with the queue window at offset OFF (0 or 1)
    auto iteration = [&](auto off, int n) {
        constexpr int OFF = decltype(off)::value;
        mbar_wait(full + s, fph);
        const float* st = ring + s * STAGE;
        {
            const float4 v0 = *reinterpret_cast<const float4*>(st + aown);
            const float4 v1 = *reinterpret_cast<const float4*>(st + aown + TX);
            float* qn = q[Q - 1 + OFF];
            qn[0] = v0.x; qn[1] = v0.y; qn[2] = v0.z; qn[3] = v0.w;
            qn[4] = v1.x; qn[5] = v1.y; qn[6] = v1.z; qn[7] = v1.w;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release2(done + s, q[Q - 1 + OFF][0], q[Q - 1 + OFF][7]);
        } else {
            const float* ap = st + ABOX + CPAD + aown;
            float ov[8], rv[8], dv[8];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const float4 o4 = *reinterpret_cast<const float4*>(ap + r * TX);
                const float4 r4 = *reinterpret_cast<const float4*>(ap + ABOX + r * TX);
                ov[4 * r] = o4.x; ov[4 * r + 1] = o4.y; ov[4 * r + 2] = o4.z; ov[4 * r + 3] = o4.w;
                rv[4 * r] = r4.x; rv[4 * r + 1] = r4.y; rv[4 * r + 2] = r4.z; rv[4 * r + 3] = r4.w;
                if (!SEP) {
                    const float4 d4 = *reinterpret_cast<const float4*>(ap + 2 * ABOX + r * TX);
                    dv[4 * r] = d4.x; dv[4 * r + 1] = d4.y; dv[4 * r + 2] = d4.z; dv[4 * r + 3] = d4.w;
                }
            }
            const float dzv = dzn;
            if (SEP && n + 1 < nplanes) dzn = __ldg(p.dz + (zo0 + dir * (n + 1 - 2 * K)));

            float acc[8];
            tall_stencil<K, KP, SW, OFF>(p.k, q, st + ABOX, tx, ty2, acc);

            const float* uc = q[K + OFF];
            bool damped;
            if (SEP) {
                damped = warp_dxy || dzv != 0.f;
#pragma unroll
                for (int c = 0; c < 8; ++c) dv[c] = dxy[c] + dzv;
            } else {
                damped = __any_sync(0xffffffffu, ((dv[0] + dv[1]) + (dv[2] + dv[3])) +
                                                     ((dv[4] + dv[5]) + (dv[6] + dv[7])) != 0.f);
            }
            float un[8];
            if (damped) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float qq = dv[c] * rv[c] * p.k.qscale;
                    const float c1 = fast_rcp(1.f + qq);
                    const float c2 = (1.f - qq) * c1;
                    const float t = fmaf(rv[c], acc[c], 2.f * uc[c]);
                    un[c] = fmaf(c1, t, -c2 * ov[c]);
                }
            } else {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float2 u2 = make_float2(uc[2 * h], uc[2 * h + 1]);
                    const float2 t2 = f2_fma(make_float2(rv[2 * h], rv[2 * h + 1]),
                                             make_float2(acc[2 * h], acc[2 * h + 1]), f2_add(u2, u2));
                    const float2 n2 = f2_add(t2, make_float2(-ov[2 * h], -ov[2 * h + 1]));
                    un[2 * h] = n2.x;
                    un[2 * h + 1] = n2.y;
                }
            }
            // the corner nodes together depend on every shared-memory load of the iteration
            __syncwarp();
            if (lane0) mbar_release4(done + s, un[0], un[3], un[4], un[7]);
            [[maybe_unused]] const bool push_now = PUSH && n - 2 * K < p.push_planes;
            [[maybe_unused]] long long peer_delta = 0;
            if constexpr (PUSH)
                peer_delta = blockIdx.z == 0 ? p.peer_delta0
                                             : (blockIdx.z == gridDim.z - 1 ? p.peer_delta1 : 0);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (!(r ? rin1 : rin0)) continue;
                const long long ro = (long long)r * p.pitch;
                const float4 nv = make_float4(un[4 * r], un[4 * r + 1], un[4 * r + 2], un[4 * r + 3]);
                __stcs(reinterpret_cast<float4*>(po + ro), nv);
                if constexpr (PUSH) {
                    if (peer_delta && push_now) *reinterpret_cast<float4*>(po + ro + peer_delta) = nv;
                }
                if (p.snap) __stcs(reinterpret_cast<float4*>(p.snap + gc + ro), nv);
                if (p.usave) {
                    const float4 g4 = __ldcs(reinterpret_cast<const float4*>(p.grad + gc + ro));
                    const float4 s4 = __ldcs(reinterpret_cast<const float4*>(p.usave + gc + ro));
                    const float* u_ = un + 4 * r;
                    const float* c_ = uc + 4 * r;
                    const float* o_ = ov + 4 * r;
                    float4 gn;
                    gn.x = fmaf(-s4.x * p.k.inv_dt2, (u_[0] - 2.f * c_[0]) + o_[0], g4.x);
                    gn.y = fmaf(-s4.y * p.k.inv_dt2, (u_[1] - 2.f * c_[1]) + o_[1], g4.y);
                    gn.z = fmaf(-s4.z * p.k.inv_dt2, (u_[2] - 2.f * c_[2]) + o_[2], g4.z);
                    gn.w = fmaf(-s4.w * p.k.inv_dt2, (u_[3] - 2.f * c_[3]) + o_[3], g4.w);
                    __stcs(reinterpret_cast<float4*>(p.grad + gc + ro), gn);
                }
            }
            po += zstep;
            gc += zstep;
        }
        if (++s == NS) {
            s = 0;
            fph ^= 1;
        }
    };

    for (int n = 0; n < nplanes; n += 2) {
        iteration(std::integral_constant<int, 0>{}, n);
        if (n + 1 < nplanes) iteration(std::integral_constant<int, 1>{}, n + 1);
        // slide the window by two planes
#pragma unroll
        for (int j = 0; j < Q - 1; ++j)
#pragma unroll
            for (int c = 0; c < 8; ++c) q[j][c] = q[j + 2][c];
    }
}

}  // namespace sfb
