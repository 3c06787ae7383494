// acoustic_patch_kernel.cuh -- "patch" variant of the dual-stream acoustic step kernel for
// the high space orders (K >= 6), sm_100a.
//
// The dual-stream kernel (acoustic_kernel.cuh) gives a thread one row of four nodes.  Its d1
// part then costs 2K LDS.128 per four nodes, and from order 14 up the kernel is bound by the
// shared-memory pipe, not by HBM (profiles/r01_acoustic_so16_592_dual.md: 0.74 LSU
// wavefronts / clk / SM, DRAM at 54 %).  Here a thread owns a 2 x 2 patch (two rows of two
// nodes): the register queue is the same size (2K+1 planes of four values), but every row
// loaded for the d1 part feeds both output rows of the patch, so the column strip costs 2K
// LDS.64 for four nodes -- half the shared-memory wavefronts -- at the price of two row
// segments instead of one for the d2 part.  Per 128 nodes: 76 wavefronts instead of 92 at
// order 16.
//
// The register queue is not shifted every plane: the loop is unrolled by two over a window
// of 2K+2 slots (plane n uses slots [0, 2K], plane n+1 slots [1, 2K+1]) and shifted by two
// afterwards, which halves the register moves per plane (64 of ~350 instructions per thread
// and plane at order 16).
//
// Everything else -- tile (64 x 14), stage layout, TMA boxes, barriers, the arithmetic and
// its order per node, the fused snapshot / imaging / halo-push outputs -- is the dual-stream
// kernel's: the two kernels produce identical bits.
#pragma once

#include "acoustic_kernel.cuh"

namespace sfb {

// release carrying a dependency on two values (the two rows of a patch load different rows)
__device__ __forceinline__ void mbar_release2(uint64_t* bar, float dep0, float dep1) {
    const uint32_t zero = blockDim.z - 1u;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     smem_u32(bar) + ((__float_as_uint(dep0) | __float_as_uint(dep1)) & zero))
                 : "memory");
}

template <int K, int NS, bool SEP>
struct PatchShape : DualShape<K, 16, 14, NS, SEP> {
    static constexpr int TXP = 32;   // threads along d2, two nodes each
    static constexpr int TYP = 7;    // thread rows, two rows each
    static constexpr int KE = (K + 1) & ~1;   // d2 reach rounded up to a float2
    static_assert(TXP * 2 == DualShape<K, 16, 14, NS, SEP>::TX, "tile width");
    static_assert(DualShape<K, 16, 14, NS, SEP>::KP >= KE, "x halo must cover the float2 reach");
};

// L(u) of one 2 x 2 patch.  q window offset OFF: logical plane i of the queue is q[i + OFF].
// Arithmetic order per node as in stencil_acc: centre, d0 pairs, d1 pairs (packed), then the
// d2 part in a scalar accumulator that is added last.
template <int K, int KP, int SW, int KE, int OFF>
__device__ __forceinline__ void patch_stencil(const StencilCoef& k, const float (&q)[2 * K + 2][4],
                                              const float* cp, int tx, int ty2, float (&acc)[4]) {
#define SFB_Q(i) q[(i) + OFF]
    float2 a01 = f2_mul(f2_splat(k.c0), make_float2(SFB_Q(K)[0], SFB_Q(K)[1]));
    float2 a23 = f2_mul(f2_splat(k.c0), make_float2(SFB_Q(K)[2], SFB_Q(K)[3]));
#pragma unroll
    for (int j = 1; j <= K; ++j) {
        const float2 w = f2_splat(k.cz[j - 1]);
        a01 = f2_fma(w, f2_add(make_float2(SFB_Q(K - j)[0], SFB_Q(K - j)[1]),
                               make_float2(SFB_Q(K + j)[0], SFB_Q(K + j)[1])), a01);
        a23 = f2_fma(w, f2_add(make_float2(SFB_Q(K - j)[2], SFB_Q(K - j)[3]),
                               make_float2(SFB_Q(K + j)[2], SFB_Q(K + j)[3])), a23);
    }
    {   // d1: rows above (L_j = own row 0 - j) and below (H_j = own row 1 + j); row 0 pairs
        // L_j with H_{j-1}, row 1 pairs L_{j-1} with H_j: every loaded row is used twice
        const float* colp = cp + (ty2 + K) * SW + KP + 2 * tx;   // own row 0, own columns
        float2 lprev = make_float2(SFB_Q(K)[0], SFB_Q(K)[1]);    // L_0 = own row 0
        float2 hprev = make_float2(SFB_Q(K)[2], SFB_Q(K)[3]);    // H_0 = own row 1
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const float2 lj = *reinterpret_cast<const float2*>(colp - j * SW);
            const float2 hj = *reinterpret_cast<const float2*>(colp + (1 + j) * SW);
            const float2 w = f2_splat(k.cy[j - 1]);
            a01 = f2_fma(w, f2_add(lj, hprev), a01);
            a23 = f2_fma(w, f2_add(lprev, hj), a23);
            lprev = lj;
            hprev = hj;
        }
    }
    // d2: one row segment per patch row; even j: the operand pair (xr[KE-j], xr[KE+1-j]) is a
    // register-aligned float2 and runs packed, odd j stays scalar (same roundings per node)
    float ax[4];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        float xr[2 * KE + 2];
        const float* rowp = cp + (ty2 + K + r) * SW + KP + 2 * tx - KE;
#pragma unroll
        for (int v = 0; v < KE + 1; ++v) {
            if (v == KE / 2) {   // own float2: already in the queue
                xr[2 * v] = SFB_Q(K)[2 * r];
                xr[2 * v + 1] = SFB_Q(K)[2 * r + 1];
            } else {
                const float2 t2 = *reinterpret_cast<const float2*>(rowp + 2 * v);
                xr[2 * v] = t2.x;
                xr[2 * v + 1] = t2.y;
            }
        }
        float2 x2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            if (j % 2 == 0) {
                x2 = f2_fma(f2_splat(k.cx[j - 1]),
                            f2_add(make_float2(xr[KE - j], xr[KE + 1 - j]),
                                   make_float2(xr[KE + j], xr[KE + 1 + j])), x2);
            } else {
                x2.x = fmaf(k.cx[j - 1], xr[KE - j] + xr[KE + j], x2.x);
                x2.y = fmaf(k.cx[j - 1], xr[KE + 1 - j] + xr[KE + 1 + j], x2.y);
            }
        }
        ax[2 * r] = x2.x;
        ax[2 * r + 1] = x2.y;
    }
    a01 = f2_add(a01, make_float2(ax[0], ax[1]));
    a23 = f2_add(a23, make_float2(ax[2], ax[3]));
    acc[0] = a01.x;
    acc[1] = a01.y;
    acc[2] = a23.x;
    acc[3] = a23.y;
#undef SFB_Q
}

template <int K, int NS, bool SEP, int MINB, bool PUSH = false>
__global__ void __launch_bounds__(PatchShape<K, NS, SEP>::NTHREADS, MINB)
acoustic_step_patch_kernel(const __grid_constant__ StepMaps tm,
                           const __grid_constant__ StepParams p) {
    using S = PatchShape<K, NS, SEP>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1, KE = S::KE;
    constexpr int NARR = S::NARR, ABOX = S::ABOX, CPAD = S::CPAD, TX = S::TX, TY = 14;
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
        // producer: identical to acoustic_step_dual_kernel (same boxes, same stage layout)
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

    const int tx = tid & 31, ty2 = 2 * (tid >> 5);
    const int x = x0 + 2 * tx, y = y0 + ty2;
    const bool rin0 = x < p.N2 && y < p.N1, rin1 = x < p.N2 && y + 1 < p.N1;
    const bool lane0 = tx == 0;

    float dxy[4] = {0.f, 0.f, 0.f, 0.f};
    bool warp_dxy = false;
    if (SEP) {
        if (rin0) {
            const float2 dx2 = __ldg(reinterpret_cast<const float2*>(p.dx + x));
            const float dy0 = __ldg(p.dy + y);
            const float dy1 = rin1 ? __ldg(p.dy + y + 1) : 0.f;
            dxy[0] = dx2.x + dy0;
            dxy[1] = dx2.y + dy0;
            dxy[2] = dx2.x + dy1;
            dxy[3] = dx2.y + dy1;
        }
        warp_dxy = __any_sync(0xffffffffu, (dxy[0] + dxy[1]) + (dxy[2] + dxy[3]) != 0.f);
    }

    float q[Q + 1][4];
#pragma unroll
    for (int j = 0; j < Q + 1; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) q[j][c] = 0.f;

    const int aown = ty2 * TX + 2 * tx;   // own float2 of patch row 0 in a plain box
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
            const float2 v0 = *reinterpret_cast<const float2*>(st + aown);
            const float2 v1 = *reinterpret_cast<const float2*>(st + aown + TX);
            q[Q - 1 + OFF][0] = v0.x;
            q[Q - 1 + OFF][1] = v0.y;
            q[Q - 1 + OFF][2] = v1.x;
            q[Q - 1 + OFF][3] = v1.y;
        }
        if (n < 2 * K) {
            __syncwarp();
            if (lane0) mbar_release2(done + s, q[Q - 1 + OFF][0], q[Q - 1 + OFF][3]);
        } else {
            const float* ap = st + ABOX + CPAD + aown;
            const float2 o0 = *reinterpret_cast<const float2*>(ap);
            const float2 o1 = *reinterpret_cast<const float2*>(ap + TX);
            const float2 r0 = *reinterpret_cast<const float2*>(ap + ABOX);
            const float2 r1 = *reinterpret_cast<const float2*>(ap + ABOX + TX);
            float dv[4] = {0.f, 0.f, 0.f, 0.f};
            if (!SEP) {
                const float2 d0 = *reinterpret_cast<const float2*>(ap + 2 * ABOX);
                const float2 d1 = *reinterpret_cast<const float2*>(ap + 2 * ABOX + TX);
                dv[0] = d0.x;
                dv[1] = d0.y;
                dv[2] = d1.x;
                dv[3] = d1.y;
            }
            const float dzv = dzn;
            if (SEP && n + 1 < nplanes) dzn = __ldg(p.dz + (zo0 + dir * (n + 1 - 2 * K)));

            float acc[4];
            patch_stencil<K, KP, SW, KE, OFF>(p.k, q, st + ABOX, tx, ty2, acc);

            const float rv[4] = {r0.x, r0.y, r1.x, r1.y};
            const float ov[4] = {o0.x, o0.y, o1.x, o1.y};
            const float* uc = q[K + OFF];
            bool damped;
            if (SEP) {
                damped = warp_dxy || dzv != 0.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) dv[c] = dxy[c] + dzv;
            } else {
                damped = __any_sync(0xffffffffu, (dv[0] + dv[1]) + (dv[2] + dv[3]) != 0.f);
            }
            float un[4];
            if (damped) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float qq = dv[c] * rv[c] * p.k.qscale;
                    const float c1 = fast_rcp(1.f + qq);
                    const float c2 = (1.f - qq) * c1;
                    const float t = fmaf(rv[c], acc[c], 2.f * uc[c]);
                    un[c] = fmaf(c1, t, -c2 * ov[c]);
                }
            } else {
                const float2 u01 = make_float2(uc[0], uc[1]), u23 = make_float2(uc[2], uc[3]);
                const float2 t01 = f2_fma(make_float2(rv[0], rv[1]), make_float2(acc[0], acc[1]),
                                          f2_add(u01, u01));
                const float2 t23 = f2_fma(make_float2(rv[2], rv[3]), make_float2(acc[2], acc[3]),
                                          f2_add(u23, u23));
                const float2 n01 = f2_add(t01, make_float2(-ov[0], -ov[1]));
                const float2 n23 = f2_add(t23, make_float2(-ov[2], -ov[3]));
                un[0] = n01.x;
                un[1] = n01.y;
                un[2] = n23.x;
                un[3] = n23.y;
            }
            // un[0] and un[3] together depend on every shared-memory load of the iteration
            __syncwarp();
            if (lane0) mbar_release2(done + s, un[0], un[3]);
            const bool push_now = PUSH && n - 2 * K < p.push_planes;
            long long peer_delta = 0;
            if constexpr (PUSH)
                peer_delta = blockIdx.z == 0 ? p.peer_delta0
                                             : (blockIdx.z == gridDim.z - 1 ? p.peer_delta1 : 0);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (!(r ? rin1 : rin0)) continue;
                const long long ro = (long long)r * p.pitch;
                const float2 nv = make_float2(un[2 * r], un[2 * r + 1]);
                __stcs(reinterpret_cast<float2*>(po + ro), nv);
                if constexpr (PUSH) {
                    if (peer_delta && push_now)
                        *reinterpret_cast<float2*>(po + ro + peer_delta) = nv;
                }
                if (p.snap) __stcs(reinterpret_cast<float2*>(p.snap + gc + ro), nv);
                if (p.usave) {
                    const float2 g2 = __ldcs(reinterpret_cast<const float2*>(p.grad + gc + ro));
                    const float2 s2 = __ldcs(reinterpret_cast<const float2*>(p.usave + gc + ro));
                    float2 gn;
                    gn.x = fmaf(-s2.x * p.k.inv_dt2, (un[2 * r] - 2.f * uc[2 * r]) + ov[2 * r], g2.x);
                    gn.y = fmaf(-s2.y * p.k.inv_dt2,
                                (un[2 * r + 1] - 2.f * uc[2 * r + 1]) + ov[2 * r + 1], g2.y);
                    __stcs(reinterpret_cast<float2*>(p.grad + gc + ro), gn);
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
            for (int c = 0; c < 4; ++c) q[j][c] = q[j + 2][c];
    }
}

}  // namespace sfb
