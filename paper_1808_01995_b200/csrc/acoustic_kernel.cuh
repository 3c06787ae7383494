// acoustic_kernel.cuh -- space-order-k 3-D star-stencil step for the damped acoustic
// wave equation, sm_100a.
//
// Computes, for every owned node of one slab (the closed
// form the reference pins at proj/tests/test_compiler.cpp:80,84):
//     u[t+1] = ( L(u[t]) - m (u[t-1] - 2 u[t]) / dt^2 + damp u[t-1] / (2 dt) ) * inv0
// evaluated in the algebraically identical, better conditioned fp32 form
//     u[t+1] = c1 (2 u[t] + r L(u[t])) - c2 u[t-1],
//     r = dt^2/m,  q = damp r / (2 dt),  c1 = 1/(1+q),  c2 = (1-q) c1.
// The adjoint update (proj/src/seismic_ops.cpp:97-100) is the same expression with the
// roles of t-1 and t+1 swapped, so this kernel serves forward, adjoint and gradient.
//
// Data movement.  u[t] is streamed along the slowest axis d0 in (d1,d2) tiles: a producer
// warp issues one TMA box load (cp.async.bulk.tensor.3d, zero fill outside the grid =
// the reference's zero halo, proj/include/sf/function.hpp:17) per plane into a shared
// memory ring; consumer threads keep the 2K+1 d0 neighbours of their own points in a
// register queue and read the in-plane neighbours of the centre plane from the ring.
// u[t-1], r and damp are read once with 128-bit loads and u[t+1] overwrites u[t-1] in
// place, so a node costs its compulsory 20 bytes (16 with the separable damping
// profiles).  Optional fused outputs: forward snapshot (save) and the imaging
// condition grad -= u_saved * v.dt2 (proj/src/seismic_ops.cpp:132).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sfb {

constexpr int kMaxK = 8;

struct StencilCoef {
    float c0;           // w_0 * sum_d 1/h_d^2 over active axes
    float cx[kMaxK];    // w_j / h_2^2 (contiguous axis)
    float cy[kMaxK];    // w_j / h_1^2
    float cz[kMaxK];    // w_j / h_0^2 (streaming axis)
    float qscale;       // 1 / (2 dt)
    float inv_dt2;      // 1 / dt^2
};

struct StepParams {
    StencilCoef k;
    const float* r;      // dt^2/m, compact [n0][N1][pitch]
    const float* damp;   // dense damping (null when separable)
    const float* dz;     // separable profiles: damp = dz[i0] + dy[i1] + dx[i2]
    const float* dy;
    const float* dx;
    float* uo;           // in: level t-1 (t+1 for the adjoint); out: the new level; has K ghost planes per side
    float* snap;         // optional copy of the new level (compact)
    const float* usave;  // optional saved forward level (compact) -> imaging
    float* grad;         // imaging accumulator (compact)
    int N1, N2;
    int pitch;           // floats per row (multiple of 4)
    long long plane;     // floats per plane
    int z_lo, z_hi;      // owned output planes [z_lo, z_hi) handled by this launch
    int chunk;           // output planes per block
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar), ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

template <int K, int TXV, int TY, int R, int NST>
struct StepShape {
    static constexpr int KP = (K + 3) & ~3;       // x halo rounded to a float4
    static constexpr int TX = TXV * 4;
    static constexpr int SW = TX + 2 * KP;        // ring row width (floats)
    static constexpr int SH = TY + 2 * K;         // ring rows
    static constexpr int BOX = SW * SH;           // floats moved per TMA box
    static constexpr int STAGE = ((BOX + 31) / 32) * 32;
    static constexpr int NCONS = TXV * (TY / R);  // consumer threads
    static constexpr int NTHREADS = NCONS + 32;   // + producer warp
    static constexpr size_t SMEM = size_t(NST) * STAGE * 4 + 2 * NST * 8 + 128;
    static_assert(TY % R == 0 && NCONS % 32 == 0, "tile shape");
    static_assert(NST >= K + 2, "ring must hold the centre plane and the newest plane");
};

template <int K, int TXV, int TY, int R, int NST, bool SEP>
__global__ void __launch_bounds__(StepShape<K, TXV, TY, R, NST>::NTHREADS)
acoustic_step_kernel(const __grid_constant__ CUtensorMap tmU,
                     const __grid_constant__ StepParams p) {
    using S = StepShape<K, TXV, TY, R, NST>;
    constexpr int KP = S::KP, SW = S::SW, STAGE = S::STAGE, Q = 2 * K + 1;
    constexpr int NCW = S::NCONS / 32;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t mis = smem_u32(smem_raw) & 127u;
    float* ring = reinterpret_cast<float*>(smem_raw + ((128u - mis) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NST * STAGE);
    uint64_t* empty = full + NST;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * S::TX, y0 = blockIdx.y * TY;
    const int zb = p.z_lo + blockIdx.z * p.chunk;
    const int ze = min(zb + p.chunk, p.z_hi);
    const int nplanes = (ze - zb) + 2 * K;  // buffer planes zb .. ze+2K-1 (ghost offset K)

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid >= S::NCONS) {
        // ---- producer warp: one elected lane streams the planes of this block -------
        if (tid == S::NCONS) {
            int s = 0;
            uint32_t ph = 0;  // parity of the release that must precede refill
            for (int n = 0; n < nplanes; ++n) {
                if (n >= NST) mbar_wait(empty + s, ph);
                mbar_arrive_expect_tx(full + s, S::BOX * 4);
                tma_load_3d(ring + s * STAGE, &tmU, x0 - KP, y0 - K, zb + n, full + s);
                if (++s == NST) {
                    s = 0;
                    if (n >= NST) ph ^= 1;
                }
            }
        }
        return;
    }

    // ---- consumers -------------------------------------------------------------------
    const int tx = tid % TXV, ty0 = (tid / TXV) * R;
    const int x = x0 + 4 * tx;
    const bool xin = x < p.N2;
    bool rin[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) rin[rr] = xin && (y0 + ty0 + rr) < p.N1;
    const long long rowoff = (long long)(y0 + ty0) * p.pitch + x;

    float dxy[R][4];
    if (SEP) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            float4 dx4 = make_float4(0.f, 0.f, 0.f, 0.f);
            float dyv = 0.f;
            if (rin[rr]) {
                dx4 = __ldg(reinterpret_cast<const float4*>(p.dx + x));
                dyv = __ldg(p.dy + y0 + ty0 + rr);
            }
            dxy[rr][0] = dx4.x + dyv;
            dxy[rr][1] = dx4.y + dyv;
            dxy[rr][2] = dx4.z + dyv;
            dxy[rr][3] = dx4.w + dyv;
        }
    }

    float q[R][Q][4];
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
        for (int j = 0; j < Q; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) q[rr][j][c] = 0.f;

    int s = 0, cs = K;     // ring stage of the newest plane / of the centre plane (plane K is the first centre)
    uint32_t fph = 0;      // parity of the fill we wait for on stage s
    const int own = (ty0 + K) * SW + KP + 4 * tx;  // own point inside a stage

    for (int n = 0; n < nplanes; ++n) {
        mbar_wait(full + s, fph);
        const float* sp = ring + s * STAGE;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const float4 v = *reinterpret_cast<const float4*>(sp + own + rr * SW);
            q[rr][Q - 1][0] = v.x;
            q[rr][Q - 1][1] = v.y;
            q[rr][Q - 1][2] = v.z;
            q[rr][Q - 1][3] = v.w;
        }
        if (n < K) {  // the first K planes are d0 halo only: never a centre
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(empty + s);
        }
        if (n >= 2 * K) {
            const int zo = zb + n - 2 * K;
            const long long gc = (long long)zo * p.plane + rowoff;         // compact arrays
            const long long gu = (long long)(zo + K) * p.plane + rowoff;   // u buffers
            float4 r4[R], o4[R], d4[R], g4[R], s4[R];
            const bool img = p.usave != nullptr;
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                r4[rr] = o4[rr] = d4[rr] = g4[rr] = s4[rr] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (rin[rr]) {
                    const long long o = (long long)rr * p.pitch;
                    r4[rr] = __ldcs(reinterpret_cast<const float4*>(p.r + gc + o));
                    o4[rr] = __ldcs(reinterpret_cast<const float4*>(p.uo + gu + o));
                    if (!SEP) d4[rr] = __ldcs(reinterpret_cast<const float4*>(p.damp + gc + o));
                    if (img) {
                        g4[rr] = __ldcs(reinterpret_cast<const float4*>(p.grad + gc + o));
                        s4[rr] = __ldcs(reinterpret_cast<const float4*>(p.usave + gc + o));
                    }
                }
            }
            float dzv = 0.f;
            if (SEP) dzv = __ldg(p.dz + zo);

            const float* cp = ring + cs * STAGE;
            float acc[R][4];
            // centre and streaming-axis neighbours from the register queue
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float a = p.k.c0 * q[rr][K][c];
#pragma unroll
                    for (int j = 1; j <= K; ++j)
                        a = fmaf(p.k.cz[j - 1], q[rr][K - j][c] + q[rr][K + j][c], a);
                    acc[rr][c] = a;
                }
            // contiguous-axis neighbours: one aligned row segment per own row
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                float xr[2 * KP + 4];
                const float* rowp = cp + (ty0 + rr + K) * SW + 4 * tx;
#pragma unroll
                for (int v = 0; v < (2 * KP + 4) / 4; ++v) {
                    if (v == KP / 4) {  // own float4: already in the queue
                        xr[4 * v + 0] = q[rr][K][0];
                        xr[4 * v + 1] = q[rr][K][1];
                        xr[4 * v + 2] = q[rr][K][2];
                        xr[4 * v + 3] = q[rr][K][3];
                    } else {
                        const float4 t4 = *reinterpret_cast<const float4*>(rowp + 4 * v);
                        xr[4 * v + 0] = t4.x;
                        xr[4 * v + 1] = t4.y;
                        xr[4 * v + 2] = t4.z;
                        xr[4 * v + 3] = t4.w;
                    }
                }
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 1; j <= K; ++j)
                        acc[rr][c] = fmaf(p.k.cx[j - 1], xr[KP + c - j] + xr[KP + c + j], acc[rr][c]);
            }
            // d1 neighbours: a column strip of R + 2K rows shared by the R own rows
            {
                float col[R + 2 * K][4];
                const float* colp = cp + ty0 * SW + KP + 4 * tx;
#pragma unroll
                for (int i = 0; i < R + 2 * K; ++i) {
                    if (i >= K && i < K + R) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) col[i][c] = q[i - K][K][c];
                    } else {
                        const float4 t4 = *reinterpret_cast<const float4*>(colp + i * SW);
                        col[i][0] = t4.x;
                        col[i][1] = t4.y;
                        col[i][2] = t4.z;
                        col[i][3] = t4.w;
                    }
                }
#pragma unroll
                for (int rr = 0; rr < R; ++rr)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 1; j <= K; ++j)
                            acc[rr][c] = fmaf(p.k.cy[j - 1],
                                              col[rr + K - j][c] + col[rr + K + j][c], acc[rr][c]);
            }
            // centre plane fully read: hand its stage back to the producer
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(empty + cs);
            if (++cs == NST) cs = 0;

#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                if (!rin[rr]) continue;
                const float rv[4] = {r4[rr].x, r4[rr].y, r4[rr].z, r4[rr].w};
                const float ov[4] = {o4[rr].x, o4[rr].y, o4[rr].z, o4[rr].w};
                const float dv[4] = {d4[rr].x, d4[rr].y, d4[rr].z, d4[rr].w};
                float un[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float dmp = SEP ? (dxy[rr][c] + dzv) : dv[c];
                    const float qq = dmp * rv[c] * p.k.qscale;
                    const float c1 = __frcp_rn(1.f + qq);
                    const float c2 = (1.f - qq) * c1;
                    const float t = fmaf(rv[c], acc[rr][c], 2.f * q[rr][K][c]);
                    un[c] = fmaf(c1, t, -c2 * ov[c]);
                }
                const long long o = (long long)rr * p.pitch;
                __stcs(reinterpret_cast<float4*>(p.uo + gu + o),
                       make_float4(un[0], un[1], un[2], un[3]));
                if (p.snap)
                    __stcs(reinterpret_cast<float4*>(p.snap + gc + o),
                           make_float4(un[0], un[1], un[2], un[3]));
                if (img) {
                    const float gv[4] = {g4[rr].x, g4[rr].y, g4[rr].z, g4[rr].w};
                    const float sv[4] = {s4[rr].x, s4[rr].y, s4[rr].z, s4[rr].w};
                    float gn[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        gn[c] = fmaf(-sv[c] * p.k.inv_dt2,
                                     (un[c] - 2.f * q[rr][K][c]) + ov[c], gv[c]);
                    __stcs(reinterpret_cast<float4*>(p.grad + gc + o),
                           make_float4(gn[0], gn[1], gn[2], gn[3]));
                }
            }
        }
        // slide the register queue one plane along d0
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int j = 0; j < Q - 1; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) q[rr][j][c] = q[rr][j + 1][c];
        if (++s == NST) {
            s = 0;
            fph ^= 1;
        }
    }
}

}  // namespace sfb
